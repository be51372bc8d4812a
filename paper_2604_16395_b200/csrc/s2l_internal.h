// Internal declarations shared by the host runtime and the kernels of libs2l.
// Product code only — nothing here is shared with oracle/ (see DESIGN.md §Boundary).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifndef S2L_HEAD_MAJOR
#define S2L_HEAD_MAJOR 1   // v2 unit order inside an item: 0 = pair-major, 1 = kv-head-major
#endif
// Programmatic dependent launch between the library's consecutive kernels on the compute
// stream (append -> attention -> append ...): a kernel launched with it may be scheduled while
// its predecessor drains; it executes griddepcontrol.wait (predecessor complete, its writes
// visible) before touching global memory, so only the launch latency overlaps.  Off: measured
// 0.5-1.7 % slower on the C2 step (profiles/r01/pdl_ab.txt), the gaps it hides are ~3 us.
#ifndef S2L_PDL
#define S2L_PDL 0
#endif

#include <utility>

namespace s2l {

#ifdef __CUDACC__
// Kernel prologue of a PDL-launched kernel: wait for the predecessor grid, then allow the
// successor grid to be scheduled (it waits for this one in turn).
__device__ __forceinline__ void pdl_prologue() {
#if S2L_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
// Launch with the programmatic-stream-serialization attribute (S2L_PDL) or plainly.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = S2L_PDL ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
#endif

// ---- device-side descriptors written into the staging ring by the host -------------------

// One item of an append launch.  Positions [nc, nc+n_kv) of the request are written; the
// block ids covering them are ids[id_off .. id_off + n_ids) (first one = block nc/k).
struct AppendItemDev {
  int64_t nc;        // num_computed before the append
  int64_t n_kv;
  int64_t kv_row;    // first row in the caller's k/v
  int64_t row_begin; // prefix sum of n_kv over items (thread -> item lookup)
  int32_t id_off;
  int32_t pad;
};

// One entry of the device block-table patch list: table[idx] = value.
struct TablePatch {
  int32_t idx;
  int32_t value;
};

// One item of an attention launch (items sorted by descending kv length on the host).
struct AttnItemDev {
  int64_t q_pos;
  int64_t q_row;
  int32_t n_q;
  int32_t slot;        // row of the device block table
  int32_t tiles;       // 128-row (token x head-in-group) Q tiles of this item
  int32_t unit_begin;  // prefix sum of tiles * h_kv over items
};

// Descriptors of small calls travel inside the kernel's parameter block (read through the
// constant bank) instead of the staging ring: a staged upload is a cudaMemcpyAsync that queues
// on the copy engine behind bulk H2D traffic (inputs, swap-ins) and would stall the compute
// stream behind it.  Larger calls fall back to the staging ring.
constexpr int kInlineBytes = 6144;      // append: items + block ids + table patches
struct InlineBlob {
  alignas(16) uint8_t b[kInlineBytes];
};
constexpr int kInlineAttnItems = 64;    // attention: items inline up to this many
constexpr int kInlinePatches = 512;     // table-patch kernel
struct InlinePatches {
  TablePatch p[kInlinePatches];
};

struct Geometry {
  int32_t L, h_q, h_kv, d, k;
  int32_t max_blocks;  // columns of the device block table
  bool fp8 = false;    // K/V stored as FP8 E4M3 (s2l_config.kv_dtype = 1): 1 byte per value
};

// ---- kernel launchers (kernels_*.cu) ----------------------------------------------------

cudaError_t launch_table_patch(const TablePatch* patches, int32_t n, int32_t* table,
                               cudaStream_t st);
// Same with the patches (n <= kInlinePatches) passed by value from host memory.
cudaError_t launch_table_patch_inline(const TablePatch* host_patches, int32_t n, int32_t* table,
                                      cudaStream_t st);

// Writes K/V rows into the pool and applies the table patches (fused).  k / v hold layers
// layer0 .. layer0+nl-1 ([nl][kv_rows][h_kv][d]); nl = 0 means all L layers from layer 0.
cudaError_t launch_append(const Geometry& g, const AppendItemDev* items, int32_t n_items,
                          int64_t total_rows, const int32_t* ids, int32_t n_ids,
                          const TablePatch* patches,
                          int32_t n_patches, int32_t* table, const void* k, const void* v,
                          int64_t kv_rows, void* pool, cudaStream_t st, int32_t layer0 = 0,
                          int32_t nl = 0);
// Same with items / ids / patches laid out in a host blob (items at 0, ids at off_ids,
// patches at off_patch; total <= kInlineBytes) passed by value.
cudaError_t launch_append_inline(const Geometry& g, const InlineBlob& blob, int32_t n_items,
                                 int64_t total_rows, int32_t off_ids, int32_t n_ids,
                                 int32_t off_patch, int32_t n_patches, int32_t* table,
                                 const void* k, const void* v, int64_t kv_rows, void* pool,
                                 cudaStream_t st, int32_t layer0 = 0, int32_t nl = 0);

// Swap staging (a5 / a6 with scattered GPU ids): copies GPU blocks ids[0..n) of the pool
// into consecutive block slots of `stage` (to_stage) or back (scatter), on stream st.
constexpr int kSwapIdsPerLaunch = 1024;
cudaError_t launch_swap_stage(const int32_t* host_ids, int32_t n, void* pool, void* stage, int64_t block_bytes,
                              bool to_stage, cudaStream_t st);

// CUDA-core attention for any geometry (one warp per (query row, q head)).
cudaError_t launch_attn_generic(const Geometry& g, const AttnItemDev* items, int32_t n_items,
                                int64_t total_q, const int32_t* table, int32_t layer,
                                const void* q, void* o, float* lse, const void* pool,
                                cudaStream_t st);

// tcgen05 / TMEM / TMA attention (head_dim 128, 16 <= k <= 128, 128 % (h_q/h_kv) == 0).
// tmap_q points to one host CUtensorMap (128 bytes), tmap_kv to the two pool maps (256 bytes).
// One work unit (CTA) = one (item, kv head, pair of 128-row Q tiles).
bool attn_tc_supported(const Geometry& g);
constexpr int kMaxDevices = 64;
// Grid = split_begin + (total_units - split_begin) * split_s CTAs: units below split_begin
// run whole, the remaining (tail-wave) units run as split_s KV-range pieces whose partials
// (ws: O partials of max_pieces pieces, then their (m, l)) are merged by the last piece (ws_cnt).
// items: device pointer, or (n_items <= kInlineAttnItems and items_host != nullptr) the host
// array is copied into the kernel's parameters instead.
cudaError_t launch_attn_tc(const Geometry& g, const AttnItemDev* items, const AttnItemDev* items_host,
                           int32_t n_items,
                           int32_t total_units, int32_t split_begin, int32_t split_s,
                           float* ws, int32_t max_pieces, int32_t* ws_cnt,
                           const int32_t* table, int32_t layer, const void* tmap_q,
                           const void* tmap_kv, const void* tmap_o, void* o, float* lse,
                           int32_t flags, cudaStream_t st, const void* tmap_in = nullptr,
                           void* pool = nullptr, uint64_t fuse_mask = ~0ull);
// fuse_mask (kAttnFuseAppend, items inline): bit i set = item i (in the items array's order)
// has its append fused; the others were appended before the launch and read from the pool.
// flags of launch_attn_tc
// Fused append (NEXT-2).  For every item selected by fuse_mask (q_pos a multiple of
// the block size) the chunk rows [q_pos, q_pos+n_q) of this layer are read from tmap_in
// (make_tmap_in) and written to the pool by the kernel.  No two items may share a request.
constexpr int32_t kAttnFuseAppend = 8;
constexpr int32_t kAttnNoDirectMerge = 16;   // tests: split pieces always merge through the workspace
// Experiments: device buffer receiving kernel timeline stamps (S2L_TRACE builds); nullptr = off.
void set_attn_trace(uint32_t* buf);
constexpr int64_t kSplitPieceFloats = 2 * 128 * 130;   // O [2][128][128] + (m, l) [2][128][2]
// TMA descriptors (host).  Returns false on failure (message in *err).
bool make_tmap_q(void* out128, const void* q, int64_t q_rows, int32_t h_q, int32_t d,
                 int32_t group, const char** err);
// One layer's K and V input rows ([rows][h_kv][d] bf16) into out512: per-block boxes (K at 0,
// V at 128) and whole-tile boxes (K at 256, V at 384).
bool make_tmap_in(void* out512, const void* k, const void* v, int64_t rows, int32_t h_kv,
                  int32_t d, int32_t kb, const char** err);
// Maps of the pool into out256: [0,128) per-block boxes, [128,256) 128-key block runs.
bool make_tmap_kv(void* out256, const void* pool, int64_t num_blocks, int32_t L, int32_t h_kv,
                  int32_t d, int32_t k, bool fp8, const char** err);

}  // namespace s2l
