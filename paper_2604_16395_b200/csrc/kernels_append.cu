// Paged KV append (a3) and device block-table patching.
//
// a3, P:L59 / P:L67: the K/V rows of positions [nc, nc+n_kv) of each request are stored in
// block table[pos / k] at slot pos % k of every layer.  Pool layout (include/s2l.h):
//   pool[block][layer][2][kv_head][slot][d]  bf16.
// One thread moves one 16-byte vector (8 bf16).  Consecutive threads walk d, then kv heads,
// then tokens, so reads of the caller's [L][rows][h_kv][d] rows are fully coalesced and each
// written row (d*2 bytes) is one contiguous run.  blockIdx.y = layer*2 + (0:K, 1:V).
// The block ids come from the staged id list (not the table), so the same launch can also
// apply the table patches without a read/write race.
#include "s2l_internal.h"

#include <cuda_bf16.h>

#include <cstring>

namespace s2l {
namespace {

__global__ void table_patch_kernel(const TablePatch* __restrict__ patches, int32_t n,
                                   int32_t* __restrict__ table) {
  pdl_prologue();
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    table[patches[i].idx] = patches[i].value;
}
__global__ void table_patch_inline_kernel(const __grid_constant__ InlinePatches ps, int32_t n,
                                          int32_t* __restrict__ table) {
  pdl_prologue();
  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) table[ps.p[i].idx] = ps.p[i].value;
}

constexpr int kSmemItems = 256;    // items / ids staged in shared memory when they fit (38 KB)
constexpr int kSmemIds = 6144;

__device__ __forceinline__ int32_t find_item(const AppendItemDev* items, int32_t n, int64_t row) {
  int32_t lo = 0, hi = n - 1;     // last item with row_begin <= row
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (items[mid].row_begin <= row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// One warp moves whole token rows: for each of its kRowsPerWarp rows it looks the item up once
// (items and block ids are staged in shared memory), then each lane loads its 16-byte vectors
// of the row ([h_kv][d] contiguous, so the warp reads the row coalesced) and stores them to
// (block, slot) of every kv head (each head's d*2 bytes contiguous in the pool).  All loads of
// a warp are issued before its stores.  blockIdx.y = layer * 2 + (0: K, 1: V).
#ifndef S2L_APPEND_ROWS
#define S2L_APPEND_ROWS 4
#endif
constexpr int kRowsPerWarp = S2L_APPEND_ROWS;
// Wide token rows (more than 4 16-byte vectors per lane, h_kv * d > 1024) go one row per warp,
// their vectors in chunks of 16 per lane, so the values in flight stay within registers.
template <int kMaxVecPerLane> constexpr int kRowsFor = kMaxVecPerLane <= 4 ? kRowsPerWarp : 1;
template <int kMaxVecPerLane> constexpr int kChunkFor = kMaxVecPerLane < 16 ? kMaxVecPerLane : 16;

// 8 bf16 -> 8 E4M3 codes (FP8 KV cache, kv_dtype 1): round to nearest even, saturating to
// +-448 (reading Z20; the same rule as oracle/fp8.py); low element in the low byte.
__device__ __forceinline__ uint2 bf16x8_to_e4m3x8(uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t o[2] = {0, 0};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xffff0000u);
    uint16_t c;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(c) : "f"(hi), "f"(lo));
    o[i >> 1] |= (uint32_t)c << (16 * (i & 1));
  }
  return make_uint2(o[0], o[1]);
}

// kMaxVecPerLane >= vectors per lane per row (vpt/32: 4 at Llama-3 h_kv 8, d 128).
// kVpr = d/8 vectors per head row when known at compile time (16 at d = 128), else 0.
// Descriptors either through device pointers (staging ring) or, when blob_mode != 0, from
// the kernel's by-value parameter blob (items at 0, ids at off_ids, patches at off_patch).
// kFp8: the pool holds E4M3 codes (1 byte per value): vector index i of 8 values is the uint2
// at i (instead of the uint4 at i).
template <int kMaxVecPerLane, int kVpr, bool kFp8>
__global__ void __launch_bounds__(256) append_kernel(
    const AppendItemDev* __restrict__ items_p, int32_t n_items, int64_t total_rows,
    const int32_t* __restrict__ ids_p, int32_t n_ids, const TablePatch* __restrict__ patches_p,
    int32_t n_patches, int32_t* __restrict__ table, const uint4* __restrict__ k,
    const uint4* __restrict__ v, int64_t kv_rows, uint4* __restrict__ pool, int32_t L,
    int32_t h_kv, int32_t vec_per_row, int32_t kb_log2, const __grid_constant__ InlineBlob blob,
    int32_t blob_mode, int32_t off_ids, int32_t off_patch, int32_t layer0) {
  pdl_prologue();
  const AppendItemDev* items_g = blob_mode ? reinterpret_cast<const AppendItemDev*>(blob.b) : items_p;
  const int32_t* ids_g = blob_mode ? reinterpret_cast<const int32_t*>(blob.b + off_ids) : ids_p;
  const TablePatch* patches = blob_mode ? reinterpret_cast<const TablePatch*>(blob.b + off_patch) : patches_p;
  __shared__ AppendItemDev s_items[kSmemItems];
  __shared__ int32_t s_ids[kSmemIds];
  const bool staged = n_items <= kSmemItems && n_ids <= kSmemIds;
  if (staged) {
    for (int32_t i = threadIdx.x; i < n_items; i += blockDim.x) s_items[i] = items_g[i];
    for (int32_t i = threadIdx.x; i < n_ids; i += blockDim.x) s_ids[i] = ids_g[i];
    __syncthreads();
  }
  const AppendItemDev* items = staged ? s_items : items_g;
  const int32_t* ids = staged ? s_ids : ids_g;
  const int32_t lk = blockIdx.y;
  const int32_t layer = layer0 + (lk >> 1), kind = lk & 1;   // k/v hold layers layer0 ..

  if (lk == 0 && blockIdx.x == 0) {
    for (int32_t i = threadIdx.x; i < n_patches; i += blockDim.x) table[patches[i].idx] = patches[i].value;
  }
  const int32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint4* src = (kind ? v : k) + (int64_t)(lk >> 1) * kv_rows * h_kv * vec_per_row;
  const int32_t vpt = h_kv * vec_per_row;                 // vectors per token row
  const int32_t kb = 1 << kb_log2;
  if constexpr (kMaxVecPerLane <= 4) {
    // narrow rows (the measured configurations): each row's loads right after its lookup
    const int64_t row0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * kRowsPerWarp;
    const int64_t stride_rows = (int64_t)gridDim.x * (blockDim.x >> 5) * kRowsPerWarp;
    for (int64_t rb = row0; rb < total_rows; rb += stride_rows) {
      uint4 val[kRowsPerWarp][kMaxVecPerLane];
      int64_t dst_row[kRowsPerWarp];        // pool vector index of (block, layer, kind, head 0, slot)
      int64_t src_row[kRowsPerWarp];
  #pragma unroll
      for (int rr = 0; rr < kRowsPerWarp; ++rr) {
        const int64_t row = rb + rr;
        dst_row[rr] = -1;
        if (row < total_rows) {
          const AppendItemDev& it = items[find_item(items, n_items, row)];
          const int64_t t = row - it.row_begin;
          const int64_t pos = it.nc + t;
          const int32_t blk = ids[it.id_off + (int32_t)((pos >> kb_log2) - (it.nc >> kb_log2))];
          const int32_t slot = (int32_t)(pos & (kb - 1));
          src_row[rr] = (it.kv_row + t) * vpt;
          dst_row[rr] = ((((int64_t)blk * L + layer) * 2 + kind) * h_kv * kb + slot) * vec_per_row;
  #pragma unroll
          for (int u = 0; u < kMaxVecPerLane; ++u) {
            const int32_t gi = lane + 32 * u;
            if (gi < vpt) val[rr][u] = src[src_row[rr] + gi];
          }
        }
      }
  #pragma unroll
      for (int rr = 0; rr < kRowsPerWarp; ++rr) {
        if (dst_row[rr] < 0) continue;
  #pragma unroll
        for (int u = 0; u < kMaxVecPerLane; ++u) {
          const int32_t gi = lane + 32 * u;
          if (gi < vpt) {
            const int32_t vpr = kVpr ? kVpr : vec_per_row;
            const int32_t head = gi / vpr, vec = gi - head * vpr;
            const int64_t di = dst_row[rr] + (int64_t)head * kb * vpr + vec;
            if constexpr (kFp8) reinterpret_cast<uint2*>(pool)[di] = bf16x8_to_e4m3x8(val[rr][u]);
            else pool[di] = val[rr][u];
          }
        }
      }
    }
  } else {
    constexpr int kRows = kRowsFor<kMaxVecPerLane>, kChunk = kChunkFor<kMaxVecPerLane>;
    const int64_t row0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * kRows;
    const int64_t stride_rows = (int64_t)gridDim.x * (blockDim.x >> 5) * kRows;
    for (int64_t rb = row0; rb < total_rows; rb += stride_rows) {
      int64_t dst_row[kRows];               // pool vector index of (block, layer, kind, head 0, slot)
      int64_t src_row[kRows];
  #pragma unroll
      for (int rr = 0; rr < kRows; ++rr) {
        const int64_t row = rb + rr;
        dst_row[rr] = -1;
        if (row < total_rows) {
          const AppendItemDev& it = items[find_item(items, n_items, row)];
          const int64_t t = row - it.row_begin;
          const int64_t pos = it.nc + t;
          const int32_t blk = ids[it.id_off + (int32_t)((pos >> kb_log2) - (it.nc >> kb_log2))];
          const int32_t slot = (int32_t)(pos & (kb - 1));
          src_row[rr] = (it.kv_row + t) * vpt;
          dst_row[rr] = ((((int64_t)blk * L + layer) * 2 + kind) * h_kv * kb + slot) * vec_per_row;
        }
      }
  #pragma unroll
      for (int c0 = 0; c0 < kMaxVecPerLane; c0 += kChunk) {
        uint4 val[kRows][kChunk];
  #pragma unroll
        for (int rr = 0; rr < kRows; ++rr) {
          if (dst_row[rr] < 0) continue;
  #pragma unroll
          for (int u = 0; u < kChunk; ++u) {
            const int32_t gi = lane + 32 * (c0 + u);
            if (gi < vpt) val[rr][u] = src[src_row[rr] + gi];
          }
        }
  #pragma unroll
        for (int rr = 0; rr < kRows; ++rr) {
          if (dst_row[rr] < 0) continue;
  #pragma unroll
          for (int u = 0; u < kChunk; ++u) {
            const int32_t gi = lane + 32 * (c0 + u);
            if (gi < vpt) {
              const int32_t vpr = kVpr ? kVpr : vec_per_row;
              const int32_t head = gi / vpr, vec = gi - head * vpr;
              const int64_t di = dst_row[rr] + (int64_t)head * kb * vpr + vec;
              if constexpr (kFp8) reinterpret_cast<uint2*>(pool)[di] = bf16x8_to_e4m3x8(val[rr][u]);
              else pool[di] = val[rr][u];
            }
          }
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_table_patch_inline(const TablePatch* host_patches, int32_t n, int32_t* table,
                                      cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > kInlinePatches) return cudaErrorInvalidValue;
  InlinePatches ps;
  memcpy(ps.p, host_patches, (size_t)n * sizeof(TablePatch));
  return launch_k(table_patch_inline_kernel, dim3(1), dim3(256), 0, st, ps, n, table);
}

cudaError_t launch_table_patch(const TablePatch* patches, int32_t n, int32_t* table,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int blocks = (n + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  return launch_k(table_patch_kernel, dim3(blocks), dim3(256), 0, st, patches, n, table);
}

namespace {
cudaError_t launch_append_impl(const Geometry& g, const AppendItemDev* items, int32_t n_items,
                               int64_t total_rows, const int32_t* ids, int32_t n_ids,
                               const TablePatch* patches, int32_t n_patches, int32_t* table,
                               const void* k, const void* v, int64_t kv_rows, void* pool,
                               const InlineBlob& blob, int32_t blob_mode, int32_t off_ids,
                               int32_t off_patch, cudaStream_t st, int32_t layer0, int32_t nl) {
  const int32_t vec_per_row = g.d / 8;
  const int64_t vpt = (int64_t)g.h_kv * vec_per_row;
  int kb_log2 = 0;
  while ((1 << kb_log2) < g.k) ++kb_log2;
  const int32_t rows_per_warp = vpt <= 128 ? kRowsPerWarp : 1;   // kRowsFor of the dispatched MAXV
  const int64_t warps = (total_rows + rows_per_warp - 1) / rows_per_warp;
  int64_t blocks = (warps + 7) / 8;                  // 8 warps per CTA
  if (blocks < 1) blocks = 1;
  if (blocks > 65535) blocks = 65535;
  if (nl <= 0) nl = g.L;
  dim3 grid((unsigned)blocks, nl * 2);
#define S2L_APPEND(MAXV, VPR)                                                                     \
  e = g.fp8 ? launch_k(append_kernel<MAXV, VPR, true>, grid, dim3(256), 0, st, items, n_items, total_rows, ids, \
               n_ids, patches, n_patches, table, (const uint4*)k, (const uint4*)v, kv_rows,         \
               (uint4*)pool, g.L, g.h_kv, vec_per_row, kb_log2, blob, blob_mode, off_ids, off_patch, \
               layer0)                                                                               \
            : launch_k(append_kernel<MAXV, VPR, false>, grid, dim3(256), 0, st, items, n_items, total_rows, ids,   \
               n_ids, patches, n_patches, table, (const uint4*)k, (const uint4*)v, kv_rows,         \
               (uint4*)pool, g.L, g.h_kv, vec_per_row, kb_log2, blob, blob_mode, off_ids, off_patch, \
               layer0)
  cudaError_t e = cudaSuccess;
  if (vec_per_row == 16 && vpt <= 128) S2L_APPEND(4, 16);          // d = 128, h_kv <= 8
  else if (vec_per_row == 16 && vpt <= 512) S2L_APPEND(16, 16);
  else if (vpt <= 32) S2L_APPEND(1, 0);
  else if (vpt <= 128) S2L_APPEND(4, 0);
  else if (vpt <= 512) S2L_APPEND(16, 0);
  else if (vpt <= 2048) S2L_APPEND(64, 0);
  else return cudaErrorInvalidValue;
#undef S2L_APPEND
  return e;
}
}  // namespace

cudaError_t launch_append(const Geometry& g, const AppendItemDev* items, int32_t n_items,
                          int64_t total_rows, const int32_t* ids, int32_t n_ids,
                          const TablePatch* patches,
                          int32_t n_patches, int32_t* table, const void* k, const void* v,
                          int64_t kv_rows, void* pool, cudaStream_t st, int32_t layer0, int32_t nl) {
  static InlineBlob empty;   // unused in pointer mode (still copied as a parameter)
  return launch_append_impl(g, items, n_items, total_rows, ids, n_ids, patches, n_patches, table,
                            k, v, kv_rows, pool, empty, 0, 0, 0, st, layer0, nl);
}

cudaError_t launch_append_inline(const Geometry& g, const InlineBlob& blob, int32_t n_items,
                                 int64_t total_rows, int32_t off_ids, int32_t n_ids,
                                 int32_t off_patch, int32_t n_patches, int32_t* table,
                                 const void* k, const void* v, int64_t kv_rows, void* pool,
                                 cudaStream_t st, int32_t layer0, int32_t nl) {
  return launch_append_impl(g, nullptr, n_items, total_rows, nullptr, n_ids, nullptr, n_patches,
                            table, k, v, kv_rows, pool, blob, 1, off_ids, off_patch, st, layer0, nl);
}

}  // namespace s2l

// ---- swap gather / scatter (a5 / a6 with scattered GPU block ids) --------------------------
// The copy engines move each contiguous run of blocks as one DMA; when the GPU ids of a swap
// are scattered (short runs), the runs are staged: swap-out gathers the blocks of a CPU-id run
// into a contiguous device staging buffer (HBM -> HBM) and moves it with one D2H; swap-in
// moves a CPU run into staging with one H2D and scatters it to its GPU blocks.  One CTA moves
// one block (16-byte vectors); block ids travel by value (<= kSwapIdsPerLaunch per launch).
namespace s2l {
namespace {
struct SwapIds {
  int32_t id[kSwapIdsPerLaunch];
};
__global__ void __launch_bounds__(256) swap_stage_kernel(const __grid_constant__ SwapIds ids, int32_t n,
                                                          uint4* __restrict__ pool, uint4* __restrict__ stage,
                                                          int64_t vec_per_block, int32_t to_stage) {
  pdl_prologue();
  for (int32_t b = blockIdx.x; b < n; b += gridDim.x) {
    uint4* g = pool + (int64_t)ids.id[b] * vec_per_block;
    uint4* s = stage + (int64_t)b * vec_per_block;
    if (to_stage) {
      for (int64_t i = threadIdx.x; i < vec_per_block; i += blockDim.x) s[i] = __ldcs(g + i);
    } else {
      for (int64_t i = threadIdx.x; i < vec_per_block; i += blockDim.x) g[i] = s[i];
    }
  }
}
}  // namespace

cudaError_t launch_swap_stage(const int32_t* host_ids, int32_t n, void* pool, void* stage, int64_t block_bytes,
                              bool to_stage, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n > kSwapIdsPerLaunch || block_bytes % 16) return cudaErrorInvalidValue;
  SwapIds ids;
  memcpy(ids.id, host_ids, (size_t)n * sizeof(int32_t));
  return launch_k(swap_stage_kernel, dim3(n), dim3(256), 0, st, ids, n, (uint4*)pool, (uint4*)stage,
                  block_bytes / 16, to_stage ? 1 : 0);
}
}  // namespace s2l
