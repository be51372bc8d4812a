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

namespace s2l {
namespace {

__global__ void table_patch_kernel(const TablePatch* __restrict__ patches, int32_t n,
                                   int32_t* __restrict__ table) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    table[patches[i].idx] = patches[i].value;
}

constexpr int kVecPerThread = 8;   // 8 x 16-byte loads in flight per thread, then 8 stores
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

// One thread moves kVecPerThread 16-byte vectors of the concatenated [rows][h_kv][d] input of
// one (layer, K|V) (blockIdx.y) to their (block, slot) in the pool.  The item descriptors and
// the block ids are staged in shared memory first, so the only global load on each vector's
// critical path is the data itself.
__global__ void __launch_bounds__(256) append_kernel(
    const AppendItemDev* __restrict__ items_g, int32_t n_items, int64_t total_vecs_per_lk,
    const int32_t* __restrict__ ids_g, int32_t n_ids, const TablePatch* __restrict__ patches,
    int32_t n_patches, int32_t* __restrict__ table, const uint4* __restrict__ k,
    const uint4* __restrict__ v, int64_t kv_rows, uint4* __restrict__ pool, int32_t L,
    int32_t h_kv, int32_t vec_per_row, int32_t kb_log2, int32_t vpt_log2) {
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
  const int32_t lk = blockIdx.y;          // layer * 2 + kind
  const int32_t layer = lk >> 1, kind = lk & 1;
  if (lk == 0 && blockIdx.x == 0) {
    for (int32_t i = threadIdx.x; i < n_patches; i += blockDim.x) table[patches[i].idx] = patches[i].value;
  }
  const uint4* src = (kind ? v : k) + (int64_t)layer * kv_rows * h_kv * vec_per_row;
  const int32_t vpt = h_kv * vec_per_row;                   // vectors per token row
  const int32_t total = (int32_t)total_vecs_per_lk;        // host checks < 2^31
  const int32_t kb = 1 << kb_log2;
  const int32_t stride = gridDim.x * blockDim.x;
  for (int32_t g0 = blockIdx.x * blockDim.x + threadIdx.x; g0 < total; g0 += stride * kVecPerThread) {
    uint4 val[kVecPerThread];
    int64_t dst[kVecPerThread];
#pragma unroll
    for (int u = 0; u < kVecPerThread; ++u) {
      const int32_t g = g0 + u * stride;
      dst[u] = -1;
      if (g < total) {
        const int32_t row = vpt_log2 >= 0 ? (g >> vpt_log2) : g / vpt;   // token row
        const int32_t rem = g - row * vpt;
        const int32_t head = rem / vec_per_row;
        const int32_t vec = rem - head * vec_per_row;
        const AppendItemDev& it = items[find_item(items, n_items, row)];
        const int64_t t = (int64_t)row - it.row_begin;
        const int64_t pos = it.nc + t;
        const int32_t blk = ids[it.id_off + (int32_t)((pos >> kb_log2) - (it.nc >> kb_log2))];
        const int32_t slot = (int32_t)(pos & (kb - 1));
        val[u] = src[((it.kv_row + t) * h_kv + head) * vec_per_row + vec];
        dst[u] = (((((int64_t)blk * L + layer) * 2 + kind) * h_kv + head) * kb + slot) * vec_per_row + vec;
      }
    }
#pragma unroll
    for (int u = 0; u < kVecPerThread; ++u)
      if (dst[u] >= 0) pool[dst[u]] = val[u];
  }
}

}  // namespace

cudaError_t launch_table_patch(const TablePatch* patches, int32_t n, int32_t* table,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int blocks = (n + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  table_patch_kernel<<<blocks, 256, 0, st>>>(patches, n, table);
  return cudaGetLastError();
}

cudaError_t launch_append(const Geometry& g, const AppendItemDev* items, int32_t n_items,
                          int64_t total_rows, const int32_t* ids, int32_t n_ids,
                          const TablePatch* patches,
                          int32_t n_patches, int32_t* table, const void* k, const void* v,
                          int64_t kv_rows, void* pool, cudaStream_t st) {
  const int32_t vec_per_row = g.d / 8;
  const int64_t total = total_rows * g.h_kv * vec_per_row;
  if (total >= (1ll << 31)) return cudaErrorInvalidValue;
  int kb_log2 = 0;
  while ((1 << kb_log2) < g.k) ++kb_log2;
  const int32_t vpt = g.h_kv * vec_per_row;
  int vpt_log2 = -1;
  if ((vpt & (vpt - 1)) == 0) {
    vpt_log2 = 0;
    while ((1 << vpt_log2) < vpt) ++vpt_log2;
  }
  // one pass: each thread moves kVecPerThread vectors; at most one wave of resident CTAs
  int64_t threads = (total + kVecPerThread - 1) / kVecPerThread;
  int64_t blocks = (threads + 255) / 256;
  const int64_t wave = 148 * 4;                 // 4 x 256-thread CTAs resident per SM (64 regs)
  const int64_t per_lk = blocks;
  if (blocks * g.L * 2 > wave && per_lk > 1) {
    blocks = (wave + g.L * 2 - 1) / (g.L * 2);
    if (blocks < 1) blocks = 1;
  }
  if (blocks < 1) blocks = 1;
  if (blocks > 65535) blocks = 65535;
  dim3 grid((unsigned)blocks, g.L * 2);
  append_kernel<<<grid, 256, 0, st>>>(items, n_items, total, ids, n_ids, patches, n_patches, table,
                                      (const uint4*)k, (const uint4*)v, kv_rows, (uint4*)pool,
                                      g.L, g.h_kv, vec_per_row, kb_log2, vpt_log2);
  return cudaGetLastError();
}

}  // namespace s2l
