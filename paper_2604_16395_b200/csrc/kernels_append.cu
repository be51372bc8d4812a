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

__global__ void __launch_bounds__(256) append_kernel(
    const AppendItemDev* __restrict__ items, int32_t n_items, int64_t total_vecs_per_lk,
    const int32_t* __restrict__ ids, const TablePatch* __restrict__ patches, int32_t n_patches,
    int32_t* __restrict__ table, const uint4* __restrict__ k, const uint4* __restrict__ v,
    int64_t kv_rows, uint4* __restrict__ pool, int32_t L, int32_t h_kv, int32_t vec_per_row,
    int32_t kb) {
  const int32_t lk = blockIdx.y;          // layer * 2 + kind
  const int32_t layer = lk >> 1, kind = lk & 1;
  if (lk == 0 && blockIdx.x == 0) {
    for (int32_t i = threadIdx.x; i < n_patches; i += blockDim.x) table[patches[i].idx] = patches[i].value;
  }
  const uint4* src = (kind ? v : k) + (int64_t)layer * kv_rows * h_kv * vec_per_row;
  const int64_t vecs_per_token = (int64_t)h_kv * vec_per_row;
  const int32_t total = (int32_t)total_vecs_per_lk;   // host checks < 2^31
  const int32_t vpt = (int32_t)vecs_per_token;
  for (int32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x) {
    const int32_t row = g / vpt;                      // token row in the concatenated items
    const int32_t rem = g - row * vpt;
    const int32_t head = rem / vec_per_row;
    const int32_t vec = rem - head * vec_per_row;
    // item lookup: last item with row_begin <= row
    int32_t lo = 0, hi = n_items - 1;
    while (lo < hi) {
      int32_t mid = (lo + hi + 1) >> 1;
      if (items[mid].row_begin <= row) lo = mid; else hi = mid - 1;
    }
    const AppendItemDev it = items[lo];
    const int64_t t = (int64_t)row - it.row_begin;
    const int64_t pos = it.nc + t;
    const int32_t blk = ids[it.id_off + (int32_t)(pos / kb - it.nc / kb)];
    const int32_t slot = (int32_t)(pos % kb);
    const uint4 val = src[((it.kv_row + t) * h_kv + head) * vec_per_row + vec];
    const int64_t dst = ((((int64_t)blk * L + layer) * 2 + kind) * h_kv + head) * kb + slot;
    pool[dst * vec_per_row + vec] = val;
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
                          int64_t total_rows, const int32_t* ids, const TablePatch* patches,
                          int32_t n_patches, int32_t* table, const void* k, const void* v,
                          int64_t kv_rows, void* pool, cudaStream_t st) {
  const int32_t vec_per_row = g.d / 8;
  const int64_t total = total_rows * g.h_kv * vec_per_row;
  if (total >= (1ll << 31)) return cudaErrorInvalidValue;
  int64_t want = (total + 255) / 256;
  // enough CTAs to cover the data, capped at 8 waves of 148 SMs x 8 CTAs
  int64_t cap = 148 * 8 * 8;
  int blocks = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  dim3 grid(blocks, g.L * 2);
  append_kernel<<<grid, 256, 0, st>>>(items, n_items, total, ids, patches, n_patches, table,
                                      (const uint4*)k, (const uint4*)v, kv_rows, (uint4*)pool,
                                      g.L, g.h_kv, vec_per_row, g.k);
  return cudaGetLastError();
}

}  // namespace s2l
