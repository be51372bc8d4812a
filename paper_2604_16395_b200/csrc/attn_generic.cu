// CUDA-core paged chunked-prefill attention for geometries the tensor-core kernel does not
// cover (e.g. C1: head_dim 16, block 4).  Same definition as attn_tc.cu (a4):
// query row t of an item sits at position q_pos + t and attends to keys 0..q_pos+t of kv head
// g(h) = h / (h_q / h_kv) (Z2), scale 1/sqrt(d) (Z1), K/V read through the block table.
// One warp per (query row, q head); lanes split head_dim (<= 8 dims per lane); keys are
// walked in order with an online softmax in fp32 (exp2 with log2(e) folded into the scale).
#include "s2l_internal.h"

#include <cuda_bf16.h>
#include <cuda_fp8.h>

namespace s2l {
namespace {

__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }
// pool element e of a bf16 or an FP8 E4M3 pool (kv_dtype 1; exact dequantization)
template <bool kFp8>
__device__ __forceinline__ float kv_at(const void* pool, int64_t e) {
  if constexpr (kFp8) {
    __nv_fp8_e4m3 x;
    x.__x = reinterpret_cast<const __nv_fp8_storage_t*>(pool)[e];
    return float(x);
  } else {
    return bf2f(reinterpret_cast<const __nv_bfloat16*>(pool)[e]);
  }
}

template <bool kFp8>
__global__ void __launch_bounds__(128) attn_generic_kernel(
    const AttnItemDev* __restrict__ items, int32_t n_items, int64_t total_q,
    const int32_t* __restrict__ table, int32_t layer, const __nv_bfloat16* __restrict__ q,
    __nv_bfloat16* __restrict__ o, float* __restrict__ lse,
    const void* __restrict__ pool, int32_t L, int32_t h_q, int32_t h_kv, int32_t d,
    int32_t kb, int32_t max_blocks, float scale_log2) {
  const int32_t lane = threadIdx.x & 31;
  const int64_t wid = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= total_q * h_q) return;
  const int32_t h = (int32_t)(wid % h_q);
  int64_t rank = wid / h_q;  // query row rank across items (items in staged order)
  int32_t i = 0;
  for (; i < n_items; ++i) {
    if (rank < items[i].n_q) break;
    rank -= items[i].n_q;
  }
  const AttnItemDev it = items[i];
  const int64_t t = rank;
  const int64_t row = it.q_row + t;
  const int64_t limit = it.q_pos + t;  // last visible key (inclusive)
  const int32_t g = h / (h_q / h_kv);
  const int32_t per = (d + 31) / 32;   // dims per lane (d <= 256 -> <= 8)
  float qv[8], acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int dim = lane * per + c;
    qv[c] = (c < per && dim < d) ? bf2f(q[(row * h_q + h) * d + dim]) : 0.f;
    acc[c] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  const int32_t* trow = table + (int64_t)it.slot * max_blocks;
  for (int64_t j = 0; j <= limit; ++j) {
    const int32_t blk = trow[j / kb];
    const int32_t slot = (int32_t)(j % kb);
    const int64_t kbase = (((((int64_t)blk * L + layer) * 2 + 0) * h_kv + g) * kb + slot) * d;
    const int64_t vbase = (((((int64_t)blk * L + layer) * 2 + 1) * h_kv + g) * kb + slot) * d;
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int dim = lane * per + c;
      if (c < per && dim < d) s += qv[c] * kv_at<kFp8>(pool, kbase + dim);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    s *= scale_log2;
    const float m_new = fmaxf(m, s);
    const float alpha = exp2f(m - m_new);
    const float p = exp2f(s - m_new);
    l = l * alpha + p;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int dim = lane * per + c;
      const float vv = (c < per && dim < d) ? kv_at<kFp8>(pool, vbase + dim) : 0.f;
      acc[c] = acc[c] * alpha + p * vv;
    }
    m = m_new;
  }
  const float inv = 1.f / l;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int dim = lane * per + c;
    if (c < per && dim < d) o[(row * h_q + h) * d + dim] = __float2bfloat16_rn(acc[c] * inv);
  }
  if (lse && lane == 0) lse[row * h_q + h] = (m + log2f(l)) * 0.69314718055994531f;
}

}  // namespace

cudaError_t launch_attn_generic(const Geometry& g, const AttnItemDev* items, int32_t n_items,
                                int64_t total_q, const int32_t* table, int32_t layer,
                                const void* q, void* o, float* lse, const void* pool,
                                cudaStream_t st) {
  const int64_t warps = total_q * g.h_q;
  const int64_t blocks = (warps + 3) / 4;
  if (blocks <= 0) return cudaSuccess;
  if (blocks > 0x7fffffffll) return cudaErrorInvalidValue;
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)g.d);
  if (g.fp8)
    attn_generic_kernel<true><<<(unsigned)blocks, 128, 0, st>>>(
        items, n_items, total_q, table, layer, (const __nv_bfloat16*)q, (__nv_bfloat16*)o, lse,
        pool, g.L, g.h_q, g.h_kv, g.d, g.k, g.max_blocks, scale_log2);
  else
    attn_generic_kernel<false><<<(unsigned)blocks, 128, 0, st>>>(
        items, n_items, total_q, table, layer, (const __nv_bfloat16*)q, (__nv_bfloat16*)o, lse,
        pool, g.L, g.h_q, g.h_kv, g.d, g.k, g.max_blocks, scale_log2);
  return cudaGetLastError();
}

}  // namespace s2l
