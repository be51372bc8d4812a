// Microbenchmark: instruction-schedule variants of the attention softmax's exp phase for one
// 128-column row per thread (scale FFMA2, 2^x on MUFU or the FMA-pipe polynomial, FADD2 row
// sum, bf16 pack), 1 or 2 warps per SMSP.  Reports cycles per 128-column tile per warp.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/softmax_bench2.cu -o /tmp/sb2
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pack(float lo, float hi) { uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ float2 poly2(float2 x) {
  x.x = fmaxf(x.x, -127.f); x.y = fmaxf(x.y, -127.f);
  const float2 y = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 t = __fadd2_rn(y, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-t.x, -t.y));
  float2 q = __ffma2_rn(f, make_float2(0.0551704f, 0.0551704f), make_float2(0.24260826f, 0.24260826f));
  q = __ffma2_rn(q, f, make_float2(0.69326098f, 0.69326098f));
  q = __ffma2_rn(q, f, make_float2(0.99992833f, 0.99992833f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(y.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(y.y) << 23)));
}
// poly choice for pair c (0..63): MODE 0 contiguous (c&7)<P, MODE 1 spread (c % (8/P) == 0 for P in {1,2,4})
template <int P, int MODE>
__device__ __forceinline__ bool is_poly(int c) {
  if (P == 0) return false;
  if (MODE == 0) return (c & 7) < P;
  return (c % (8 / P)) == 0;
}

// CH = pairs per phase group (16: current 32-col chunks; 32: 64-col chunks; 64: whole row)
template <int CH, int P, int MODE>
__device__ __forceinline__ float tile(const float (&s)[128], float2 sc, float2 nm, uint32_t& sink) {
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int g = 0; g < 64; g += CH) {
    float2 x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __ffma2_rn(make_float2(s[2 * (g + c)], s[2 * (g + c) + 1]), sc, nm);
#pragma unroll
    for (int c = 0; c < CH; ++c)
      x[c] = is_poly<P, MODE>(g + c) ? poly2(x[c]) : make_float2(ex2(x[c].x), ex2(x[c].y));
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      acc[c & 3] = __fadd2_rn(acc[c & 3], x[c]);
      sink ^= pack(x[c].x, x[c].y);
    }
  }
  const float2 a = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
  return a.x + a.y;
}

// software-pipelined: scale of group g+1 issued with the exps of group g
template <int CH, int P, int MODE>
__device__ __forceinline__ float tile_sw(const float (&s)[128], float2 sc, float2 nm, uint32_t& sink) {
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  float2 x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = __ffma2_rn(make_float2(s[2 * c], s[2 * c + 1]), sc, nm);
#pragma unroll
  for (int g = 0; g < 64; g += CH) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (g + CH < 64) y[c] = __ffma2_rn(make_float2(s[2 * (g + CH + c)], s[2 * (g + CH + c) + 1]), sc, nm);
      x[c] = is_poly<P, MODE>(g + c) ? poly2(x[c]) : make_float2(ex2(x[c].x), ex2(x[c].y));
      acc[c & 3] = __fadd2_rn(acc[c & 3], x[c]);
      sink ^= pack(x[c].x, x[c].y);
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = y[c];
  }
  const float2 a = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
  return a.x + a.y;
}

// pure MUFU.EX2 throughput: 128 independent ex2 per thread per iteration
__global__ void mufu_only(const float* __restrict__ in, uint32_t* out, int iters, long long* cycles) {
  float s[128];
#pragma unroll
  for (int c = 0; c < 128; ++c) s[c] = in[(threadIdx.x * 7 + c) & 1023];
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 128; ++c) s[c] = ex2(s[c]);
  }
  long long t1 = clock64();
#pragma unroll
  for (int c = 0; c < 128; ++c) acc += s[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(acc);
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = (t1 - t0) / iters;
}

template <int V, int CH, int P, int MODE>
__global__ void k(const float* __restrict__ in, uint32_t* out, int iters, long long* cycles) {
  float s[128];
#pragma unroll
  for (int c = 0; c < 128; ++c) s[c] = in[(threadIdx.x * 7 + c) & 1023];
  uint32_t sink = 0;
  float l = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float2 sc = make_float2(0.18f, 0.18f), nm = make_float2(-1.f, -1.f);
    l += V == 0 ? tile<CH, P, MODE>(s, sc, nm, sink) : tile_sw<CH, P, MODE>(s, sc, nm, sink);
    s[it & 127] += 1e-3f;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink ^ __float_as_uint(l);
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = (t1 - t0) / iters;
}

template <int V, int CH, int P, int MODE>
void run(const char* name, float* in, uint32_t* out, long long* cyc) {
  for (int w = 1; w <= 2; ++w) {
    k<V, CH, P, MODE><<<148, 128 * w>>>(in, out, 200, cyc);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s poly %d/8 %s  %d warp(s)/SMSP: %5lld cycles per tile per warp\n", name, P, MODE ? "spread" : "contig", w, h);
  }
}

int main() {
  float* in; cudaMalloc(&in, 4096); cudaMemset(in, 0, 4096);
  uint32_t* out; cudaMalloc(&out, 148 * 256 * 4);
  long long* cyc; cudaMalloc(&cyc, 8);
  for (int w = 1; w <= 2; ++w) {
    mufu_only<<<148, 128 * w>>>(in, out, 200, cyc);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %d warp(s)/SMSP: %5lld cycles per 128 ex2 per warp\n", "MUFU.EX2 only", w, h);
  }
  run<0, 32, 1, 1>("phases of 32 pairs (kernel)", in, out, cyc);
  run<0, 16, 2, 0>("phases of 16 pairs", in, out, cyc);
  run<0, 16, 2, 1>("phases of 16 pairs", in, out, cyc);
  run<0, 32, 2, 1>("phases of 32 pairs", in, out, cyc);
  run<0, 64, 2, 1>("phases of 64 pairs", in, out, cyc);
  run<1, 8, 2, 1>("sw-pipelined 8", in, out, cyc);
  run<1, 16, 2, 1>("sw-pipelined 16", in, out, cyc);
  run<0, 16, 0, 0>("phases of 16, all MUFU", in, out, cyc);
  run<0, 16, 4, 1>("phases of 16", in, out, cyc);
  run<1, 16, 4, 1>("sw-pipelined 16", in, out, cyc);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
