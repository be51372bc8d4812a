// Microbenchmark: MUFU throughput of ex2.approx.ftz.f32 (one element) vs ex2.approx.ftz.bf16x2
// (two elements per instruction) on sm_100a, 4 warps per SMSP, independent chains.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/ex2_bf16x2_bench.cu -o /tmp/ex2b
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(uint32_t* out, int iters, long long* cycles) {
  uint32_t r[16];
  float f[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    f[i] = -0.001f * (threadIdx.x + i);
    r[i] = 0x3f00bf00u + threadIdx.x + i;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      else asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[i]));
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc ^= r[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

int main() {
  uint32_t* out; cudaMalloc(&out, 148 * 1024 * 4);
  long long* cyc; cudaMalloc(&cyc, 8);
  const int iters = 2000;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<148, 512>>>(out, iters, cyc); else k<1><<<148, 512>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      // per SMSP: 4 warps x iters x 16 instructions
      const double instr = 4.0 * iters * 16;
      const double elems = instr * 32 * (mode ? 2 : 1);
      if (rep) printf("%-28s %6.2f cycles per warp-instruction per SMSP, %5.2f elements/clk/SMSP\n",
                      mode ? "ex2.approx.ftz.bf16x2" : "ex2.approx.ftz.f32", h / instr, elems / h);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
