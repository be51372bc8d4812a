// Microbenchmark: MUFU.EX2 (f32, f16x2) and FMA-pipe throughput per SM on this GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = (threadIdx.x + i) * -1e-3f;
  uint32_t h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = 0x3c003c00u + i + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 1 && i < 8) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
      if (MODE == 2) asm volatile("fma.rn.f32 %0, %0, 0f3F7FF000, 0f3A000000;" : "+f"(a[i]));
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __half2float(__ushort_as_half((unsigned short)h[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int ops_per_iter) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out; cudaMalloc(&out, sms * 8 * 512 * sizeof(float));
  const int iters = 4096;
  for (int w = 0; w < 2; ++w) k<MODE><<<sms * 4, 512>>>(out, iters);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<sms * 4, 512>>>(out, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (double)sms * 4 * 512 * iters * ops_per_iter;
  double per_s = ops / (ms * 1e-3);
  printf("%-12s %.3f Tops/s  = %.1f per SM per clock at %d MHz (nominal clockRate)\n", name, per_s / 1e12,
         per_s / sms / (clk * 1e3), clk / 1000);
  cudaFree(out);
}

int main() {
  run<0>("ex2.f32", 16);
  run<1>("ex2.f16x2", 16);   // 8 instructions x 2 values
  run<2>("ffma.f32", 16);
  return 0;
}
