// Launch cost vs kernel-parameter size (sm_100a): back-to-back launches of a copy kernel that
// moves 16 MiB (read) + 16 MiB (write) like the C2 append, with a by-value parameter block of
// N bytes (only the first 16 bytes are read).  Prints the average time per launch from CUDA
// events around 200 launches, for N = 64 .. 6144, and for an empty kernel.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o param_size_bench param_size_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
struct Blob {
  alignas(16) unsigned char b[N];
};

template <int N>
__global__ void __launch_bounds__(256) copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, long n,
                                                   const __grid_constant__ Blob<N> blob) {
  const int off = blob.b[0];
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    dst[i + off] = src[i];
}
template <int N>
__global__ void empty_kernel(const __grid_constant__ Blob<N> blob) {
  if (blob.b[1] == 77 && threadIdx.x == 1000) printf("x");
}

template <int N>
void run(uint4* const* src, uint4* dst, long n, cudaStream_t st) {
  Blob<N> b{};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * 8;
  for (int i = 0; i < 20; ++i) copy_kernel<N><<<grid, 256, 0, st>>>(src[i & 7], dst, n, b);
  cudaEventRecord(e0, st);
  for (int i = 0; i < 200; ++i) copy_kernel<N><<<grid, 256, 0, st>>>(src[i & 7], dst, n, b);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const float us = ms * 1e3f / 200;
  for (int i = 0; i < 20; ++i) empty_kernel<N><<<1, 32, 0, st>>>(b);
  cudaEventRecord(e0, st);
  for (int i = 0; i < 200; ++i) empty_kernel<N><<<1, 32, 0, st>>>(b);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms2 = 0;
  cudaEventElapsedTime(&ms2, e0, e1);
  printf("param %5d B: copy 32 MiB %7.2f us/launch (%6.0f GB/s)   empty kernel %6.2f us/launch\n", N, us,
         2.0 * n * 16 / (us * 1e-6) / 1e9, ms2 * 1e3f / 200);
}

int main() {
  const long n = (16l << 20) / 16;
  uint4 *src[8], *dst;        // 8 sources of 16 MiB (128 MiB > L2): reads come from HBM
  for (int i = 0; i < 8; ++i) {
    cudaMalloc(&src[i], n * 16 + 4096);
    cudaMemset(src[i], 1, n * 16);
  }
  cudaMalloc(&dst, n * 16 + 4096);
  cudaStream_t st;
  cudaStreamCreate(&st);
  run<64>(src, dst, n, st);
  run<1024>(src, dst, n, st);
  run<2048>(src, dst, n, st);
  run<4096>(src, dst, n, st);
  run<6144>(src, dst, n, st);
  run<64>(src, dst, n, st);
  return 0;
}
