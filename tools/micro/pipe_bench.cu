// Microbenchmark: issue cost per warp instruction on one SMSP for the instructions of the
// attention softmax (which pipe each one uses decides the softmax's critical resource).
// Each kernel runs 8 independent chains per thread, W warps per SMSP; reports cycles per warp
// instruction per SMSP (1.0 = one per clock).  Pairs (A + B in the same loop) show whether two
// instructions share a pipe (cost adds) or not (cost = max).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/pipe_bench.cu -o /tmp/pipe_bench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t f2bf(float lo, float hi) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b) { uint32_t r; asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ float mx3(float a, float b, float c) { float r; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ uint32_t iadd(uint32_t a, uint32_t b) { uint32_t r; asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ uint32_t shl(uint32_t a) { uint32_t r; asm volatile("shl.b32 %0, %1, 23;" : "=r"(r) : "r"(a)); return r; }
__device__ __forceinline__ float fadd(float a, float b) { float r; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float fmul(float a, float b) { float r; asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ uint32_t f2h2(float lo, float hi) { uint32_t r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ uint32_t lop(uint32_t a, uint32_t b) { uint32_t r; asm volatile("and.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b)); return r; }
__device__ __forceinline__ float frnd(float a) { float r; asm volatile("cvt.rni.f32.f32 %0, %1;" : "=f"(r) : "f"(a)); return r; }
__device__ __forceinline__ int f2i(float a) { int r; asm volatile("cvt.rni.s32.f32 %0, %1;" : "=r"(r) : "f"(a)); return r; }

// op ids
enum { EX2 = 0, F2BF, PRMT, MX3, FFMA2, IADD, SHL, FADD, FMUL, F2H2, LOP, FRND, F2I,
       EX2_F2BF, EX2_PRMT, EX2_FFMA2, EX2_MX3, F2BF_FFMA2, EX2_IADD, F2BF_MX3, NOPS };
static const char* names[] = {"MUFU.EX2", "F2FP.BF16 (cvt.rn.bf16x2)", "PRMT", "FMNMX3", "FFMA2", "IADD", "SHL",
                              "FADD", "FMUL", "F2FP.F16 (cvt.rn.f16x2)", "LOP3", "FRND", "F2I",
                              "EX2+F2BF", "EX2+PRMT", "EX2+FFMA2", "EX2+FMNMX3", "F2BF+FFMA2", "EX2+IADD", "F2BF+FMNMX3"};

template <int OP>
__global__ void k(uint32_t* out, int iters, long long* cycles) {
  float f[8];
  uint32_t u[8];
  float2 g[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    f[i] = 0.001f * (threadIdx.x + i);
    u[i] = threadIdx.x * 3 + i;
    g[i] = make_float2(f[i], f[i] + 1.f);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 4; ++rep) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == EX2 || OP == EX2_F2BF || OP == EX2_PRMT || OP == EX2_FFMA2 || OP == EX2_MX3 || OP == EX2_IADD)
          f[i] = ex2(f[i]);
        if (OP == F2BF || OP == EX2_F2BF || OP == F2BF_FFMA2 || OP == F2BF_MX3)
          u[i] = f2bf(__uint_as_float(u[i]), f[i]);
        if (OP == PRMT || OP == EX2_PRMT) u[i] = prmt(u[i], __float_as_uint(f[i]));
        if (OP == MX3 || OP == EX2_MX3 || OP == F2BF_MX3) g[i].x = mx3(g[i].x, g[i].y, f[(i + 1) & 7]);
        if (OP == FFMA2 || OP == EX2_FFMA2 || OP == F2BF_FFMA2) g[i] = ffma2(g[i], g[i], g[(i + 3) & 7]);
        if (OP == IADD || OP == EX2_IADD) u[i] = iadd(u[i], u[(i + 1) & 7]);
        if (OP == SHL) u[i] = shl(u[i]);
        if (OP == FADD) f[i] = fadd(f[i], f[(i + 1) & 7]);
        if (OP == FMUL) f[i] = fmul(f[i], f[(i + 1) & 7]);
        if (OP == F2H2) u[i] = f2h2(__uint_as_float(u[i]), f[i]);
        if (OP == LOP) u[i] = lop(u[i], u[(i + 1) & 7]);
        if (OP == FRND) f[i] = frnd(f[i]);
        if (OP == F2I) u[i] = f2i(__uint_as_float(u[i]));
      }
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= u[i] ^ __float_as_uint(f[i]) ^ __float_as_uint(g[i].x) ^ __float_as_uint(g[i].y);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = (t1 - t0);
}

template <int OP>
void run(int wps, uint32_t* out, long long* cyc) {
  const int iters = 2000;
  k<OP><<<1, 128 * wps>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  // warp instructions per SMSP of each kind = wps * iters * 32
  const double per = (double)h / ((double)wps * iters * 32);
  printf("%-28s W=%d  %.3f cycles / warp-instr / SMSP  (%.1f lanes/clk/SM)\n", names[OP], wps, per, 128.0 / per);
}

template <int OP>
void runall(uint32_t* out, long long* cyc) {
  run<OP>(1, out, cyc);
  run<OP>(4, out, cyc);
}

int main() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 8);
  runall<EX2>(out, cyc); runall<F2BF>(out, cyc); runall<PRMT>(out, cyc); runall<MX3>(out, cyc);
  runall<FFMA2>(out, cyc); runall<IADD>(out, cyc); runall<SHL>(out, cyc); runall<FADD>(out, cyc);
  runall<FMUL>(out, cyc); runall<F2H2>(out, cyc); runall<LOP>(out, cyc); runall<FRND>(out, cyc);
  runall<F2I>(out, cyc);
  runall<EX2_F2BF>(out, cyc); runall<EX2_PRMT>(out, cyc); runall<EX2_FFMA2>(out, cyc);
  runall<EX2_MX3>(out, cyc); runall<F2BF_FFMA2>(out, cyc); runall<EX2_IADD>(out, cyc);
  runall<F2BF_MX3>(out, cyc);
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
