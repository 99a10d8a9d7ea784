// Issue/pipe throughput of the FP32 instruction forms the FFT engine uses (B200, sm_100a).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_fp32 scripts/ubench_fp32.cu
// Each kernel runs 8 independent dependency chains per thread, 16 warps per SM, and reports
// warp-instructions per clock per SM (4.0 = one per SMSP per clock).
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ unsigned long long a2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long m2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <int MODE>
__global__ void k(float* out, float s, long long* cyc) {
  unsigned long long x[8], y[8];
  float fx[8], fy[8];
  const unsigned long long c = __double_as_longlong((double)s);
  for (int i = 0; i < 8; ++i) {
    x[i] = __double_as_longlong((double)(threadIdx.x + i));
    y[i] = __double_as_longlong((double)(threadIdx.x * 3 + i));
    fx[i] = threadIdx.x + i;
    fy[i] = threadIdx.x * 0.5f + i;
  }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (MODE == 0) x[i] = f2(x[i], y[i], c);                   // FFMA2, 3 registers
      if constexpr (MODE == 1) x[i] = a2(x[i], y[i]);                      // FADD2
      if constexpr (MODE == 2) x[i] = m2(x[i], y[i]);                      // FMUL2
      if constexpr (MODE == 3) fx[i] = fmaf(fx[i], fy[i], fy[(i + 1) & 7]); // FFMA 3 registers
      if constexpr (MODE == 4) fx[i] = fmaf(fx[i], 1.0001f, 0.5f);         // FFMA immediate
      if constexpr (MODE == 5) { x[i] = f2(x[i], y[i], c); fx[i] = fmaf(fx[i], fy[i], s); }  // mixed
      if constexpr (MODE == 7) x[i] = f2(x[i], 0x3f8000003f800000ull, y[i]);   // FFMA2 broadcast immediate
      if constexpr (MODE == 6) { x[i] = f2(x[i], y[i], c); fx[i] = fx[i] + fy[i]; }          // FFMA2 + FADD
      if constexpr (MODE == 8) { x[i] = f2(x[i], y[i], c); y[i] = a2(y[i], c); }              // FFMA2 + FADD2
      if constexpr (MODE == 9) { x[i] = m2(x[i], c); y[i] = a2(y[i], c); }                   // FMUL2 + FADD2
      if constexpr (MODE == 10) { x[i] = f2(x[i], y[i], c); x[(i + 4) & 7] = f2(x[(i + 4) & 7], y[i], c); y[i] = a2(y[i], c); }  // 2 FFMA2 + FADD2
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
  for (int i = 0; i < 8; ++i) acc += (float)__longlong_as_double(x[i]) + fx[i];
  if (acc == 12345.f) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 8);
  const char* names[] = {"FFMA2 (3 reg)", "FADD2", "FMUL2", "FFMA (3 reg)", "FFMA (imm)", "FFMA2 + FFMA", "FFMA2 + FADD", "FFMA2 (imm)", "FFMA2 + FADD2", "FMUL2 + FADD2", "2 FFMA2 + FADD2"};
  const int per_iter[] = {8, 8, 8, 8, 8, 16, 16, 8, 16, 16, 24};
  for (int warps : {8, 16, 32}) {
    for (int mode = 0; mode < 11; ++mode) {
      auto run = [&]() {
        switch (mode) {
          case 0: k<0><<<148, warps * 32>>>(out, 1.f, cyc); break;
          case 1: k<1><<<148, warps * 32>>>(out, 1.f, cyc); break;
          case 2: k<2><<<148, warps * 32>>>(out, 1.f, cyc); break;
          case 3: k<3><<<148, warps * 32>>>(out, 1.f, cyc); break;
          case 4: k<4><<<148, warps * 32>>>(out, 1.f, cyc); break;
          case 5: k<5><<<148, warps * 32>>>(out, 1.f, cyc); break;
          case 6: k<6><<<148, warps * 32>>>(out, 1.f, cyc); break;
          case 7: k<7><<<148, warps * 32>>>(out, 1.f, cyc); break;
          case 8: k<8><<<148, warps * 32>>>(out, 1.f, cyc); break;
          case 9: k<9><<<148, warps * 32>>>(out, 1.f, cyc); break;
          case 10: k<10><<<148, warps * 32>>>(out, 1.f, cyc); break;
        }
      };
      run();
      cudaDeviceSynchronize();
      run();
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double instr = (double)warps * ITERS * per_iter[mode];
      printf("warps/SM %2d  %-16s  %6.3f warp-instr/clk/SM  (%lld clk)\n", warps, names[mode], instr / c, c);
    }
  }
  return 0;
}
