// Which FP32 instruction forms share an issue pipe on B200 (sm_100a): every pair of
// {FFMA2, FADD2, FMUL2, FFMA, FADD, FMUL, MUFU.SIN} interleaved 1:1 in 16 independent chains per
// thread, 16 warps per SM.  Reports warp-instructions per clock per SM for the pair; a pair that runs
// at the sum of its members' solo rates issues on two different pipes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_pipes scripts/ubench_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048
typedef unsigned long long u64;

template <int OP>
__device__ __forceinline__ void op(u64& x, float& f, u64 y, u64 c, float fy) {
  if constexpr (OP == 0) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(y), "l"(c));
  if constexpr (OP == 1) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
  if constexpr (OP == 2) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
  if constexpr (OP == 3) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f) : "f"(fy), "f"(fy));
  if constexpr (OP == 4) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(f) : "f"(fy));
  if constexpr (OP == 5) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(f) : "f"(fy));
  if constexpr (OP == 6) asm volatile("sin.approx.f32 %0, %0;" : "+f"(f));
}

template <int A, int B>
__global__ void k(float* out, float s, long long* cyc) {
  u64 x[8], z[8];
  float fx[8], fz[8];
  const u64 c = __double_as_longlong((double)s);
  const u64 y = __double_as_longlong((double)(threadIdx.x * 3));
  const float fy = threadIdx.x * 0.5f;
  for (int i = 0; i < 8; ++i) {
    x[i] = __double_as_longlong((double)(threadIdx.x + i));
    z[i] = x[i] + 1;
    fx[i] = threadIdx.x + i;
    fz[i] = fx[i] + 1.f;
  }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 2
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      op<A>(x[i], fx[i], y, c, fy);
      op<B>(z[i], fz[i], y, c, fy);
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
  for (int i = 0; i < 8; ++i) acc += (float)__longlong_as_double(x[i]) + (float)__longlong_as_double(z[i]) + fx[i] + fz[i];
  if (acc == 12345.f) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

const char* names[] = {"FFMA2", "FADD2", "FMUL2", "FFMA", "FADD", "FMUL", "MUFU"};
float* out;
long long* cyc;

template <int A, int B>
void run1() {
  const int warps = 16;
  k<A, B><<<148, warps * 32>>>(out, 1.f, cyc);
  cudaDeviceSynchronize();
  k<A, B><<<148, warps * 32>>>(out, 1.f, cyc);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-6s + %-6s  %6.3f warp-instr/clk/SM\n", names[A], names[B], (double)warps * ITERS * 16 / c);
}

template <int A, int B>
void row() {
  if constexpr (B <= 6) {
    run1<A, B>();
    row<A, B + 1>();
  }
}
template <int A>
void all() {
  if constexpr (A <= 6) {
    row<A, A>();
    all<A + 1>();
  }
}

int main() {
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 8);
  all<0>();
  return 0;
}
