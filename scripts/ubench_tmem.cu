// TMEM as per-thread storage outside MMA (B200, sm_100a): 2 CTAs x 8 warps per SM, each CTA allocates
// 256 columns; warp w uses lanes 32*(w%4).. and columns 128*(w/4)...  Measures the rate of
// tcgen05.ld.32x32b.x16 (+ wait) and checks that values written with tcgen05.st read back.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/ubench_tmem scripts/ubench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(256, 2) k(float* out, int iters, int* bad) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t base = taddr_s + ((uint32_t)(32 * (warp % 4)) << 16) + 128u * (warp / 4);
  // write 128 columns: value = f(thread, col)
  for (int c = 0; c < 128; c += 8) {
    uint32_t v[8];
    for (int i = 0; i < 8; ++i) v[i] = __float_as_uint((float)(threadIdx.x * 1000 + c + i + blockIdx.x));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(base + c),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;\n");
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 128; c += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15}, [%16];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(base + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (it == 0) {
        for (int i = 0; i < 16; ++i)
          if (__uint_as_float(v[i]) != (float)(threadIdx.x * 1000 + c + i + blockIdx.x)) atomicAdd(bad, 1);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc += __uint_as_float(v[i]);
    }
  }
  if (acc == 1.2345f) out[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(taddr_s));
}

int main() {
  float* out;
  int* bad;
  cudaMalloc(&out, 4);
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  const int iters = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<0><<<296, 256>>>(out, 4, bad);
  cudaDeviceSynchronize();
  printf("warmup: %s\n", cudaGetErrorString(cudaGetLastError()));
  cudaEventRecord(e0);
  k<0><<<296, 256>>>(out, iters, bad);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int hb;
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  const double bytes = 296.0 * 256 * iters * 128 * 4;  // per-thread 128 columns x 4 B per iteration
  printf("tcgen05.ld 32x32b.x16: %.3f ms, %.1f TB/s total, %.1f B/clk/SM at 1.965 GHz, mismatches %d (%s)\n", ms,
         bytes / ms / 1e9, bytes / (ms * 1e-3) / 148 / 1.965e9, hb, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
