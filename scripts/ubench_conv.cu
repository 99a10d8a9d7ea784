// FFT-engine ceiling on B200: the 8192-point pruned convolution core of K3 (block_conv /
// block_conv_pp from csrc/fft.cuh) run back to back on shared-memory-resident data, no
// global traffic except a final checksum.  Reports microseconds per 2049 column transforms
// (one 2048^2 slice's worth of K3 work) for the launch shapes K3 can take.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_1608_03589_b200/csrc -o scripts/ubench_conv scripts/ubench_conv.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "fft.cuh"

using namespace lpbp;
constexpr int L = 8192;
constexpr int T = FftPlan<L, false>::T;

struct Sync1 {
  __device__ void operator()() const { __syncthreads(); }
};
struct GSync {
  int id;
  __device__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(T) : "memory"); }
};
struct PP {
  int mine, other;
  bool on, skip_last;
  __device__ void enter() const {
    if (on) asm volatile("bar.sync %0, %1;" ::"r"(mine), "r"(2 * T) : "memory");
  }
  __device__ void leave() const {
    if (on) asm volatile("bar.arrive %0, %1;" ::"r"(other), "r"(2 * T) : "memory");
  }
  __device__ void leave_last() const {
    if (on && !skip_last) asm volatile("bar.arrive %0, %1;" ::"r"(other), "r"(2 * T) : "memory");
  }
};

// MODE 0: block_conv, one group per CTA (2 CTAs/SM); MODE 1: block_conv_pp, one group per CTA;
// MODE 2: block_conv_pp two free-running groups per CTA; MODE 3: two groups with the token.
template <int MODE>
__global__ void __launch_bounds__(MODE >= 2 ? 2 * T : T, MODE >= 2 ? 1 : 2)
k(const float2* __restrict__ tw, float* out, int iters) {
  extern __shared__ __align__(16) float2 sm[];
  const int g = MODE >= 2 ? threadIdx.x / T : 0, ti = threadIdx.x % T;
  float2* buf = sm + g * padded_len(L);
  float acc = 0.f;
  const float2 kc = make_float2(0.999f, 0.001f);
  auto load = [&](int idx) { return make_float2((float)(idx & 7) * 0.125f, (float)(idx & 3)); };
  auto mul = [&](int idx, float2 v) { return cmul(v, kc); };
  auto store = [&](int idx, float2 v) { acc += v.x; };
  const GSync gs{1 + g};
  const PP ph{3 + g, 4 - g, MODE == 3, false};
  if (MODE == 3 && g == 1) ph.leave();
  for (int it = 0; it < iters; ++it) {
    if constexpr (MODE == 0) {
      block_conv<L, true, 16>(buf, ti, tw, load, mul, store, Sync1{});
      __syncthreads();
    } else if constexpr (MODE == 1) {
      block_conv_pp<L, true, 16>(buf, ti, tw, load, mul, store, Sync1{}, NoPhase{});
      __syncthreads();
    } else {
      const PP q{ph.mine, ph.other, ph.on, g == 1 && it + 1 == iters};
      block_conv_pp<L, true, 16>(buf, ti, tw, load, mul, store, gs, q);
      gs();
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  float2* tw;
  float* out;
  cudaMalloc(&tw, TwTable<L>::len * sizeof(float2));
  cudaMalloc(&out, 4);
  k_init_twiddles<L><<<(TwTable<L>::len + 255) / 256, 256>>>(tw);
  const int iters = 64;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"block_conv 256 thr x 2 CTA/SM", "block_conv_pp (no hooks) 256 x 2", "pp 2 groups free", "pp 2 groups token"};
  for (int mode = 0; mode < 4; ++mode) {
    const int thr = mode >= 2 ? 2 * T : T;
    const size_t smem = (mode >= 2 ? 2 : 1) * padded_len(L) * sizeof(float2);
    const int ctas = mode >= 2 ? 148 : 296;
    auto launch = [&]() {
      switch (mode) {
        case 0: k<0><<<ctas, thr, smem>>>(tw, out, iters); break;
        case 1: k<1><<<ctas, thr, smem>>>(tw, out, iters); break;
        case 2: k<2><<<ctas, thr, smem>>>(tw, out, iters); break;
        case 3: k<3><<<ctas, thr, smem>>>(tw, out, iters); break;
      }
    };
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double transforms = 296.0 * iters;  // column transforms (fwd + mul + inv) per launch
    printf("%-36s %8.3f ms  %6.1f us per 2049 columns  (%s)\n", names[mode], ms, ms * 1e3 / transforms * 2049,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
