// BST engine kernels: launchers and device-side tables (see bst_kernels.cu).
#pragma once
#include <cuda_runtime.h>

namespace lpbp {

struct BstTables {
  const int2* tap_base;   // [ns] semi-polar lerp bases (+s, -s)
  const float4* tap_w;    // [ns] weights with the window folded in
  const float* kern;      // [m_need] radial kernel incl. ds and the Hermitian 1/2
  const float2* tau;      // [big] phase ramp
  const float2* cmean;    // [big] crop-mean weights
  const float4* chord;    // [ntheta] chord trapezoid (t1, t2, Lmax dt dtheta / 4, 1/(t2 - t1)) (subtract_mean)
  const uint2* grid_q;    // [big/2][big/2 + 1] quadrant gridding coordinates
  const float2* tw_L;     // pass twiddles, N = L
  const float2* tw_big;   // pass twiddles, N = big
  // generic sizes (Bluestein): chirps of the DFT lengths and the convolution filters
  const float2* chirp_L;  // [L]
  const float2* bhat_L;   // [mb_L] forward filter spectrum / mb_L
  const float2* tw_mbL;   // pass twiddles, N = mb_L
  const float2* chirp_big;  // [big]
  const float2* bhat_big;   // [mb_big] inverse filter spectrum / mb_big
  const float2* tw_mbbig;   // pass twiddles, N = mb_big
};

struct BstDims {
  int nt, ntheta, n, ns, nray, L, m_need, m_pad, big, p0;
  int mb_L, mb_big;  // Bluestein convolution sizes (0 = power-of-two direct FFT)
  int subtract_mean;
  double dsigma, dw;
  float s_img;   // output scale (BST_SCALE / (4 d^2), x 1/(2 pi) for fbp)
  float s_mean;  // BST_SCALE / (4 d^2): crop-mean accumulator -> BST image units
  float fbp;     // 1 or 1/(2 pi)
};

// P: [B][nray][m_pad] complex; acc: [B][2] doubles (zeroed by the caller)
cudaError_t launch_bst_radial(const BstDims& d, const BstTables& t, const float* g, float2* P, double* acc, int batch,
                              cudaStream_t s);
// X: [B][n][big/2] complex workspace; img: [B][n][n]
// mid (optional): recorded on s between the grid_x and grid_y launches (stage profiling)
cudaError_t launch_bst_grid(const BstDims& d, const BstTables& t, const float2* P, float2* X, float* img, double* acc,
                            int batch, cudaStream_t s, cudaEvent_t mid = nullptr);

}  // namespace lpbp
