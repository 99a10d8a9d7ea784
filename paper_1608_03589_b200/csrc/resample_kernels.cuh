// Standalone resampling kernels (see resample_kernels.cu).
#pragma once
#include <cuda_runtime.h>

namespace lpbp {

// g [batch][nt][ntheta] -> p [batch][ns][2 ntheta]
cudaError_t launch_semipolar(const float* g, float* p, int nt, int ntheta, int ns, int batch, cudaStream_t s);
// p [batch][ns][nphi] -> lp [batch][nrho][nphi]
cudaError_t launch_semipolar_to_logpolar(const float* p, float* lp, int ns, int nphi, double rho0, int nrho, int batch,
                                         cudaStream_t s);
// lp [batch][nrho][nphi] -> img [batch][ny][nx]
cudaError_t launch_logpolar_to_cartesian(const float* lp, float* img, int nrho, int nphi, double rho0, int nx, int ny,
                                         int batch, cudaStream_t s);

// P [batch] x strided [nsig][nray] complex -> out [batch][ny][nx] complex (Hermitian-averaged)
cudaError_t launch_polar_to_cartesian_frequency(const float2* P, float2* out, int nsig, int nray, long long sm,
                                                long long sr, long long pslice, double dsigma, int nx, int ny,
                                                double dw, float scale, int batch, cudaStream_t s);
// per-slice <g, chord> dt dtheta / 4 (chord_params: [ntheta] trapezoids, bst_host)
cudaError_t launch_mean_backprojection(const float* g, const float4* chord_params, double* out, int nt, int ntheta,
                                       int batch, cudaStream_t s);

}  // namespace lpbp
