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

}  // namespace lpbp
