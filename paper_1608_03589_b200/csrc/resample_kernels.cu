// Standalone device versions of the reference's resampling functions on the
// log-polar path (the fused pipeline computes them implicitly):
//   k_semipolar        sinogram_to_semipolar   grids.py:290-311
//   k_semi_to_lp       semipolar_to_logpolar   grids.py:332-347
//   k_lp_to_cart       logpolar_to_cartesian   grids.py:399-443 (any nx x ny, fp64 coordinates)
// All use _lerp_axis0 semantics (grids.py:255-269): taps outside the array read zero.
#include <cuda_runtime.h>

#include "resample_kernels.cuh"

namespace lpbp {
namespace {

// v[f] along a strided column with the reference's out-of-range-reads-zero rule
__device__ __forceinline__ float lerp_col(const float* col, size_t stride, int n, double f) {
  const double fl = floor(f);
  const float w = (float)(f - fl);
  const long long i0 = (long long)fl;
  const float a = (i0 >= 0 && i0 < n) ? __ldg(col + (size_t)i0 * stride) : 0.f;
  const float b = (i0 + 1 >= 0 && i0 + 1 < n) ? __ldg(col + (size_t)(i0 + 1) * stride) : 0.f;
  return a * (1.f - w) + b * w;
}

// p[k][j] = g(+s_k, theta_j) for j < ntheta, g(-s_k, theta_{j - ntheta}) otherwise; s_k = k/(ns-1)
__global__ void __launch_bounds__(256)
k_semipolar(const float* __restrict__ g, float* __restrict__ p, int nt, int ntheta, int ns) {
  const int j = blockIdx.x * 256 + threadIdx.x;
  const int k = blockIdx.y;
  const int nphi = 2 * ntheta;
  if (j >= nphi) return;
  const size_t b = blockIdx.z;
  const bool neg = j >= ntheta;
  const int col = neg ? j - ntheta : j;
  const double s = k / (ns - 1.0);
  const double f = ((neg ? -s : s) + 1.0) / (2.0 / nt);
  p[(b * ns + k) * nphi + j] = lerp_col(g + b * nt * ntheta + col, ntheta, nt, f);
}

// lp[i][j] = p(s = e^{rho_i}, phi_j), rho_i = rho0 + (i+1) drho, f = e^rho (ns - 1)
__global__ void __launch_bounds__(256)
k_semi_to_lp(const float* __restrict__ p, float* __restrict__ lp, int ns, int nphi, double rho0, int nrho) {
  const int j = blockIdx.x * 256 + threadIdx.x;
  const int i = blockIdx.y;
  if (j >= nphi) return;
  const size_t b = blockIdx.z;
  const double drho = -rho0 / nrho;
  const double f = exp(rho0 + (i + 1) * drho) * (ns - 1.0);
  lp[(b * nrho + i) * nphi + j] = lerp_col(p + b * ns * nphi + j, nphi, ns, f);
}

// Cartesian readout of a log-polar image at pixel centres (x_j, y_i) of an nx x ny image.
__global__ void __launch_bounds__(256)
k_lp_to_cart(const float* __restrict__ lp, float* __restrict__ img, int nrho, int nphi, double rho0, int nx, int ny) {
  const int jx = blockIdx.x * 32 + threadIdx.x;
  const int iy = blockIdx.y * 8 + threadIdx.y;
  if (jx >= nx || iy >= ny) return;
  const size_t b = blockIdx.z;
  const double x = -1.0 + (jx + 0.5) * (2.0 / nx), y = -1.0 + (iy + 0.5) * (2.0 / ny);
  const double r = hypot(x, y);
  float out = 0.f;
  if (r <= 1.0 && r > 0.0) {
    const double rho = log(r);
    if (rho >= rho0) {
      const double drho = -rho0 / nrho, two_pi = 2.0 * 3.14159265358979323846;
      double fi = (rho - rho0) / drho - 1.0;
      if (fi >= -1.0 && fi < 0.0) fi = 0.0;
      fi = fmin(fmax(fi, 0.0), nrho - 1.0);
      double phi = atan2(y, x);
      if (phi < 0.0) phi += two_pi;
      const double fj = phi / (two_pi / nphi);
      const double fil = floor(fi), fjl = floor(fj);
      const int i0 = (int)fil, i1 = min(i0 + 1, nrho - 1);
      int j0 = (int)fjl % nphi;
      if (j0 < 0) j0 += nphi;
      const int j1 = (j0 + 1) % nphi;
      const float wi = (float)(fi - fil), wj = (float)(fj - fjl);
      const float* v = lp + b * nrho * nphi;
      const float* r0 = v + (size_t)i0 * nphi;
      const float* r1 = v + (size_t)i1 * nphi;
      out = __ldg(r0 + j0) * (1.f - wi) * (1.f - wj) + __ldg(r1 + j0) * wi * (1.f - wj) +
            __ldg(r0 + j1) * (1.f - wi) * wj + __ldg(r1 + j1) * wi * wj;
    }
  }
  img[(b * ny + iy) * nx + jx] = out;
}

// Polar -> Cartesian frequency gridding on an nx x ny FFT-ordered lattice omega = dw k
// (grids.py:456-508): bilinear in (sigma, theta), theta periodic, then the Hermitian
// average 0.5 (G(k) + conj G(-k mod n)), each bin's mirror sampled at its own
// lattice frequency.  fp64 coordinates.  P[m][ray] is read through strides (sm, sr).
__device__ __forceinline__ double fftfreq_k(int k, int n) { return (double)(k < (n + 1) / 2 ? k : k - n); }

__device__ float2 polar_sample(const float2* P, long long sm, long long sr, int nsig, int nray, double dsigma,
                               double wx, double wy) {
  const double two_pi = 2.0 * 3.14159265358979323846;
  const double fi = fmin(hypot(wx, wy) / dsigma, nsig - 1.0);
  const double fil = floor(fi);
  const int i0 = (int)fil, i1 = min(i0 + 1, nsig - 1);
  const double wi = fi - fil;
  double th = atan2(wy, wx);
  if (th < 0.0) th += two_pi;
  const double fj = th / (two_pi / nray);
  const double fjl = floor(fj);
  const double wj = fj - fjl;
  int j0 = (int)fjl % nray;
  if (j0 < 0) j0 += nray;
  const int j1 = (j0 + 1) % nray;
  const float2 a = P[i0 * sm + j0 * sr], b = P[i1 * sm + j0 * sr], c = P[i0 * sm + j1 * sr], d = P[i1 * sm + j1 * sr];
  const float c00 = (float)((1 - wi) * (1 - wj)), c10 = (float)(wi * (1 - wj)), c01 = (float)((1 - wi) * wj),
              c11 = (float)(wi * wj);
  return make_float2(a.x * c00 + b.x * c10 + c.x * c01 + d.x * c11, a.y * c00 + b.y * c10 + c.y * c01 + d.y * c11);
}

__global__ void __launch_bounds__(256)
k_polar_to_cart_freq(const float2* __restrict__ P, float2* __restrict__ out, int nsig, int nray, long long sm,
                     long long sr, long long pslice, double dsigma, int nx, int ny, double dw, float scale) {
  const int ix = blockIdx.x * 32 + threadIdx.x;
  const int iy = blockIdx.y * 8 + threadIdx.y;
  if (ix >= nx || iy >= ny) return;
  const size_t b = blockIdx.z;
  const float2* Pb = P + b * pslice;
  // wx = cartesian_frequencies(nx) * (dw / pi) = pi * k * (dw / pi)
  const double pi = 3.14159265358979323846;
  auto w = [&](int k, int n) { return (pi * fftfreq_k(k, n)) * (dw / pi); };
  const float2 g = polar_sample(Pb, sm, sr, nsig, nray, dsigma, w(ix, nx), w(iy, ny));
  const int mx = (nx - ix) % nx, my = (ny - iy) % ny;
  const float2 h = polar_sample(Pb, sm, sr, nsig, nray, dsigma, w(mx, nx), w(my, ny));
  out[(b * ny + iy) * nx + ix] = make_float2(0.5f * scale * (g.x + h.x), 0.5f * scale * (g.y - h.y));
}

// Spatial mean of the backprojection over [-1, 1]^2 via <g, chord> dt dtheta / 4
// (bst.py:173-180); chord as the per-angle trapezoid (t1, t2, Lmax, 1/(t2-t1)) built
// on the host; fp64 accumulation, one block per slice.
__global__ void __launch_bounds__(256)
k_mean_bp(const float* __restrict__ g, const float4* __restrict__ cp, double* __restrict__ out, int nt, int ntheta) {
  const size_t b = blockIdx.x;
  const float* gb = g + b * nt * ntheta;
  const float dt = 2.f / nt;
  double part = 0.0;
  for (int e = threadIdx.x; e < nt * ntheta; e += blockDim.x) {
    const int t = e / ntheta, j = e - t * ntheta;
    const float4 c = __ldg(cp + j);
    const float a = fabsf(-1.f + t * dt);
    const float ch = a <= c.x ? c.z : (a < c.y ? c.z * (c.y - a) * c.w : 0.f);
    part += (double)__ldg(gb + e) * (double)ch;
  }
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  __shared__ double red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += red[i];
    out[b] = s;
  }
}

}  // namespace

cudaError_t launch_polar_to_cartesian_frequency(const float2* P, float2* out, int nsig, int nray, long long sm,
                                                long long sr, long long pslice, double dsigma, int nx, int ny,
                                                double dw, float scale, int batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  k_polar_to_cart_freq<<<dim3((nx + 31) / 32, (ny + 7) / 8, batch), dim3(32, 8), 0, s>>>(
      P, out, nsig, nray, sm, sr, pslice, dsigma, nx, ny, dw, scale);
  return cudaGetLastError();
}

cudaError_t launch_mean_backprojection(const float* g, const float4* chord_params, double* out, int nt, int ntheta,
                                       int batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  k_mean_bp<<<batch, 256, 0, s>>>(g, chord_params, out, nt, ntheta);
  return cudaGetLastError();
}

cudaError_t launch_semipolar(const float* g, float* p, int nt, int ntheta, int ns, int batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  k_semipolar<<<dim3((2 * ntheta + 255) / 256, ns, batch), 256, 0, s>>>(g, p, nt, ntheta, ns);
  return cudaGetLastError();
}

cudaError_t launch_semipolar_to_logpolar(const float* p, float* lp, int ns, int nphi, double rho0, int nrho, int batch,
                                         cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  k_semi_to_lp<<<dim3((nphi + 255) / 256, nrho, batch), 256, 0, s>>>(p, lp, ns, nphi, rho0, nrho);
  return cudaGetLastError();
}

cudaError_t launch_logpolar_to_cartesian(const float* lp, float* img, int nrho, int nphi, double rho0, int nx, int ny,
                                         int batch, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  k_lp_to_cart<<<dim3((nx + 31) / 32, (ny + 7) / 8, batch), dim3(32, 8), 0, s>>>(lp, img, nrho, nphi, rho0, nx, ny);
  return cudaGetLastError();
}

}  // namespace lpbp
