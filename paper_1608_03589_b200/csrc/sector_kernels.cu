// Device kernels of the sector (partial) log-polar backprojection
// (fastbp.logpolar.partial_backproject, logpolar.py:210-299).  The per-sector
// log-polar stage reuses the backprojection kernels through a sub-plan; these
// two kernels are the steps around it.
#include <cuda_runtime.h>

#include "sector_kernels.cuh"

namespace lpbp {
namespace {

// Working-frame sinogram of one sector, one output sample per thread:
//   rolled(m, j)  = g(m, src_j), or g(nt - m, src_j) (0 at m = 0) for flipped columns
//   scaled(k, j)  = a_r * lerp_m(w_j * rolled(., j), fi1_k),  fi1_k = (t_k / a_r + 1) / dt
//   out(i, j)     = lerp_k(scaled(., j), (t_i - off_j + 1) / dt)
// with zero outside [0, nt) at both levels (grids.py:255-269), i.e. the reference's
// _roll_angles -> weights -> _rescale_support -> shift_sinogram chain
// (logpolar.py:153-179, 260-271; radon.py:137-158).  Weights and bases come from
// fp64 host tables (per column: source, flip, weight, shift base; per row: the
// shrink lerp), so a sample is 4 gathers and a few FMAs.
__global__ void __launch_bounds__(256)
k_sector_prep(const float* __restrict__ g, float* __restrict__ out, int nt, int ntheta, int nin,
              const SectorCol* __restrict__ cols, const SectorRow* __restrict__ rows, double a_r, int klo, int khi) {
  const int j = blockIdx.x * 32 + threadIdx.x;
  const int i = blockIdx.y * 8 + threadIdx.y;
  if (j >= ntheta || i >= nt) return;
  const size_t slice_in = (size_t)blockIdx.z * nt * nin;
  const size_t slice_out = (size_t)blockIdx.z * nt * ntheta;
  const SectorCol c = cols[j];
  const float w2 = c.w2;
  const int k2 = i + c.d;  // floor((t_i - off + 1) / dt) with the per-column fraction w2
  // zero-weight angle (outside this sector's extended mask) or both shrink taps outside the
  // rows that can be nonzero: the sample is exactly zero, skip the loads
  if (c.w == 0.f || k2 + 1 < klo || k2 > khi) {
    out[slice_out + (size_t)i * ntheta + j] = 0.f;
    return;
  }
  const float* col = g + slice_in + c.src;
  auto rolled = [&](int m) -> float {
    if (m < 0 || m >= nt) return 0.f;
    if (c.flip) {
      if (m == 0) return 0.f;  // t = -1 maps to +1, off the grid
      m = nt - m;
    }
    return __ldg(col + (size_t)m * nin);
  };
  const float a = (float)a_r;
  auto scaled = [&](int k) -> float {
    if (k < 0 || k >= nt) return 0.f;
    const SectorRow r = rows[k];
    return a * ((rolled(r.k1) * c.w) * (1.f - r.w1) + (rolled(r.k1 + 1) * c.w) * r.w1);
  };
  out[slice_out + (size_t)i * ntheta + j] = scaled(k2) * (1.f - w2) + scaled(k2 + 1) * w2;
}

// Sum of every sector's bilinear log-polar sample at the working-frame image of
// each pixel, x_w = (1 - a_r, 0) + a_r R(-theta_c) x, divided by a_r
// (logpolar.py:191-215, 289-297).  Coordinates and the discontinuous predicates
// (0 < r <= 1, ln r >= rho0) in fp64, once per pixel and sector for a group of G
// slices; the pixel is written once.
template <int G>
__global__ void __launch_bounds__(256)
k_sector_readout(const __grid_constant__ SectorArgs secs, int nsec, float* __restrict__ img, int n, int nphi,
                 int batch) {
  const int jx = blockIdx.x * 32 + threadIdx.x;
  const int iy = blockIdx.y * 8 + threadIdx.y;
  if (jx >= n || iy >= n) return;
  const int b0 = blockIdx.z * G;
  const int nb = min(G, batch - b0);
  const double h = 2.0 / n;
  const double x = -1.0 + (jx + 0.5) * h, y = -1.0 + (iy + 0.5) * h;
  const double two_pi = 2.0 * 3.14159265358979323846;
  const double dphi = two_pi / nphi;
  float acc[G];
#pragma unroll
  for (int b = 0; b < G; ++b) acc[b] = 0.f;
  for (int s = 0; s < nsec; ++s) {
    const SectorDev& S = secs.s[s];
    const double xw = (1.0 - S.a_r) + S.a_r * (S.ct * x + S.st * y);
    const double yw = S.a_r * (-S.st * x + S.ct * y);
    const double r = hypot(xw, yw);
    if (!(r <= 1.0 && r > 0.0)) continue;
    const double rho = log(r);
    if (!(rho >= S.rho0)) continue;
    double fi = (rho - S.rho0) / S.drho - 1.0;
    if (fi >= -1.0 && fi < 0.0) fi = 0.0;
    fi = fmin(fmax(fi, 0.0), S.nrho - 1.0);
    double phi = atan2(yw, xw);
    if (phi < 0.0) phi += two_pi;  // np.mod(phi, 2 pi) for phi in [-pi, pi]
    const double fj = phi / dphi;
    const double fjl = floor(fj);
    const double fil = floor(fi);
    const int i0 = (int)fil;
    const int i1 = min(i0 + 1, S.nrho - 1);
    int j0 = (int)fjl % nphi;
    if (j0 < 0) j0 += nphi;
    const int j1 = (j0 + 1) % nphi;
    const float wi = (float)(fi - fil), wj = (float)(fj - fjl);
    const float c00 = (1.f - wi) * (1.f - wj), c10 = wi * (1.f - wj), c01 = (1.f - wi) * wj, c11 = wi * wj;
    const float inv_a = S.inv_a;
    const float* base = S.lp + (size_t)b0 * S.lp_slice;
#pragma unroll
    for (int b = 0; b < G; ++b) {
      if (b < nb) {
        const float* v = base + (size_t)b * S.lp_slice;
        const float* r0 = v + (size_t)i0 * nphi;
        const float* r1 = v + (size_t)i1 * nphi;
        const float val = __ldg(r0 + j0) * c00 + __ldg(r1 + j0) * c10 + __ldg(r0 + j1) * c01 + __ldg(r1 + j1) * c11;
        acc[b] += val * inv_a;
      }
    }
  }
  float* o = img + (size_t)b0 * n * n + (size_t)iy * n + jx;
#pragma unroll
  for (int b = 0; b < G; ++b)
    if (b < nb) o[(size_t)b * n * n] = acc[b];
}

}  // namespace

cudaError_t launch_sector_prep(const float* g, float* out, int nt, int ntheta, int nin, int batch,
                               const SectorCol* cols, const SectorRow* rows, double a_r, int klo, int khi,
                               cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  const dim3 grid((ntheta + 31) / 32, (nt + 7) / 8, batch);
  k_sector_prep<<<grid, dim3(32, 8), 0, s>>>(g, out, nt, ntheta, nin, cols, rows, a_r, klo, khi);
  return cudaGetLastError();
}

cudaError_t launch_sector_readout(const SectorArgs& secs, int nsec, float* img, int n, int nphi, int batch,
                                  cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  constexpr int G = kSectorGroup;
  const dim3 grid((n + 31) / 32, (n + 7) / 8, (batch + G - 1) / G);
  k_sector_readout<G><<<grid, dim3(32, 8), 0, s>>>(secs, nsec, img, n, nphi, batch);
  return cudaGetLastError();
}

}  // namespace lpbp
