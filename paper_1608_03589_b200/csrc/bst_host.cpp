// fp64 tables of the BST engine.  Every formula restates
// /root/reference/pkg/src/fastbp/bst.py (and grids.py:290-311, 451-508).
#include "bst_host.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <thread>

namespace lpbp {
namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kBstScale = 4.0 * kPi;  // bst.py:47
constexpr int kOversample = 2;           // bst.py:52
constexpr int kDomainPad = 2;            // bst.py:58

// Modified Bessel function I0 by its power series (scipy.special.i0 to ~1e-16
// for the arguments a window uses; the terms are all positive).
double bessel_i0(double x) {
  const double q = 0.25 * x * x;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 500; ++k) {
    term *= q / ((double)k * k);
    sum += term;
    if (term < 1e-17 * sum) break;
  }
  return sum;
}

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

// (13-bit index, 19-bit fixed-point weight) of a clamped fractional coordinate
uint32_t pack_coord(double f) {
  double fl = std::floor(f);
  long long q = std::llround((f - fl) * 524288.0);
  if (q >= 524288) {
    q = 0;
    fl += 1.0;
  }
  return (uint32_t)(long long)fl | ((uint32_t)q << 13);
}

}  // namespace

std::string build_bst_host(const BstParams& p, BstHost& h) {
  // BstOptions (bst.py:79-87), in the reference's order
  if (p.n < 2) return "n_out must be >= 2";
  if (p.beta < 0) return "beta must be >= 0";
  if (p.zero_pad < 1) return "zero_pad must be >= 1";
  if (p.dc_mode != 0 && p.dc_mode != 1) return "dc_mode must be 'subtract_mean' or 'kernel_cap'";
  if (p.filter) {
    if (p.lam < 0) return "lambda must be >= 0";
    if (!(0.0 < p.cutoff && p.cutoff <= 1.0)) return "cutoff must lie in (0, 1]";
  }
  if (p.nt < 4 || p.ntheta < 1) return "sinogram must have nt >= 4 and ntheta >= 1";
  h = BstHost{};
  h.p = p;
  const int nt = p.nt;
  h.ns = kOversample * (nt / 2);
  const int ns = h.ns;
  h.nray = 2 * p.ntheta;
  h.ds = 1.0 / (ns - 1);
  h.L = next_fast_len(std::max((int)std::ceil(2.0 * p.zero_pad * (ns - 1)), ns));
  h.dsigma = 2.0 * kPi / (h.L * h.ds);
  const double sigma_need = std::sqrt(2.0) * kPi * p.n / 2.0;
  h.m_need = (int)std::floor(sigma_need / h.dsigma) + 2;
  if (h.m_need > h.L / 2 + 1) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "n_out = %d exceeds the resolution supported by an nt = %d sinogram (max ~ %d)",
                  p.n, nt, (int)(std::sqrt(2.0) * (ns - 1)));
    return buf;
  }
  h.m_pad = (h.m_need + 4) / 4 * 4;  // >= m_need + 1: the gridding reads bin i0 + 1 unguarded
  h.big = kDomainPad * p.n;
  h.dw = kPi / kDomainPad;
  h.p0 = ((kDomainPad - 1) * p.n) / 2;
  h.out_scale = kBstScale / (4.0 * kDomainPad * kDomainPad);  // ifft2 1/big^2 x big^2/(4 d^2); unnormalised FFTs here
  if (p.filter) h.out_scale *= 1.0 / (2.0 * kPi);                // filtering.py:27, 98

  // semi-polar taps on s_k = k/(ns-1), window w_k (bst.py:90-102, 131-136)
  const double dt = 2.0 / nt;
  const double i0b = std::fabs(bessel_i0(p.beta));
  h.tap_base.resize(ns);
  h.tap_w.resize(ns);
  for (int k = 0; k < ns; ++k) {
    const double s = k / (ns - 1.0);
    const double u = (2.0 * k - ns + 1.0) / (ns - 1.0);
    double win = std::fabs(bessel_i0(p.beta * std::sqrt(std::max(1.0 - u * u, 0.0)))) / i0b;
    if (k == 0) win *= 0.5;  // s = 0 is shared by the two half-lines (bst.py:133-135)
    int32_t bp, bn;
    double pw0, pw1, nw0, nw1;
    lerp_tap_public((s + 1.0) / dt, nt, bp, pw0, pw1);
    lerp_tap_public((-s + 1.0) / dt, nt, bn, nw0, nw1);
    h.tap_base[k] = I2{bp, bn};
    h.tap_w[k] = F4{(float)(pw0 * win), (float)(pw1 * win), (float)(nw0 * win), (float)(nw1 * win)};
  }
  // radial kernel (bst.py:105-117, 188-193) with ds and the Hermitian 1/2 folded in
  h.kern.resize(h.m_need);
  for (int m = 0; m < h.m_need; ++m) {
    double k;
    if (m == 0) k = (p.dc_mode == 0) ? 0.0 : 1.0 / h.dsigma;
    else k = 1.0 / (m * h.dsigma);
    h.kern[m] = (float)(0.5 * h.ds * k);
  }
  // phase ramp and crop-mean weights (bst.py:159-169)
  const int big = h.big;
  const double dx = 2.0 / p.n;
  const double ph = (0.5 - h.p0) * dx - 1.0;
  h.tau.resize(big);
  h.cmean.resize(big);
  for (int k = 0; k < big; ++k) {
    const long long kf = k < (big + 1) / 2 ? k : (long long)k - big;  // fftfreq(big) * big
    const double a = h.dw * (double)kf * ph;
    h.tau[k] = F2{(float)std::cos(a), (float)std::sin(a)};
    double cr = 0.0, ci = 0.0;
    for (int y = h.p0; y < h.p0 + p.n; ++y) {
      const double b = 2.0 * kPi * (double)(((long long)k * y) % big) / big;
      cr += std::cos(b);
      ci += std::sin(b);
    }
    const double inv = 1.0 / ((double)p.n * p.n);
    h.cmean[k] = F2{(float)(cr * inv), (float)(ci * inv)};
  }
  if (p.filter) build_ramp_taps(nt, p.lam, p.cutoff, h.M, h.Lr, h.ramp);
  // chord weights of the exact mean (bst.py:173-180): for |cos|, |sin| the chord of the line
  // x . xi = t through [-1, 1]^2 is a trapezoid in t; the reference's degenerate axes
  // (|cos| or |sin| <= 1e-15) give 2 on |t| <= 1
  if (p.dc_mode == 0) {
    h.chord_col.resize(p.ntheta);
    const double dth = kPi / p.ntheta;
    for (int j = 0; j < p.ntheta; ++j) {
      const double c = std::fabs(std::cos(j * dth)), sn = std::fabs(std::sin(j * dth));
      const bool deg = c <= 1e-15 || sn <= 1e-15;
      const double t1 = deg ? 1.0 : std::fabs(c - sn), t2 = deg ? 1.0 : c + sn;
      const double lmax = deg ? 2.0 : 2.0 / std::max(c, sn);
      h.chord_col[j] = F4{(float)t1, (float)t2, (float)(lmax * dt * dth / 4.0), t2 > t1 ? (float)(1.0 / (t2 - t1)) : 0.f};
    }
  }
  // gridding coordinates on the quadrant (grids.py:477-494), fp64
  {
    const int hb = big / 2;
    h.qw_pitch = hb + 1;
    h.grid_q.assign((size_t)hb * h.qw_pitch * 2, 0u);
    const int nsig = h.m_need, nray = h.nray;
    const double dphi = 2.0 * kPi / nray;
    const int nthreads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int tid = 0; tid < nthreads; ++tid) {
      pool.emplace_back([&, tid]() {
        for (int ky = tid; ky < hb; ky += nthreads) {
          const double wy = (kPi * (double)ky) * (h.dw / kPi);
          for (int qx = 0; qx <= hb; ++qx) {
            const double wx = (kPi * (double)qx) * (h.dw / kPi);
            const double fi = std::min(std::hypot(wx, wy) / h.dsigma, nsig - 1.0);
            double th = std::atan2(wy, wx);
            if (th < 0) th += 2.0 * kPi;
            const double fj = th / dphi;
            uint32_t* e = &h.grid_q[((size_t)ky * h.qw_pitch + qx) * 2];
            e[0] = pack_coord(fi);
            e[1] = pack_coord(fj);
          }
        }
      });
    }
    for (auto& t : pool) t.join();
  }
  auto pow2_at_least = [](int v) { int q = 1; while (q < v) q <<= 1; return q; };
  const bool L_direct = is_pow2(h.L) && h.L >= 512 && h.L <= 8192;
  const bool big_direct = is_pow2(big) && big >= 128 && big <= 4096;
  if (!L_direct) h.mb_L = std::max(512, pow2_at_least(2 * h.L));
  if (!big_direct) h.mb_big = std::max(256, pow2_at_least(2 * big));
  h.supported = (L_direct || h.mb_L <= 8192) && (big_direct || h.mb_big <= 8192) &&
                h.m_need < 8192 && h.nray / 4 + 1 < 8192 &&  // 13-bit gridding indices
                (nt % 2) == 0 && (!p.filter || h.M <= 4096);
  if (h.supported && h.mb_L) bluestein_tables(h.L, h.mb_L, false, h.chirp_L, h.bhat_L);
  if (h.supported && h.mb_big) bluestein_tables(big, h.mb_big, true, h.chirp_big, h.bhat_big);
  return "";
}

}  // namespace lpbp
