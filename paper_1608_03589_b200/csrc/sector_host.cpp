// fp64 host construction of the sector backprojection tables.  Every formula
// restates /root/reference/pkg/src/fastbp/logpolar.py:153-299 (and radon.py:137-158).
#include "sector_host.h"

#include <cmath>
#include <cstdio>

#include "plan_host.h"

namespace lpbp {
namespace {

constexpr double kPi = 3.14159265358979323846;

// |theta - center| folded to [0, pi/2] modulo pi (logpolar.py:186-188); Python's
// float % has the sign of the divisor, so fold into [0, pi) first.
double angular_distance_mod_pi(double theta, double center) {
  double d = std::fmod(theta - center + kPi / 2.0, kPi);
  if (d < 0) d += kPi;
  return std::fabs(d - kPi / 2.0);
}

}  // namespace

std::string build_sector_set(int nt, int ntheta, int n_out, const std::vector<SectorSpec>& sectors,
                             SectorSetHost& out) {
  // argument checks in the reference's order (logpolar.py:218-227)
  if (n_out < 2) return "n_out must be >= 2";
  if (sectors.empty()) return "at least one sector is required";
  for (const auto& s : sectors) {
    if (!(0.0 < s.beta && s.beta <= kPi / 2.0)) return "sector half-width beta must lie in (0, pi/2]";
    if (!(0.0 < s.a_r && s.a_r < 0.5)) return "sector rescale a_r must lie in (0, 1/2)";
  }
  if (nt < 4 || ntheta < 1) return "sinogram must have nt >= 4 and ntheta >= 1";
  out = SectorSetHost{};
  out.nt = nt;
  out.ntheta = ntheta;
  out.n = n_out;
  const int ns = nt / 2;
  const double dtheta = kPi / ntheta;
  const double dt = 2.0 / nt;
  const double ext = 2.0 * dtheta;

  // extended masks and coverage (logpolar.py:238-246)
  std::vector<std::vector<char>> mask(sectors.size(), std::vector<char>(ntheta, 0));
  out.coverage.assign(ntheta, 0.0);
  for (size_t q = 0; q < sectors.size(); ++q) {
    const double center = sectors[q].theta0 + sectors[q].beta;
    for (int j = 0; j < ntheta; ++j) {
      const double theta = j * dtheta;
      if (angular_distance_mod_pi(theta, center) <= sectors[q].beta + ext + 1e-12) {
        mask[q][j] = 1;
        out.coverage[j] += 1.0;
      }
    }
  }
  for (int j = 0; j < ntheta; ++j) {
    if (out.coverage[j] == 0.0) {
      char buf[128];
      std::snprintf(buf, sizeof buf, "sectors do not cover the angle range: theta = %.4f uncovered", j * dtheta);
      return buf;
    }
  }

  for (size_t q = 0; q < sectors.size(); ++q) {
    const SectorSpec& sp = sectors[q];
    SectorHost S;
    S.spec = sp;
    const double center = sp.theta0 + sp.beta;
    S.jc = (int)std::nearbyint(center / dtheta);  // Python round(): half to even, as nearbyint in the default mode
    S.theta_c = S.jc * dtheta;
    // mesh depth (logpolar.py:272-283)
    S.support_min = (1.0 - sp.a_r) * std::cos(std::min(sp.beta + ext, kPi / 2.0)) - sp.a_r;
    if (S.support_min > 0.05)
      S.rho0 = std::min(std::log(S.support_min), std::log(1.0 - 2.0 * sp.a_r)) - 0.2;
    else
      S.rho0 = std::log(sp.a_r) + adaptive_rho0(n_out, n_out);
    std::string err = mesh_for(ns, S.rho0, 0, S.nrho);
    if (!err.empty()) return err;

    // working-frame columns: roll by jc with the t-flip past pi, weights, shift offsets
    int shift = S.jc % ntheta;
    if (shift < 0) shift += ntheta;
    S.cols.resize(ntheta);
    for (int j = 0; j < ntheta; ++j) {
      SectorCol c{};
      const int src = j + shift;
      c.src = src % ntheta;
      c.flip = src >= ntheta ? 1 : 0;
      const int rot = (j + S.jc % ntheta + ntheta) % ntheta;  // (arange + jc) % ntheta
      c.w = mask[q][rot] ? (float)(1.0 / out.coverage[rot]) : 0.0f;
      c.off = (1.0 - sp.a_r) * std::cos(j * dtheta);
      // reference: fi = (t_i - off + 1) / dt with t_i = -1 + i dt, i.e. i - off / dt
      const double base = -c.off / dt;
      const double fl = std::floor(base);
      c.d = (int32_t)fl;
      c.w2 = (float)(base - fl);
      S.cols[j] = c;
    }
    // compacted columns: nonzero weights form the cyclic block [ntheta - a, ntheta) u [0, b]
    {
      int b = -1, a = 0;
      while (b + 1 < ntheta && S.cols[b + 1].w != 0.f) ++b;
      while (a < ntheta - (b + 1) && S.cols[ntheta - 1 - a].w != 0.f) ++a;
      int nz = 0;
      for (const auto& c : S.cols) nz += c.w != 0.f;
      const int lo = b + 1, W = a + lo;
      const int wpad = (W + 3) / 4 * 4;
      if (nz == W && wpad < ntheta) {  // one cyclic block, narrower than the row: compact it
        S.lo = lo;
        S.wpad = wpad;
        S.ccols.assign(wpad, SectorCol{});  // padding columns: weight 0, written as zeros
        for (int w = 0; w < lo; ++w) S.ccols[w] = S.cols[w];
        for (int w = 0; w < a; ++w) S.ccols[wpad - a + w] = S.cols[ntheta - a + w];
      } else {  // wide or split sectors: full width
        S.lo = ntheta;
        S.wpad = ntheta;
        S.ccols = S.cols;
      }
    }
    // shrunk support rows: fi = (t_k / a_r + 1) / dt
    S.rows.resize(nt);
    S.klo = 0;
    S.khi = -1;
    for (int k = 0; k < nt; ++k) {
      const double t = -1.0 + k * dt;
      const double fi = (t / sp.a_r + 1.0) / dt;
      const double fl = std::floor(fi);
      SectorRow r{};
      r.k1 = (fl < -2.0) ? -2 : (fl > nt + 1.0 ? nt + 1 : (int32_t)fl);  // outside: both taps read zero
      r.w1 = (float)(fi - fl);
      S.rows[k] = r;
      if (r.k1 + 1 >= 0 && r.k1 < nt) {  // at least one tap inside the sinogram
        if (S.khi < S.klo) S.klo = k;
        S.khi = k;
      }
    }
    out.sec.push_back(std::move(S));
  }
  return "";
}

}  // namespace lpbp
