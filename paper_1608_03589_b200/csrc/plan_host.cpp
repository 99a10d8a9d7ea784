// fp64 host construction of plan tables.  See plan_host.h.
#include "plan_host.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <thread>

namespace lpbp {

namespace {

using cd = std::complex<double>;
constexpr double kPi = 3.14159265358979323846;

int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// In-place iterative radix-2 complex FFT (forward, exp(-2 pi i nk/N)), fp64.
void fft_pow2(std::vector<cd>& a, const std::vector<cd>& w /* w[k] = exp(-2 pi i k/N), k < N/2 */) {
  const int n = (int)a.size();
  for (int i = 1, j = 0; i < n; ++i) {
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (int len = 2; len <= n; len <<= 1) {
    const int step = n / len;
    for (int i = 0; i < n; i += len) {
      for (int k = 0; k < len / 2; ++k) {
        const cd u = a[i + k], v = a[i + k + len / 2] * w[k * step];
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
    }
  }
}

// Linear-interpolation tap of fastbp.grids._lerp_axis0 (grids.py:255-269):
//   value = [0<=i0<n] v[i0] (1-w) + [0<=i0+1<n] v[i0+1] w,  i0 = floor(f), w = f - i0
// re-expressed as (base, w0, w1) over rows base, base+1 with base in [0, n-2]
// and out-of-range terms folded to zero weight.
void lerp_tap(double f, int n, int32_t& base, double& w0, double& w1) {
  const double fl = std::floor(f);
  const long long i0 = (long long)fl;
  const double w = f - fl;
  const double a0 = (i0 >= 0 && i0 < n) ? (1.0 - w) : 0.0;       // weight of row i0
  const double a1 = (i0 + 1 >= 0 && i0 + 1 < n) ? w : 0.0;        // weight of row i0+1
  if (i0 >= 0 && i0 <= n - 2) {
    base = (int32_t)i0; w0 = a0; w1 = a1;
  } else if (i0 == n - 1) {
    base = n - 2; w0 = 0.0; w1 = a0;
  } else if (i0 == -1) {
    base = 0; w0 = a1; w1 = 0.0;
  } else {
    base = i0 < 0 ? 0 : n - 2; w0 = 0.0; w1 = 0.0;
  }
}

}  // namespace

void lerp_tap_public(double f, int n, int32_t& base, double& w0, double& w1) { lerp_tap(f, n, base, w0, w1); }

void bluestein_tables(int len, int MB, bool inverse, std::vector<F2>& chirp, std::vector<F2>& bhat) {
  // c[k] = exp(-i pi k^2 / len) with exact phase reduction; filter b[j] = conj c[|j|] (forward)
  // or c[|j|] (inverse) for |j| < len on the MB-point circle; bhat = FFT_MB(b) / MB
  std::vector<cd> c(len);
  chirp.resize(len);
  for (int k = 0; k < len; ++k) {
    const long long q = ((long long)k * k) % (2LL * len);
    c[k] = std::polar(1.0, -kPi * (double)q / len);
    chirp[k] = F2{(float)c[k].real(), (float)c[k].imag()};
  }
  std::vector<cd> wM(MB / 2);
  for (int k = 0; k < MB / 2; ++k) wM[k] = std::polar(1.0, -2.0 * kPi * (double)k / MB);
  std::vector<cd> b(MB, cd(0, 0));
  for (int j = 0; j < len; ++j) {
    const cd v = inverse ? c[j] : std::conj(c[j]);
    b[j] = v;
    if (j) b[MB - j] = v;
  }
  fft_pow2(b, wM);
  bhat.resize(MB);
  for (int q = 0; q < MB; ++q) bhat[q] = F2{(float)(b[q].real() / MB), (float)(b[q].imag() / MB)};
}

void build_bands(HostPlan& h, int band_rows) {
  // Steps of band_rows (2 or 4) rows for the streaming fused readout: step b owns
  // the pixels with i0 in [r0 - 1, r0 + band_rows - 1), r0 = row_min + band_rows*b,
  // so its taps are the previous step's last row (still resident) and its own.
  const size_t nqq = (size_t)h.nq * h.nq;
  int rmin = h.nrho;
  for (size_t e = 0; e < nqq; ++e)
    if (h.qidx[e] != 0xFFFFFFFFu) rmin = std::min(rmin, (int)(h.qidx[e] & 0xFFFFu));
  if (rmin == h.nrho) rmin = 0;
  rmin &= ~3;  // steps start at multiples of 4 rows: TMA box rows start 16/32-B aligned
  h.band_rows = band_rows;
  h.row_min = rmin;
  h.nbands = (h.nrho - rmin) / band_rows + 1;
  std::vector<std::vector<uint32_t>> valid(h.nbands), zero(h.nbands);
  std::vector<uint32_t> zeros;  // raster order
  h.band_need.assign(h.nbands, 0);
  for (size_t e = 0; e < nqq; ++e) {
    const uint32_t q = h.qidx[e];
    if (q == 0xFFFFFFFFu) {
      zeros.push_back((uint32_t)e | 0x80000000u);
    } else {
      const int i0 = (int)(q & 0xFFFFu), i1 = std::min(i0 + 1, h.nrho - 1);
      const int b = (i0 + 1 - rmin) / band_rows;
      valid[b].push_back((uint32_t)e);
      h.band_need[(i0 - rmin) / band_rows] = 1;  // the bands holding the two tapped rows
      h.band_need[(i1 - rmin) / band_rows] = 1;
    }
  }
  // zero-writes: contiguous raster chunks dealt to the needed bands, so they fill whole sectors
  std::vector<int> needed;
  for (int b = 0; b < h.nbands; ++b)
    if (h.band_need[b]) needed.push_back(b);
  if (needed.empty() && h.nbands > 0) {  // no pixel in range at all: band 0 writes the zeros
    h.band_need[0] = 1;
    needed.push_back(0);
  }
  for (size_t k = 0; k < needed.size(); ++k) {
    const size_t lo = zeros.size() * k / needed.size(), hi = zeros.size() * (k + 1) / needed.size();
    zero[needed[k]].assign(zeros.begin() + lo, zeros.begin() + hi);
  }
  h.band_entries.clear();
  h.band_off.assign(h.nbands + 1, 0);
  for (int b = 0; b < h.nbands; ++b) {
    h.band_off[b] = (uint32_t)h.band_entries.size();
    h.band_entries.insert(h.band_entries.end(), valid[b].begin(), valid[b].end());
    h.band_entries.insert(h.band_entries.end(), zero[b].begin(), zero[b].end());
  }
  h.band_off[h.nbands] = (uint32_t)h.band_entries.size();
  // Work units, built from the outermost band inward.  A needed band costs one transform step plus its
  // pixel entries (kEntryEquiv entries ~ one step); a unit closes once its cost reaches kUnitCost or it
  // spans kMaxUnitBands bands.  Pixel-heavy outer bands thus come in short units (the heaviest
  // unit bounds the kernel: units are taken dynamically, largest-first), the sparse inner bands in long
  // ones (each unit re-transforms the band before it for its carried row).
  {
    // measured on B200 at 2048^2 with the warp-specialised kernel (E0 x cost target in {2000, 3000, 5000} x
    // {4, 6, 8, 12}: 28.7 - 32.5 us/slice)
    const double kEntryEquiv = 2000.0, kUnitCost = 8.0;
    std::vector<std::pair<uint32_t, uint32_t>> us;
    int hi = h.nbands;
    while (hi > 0) {
      int lo = hi;
      double cost = 0.0;
      while (lo > 0 && hi - lo < kMaxUnitBands && cost < kUnitCost) {
        --lo;
        cost += (h.band_need[lo] ? 1.0 : 0.0) + (double)(h.band_off[lo + 1] - h.band_off[lo]) / kEntryEquiv;
      }
      us.push_back({(uint32_t)lo, (uint32_t)hi});
      hi = lo;
    }
    h.nunits = (int)us.size();
    h.units.resize(2 * us.size());
    for (size_t u = 0; u < us.size(); ++u) {
      h.units[2 * u] = us[u].first;
      h.units[2 * u + 1] = us[u].second;
    }
  }
  h.row_need.assign(((size_t)h.nrho_pad + 31) / 32 + 1, 0u);
  for (int b = 0; b < h.nbands; ++b)
    if (h.band_need[b])
      for (int r = rmin + band_rows * b; r < rmin + band_rows * (b + 1) && r < h.nrho_pad; ++r)
        h.row_need[(size_t)r >> 5] |= 1u << (r & 31);
  h.row_end = rmin + band_rows * h.nbands;
  h.rowmap_cp.assign((size_t)h.row_end, -1);
  h.rowmap_id.assign((size_t)h.row_end, -1);
  h.band_row_cp.assign((size_t)h.nbands, 0u);
  h.band_row_id.assign((size_t)h.nbands, 0u);
  {
    int cpos = 0;
    for (int b = 0; b < h.nbands; ++b) {
      if (!h.band_need[b]) continue;
      const int r0 = rmin + band_rows * b;
      h.band_row_cp[b] = (uint32_t)cpos + 1u;
      h.band_row_id[b] = (uint32_t)r0 + 1u;
      for (int j = 0; j < band_rows; ++j) {
        h.rowmap_cp[(size_t)r0 + j] = cpos + j;
        h.rowmap_id[(size_t)r0 + j] = r0 + j;
      }
      cpos += band_rows;
    }
  }
  h.band_packed.resize(h.band_entries.size() * 4);
  for (size_t e = 0; e < h.band_entries.size(); ++e) {
    const uint32_t ent = h.band_entries[e];
    const uint32_t qq = ent & 0x7FFFFFFFu;
    uint32_t wi = 0, wj = 0;
    std::memcpy(&wi, &h.qw[qq].x, 4);
    std::memcpy(&wj, &h.qw[qq].y, 4);
    // qy | qx << 15 | zero flag << 31: the device reads the quadrant position without a division
    const uint32_t qy = qq / (uint32_t)h.nq, qx = qq % (uint32_t)h.nq;
    h.band_packed[4 * e + 0] = qy | (qx << 15) | (ent & 0x80000000u);
    h.band_packed[4 * e + 1] = h.qidx[qq];
    h.band_packed[4 * e + 2] = wi;
    h.band_packed[4 * e + 3] = wj;
  }
}

double adaptive_rho0(int nx, int ny) { return std::log(std::min(2.0 / nx, 2.0 / ny)) - std::log(2.0); }

std::string mesh_for(int ns, double rho0, int nrho_in, int& nrho_out) {
  const double ds = 2.0 / ns;
  int nrho = nrho_in;
  if (nrho <= 0) nrho = std::max(2, (int)std::ceil(-rho0 / -std::log1p(-ds)));
  const double drho = -rho0 / nrho;
  if (1.0 - std::exp(-drho) > ds * (1.0 + 1e-9)) {
    char buf[256];
    std::snprintf(buf, sizeof buf,
                  "log-polar mesh too coarse: largest radial step %.3e exceeds the sinogram step %.3e",
                  1.0 - std::exp(-drho), ds);
    return buf;
  }
  nrho_out = nrho;
  return "";
}

int next_fast_len(int target) {
  if (target <= 1) return 1;
  for (int v = target;; ++v) {
    int r = v;
    for (int p : {2, 3, 5, 7, 11})
      while (r % p == 0) r /= p;
    if (r == 1) return v;
  }
}

// Ramp / Tikhonov filter (filtering.py:54-70).  The reference multiplies by resp
// on an Lr = next_fast_len(8 nt) grid; that is a convolution with the real even
// taps h[d] = (1/Lr) sum_k resp_k cos(2 pi k d / Lr), |d| < nt.  The same taps
// periodised on M = pow2 >= 2 nt give an exact circular embedding; the table is
// their M-point spectrum / M.
void build_ramp_taps(int nt, double lam, double cutoff, int& M_out, int& Lr_out, std::vector<float>& ramp) {
  const double dt = 2.0 / nt;
  const int Lr = next_fast_len(8 * nt);
  Lr_out = Lr;
  const double val = 1.0 / (Lr * dt);  // numpy.fft.fftfreq
  const double cut = cutoff * kPi / dt;
  std::vector<double> resp(Lr);
  const int Npos = (Lr - 1) / 2 + 1;
  for (int k = 0; k < Lr; ++k) {
    const long long f = k < Npos ? k : (long long)k - Lr;
    const double sigma = 2.0 * kPi * ((double)f * val);
    const double a = std::fabs(sigma);
    resp[k] = (std::fabs(sigma) > cut) ? 0.0 : a / (1.0 + lam * a);
  }
  std::vector<double> cosr(Lr);
  for (int q = 0; q < Lr; ++q) cosr[q] = std::cos(2.0 * kPi * (double)q / Lr);
  std::vector<double> taps(nt);
  for (int d = 0; d < nt; ++d) {
    double acc = 0.0;
    long long ph = 0;
    for (int k = 0; k < Lr; ++k) {
      acc += resp[k] * cosr[ph];
      ph += d;
      if (ph >= Lr) ph -= Lr;
    }
    taps[d] = acc / Lr;
  }
  M_out = std::max(512, next_pow2(2 * nt));  // any M >= 2 nt - 1 embeds the Toeplitz filter
  const int M = M_out;
  std::vector<double> cosm(M);
  for (int q = 0; q < M; ++q) cosm[q] = std::cos(2.0 * kPi * (double)q / M);
  ramp.resize(M);
  for (int kap = 0; kap < M; ++kap) {
    double acc = taps[0];
    long long ph = 0;
    for (int d = 1; d < nt; ++d) {
      ph += kap;
      if (ph >= M) ph -= M;
      acc += 2.0 * taps[d] * cosm[ph];
    }
    ramp[kap] = (float)(acc / M);
  }
}

std::string build_host_plan(const HostPlanParams& p, HostPlan& h) {
  if (p.nt < 2 || p.ntheta < 1) return "nt must be >= 2 and ntheta >= 1";
  if (p.n < 2) return "n_out must be >= 2";
  if (p.has_rho0 && !(p.rho0 < 0)) return "rho0 must be negative";
  if (p.nrho != 0 && p.nrho < 2) return "nrho must be >= 2";
  if (p.filter) {
    if (p.lam < 0) return "lambda must be >= 0";
    if (!(p.cutoff > 0.0 && p.cutoff <= 1.0)) return "cutoff must lie in (0, 1]";
  }
  h.nt = p.nt;
  h.ntheta = p.ntheta;
  h.n = p.n;
  h.filter = p.filter;
  h.ns = p.nt / 2;  // logpolar.py:131
  if (h.ns < 2) return "ns must be >= 2";
  h.nphi = 2 * p.ntheta;  // grids.py:303
  h.nh = h.nphi / 2 + 1;
  h.rho0 = p.has_rho0 ? p.rho0 : adaptive_rho0(p.n, p.n);  // logpolar.py:132
  std::string err = mesh_for(h.ns, h.rho0, p.nrho, h.nrho);  // logpolar.py:133
  if (!err.empty()) return err;
  h.drho = -h.rho0 / h.nrho;              // grids.py:183
  h.dphi = 2.0 * kPi / h.nphi;            // grids.py:187
  h.nrho_pad = (h.nrho + 15) / 16 * 16;
  h.out_scale = p.filter ? 1.0 / (2.0 * kPi) : 1.0;  // filtering.py:27,98
  const int nt = p.nt, ns = h.ns, nrho = h.nrho, nphi = h.nphi, nh = h.nh;
  const double dt = 2.0 / nt;  // grids.py:112

  // --- semi-polar taps (grids.py:290-311): s_k = k/(ns-1), f = (+-s + 1)/dt
  h.ab.resize(ns);
  h.wab.resize(ns);
  for (int k = 0; k < ns; ++k) {
    const double s = (double)k / (ns - 1.0);
    int32_t a, b;
    double wa0, wa1, wb0, wb1;
    lerp_tap((s + 1.0) / dt, nt, a, wa0, wa1);
    lerp_tap((-s + 1.0) / dt, nt, b, wb0, wb1);
    h.ab[k] = I2{a, b};
    h.wab[k] = F4{(float)wa0, (float)wa1, (float)wb0, (float)wb1};
  }
  // packed semi-polar taps for K3 (8 bytes per s-row instead of 24): row floor(f) with weights
  // (1 - w, w); f = (+-s + 1)/dt lies in [0, nt], so rows nt and nt + 1 (zero in K3's column
  // buffer) stand in for the reference's out-of-range zeros; w keeps 19 fractional bits
  if (nt > 8191) return "nt too large for the packed semi-polar taps (nt < 8192)";
  h.abw.resize(2 * (size_t)ns);
  for (int k = 0; k < ns; ++k) {
    const double s = (double)k / (ns - 1.0);
    for (int side = 0; side < 2; ++side) {
      const double f = ((side ? -s : s) + 1.0) / dt;
      const double fl = std::floor(f);
      long long wq = std::llround((f - fl) * 524288.0);
      if (wq > 524287) wq = 524287;
      h.abw[2 * (size_t)k + side] = (uint32_t)fl | ((uint32_t)wq << 13);
    }
  }
  // --- K2p tiles: 4 semi-polar rows, the sinogram rows their non-zero taps touch on each side
  h.pmix = 0;
  h.ptile.clear();
  h.ploc.clear();
  if (ns % 4 == 0) {
    constexpr int kSide = 5;  // rows per side a K2p input slot holds
    bool ok = true;
    h.ptile.assign((size_t)ns, 0);
    h.ploc.assign((size_t)ns, 0u);
    for (int k0 = 0; k0 < ns && ok; k0 += 4) {
      int lo[2] = {nt, nt}, hi[2] = {-1, -1};
      for (int k = k0; k < k0 + 4; ++k) {
        const int base[2] = {h.ab[k].x, h.ab[k].y};
        const float w[4] = {h.wab[k].x, h.wab[k].y, h.wab[k].z, h.wab[k].w};
        for (int side = 0; side < 2; ++side)
          for (int j = 0; j < 2; ++j)
            if (w[2 * side + j] != 0.f) {
              lo[side] = std::min(lo[side], base[side] + j);
              hi[side] = std::max(hi[side], base[side] + j);
            }
      }
      for (int side = 0; side < 2; ++side) {
        if (hi[side] < 0) lo[side] = hi[side] = 0;  // no tap on this side: one (unused) row
        if (hi[side] - lo[side] + 1 > kSide || lo[side] < 0 || hi[side] >= nt) ok = false;
        h.ptile[(size_t)k0 + 2 * side] = lo[side];
        h.ptile[(size_t)k0 + 2 * side + 1] = hi[side] - lo[side] + 1;
      }
      for (int k = k0; k < k0 + 4 && ok; ++k) {
        const int base[2] = {h.ab[k].x, h.ab[k].y};
        const float w[4] = {h.wab[k].x, h.wab[k].y, h.wab[k].z, h.wab[k].w};
        uint32_t loc = 0;
        for (int side = 0; side < 2; ++side)
          for (int j = 0; j < 2; ++j) {
            const int l = w[2 * side + j] != 0.f ? base[side] + j - lo[side] : 0;
            loc |= (uint32_t)l << (4 * (2 * side + j));
          }
        h.ploc[k] = loc;
      }
    }
    h.pmix = ok ? 1 : 0;
  }
  // --- log-polar taps (grids.py:332-347): rho_i = rho0 + (i+1) drho, f = e^rho (ns-1)
  h.ki.resize(nrho);
  h.wi.resize(nrho);
  for (int i = 0; i < nrho; ++i) {
    const double rho = h.rho0 + (double)(i + 1) * h.drho;
    int32_t k;
    double w0, w1;
    lerp_tap(std::exp(rho) * (ns - 1.0), ns, k, w0, w1);
    h.ki[i] = k;
    h.wi[i] = F2{(float)w0, (float)w1};
  }
  // packed taps for K3's shared-memory copy: f = e^rho (ns-1) lies in (0, ns-1], so
  // lerp_tap always gives w0 = 1 - w1 here; w1 keeps 20 fractional bits (error <= 2^-21)
  if (ns - 1 > 0x7FF) return "ns too large for the packed log-polar taps (ns <= 2048)";
  h.kw.resize(nrho);
  for (int i = 0; i < nrho; ++i) {
    const long long wq = std::llround((double)h.wi[i].y * 1048576.0);
    h.kw[i] = (uint32_t)h.ki[i] | ((uint32_t)wq << 11);
  }

  // --- kernel support (logpolar.py:66-81, rolled by -nphi/2 at :110):
  // cell (k, l) holds 1/drho iff |e^{k drho} cos(theta_j) - 1| <= drho with
  // theta_j = -pi + j*2pi/nphi and j = (l + nphi/2) mod nphi.
  std::vector<double> costab(nphi);
  for (int j = 0; j < nphi; ++j) costab[j] = std::cos(-kPi + (double)j * (2.0 * kPi / nphi));
  std::vector<std::vector<int>> cells(nrho);
  h.kmax = 0;
  h.nnz = 0;
  h.cell_k.clear();
  h.cell_l.clear();
  for (int k = 0; k < nrho; ++k) {
    const double e = std::exp((double)k * h.drho);
    for (int l = 0; l < nphi; ++l) {
      const int j = (l + nphi / 2) % nphi;
      if (std::fabs(e * costab[j] - 1.0) <= h.drho) {
        cells[k].push_back(l);
        h.cell_k.push_back(k);
        h.cell_l.push_back(l);
        h.kmax = k;
        ++h.nnz;
      }
    }
  }
  h.L = std::max(512, next_pow2(nrho + h.kmax));
  const int L = h.L;

  // --- kernel spectrum Khat[m][kappa] = FFT_L over k of KPhi[k][m], with
  // KPhi[k][m] = sum_{l in cells_k} (1/drho) e^{-2 pi i l m / nphi} and the
  // output scale LOGPOLAR_SCALE * drho * dphi (logpolar.py:47,117) plus the
  // unnormalised inverse FFTs' 1/(L * nphi) folded in.
  std::vector<cd> ctab(nphi);
  for (int q = 0; q < nphi; ++q) ctab[q] = std::polar(1.0, -2.0 * kPi * (double)q / nphi);
  std::vector<cd> wL(L / 2);
  for (int k = 0; k < L / 2; ++k) wL[k] = std::polar(1.0, -2.0 * kPi * (double)k / L);
  const double kscale = 0.5 * h.drho * h.dphi / ((double)L * nphi) / h.drho;  // cell value 1/drho
  h.khat.assign((size_t)nh * L, F2{0, 0});
  {
    const int nthreads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int tid = 0; tid < nthreads; ++tid) {
      pool.emplace_back([&, tid]() {
        std::vector<cd> col(L);
        for (int m = tid; m < nh; m += nthreads) {
          std::fill(col.begin(), col.end(), cd(0, 0));
          for (int k = 0; k <= h.kmax; ++k) {
            cd acc(0, 0);
            for (int l : cells[k]) acc += ctab[(int)(((long long)l * m) % nphi)];
            col[k] = acc;
          }
          fft_pow2(col, wL);
          F2* dst = h.khat.data() + (size_t)m * L;
          for (int q = 0; q < L; ++q) dst[q] = F2{(float)(col[q].real() * kscale), (float)(col[q].imag() * kscale)};
        }
      });
    }
    for (auto& t : pool) t.join();
  }

  // (FFT twiddle tables are generated on the device from the compile-time radix plans.)

  // --- generic-size path: Bluestein chirps for the length-nphi DFTs
  const bool pow2_phi = (nphi & (nphi - 1)) == 0 && nphi >= 512 && nphi <= 4096;
  h.generic = !pow2_phi || (nt % 4) != 0 || (p.filter && (p.ntheta % 8) != 0);
  if (h.generic) {
    h.MB = std::max(512, next_pow2(2 * nphi));
    const int MB = h.MB;
    h.chirp.resize(nphi);
    std::vector<cd> c(nphi);
    for (int k = 0; k < nphi; ++k) {
      const long long q = ((long long)k * k) % (2LL * nphi);  // exact phase reduction
      c[k] = std::polar(1.0, -kPi * (double)q / nphi);
      h.chirp[k] = F2{(float)c[k].real(), (float)c[k].imag()};
    }
    std::vector<cd> wM(MB / 2);
    for (int k = 0; k < MB / 2; ++k) wM[k] = std::polar(1.0, -2.0 * kPi * (double)k / MB);
    for (int dir = 0; dir < 2; ++dir) {  // forward: b[j] = conj c[|j|]; inverse: b[j] = c[|j|]
      std::vector<cd> b(MB, cd(0, 0));
      for (int j = 0; j < nphi; ++j) {
        const cd v = dir == 0 ? std::conj(c[j]) : c[j];
        b[j] = v;
        if (j) b[MB - j] = v;
      }
      fft_pow2(b, wM);
      auto& dst = dir == 0 ? h.bhat_f : h.bhat_i;
      dst.resize(MB);
      for (int q = 0; q < MB; ++q) dst[q] = F2{(float)(b[q].real() / MB), (float)(b[q].imag() / MB)};
    }
  }

  // --- ramp / Tikhonov filter (filtering.py:54-70)
  if (p.filter) build_ramp_taps(nt, p.lam, p.cutoff, h.M, h.ramp_len_ref, h.ramp);

  // --- readout quadrant table (grids.py:399-443) at x, y >= 0; the device
  // reflects phi for the other quadrants.
  const int c = p.n / 2;
  h.nq = p.n - c;
  h.qidx.assign((size_t)h.nq * h.nq, 0xFFFFFFFFu);
  h.qw.assign((size_t)h.nq * h.nq, F2{0, 0});
  for (int qy = 0; qy < h.nq; ++qy) {
    const double y = -1.0 + ((double)(c + qy) + 0.5) * (2.0 / p.n);
    for (int qx = 0; qx < h.nq; ++qx) {
      const double x = -1.0 + ((double)(c + qx) + 0.5) * (2.0 / p.n);
      const double r = std::hypot(x, y);
      if (!(r <= 1.0 && r > 0.0)) continue;
      const double rho = std::log(r);
      if (!(rho >= h.rho0)) continue;
      double fi = (rho - h.rho0) / h.drho - 1.0;
      if (fi >= -1.0 && fi < 0.0) fi = 0.0;
      fi = std::min(std::max(fi, 0.0), (double)(nrho - 1));
      double phi = std::fmod(std::atan2(y, x), 2.0 * kPi);
      if (phi < 0) phi += 2.0 * kPi;
      const double fj = phi / h.dphi;
      const double i0 = std::floor(fi), j0 = std::floor(fj);
      const int ji = ((int)j0 % nphi + nphi) % nphi;
      h.qidx[(size_t)qy * h.nq + qx] = (uint32_t)i0 | ((uint32_t)ji << 16);
      h.qw[(size_t)qy * h.nq + qx] = F2{(float)(fi - i0), (float)(fj - j0)};
    }
  }
  if (h.generic) {  // tapped row pairs; the first one (even row) bounds the rows K3 must store
    std::vector<uint8_t> need((nrho + 1) / 2, 0);
    for (const uint32_t e : h.qidx) {
      if (e == 0xFFFFFFFFu) continue;
      const int i0 = (int)(e & 0xFFFFu), i1 = std::min(i0 + 1, nrho - 1);
      need[i0 / 2] = need[i1 / 2] = 1;
    }
    h.pair_list.clear();
    for (int j = 0; j < (int)need.size(); ++j)
      if (need[j]) h.pair_list.push_back((uint32_t)j);
    h.row_min = h.pair_list.empty() ? 0 : 2 * (int)h.pair_list[0];
  }

  // --- distinct 32-byte sectors of the fp32 log-polar image read by the readout
  // taps over the whole image (reflections as on the device): the readout's
  // compulsory read traffic.
  {
    std::vector<uint8_t> hit(((size_t)nrho * nphi + 7) / 8 + 1, 0);
    auto mark = [&](int i, int j) { hit[((size_t)i * nphi + j) / 8] = 1; };
    for (int iy = 0; iy < p.n; ++iy) {
      for (int jx = 0; jx < p.n; ++jx) {
        const bool yneg = iy < c, xneg = jx < c;
        const int qy = yneg ? (p.n - 1 - iy) - c : iy - c;
        const int qx = xneg ? (p.n - 1 - jx) - c : jx - c;
        const uint32_t e = h.qidx[(size_t)qy * h.nq + qx];
        if (e == 0xFFFFFFFFu) continue;
        const float wjr = h.qw[(size_t)qy * h.nq + qx].y;
        const int i0 = (int)(e & 0xFFFFu), jr = (int)(e >> 16);
        int j0;
        if (!xneg && !yneg) j0 = jr;
        else if (xneg && yneg) j0 = nphi / 2 + jr;
        else {
          const int Q = xneg ? nphi / 2 : nphi;
          j0 = (wjr == 0.f) ? Q - jr : Q - jr - 1;
        }
        if (j0 >= nphi) j0 -= nphi;
        const int j1 = (j0 + 1 == nphi) ? 0 : j0 + 1;
        const int i1 = std::min(i0 + 1, nrho - 1);
        mark(i0, j0); mark(i0, j1); mark(i1, j0); mark(i1, j1);
      }
    }
    size_t cnt = 0;
    for (uint8_t v : hit) cnt += v;
    h.readout_sector_bytes = cnt * 32;
  }

  // --- direct backprojector angle table (reference.py:30-36)
  h.naive_cs.resize(p.ntheta);
  const double dtheta = kPi / p.ntheta;
  for (int k = 0; k < p.ntheta; ++k) {
    const double th = k * dtheta;
    h.naive_cs[k] = F2{(float)(std::cos(th) * nt / (2.0 * p.n)), (float)(std::sin(th) * nt / (2.0 * p.n))};
  }
  return "";
}

}  // namespace lpbp
