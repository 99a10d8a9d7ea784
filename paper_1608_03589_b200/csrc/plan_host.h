// Host-side (fp64) construction of the constant tables of a log-polar
// backprojection plan.  Every formula restates the fastbp reference so the
// device pipeline reproduces it; file:line citations refer to
// /root/reference/pkg/src/fastbp.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace lpbp {

struct F2 { float x, y; };
struct I2 { int32_t x, y; };
struct F4 { float x, y, z, w; };

struct HostPlanParams {
  int nt, ntheta, n;
  bool has_rho0;
  double rho0;
  int nrho;       // 0 = automatic (_mesh_for)
  bool filter;    // fbp: filter_sinogram + 1/(2 pi)
  double lam, cutoff;
};

struct HostPlan {
  // geometry
  int nt = 0, ntheta = 0, n = 0, ns = 0, nphi = 0, nh = 0, nrho = 0, nrho_pad = 0, L = 0, M = 0, nq = 0;
  int kmax = 0, nnz = 0, ramp_len_ref = 0;
  size_t readout_sector_bytes = 0;
  double rho0 = 0, drho = 0, dphi = 0, out_scale = 1;
  bool filter = false;
  // tables (uploaded to the device)
  std::vector<F2> khat, wi, qw, naive_cs;
  std::vector<float> ramp;
  std::vector<I2> ab;
  std::vector<F4> wab;
  std::vector<uint32_t> abw;  // [2 ns] packed semi-polar taps for K3: a | w1a << 13, b | w1b << 13 (rows past nt read zero)
  // K2p (row DFT of the semi-polar rows, grids.py:290-311 before logpolar.py:112): tiles of 4 semi-polar
  // rows; ptile[4 j] = {a_lo, na, b_lo, nb}: the sinogram rows [a_lo, a_lo + na) hold every non-zero
  // t >= 0 tap of rows 4j .. 4j+3 and [b_lo, b_lo + nb) every t <= 0 tap (na, nb <= 5), ploc[k] = the
  // taps' rows inside those ranges (la0 | la1 << 4 | lb0 << 8 | lb1 << 12; zero-weight taps point at
  // row 0 of the range), weights = wab[k].  pmix = 1 when every tile fits (ns % 4 == 0 too).
  int pmix = 0;
  std::vector<int32_t> ptile;
  std::vector<uint32_t> ploc;
  std::vector<int32_t> ki;
  std::vector<uint32_t> kw;  // [nrho] packed log-polar tap: ki | round(w1 * 2^20) << 11 (w0 = 1 - w1)
  std::vector<uint32_t> qidx;
  // fused inverse-DFT + readout: quads of band_rows (4) log-polar rows starting at
  // r0 = row_min + 4b (row_min even); band_entries lists the quadrant pixels (qy*nq + qx)
  // with i0 in [r0 - 1, r0 + 3) (bit 31 set = write zero), band_off[b..b+1).
  int band_rows = 0, row_min = 0, nbands = 0;
  std::vector<uint32_t> band_entries, band_off;
  // band_need[b] = 1 iff some pixel taps one of band b's rows: the fused kernel neither loads nor
  // transforms the others (~1/3 of the bands at 2048^2 lie between the discrete radii of the
  // innermost pixels); zero-writes are dealt to needed bands only
  std::vector<uint32_t> band_need;
  // fused-kernel work units: contiguous band ranges [units[2u], units[2u+1]), outermost first, cut
  // so each unit's cost (needed bands + pixel entries / unit_entry_equiv) is about unit_cost; at most
  // kMaxUnitBands bands per unit
  std::vector<uint32_t> units;
  int nunits = 0;
  // bitmap over the log-polar rows [0, nrho_pad): 1 = the row belongs to a needed band (the fused kernel
  // loads and transforms whole bands, so every row of a needed band must hold K3's output); K3 writes
  // these rows only
  std::vector<uint32_t> row_need;
  // the same as maps (see kernels.cuh DevTables): rows [0, row_end), row_end = row_min + band_rows * nbands
  int row_end = 0;
  std::vector<int32_t> rowmap_cp, rowmap_id;
  std::vector<uint32_t> band_row_cp, band_row_id;
  // self-contained 16-byte entries {qy | qx << 15 | zero flag << 31, qidx, wi bits, wj bits}
  std::vector<uint32_t> band_packed;
  // generic sizes (nphi not a power of two in [512, 4096], ...): Bluestein DFTs of
  // length nphi through MB-point convolutions, MB = pow2 >= 2 nphi
  bool generic = false;
  int MB = 0;
  // generic path (unfused inverse DFT + readout): the row pairs (2j, 2j+1) some pixel taps, ascending;
  // the inverse DFT runs over these only (a third of the rows at 2048^2 are tapped by no pixel)
  std::vector<uint32_t> pair_list;
  std::vector<F2> chirp;          // [nphi] exp(-i pi n^2 / nphi)
  std::vector<F2> bhat_f, bhat_i; // [MB] FFT_MB of the forward / inverse chirp filter, incl. 1/MB
  // kernel support (for diagnostics/tests): cells (k, l) of the rolled kernel
  std::vector<int32_t> cell_k, cell_l;
};

// Returns "" on success, else the error message (ValueError semantics).
std::string build_host_plan(const HostPlanParams& p, HostPlan& out);
// Fill band_* for bands of `band_rows` rows (needs qidx built).
constexpr int kMaxUnitBands = 24;  // the fused kernel's per-unit arrays (one lane per band + 1)
void build_bands(HostPlan& h, int band_rows);

// fastbp.grids.adaptive_rho0 (grids.py:385-391)
double adaptive_rho0(int nx, int ny);
// fastbp.logpolar._mesh_for (logpolar.py:84-97); returns "" or error message
std::string mesh_for(int ns, double rho0, int nrho_in, int& nrho_out);
// scipy.fft.next_fast_len(target) for complex transforms: smallest 11-smooth >= target
int next_fast_len(int target);
// Ramp / Tikhonov filter spectrum on the circular embedding M = pow2 >= 2 nt (filtering.py:54-70)
void build_ramp_taps(int nt, double lam, double cutoff, int& M_out, int& Lr_out, std::vector<float>& ramp);
// _lerp_axis0 tap (grids.py:255-269) as (base in [0, n-2], w0, w1), out-of-range terms weight 0
void lerp_tap_public(double f, int n, int32_t& base, double& w0, double& w1);
// Bluestein tables of a length-len DFT on an MB-point circular convolution (MB pow2 >= 2 len)
void bluestein_tables(int len, int MB, bool inverse, std::vector<F2>& chirp, std::vector<F2>& bhat);

}  // namespace lpbp
