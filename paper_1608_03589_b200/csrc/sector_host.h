// Host-side (fp64) geometry and tables of the sector (partial) log-polar
// backprojection, fastbp.logpolar.partial_backproject (logpolar.py:210-299).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace lpbp {

struct SectorSpec { double theta0, beta, a_r; };

// Per output column j of a sector's working-frame sinogram: which input column
// it reads (angles rolled by jc, logpolar.py:162-172), whether that column is
// the t-flipped copy (it wrapped past pi, :153-159), its mask/coverage weight
// (:263-268) and the shift offset (1 - a_r) cos(theta_j) (radon.py:144-147).
struct SectorCol {
  double off;
  int32_t src;
  int32_t flip;
  float w;
  // fi(i) = (t_i - off + 1) / dt = i - off / dt: floor = i + d, weight w2 constant per column
  int32_t d;
  float w2;
  float pad;
};
// Per row k of the shrunk sinogram out(t_k) = a_r g(t_k / a_r)  (logpolar.py:175-179):
// lerp base row and weight of fi = (t_k / a_r + 1) / dt.
struct SectorRow {
  int32_t k1;
  float w1;
};

struct SectorHost {
  SectorSpec spec{};
  int jc = 0;               // centre snapped to the angle grid
  double theta_c = 0;       // jc * dtheta
  double support_min = 0;   // logpolar.py:278
  double rho0 = 0;          // sector mesh depth (logpolar.py:279-283)
  int nrho = 0;             // _mesh_for(ns, rho0, None)
  std::vector<SectorCol> cols;  // [ntheta] the reference's working-frame columns
  // Compacted storage of the working sinogram for the log-polar stage: the nonzero-weight
  // columns form the cyclic block [0, lo) u [ntheta - hi, ntheta); rows are stored as
  // [lo leading columns][zero padding][hi trailing columns], wpad wide (multiple of 4).  The
  // row DFT maps the trailing part back to the row's end, so the values are exactly the
  // reference's; only the zero columns are never written or read.
  int lo = 0, wpad = 0;
  std::vector<SectorCol> ccols;  // [wpad]
  std::vector<SectorRow> rows;  // [nt]
  int klo = 0, khi = -1;        // rows k of the shrunk sinogram that can be nonzero (a tap in [0, nt))
};

struct SectorSetHost {
  int nt = 0, ntheta = 0, n = 0;
  std::vector<SectorHost> sec;
  std::vector<double> coverage;  // [ntheta]
};

// Validates like the reference (ValueError messages verbatim) and builds every
// sector's geometry and tables.  Returns "" on success.
std::string build_sector_set(int nt, int ntheta, int n_out, const std::vector<SectorSpec>& sectors,
                             SectorSetHost& out);

}  // namespace lpbp
