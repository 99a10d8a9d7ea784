// Sector (partial) backprojection kernels: launchers and device-side tables.
#pragma once
#include <cuda_runtime.h>

#include "sector_host.h"

namespace lpbp {

// One sector as the readout sees it (device array of nsec entries).
struct SectorDev {
  const float* lp;        // [batch][nrho][nphi] convolved log-polar images of this sector
  long long lp_slice;     // nrho * nphi
  int nrho;
  int pad;
  double rho0, drho;      // sector mesh
  double ct, st, a_r;     // working frame: x_w = (1 - a_r, 0) + a_r R(-theta_c) x
  float inv_a;
  float pad2;
};

constexpr int kSectorGroup = 16;  // slices per readout thread (coordinates computed once per group)
constexpr int kMaxSectors = 32;   // sectors per plan (the readout takes them as one kernel argument)

struct SectorArgs {
  SectorDev s[kMaxSectors];
};

// out [batch][nt][ntheta] (ntheta = output columns, the cols table's length); g [batch][nt][nin]
cudaError_t launch_sector_prep(const float* g, float* out, int nt, int ntheta, int nin, int batch,
                               const SectorCol* cols, const SectorRow* rows, double a_r, int klo, int khi,
                               cudaStream_t s);
cudaError_t launch_sector_readout(const SectorArgs& secs, int nsec, float* img, int n, int nphi, int batch,
                                  cudaStream_t s);

}  // namespace lpbp
