// Launch wrappers for the log-polar backprojection kernels (sm_100a).
// Layouts (all C-contiguous, fp32 / complex64 as float2):
//   sinogram  g  [B][nt][ntheta]              (fastbp Sinogram.values, t outer)
//   row spectra G [B][nh][nt]    nh = nphi/2+1 (phi-frequency major, t contiguous)
//   semi-polar row spectra P [B][nh][ns]      (d.pmix plans: K2p's output instead of G)
//   conv spectra Y [B][nh][nrho_pad]          (phi-frequency major, rho contiguous)
//   log-polar  lp [B][nrho][nphi]             (fastbp LogPolarImage.values)
//   image     img [B][n][n]                   (fastbp CartesianImage.values, y outer)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lpbp {

struct DevTables {
  // pass-twiddle tables (fft.cuh TwTable layout) of size
  const float2* tw_phi;   // N = nphi
  const float2* tw_rho;   // N = L
  const float2* tw_ramp;  // N = M = 2 nt (FBP only)
  const float* ramp;      // [M] real even filter response incl. 1/M (FBP only)
  const int2* ab;         // [ns] t-rows (a_k, b_k) of the semi-polar lerp
  const float4* wab;      // [ns] weights (wa0, wa1, wb0, wb1)
  const uint2* abw;       // [ns] packed (a | w1a << 13, b | w1b << 13), plan_host abw
  const int32_t* ptile;   // [ns] K2p tiles: {a_lo, na, b_lo, nb} per 4 semi-polar rows (plan_host ptile)
  const uint32_t* ploc;   // [ns] K2p tap rows inside the tile's ranges (plan_host ploc)
  const int* ki;          // [nrho] s-row of the log-polar lerp
  const float2* wi;       // [nrho] weights (w0, w1)
  const uint32_t* kw;     // [nrho] packed ki | w1 * 2^20 << 11 (K3 stages it in shared memory)
  const float2* khat;     // [nh][L] kernel spectrum incl. 0.5*drho*dphi/(L*nphi)
  const uint32_t* qidx;   // [nq][nq] readout quadrant table: i0 | j0 << 16, ~0 = zero pixel
  const float2* qw;       // [nq][nq] readout weights (wi, wj)
  const float2* naive_cs; // [ntheta] (cos, sin) * nt/(2n) for the direct backprojector
  const uint32_t* band_off;      // [nbands+1] fused readout: entry range per band
  const uint32_t* band_entries;  // per band: uint4 {qq | bit31 zero, qidx, wi, wj} (plan_host band_packed)
  const uint32_t* band_need;     // [nbands] 1 = some pixel taps one of the band's rows
  const uint32_t* units;         // [nunits][2] fused work units: band range [k0, k1), outermost first
  // where the fused path keeps the convolved spectra's rows inside a Y column (plan_host build_bands):
  // rowmap_*[row] = position or -1 (a band nobody taps: never written, never read), band_row_*[band] =
  // 1 + position of the band's first row or 0; _id: rows stay in place, _cp: needed bands back to back
  const int32_t* rowmap_cp;
  const int32_t* rowmap_id;
  const uint32_t* band_row_cp;
  const uint32_t* band_row_id;
  // generic sizes (Bluestein)
  const float2* chirp;   // [nphi]
  const float2* bhat_f;  // [MB]
  const float2* bhat_i;  // [MB]
  const float2* tw_blue; // pass twiddles, N = MB
  const uint32_t* pairs; // [npairs] row pairs the readout taps (generic path's inverse DFT), ascending
};

struct Dims {
  int nt, ntheta, n, ns, nphi, nh, nrho, nrho_pad, L, M, nq;
  int row_min, nbands, band_rows;  // fused inverse-DFT + readout quads (band_rows = 4)
  int nunits;                      // fused work units (plan_host build_bands)
  int nsm;                         // SMs of the plan's device (persistent grids)
  int generic, MB;                 // generic-size path (Bluestein length-nphi DFTs via MB-point convolutions)
  int gp;                          // column pitch of the row spectra G[m][.] (nt rounded up to even: TMA bulk
                                   // column loads are 16-byte multiples); 0 = nt
  int win, win_lo;                 // compacted row-DFT input (0 = plain rows of ntheta): rows of `win` floats,
                                   // win_lo leading columns + the row's last win - win_lo columns
  float out_scale;        // 1 (backprojection) or 1/(2 pi) (fbp)
  int npairs;             // > 0: the generic inverse DFT runs over t.pairs only (0 = every row pair)
  int ycompact;           // 1: the fused path packs the needed bands of Y back to back (rowmap_cp / band_row_cp)
  int row_end;            // rows the band tables span: row_min + band_rows * nbands (>= nrho)
  int pmix;               // 2: the same through the mixed-radix row DFT of a generic plan (k_row_rdft_mixed_p); 1: K2p emits the semi-polar row spectra P[b][m][ns] and K3 takes them as they are
};

// Each returns cudaGetLastError() after the launch (0 on success) or
// cudaErrorNotSupported when no instantiation exists for the size.
cudaError_t launch_ramp(const Dims& d, const DevTables& t, const float* g, float* out, int batch, cudaStream_t s);
cudaError_t launch_row_rdft(const Dims& d, const DevTables& t, const float* g, float2* G, int batch, cudaStream_t s);
// generic plan whose mixed-radix row DFT can transform the semi-polar rows (d.pmix = 2)
bool mixed_p_available(int nphi, int ns, int nrho, int L);
// semi-polar row spectra P[b][nh][ns] (d.pmix plans; cudaErrorNotSupported otherwise)
cudaError_t launch_row_rdft_p(const Dims& d, const DevTables& t, const float* g, float2* P, int batch, cudaStream_t s);
// rows < row_lo of Y are not written (0 = all rows); pin: the input is K2p's P[b][nh][ns] (no row mix)
// fused_rows: only the rows of bands the fused inverse DFT + readout loads are written (t.rowmap_*)
cudaError_t launch_rho_conv(const Dims& d, const DevTables& t, const float2* G, float2* Y, int batch, int row_lo,
                            cudaStream_t s, bool pin = false, bool fused_rows = false);
cudaError_t launch_row_irdft(const Dims& d, const DevTables& t, const float2* Y, float* lp, int batch, cudaStream_t s);
// counter: one device int of workspace (zeroed by the launcher on s)
cudaError_t launch_irdft_readout(const Dims& d, const DevTables& t, const float2* Y, float* img, int batch,
                                 int* counter, cudaStream_t s);
int fused_band_rows(int nphi);
// generic plan whose mixed-radix nphi runs the fused inverse DFT + readout (bands of 2 rows)
bool fused_mixed_available(const Dims& d);
constexpr int kFusedMaxUnit = 24;  // longest fused work unit in bands (per-unit arrays, one lane per band + 1)
cudaError_t launch_readout(const Dims& d, const DevTables& t, const float* lp, float* img, int batch, cudaStream_t s);

cudaError_t launch_radon_ellipses(const double* params, int K, int nt, int ntheta, int batch, float* out,
                                  cudaStream_t s);
cudaError_t launch_radon_ellipses(const double* params, int K, int nt, int ntheta, int batch, double* out,
                                  cudaStream_t s);

bool sizes_supported(int nt, int ntheta, int L, int M, int MB, bool filter, bool generic);
// generic-size kernels: ramp over bounds-checked column pairs, Bluestein row DFT / inverse DFT
cudaError_t launch_ramp_generic(const Dims& d, const DevTables& t, const float* g, float* out, int batch,
                                cudaStream_t s);
cudaError_t launch_row_rdft_generic(const Dims& d, const DevTables& t, const float* g, float2* G, int batch,
                                    cudaStream_t s);
// nphi has a direct mixed-radix kernel (Q P, Q in {3, 5, 9, 15, 25}); otherwise Bluestein
bool mixed_radix_length(int nphi);
cudaError_t launch_row_irdft_generic(const Dims& d, const DevTables& t, const float2* Y, float* lp, int batch,
                                     cudaStream_t s);
// Pass-twiddle tables (fft.cuh TwTable): entry count for size N (-1 if unsupported)
// and a device fill kernel.
int twiddle_table_len(int N);
cudaError_t launch_init_twiddles(int N, float2* out, cudaStream_t s);

}  // namespace lpbp
