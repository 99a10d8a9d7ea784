/*
 * lpbp.h — C ABI of the B200-native log-polar backprojection library
 * (liblpbp.so, sm_100a).  Drop-in for the fastbp backprojection / FBP path.
 *
 * Reference interfaces replaced (paths under pkg/src/fastbp of arXiv 1608.03589's
 * reference package):
 *   lpbp_execute (filter = 0)    logpolar_backproject(g, n_out, opts)        logpolar.py:121-136
 *   lpbp_execute (filter = 1)    fbp(g, spec, engine="logpolar", n, opts)    filtering.py:73-98
 *   lpbp_filter                  filter_sinogram(g, spec)                    filtering.py:54-70
 *   lpbp_logpolar                _logpolar_convolve(sinogram_to_semipolar(g), rho0, nrho)
 *                                                                            logpolar.py:100-118, grids.py:290-347
 *   lpbp_readout                 logpolar_to_cartesian(l, n, n)              grids.py:399-443
 *   lpbp_naive_backproject       backproject_naive(g, n)                     reference.py:21-37
 *   lpbp_plan_create             LogPolarOptions / FilterSpec validation, adaptive_rho0, _mesh_for,
 *                                make_logpolar_kernel, the kernel spectrum   logpolar.py:50-97, grids.py:385-391,
 *                                                                            filtering.py:30-51
 *
 * Layouts (C-contiguous fp32, as the reference's .values arrays):
 *   sinogram [batch][nt][ntheta]    image [batch][n][n]    log-polar [batch][nrho][2*ntheta]
 * Pointers named *_dev are device pointers on the plan's device; *_host are host
 * pointers (page-locked memory gives copy/compute overlap).  `stream` is a
 * cudaStream_t (NULL = legacy default stream).  Calls are asynchronous with
 * respect to the host unless stated otherwise.
 *
 * Errors: every function returns an LPBP_* status; lpbp_last_error() returns the
 * message of the last failure on the calling thread.  LPBP_EINVAL carries the
 * reference's ValueError messages.
 */
#ifndef LPBP_H_
#define LPBP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LPBP_OK 0
#define LPBP_EINVAL 1       /* invalid argument (reference ValueError)            */
#define LPBP_ECUDA 2        /* CUDA runtime / launch failure                      */
#define LPBP_EUNSUPPORTED 3 /* size has no compiled kernel instantiation          */
#define LPBP_ENOMEM 4       /* device or host allocation failed                   */

typedef struct lpbp_plan lpbp_plan;

typedef struct lpbp_params {
  int32_t nt;        /* detector bins (Sinogram.nt)                                      */
  int32_t ntheta;    /* projection angles (Sinogram.ntheta); nphi = 2*ntheta             */
  int32_t n_out;     /* output image side                                               */
  int32_t has_rho0;  /* 0: adaptive_rho0(n_out, n_out); 1: use rho0 (LogPolarOptions.rho0) */
  double rho0;
  int32_t nrho;      /* 0: _mesh_for default; else LogPolarOptions.nrho                 */
  int32_t filter;    /* 0: backprojection; 1: FBP = filter_sinogram, backproject, 1/(2pi) */
  double lam;        /* FilterSpec.lam (filter = 1)                                     */
  double cutoff;     /* FilterSpec.cutoff (filter = 1)                                  */
  int32_t device;    /* CUDA device ordinal; < 0 builds a host-only plan (tables and info
                        only, no device memory, every execute call fails with EINVAL)   */
} lpbp_params;

typedef struct lpbp_plan_info {
  int32_t nt, ntheta, n_out, ns, nphi, nrho, L, M, kernel_nnz, kmax, filter, device;
  double rho0, drho, dphi, out_scale;
  size_t table_bytes;          /* device bytes of constant tables owned by the plan */
  size_t workspace_per_slice;  /* lpbp_execute workspace bytes per slice in flight  */
  size_t readout_sector_bytes; /* distinct 32-byte log-polar sectors the readout taps (x32) */
  int32_t band_rows, row_min, nbands; /* fused inverse-DFT + readout banding               */
  int32_t generic, MB;         /* 1: any-size path (Bluestein length-nphi DFTs on MB-point FFTs) */
  int32_t phi_q;               /* generic path with mixed-radix length-nphi DFTs (nphi = phi_q x 2^k,
                                  phi_q in {3, 5, 9, 15, 25}) instead of Bluestein; 0 otherwise */
  int32_t p_rows;              /* 1: the row-DFT stage forms the semi-polar rows (grids.py:290-311) first and
                                  emits their ns = nt/2 spectra; 0: nt row spectra, mixed in the rho stage */
} lpbp_plan_info;

int lpbp_plan_create(const lpbp_params* params, lpbp_plan** plan);
void lpbp_plan_destroy(lpbp_plan* plan);
int lpbp_plan_get_info(const lpbp_plan* plan, lpbp_plan_info* info);

/* Workspace for lpbp_execute / lpbp_logpolar processing `chunk` slices at a time. */
int lpbp_workspace_bytes(const lpbp_plan* plan, int32_t chunk, size_t* bytes);

/* Full path: sinogram -> image for `batch` slices (device pointers).  The batch is
 * processed in chunks that fit ws_bytes (>= one slice).  ws = NULL uses a workspace
 * owned by the plan (then calls on one plan must not overlap).  Alignment: sino_dev
 * 16 bytes (TMA bulk loads), ws 256 bytes (cudaMalloc pointers satisfy both). */
int lpbp_execute(const lpbp_plan* plan, const float* sino_dev, float* img_dev, int32_t batch, void* ws,
                 size_t ws_bytes, void* stream);

/* Same, from host to host: chunked H2D / compute / D2H overlapped on internal
 * streams.  Blocks until the images are in img_host. */
int lpbp_execute_host(lpbp_plan* plan, const float* sino_host, float* img_host, int32_t batch, int32_t chunk);

/* Stages (parity testing and composition). */
int lpbp_filter(const lpbp_plan* plan, const float* sino_dev, float* out_dev, int32_t batch, void* stream);
int lpbp_logpolar(const lpbp_plan* plan, const float* sino_dev, float* lp_dev, int32_t batch, void* ws,
                  size_t ws_bytes, void* stream);
int lpbp_readout(const lpbp_plan* plan, const float* lp_dev, float* img_dev, int32_t batch, void* stream);

/* Direct O(n^2 ntheta) pixel-driven backprojector (reference.py:21-37, configs[4]).
 * ws_dev: lpbp_naive_workspace_bytes, 256-byte aligned (the fp64-built angle table and a
 * zero-padded angle-major copy of the batch, 4 slices interleaved per entry).  Two kernel
 * launches on `stream`; asynchronous (no host synchronisation). */
int lpbp_naive_workspace_bytes(int32_t nt, int32_t ntheta, int32_t batch, size_t* bytes);
int lpbp_naive_backproject(const float* sino_dev, float* img_dev, int32_t nt, int32_t ntheta, int32_t n,
                           int32_t batch, float* ws_dev, void* stream);

/* Host copies of plan tables for tests: which = "kernel_cells" (int32 pairs k,l),
 * "ramp" (float M), "khat" (float2 nh*L), "ab" (int32 pairs ns), "wab" (float4 ns),
 * "ki" (int32 nrho), "wi" (float2 nrho), "qidx" (uint32 nq*nq), "qw" (float2 nq*nq),
 * "band_off" (uint32 nbands+1), "band_entries" (uint32), "chirp" (float2 nphi),
 * "bhat_f" / "bhat_i" (float2 MB; generic-size plans only).  Returns the element count in *count;
 * if dst is non-NULL copies min(count, capacity) elements. */
int lpbp_plan_table(const lpbp_plan* plan, const char* which, void* dst, size_t capacity, size_t* count);

/* Per-stage CUDA-event timing of lpbp_execute / lpbp_logpolar / lpbp_execute_host
 * launches (stages: 0 ramp filter, 1 row DFT, 2 rho convolution, 3 row inverse DFT,
 * 4 readout, 5 fused row inverse DFT + readout).  Events are recorded on the launching stream around each kernel;
 * lpbp_profile_read waits for them, returns the sums since the last read and resets. */
int lpbp_profile_enable(lpbp_plan* plan, int32_t enable);
int lpbp_profile_read(lpbp_plan* plan, double* stage_ms, int64_t* stage_launches, int64_t* stage_slices,
                      int32_t nstages);

/* Analytic ellipse-phantom sinograms: fastbp.radon.radon_ellipses (radon.py:38-61), the
 * step before the path, in fp64 on the device with the reference's accumulation order.
 * params_dev: [batch][k][6] doubles (cx, cy, a, b, tilt, rho), any k >= 1;
 * out: [batch][nt][ntheta], fp32 (lpbp_radon_ellipses) or fp64 (lpbp_radon_ellipses_f64). */
int lpbp_radon_ellipses(const double* params_dev, int32_t k, int32_t nt, int32_t ntheta, int32_t batch,
                        float* out_dev, void* stream);
int lpbp_radon_ellipses_f64(const double* params_dev, int32_t k, int32_t nt, int32_t ntheta, int32_t batch,
                            double* out_dev, void* stream);
/* Same from host buffers (fp64 params in, fp64 sinograms out; synchronous on `device`). */
int lpbp_radon_ellipses_host(const double* params, int32_t k, int32_t nt, int32_t ntheta, int32_t batch, double* out,
                             int32_t device);

/* ---- sector (partial) backprojection: partial_backproject(g, sectors, n_out), logpolar.py:210-299 ----
 * Each sector (theta0, beta, a_r) covers ray angles [theta0, theta0 + 2 beta] mod pi.  Its
 * working-frame sinogram (angles rolled to the sector centre with the t-flip past pi,
 * mask / coverage weights, support shrunk by a_r and shifted by 1 - a_r; logpolar.py:153-179,
 * 260-271, radon.py:137-158) runs through the log-polar stage on the sector's own shallow mesh
 * (logpolar.py:272-287); the sector images are sampled at x_w = (1 - a_r, 0) + a_r R(-theta_c) x,
 * divided by a_r and summed (logpolar.py:289-297).  Validation returns LPBP_EINVAL with the
 * reference's ValueError messages.  No filtering (the reference does not filter here). */
typedef struct lpbp_sector_plan lpbp_sector_plan;

typedef struct lpbp_sector {
  double theta0; /* first ray angle of the sector */
  double beta;   /* half-width, (0, pi/2]          */
  double a_r;    /* rescale, (0, 1/2)              */
} lpbp_sector;

typedef struct lpbp_sector_info {
  int32_t jc;          /* centre angle index round((theta0 + beta) / dtheta)      */
  int32_t nrho;        /* sector mesh rows (_mesh_for(ns, rho0, None))            */
  int32_t L;           /* rho FFT length of the sector's log-polar stage          */
  int32_t nphi;        /* 2 * ntheta                                              */
  double theta_c;      /* jc * dtheta                                             */
  double rho0;         /* sector mesh depth (logpolar.py:279-283)                 */
  double drho;         /* -rho0 / nrho                                            */
  double support_min;  /* logpolar.py:278                                         */
  double a_r;
  size_t table_bytes;  /* device bytes of this sector's constant tables           */
} lpbp_sector_info;

int lpbp_sector_plan_create(int32_t nt, int32_t ntheta, int32_t n_out, const lpbp_sector* sectors,
                            int32_t nsectors, int32_t device, lpbp_sector_plan** plan);
void lpbp_sector_plan_destroy(lpbp_sector_plan* plan);
int lpbp_sector_get_info(const lpbp_sector_plan* plan, int32_t index, lpbp_sector_info* info);
/* Workspace for `chunk` slices in flight (256-byte aligned). */
int lpbp_sector_workspace_bytes(const lpbp_sector_plan* plan, int32_t chunk, size_t* bytes);
/* sino [batch][nt][ntheta] -> img [batch][n][n]; ws NULL = plan-owned workspace (calls serialise). */
int lpbp_sector_execute(lpbp_sector_plan* plan, const float* sino_dev, float* img_dev, int32_t batch, void* ws,
                        size_t ws_bytes, void* stream);
/* Host -> host: chunked copies around lpbp_sector_execute on a plan-owned stream; blocks. */
int lpbp_sector_execute_host(lpbp_sector_plan* plan, const float* sino_host, float* img_host, int32_t batch,
                             int32_t chunk);
/* Stage: sector `index`'s working-frame sinogram [batch][nt][ntheta]. */
int lpbp_sector_prepare(const lpbp_sector_plan* plan, int32_t index, const float* sino_dev, float* out_dev,
                        int32_t batch, void* stream);
/* Stage: the log-polar stage of sector `index` on a working-frame sinogram -> [batch][nrho][nphi]. */
int lpbp_sector_logpolar(const lpbp_sector_plan* plan, int32_t index, const float* work_dev, float* lp_dev,
                         int32_t batch, void* stream);

/* ---- BST engine: bst_backproject(g, BstOptions), bst.py:183-203, and fbp(g, spec, engine="bst"),
 * the reference fbp's default engine (filtering.py:73-98) ----
 * Semi-polar unfolding on 2*(nt/2) radial samples with the Kaiser window, per-ray zero-padded
 * real DFTs along s (bst.py:120-143), 1/sigma kernel, bilinear polar -> Cartesian frequency
 * gridding with Hermitian averaging on the 2x padded lattice (grids.py:456-508), inverse 2-D
 * DFT with the phase ramps, crop (bst.py:146-170), BST_SCALE, and in subtract_mean mode the
 * exact spatial mean from <g, chord> (bst.py:173-180, 196-202).  This build runs radial DFT
 * lengths L that are powers of two in [512, 8192] or at most 4096 (Bluestein), padded sides 2 n
 * that are powers of two in [128, 4096] or at most 4096 (Bluestein), and even nt; other sizes
 * return LPBP_EUNSUPPORTED after validation. */
typedef struct lpbp_bst_plan lpbp_bst_plan;

typedef struct lpbp_bst_params {
  int32_t nt, ntheta, n_out;
  double beta;       /* BstOptions.beta (Kaiser window; 0 = none)          */
  double zero_pad;   /* BstOptions.zero_pad (>= 1)                         */
  int32_t dc_mode;   /* 0 = "subtract_mean", 1 = "kernel_cap"              */
  int32_t filter;    /* 1: fbp = filter_sinogram(FilterSpec(lam, cutoff)) first, x 1/(2 pi) */
  double lam, cutoff;
  int32_t device;    /* < 0: host-only plan (validation and info only)     */
} lpbp_bst_params;

typedef struct lpbp_bst_info {
  int32_t ns, nray, L, m_need, m_pad, big, p0, supported;
  double ds, dsigma, out_scale;
  size_t table_bytes, workspace_per_slice;
} lpbp_bst_info;

int lpbp_bst_plan_create(const lpbp_bst_params* params, lpbp_bst_plan** plan);
void lpbp_bst_plan_destroy(lpbp_bst_plan* plan);
int lpbp_bst_get_info(const lpbp_bst_plan* plan, lpbp_bst_info* info);
int lpbp_bst_workspace_bytes(const lpbp_bst_plan* plan, int32_t chunk, size_t* bytes);
/* Per-stage CUDA-event timing of lpbp_bst_execute / _execute_host (stages: 0 ramp filter (fbp
 * plans), 1 radial spectra, 2 gridding + inverse DFT along x, 3 inverse DFT along y + crop);
 * lpbp_bst_profile_read waits for the events, returns the sums since the last read and resets. */
int lpbp_bst_profile_enable(lpbp_bst_plan* plan, int32_t enable);
int lpbp_bst_profile_read(lpbp_bst_plan* plan, double* stage_ms, int64_t* stage_launches, int64_t* stage_slices,
                          int32_t nstages);
/* sino [batch][nt][ntheta] -> img [batch][n][n]; ws NULL = plan-owned workspace. */
int lpbp_bst_execute(lpbp_bst_plan* plan, const float* sino_dev, float* img_dev, int32_t batch, void* ws,
                     size_t ws_bytes, void* stream);
int lpbp_bst_execute_host(lpbp_bst_plan* plan, const float* sino_host, float* img_host, int32_t batch,
                          int32_t chunk);
/* Stage: the weighted radial spectra of an unfiltered batch, laid out as ray pairs
 * P[batch][ntheta + 2][m_pad][2] complex64 (pair c = rays c and c + ntheta, the two half-lines
 * of angle c; pair ntheta repeats pair 0 swapped: rays ntheta and 0; pair ntheta + 1 and the
 * bins m >= m_need are zero); bins m < m_need hold 0.5 x the reference's spectra * sigma_kernel, the 1/2 being
 * the Hermitian averaging of the gridding; the DC bin is zero in subtract_mean mode. */
int lpbp_bst_radial(const lpbp_bst_plan* plan, const float* sino_dev, float* spectra_dev, int32_t batch,
                    void* stream);

/* ---- the path's resampling steps as standalone operations (the fused pipeline computes them
 * implicitly); reference semantics and ValueError texts ----
 * sinogram_to_semipolar(g, ns)   grids.py:290-311   sino [batch][nt][ntheta] -> p [batch][ns][2 ntheta]
 *                                                   (ns = 0: nt / 2)
 * semipolar_to_logpolar(p, rho0, nrho)  grids.py:332-347   p [batch][ns][nphi] -> lp [batch][nrho][nphi]
 * logpolar_to_cartesian(l, nx, ny)      grids.py:399-443   lp -> img [batch][ny][nx] (fp64 coordinates)
 * make_logpolar_kernel(nrho, nphi, drho) logpolar.py:66-81  dense [nrho][nphi] float64 on the host */
int lpbp_sinogram_to_semipolar(const float* sino_dev, float* p_dev, int32_t nt, int32_t ntheta, int32_t ns,
                               int32_t batch, void* stream);
int lpbp_semipolar_to_logpolar(const float* p_dev, float* lp_dev, int32_t ns, int32_t nphi, double rho0, int32_t nrho,
                               int32_t batch, void* stream);
int lpbp_logpolar_to_cartesian(const float* lp_dev, float* img_dev, int32_t nrho, int32_t nphi, double rho0,
                               int32_t nx, int32_t ny, int32_t batch, void* stream);
int lpbp_logpolar_kernel(int32_t nrho, int32_t nphi, double drho, double* out_host);

/* ---- BST helpers ----
 * polar_to_cartesian_frequency(ps, nx, ny, dw)  grids.py:456-508: spectra [batch] x complex64 P with
 *   element (m, ray) at P[m * stride_m + ray * stride_ray] (slice pitch slice_pitch, in complex
 *   elements) -> out [batch][ny][nx] complex64, times `scale`; fp64 coordinates.
 * mean_backprojection(g)   bst.py:173-180 -> out_dev [batch] doubles.
 * kaiser_window(ns, beta)  bst.py:90-102 -> out_host [ns] doubles. */
int lpbp_polar_to_cartesian_frequency(const float* spec_dev, float* out_dev, int32_t nsigma, int32_t nray,
                                      int64_t stride_m, int64_t stride_ray, int64_t slice_pitch, double dsigma,
                                      int32_t nx, int32_t ny, double dw, float scale, int32_t batch, void* stream);
int lpbp_mean_backprojection(const float* sino_dev, double* out_dev, int32_t nt, int32_t ntheta, int32_t batch,
                             void* stream);
int lpbp_kaiser_window(int32_t ns, double beta, double* out_host);

/* Number of kernel launches the last lpbp_execute/lpbp_execute_host issued on the calling thread. */
int64_t lpbp_last_launch_count(void);

const char* lpbp_last_error(void);
int32_t lpbp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LPBP_H_ */
