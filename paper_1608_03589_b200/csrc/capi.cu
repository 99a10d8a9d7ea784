// C ABI (include/lpbp.h): plan lifetime, device tables, chunked executors.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges per stage for timeline tools

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/lpbp.h"
#include "kernels.cuh"
#include "direct_kernels.cuh"
#include "plan_host.h"
#include "sector_kernels.cuh"
#include "bst_host.h"
#include "bst_kernels.cuh"
#include "resample_kernels.cuh"

using lpbp::DevTables;
using lpbp::Dims;
using lpbp::HostPlan;

namespace {

thread_local std::string g_last_error;
thread_local int64_t g_launches = 0;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(LPBP_ECUDA, std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}
int launch_fail(cudaError_t e, const char* where) {
  if (e == cudaErrorNotSupported) return fail(LPBP_EUNSUPPORTED, std::string(where) + ": size not supported");
  return cuda_fail(e, where);
}

struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = (prev == dev) || cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

size_t align256(size_t v) { return (v + 255) / 256 * 256; }


// Error exit of a host pipeline: copies already queued on the three streams still read the
// caller's host buffers, so wait for them before handing the (first) error back.
int drain_streams(cudaStream_t a, cudaStream_t b, cudaStream_t c, int rc) {
  if (a) cudaStreamSynchronize(a);
  if (b) cudaStreamSynchronize(b);
  if (c) cudaStreamSynchronize(c);
  return rc;
}

}  // namespace

struct lpbp_plan {
  HostPlan h;
  Dims d{};
  DevTables t{};
  int device = 0;
  std::vector<void*> allocs;
  size_t table_bytes = 0;
  size_t szA = 0, szB = 0;  // per-slice workspace regions (aliased by stage lifetime)

  // optional per-stage CUDA-event profiling (lpbp_profile_enable / _read)
  struct Rec { int stage; int slices; cudaEvent_t a, b; };
  bool profiling = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> ev_pool;
  std::mutex prof_mu;

  std::mutex mu;  // guards the owned workspace and the host pipeline
  void* own_ws = nullptr;
  size_t own_ws_bytes = 0;
  struct Pipe {
    int chunk = 0;
    cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
    cudaEvent_t ev_in[2] = {}, ev_comp[2] = {}, ev_out[2] = {};
    float* in[2] = {};
    float* out[2] = {};
    void* ws = nullptr;
    size_t ws_bytes = 0;
  } pipe;

  template <typename T>
  int upload(const std::vector<T>& v, const T** dst) {
    if (v.empty()) {
      *dst = nullptr;
      return LPBP_OK;
    }
    void* p = nullptr;
    const size_t bytes = v.size() * sizeof(T);
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(plan table)");
    allocs.push_back(p);
    e = cudaMemcpy(p, v.data(), bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(plan table)");
    table_bytes += bytes;
    *dst = static_cast<const T*>(p);
    return LPBP_OK;
  }

  // device-generated pass-twiddle table for FFT size N
  int twiddles(int N, const float2** dst) {
    const int len = lpbp::twiddle_table_len(N);
    if (len < 0) return fail(LPBP_EUNSUPPORTED, "no FFT plan for size " + std::to_string(N));
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)len * sizeof(float2));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(twiddles)");
    allocs.push_back(p);
    e = lpbp::launch_init_twiddles(N, static_cast<float2*>(p), nullptr);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "init_twiddles");
    table_bytes += (size_t)len * sizeof(float2);
    *dst = static_cast<const float2*>(p);
    return LPBP_OK;
  }

  void release_pipe() {
    for (int i = 0; i < 2; ++i) {
      if (pipe.ev_in[i]) cudaEventDestroy(pipe.ev_in[i]);
      if (pipe.ev_comp[i]) cudaEventDestroy(pipe.ev_comp[i]);
      if (pipe.ev_out[i]) cudaEventDestroy(pipe.ev_out[i]);
      if (pipe.in[i]) cudaFree(pipe.in[i]);
      if (pipe.out[i]) cudaFree(pipe.out[i]);
    }
    if (pipe.ws) cudaFree(pipe.ws);
    if (pipe.s_in) cudaStreamDestroy(pipe.s_in);
    if (pipe.s_comp) cudaStreamDestroy(pipe.s_comp);
    if (pipe.s_out) cudaStreamDestroy(pipe.s_out);
    pipe = Pipe{};
  }

  ~lpbp_plan() {
    DeviceGuard g(device);
    for (auto& r : recs) { ev_pool.push_back(r.a); ev_pool.push_back(r.b); }
    for (auto e : ev_pool) cudaEventDestroy(e);
    release_pipe();
    if (own_ws) cudaFree(own_ws);
    for (void* p : allocs) cudaFree(p);
  }
};

namespace {

// Stage ids for profiling: 0 ramp, 1 row_rdft, 2 rho_conv, 3 row_irdft, 4 readout,
// 5 fused row_irdft + readout.
constexpr int kStages = 6;

cudaEvent_t take_event(lpbp_plan* P) {
  if (!P->ev_pool.empty()) {
    cudaEvent_t e = P->ev_pool.back();
    P->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

constexpr const char* kStageNames[kStages] = {"lpbp.ramp_filter", "lpbp.row_rdft", "lpbp.rho_conv",
                                               "lpbp.row_irdft", "lpbp.readout", "lpbp.irdft_readout"};

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

template <typename F>
cudaError_t staged(const lpbp_plan* Pc, int stage, int slices, cudaStream_t s, F&& launch) {
  lpbp_plan* P = const_cast<lpbp_plan*>(Pc);
  NvtxRange range(kStageNames[stage]);
  if (!P->profiling) return launch();
  std::lock_guard<std::mutex> lk(P->prof_mu);
  cudaEvent_t a = take_event(P), b = take_event(P);
  cudaEventRecord(a, s);
  cudaError_t e = launch();
  cudaEventRecord(b, s);
  P->recs.push_back({stage, slices, a, b});
  return e;
}

// Run the stages for one chunk already resident on the device.
// stop_after_lp: write the log-polar image to lp_out and skip filter/readout.
// win > 0: compacted input rows (sector path) of `win` floats: `win_lo` leading columns,
// then the row's last win - win_lo columns; everything between is zero.

// The ramp filter acts along t only: a generic plan (length-nphi DFTs by Bluestein) still takes the
// power-of-two ramp kernels whenever they cover (nt, ntheta); the Bluestein-capable kernel otherwise.
static cudaError_t ramp_any(const lpbp::Dims& d, const lpbp::DevTables& t, const float* in, float* out, int c,
                            cudaStream_t s) {
  cudaError_t r = lpbp::launch_ramp(d, t, in, out, c, s);
  if (r == cudaErrorNotSupported && d.generic) {
    (void)cudaGetLastError();
    r = lpbp::launch_ramp_generic(d, t, in, out, c, s);
  }
  return r;
}

int run_chunk(const lpbp_plan* P, const float* in, float* out, int c, char* ws, cudaStream_t s, bool stop_after_lp,
              float* lp_out, int win = 0, int win_lo = 0) {
  Dims dl = P->d;
  if (win > 0) {
    dl.win = win;
    dl.win_lo = win_lo;
  }
  const Dims& d = dl;
  char* A = ws;
  char* B = ws + align256(P->szA * c);
  int* counter = reinterpret_cast<int*>(B + align256(P->szB * c));
  const float* src = in;
  cudaError_t e;
  const bool gen = d.generic != 0;
  if (P->h.filter && !stop_after_lp) {
    e = staged(P, 0, c, s, [&] { return ramp_any(d, P->t, in, reinterpret_cast<float*>(A), c, s); });
    if (e) return launch_fail(e, "ramp_filter");
    ++g_launches;
    src = reinterpret_cast<const float*>(A);
  }
  const bool pin = (gen ? d.pmix == 2 : d.pmix == 1) && win == 0;  // semi-polar row spectra, no row mix in K3
  e = staged(P, 1, c, s, [&] {
    return pin   ? lpbp::launch_row_rdft_p(d, P->t, src, reinterpret_cast<float2*>(B), c, s)
           : gen ? lpbp::launch_row_rdft_generic(d, P->t, src, reinterpret_cast<float2*>(B), c, s)
                 : lpbp::launch_row_rdft(d, P->t, src, reinterpret_cast<float2*>(B), c, s);
  });
  if (e) return launch_fail(e, "row_rdft");
  ++g_launches;
  const bool unfused = stop_after_lp || (gen && !lpbp::fused_mixed_available(d));
  e = staged(P, 2, c, s, [&] {  // rows below the first tapped one (pair) are never read downstream; ahead of the
                                // fused inverse DFT + readout only the rows of the bands it loads are written
    return lpbp::launch_rho_conv(d, P->t, reinterpret_cast<const float2*>(B), reinterpret_cast<float2*>(A), c,
                                 stop_after_lp ? 0 : d.row_min, s, pin, !unfused && P->t.rowmap_id != nullptr);
  });
  if (e) return launch_fail(e, "rho_conv");
  ++g_launches;
  if (stop_after_lp || (gen && !lpbp::fused_mixed_available(d))) {
    // generic sizes: unfused inverse DFT into B (or the caller's buffer), then the readout
    float* lp = stop_after_lp ? lp_out : reinterpret_cast<float*>(B);
    lpbp::Dims dp = d;  // the full log-polar image for the stage API; the tapped row pairs otherwise
    if (stop_after_lp) dp.npairs = 0;
    e = staged(P, 3, c, s, [&] {
      return gen ? lpbp::launch_row_irdft_generic(dp, P->t, reinterpret_cast<const float2*>(A), lp, c, s)
                 : lpbp::launch_row_irdft(d, P->t, reinterpret_cast<const float2*>(A), lp, c, s);
    });
    if (e) return launch_fail(e, "row_irdft");
    ++g_launches;
    if (stop_after_lp) return LPBP_OK;
    e = staged(P, 4, c, s, [&] { return lpbp::launch_readout(d, P->t, lp, out, c, s); });
    if (e) return launch_fail(e, "readout");
    ++g_launches;
    return LPBP_OK;
  }
  e = staged(P, 5, c, s,
             [&] { return lpbp::launch_irdft_readout(d, P->t, reinterpret_cast<const float2*>(A), out, c, counter, s); });
  if (e) return launch_fail(e, "irdft_readout");
  ++g_launches;
  return LPBP_OK;
}

size_t ws_bytes_for(const lpbp_plan* P, int chunk) { return align256(P->szA * chunk) + align256(P->szB * chunk) + 256; }
size_t ws_per_slice(const lpbp_plan* P) { return ws_bytes_for(P, 1); }

int ensure_own_ws(lpbp_plan* P, size_t bytes) {
  if (P->own_ws_bytes >= bytes) return LPBP_OK;
  if (P->own_ws) cudaFree(P->own_ws);
  P->own_ws = nullptr;
  P->own_ws_bytes = 0;
  cudaError_t e = cudaMalloc(&P->own_ws, bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(workspace)");
  P->own_ws_bytes = bytes;
  return LPBP_OK;
}

int run_batched(const lpbp_plan* Pc, const float* in, float* out, int batch, void* ws, size_t ws_bytes,
                cudaStream_t s, bool stop_after_lp) {
  lpbp_plan* P = const_cast<lpbp_plan*>(Pc);
  // TMA bulk loads read the sinogram rows and the workspace regions directly
  if (reinterpret_cast<uintptr_t>(in) % 16) return fail(LPBP_EINVAL, "sinogram pointer must be 16-byte aligned");
  if (ws && reinterpret_cast<uintptr_t>(ws) % 256) return fail(LPBP_EINVAL, "workspace must be 256-byte aligned");
  const size_t per = P->szA + P->szB;
  std::unique_lock<std::mutex> lock(P->mu, std::defer_lock);
  if (!ws) {
    lock.lock();
    const int chunk = std::max(1, std::min(batch, 16));
    int rc = ensure_own_ws(P, ws_bytes_for(P, chunk));
    if (rc) return rc;
    ws = P->own_ws;
    ws_bytes = P->own_ws_bytes;
  }
  int chunk = 1;
  while (chunk < batch && ws_bytes_for(P, chunk + 1) <= ws_bytes) ++chunk;
  if (ws_bytes_for(P, chunk) > ws_bytes)
    return fail(LPBP_EINVAL, "workspace too small for one slice (need " + std::to_string(ws_per_slice(P)) + " bytes)");
  (void)per;
  const size_t in_slice = (size_t)P->d.nt * P->d.ntheta;
  const size_t out_slice = stop_after_lp ? (size_t)P->d.nrho * P->d.nphi : (size_t)P->d.n * P->d.n;
  for (int off = 0; off < batch; off += chunk) {
    const int c = std::min(chunk, batch - off);
    int rc = run_chunk(P, in + off * in_slice, stop_after_lp ? nullptr : out + off * out_slice, c,
                       static_cast<char*>(ws), s, stop_after_lp, stop_after_lp ? out + off * out_slice : nullptr);
    if (rc) return rc;
  }
  return LPBP_OK;
}

}  // namespace

static_assert(lpbp::kMaxUnitBands == lpbp::kFusedMaxUnit, "host work units must fit the fused kernel's arrays");

extern "C" {

int lpbp_plan_create(const lpbp_params* params, lpbp_plan** plan) {
  g_last_error.clear();
  if (!params || !plan) return fail(LPBP_EINVAL, "null argument");
  *plan = nullptr;
  lpbp::HostPlanParams hp{params->nt, params->ntheta, params->n_out, params->has_rho0 != 0, params->rho0,
                          params->nrho, params->filter != 0, params->lam, params->cutoff};
  lpbp_plan* P = new (std::nothrow) lpbp_plan();
  if (!P) return fail(LPBP_ENOMEM, "host allocation failed");
  std::string err = lpbp::build_host_plan(hp, P->h);
  if (!err.empty()) {
    delete P;
    return fail(LPBP_EINVAL, err);
  }
  const HostPlan& h = P->h;
  if (params->device >= 0 && !lpbp::sizes_supported(h.nt, h.ntheta, h.L, h.M, h.MB, h.filter, h.generic)) {
    delete P;
    return fail(LPBP_EUNSUPPORTED, "no kernel instantiation for nt=" + std::to_string(h.nt) + ", ntheta=" +
                                       std::to_string(h.ntheta) + ", L=" + std::to_string(h.L) +
                                       " (this build: ramp embedding 2*nt <= 8192, rho FFT <= 16384, row DFTs of length 2*ntheta: Bluestein on <= 16384 points or mixed-radix Q x 2^k, Q in {3, 5, 9, 15, 25})");
  }
  P->device = params->device;
  if (lpbp::fused_band_rows(P->h.nphi) > 0) lpbp::build_bands(P->h, lpbp::fused_band_rows(P->h.nphi));
  if (P->device >= 0) {
    DeviceGuard g(P->device);
    if (!g.ok) {
      delete P;
      return fail(LPBP_ECUDA, "cannot select CUDA device " + std::to_string(params->device));
    }
    int rc = LPBP_OK;
    if (!h.generic) rc = rc ? rc : P->twiddles(h.nphi, &P->t.tw_phi);
    rc = rc ? rc : P->twiddles(h.L, &P->t.tw_rho);
    if (h.filter) rc = rc ? rc : P->twiddles(h.M, &P->t.tw_ramp);
    if (h.generic) {
      if (h.MB <= 16384) rc = rc ? rc : P->twiddles(h.MB, &P->t.tw_blue);  // (longer: mixed-radix lengths only)
      rc = rc ? rc : P->upload(h.chirp, reinterpret_cast<const lpbp::F2**>(&P->t.chirp));
      rc = rc ? rc : P->upload(h.bhat_f, reinterpret_cast<const lpbp::F2**>(&P->t.bhat_f));
      rc = rc ? rc : P->upload(h.bhat_i, reinterpret_cast<const lpbp::F2**>(&P->t.bhat_i));
    }
    rc = rc ? rc : P->upload(h.ramp, &P->t.ramp);
    rc = rc ? rc : P->upload(h.ab, reinterpret_cast<const lpbp::I2**>(&P->t.ab));
    rc = rc ? rc : P->upload(h.wab, reinterpret_cast<const lpbp::F4**>(&P->t.wab));
    rc = rc ? rc : P->upload(h.abw, reinterpret_cast<const uint32_t**>(&P->t.abw));
    if (h.pmix) {
      rc = rc ? rc : P->upload(h.ptile, &P->t.ptile);
      rc = rc ? rc : P->upload(h.ploc, &P->t.ploc);
    }
    rc = rc ? rc : P->upload(h.ki, &P->t.ki);
    rc = rc ? rc : P->upload(h.wi, reinterpret_cast<const lpbp::F2**>(&P->t.wi));
    rc = rc ? rc : P->upload(h.kw, &P->t.kw);
    rc = rc ? rc : P->upload(h.khat, reinterpret_cast<const lpbp::F2**>(&P->t.khat));
    rc = rc ? rc : P->upload(h.qidx, &P->t.qidx);
    rc = rc ? rc : P->upload(h.qw, reinterpret_cast<const lpbp::F2**>(&P->t.qw));
    rc = rc ? rc : P->upload(h.naive_cs, reinterpret_cast<const lpbp::F2**>(&P->t.naive_cs));
    if (!rc) {
      rc = P->upload(P->h.band_off, &P->t.band_off);
      rc = rc ? rc : P->upload(P->h.band_packed, &P->t.band_entries);
      rc = rc ? rc : P->upload(P->h.band_need, &P->t.band_need);
      rc = rc ? rc : P->upload(P->h.units, &P->t.units);
      rc = rc ? rc : P->upload(P->h.rowmap_cp, &P->t.rowmap_cp);
      rc = rc ? rc : P->upload(P->h.rowmap_id, &P->t.rowmap_id);
      rc = rc ? rc : P->upload(P->h.band_row_cp, &P->t.band_row_cp);
      rc = rc ? rc : P->upload(P->h.band_row_id, &P->t.band_row_id);
      rc = rc ? rc : P->upload(P->h.pair_list, &P->t.pairs);
    }
    if (rc) {
      std::string msg = g_last_error;
      delete P;
      return fail(rc, msg);
    }
  }
  Dims& d = P->d;
  d.nt = h.nt;
  d.gp = h.nt + (h.nt & 1);
  d.ntheta = h.ntheta;
  d.n = h.n;
  d.ns = h.ns;
  d.nphi = h.nphi;
  d.nh = h.nh;
  d.nrho = h.nrho;
  d.nrho_pad = h.nrho_pad;
  d.L = h.L;
  d.M = h.M;
  d.nq = h.nq;
  d.out_scale = (float)h.out_scale;
  d.row_min = h.row_min;
  d.nbands = h.nbands;
  d.nunits = h.nunits;
  d.band_rows = h.band_rows;
  d.generic = h.generic ? 1 : 0;
  d.MB = h.MB;
  d.npairs = (int)h.pair_list.size();
  // K2p + K3 on semi-polar row spectra: power-of-two path only; LPBP_K2P=0 keeps K2's row spectra and
  // K3's frequency-domain row mix (A/B checks)
  static const bool k2p = [] {
    const char* v = getenv("LPBP_K2P");
    return v ? atoi(v) != 0 : true;
  }();
  d.pmix = (h.pmix && !h.generic && k2p && 2 * h.nrho <= h.L) ? 1 : 0;
  if (h.generic && k2p && lpbp::mixed_p_available(h.nphi, h.ns, h.nrho, h.L)) d.pmix = 2;  // mixed-radix lengths
  // the fused path's Y columns hold the needed bands back to back; LPBP_YCOMPACT=0 leaves every row in place
  static const bool ycp = [] {
    const char* v = getenv("LPBP_YCOMPACT");
    return v ? atoi(v) != 0 : true;
  }();
  d.ycompact = ycp ? 1 : 0;
  d.row_end = P->h.row_end;
  d.nsm = 148;
  if (P->device >= 0) cudaDeviceGetAttribute(&d.nsm, cudaDevAttrMultiProcessorCount, P->device);
  const size_t fg = h.filter ? (size_t)h.nt * h.ntheta * sizeof(float) : 0;
  const size_t Y = (size_t)h.nh * h.nrho_pad * sizeof(float2);
  const size_t G = (size_t)h.nh * (h.nt + (h.nt & 1)) * sizeof(float2);
  const size_t lp = (size_t)h.nrho * h.nphi * sizeof(float);
  P->szA = std::max(fg, Y);
  P->szB = std::max(G, lp);
  *plan = P;
  return LPBP_OK;
}

void lpbp_plan_destroy(lpbp_plan* plan) { delete plan; }

int lpbp_plan_get_info(const lpbp_plan* P, lpbp_plan_info* info) {
  if (!P || !info) return fail(LPBP_EINVAL, "null argument");
  const HostPlan& h = P->h;
  info->nt = h.nt;
  info->ntheta = h.ntheta;
  info->n_out = h.n;
  info->ns = h.ns;
  info->nphi = h.nphi;
  info->nrho = h.nrho;
  info->L = h.L;
  info->M = h.M;
  info->kernel_nnz = h.nnz;
  info->kmax = h.kmax;
  info->filter = h.filter ? 1 : 0;
  info->device = P->device;
  info->rho0 = h.rho0;
  info->drho = h.drho;
  info->dphi = h.dphi;
  info->out_scale = h.out_scale;
  info->table_bytes = P->table_bytes;
  info->workspace_per_slice = ws_per_slice(P);
  info->readout_sector_bytes = h.readout_sector_bytes;
  info->band_rows = h.band_rows;
  info->row_min = h.row_min;
  info->nbands = h.nbands;
  info->generic = h.generic ? 1 : 0;
  info->MB = h.MB;
  info->p_rows = P->d.pmix ? 1 : 0;
  info->phi_q = 0;
  if (h.generic && lpbp::mixed_radix_length(h.nphi)) {
    int q = h.nphi;
    while (q % 2 == 0) q /= 2;
    info->phi_q = q;
  }
  return LPBP_OK;
}

int lpbp_workspace_bytes(const lpbp_plan* P, int32_t chunk, size_t* bytes) {
  if (!P || !bytes || chunk < 1) return fail(LPBP_EINVAL, "invalid argument");
  *bytes = ws_bytes_for(P, chunk);
  return LPBP_OK;
}

int lpbp_execute(const lpbp_plan* P, const float* sino_dev, float* img_dev, int32_t batch, void* ws,
                 size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (!P || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (batch == 0) return LPBP_OK;
  if (!sino_dev || !img_dev) return fail(LPBP_EINVAL, "invalid argument");
  DeviceGuard g(P->device);
  return run_batched(P, sino_dev, img_dev, batch, ws, ws_bytes, static_cast<cudaStream_t>(stream), false);
}

int lpbp_logpolar(const lpbp_plan* P, const float* sino_dev, float* lp_dev, int32_t batch, void* ws,
                  size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (!P || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (batch == 0) return LPBP_OK;
  if (!sino_dev || !lp_dev) return fail(LPBP_EINVAL, "invalid argument");
  DeviceGuard g(P->device);
  return run_batched(P, sino_dev, lp_dev, batch, ws, ws_bytes, static_cast<cudaStream_t>(stream), true);
}

int lpbp_filter(const lpbp_plan* P, const float* sino_dev, float* out_dev, int32_t batch, void* stream) {
  g_launches = 0;
  if (!P || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (!P->h.filter) return fail(LPBP_EINVAL, "plan was created without a filter (filter = 0)");
  if (batch == 0) return LPBP_OK;
  if (!sino_dev || !out_dev) return fail(LPBP_EINVAL, "invalid argument");
  DeviceGuard g(P->device);
  cudaError_t e = ramp_any(P->d, P->t, sino_dev, out_dev, batch, static_cast<cudaStream_t>(stream));
  if (e) return launch_fail(e, "ramp_filter");
  ++g_launches;
  return LPBP_OK;
}

int lpbp_readout(const lpbp_plan* P, const float* lp_dev, float* img_dev, int32_t batch, void* stream) {
  g_launches = 0;
  if (!P || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (batch == 0) return LPBP_OK;
  if (!lp_dev || !img_dev) return fail(LPBP_EINVAL, "invalid argument");
  DeviceGuard g(P->device);
  cudaError_t e = lpbp::launch_readout(P->d, P->t, lp_dev, img_dev, batch, static_cast<cudaStream_t>(stream));
  if (e) return launch_fail(e, "readout");
  ++g_launches;
  return LPBP_OK;
}

int lpbp_execute_host(lpbp_plan* P, const float* sino_host, float* img_host, int32_t batch, int32_t chunk) {
  g_launches = 0;
  if (!P || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (batch == 0) return LPBP_OK;
  if (!sino_host || !img_host) return fail(LPBP_EINVAL, "invalid argument");
  if (chunk <= 0) chunk = 4;
  chunk = std::min(chunk, batch);
  DeviceGuard g(P->device);
  std::lock_guard<std::mutex> lock(P->mu);
  auto& pp = P->pipe;
  const size_t in_slice = (size_t)P->d.nt * P->d.ntheta * sizeof(float);
  const size_t out_slice = (size_t)P->d.n * P->d.n * sizeof(float);
  if (pp.chunk < chunk) {
    P->release_pipe();
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaMalloc(&pp.in[i], in_slice * chunk);
      if (e == cudaSuccess) e = cudaMalloc(&pp.out[i], out_slice * chunk);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pp.ev_in[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pp.ev_comp[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pp.ev_out[i], cudaEventDisableTiming);
    }
    pp.ws_bytes = ws_bytes_for(P, chunk);
    if (e == cudaSuccess) e = cudaMalloc(&pp.ws, pp.ws_bytes);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pp.s_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pp.s_comp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pp.s_out, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      P->release_pipe();
      return cuda_fail(e, "host pipeline setup");
    }
    pp.chunk = chunk;
  }
  const int nchunks = (batch + chunk - 1) / chunk;
  for (int ci = 0; ci < nchunks; ++ci) {
    const int slot = ci & 1;
    const int off = ci * chunk;
    const int c = std::min(chunk, batch - off);
    cudaError_t e;
    if (ci >= 2) cudaStreamWaitEvent(pp.s_in, pp.ev_comp[slot], 0);
    e = cudaMemcpyAsync(pp.in[slot], sino_host + (size_t)off * (in_slice / sizeof(float)), in_slice * c,
                        cudaMemcpyHostToDevice, pp.s_in);
    if (e) return drain_streams(pp.s_in, pp.s_comp, pp.s_out, cuda_fail(e, "H2D"));
    cudaEventRecord(pp.ev_in[slot], pp.s_in);
    cudaStreamWaitEvent(pp.s_comp, pp.ev_in[slot], 0);
    if (ci >= 2) cudaStreamWaitEvent(pp.s_comp, pp.ev_out[slot], 0);
    const int64_t before = g_launches;
    int rc = run_chunk(P, pp.in[slot], pp.out[slot], c, static_cast<char*>(pp.ws), pp.s_comp, false, nullptr);  // cudaMalloc'd: aligned
    if (rc) return drain_streams(pp.s_in, pp.s_comp, pp.s_out, rc);
    (void)before;
    cudaEventRecord(pp.ev_comp[slot], pp.s_comp);
    cudaStreamWaitEvent(pp.s_out, pp.ev_comp[slot], 0);
    e = cudaMemcpyAsync(img_host + (size_t)off * (out_slice / sizeof(float)), pp.out[slot], out_slice * c,
                        cudaMemcpyDeviceToHost, pp.s_out);
    if (e) return drain_streams(pp.s_in, pp.s_comp, pp.s_out, cuda_fail(e, "D2H"));
    cudaEventRecord(pp.ev_out[slot], pp.s_out);
  }
  cudaError_t e = cudaStreamSynchronize(pp.s_out);
  if (e == cudaSuccess) e = cudaStreamSynchronize(pp.s_comp);
  if (e) return drain_streams(pp.s_in, pp.s_comp, pp.s_out, cuda_fail(e, "execute_host sync"));
  return LPBP_OK;
}

int lpbp_naive_workspace_bytes(int32_t nt, int32_t ntheta, int32_t batch, size_t* bytes) {
  if (!bytes || nt < 2 || ntheta < 1 || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  *bytes = lpbp::direct_geom(nt, ntheta, 2, batch).ws_bytes;  // independent of n
  return LPBP_OK;
}

int lpbp_naive_backproject(const float* sino_dev, float* img_dev, int32_t nt, int32_t ntheta, int32_t n,
                           int32_t batch, float* ws_dev, void* stream) {
  g_launches = 0;
  if (batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (n < 2) return fail(LPBP_EINVAL, "n must be >= 2");
  if (nt < 2 || ntheta < 1) return fail(LPBP_EINVAL, "nt must be >= 2 and ntheta >= 1");
  if (batch == 0) return LPBP_OK;
  if (!sino_dev || !img_dev || !ws_dev) return fail(LPBP_EINVAL, "invalid argument");
  if (reinterpret_cast<uintptr_t>(ws_dev) % 256) return fail(LPBP_EINVAL, "workspace must be 256-byte aligned");
  const lpbp::DirectGeom g = lpbp::direct_geom(nt, ntheta, n, batch);
  cudaError_t e = lpbp::launch_direct(g, sino_dev, ws_dev, img_dev, batch, static_cast<cudaStream_t>(stream));
  g_launches += 2;
  if (e) return cuda_fail(e, "naive_backproject");
  return LPBP_OK;
}

int lpbp_plan_table(const lpbp_plan* P, const char* which, void* dst, size_t capacity, size_t* count) {
  if (!P || !which || !count) return fail(LPBP_EINVAL, "invalid argument");
  const HostPlan& h = P->h;
  if (!std::strcmp(which, "kernel_cells")) {
    *count = h.cell_k.size();
    if (dst) {
      int32_t* o = static_cast<int32_t*>(dst);
      for (size_t i = 0; i < std::min(capacity, *count); ++i) {
        o[2 * i] = h.cell_k[i];
        o[2 * i + 1] = h.cell_l[i];
      }
    }
    return LPBP_OK;
  }
  if (!std::strcmp(which, "ramp")) {
    *count = h.ramp.size();
    if (dst) std::memcpy(dst, h.ramp.data(), std::min(capacity, *count) * sizeof(float));
    return LPBP_OK;
  }
  if (!std::strcmp(which, "khat")) {
    *count = h.khat.size();
    if (dst) std::memcpy(dst, h.khat.data(), std::min(capacity, *count) * sizeof(lpbp::F2));
    return LPBP_OK;
  }
  auto copy_vec = [&](const auto& v) {
    *count = v.size();
    if (dst) std::memcpy(dst, v.data(), std::min(capacity, *count) * sizeof(v[0]));
    return LPBP_OK;
  };
  if (!std::strcmp(which, "ab")) return copy_vec(h.ab);         // int32 pairs (a_k, b_k)
  if (!std::strcmp(which, "wab")) return copy_vec(h.wab);       // float quads
  if (!std::strcmp(which, "ptile")) return copy_vec(h.ptile);   // int32 [ns]: {a_lo, na, b_lo, nb} per 4 semi-polar rows
  if (!std::strcmp(which, "ploc")) return copy_vec(h.ploc);     // uint32 [ns]: tap rows inside the tile's ranges
  if (!std::strcmp(which, "ki")) return copy_vec(h.ki);         // int32
  if (!std::strcmp(which, "wi")) return copy_vec(h.wi);         // float pairs
  if (!std::strcmp(which, "qidx")) return copy_vec(h.qidx);     // uint32
  if (!std::strcmp(which, "qw")) return copy_vec(h.qw);         // float pairs
  if (!std::strcmp(which, "chirp")) return copy_vec(h.chirp);      // float2 nphi (generic sizes)
  if (!std::strcmp(which, "bhat_f")) return copy_vec(h.bhat_f);    // float2 MB
  if (!std::strcmp(which, "bhat_i")) return copy_vec(h.bhat_i);    // float2 MB
  if (!std::strcmp(which, "band_off")) return copy_vec(h.band_off);          // uint32 nbands+1
  if (!std::strcmp(which, "band_entries")) return copy_vec(h.band_entries);  // uint32
  if (!std::strcmp(which, "band_need")) return copy_vec(h.band_need);        // uint32 nbands
  if (!std::strcmp(which, "units")) return copy_vec(h.units);                // uint32 pairs [k0, k1), outermost first
  if (!std::strcmp(which, "row_need")) return copy_vec(h.row_need);          // uint32 bitmap over log-polar rows
  if (!std::strcmp(which, "rowmap_cp")) return copy_vec(h.rowmap_cp);        // int32 [row_end]: compacted position or -1
  if (!std::strcmp(which, "rowmap_id")) return copy_vec(h.rowmap_id);        // int32 [row_end]: the row itself or -1
  if (!std::strcmp(which, "band_row_cp")) return copy_vec(h.band_row_cp);    // uint32 [nbands]: 1 + compacted first row, 0 = unneeded
  if (!std::strcmp(which, "band_row_id")) return copy_vec(h.band_row_id);    // uint32 [nbands]: 1 + first row, 0 = unneeded
  return fail(LPBP_EINVAL, std::string("unknown table ") + which);
}

int lpbp_profile_enable(lpbp_plan* P, int32_t enable) {
  if (!P) return fail(LPBP_EINVAL, "invalid argument");
  std::lock_guard<std::mutex> lk(P->prof_mu);
  P->profiling = enable != 0;
  return LPBP_OK;
}

int lpbp_profile_read(lpbp_plan* P, double* stage_ms, int64_t* stage_launches, int64_t* stage_slices,
                      int32_t nstages) {
  if (!P || !stage_ms || !stage_launches || !stage_slices || nstages < kStages)
    return fail(LPBP_EINVAL, "invalid argument");
  DeviceGuard g(P->device);
  std::lock_guard<std::mutex> lk(P->prof_mu);
  for (int i = 0; i < nstages; ++i) {
    stage_ms[i] = 0;
    stage_launches[i] = 0;
    stage_slices[i] = 0;
  }
  int rc = LPBP_OK;
  for (auto& r : P->recs) {
    cudaError_t e = cudaEventSynchronize(r.b);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
    if (e != cudaSuccess && rc == LPBP_OK) rc = cuda_fail(e, "profile_read");
    stage_ms[r.stage] += ms;
    stage_launches[r.stage] += 1;
    stage_slices[r.stage] += r.slices;
    P->ev_pool.push_back(r.a);
    P->ev_pool.push_back(r.b);
  }
  P->recs.clear();
  return rc;
}

extern "C++" {
namespace {
template <typename OutT>
int radon_ellipses_abi(const double* params_dev, int32_t k, int32_t nt, int32_t ntheta, int32_t batch, OutT* out_dev,
                       void* stream) {
  if (!params_dev || !out_dev || k < 1 || nt < 2 || ntheta < 1 || batch < 0 || batch > 65535)
    return fail(LPBP_EINVAL, "invalid argument");
  if (batch == 0) return LPBP_OK;
  cudaError_t e = lpbp::launch_radon_ellipses(params_dev, k, nt, ntheta, batch, out_dev,
                                              static_cast<cudaStream_t>(stream));
  if (e) return cuda_fail(e, "radon_ellipses");
  return LPBP_OK;
}
}  // namespace
}  // extern "C++"

int lpbp_radon_ellipses(const double* params_dev, int32_t k, int32_t nt, int32_t ntheta, int32_t batch,
                        float* out_dev, void* stream) {
  return radon_ellipses_abi(params_dev, k, nt, ntheta, batch, out_dev, stream);
}

int lpbp_radon_ellipses_f64(const double* params_dev, int32_t k, int32_t nt, int32_t ntheta, int32_t batch,
                            double* out_dev, void* stream) {
  return radon_ellipses_abi(params_dev, k, nt, ntheta, batch, out_dev, stream);
}

int lpbp_radon_ellipses_host(const double* params, int32_t k, int32_t nt, int32_t ntheta, int32_t batch, double* out,
                             int32_t device) {
  if (!params || !out || k < 1 || nt < 2 || ntheta < 1 || batch < 0 || batch > 65535 || device < 0)
    return fail(LPBP_EINVAL, "invalid argument");
  if (batch == 0) return LPBP_OK;
  DeviceGuard g(device);
  if (!g.ok) return fail(LPBP_ECUDA, "cannot select the device");
  const size_t pb = (size_t)batch * k * 6 * sizeof(double), ob = (size_t)batch * nt * ntheta * sizeof(double);
  void *dp = nullptr, *dout = nullptr;
  cudaError_t e = cudaMalloc(&dp, pb);
  if (!e) e = cudaMalloc(&dout, ob);
  if (!e) e = cudaMemcpy(dp, params, pb, cudaMemcpyHostToDevice);
  if (!e) e = lpbp::launch_radon_ellipses(static_cast<const double*>(dp), k, nt, ntheta, batch,
                                          static_cast<double*>(dout), nullptr);
  if (!e) e = cudaMemcpy(out, dout, ob, cudaMemcpyDeviceToHost);
  if (dp) cudaFree(dp);
  if (dout) cudaFree(dout);
  if (e) return cuda_fail(e, "radon_ellipses_host");
  return LPBP_OK;
}


// ---------------------------------------------------------------------------
// sector (partial) backprojection
// ---------------------------------------------------------------------------
}  // extern "C"

// Host-to-host pipeline shared by the sector and BST plans: two device staging slots, chunk k+1's
// H2D and chunk k-1's D2H on their own streams beside chunk k's kernels (the log-polar plan's
// lpbp_execute_host does the same with its own workspace layout).
struct HostPipe {
  int chunk = 0;
  size_t ws_bytes = 0;
  float* in[2] = {nullptr, nullptr};
  float* out[2] = {nullptr, nullptr};
  void* ws = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  std::mutex mu;
  void release() {  // the owner's device must be current
    for (int i = 0; i < 2; ++i) {
      if (in[i]) cudaFree(in[i]);
      if (out[i]) cudaFree(out[i]);
      if (ev_in[i]) cudaEventDestroy(ev_in[i]);
      if (ev_comp[i]) cudaEventDestroy(ev_comp[i]);
      if (ev_out[i]) cudaEventDestroy(ev_out[i]);
      in[i] = out[i] = nullptr;
      ev_in[i] = ev_comp[i] = ev_out[i] = nullptr;
    }
    if (ws) cudaFree(ws);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_comp) cudaStreamDestroy(s_comp);
    if (s_out) cudaStreamDestroy(s_out);
    ws = nullptr;
    s_in = s_comp = s_out = nullptr;
    chunk = 0;
    ws_bytes = 0;
  }
};

// run(in_dev, out_dev, c, ws, ws_bytes, stream) -> LPBP status; counts its launches in g_launches
template <typename Run>
int host_pipeline(HostPipe& pp, int batch, int chunk, size_t in_slice, size_t out_slice, size_t ws_bytes,
                  const float* sino_host, float* img_host, Run&& run) {
  std::lock_guard<std::mutex> lk(pp.mu);
  if (pp.chunk < chunk || pp.ws_bytes < ws_bytes) {
    pp.release();
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaMalloc(&pp.in[i], in_slice * chunk * sizeof(float));
      if (e == cudaSuccess) e = cudaMalloc(&pp.out[i], out_slice * chunk * sizeof(float));
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pp.ev_in[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pp.ev_comp[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pp.ev_out[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaMalloc(&pp.ws, ws_bytes);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pp.s_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pp.s_comp, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&pp.s_out, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      pp.release();
      return cuda_fail(e, "host pipeline setup");
    }
    pp.chunk = chunk;
    pp.ws_bytes = ws_bytes;
  }
  int64_t launches = 0;
  const int nchunks = (batch + chunk - 1) / chunk;
  for (int ci = 0; ci < nchunks; ++ci) {
    const int slot = ci & 1;
    const int off = ci * chunk;
    const int c = std::min(chunk, batch - off);
    if (ci >= 2) cudaStreamWaitEvent(pp.s_in, pp.ev_comp[slot], 0);  // slot's previous input consumed
    cudaError_t e = cudaMemcpyAsync(pp.in[slot], sino_host + (size_t)off * in_slice, in_slice * c * sizeof(float),
                                    cudaMemcpyHostToDevice, pp.s_in);
    if (e) return drain_streams(pp.s_in, pp.s_comp, pp.s_out, cuda_fail(e, "H2D"));
    cudaEventRecord(pp.ev_in[slot], pp.s_in);
    cudaStreamWaitEvent(pp.s_comp, pp.ev_in[slot], 0);
    if (ci >= 2) cudaStreamWaitEvent(pp.s_comp, pp.ev_out[slot], 0);  // slot's previous output copied out
    g_launches = 0;
    const int rc = run(pp.in[slot], pp.out[slot], c, pp.ws, pp.ws_bytes, pp.s_comp);
    if (rc) return drain_streams(pp.s_in, pp.s_comp, pp.s_out, rc);
    launches += g_launches;
    cudaEventRecord(pp.ev_comp[slot], pp.s_comp);
    cudaStreamWaitEvent(pp.s_out, pp.ev_comp[slot], 0);
    e = cudaMemcpyAsync(img_host + (size_t)off * out_slice, pp.out[slot], out_slice * c * sizeof(float),
                        cudaMemcpyDeviceToHost, pp.s_out);
    if (e) return drain_streams(pp.s_in, pp.s_comp, pp.s_out, cuda_fail(e, "D2H"));
    cudaEventRecord(pp.ev_out[slot], pp.s_out);
  }
  cudaError_t e = cudaStreamSynchronize(pp.s_out);
  if (e == cudaSuccess) e = cudaStreamSynchronize(pp.s_comp);
  if (e) return drain_streams(pp.s_in, pp.s_comp, pp.s_out, cuda_fail(e, "execute_host sync"));
  g_launches = launches;
  return LPBP_OK;
}

struct lpbp_sector_plan {
  lpbp::SectorSetHost h;
  // log-polar stage per sector (explicit rho0, no filter).  Sectors whose meshes coincide
  // (same rho0_s and nrho_s, e.g. equal beta and a_r) share one plan and run as one batch.
  std::vector<lpbp_plan*> sub;     // per sector (aliases the group's plan)
  std::vector<lpbp_plan*> owned;   // one per group
  std::vector<std::vector<int>> groups;  // sector indices per group
  std::vector<const lpbp::SectorCol*> cols;   // full-width (reference layout; stage API)
  std::vector<const lpbp::SectorCol*> ccols;  // compacted (execute)
  std::vector<const lpbp::SectorRow*> rows;
  std::vector<size_t> own_table_bytes;
  std::vector<void*> allocs;
  int device = 0;
  std::mutex mu;
  void* own_ws = nullptr;
  size_t own_ws_bytes = 0;
  HostPipe pipe;  // host path (lpbp_sector_execute_host)
  ~lpbp_sector_plan() {
    DeviceGuard g(device);
    pipe.release();
    for (auto* p : owned) delete p;
    for (void* p : allocs) cudaFree(p);
    if (own_ws) cudaFree(own_ws);
  }
};

namespace {

// [working sinograms of the largest group][log-polar images, per group: members x chunk][sub-plan ws]
size_t sector_ws_bytes(const lpbp_sector_plan* P, int chunk) {
  const auto& h = P->h;
  size_t sub = 0, lp = 0, work = 0;
  for (size_t g = 0; g < P->groups.size(); ++g) {
    const lpbp_plan* S = P->owned[g];
    const size_t m = P->groups[g].size();
    work = std::max(work, m * chunk * h.nt * (size_t)h.sec[P->groups[g][0]].wpad);
    sub = std::max(sub, ws_bytes_for(S, (int)(m * chunk)));
    lp += align256(m * chunk * S->d.nrho * S->d.nphi * sizeof(float));
  }
  return align256(work * sizeof(float)) + lp + sub;
}

int sector_chunk(const lpbp_sector_plan* P, const float* in, float* out, int c, char* ws, cudaStream_t st) {
  const auto& h = P->h;
  size_t work_floats = 0;
  for (const auto& g : P->groups) work_floats = std::max(work_floats, g.size() * c * h.nt * (size_t)h.sec[g[0]].wpad);
  float* work = reinterpret_cast<float*>(ws);
  char* cur = ws + align256(work_floats * sizeof(float));
  lpbp::SectorArgs args{};
  const int nsec = (int)P->sub.size();
  std::vector<float*> lp_group(P->groups.size());
  for (size_t g = 0; g < P->groups.size(); ++g) {
    const lpbp_plan* S = P->owned[g];
    const size_t per = (size_t)c * S->d.nrho * S->d.nphi;  // one sector's images for the chunk
    lp_group[g] = reinterpret_cast<float*>(cur);
    for (size_t k = 0; k < P->groups[g].size(); ++k) {
      const int s = P->groups[g][k];
      auto& a = args.s[s];
      a.lp = lp_group[g] + k * per;
      a.lp_slice = (long long)S->d.nrho * S->d.nphi;
      a.nrho = S->d.nrho;
      a.rho0 = S->h.rho0;
      a.drho = S->h.drho;
      a.ct = std::cos(h.sec[s].theta_c);
      a.st = std::sin(h.sec[s].theta_c);
      a.a_r = h.sec[s].spec.a_r;
      a.inv_a = (float)(1.0 / h.sec[s].spec.a_r);
    }
    cur += align256(P->groups[g].size() * per * sizeof(float));
  }
  char* subws = cur;
  for (size_t g = 0; g < P->groups.size(); ++g) {
    const auto& members = P->groups[g];
    const int wpad = h.sec[members[0]].wpad;
    const size_t w_slice = (size_t)h.nt * wpad;
    for (size_t k = 0; k < members.size(); ++k) {  // compacted working sinograms of the group, back to back
      const int s = members[k];
      cudaError_t e = lpbp::launch_sector_prep(in, work + k * c * w_slice, h.nt, wpad, h.ntheta, c, P->ccols[s],
                                               P->rows[s], h.sec[s].spec.a_r, h.sec[s].klo, h.sec[s].khi, st);
      if (e) return launch_fail(e, "sector_prep");
      ++g_launches;
    }
    int rc = run_chunk(P->owned[g], work, nullptr, (int)(members.size() * c), subws, st, true, lp_group[g], wpad,
                       h.sec[members[0]].lo);
    if (rc) return rc;
  }
  cudaError_t e = lpbp::launch_sector_readout(args, nsec, out, h.n, 2 * h.ntheta, c, st);
  if (e) return launch_fail(e, "sector_readout");
  ++g_launches;
  return LPBP_OK;
}

}  // namespace

extern "C" {

int lpbp_sector_plan_create(int32_t nt, int32_t ntheta, int32_t n_out, const lpbp_sector* sectors,
                            int32_t nsectors, int32_t device, lpbp_sector_plan** plan) {
  g_last_error.clear();
  if (!plan || nsectors < 0 || (nsectors > 0 && !sectors)) return fail(LPBP_EINVAL, "invalid argument");
  *plan = nullptr;
  if (nsectors > lpbp::kMaxSectors)
    return fail(LPBP_EINVAL, "at most " + std::to_string(lpbp::kMaxSectors) + " sectors per plan");
  std::vector<lpbp::SectorSpec> specs;
  for (int i = 0; i < nsectors; ++i) specs.push_back({sectors[i].theta0, sectors[i].beta, sectors[i].a_r});
  auto* P = new (std::nothrow) lpbp_sector_plan();
  if (!P) return fail(LPBP_ENOMEM, "host allocation failed");
  std::string err = lpbp::build_sector_set(nt, ntheta, n_out, specs, P->h);
  if (!err.empty()) {
    delete P;
    return fail(LPBP_EINVAL, err);
  }
  P->device = device;
  for (size_t q = 0; q < P->h.sec.size(); ++q) {
    const auto& S = P->h.sec[q];
    bool shared = false;  // an existing plan with the same mesh
    for (size_t g = 0; g < P->groups.size() && !shared; ++g) {
      const lpbp_plan* o = P->owned[g];
      const auto& S0 = P->h.sec[P->groups[g][0]];
      if (o->h.rho0 == S.rho0 && o->h.nrho == S.nrho && S0.wpad == S.wpad && S0.lo == S.lo) {
        P->groups[g].push_back((int)q);
        P->sub.push_back(P->owned[g]);
        shared = true;
      }
    }
    if (shared) continue;
    lpbp_params sp{};
    sp.nt = nt;
    sp.ntheta = ntheta;
    sp.n_out = 2;  // the sub-plan's own Cartesian readout is never used
    sp.has_rho0 = 1;
    sp.rho0 = S.rho0;
    sp.nrho = S.nrho;
    sp.filter = 0;
    sp.device = device;
    lpbp_plan* sub = nullptr;
    int rc = lpbp_plan_create(&sp, &sub);
    if (rc) {
      std::string msg = g_last_error;
      delete P;
      return fail(rc, msg);
    }
    P->owned.push_back(sub);
    P->groups.push_back({(int)q});
    P->sub.push_back(sub);
  }
  if (device >= 0) {
    DeviceGuard g(device);
    for (const auto& S : P->h.sec) {
      void *c = nullptr, *cc = nullptr, *r = nullptr;
      const size_t cb = S.cols.size() * sizeof(lpbp::SectorCol), ccb = S.ccols.size() * sizeof(lpbp::SectorCol);
      const size_t rb = S.rows.size() * sizeof(lpbp::SectorRow);
      cudaError_t e = cudaMalloc(&c, cb);
      if (e == cudaSuccess) P->allocs.push_back(c);
      if (e == cudaSuccess) e = cudaMalloc(&cc, ccb);
      if (e == cudaSuccess) P->allocs.push_back(cc);
      if (e == cudaSuccess) e = cudaMalloc(&r, rb);
      if (e == cudaSuccess) P->allocs.push_back(r);
      if (e == cudaSuccess) e = cudaMemcpy(c, S.cols.data(), cb, cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = cudaMemcpy(cc, S.ccols.data(), ccb, cudaMemcpyHostToDevice);
      if (e == cudaSuccess) e = cudaMemcpy(r, S.rows.data(), rb, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) {
        delete P;
        return cuda_fail(e, "sector tables");
      }
      P->cols.push_back(static_cast<const lpbp::SectorCol*>(c));
      P->ccols.push_back(static_cast<const lpbp::SectorCol*>(cc));
      P->rows.push_back(static_cast<const lpbp::SectorRow*>(r));
      P->own_table_bytes.push_back(cb + ccb + rb);
    }
  } else {
    P->own_table_bytes.assign(P->h.sec.size(), 0);
  }
  *plan = P;
  return LPBP_OK;
}

void lpbp_sector_plan_destroy(lpbp_sector_plan* plan) { delete plan; }

int lpbp_sector_get_info(const lpbp_sector_plan* P, int32_t index, lpbp_sector_info* info) {
  if (!P || !info || index < 0 || index >= (int)P->sub.size()) return fail(LPBP_EINVAL, "invalid argument");
  const auto& S = P->h.sec[index];
  const lpbp_plan* sub = P->sub[index];
  info->jc = S.jc;
  info->nrho = sub->h.nrho;
  info->L = sub->h.L;
  info->nphi = sub->h.nphi;
  info->theta_c = S.theta_c;
  info->rho0 = sub->h.rho0;
  info->drho = sub->h.drho;
  info->support_min = S.support_min;
  info->a_r = S.spec.a_r;
  info->table_bytes = sub->table_bytes + P->own_table_bytes[index];
  return LPBP_OK;
}

int lpbp_sector_workspace_bytes(const lpbp_sector_plan* P, int32_t chunk, size_t* bytes) {
  if (!P || !bytes || chunk < 1) return fail(LPBP_EINVAL, "invalid argument");
  *bytes = sector_ws_bytes(P, chunk);
  return LPBP_OK;
}

int lpbp_sector_execute(lpbp_sector_plan* P, const float* sino_dev, float* img_dev, int32_t batch, void* ws,
                        size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (!P || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (batch == 0) return LPBP_OK;
  if (!sino_dev || !img_dev) return fail(LPBP_EINVAL, "invalid argument");
  if (ws && reinterpret_cast<uintptr_t>(ws) % 256) return fail(LPBP_EINVAL, "workspace must be 256-byte aligned");
  DeviceGuard g(P->device);
  std::unique_lock<std::mutex> lock(P->mu, std::defer_lock);
  if (!ws) {
    lock.lock();
    const size_t need = sector_ws_bytes(P, std::max(1, std::min((int)batch, 8)));
    if (P->own_ws_bytes < need) {
      if (P->own_ws) cudaFree(P->own_ws);
      P->own_ws = nullptr;
      P->own_ws_bytes = 0;
      cudaError_t e = cudaMalloc(&P->own_ws, need);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(sector workspace)");
      P->own_ws_bytes = need;
    }
    ws = P->own_ws;
    ws_bytes = P->own_ws_bytes;
  }
  int chunk = 1;
  while (chunk < batch && sector_ws_bytes(P, chunk + 1) <= ws_bytes) ++chunk;
  if (sector_ws_bytes(P, chunk) > ws_bytes)
    return fail(LPBP_EINVAL, "workspace too small for one slice (need " + std::to_string(sector_ws_bytes(P, 1)) +
                                 " bytes)");
  const size_t in_slice = (size_t)P->h.nt * P->h.ntheta, out_slice = (size_t)P->h.n * P->h.n;
  int64_t launches = 0;
  for (int off = 0; off < batch; off += chunk) {
    const int c = std::min(chunk, batch - off);
    int rc = sector_chunk(P, sino_dev + off * in_slice, img_dev + off * out_slice, c, static_cast<char*>(ws),
                          static_cast<cudaStream_t>(stream));
    if (rc) return rc;
    launches += g_launches;
    g_launches = 0;
  }
  g_launches = launches;
  return LPBP_OK;
}

int lpbp_sector_execute_host(lpbp_sector_plan* P, const float* sino_host, float* img_host, int32_t batch,
                             int32_t chunk) {
  g_launches = 0;
  if (!P || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (batch == 0) return LPBP_OK;
  if (!sino_host || !img_host) return fail(LPBP_EINVAL, "invalid argument");
  if (chunk <= 0) chunk = 4;
  chunk = std::min(chunk, batch);
  DeviceGuard g(P->device);
  const size_t in_slice = (size_t)P->h.nt * P->h.ntheta, out_slice = (size_t)P->h.n * P->h.n;
  return host_pipeline(P->pipe, batch, chunk, in_slice, out_slice, sector_ws_bytes(P, chunk), sino_host, img_host,
                       [&](const float* in, float* out, int c, void* ws, size_t wsb, cudaStream_t st) {
                         return lpbp_sector_execute(P, in, out, c, ws, wsb, st);
                       });
}

int lpbp_sector_prepare(const lpbp_sector_plan* P, int32_t index, const float* sino_dev, float* out_dev,
                        int32_t batch, void* stream) {
  g_launches = 0;
  if (!P || batch < 0 || index < 0 || index >= (int)P->sub.size()) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (batch == 0) return LPBP_OK;
  if (!sino_dev || !out_dev) return fail(LPBP_EINVAL, "invalid argument");
  DeviceGuard g(P->device);
  const auto& S = P->h.sec[index];
  cudaError_t e = lpbp::launch_sector_prep(sino_dev, out_dev, P->h.nt, P->h.ntheta, P->h.ntheta, batch,
                                           P->cols[index], P->rows[index], S.spec.a_r, S.klo, S.khi,
                                           static_cast<cudaStream_t>(stream));
  if (e) return launch_fail(e, "sector_prep");
  ++g_launches;
  return LPBP_OK;
}

int lpbp_sector_logpolar(const lpbp_sector_plan* P, int32_t index, const float* work_dev, float* lp_dev,
                         int32_t batch, void* stream) {
  if (!P || index < 0 || index >= (int)P->sub.size()) return fail(LPBP_EINVAL, "invalid argument");
  return lpbp_logpolar(P->sub[index], work_dev, lp_dev, batch, nullptr, 0, stream);
}


// ---------------------------------------------------------------------------
// BST engine
// ---------------------------------------------------------------------------
}  // extern "C"

struct lpbp_bst_plan {
  lpbp::BstHost h;
  lpbp::BstDims d{};
  lpbp::BstTables t{};
  Dims rd{};        // ramp-filter dims (fbp)
  DevTables rt{};   // ramp-filter tables (fbp)
  int device = 0;
  std::vector<void*> allocs;
  size_t table_bytes = 0;
  std::mutex mu;
  void* own_ws = nullptr;
  size_t own_ws_bytes = 0;
  HostPipe pipe;  // host path (lpbp_bst_execute_host)
  // optional per-stage CUDA-event profiling (lpbp_bst_profile_enable / _read):
  // ev[0..4] = before ramp, before radial, before grid_x, between grid_x and grid_y, after grid_y
  struct Rec { int slices; bool ramp; cudaEvent_t ev[5]; };
  bool profiling = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> ev_pool;
  std::mutex prof_mu;
  cudaEvent_t take_event() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  template <typename T>
  int upload(const std::vector<T>& v, const void** dst) {
    void* p = nullptr;
    const size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(bst table)");
    allocs.push_back(p);
    if (!v.empty()) e = cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(bst table)");
    table_bytes += bytes;
    *dst = p;
    return LPBP_OK;
  }
  int twiddles(int N, const float2** dst) {
    const int len = lpbp::twiddle_table_len(N);
    if (len < 0) return fail(LPBP_EUNSUPPORTED, "no FFT plan for size " + std::to_string(N));
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)len * sizeof(float2));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(twiddles)");
    allocs.push_back(p);
    e = lpbp::launch_init_twiddles(N, static_cast<float2*>(p), nullptr);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, "init_twiddles");
    table_bytes += (size_t)len * sizeof(float2);
    *dst = static_cast<const float2*>(p);
    return LPBP_OK;
  }
  ~lpbp_bst_plan() {
    DeviceGuard g(device);
    pipe.release();
    for (auto& r : recs)
      for (cudaEvent_t e : r.ev) ev_pool.push_back(e);
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    for (void* p : allocs) cudaFree(p);
    if (own_ws) cudaFree(own_ws);
  }
};

namespace {

// per slice: filtered sinogram (fbp) | P [nray/2 + 2][m_pad] ray pairs | X [n][big/2] complex; + 2 doubles per slice
size_t bst_slice_bytes(const lpbp::BstHost& h, size_t* off_p, size_t* off_x) {
  const size_t f = h.p.filter ? align256((size_t)h.p.nt * h.p.ntheta * sizeof(float)) : 0;
  const size_t pb = align256((size_t)(h.nray + 4) * h.m_pad * sizeof(float2));
  const size_t xb = align256((size_t)h.p.n * (h.big / 2) * sizeof(float2));
  if (off_p) *off_p = f;
  if (off_x) *off_x = f + pb;
  return f + pb + xb;
}
size_t bst_ws_bytes(const lpbp_bst_plan* P, int chunk) {
  return bst_slice_bytes(P->h, nullptr, nullptr) * chunk + align256((size_t)chunk * 2 * sizeof(double));
}

int bst_chunk(const lpbp_bst_plan* P, const float* in, float* out, int c, char* ws, cudaStream_t st,
              float2* spectra_only) {
  const auto& h = P->h;
  size_t off_p, off_x;
  const size_t per = bst_slice_bytes(h, &off_p, &off_x);
  (void)per;
  // regions laid out per chunk: [filtered c slices][P c slices][X c slices][acc]
  const size_t fb = h.p.filter ? align256((size_t)h.p.nt * h.p.ntheta * sizeof(float)) : 0;
  const size_t pb = align256((size_t)(h.nray + 4) * h.m_pad * sizeof(float2));
  const size_t xb = align256((size_t)h.p.n * (h.big / 2) * sizeof(float2));
  float* filt = reinterpret_cast<float*>(ws);
  float2* Pw = spectra_only ? spectra_only : reinterpret_cast<float2*>(ws + fb * c);
  float2* Xw = reinterpret_cast<float2*>(ws + (fb + pb) * c);
  double* acc = reinterpret_cast<double*>(ws + (fb + pb + xb) * c);
  cudaError_t e = cudaMemsetAsync(acc, 0, (size_t)c * 2 * sizeof(double), st);
  if (e) return cuda_fail(e, "bst acc");
  const float* src = in;
  lpbp_bst_plan* Pm = const_cast<lpbp_bst_plan*>(P);
  std::unique_lock<std::mutex> plk(Pm->prof_mu, std::defer_lock);
  lpbp_bst_plan::Rec rec{c, false, {}};
  const bool prof = Pm->profiling && !spectra_only;
  if (prof) {
    plk.lock();
    for (auto& ev : rec.ev) ev = Pm->take_event();
    cudaEventRecord(rec.ev[0], st);
  }
  // error exits hand the events taken for this chunk back to the pool
  auto fail_chunk = [&](cudaError_t err, const char* where) {
    if (prof)
      for (cudaEvent_t ev : rec.ev) Pm->ev_pool.push_back(ev);
    return launch_fail(err, where);
  };
  if (h.p.filter && !spectra_only) {
    rec.ramp = true;
    e = lpbp::launch_ramp(P->rd, P->rt, in, filt, c, st);  // column tiles need ntheta % TC == 0
    if (e == cudaErrorNotSupported) {
      (void)cudaGetLastError();
      e = lpbp::launch_ramp_generic(P->rd, P->rt, in, filt, c, st);
    }
    if (e) return fail_chunk(e, "bst ramp_filter");
    ++g_launches;
    src = filt;
  }
  if (prof) cudaEventRecord(rec.ev[1], st);
  e = lpbp::launch_bst_radial(P->d, P->t, src, Pw, acc, c, st);
  if (e) return fail_chunk(e, "bst_radial");
  ++g_launches;
  if (spectra_only) return LPBP_OK;
  if (prof) cudaEventRecord(rec.ev[2], st);
  e = lpbp::launch_bst_grid(P->d, P->t, Pw, Xw, out, acc, c, st, prof ? rec.ev[3] : nullptr);
  if (e) return fail_chunk(e, "bst_grid");
  g_launches += 2;
  if (prof) {
    cudaEventRecord(rec.ev[4], st);
    Pm->recs.push_back(rec);
  }
  return LPBP_OK;
}

}  // namespace

extern "C" {

int lpbp_bst_profile_enable(lpbp_bst_plan* P, int32_t enable) {
  if (!P) return fail(LPBP_EINVAL, "invalid argument");
  std::lock_guard<std::mutex> lk(P->prof_mu);
  P->profiling = enable != 0;
  return LPBP_OK;
}

int lpbp_bst_profile_read(lpbp_bst_plan* P, double* stage_ms, int64_t* stage_launches, int64_t* stage_slices,
                          int32_t nstages) {
  constexpr int kBstStages = 4;  // ramp filter, radial, grid_x, grid_y
  if (!P || !stage_ms || !stage_launches || !stage_slices || nstages < kBstStages)
    return fail(LPBP_EINVAL, "invalid argument");
  DeviceGuard g(P->device);
  std::lock_guard<std::mutex> lk(P->prof_mu);
  for (int i = 0; i < nstages; ++i) {
    stage_ms[i] = 0;
    stage_launches[i] = 0;
    stage_slices[i] = 0;
  }
  int rc = LPBP_OK;
  for (auto& r : P->recs) {
    cudaError_t e = cudaEventSynchronize(r.ev[4]);
    for (int k = 0; k < kBstStages; ++k) {
      if (k == 0 && !r.ramp) continue;
      float ms = 0.f;
      if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.ev[k], r.ev[k + 1]);
      stage_ms[k] += ms;
      stage_launches[k] += 1;
      stage_slices[k] += r.slices;
    }
    if (e != cudaSuccess && rc == LPBP_OK) rc = cuda_fail(e, "bst profile_read");
    for (cudaEvent_t ev : r.ev) P->ev_pool.push_back(ev);
  }
  P->recs.clear();
  return rc;
}

int lpbp_bst_plan_create(const lpbp_bst_params* params, lpbp_bst_plan** plan) {
  g_last_error.clear();
  if (!params || !plan) return fail(LPBP_EINVAL, "null argument");
  *plan = nullptr;
  lpbp::BstParams bp{params->nt, params->ntheta, params->n_out, params->beta, params->zero_pad, params->dc_mode,
                     params->filter != 0, params->lam, params->cutoff};
  auto* P = new (std::nothrow) lpbp_bst_plan();
  if (!P) return fail(LPBP_ENOMEM, "host allocation failed");
  std::string err = lpbp::build_bst_host(bp, P->h);
  if (!err.empty()) {
    delete P;
    return fail(LPBP_EINVAL, err);
  }
  const auto& h = P->h;
  P->device = params->device;
  if (params->device >= 0 && !h.supported) {
    const int n = h.p.n, L = h.L;
    delete P;
    return fail(LPBP_EUNSUPPORTED, "BST engine: no kernel instantiation for radial DFT length L=" + std::to_string(L) +
                                       " / padded side " + std::to_string(2 * n) +
                                       " (this build: L a power of two in [512, 8192] or L <= 4096; padded side a "
                                       "power of two in [128, 4096] or <= 4096; even nt)");
  }
  auto& d = P->d;
  d.nt = h.p.nt;
  d.ntheta = h.p.ntheta;
  d.n = h.p.n;
  d.ns = h.ns;
  d.nray = h.nray;
  d.L = h.L;
  d.m_need = h.m_need;
  d.m_pad = h.m_pad;
  d.big = h.big;
  d.p0 = h.p0;
  d.mb_L = h.mb_L;
  d.mb_big = h.mb_big;
  d.subtract_mean = h.p.dc_mode == 0 ? 1 : 0;
  d.dsigma = h.dsigma;
  d.dw = h.dw;
  d.s_img = (float)h.out_scale;
  d.fbp = h.p.filter ? (float)(1.0 / (2.0 * 3.14159265358979323846)) : 1.f;
  d.s_mean = (float)(h.out_scale / d.fbp);
  if (P->device >= 0) {
    DeviceGuard g(P->device);
    if (!g.ok) {
      delete P;
      return fail(LPBP_ECUDA, "cannot select CUDA device " + std::to_string(params->device));
    }
    int rc = LPBP_OK;
    const void* p;
    rc = rc ? rc : P->upload(h.tap_base, &p);
    if (!rc) P->t.tap_base = static_cast<const int2*>(p);
    rc = rc ? rc : P->upload(h.tap_w, &p);
    if (!rc) P->t.tap_w = static_cast<const float4*>(p);
    rc = rc ? rc : P->upload(h.kern, &p);
    if (!rc) P->t.kern = static_cast<const float*>(p);
    rc = rc ? rc : P->upload(h.tau, &p);
    if (!rc) P->t.tau = static_cast<const float2*>(p);
    rc = rc ? rc : P->upload(h.cmean, &p);
    if (!rc) P->t.cmean = static_cast<const float2*>(p);
    rc = rc ? rc : P->upload(h.chord_col, &p);
    if (!rc) P->t.chord = h.chord_col.empty() ? nullptr : static_cast<const float4*>(p);
    rc = rc ? rc : P->upload(h.grid_q, &p);
    if (!rc) P->t.grid_q = static_cast<const uint2*>(p);
    if (h.mb_L) {
      rc = rc ? rc : P->twiddles(h.mb_L, &P->t.tw_mbL);
      rc = rc ? rc : P->upload(h.chirp_L, &p);
      if (!rc) P->t.chirp_L = static_cast<const float2*>(p);
      rc = rc ? rc : P->upload(h.bhat_L, &p);
      if (!rc) P->t.bhat_L = static_cast<const float2*>(p);
    } else {
      rc = rc ? rc : P->twiddles(h.L, &P->t.tw_L);
    }
    if (h.mb_big) {
      rc = rc ? rc : P->twiddles(h.mb_big, &P->t.tw_mbbig);
      rc = rc ? rc : P->upload(h.chirp_big, &p);
      if (!rc) P->t.chirp_big = static_cast<const float2*>(p);
      rc = rc ? rc : P->upload(h.bhat_big, &p);
      if (!rc) P->t.bhat_big = static_cast<const float2*>(p);
    } else {
      rc = rc ? rc : P->twiddles(h.big, &P->t.tw_big);
    }
    if (h.p.filter) {
      rc = rc ? rc : P->upload(h.ramp, &p);
      if (!rc) P->rt.ramp = static_cast<const float*>(p);
      rc = rc ? rc : P->twiddles(h.M, &P->rt.tw_ramp);
      P->rd.nt = h.p.nt;
      P->rd.ntheta = h.p.ntheta;
      P->rd.M = h.M;
      P->rd.nsm = 148;
      cudaDeviceGetAttribute(&P->rd.nsm, cudaDevAttrMultiProcessorCount, P->device);
    }
    if (rc) {
      std::string msg = g_last_error;
      delete P;
      return fail(rc, msg);
    }
  }
  *plan = P;
  return LPBP_OK;
}

void lpbp_bst_plan_destroy(lpbp_bst_plan* plan) { delete plan; }

int lpbp_bst_get_info(const lpbp_bst_plan* P, lpbp_bst_info* info) {
  if (!P || !info) return fail(LPBP_EINVAL, "null argument");
  const auto& h = P->h;
  info->ns = h.ns;
  info->nray = h.nray;
  info->L = h.L;
  info->m_need = h.m_need;
  info->m_pad = h.m_pad;
  info->big = h.big;
  info->p0 = h.p0;
  info->supported = h.supported ? 1 : 0;
  info->ds = h.ds;
  info->dsigma = h.dsigma;
  info->out_scale = h.out_scale;
  info->table_bytes = P->table_bytes;
  info->workspace_per_slice = bst_ws_bytes(P, 1);
  return LPBP_OK;
}

int lpbp_bst_workspace_bytes(const lpbp_bst_plan* P, int32_t chunk, size_t* bytes) {
  if (!P || !bytes || chunk < 1) return fail(LPBP_EINVAL, "invalid argument");
  *bytes = bst_ws_bytes(P, chunk);
  return LPBP_OK;
}

int lpbp_bst_execute(lpbp_bst_plan* P, const float* sino_dev, float* img_dev, int32_t batch, void* ws,
                     size_t ws_bytes, void* stream) {
  g_launches = 0;
  if (!P || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (batch == 0) return LPBP_OK;
  if (!sino_dev || !img_dev) return fail(LPBP_EINVAL, "invalid argument");
  if (reinterpret_cast<uintptr_t>(sino_dev) % 16) return fail(LPBP_EINVAL, "sinogram pointer must be 16-byte aligned");
  if (ws && reinterpret_cast<uintptr_t>(ws) % 256) return fail(LPBP_EINVAL, "workspace must be 256-byte aligned");
  DeviceGuard g(P->device);
  std::unique_lock<std::mutex> lock(P->mu, std::defer_lock);
  if (!ws) {
    lock.lock();
    const size_t need = bst_ws_bytes(P, std::max(1, std::min((int)batch, 4)));
    if (P->own_ws_bytes < need) {
      if (P->own_ws) cudaFree(P->own_ws);
      P->own_ws = nullptr;
      P->own_ws_bytes = 0;
      cudaError_t e = cudaMalloc(&P->own_ws, need);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(bst workspace)");
      P->own_ws_bytes = need;
    }
    ws = P->own_ws;
    ws_bytes = P->own_ws_bytes;
  }
  int chunk = 1;
  while (chunk < batch && bst_ws_bytes(P, chunk + 1) <= ws_bytes) ++chunk;
  if (bst_ws_bytes(P, chunk) > ws_bytes)
    return fail(LPBP_EINVAL, "workspace too small for one slice (need " + std::to_string(bst_ws_bytes(P, 1)) + " bytes)");
  const size_t in_slice = (size_t)P->h.p.nt * P->h.p.ntheta, out_slice = (size_t)P->h.p.n * P->h.p.n;
  int64_t launches = 0;
  for (int off = 0; off < batch; off += chunk) {
    const int c = std::min(chunk, batch - off);
    int rc = bst_chunk(P, sino_dev + off * in_slice, img_dev + off * out_slice, c, static_cast<char*>(ws),
                       static_cast<cudaStream_t>(stream), nullptr);
    if (rc) return rc;
    launches += g_launches;
    g_launches = 0;
  }
  g_launches = launches;
  return LPBP_OK;
}

int lpbp_bst_execute_host(lpbp_bst_plan* P, const float* sino_host, float* img_host, int32_t batch, int32_t chunk) {
  g_launches = 0;
  if (!P || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (batch == 0) return LPBP_OK;
  if (!sino_host || !img_host) return fail(LPBP_EINVAL, "invalid argument");
  if (chunk <= 0) chunk = 4;
  chunk = std::min(chunk, batch);
  DeviceGuard g(P->device);
  const size_t in_slice = (size_t)P->h.p.nt * P->h.p.ntheta, out_slice = (size_t)P->h.p.n * P->h.p.n;
  return host_pipeline(P->pipe, batch, chunk, in_slice, out_slice, bst_ws_bytes(P, chunk), sino_host, img_host,
                       [&](const float* in, float* out, int c, void* ws, size_t, cudaStream_t st) {
                         return bst_chunk(P, in, out, c, static_cast<char*>(ws), st, nullptr);
                       });
}

int lpbp_bst_radial(const lpbp_bst_plan* P, const float* sino_dev, float* spectra_dev, int32_t batch, void* stream) {
  g_launches = 0;
  if (!P || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (P->device < 0) return fail(LPBP_EINVAL, "host-only plan (device < 0) cannot execute");
  if (batch == 0) return LPBP_OK;
  if (!sino_dev || !spectra_dev) return fail(LPBP_EINVAL, "invalid argument");
  DeviceGuard g(P->device);
  // spectra_dev holds [batch][ntheta + 2][m_pad] ray pairs; the accumulators go to a small scratch
  void* acc = nullptr;
  cudaError_t e = cudaMallocAsync(&acc, (size_t)batch * 2 * sizeof(double) + 256, static_cast<cudaStream_t>(stream));
  if (e) return cuda_fail(e, "bst radial scratch");
  e = cudaMemsetAsync(acc, 0, (size_t)batch * 2 * sizeof(double), static_cast<cudaStream_t>(stream));
  if (!e) e = lpbp::launch_bst_radial(P->d, P->t, sino_dev, reinterpret_cast<float2*>(spectra_dev),
                                      static_cast<double*>(acc), batch, static_cast<cudaStream_t>(stream));
  cudaFreeAsync(acc, static_cast<cudaStream_t>(stream));
  if (e) return launch_fail(e, "bst_radial");
  ++g_launches;
  return LPBP_OK;
}


// ---------------------------------------------------------------------------
// standalone resampling steps
// ---------------------------------------------------------------------------
int lpbp_sinogram_to_semipolar(const float* sino_dev, float* p_dev, int32_t nt, int32_t ntheta, int32_t ns,
                               int32_t batch, void* stream) {
  g_launches = 0;
  if (ns == 0) ns = nt / 2;
  if (ns < 2) return fail(LPBP_EINVAL, "ns must be >= 2");
  if (nt < 2 || ntheta < 1) return fail(LPBP_EINVAL, "nt must be >= 2 and ntheta >= 1");
  if (batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (batch == 0) return LPBP_OK;
  if (!sino_dev || !p_dev) return fail(LPBP_EINVAL, "invalid argument");
  cudaError_t e = lpbp::launch_semipolar(sino_dev, p_dev, nt, ntheta, ns, batch, static_cast<cudaStream_t>(stream));
  if (e) return cuda_fail(e, "sinogram_to_semipolar");
  ++g_launches;
  return LPBP_OK;
}

int lpbp_semipolar_to_logpolar(const float* p_dev, float* lp_dev, int32_t ns, int32_t nphi, double rho0, int32_t nrho,
                               int32_t batch, void* stream) {
  g_launches = 0;
  if (nrho < 2) return fail(LPBP_EINVAL, "nrho must be >= 2");
  if (!(rho0 < 0)) return fail(LPBP_EINVAL, "rho0 must be negative");
  if (ns < 2 || nphi < 2) return fail(LPBP_EINVAL, "ns and nphi must be >= 2");
  if (batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (batch == 0) return LPBP_OK;
  if (!p_dev || !lp_dev) return fail(LPBP_EINVAL, "invalid argument");
  cudaError_t e = lpbp::launch_semipolar_to_logpolar(p_dev, lp_dev, ns, nphi, rho0, nrho, batch,
                                                     static_cast<cudaStream_t>(stream));
  if (e) return cuda_fail(e, "semipolar_to_logpolar");
  ++g_launches;
  return LPBP_OK;
}

int lpbp_logpolar_to_cartesian(const float* lp_dev, float* img_dev, int32_t nrho, int32_t nphi, double rho0,
                               int32_t nx, int32_t ny, int32_t batch, void* stream) {
  g_launches = 0;
  if (nx < 2 || ny < 2) return fail(LPBP_EINVAL, "nx and ny must be >= 2");
  if (nrho < 2 || nphi < 2) return fail(LPBP_EINVAL, "nrho and nphi must be >= 2");
  if (!(rho0 < 0)) return fail(LPBP_EINVAL, "rho0 must be negative");
  if (batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (batch == 0) return LPBP_OK;
  if (!lp_dev || !img_dev) return fail(LPBP_EINVAL, "invalid argument");
  cudaError_t e = lpbp::launch_logpolar_to_cartesian(lp_dev, img_dev, nrho, nphi, rho0, nx, ny, batch,
                                                     static_cast<cudaStream_t>(stream));
  if (e) return cuda_fail(e, "logpolar_to_cartesian");
  ++g_launches;
  return LPBP_OK;
}

int lpbp_logpolar_kernel(int32_t nrho, int32_t nphi, double drho, double* out_host) {
  if (nrho < 2 || nphi < 2) return fail(LPBP_EINVAL, "kernel mesh must be at least 2 x 2");
  if (!(drho > 0)) return fail(LPBP_EINVAL, "drho must be positive");
  if (!out_host) return fail(LPBP_EINVAL, "invalid argument");
  constexpr double kPi = 3.14159265358979323846;
  std::vector<double> ct(nphi);
  for (int j = 0; j < nphi; ++j) ct[j] = std::cos(-kPi + (double)j * (2.0 * kPi / nphi));
  for (int i = 0; i < nrho; ++i) {
    const double e = std::exp((double)i * drho);
    for (int j = 0; j < nphi; ++j)
      out_host[(size_t)i * nphi + j] = std::fabs(e * ct[j] - 1.0) <= drho ? 1.0 / drho : 0.0;
  }
  return LPBP_OK;
}


int lpbp_polar_to_cartesian_frequency(const float* spec_dev, float* out_dev, int32_t nsigma, int32_t nray,
                                      int64_t stride_m, int64_t stride_ray, int64_t slice_pitch, double dsigma,
                                      int32_t nx, int32_t ny, double dw, float scale, int32_t batch, void* stream) {
  g_launches = 0;
  if (nx < 2 || ny < 2) return fail(LPBP_EINVAL, "nx and ny must be >= 2");
  if (nsigma < 2 || nray < 2) return fail(LPBP_EINVAL, "nsigma and ntheta must be >= 2");
  if (!(dsigma > 0)) return fail(LPBP_EINVAL, "dsigma must be positive");
  const double nyq = std::sqrt(2.0) * dw * std::max(nx, ny) / 2.0, smax = (nsigma - 1) * dsigma;
  if (smax < nyq * (1.0 - 1e-12)) {
    char buf[200];
    std::snprintf(buf, sizeof buf,
                  "polar spectrum reaches sigma = %.3f but the cartesian grid requires coverage up to the Nyquist "
                  "radius %.3f", smax, nyq);
    return fail(LPBP_EINVAL, buf);
  }
  if (batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (batch == 0) return LPBP_OK;
  if (!spec_dev || !out_dev) return fail(LPBP_EINVAL, "invalid argument");
  cudaError_t e = lpbp::launch_polar_to_cartesian_frequency(
      reinterpret_cast<const float2*>(spec_dev), reinterpret_cast<float2*>(out_dev), nsigma, nray, stride_m, stride_ray,
      slice_pitch, dsigma, nx, ny, dw, scale, batch, static_cast<cudaStream_t>(stream));
  if (e) return cuda_fail(e, "polar_to_cartesian_frequency");
  ++g_launches;
  return LPBP_OK;
}

int lpbp_mean_backprojection(const float* sino_dev, double* out_dev, int32_t nt, int32_t ntheta, int32_t batch,
                             void* stream) {
  g_launches = 0;
  if (nt < 2 || ntheta < 1 || batch < 0) return fail(LPBP_EINVAL, "invalid argument");
  if (batch == 0) return LPBP_OK;
  if (!sino_dev || !out_dev) return fail(LPBP_EINVAL, "invalid argument");
  // chord of the square per angle as a trapezoid in t (same fp64 construction as the BST plan)
  const double kPi = 3.14159265358979323846, dt = 2.0 / nt, dth = kPi / ntheta;
  std::vector<lpbp::F4> cp(ntheta);
  for (int j = 0; j < ntheta; ++j) {
    const double c = std::fabs(std::cos(j * dth)), sn = std::fabs(std::sin(j * dth));
    const bool deg = c <= 1e-15 || sn <= 1e-15;
    const double t1 = deg ? 1.0 : std::fabs(c - sn), t2 = deg ? 1.0 : c + sn;
    const double lmax = deg ? 2.0 : 2.0 / std::max(c, sn);
    cp[j] = lpbp::F4{(float)t1, (float)t2, (float)(lmax * dt * dth / 4.0), t2 > t1 ? (float)(1.0 / (t2 - t1)) : 0.f};
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, cp.size() * sizeof(lpbp::F4), st);
  if (!e) e = cudaMemcpyAsync(d, cp.data(), cp.size() * sizeof(lpbp::F4), cudaMemcpyHostToDevice, st);
  if (!e) e = cudaStreamSynchronize(st);  // the host vector goes out of scope
  if (!e) e = lpbp::launch_mean_backprojection(sino_dev, static_cast<const float4*>(d), out_dev, nt, ntheta, batch, st);
  if (d) cudaFreeAsync(d, st);
  if (e) return cuda_fail(e, "mean_backprojection");
  ++g_launches;
  return LPBP_OK;
}

int lpbp_kaiser_window(int32_t ns, double beta, double* out_host) {
  if (ns < 2) return fail(LPBP_EINVAL, "ns must be >= 2");
  if (!out_host) return fail(LPBP_EINVAL, "invalid argument");
  auto i0 = [](double x) {  // power series of I0 (all terms positive)
    const double q = 0.25 * x * x;
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 500; ++k) {
      term *= q / ((double)k * k);
      sum += term;
      if (term < 1e-17 * sum) break;
    }
    return sum;
  };
  const double den = std::fabs(i0(beta));
  for (int i = 0; i < ns; ++i) {
    const double u = (2.0 * i - ns + 1.0) / (ns - 1.0);
    out_host[i] = std::fabs(i0(beta * std::sqrt(std::max(1.0 - u * u, 0.0)))) / den;
  }
  return LPBP_OK;
}

int64_t lpbp_last_launch_count(void) { return g_launches; }
const char* lpbp_last_error(void) { return g_last_error.c_str(); }
int32_t lpbp_version(void) { return 100; }

}  // extern "C"
