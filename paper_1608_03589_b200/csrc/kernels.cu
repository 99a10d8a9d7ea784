// Device kernels of the log-polar backprojection hot path (sm_100a, fp32).
//
// Pipeline per slice (fastbp reference in parentheses):
//   K1 ramp_filter   g -> g_f                  (filtering.py:54-70 filter_sinogram)
//   K2 row_rdft      g -> G[m][t]              (first half of the rfft2 in logpolar.py:113,
//                                               applied to sinogram rows, see below)
//   K3 rho_conv      G -> Y[m][rho]            (grids.py:290-347 resampling + logpolar.py:100-118
//                                               rho-axis FFT convolution with the kernel)
//   K4 row_irdft     Y -> lp[rho][phi]         (phi-axis half of irfft2, logpolar.py:113-117)
//   K5 readout       lp -> img                 (grids.py:399-443 logpolar_to_cartesian)
//
// Why K2 transforms sinogram rows rather than log-polar rows: both resampling
// steps (sinogram->semi-polar->log-polar) act only along t/s with weights that
// depend only on the row, and the phi<pi / phi>=pi halves are the same sinogram
// columns.  So the phi-DFT of log-polar row i is a <=8-term combination of the
// phi-DFTs of sinogram rows (the phi>=pi half picks up (-1)^m from its nphi/2
// shift).  nt row FFTs replace nrho (~1.9x fewer) and the row mix moves into K3,
// where it feeds the first rho-FFT pass straight from shared memory.
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "async.cuh"
#include "fft.cuh"
#include "tmem.cuh"
#include "mixed.cuh"
#include "kernels.cuh"

namespace lpbp {

namespace {
__device__ __forceinline__ void block_sync() { __syncthreads(); }
// named barrier for one FFT group of `count` threads (ids 1.. ; 0 is __syncthreads)
struct GroupSync {
  int id, count;
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
  }
};
}  // namespace

// ---------------------------------------------------------------------------
// K1: ramp filter along t (strided columns of g).  Two theta-columns are packed
// as re/im of one complex M-point FFT (the response is real and even, so no
// unpacking is needed).  Tile: all nt rows x TC columns staged in smem.
// ---------------------------------------------------------------------------
template <int M, int TC, int G>
__global__ void __launch_bounds__(G * FftPlan<M, false>::T, (G == 1 ? 2 : 1))
k_ramp(const float* __restrict__ g, float* __restrict__ out, int nt, int ntheta,
       const float* __restrict__ resp, const float2* __restrict__ tw) {
  constexpr int T = FftPlan<M, false>::T;
  constexpr int TP = TC + 1;  // tile pitch (floats): conflict-free column reads
  constexpr int V = TC / 4;   // float4 per tile row
  extern __shared__ __align__(16) float2 smem_k1[];
  float* tile = reinterpret_cast<float*>(smem_k1);  // nt * TP floats
  float2* bufs = smem_k1 + ((nt * TP + 1) / 2);
  const int gi = threadIdx.x / T, ti = threadIdx.x % T;
  float2* buf = bufs + gi * padded_len(M);
  const int c0 = blockIdx.x * TC;
  const size_t slice = (size_t)blockIdx.y * nt * ntheta;
  const float* src = g + slice + c0;
  float* dst = out + slice + c0;

  // 16-byte loads, 8 in flight per thread
  const int total = nt * V;
#pragma unroll 8
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int t = e / V, c = (e % V) * 4;
    const float4 v = __ldg(reinterpret_cast<const float4*>(src + (size_t)t * ntheta + c));
    float* r = tile + t * TP + c;
    r[0] = v.x;
    r[1] = v.y;
    r[2] = v.z;
    r[3] = v.w;
  }
  __syncthreads();
  for (int round = 0; round < TC / 2 / G; ++round) {
    const int q = round * G + gi;
    auto load = [&](int idx) -> float2 {
      return idx < nt ? make_float2(tile[idx * TP + 2 * q], tile[idx * TP + 2 * q + 1]) : make_float2(0.f, 0.f);
    };
    auto mul = [&](int idx, float2 v) -> float2 { return cscale(v, __ldg(resp + idx)); };
    auto store = [&](int idx, float2 v) {
      if (idx < nt) {
        tile[idx * TP + 2 * q] = v.x;
        tile[idx * TP + 2 * q + 1] = v.y;
      }
    };
    block_conv<M, true, 16>(buf, ti, tw, load, mul, store, block_sync);  // M = 2 nt: half-zero in, low half out
    __syncthreads();
  }
#pragma unroll 8
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int t = e / V, c = (e % V) * 4;
    const float* r = tile + t * TP + c;
    *reinterpret_cast<float4*>(dst + (size_t)t * ntheta + c) = make_float4(r[0], r[1], r[2], r[3]);
  }
}

// Persistent TMA variant (nt a multiple of 256): one CTA per SM, two FFT groups,
// two tile slots.  Tiles of 8 columns x nt rows arrive by 2-D TMA boxes {8, 256}
// and leave by TMA stores, both issued by one thread, so HBM traffic runs behind
// the convolutions of the other slot with no load/store instructions in the
// warps.  The slot layout is TMA's 32-byte swizzle: float (t, c) sits at
// t*8 + (c ^ 4*((t >> 2) & 1)), which spreads a column pair of 16 consecutive rows
// over 8 bank pairs (2-way) instead of 4 (4-way) for the dense layout.
template <int M>
struct RampTmaShape {
  static constexpr int G = 2, TC = 8, BOXR = 256;
  static constexpr int T = FftPlan<M, false>::T;
  static size_t smem(int nt) {
    return 1024 + 2 * (size_t)nt * TC * sizeof(float) + (size_t)G * padded_len(M) * sizeof(float2) +
           (size_t)M * sizeof(float) + 64;
  }
};

template <int M>
__global__ void __launch_bounds__(RampTmaShape<M>::G * FftPlan<M, false>::T, 1)
k_ramp_tma(const __grid_constant__ CUtensorMap gmap, const __grid_constant__ CUtensorMap omap, int nt,
           int tiles_per_slice, int ntiles, const float* __restrict__ resp, const float2* __restrict__ tw) {
  using RS = RampTmaShape<M>;
  constexpr int T = RS::T, G = RS::G, TC = RS::TC, BOXR = RS::BOXR;
  static_assert((M / 16) % 8 == 0 && T % 8 == 0, "pass-0 rows must keep (idx >> 2) & 1 = (ti >> 2) & 1");
  extern __shared__ unsigned char smem_k1t[];
  // 1024-byte aligned slots (TMA swizzle atoms); offset from the shared symbol itself so the
  // compiler keeps every access in the shared window (LDS/STS, not generic LD/ST)
  float* slots = reinterpret_cast<float*>(smem_k1t + ((1024u - (smem_u32(smem_k1t) & 1023u)) & 1023u));
  const int slot_floats = nt * TC;
  float2* bufs = reinterpret_cast<float2*>(slots + 2 * slot_floats);
  float* resp_s = reinterpret_cast<float*>(bufs + G * padded_len(M));  // the response, read by every convolution
  uint64_t* bars = reinterpret_cast<uint64_t*>(resp_s + M);
  const int gi = threadIdx.x / T, ti = threadIdx.x % T;
  float2* buf = bufs + gi * padded_len(M);
  const uint32_t tile_bytes = (uint32_t)slot_floats * sizeof(float);
  const int first = blockIdx.x, stride = gridDim.x;
  auto corner = [&](int tile, int& c0, int& r0) {
    const int b = tile / tiles_per_slice;
    c0 = (tile - b * tiles_per_slice) * TC;
    r0 = b * nt;
  };
  auto load_tile = [&](int tile, int s) {  // warp 0: lane 0 arms the barrier, one box per lane
    const int lane = threadIdx.x;
    int c0, r0;
    corner(tile, c0, r0);
    if (lane == 0) mbar_arrive_expect_tx(&bars[s], tile_bytes);
    __syncwarp();
    for (int k = lane; k < nt / BOXR; k += 32)
      tma_load_2d(slots + s * slot_floats + k * BOXR * TC, &gmap, c0, r0 + k * BOXR, &bars[s]);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  for (int i = threadIdx.x; i < M; i += blockDim.x) resp_s[i] = __ldg(resp + i);
  __syncthreads();
  if (threadIdx.x < 32) {
    if (first < ntiles) load_tile(first, 0);
    if (first + stride < ntiles) load_tile(first + stride, 1);
  }
  const int sw = ((ti >> 2) & 1) << 2;  // this thread's rows all share the swizzle bit
  const GroupSync gsync{1 + gi, T};
  int it = 0;
  int refill = -1;  // (thread 0) tile whose slot waits to be refilled once its TMA stores have read it
#pragma unroll 1
  for (int tile = first; tile < ntiles; tile += stride, ++it) {
    const int s = it & 1;
    float* tl = slots + s * slot_floats;
    mbar_wait(&bars[s], (it >> 1) & 1);
#pragma unroll 1
    for (int round = 0; round < TC / 2 / G; ++round) {
      if (round == 1 && threadIdx.x < 32 && refill >= 0) {
        // the previous tile's stores (one per lane) have had a round to drain: refill the slot two tiles ahead
        bulk_wait_group_read<0>();
        __syncwarp();
        load_tile(refill + 2 * stride, s ^ 1);
        refill = -1;
      }
      const int q = round * G + gi;
      float* col = tl + ((2 * q) ^ sw);  // row idx at col + 8 idx
      auto load = [&](int idx) -> float2 {
        return idx < nt ? *reinterpret_cast<const float2*>(col + idx * TC) : make_float2(0.f, 0.f);
      };
      auto mul = [&](int idx, float2 v) -> float2 { return cscale(v, resp_s[idx]); };
      auto store = [&](int idx, float2 v) {
        if (idx < nt) *reinterpret_cast<float2*>(col + idx * TC) = v;
      };
      block_conv<M, true, 16>(buf, ti, tw, load, mul, store, gsync);  // M = 2 nt: half-zero in, low half out
      gsync();                                                       // buf is reused by the next round
    }
    __syncthreads();  // every group's results are in the slot
    if (threadIdx.x < 32) {  // one TMA store box per lane
      int c0, r0;
      corner(tile, c0, r0);
      fence_proxy_async_smem();  // the convolutions' generic stores before this lane's TMA reads
      for (int k = threadIdx.x; k < nt / BOXR; k += 32) tma_store_2d(&omap, c0, r0 + k * BOXR, tl + k * BOXR * TC);
      bulk_commit_group();
      if (tile + 2 * stride < ntiles) refill = tile;
    }
  }
  if (threadIdx.x < 32) bulk_wait_group<0>();
}

// ---------------------------------------------------------------------------
// K2: real DFT of sinogram rows, zero-padded from ntheta to nphi = 2 ntheta.
// Rows t, t+1 are packed as re/im; spectra are separated with
//   A[m] = (Z[m] + conj Z[-m]) / 2,  B[m] = (Z[m] - conj Z[-m]) / 2i
// and staged as [m][TR] (TMA 32-byte swizzle) so G[m][t0..t0+TR) leaves by TMA stores.
// ---------------------------------------------------------------------------

// Persistent: each CTA walks tiles (slice, 4 consecutive rows); a tile's rows are
// contiguous (4 x NTH floats) and arrive by one TMA bulk copy into a double
// buffer, two tiles ahead of use.  Group g (of 2) transforms row pair g.
template <int NPHI>
struct RdftShape {
  static constexpr int TR = 4, G = 2;
  static constexpr int NTH = NPHI / 2, NH = NPHI / 2 + 1;
  static constexpr int IN = TR * NTH / 2;                    // float2 per input tile
  static constexpr int STG = ((NH * TR) + 15) & ~15;         // float2 staging
  static constexpr int BUF = (padded_len(NPHI) + 15) & ~15;  // float2 per FFT buffer
  static constexpr size_t SMEM = ((size_t)2 * IN + STG + G * BUF) * 8 + 64 + 1024;  // + alignment slack
  static constexpr int NFULL = (NPHI / 2) / 256;  // 256-row TMA store boxes of the spectra; one 1-row tail box
};

// NARROW: compacted input rows (the sector path): `win` (multiple of 4) floats holding the
// row's first win_lo columns followed by its last win - win_lo columns; the rest is zero.
template <int NPHI, bool NARROW>
__global__ void __launch_bounds__(RdftShape<NPHI>::G * FftPlan<NPHI, false>::T, 1)
k_row_rdft(const __grid_constant__ CUtensorMap gmap, const __grid_constant__ CUtensorMap gtail,
           const float* __restrict__ g, int nt, int ntiles_per_slice, int ntiles,
           const float2* __restrict__ tw, int win, int win_lo) {
  using RS = RdftShape<NPHI>;
  constexpr int T = FftPlan<NPHI, false>::T;
  constexpr int TR = RS::TR, NTH = RS::NTH, NH = RS::NH, NFULL = RS::NFULL;
  static_assert(TR == 4 && NFULL * 256 + 1 == NH && NFULL < 32, "32-byte staging rows, full boxes + one tail row");
  extern __shared__ __align__(128) float2 smem_k2_raw[];
  // 1024-byte aligned base (TMA swizzle atoms), offset from the shared symbol to stay in the shared window
  float2* smem_k2 = smem_k2_raw + ((1024u - (smem_u32(smem_k2_raw) & 1023u)) & 1023u) / sizeof(float2);
  float* in0 = reinterpret_cast<float*>(smem_k2);               // 2 x TR*NTH floats
  // [NH][TR] spectra staging in TMA's 32-byte swizzle: complex (m, c) at m*TR + (c ^ 2*((m >> 2) & 1));
  // leaves by TMA stores into G[b][m][t0 .. t0+TR)
  float2* stg = smem_k2 + 2 * RS::IN;
  float2* buf = stg + RS::STG + (threadIdx.x / T) * RS::BUF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + RS::STG + RS::G * RS::BUF);
  const int gi = threadIdx.x / T, ti = threadIdx.x % T;
  const int W = NARROW ? win : NTH;  // input row pitch (floats)
  const uint32_t TILE_BYTES = TR * W * 4;
  auto tile_src = [&](int tile) {
    const int b = tile / ntiles_per_slice, t0 = (tile - b * ntiles_per_slice) * TR;
    return g + ((size_t)b * nt + t0) * W;
  };
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int first = blockIdx.x, stride = gridDim.x;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) {
      const int tile = first + k * stride;
      if (tile < ntiles) {
        mbar_arrive_expect_tx(&bars[k], TILE_BYTES);
        tma_bulk_g2s(in0 + k * TR * NTH, tile_src(tile), TILE_BYTES, &bars[k]);
      }
    }
  }
  int it = 0;
#pragma unroll 1
  for (int tile = first; tile < ntiles; tile += stride, ++it) {
    const int sl = it & 1;
    mbar_wait(&bars[sl], (it >> 1) & 1);
    const float* ra = in0 + sl * TR * NTH + (2 * gi) * W;
    const float* rb = ra + W;
    auto load = [&](int idx) -> float2 {  // idx < NTH (IN_HALF)
      if constexpr (NARROW) {
        const int tail = NTH - (W - win_lo);  // first row position of the trailing block
        if (idx >= win_lo && idx < tail) return make_float2(0.f, 0.f);
        if (idx >= tail) idx -= tail - win_lo;
      }
      return make_float2(ra[idx], rb[idx]);
    };
    auto store = [&](int idx, float2 v) { buf[pad16(idx)] = v; };
    block_fft<NPHI, false, true, false, true, 16>(buf, ti, tw, load, store, GroupSync{1 + gi, T});
    if (threadIdx.x < 32) bulk_wait_group_read<0>();  // the previous tile's TMA stores (warp 0's lanes) have read stg
    __syncthreads();
    // every thread is past pass 0: the input slot is free for the tile two ahead
    if (threadIdx.x == 0 && tile + 2 * stride < ntiles) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bars[sl], TILE_BYTES);
      tma_bulk_g2s(in0 + sl * TR * NTH, tile_src(tile + 2 * stride), TILE_BYTES, &bars[sl]);
    }
    for (int m = ti; m < NH; m += T) {
      const float2 z = buf[pad16(m)];
      const float2 w = buf[pad16((NPHI - m) & (NPHI - 1))];
      const int sw = ((m >> 2) & 1) << 1;
      // rows 2 gi and 2 gi + 1 sit side by side in the swizzled [m][4] staging (sw is even): one
      // 16-byte store (a warp's 32 stores fill 8 distinct 16-byte bank groups: 4 wavefronts, no conflict)
      *reinterpret_cast<float4*>(stg + m * TR + ((2 * gi) ^ sw)) =
          make_float4(0.5f * (z.x + w.x), 0.5f * (z.y - w.y), 0.5f * (z.y + w.y), 0.5f * (w.x - z.x));
    }
    __syncthreads();
    if (threadIdx.x <= NFULL) {  // one TMA store box per lane of warp 0
      const int b = tile / ntiles_per_slice, t0 = (tile - b * ntiles_per_slice) * TR;
      const int bx = threadIdx.x;
      fence_proxy_async_smem();  // the separation's generic stores before this lane's TMA reads
      if (bx < NFULL) tma_store_2d(&gmap, 2 * t0, b * NH + bx * 256, stg + bx * 256 * TR);
      else tma_store_2d(&gtail, 2 * t0, b * NH + NFULL * 256, stg + NFULL * 256 * TR);
      bulk_commit_group();
    }
    // next tile's separation rewrites stg only after its FFT and the store-read wait above
  }
  if (threadIdx.x < 32) bulk_wait_group<0>();
}

// ---------------------------------------------------------------------------
// K2p: real DFT along phi of the SEMI-POLAR rows (grids.py:290-311 followed by the phi half of
// logpolar.py:112): row k of p is [ t >= 0 lerp of the sinogram | t <= 0 lerp ], 2 ntheta = nphi
// samples, so its spectrum is what K3's frequency-domain row mix would build from four row spectra.
// Forming p before the transform halves the transforms (ns = nt/2 full-length rows instead of nt
// zero-padded ones), K2's output and K3's column input, and takes the row mix out of K3.
// Persistent CTAs walk tiles (slice, 4 semi-polar rows); a producer warp lands the tile's sinogram
// rows — two contiguous runs of <= 5 rows, one per side (plan_host ptile) — in the single input slot
// by two TMA bulk copies as soon as every consumer warp is past the previous tile's pass-0 loads
// (the only reads of the slot), i.e. most of a tile ahead.  FFT group g forms rows 4j + 2g, 4j + 2g + 1
// inside its pass-0 loads (two taps per value, weights in registers) packed as re/im; the spectra
// are separated and staged [m][4] like K2's and leave by TMA stores into P[b][m][k0 .. k0 + 4).
// ---------------------------------------------------------------------------
template <int NPHI>
struct RdftPShape {
  static constexpr int KR = 4, G = 2, SR = 5;
  static constexpr int NTH = NPHI / 2, NH = NPHI / 2 + 1;
  static constexpr int IN = 2 * SR * NTH / 2;                // float2 in the input slot (a rows, then b rows)
  static constexpr int STG = ((NH * KR) + 15) & ~15;         // float2 staging
  static constexpr int BUF = (padded_len(NPHI) + 15) & ~15;  // float2 per FFT buffer
  static constexpr size_t SMEM = ((size_t)IN + STG + G * BUF) * 8 + 64 + 1024;  // + barriers, alignment slack
  static constexpr int NFULL = (NPHI / 2) / 256;
};

template <int NPHI>
__global__ void __launch_bounds__(RdftPShape<NPHI>::G * FftPlan<NPHI, false>::T + 32, 1)
k_row_rdft_p(const __grid_constant__ CUtensorMap pmap, const __grid_constant__ CUtensorMap ptail,
             const float* __restrict__ g, int nt, int ntiles_per_slice, int ntiles, const int4* __restrict__ ptile,
             const uint32_t* __restrict__ ploc, const float4* __restrict__ wab, const float2* __restrict__ tw) {
  using RS = RdftPShape<NPHI>;
  constexpr int T = FftPlan<NPHI, false>::T;
  constexpr int KR = RS::KR, NTH = RS::NTH, NH = RS::NH, NFULL = RS::NFULL, SR = RS::SR;
  constexpr int NC = RS::G * T;
  static_assert(KR == 4 && NFULL * 256 + 1 == NH && NFULL < 32, "32-byte staging rows, full boxes + one tail row");
  extern __shared__ __align__(128) float2 smem_k2p_raw[];
  float2* smem_k2 = smem_k2p_raw + ((1024u - (smem_u32(smem_k2p_raw) & 1023u)) & 1023u) / sizeof(float2);
  float* slot = reinterpret_cast<float*>(smem_k2);  // [2][SR][NTH]
  float2* stg = smem_k2 + RS::IN;                   // [NH][4] in TMA's 32-byte swizzle (as K2)
  float2* bufs = stg + RS::STG;
  uint64_t* bars = reinterpret_cast<uint64_t*>(bufs + RS::G * RS::BUF);  // full, consumed
  uint64_t* full = &bars[0];
  uint64_t* consumed = &bars[1];
  if (threadIdx.x == 0) {
    mbar_init(full, 1);
    mbar_init(consumed, NC / 32);
    fence_mbar_init();
  }
  __syncthreads();
  const int first = blockIdx.x, stride = gridDim.x;

  if (threadIdx.x >= NC) {  // ---- producer warp (lane 0 issues)
    if (threadIdx.x == NC) {
      int it = 0;
      for (int tile = first; tile < ntiles; tile += stride, ++it) {
        if (it > 0) mbar_wait(consumed, (uint32_t)((it - 1) & 1));
        const int b = tile / ntiles_per_slice, kb = tile - b * ntiles_per_slice;
        const int4 td = __ldg(ptile + kb);
        const float* base = g + (size_t)b * nt * NTH;
        const uint32_t ba = (uint32_t)td.y * NTH * 4u, bb = (uint32_t)td.w * NTH * 4u;
        fence_proxy_async_smem();  // the consumers' reads of the slot before these writes
        mbar_arrive_expect_tx(full, ba + bb);
        tma_bulk_g2s(slot, base + (size_t)td.x * NTH, ba, full);
        tma_bulk_g2s(slot + SR * NTH, base + (size_t)td.z * NTH, bb, full);
      }
    }
    return;
  }

  const int gi = threadIdx.x / T, ti = threadIdx.x % T;
  float2* buf = bufs + gi * RS::BUF;
  const GroupSync gsync{1 + gi, T};
  const GroupSync csync{1 + RS::G, NC};
  int it = 0;
#pragma unroll 1
  for (int tile = first; tile < ntiles; tile += stride, ++it) {
    const int b = tile / ntiles_per_slice, k0 = (tile - b * ntiles_per_slice) * KR;
    // this group's two rows: tap rows inside the slot and their weights
    const int kx = k0 + 2 * gi;
    const uint32_t lx = __ldg(ploc + kx), ly = __ldg(ploc + kx + 1);
    const float4 wx = __ldg(wab + kx), wy = __ldg(wab + kx + 1);
    const int xa0 = (int)(lx & 15u) * NTH, xa1 = (int)((lx >> 4) & 15u) * NTH;
    const int xb0 = (int)((lx >> 8) & 15u) * NTH + SR * NTH, xb1 = (int)((lx >> 12) & 15u) * NTH + SR * NTH;
    const int ya0 = (int)(ly & 15u) * NTH, ya1 = (int)((ly >> 4) & 15u) * NTH;
    const int yb0 = (int)((ly >> 8) & 15u) * NTH + SR * NTH, yb1 = (int)((ly >> 12) & 15u) * NTH + SR * NTH;
    mbar_wait(full, (uint32_t)(it & 1));
    constexpr int R0 = FftPlan<NPHI, false>::radix(0), QS = NPHI / R0;
    auto load = [&](int j, auto rc) -> float2 {
      constexpr int r = decltype(rc)::value;
      if constexpr (r < R0 / 2) {  // phi < pi: the t >= 0 taps
        const float* c = slot + j + r * QS;
        return make_float2(fmaf(wx.y, c[xa1], wx.x * c[xa0]), fmaf(wy.y, c[ya1], wy.x * c[ya0]));
      } else {  // phi >= pi: the t <= 0 taps
        const float* c = slot + j + (r - R0 / 2) * QS;
        return make_float2(fmaf(wx.w, c[xb1], wx.z * c[xb0]), fmaf(wy.w, c[yb1], wy.z * c[yb0]));
      }
    };
    auto store = [&](int idx, float2 v) { buf[pad16(idx)] = v; };
    bool first_sync = true;
    auto sync = [&]() {  // the first barrier follows pass 0's stores: this warp no longer reads the slot
      if (first_sync) {
        first_sync = false;
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(consumed);
      }
      gsync();
    };
    block_fft<NPHI, false, true, false, false, 16>(buf, ti, tw, load, store, sync);
    if (threadIdx.x < 32) bulk_wait_group_read<0>();  // the previous tile's TMA stores have read stg
    csync();
    for (int m = ti; m < NH; m += T) {
      const float2 z = buf[pad16(m)];
      const float2 w = buf[pad16((NPHI - m) & (NPHI - 1))];
      const int sw = ((m >> 2) & 1) << 1;
      *reinterpret_cast<float4*>(stg + m * KR + ((2 * gi) ^ sw)) =
          make_float4(0.5f * (z.x + w.x), 0.5f * (z.y - w.y), 0.5f * (z.y + w.y), 0.5f * (w.x - z.x));
    }
    csync();
    if (threadIdx.x <= NFULL) {  // one TMA store box per lane of warp 0
      const int bx = threadIdx.x;
      fence_proxy_async_smem();
      if (bx < NFULL) tma_store_2d(&pmap, 2 * k0, b * NH + bx * 256, stg + bx * 256 * KR);
      else tma_store_2d(&ptail, 2 * k0, b * NH + NFULL * 256, stg + NFULL * 256 * KR);
      bulk_commit_group();
    }
  }
  if (threadIdx.x < 32) bulk_wait_group<0>();
}

// ---------------------------------------------------------------------------
// K3: per phi-frequency column m (one CTA), for every slice of the batch:
//   p[k]  = wa0 G[a_k] + wa1 G[a_k+1] + (-1)^m (wb0 G[b_k] + wb1 G[b_k+1])   (semi-polar, grids.py:290-311)
//   x[i]  = w0 p[k_i] + w1 p[k_i+1], i < nrho, 0 for i >= nrho            (log-polar, grids.py:332-347)
//   Y[m]  = IFFT_L( FFT_L(x) * Khat[m] )[:nrho]                           (logpolar.py:112-117)
// The row mix is evaluated inside the first forward pass; the multiply by
// Khat is fused between the last forward and first inverse pass.  TM: each
// thread's 32 Khat values of the CTA's column are read from L2 once and kept in
// its TMEM lane (tensor memory, otherwise idle here) for all slices of the chunk.
// ---------------------------------------------------------------------------
// 16384-point columns (nt >~ 2900): 512 threads and ~200 KB of shared memory, one CTA per SM
// PIN: Gh is K2p's semi-polar row spectra P[b][m][ns] (gp = ns): the column is the p the first pass
// interpolates from, landed by TMA in one of two buffers (the other one is refilled at the top of
// the slice's iteration: its last readers were the previous slice's first pass).
template <int L, bool PRUNE, bool TM, bool PIN = false>
__global__ void __launch_bounds__(FftPlan<L, false>::T, (L >= 16384 ? 1 : 2))
k_rho_conv(const float2* __restrict__ Gh, float2* __restrict__ Yh, int batch, int nt, int gp, int ns, int nrho, int row_lo,
           int nrho_pad, int nh, const uint2* __restrict__ abw,
           const uint32_t* __restrict__ kw, const float2* __restrict__ khat, const float2* __restrict__ tw,
           const int32_t* __restrict__ rowmap, int zend) {
  constexpr int T = FftPlan<L, false>::T;
  extern __shared__ __align__(16) float2 smem_k3[];
  __shared__ __align__(8) uint64_t bars[2];
  uint64_t& bar = bars[0];
  __shared__ uint32_t tslot;
  float2* buf = smem_k3;                          // padded_len(L)
  float2* p = buf + padded_len(L);                // ns (PIN: two buffers of PS = ns + 2, the pad reads zero)
  const int PS = (ns + 3) & ~1;
  float2* gcol = PIN ? p : p + ((ns + 1) & ~1);   // gp + 2 (16-B aligned); refilled as soon as the row mix is done
  uint32_t* kws = reinterpret_cast<uint32_t*>(PIN ? p + 2 * PS : gcol + gp + 2);  // nrho packed log-polar taps, same for every column
  const int m = blockIdx.x;
  const float sg = (m & 1) ? -1.f : 1.f;
  const int ti = threadIdx.x;
  const float2* kcol = khat + (size_t)m * L;
  const uint32_t col_bytes = (uint32_t)gp * sizeof(float2);  // gp = nt rounded up to even

  // TM: loop invariants live in the thread's TMEM lane for all slices of the chunk: its E Khat values
  // of this column (one L2 read of the column per CTA instead of one per slice, columns [0, 2E)), its
  // first-pass log-polar taps ([2E, 2E + 16), TKW) and its semi-polar row-mix taps ([2E + 16, 2E + 32),
  // when ns <= 4T).  (The twiddles, also per-thread invariants, were measured slower from TMEM than
  // from the SFU: 73.0 vs 69.3 us/slice; the SFU work overlaps the pass's shared-memory loads.)
  constexpr int E = FftPlan<L, false>::E;
  constexpr int R0 = FftPlan<L, false>::radix(0), RL0 = PRUNE ? R0 / 2 : R0, KWN = (E / R0) * RL0;
  constexpr bool TKW = TM && KWN <= 16;
  constexpr bool TKF = TKW && PIN;  // taps kept unpacked (row, fp32 weight) in the 32 columns the row-mix taps left free
  constexpr int WCOLS = 2 * E + 48;  // K-hat | first-pass taps | row-mix taps (or the taps' weights) | store rows
  constexpr int TCOLS = pow2_at_least(WCOLS * (T >= 128 ? T / 128 : 1));
  const bool tab = TM && !PIN && ns <= 4 * T;  // row-mix taps from TMEM (uniform over the CTA)
  const int warp = ti >> 5;
  if (TM && warp == 0) tmem_alloc<TCOLS>(&tslot);
  if (ti == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t kt = TM ? tmem_addr(tslot, warp, (warp >> 2) * WCOLS) : 0u;
  // first column (in flight under the TMEM prologue); the packed taps ride on the first column's barrier as one more bulk copy (16-byte multiple)
  const uint32_t kw_bytes = (uint32_t)nrho * 4u;
  const bool kw_bulk = (kw_bytes & 15u) == 0 && (reinterpret_cast<uintptr_t>(kw) & 15u) == 0;
  if (ti == 0) {
    mbar_arrive_expect_tx(&bar, col_bytes + (kw_bulk && !TKW ? kw_bytes : 0u));
    tma_bulk_g2s(gcol, Gh + (size_t)m * gp, col_bytes, &bar);
    if (kw_bulk && !TKW) tma_bulk_g2s(kws, kw, kw_bytes, &bar);
  }
  if constexpr (TM) {  // value e = b R + r of the fused middle multiplies Khat[ti + b T + r L/R]
    constexpr int RL = FftPlan<L, false>::radix(FftPlan<L, false>::P - 1);
#pragma unroll 1
    for (int c = 0; c < E / 8; ++c) {
      float t16[16];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = 8 * c + q, bb = e / RL, r = e % RL;
        const float2 kv = __ldg(kcol + ti + bb * T + r * (L / RL));
        t16[2 * q] = kv.x;
        t16[2 * q + 1] = kv.y;
      }
      tmem_st16(kt + 16 * c, t16);
    }
    if constexpr (TKW) {  // first-pass input e = b RL0 + r reads taps at ti + b T + r L/R0
      uint32_t t[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int idx = ti + (q / RL0) * T + (q % RL0) * (L / R0);
        t[q] = (q < KWN && idx < nrho) ? __ldg(kw + idx) : 0u;
      }
      if constexpr (TKF) {  // (row, w1 as fp32: the 20-bit fixed-point weight x 2^-20 is exact) pairs
        uint32_t u[16];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            u[2 * q] = t[8 * h + q] & 0x7FFu;
            u[2 * q + 1] = __float_as_uint((float)(t[8 * h + q] >> 11) * (1.f / 1048576.f));
          }
          tmem_st16(kt + 2 * E + 16 * h, u);
        }
      } else {
        tmem_st16(kt + 2 * E, t);
      }
    }
    if (tab) {  // row-mix rows ti + u T
      uint32_t t[16];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = ti + u * T;
        const uint2 e = k < ns ? __ldg(abw + k) : make_uint2(0u, 0u);
        t[2 * u] = e.x;
        t[2 * u + 1] = e.y;
      }
#pragma unroll
      for (int q = 8; q < 16; ++q) t[q] = 0u;
      tmem_st16(kt + 2 * E + 16, t);
    }
    tmem_wait_st();
  }
  // The thread's output rows are the same for every slice: one bit per store of the last inverse pass
  // (row < nrho and >= row_lo).  rowmap (ahead of the fused inverse DFT + readout): row -> where the row
  // is stored in the column, -1 for rows of bands no pixel taps (never read): the bands the readout
  // loads sit back to back, so each of its 32-byte band reads shares its DRAM burst with the next band
  // it needs, not with a skipped one.  TMC: the 16 store rows live in the thread's TMEM lane.
  constexpr int RLS = FftPlan<L, true>::radix(FftPlan<L, true>::P - 1), NSL = FftPlan<L, true>::ns(FftPlan<L, true>::P - 1);
  constexpr int ROS = PRUNE ? RLS / 2 : RLS, NST = (E / RLS) * ROS;
  static_assert(NST <= 32, "one mask bit per store");
  constexpr bool TMC = TM && NST <= 16;
  uint32_t smask = 0;
  {
    uint32_t crow[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int q = 0; q < NST; ++q) {
      const int idx = ti + (q / ROS) * T + (q % ROS) * NSL;
      int c = (idx < nrho && idx >= row_lo) ? (rowmap ? __ldg(rowmap + idx) : idx) : -1;
      if (c >= nrho_pad) c = -1;
      smask |= c >= 0 ? 1u << q : 0u;
      if constexpr (TMC) crow[q] = (uint32_t)max(c, 0);
    }
    if constexpr (TMC) {
      tmem_st16(kt + 2 * E + 32, crow);
      tmem_wait_st();
    }
  }
  if (!kw_bulk && !TKW)
    for (int i = ti; i < nrho; i += T) kws[i] = __ldg(kw + i);  // visible after the row mix's barrier
  if (PIN) {
    if (ti < 4) p[(ti >> 1) * PS + ns + (ti & 1)] = make_float2(0.f, 0.f);  // p[ns], p[ns + 1] of both buffers
  } else if (ti < 2) {
    gcol[gp + ti] = make_float2(0.f, 0.f);  // rows nt, nt+1 of the packed taps read zero (visible
  }                                          // after the first mbarrier wait's __syncthreads below)
  __syncthreads();

  for (int b = 0; b < batch; ++b) {
    const float2* pc = p;
    if constexpr (PIN) {
      mbar_wait(&bars[b & 1], (uint32_t)((b >> 1) & 1));
      pc = p + (b & 1) * PS;
      if (ti == 0 && b + 1 < batch) {  // the other buffer's last readers: the previous slice's first pass
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&bars[(b + 1) & 1], col_bytes);
        tma_bulk_g2s(p + ((b + 1) & 1) * PS, Gh + ((size_t)(b + 1) * nh + m) * gp, col_bytes, &bars[(b + 1) & 1]);
      }
    } else {
    mbar_wait(&bar, b & 1);
    const float2* col = gcol;
    // p[k] = (1 - wa) G[a] + wa G[a+1] + (-1)^m ((1 - wb) G[b] + wb G[b+1]); taps for 4 rows in flight
    constexpr float kW = 1.f / 524288.f;
#pragma unroll 1
    for (int k0 = 0; k0 < ns; k0 += 4 * T) {
      uint2 e[4];
      if (tab) {
        uint32_t t[16];
        tmem_ld16(kt + 2 * E + 16, t);
#pragma unroll
        for (int u = 0; u < 4; ++u) e[u] = make_uint2(t[2 * u], t[2 * u + 1]);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int k = k0 + ti + u * T;
          e[u] = k < ns ? __ldg(abw + k) : make_uint2(0u, 0u);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + ti + u * T;
        if (k < ns) {
          const int a = (int)(e[u].x & 0x1FFFu), b = (int)(e[u].y & 0x1FFFu);
          const float wa = (float)(e[u].x >> 13) * kW, wb = (float)(e[u].y >> 13) * kW;
          const float2 g0 = col[a], g1 = col[a + 1];
          const float2 h0 = col[b], h1 = col[b + 1];
          float2 v;
          v.x = fmaf(wa, g1.x, fmaf(-wa, g0.x, g0.x)) + sg * fmaf(wb, h1.x, fmaf(-wb, h0.x, h0.x));
          v.y = fmaf(wa, g1.y, fmaf(-wa, g0.y, g0.y)) + sg * fmaf(wb, h1.y, fmaf(-wb, h0.y, h0.y));
          p[k] = v;
        }
      }
    }
    __syncthreads();
    if (ti == 0 && b + 1 < batch) {  // the column is consumed: fetch the next slice's across the transforms
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bar, col_bytes);
      tma_bulk_g2s(gcol, Gh + ((size_t)(b + 1) * nh + m) * gp, col_bytes, &bar);
    }
    }  // !PIN
    uint32_t kwr[16];
    float kwf[32];
    auto load = [&](auto ec, int idx) -> float2 {
      constexpr int q = decltype(ec)::value;
      (void)q;
      if constexpr (TKF) {
        if constexpr (q == 0) tmem_ld32(kt + 2 * E, kwf);
      } else if constexpr (TKW) {
        if constexpr (q == 0) tmem_ld16(kt + 2 * E, kwr);
      }
      if (idx >= nrho) return make_float2(0.f, 0.f);
      int k;
      float w1;
      if constexpr (TKF) {
        k = __float_as_int(kwf[2 * q]);
        w1 = kwf[2 * q + 1];
      } else {
        uint32_t e;
        if constexpr (TKW) e = kwr[q];
        else e = kws[idx];
        k = (int)(e & 0x7FFu);
        w1 = (float)(e >> 11) * (1.f / 1048576.f);
      }
      const float2 p0 = pc[k], p1 = pc[k + 1];
      return make_float2(fmaf(w1, p1.x - p0.x, p0.x), fmaf(w1, p1.y - p0.y, p0.y));
    };
    float kr[32];
    auto mul = [&](auto ec, int idx, float2 v) -> float2 {
      constexpr int e = decltype(ec)::value;
      (void)e;
      if constexpr (TM) {  // 16 values per TMEM round trip
        if constexpr (e % 16 == 0) tmem_ld32(kt + 2 * e, kr);
        return cmul(v, make_float2(kr[2 * (e % 16)], kr[2 * (e % 16) + 1]));
      } else {
        return cmul(v, __ldg(kcol + idx));
      }
    };
    float2* ycol = Yh + ((size_t)b * nh + m) * nrho_pad;
    int sq = 0;  // position among the thread's stores (block_conv's last pass is fully unrolled)
    uint32_t crs[16];
    auto store = [&](int idx, float2 v) {  // rows below row_lo / outside the readout's bands are never read downstream
      if constexpr (TMC) {
        if (sq == 0) tmem_ld16(kt + 2 * E + 32, crs);
        if ((smask >> sq) & 1u) ycol[crs[sq]] = v;
      } else {
        if ((smask >> sq) & 1u) ycol[rowmap ? __ldg(rowmap + idx) : idx] = v;
      }
      ++sq;
    };
    if (nrho + ti < zend) {  // padding rows read as zero (K45)
      const int c = rowmap ? __ldg(rowmap + nrho + ti) : nrho + ti;
      if (c >= 0 && c < nrho_pad) ycol[c] = make_float2(0.f, 0.f);
    }
    block_conv<L, PRUNE, 16>(buf, ti, tw, load, mul, store, block_sync);  // SFU twiddles for every pass
  }
  if constexpr (TM) {
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_free<TCOLS>(tslot);
  }
}

// ---------------------------------------------------------------------------
// K4: inverse real DFT along phi for TR log-polar rows per CTA.  Rows i, i+1 are
// packed: Z[k] = X_i[k] + i X_{i+1}[k] with Hermitian extension for k > nphi/2;
// DC and Nyquist imaginary parts are dropped (numpy irfft convention).
// ---------------------------------------------------------------------------
template <int NPHI, int TR, int G>
__global__ void __launch_bounds__(G * FftPlan<NPHI, true>::T)
k_row_irdft(const float2* __restrict__ Yh, float* __restrict__ lp, int nrho, int nrho_pad,
            const float2* __restrict__ tw) {
  constexpr int T = FftPlan<NPHI, true>::T;
  constexpr int NH = NPHI / 2 + 1;
  constexpr int SP = TR + 1;  // odd pitch: conflict-free FFT reads
  extern __shared__ __align__(16) float2 smem_k4[];
  float2* stg = smem_k4;
  float2* buf = smem_k4 + NH * SP + (threadIdx.x / T) * padded_len(NPHI);
  const int gi = threadIdx.x / T, ti = threadIdx.x % T;
  const int i0 = blockIdx.x * TR;
  const float2* src = Yh + (size_t)blockIdx.y * NH * nrho_pad + i0;
  float* dst = lp + (size_t)blockIdx.y * nrho * NPHI;

#pragma unroll 8
  for (int e = threadIdx.x; e < NH * TR; e += blockDim.x) {
    const int m = e / TR, c = e % TR;
    cp_async8(stg + m * SP + c, src + (size_t)m * nrho_pad + c);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int round = 0; round < TR / 2 / G; ++round) {
    const int q = round * G + gi;
    const int ia = i0 + 2 * q, ib = ia + 1;
    const bool va = ia < nrho, vb = ib < nrho;  // rows past nrho read padding: force zero
    auto load = [&](int idx) -> float2 {
      const bool hi = idx > NPHI / 2;
      const int mm = hi ? NPHI - idx : idx;
      float2 xa = stg[mm * SP + 2 * q], xb = stg[mm * SP + 2 * q + 1];
      if (!va) xa = make_float2(0.f, 0.f);
      if (!vb) xb = make_float2(0.f, 0.f);
      if (mm == 0 || mm == NPHI / 2) {
        xa.y = 0.f;
        xb.y = 0.f;
      }
      if (hi) {
        xa.y = -xa.y;
        xb.y = -xb.y;
      }
      return make_float2(xa.x - xb.y, xa.y + xb.x);
    };
    auto store = [&](int idx, float2 v) {
      if (ia < nrho) dst[(size_t)ia * NPHI + idx] = v.x;
      if (ib < nrho) dst[(size_t)ib * NPHI + idx] = v.y;
    };
    block_fft<NPHI, true, false>(buf, ti, tw, load, store, block_sync);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K5: bilinear readout at the Cartesian pixel centres.  Coordinates come from
// the plan's fp64-built quadrant table; the other quadrants reflect phi:
//   x<0,y>=0: pi - phi   x<0,y<0: pi + phi   x>=0,y<0: 2 pi - phi
// ---------------------------------------------------------------------------
__device__ __forceinline__ float readout_pixel(const float* __restrict__ l, int iy, int jx, int n, int nq, int nrho,
                                               int nphi, const uint32_t* __restrict__ qidx,
                                               const float2* __restrict__ qw) {
  const int c = n / 2;
  const bool yneg = iy < c, xneg = jx < c;
  const int qy = yneg ? (n - 1 - iy) - c : iy - c;
  const int qx = xneg ? (n - 1 - jx) - c : jx - c;
  const uint32_t e = __ldg(qidx + qy * nq + qx);
  if (e == 0xFFFFFFFFu) return 0.f;
  const float2 w = __ldg(qw + qy * nq + qx);
  const int i0 = (int)(e & 0xFFFFu);
  const int jr = (int)(e >> 16);
  int j0;
  float wj;
  if (!xneg && !yneg) {
    j0 = jr;
    wj = w.y;
  } else if (xneg && yneg) {
    j0 = nphi / 2 + jr;
    wj = w.y;
  } else {
    const int Q = xneg ? nphi / 2 : nphi;  // fj = Q - fj_rep
    if (w.y == 0.f) {
      j0 = Q - jr;
      wj = 0.f;
    } else {
      j0 = Q - jr - 1;
      wj = 1.f - w.y;
    }
  }
  if (j0 >= nphi) j0 -= nphi;
  const int j1 = (j0 + 1 == nphi) ? 0 : j0 + 1;
  const int i1 = min(i0 + 1, nrho - 1);
  const float a00 = __ldg(l + (size_t)i0 * nphi + j0), a01 = __ldg(l + (size_t)i0 * nphi + j1);
  const float a10 = __ldg(l + (size_t)i1 * nphi + j0), a11 = __ldg(l + (size_t)i1 * nphi + j1);
  const float r0 = fmaf(wj, a01 - a00, a00);
  const float r1 = fmaf(wj, a11 - a10, a10);
  return fmaf(w.x, r1 - r0, r0);
}

// 4 pixels per thread (independent gathers in flight); grid.x covers n*n/4.
__global__ void __launch_bounds__(256)
k_readout(const float* __restrict__ lp, float* __restrict__ img, int n, int nq, int nrho, int nphi,
          const uint32_t* __restrict__ qidx, const float2* __restrict__ qw, float scale) {
  const int npix = n * n;
  const int base = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (base >= npix) return;
  const float* l = lp + (size_t)blockIdx.y * nrho * nphi;
  float* o = img + (size_t)blockIdx.y * npix;
  float v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int pix = base + u;
    v[u] = 0.f;
    if (pix < npix) {
      const int iy = pix / n;
      v[u] = readout_pixel(l, iy, pix - iy * n, n, nq, nrho, nphi, qidx, qw) * scale;
    }
  }
  if (base + 3 < npix && ((reinterpret_cast<uintptr_t>(o + base) & 15) == 0)) {
    *reinterpret_cast<float4*>(o + base) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (base + u < npix) o[base + u] = v[u];
  }
}

// ---------------------------------------------------------------------------
// K45: fused inverse phi-DFT + Cartesian readout, streamed along rho.
// Bands of 4 log-polar rows ("steps"); band b owns the pixels whose taps are
// i0, i0+1 with i0 in [r0-1, r0+3), r0 = row_min + 4b, i.e. its own rows and the
// last row of band b-1.  Persistent CTAs, warp-specialised:
//  * a producer warp takes work units (host-built band ranges, cost-balanced,
//    outermost = pixel-heaviest first, slices interleaved in pairs) from an atomic counter,
//    compacts each unit's needed bands (bands no pixel taps are never loaded) plus
//    the band before the unit (its last row feeds the unit's first band), and for
//    each step waits until a ring region is free (`empty` mbarrier), publishes the
//    step descriptor and lands the spectra there by 3-D TMA boxes {2 rows, 256 m}
//    (one box set per FFT group, [m][2] inside the group's half; `full` mbarrier);
//  * the two FFT groups inverse-transform a row pair each in place, meet at one
//    consumer barrier, sample their pixels from the region (and the previous
//    region's last row), and release the previous region.
// The log-polar image never reaches HBM; there are no CTA-wide barriers per step.
// ---------------------------------------------------------------------------
template <int NPHI>
struct FusedShape {
  static constexpr int S = 4;       // log-polar rows per step (one packed pair per FFT group)
  static constexpr int G = S / 2;   // FFT groups
  static constexpr int NR = 3;      // ring regions (previous, current, next step)
  static constexpr int UQ = kFusedMaxUnit;  // max bands per work unit (plan_host kMaxUnitBands); the producer's
                                            // ballot covers them and the reloaded band before the unit
  static_assert(UQ + 1 <= 32, "one producer lane per band of a unit");
  // spectra m = 0 .. NPHI/2: NFULL boxes of 256 rows + one 1-row tail box
  static constexpr int NFULL = (NPHI / 2) / 256;
  static_assert(NFULL * 256 + 1 == NPHI / 2 + 1, "tail box is one row");
  // FFT buffer / row storage per group; +8 float2 skews the groups' rows by 16 banks
  static constexpr int HALF = (padded_len(NPHI) + 15) / 16 * 16 + 8;
  // group g's two spectra rows arrive as [m][2] at g * IN_PITCH (128-B aligned, inside its own half)
  static constexpr int IN_PITCH = (HALF + 15) / 16 * 16;
  static_assert((G - 1) * IN_PITCH + 2 * (NPHI / 2 + 1) <= G * HALF, "group input inside its FFT half");
  static constexpr int QREG = (G * HALF + 15) / 16 * 16;  // float2, 128-B multiple (TMA destination)
  static constexpr size_t SMEM = (size_t)NR * QREG * 8 + 2 * NR * 8 + 4 * 16 + 64;  // regions + full/empty + step descriptors
};

template <int NPHI>
__global__ void __launch_bounds__(FusedShape<NPHI>::G * FftPlan<NPHI, true>::T + 32, 1)
k_irdft_readout(const __grid_constant__ CUtensorMap ymap, const __grid_constant__ CUtensorMap ytail,
                float* __restrict__ img, int nrho, int n, int nq,
                int row_min, int nsteps, int batch, int* __restrict__ counter, const uint32_t* __restrict__ step_off,
                const uint32_t* __restrict__ step_need, const uint2* __restrict__ units, int nunits,
                const uint4* __restrict__ entries, float scale, const float2* __restrict__ tw) {
  using FS = FusedShape<NPHI>;
  constexpr int S = FS::S, G = FS::G, NR = FS::NR, QREG = FS::QREG, HALF = FS::HALF;
  constexpr int NFULL = FS::NFULL;
  static_assert(NR == 3, "ring = previous (its last row feeds the readout), current, next");
  constexpr int T = FftPlan<NPHI, true>::T;
  constexpr int NC = G * T, NCW = NC / 32;  // consumer threads: the FFT groups, which also sample the readout
  constexpr int RPITCH = NPHI + 8;  // floats from row a to row b inside a group half (8-bank skew)
  static_assert(RPITCH + NPHI <= 2 * HALF, "row storage");
  constexpr uint32_t STEP_BYTES = (NFULL * 256 + 1) * S * 8;
  static_assert(G * (NFULL + 1) <= 31, "one TMA box per producer lane, lane 31 prefetches entries");
  extern __shared__ __align__(128) float2 smem_k45[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_k45 + NR * QREG);  // [NR] region landed (TMA bytes)
  uint64_t* empty = full + NR;                                         // [NR] region released by the consumers
  int4* items = reinterpret_cast<int4*>(empty + NR);                   // [4] step descriptors, ring by item
  const int total_units = nunits * batch;
  const int c = n / 2;

  if (threadIdx.x == 0) {
    for (int r = 0; r < NR; ++r) {
      mbar_init(&full[r], 1);
      mbar_init(&empty[r], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (threadIdx.x >= NC) {
    // ---- producer warp: walks work units (taken dynamically, outermost first) and their needed
    // steps, runs up to two steps ahead of the consumers: waits until a ring region is released,
    // publishes the step's descriptor and lands its spectra there by TMA.
    const int lane = threadIdx.x - NC;
    int slice = 0, k0 = 0, ks = 0, nl = 0, lpos = 0;
    unsigned bits = 0, snv = 0;
    for (int i = 0;; ++i) {
      bool done = false;
      while (lpos >= nl) {  // next unit with at least one needed step
        int uu = 0;
        if (lane == 0) uu = atomicAdd(counter, 1);
        uu = __shfl_sync(0xFFFFFFFFu, uu, 0);
        if (uu >= total_units) {
          done = true;
          break;
        }
        // slices interleaved in pairs: a unit's pixel entries serve two slices from L2, and only two
        // slices' images are written at a time, so partial image sectors complete in L2 (measured:
        // all slices interleaved 28.7 us/slice with 1.39x image write traffic, pairs 26.8 us at 1.02x,
        // one slice at a time 27.7 us with the entry table re-read from DRAM)
        constexpr int SG = 2;
        const int grp = uu / (nunits * SG);
        const int gs = min(SG, batch - grp * SG);
        const int within = uu - grp * nunits * SG;
        slice = grp * SG + within % gs;
        const uint2 ub = __ldg(units + within / gs);
        k0 = (int)ub.x;
        const int k1 = (int)ub.y;
        ks = k0 > 0 ? k0 - 1 : 0;  // the band before the unit feeds its first band's carried row
        const int st = ks + lane;
        snv = st < k1 ? __ldg(step_need + st) : 0u;  // 0 = nobody taps the band, else 1 + its first row in Y
        bits = __ballot_sync(0xFFFFFFFFu, snv != 0u);
        nl = __popc(bits);
        lpos = 0;
      }
      const int r = i % NR;
      if (i >= NR) mbar_wait(&empty[r], (uint32_t)((i / NR - 1) & 1));
      if (done) {
        if (lane == 0) {
          items[i & 3] = make_int4(-1, 0, 0, 0);
          mbar_arrive(&full[r]);
        }
        break;
      }
      const int kk = ks + (int)__fns(bits, 0, lpos + 1);
      ++lpos;
      const int yrow = (int)__shfl_sync(0xFFFFFFFFu, snv, kk - ks) - 1;  // where K3 stored the band's first row
      const bool rd = kk >= k0;  // the reloaded band before the unit only provides its last row
      uint32_t e0 = 0, e1 = 0;
      if (rd && lane == 0) {
        e0 = __ldg(step_off + kk);
        e1 = __ldg(step_off + kk + 1);
      }
      if (lane == 0) {
        items[i & 3] = make_int4(slice, kk | (rd ? 1 << 30 : 0), (int)e0, (int)e1);
        fence_proxy_async_smem();  // the consumers' generic accesses to the region before the TMA writes
        mbar_arrive_expect_tx(&full[r], STEP_BYTES);  // releases the descriptor store with the arrival
      }
      __syncwarp();
      if (lane < G * (NFULL + 1)) {  // rows (r0 + 2g, r0 + 2g + 1) -> group g's input as [m][2]
        const int g = lane / (NFULL + 1), bx = lane - g * (NFULL + 1);
        const int c0 = 2 * (yrow + 2 * g);
        float2* dst = smem_k45 + r * QREG + g * FS::IN_PITCH + 2 * (bx * 256);
        if (bx < NFULL) tma_load_3d(dst, &ymap, c0, bx * 256, slice, &full[r]);
        else tma_load_3d(dst, &ytail, c0, NFULL * 256, slice, &full[r]);
      }
      const uint32_t pa = __shfl_sync(0xFFFFFFFFu, e0, 0), pb = __shfl_sync(0xFFFFFFFFu, e1, 0);
      if (lane == 31 && pb > pa) prefetch_l2_bulk(entries + pa, 16u * (pb - pa));  // warm L2 with its pixels
    }
    return;
  }

  // ---- consumers: one step per item, in the producer's order
  const int gi = threadIdx.x / T, ti = threadIdx.x % T;
  auto row_of = [&](const float2* Q, int li) -> const float* {  // row li in [0, S) of a step region
    return reinterpret_cast<const float*>(Q + (li >> 1) * HALF) + (li & 1) * RPITCH;
  };
#pragma unroll 1
  for (int i = 0;; ++i) {
    const int R = i % NR;
    mbar_wait(&full[R], (uint32_t)((i / NR) & 1));
    const int4 itm = items[i & 3];
    if (itm.x < 0) break;
    const int slice = itm.x, kk = itm.y & 0x3FFFFFFF;
    const bool rd = (itm.y >> 30) & 1;
    const uint32_t e0 = (uint32_t)itm.z, e1 = (uint32_t)itm.w;
    // a band nobody taps is never loaded and the band before a unit is reloaded, so the previous item's
    // region (Qprev) is read only when it holds band kk - 1 of the same slice
    const float2* Qprev = smem_k45 + ((i + NR - 1) % NR) * QREG;
    float2* Q = smem_k45 + R * QREG;
    const int r0 = row_min + S * kk;
    float* out = img + (size_t)slice * n * n;
    // first pixel entries of this step: loads in flight across the transforms
    uint4 pre = make_uint4(0x80000000u, 0, 0, 0), pre2 = pre;
    const uint32_t ep = e0 + threadIdx.x;
    if (ep < e1) pre = __ldg(entries + ep);
    if (ep + NC < e1) pre2 = __ldg(entries + ep + NC);

    // inverse DFTs of rows (r0 + 2 gi, r0 + 2 gi + 1), in place in this group's part
    float2* H = Q + gi * HALF;
    float* Hf = reinterpret_cast<float*>(H);
    const float2* Qin = Q + gi * FS::IN_PITCH;
    // packed Z[k] = Xa[k] + i Xb[k], Hermitian extension for k > nphi/2; element r of pass 0
    // (k = j + r*QS) sits in the low half for r < R0/2.  DC / Nyquist imaginary parts dropped.
    // Rows in [nrho, nrho_pad) are zero (written by K3), rows past nrho_pad arrive as TMA zero fill.
    constexpr int R0 = FftPlan<NPHI, true>::radix(0), QS = NPHI / R0;
    auto load = [&](int j, auto rc) -> float2 {
      constexpr int r = decltype(rc)::value;
      if constexpr (r < R0 / 2) {
        const float4 x = *reinterpret_cast<const float4*>(Qin + 2 * (j + r * QS));
        float2 z = make_float2(x.x - x.w, x.y + x.z);
        if constexpr (r == 0)
          if (j == 0) z = make_float2(x.x, x.z);
        return z;
      } else {
        const float4 x = *reinterpret_cast<const float4*>(Qin + 2 * ((R0 - r) * QS - j));
        float2 z = make_float2(x.x + x.w, x.z - x.y);
        if constexpr (r == R0 / 2)
          if (j == 0) z = make_float2(x.x, x.z);
        return z;
      }
    };
    auto store = [&](int idx, float2 v) {
      Hf[idx] = v.x;
      Hf[RPITCH + idx] = v.y;
    };
    block_fft<NPHI, true, true, true, false, 16>(H, ti, tw, load, store, GroupSync{1 + gi, T});  // group-local
    GroupSync{1 + G, NC}();  // both groups' rows are in place (consumers only; the producer runs ahead)

    if (rd) {  // readout: taps from this step's rows and the previous step's last row
      auto pixel = [&](const uint4& ent) {
        const int qy = (int)(ent.x & 0x7FFFu), qx = (int)((ent.x >> 15) & 0xFFFFu);
        const int iyp = c + qy, iyn = n - 1 - c - qy;
        const int jxp = c + qx, jxn = n - 1 - c - qx;
        const bool dupy = iyn == iyp, dupx = jxn == jxp;  // odd n: centre row / column
        float v1 = 0.f, v2 = 0.f, v3 = 0.f, v4 = 0.f;
        if (!(ent.x & 0x80000000u)) {
          const int i0 = (int)(ent.y & 0xFFFFu), jr = (int)(ent.y >> 16);
          const float wi = __uint_as_float(ent.z), wjr = __uint_as_float(ent.w);
          const int l0 = i0 - r0, l1 = min(i0 + 1, nrho - 1) - r0;
          const float* row0 = l0 < 0 ? row_of(Qprev, S - 1) : row_of(Q, l0);
          const float* row1 = row_of(Q, l1);
          auto sample = [&](int j0, float wj) {
            if (j0 >= NPHI) j0 -= NPHI;
            const int j1 = (j0 + 1 == NPHI) ? 0 : j0 + 1;
            const float a0 = fmaf(wj, row0[j1] - row0[j0], row0[j0]);
            const float a1 = fmaf(wj, row1[j1] - row1[j0], row1[j0]);
            return fmaf(wi, a1 - a0, a0) * scale;
          };
          const bool wz = wjr == 0.f;
          const float wm = wz ? 0.f : 1.f - wjr;
          v1 = sample(jr, wjr);                                      // x >= 0, y >= 0
          v2 = sample(wz ? NPHI / 2 - jr : NPHI / 2 - jr - 1, wm);  // x < 0, y >= 0: pi - phi
          v3 = sample(NPHI / 2 + jr, wjr);                           // x < 0, y < 0: pi + phi
          v4 = sample(wz ? NPHI - jr : NPHI - jr - 1, wm);          // x >= 0, y < 0: 2 pi - phi
        }
        out[(size_t)iyp * n + jxp] = v1;
        if (!dupx) out[(size_t)iyp * n + jxn] = v2;
        if (!dupy) {
          out[(size_t)iyn * n + jxp] = v4;
          if (!dupx) out[(size_t)iyn * n + jxn] = v3;
        }
      };
      if (ep < e1) {  // entry loads run two pixels ahead; three rotating registers, no copies
        uint4 ea = pre, eb = pre2, ec;
        const uint32_t stp = NC;
        uint32_t e = ep;
        auto fetch = [&](uint4& dst) {
          dst = make_uint4(0x80000000u, 0, 0, 0);
          if (e + 2 * stp < e1) dst = __ldg(entries + e + 2 * stp);
        };
#pragma unroll 1
        for (;;) {
          fetch(ec);
          pixel(ea);
          if ((e += stp) >= e1) break;
          fetch(ea);
          pixel(eb);
          if ((e += stp) >= e1) break;
          fetch(eb);
          pixel(ec);
          if ((e += stp) >= e1) break;
        }
      }
    }
    // this warp is done with the previous item's region (its last row fed this readout)
    if (i >= 1) {
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[(i + NR - 1) % NR]);
    }
  }
}

// ---------------------------------------------------------------------------
// K45 for mixed-radix lengths nphi = Q P (mixed.cuh): the same streaming scheme as
// k_irdft_readout — a producer warp walks the work units and their needed bands, the
// consumers inverse-transform each band and sample its pixels in shared memory, so the
// log-polar image never reaches HBM — with bands of 2 rows (one packed pair: the
// mixed-radix transform of a pair needs the whole CTA's Q P / 16 threads) and a
// two-stage ring: the band's spectra land by 3-D TMA boxes {2 rows, 256 m} in one of two
// input buffers (released to the producer as soon as step A has read them), and the
// transform runs in one of two row buffers (the other holds the previous band, whose
// second row is the current band's carried row).
// ---------------------------------------------------------------------------
template <int Q, int P>
struct FusedMixedShape {
  using MS = MixedShape<Q, P>;
  static constexpr int N = Q * P, NH = N / 2 + 1, S = 2;
  static constexpr int NBOX = (NH + 255) / 256;
  static constexpr int IN = NBOX * 256 * 2;        // float2 per input buffer ([m][2 rows])
  static constexpr int RB = MS::ROWS * MS::PITCH;  // float2 per row buffer (mixed layout)
  static constexpr int RBA = (RB + 15) / 16 * 16;  // 128-B multiple
  static constexpr int NC = MS::THREADS, NTHR = NC + 32;
  static constexpr uint32_t STEP_BYTES = (uint32_t)NBOX * 256 * 16;
  static constexpr size_t SMEM = ((size_t)2 * IN + 2 * (size_t)RBA) * 8 + 4 * 8 + 4 * 16 + 64;
  static_assert(NBOX <= 31, "one TMA box per producer lane, lane 31 prefetches entries");
};

template <int Q, int P>
__global__ void __launch_bounds__(FusedMixedShape<Q, P>::NTHR, 1)
k_irdft_readout_mixed(const __grid_constant__ CUtensorMap ymap, float* __restrict__ img, int nrho, int n, int nq,
                      int row_min, int batch, int* __restrict__ counter, const uint32_t* __restrict__ step_off,
                      const uint32_t* __restrict__ step_need, const uint2* __restrict__ units, int nunits,
                      const uint4* __restrict__ entries, float scale) {
  using FS = FusedMixedShape<Q, P>;
  constexpr int N = FS::N, S = FS::S, NC = FS::NC, NCW = NC / 32, IN = FS::IN, RBA = FS::RBA;
  extern __shared__ __align__(128) float2 smem_kx[];
  float2* inbuf = smem_kx;               // [2][IN]
  float2* rows = smem_kx + 2 * IN;       // [2][RBA]
  uint64_t* full = reinterpret_cast<uint64_t*>(rows + 2 * RBA);  // [2] input landed (TMA bytes)
  uint64_t* empty = full + 2;                                    // [2] input consumed by step A
  int4* items = reinterpret_cast<int4*>(empty + 2);              // [4] step descriptors, ring by item
  const int total_units = nunits * batch;
  const int c = n / 2;
  if (threadIdx.x == 0) {
    for (int r = 0; r < 2; ++r) {
      mbar_init(&full[r], 1);
      mbar_init(&empty[r], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (threadIdx.x >= NC) {  // ---- producer warp (as in k_irdft_readout, two input buffers)
    const int lane = threadIdx.x - NC;
    int slice = 0, k0 = 0, ks = 0, nl = 0, lpos = 0;
    unsigned bits = 0, snv = 0;
    for (int i = 0;; ++i) {
      bool done = false;
      while (lpos >= nl) {
        int uu = 0;
        if (lane == 0) uu = atomicAdd(counter, 1);
        uu = __shfl_sync(0xFFFFFFFFu, uu, 0);
        if (uu >= total_units) {
          done = true;
          break;
        }
        constexpr int SG = 2;  // slices in pairs (see k_irdft_readout)
        const int grp = uu / (nunits * SG);
        const int gs = min(SG, batch - grp * SG);
        const int within = uu - grp * nunits * SG;
        slice = grp * SG + within % gs;
        const uint2 ub = __ldg(units + within / gs);
        k0 = (int)ub.x;
        const int k1 = (int)ub.y;
        ks = k0 > 0 ? k0 - 1 : 0;
        const int st = ks + lane;
        snv = st < k1 ? __ldg(step_need + st) : 0u;  // 0 = nobody taps the band, else 1 + its first row in Y
        bits = __ballot_sync(0xFFFFFFFFu, snv != 0u);
        nl = __popc(bits);
        lpos = 0;
      }
      const int r = i & 1;
      if (i >= 2) mbar_wait(&empty[r], (uint32_t)((i / 2 - 1) & 1));
      if (done) {
        if (lane == 0) {
          items[i & 3] = make_int4(-1, 0, 0, 0);
          mbar_arrive(&full[r]);
        }
        break;
      }
      const int kk = ks + (int)__fns(bits, 0, lpos + 1);
      ++lpos;
      const int yrow = (int)__shfl_sync(0xFFFFFFFFu, snv, kk - ks) - 1;
      const bool rd = kk >= k0;
      uint32_t e0 = 0, e1 = 0;
      if (rd && lane == 0) {
        e0 = __ldg(step_off + kk);
        e1 = __ldg(step_off + kk + 1);
      }
      if (lane == 0) {
        items[i & 3] = make_int4(slice, kk | (rd ? 1 << 30 : 0), (int)e0, (int)e1);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&full[r], FS::STEP_BYTES);
      }
      __syncwarp();
      if (lane < FS::NBOX)  // rows (r0, r0 + 1) as [m][2]; m >= nh is zero fill
        tma_load_3d(inbuf + r * IN + 2 * (lane * 256), &ymap, 2 * yrow, lane * 256, slice, &full[r]);
      const uint32_t pa = __shfl_sync(0xFFFFFFFFu, e0, 0), pb = __shfl_sync(0xFFFFFFFFu, e1, 0);
      if (lane == 31 && pb > pa) prefetch_l2_bulk(entries + pa, 16u * (pb - pa));
    }
    return;
  }

  // ---- consumers
  const int tid = threadIdx.x;
  auto team = [] { asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory"); };
  const int ntheta = N / 2;
#pragma unroll 1
  for (int i = 0;; ++i) {
    const int r = i & 1;
    mbar_wait(&full[r], (uint32_t)((i / 2) & 1));
    const int4 itm = items[i & 3];
    if (itm.x < 0) break;
    const int slice = itm.x, kk = itm.y & 0x3FFFFFFF;
    const bool rd = (itm.y >> 30) & 1;
    const uint32_t e0 = (uint32_t)itm.z, e1 = (uint32_t)itm.w;
    const float4* stg = reinterpret_cast<const float4*>(inbuf + r * IN);
    float2* cur = rows + (i & 1) * RBA;
    const float2* prev = rows + ((i + 1) & 1) * RBA;  // the previous item's rows: band kk - 1 when used
    const int r0 = row_min + S * kk;
    float* out = img + (size_t)slice * n * n;
    uint4 pre = make_uint4(0x80000000u, 0, 0, 0), pre2 = pre;
    const uint32_t ep = e0 + tid;
    if (ep < e1) pre = __ldg(entries + ep);
    if (ep + NC < e1) pre2 = __ldg(entries + ep + NC);
    team();  // the previous item's readout is done with `cur` (it was that item's `prev`)
    auto load = [&](int idx) -> float2 {  // Hermitian assembly of the packed pair, as k_row_irdft_mixed
      const bool hi = idx > ntheta;
      const int mm = hi ? N - idx : idx;
      float4 x = stg[mm];
      if (mm == 0 || mm == ntheta) {
        x.y = 0.f;
        x.w = 0.f;
      }
      if (hi) {
        x.y = -x.y;
        x.w = -x.w;
      }
      return make_float2(x.x - x.w, x.y + x.z);
    };
    // step A reads the input buffer (returned to the producer at the first team barrier), step B
    // transforms `cur` in place; the call ends with a team barrier
    int nsync = 0;
    block_dft_mixed_team<Q, P, true, 2>(cur, tid, load, [&] {
      team();
      if (nsync++ == 0 && (tid & 31) == 0) mbar_arrive(&empty[r]);
    });
    if (rd) {  // readout: rows r0 (.x) and r0 + 1 (.y) of `cur`, row r0 - 1 = the previous band's .y
      auto val = [&](int li, int j) -> float {
        if (li < 0) return mixed_at<Q, P>(prev, j).y;
        const float2 z = mixed_at<Q, P>(cur, j);
        return li == 0 ? z.x : z.y;
      };
      auto pixel = [&](const uint4& ent) {
        const int qy = (int)(ent.x & 0x7FFFu), qx = (int)((ent.x >> 15) & 0xFFFFu);
        const int iyp = c + qy, iyn = n - 1 - c - qy;
        const int jxp = c + qx, jxn = n - 1 - c - qx;
        const bool dupy = iyn == iyp, dupx = jxn == jxp;
        float v1 = 0.f, v2 = 0.f, v3 = 0.f, v4 = 0.f;
        if (!(ent.x & 0x80000000u)) {
          const int i0 = (int)(ent.y & 0xFFFFu), jr = (int)(ent.y >> 16);
          const float wi = __uint_as_float(ent.z), wjr = __uint_as_float(ent.w);
          const int l0 = i0 - r0, l1 = min(i0 + 1, nrho - 1) - r0;
          auto sample = [&](int j0, float wj) {
            if (j0 >= N) j0 -= N;
            const int j1 = (j0 + 1 == N) ? 0 : j0 + 1;
            const float a00 = val(l0, j0), a01 = val(l0, j1), a10 = val(l1, j0), a11 = val(l1, j1);
            const float a0 = fmaf(wj, a01 - a00, a00);
            const float a1 = fmaf(wj, a11 - a10, a10);
            return fmaf(wi, a1 - a0, a0) * scale;
          };
          const bool wz = wjr == 0.f;
          const float wm = wz ? 0.f : 1.f - wjr;
          v1 = sample(jr, wjr);
          v2 = sample(wz ? N / 2 - jr : N / 2 - jr - 1, wm);
          v3 = sample(N / 2 + jr, wjr);
          v4 = sample(wz ? N - jr : N - jr - 1, wm);
        }
        out[(size_t)iyp * n + jxp] = v1;
        if (!dupx) out[(size_t)iyp * n + jxn] = v2;
        if (!dupy) {
          out[(size_t)iyn * n + jxp] = v4;
          if (!dupx) out[(size_t)iyn * n + jxn] = v3;
        }
      };
      if (ep < e1) {
        uint4 ea = pre, eb = pre2, ec;
        const uint32_t stp = NC;
        uint32_t e = ep;
        auto fetch = [&](uint4& dst) {
          dst = make_uint4(0x80000000u, 0, 0, 0);
          if (e + 2 * stp < e1) dst = __ldg(entries + e + 2 * stp);
        };
#pragma unroll 1
        for (;;) {
          fetch(ec);
          pixel(ea);
          if ((e += stp) >= e1) break;
          fetch(ea);
          pixel(eb);
          if ((e += stp) >= e1) break;
          fetch(eb);
          pixel(ec);
          if ((e += stp) >= e1) break;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Generic sizes (any nt, any ntheta; nphi = 2 ntheta need not be a power of two).
// The length-nphi DFTs use Bluestein's identity with the same pow2 block_conv:
//   X[k] = c[k] sum_n (x[n] c[n]) conj c[k-n],  c[n] = exp(-i pi n^2 / nphi),
// a circular MB-point convolution (MB = pow2 >= 2 nphi) with the plan's
// precomputed spectrum of the chirp filter.  One CTA per row (column) pair.
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(FftPlan<M, false>::T)
k_ramp_generic(const float* __restrict__ g, float* __restrict__ out, int nt, int ntheta,
               const float* __restrict__ resp, const float2* __restrict__ tw) {
  extern __shared__ __align__(16) float2 smem_g1[];
  const int ca = 2 * blockIdx.x, cb = ca + 1;
  const bool hb = cb < ntheta;
  const size_t slice = (size_t)blockIdx.y * nt * ntheta;
  const float* src = g + slice;
  float* dst = out + slice;
  auto load = [&](int idx) -> float2 {
    if (idx >= nt) return make_float2(0.f, 0.f);
    const float* r = src + (size_t)idx * ntheta;
    return make_float2(__ldg(r + ca), hb ? __ldg(r + cb) : 0.f);
  };
  auto mul = [&](int idx, float2 v) -> float2 { return cscale(v, __ldg(resp + idx)); };
  auto store = [&](int idx, float2 v) {
    if (idx < nt) {
      dst[(size_t)idx * ntheta + ca] = v.x;
      if (hb) dst[(size_t)idx * ntheta + cb] = v.y;
    }
  };
  block_conv<M, true, 16>(smem_g1, threadIdx.x, tw, load, mul, store, block_sync);  // M >= 2 nt
}

template <int MB>
__global__ void __launch_bounds__(FftPlan<MB, false>::T)
k_row_rdft_generic(const float* __restrict__ g, float2* __restrict__ Gh, int nt, int gp, int ntheta, int win, int win_lo,
                   const float2* __restrict__ chirp, const float2* __restrict__ bhat, const float2* __restrict__ tw) {
  extern __shared__ __align__(16) float2 smem_g2[];
  const int nphi = 2 * ntheta, nh = ntheta + 1;
  float2* buf = smem_g2;
  float2* Z = smem_g2 + padded_len(MB);  // [nphi]
  const int ta = 2 * blockIdx.x, tb = ta + 1;
  const bool hb = tb < nt;
  const float* ra = g + ((size_t)blockIdx.y * nt + ta) * win;  // rows of `win` (<= ntheta) columns
  const float* rb = ra + win;
  const int tail = ntheta - (win - win_lo);  // compacted rows: [0, win_lo) and [tail, ntheta) are stored
  auto load = [&](int idx) -> float2 {  // a[n] = z[n] c[n]; z is zero for n >= ntheta
    if (idx >= ntheta || (idx >= win_lo && idx < tail)) return make_float2(0.f, 0.f);
    const int src = idx >= tail ? idx - (tail - win_lo) : idx;  // storage column
    const float2 z = make_float2(__ldg(ra + src), hb ? __ldg(rb + src) : 0.f);
    return cmul(z, __ldg(chirp + idx));
  };
  auto mul = [&](int idx, float2 v) -> float2 { return cmul(v, __ldg(bhat + idx)); };
  auto store = [&](int idx, float2 v) {
    if (idx < nphi) Z[idx] = cmul(v, __ldg(chirp + idx));
  };
  block_conv<MB, true>(buf, threadIdx.x, tw, load, mul, store, block_sync);
  __syncthreads();
  float2* dst = Gh + (size_t)blockIdx.y * nh * gp + ta;
  for (int m = threadIdx.x; m < nh; m += blockDim.x) {
    const float2 z = Z[m], w = Z[m == 0 ? 0 : nphi - m];
    dst[(size_t)m * gp] = make_float2(0.5f * (z.x + w.x), 0.5f * (z.y - w.y));
    if (hb) dst[(size_t)m * gp + 1] = make_float2(0.5f * (z.y + w.y), 0.5f * (w.x - z.x));
    else if (tb < gp) dst[(size_t)m * gp + 1] = make_float2(0.f, 0.f);  // odd nt: the pad column reads zero (K3 taps)
  }
}

template <int MB>
__global__ void __launch_bounds__(FftPlan<MB, false>::T)
k_row_irdft_generic(const float2* __restrict__ Yh, float* __restrict__ lp, int nrho, int nrho_pad, int ntheta,
                    const float2* __restrict__ chirp, const float2* __restrict__ bhat, const float2* __restrict__ tw,
                    const uint32_t* __restrict__ pairs) {
  extern __shared__ __align__(16) float2 smem_g4[];
  const int nphi = 2 * ntheta, nh = ntheta + 1;
  const int ia = 2 * (pairs ? (int)pairs[blockIdx.x] : (int)blockIdx.x), ib = ia + 1;
  const bool hb = ib < nrho;
  const float2* src = Yh + (size_t)blockIdx.y * nh * nrho_pad;
  float* dst = lp + (size_t)blockIdx.y * nrho * nphi;
  auto load = [&](int idx) -> float2 {  // a[k] = Z[k] conj c[k], Z Hermitian-assembled from Y
    if (idx >= nphi) return make_float2(0.f, 0.f);
    const bool hi = idx > ntheta;
    const int mm = hi ? nphi - idx : idx;
    float2 xa = src[(size_t)mm * nrho_pad + ia];
    float2 xb = hb ? src[(size_t)mm * nrho_pad + ib] : make_float2(0.f, 0.f);
    if (mm == 0 || mm == ntheta) {
      xa.y = 0.f;
      xb.y = 0.f;
    }
    if (hi) {
      xa.y = -xa.y;
      xb.y = -xb.y;
    }
    return cmulc(make_float2(xa.x - xb.y, xa.y + xb.x), __ldg(chirp + idx));
  };
  auto mul = [&](int idx, float2 v) -> float2 { return cmul(v, __ldg(bhat + idx)); };
  auto store = [&](int idx, float2 v) {
    if (idx < nphi) {
      const float2 z = cmulc(v, __ldg(chirp + idx));
      dst[(size_t)ia * nphi + idx] = z.x;
      if (hb) dst[(size_t)ib * nphi + idx] = z.y;
    }
  };
  block_conv<MB, true>(smem_g4, threadIdx.x, tw, load, mul, store, block_sync);
}

// Mixed-radix lengths nphi = Q P (mixed.cuh): the same row transforms as the Bluestein
// kernels above, one CTA per row pair, with the length-nphi DFT computed directly
// (Q-point DFTs in registers + Q power-of-two FFTs) instead of a 2-4x longer circular
// convolution.  LNLS's 3200 angles: nphi = 6400 = 25 x 256.
template <int Q, int P>
__global__ void __launch_bounds__(MixedShape<Q, P>::THREADS)
k_row_rdft_mixed(const float* __restrict__ g, float2* __restrict__ Gh, int nt, int gp, int ntheta, int win,
                 int win_lo) {
  extern __shared__ __align__(16) float2 smem_m2[];
  constexpr int N = Q * P;  // nphi
  const int nh = ntheta + 1;
  const int ta = 2 * blockIdx.x, tb = ta + 1;
  const bool hb = tb < nt;
  const float* ra = g + ((size_t)blockIdx.y * nt + ta) * win;  // rows of `win` (<= ntheta) columns
  const float* rb = ra + win;
  const int tail = ntheta - (win - win_lo);  // compacted rows: [0, win_lo) and [tail, ntheta) are stored
  auto load = [&](int idx) -> float2 {       // rows ta, tb packed as re / im, zero for idx >= ntheta
    if (idx >= ntheta || (idx >= win_lo && idx < tail)) return make_float2(0.f, 0.f);
    const int src = idx >= tail ? idx - (tail - win_lo) : idx;
    return make_float2(__ldg(ra + src), hb ? __ldg(rb + src) : 0.f);
  };
  block_dft_mixed<Q, P, false>(smem_m2, load);
  float2* dst = Gh + (size_t)blockIdx.y * nh * gp + ta;
  for (int m = threadIdx.x; m < nh; m += blockDim.x) {
    const float2 z = mixed_at<Q, P>(smem_m2, m), w = mixed_at<Q, P>(smem_m2, m == 0 ? 0 : N - m);
    const float2 a = make_float2(0.5f * (z.x + w.x), 0.5f * (z.y - w.y));
    const float2 b = hb ? make_float2(0.5f * (z.y + w.y), 0.5f * (w.x - z.x)) : make_float2(0.f, 0.f);
    if (tb < gp) *reinterpret_cast<float4*>(dst + (size_t)m * gp) = make_float4(a.x, a.y, b.x, b.y);  // 16 bytes
    else dst[(size_t)m * gp] = a;  // (odd nt: the pad column past tb reads zero)
  }
}

// The same for the SEMI-POLAR rows (K2p's order of the two linear maps, grids.py:290-311 before the phi DFT):
// rows ka = 2 blockIdx.x and ka + 1 of p, each value two taps of the sinogram (t >= 0 taps for phi < pi,
// t <= 0 taps for phi >= pi; rows `ab`, weights `wab`: out-of-range taps carry weight 0 on a valid row);
// ns = nt/2 full-length transforms instead of nt zero-padded ones, output P[b][m][ns].
template <int Q, int P>
__global__ void __launch_bounds__(MixedShape<Q, P>::THREADS)
k_row_rdft_mixed_p(const float* __restrict__ g, float2* __restrict__ Ph, int nt, int ns, int ntheta,
                   const int2* __restrict__ ab, const float4* __restrict__ wab) {
  extern __shared__ __align__(16) float2 smem_m2p[];
  constexpr int N = Q * P;  // nphi
  const int nh = ntheta + 1;
  const int ka = 2 * blockIdx.x, kb = ka + 1;
  const bool hb = kb < ns;
  const float* base = g + (size_t)blockIdx.y * nt * ntheta;
  const int2 ia = __ldg(ab + ka), ib = hb ? __ldg(ab + kb) : ia;
  const float4 wa = __ldg(wab + ka), wb = hb ? __ldg(wab + kb) : make_float4(0.f, 0.f, 0.f, 0.f);
  const float* xa = base + (size_t)ia.x * ntheta;  // taps xa[j], xa[ntheta + j]
  const float* xb = base + (size_t)ia.y * ntheta;
  const float* ya = base + (size_t)ib.x * ntheta;
  const float* yb = base + (size_t)ib.y * ntheta;
  auto load = [&](int idx) -> float2 {  // rows ka, kb packed as re / im
    if (idx < ntheta)
      return make_float2(fmaf(wa.y, __ldg(xa + ntheta + idx), wa.x * __ldg(xa + idx)),
                         fmaf(wb.y, __ldg(ya + ntheta + idx), wb.x * __ldg(ya + idx)));
    const int j = idx - ntheta;
    return make_float2(fmaf(wa.w, __ldg(xb + ntheta + j), wa.z * __ldg(xb + j)),
                       fmaf(wb.w, __ldg(yb + ntheta + j), wb.z * __ldg(yb + j)));
  };
  block_dft_mixed<Q, P, false>(smem_m2p, load);
  float2* dst = Ph + (size_t)blockIdx.y * nh * ns + ka;  // ns even: both rows by one 16-byte store
  for (int m = threadIdx.x; m < nh; m += blockDim.x) {
    const float2 z = mixed_at<Q, P>(smem_m2p, m), w = mixed_at<Q, P>(smem_m2p, m == 0 ? 0 : N - m);
    *reinterpret_cast<float4*>(dst + (size_t)m * ns) =
        make_float4(0.5f * (z.x + w.x), 0.5f * (z.y - w.y), 0.5f * (z.y + w.y), 0.5f * (w.x - z.x));
  }
}

template <int Q, int P>
__global__ void __launch_bounds__(MixedShape<Q, P>::THREADS)
k_row_irdft_mixed(const __grid_constant__ CUtensorMap ymap, float* __restrict__ lp, int nrho, int ntheta, int nbox,
                  const uint32_t* __restrict__ pairs) {
  extern __shared__ __align__(128) float2 smem_m4[];
  // the CTA's two rows of every spectrum column, [nbox * 256][2] (3-D TMA boxes {2 rows, 256 m}), then
  // the mixed-radix rows
  const float4* stg = reinterpret_cast<const float4*>(smem_m4);
  float2* buf = smem_m4 + 2 * 256 * nbox;
  __shared__ __align__(8) uint64_t bar;
  constexpr int N = Q * P;  // nphi
  const int ia = 2 * (pairs ? (int)pairs[blockIdx.x] : (int)blockIdx.x), ib = ia + 1;
  const bool hb = ib < nrho;
  float* dst = lp + (size_t)blockIdx.y * nrho * N;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) mbar_arrive_expect_tx(&bar, (uint32_t)nbox * 256u * 16u);
    __syncwarp();
    for (int bx = threadIdx.x; bx < nbox; bx += 32)
      tma_load_3d(const_cast<float4*>(stg) + bx * 256, &ymap, 2 * ia, bx * 256, blockIdx.y, &bar);
  }
  mbar_wait(&bar, 0);
  // Z[k] = Xa[k] + i Xb[k], Hermitian-assembled from the staged columns (row ib = nrho is a zero
  // padding row of Y, written by K3)
  auto load = [&](int idx) -> float2 {
    const bool hi = idx > ntheta;
    const int mm = hi ? N - idx : idx;
    float4 x = stg[mm];
    if (mm == 0 || mm == ntheta) {  // numpy irfft drops the DC / Nyquist imaginary parts
      x.y = 0.f;
      x.w = 0.f;
    }
    if (hi) {
      x.y = -x.y;
      x.w = -x.w;
    }
    return make_float2(x.x - x.w, x.y + x.z);
  };
  block_dft_mixed<Q, P, true>(buf, load);
  for (int k = threadIdx.x; k < N; k += blockDim.x) {  // coalesced rows
    const float2 z = mixed_at<Q, P>(buf, k);
    dst[(size_t)ia * N + k] = z.x;
    if (hb) dst[(size_t)ib * N + k] = z.y;
  }
}

// ---------------------------------------------------------------------------
// Input generator: exact ellipse line integrals (radon.py:38-61) in fp64,
// 2 rho A B sqrt(w^2 - tau^2) / w^2, tau = t - c.xi_theta,
// w^2 = A^2 cos^2(theta - gamma) + B^2 sin^2(theta - gamma), summed over the
// ellipses in order (the reference's accumulation order).  Block: 32 angles x 64
// rows, 8 rows per thread in registers; per-(ellipse, angle) terms staged in smem
// in chunks of KC ellipses, so any ellipse count runs.
// ---------------------------------------------------------------------------
constexpr int kRadonKC = 64;

template <typename OutT>
__global__ void __launch_bounds__(256)
k_radon_ellipses(const double* __restrict__ params, int K, int nt, int ntheta, OutT* __restrict__ out) {
  __shared__ double w2s[kRadonKC * 32], cps[kRadonKC * 32], c2s[kRadonKC * 32];
  const int b = blockIdx.z, j0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const double* P = params + (size_t)b * K * 6;
  const double kPi = 3.14159265358979323846;
  const int j = j0 + tx;
  double acc[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) acc[r] = 0.0;
  for (int e0 = 0; e0 < K; e0 += kRadonKC) {
    const int kc = min(kRadonKC, K - e0);
    __syncthreads();  // the previous chunk's terms are consumed
    for (int idx = threadIdx.x; idx < kc * 32; idx += blockDim.x) {
      const int e = e0 + (idx >> 5), jj = idx & 31;
      const int jc = min(j0 + jj, ntheta - 1);
      const double cx = P[e * 6], cy = P[e * 6 + 1], a = P[e * 6 + 2], bb = P[e * 6 + 3];
      const double tilt = P[e * 6 + 4], rho = P[e * 6 + 5];
      const double th = (double)jc * (kPi / ntheta);
      const double ang = th - tilt;
      const double ac = a * cos(ang), bs = bb * sin(ang);
      w2s[idx] = ac * ac + bs * bs;
      cps[idx] = cx * cos(th) + cy * sin(th);
      c2s[idx] = 2.0 * rho * a * bb;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int i = blockIdx.y * 64 + ty + 8 * r;
      const double t = -1.0 + (double)i * (2.0 / nt);
      double s = acc[r];
      for (int e = 0; e < kc; ++e) {
        const double tau = t - cps[e * 32 + tx];
        const double w2 = w2s[e * 32 + tx];
        const double under = w2 - tau * tau;
        if (under > 0.0) s += c2s[e * 32 + tx] * sqrt(under) / w2;
      }
      acc[r] = s;
    }
  }
  if (j >= ntheta) return;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = blockIdx.y * 64 + ty + 8 * r;
    if (i < nt) out[((size_t)b * nt + i) * ntheta + j] = (OutT)acc[r];
  }
}

template <typename OutT>
cudaError_t radon_ellipses_impl(const double* params, int K, int nt, int ntheta, int batch, OutT* out,
                                cudaStream_t s) {
  k_radon_ellipses<OutT><<<dim3((ntheta + 31) / 32, (nt + 63) / 64, batch), 256, 0, s>>>(params, K, nt, ntheta, out);
  return cudaGetLastError();
}
cudaError_t launch_radon_ellipses(const double* params, int K, int nt, int ntheta, int batch, float* out,
                                  cudaStream_t s) {
  return radon_ellipses_impl(params, K, nt, ntheta, batch, out, s);
}
cudaError_t launch_radon_ellipses(const double* params, int K, int nt, int ntheta, int batch, double* out,
                                  cudaStream_t s) {
  return radon_ellipses_impl(params, K, nt, ntheta, batch, out, s);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
namespace {
cudaError_t encode_rowspec_map(CUtensorMap* map, const float2* G, int nt, int nh, int batch, int box_m);

template <typename K>
cudaError_t prep(K kernel, size_t smem) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template <int M, int TC, int G>
cudaError_t ramp_impl(const Dims& d, const DevTables& t, const float* g, float* out, int batch, cudaStream_t s) {
  if (d.ntheta % TC) return cudaErrorNotSupported;
  const size_t smem = ((size_t)(d.nt * (TC + 1) + 1) / 2 + (size_t)G * padded_len(M)) * sizeof(float2);
  auto k = k_ramp<M, TC, G>;
  cudaError_t e = prep(k, smem);
  if (e) return e;
  k<<<dim3(d.ntheta / TC, batch), G * FftPlan<M, false>::T, smem, s>>>(g, out, d.nt, d.ntheta, t.ramp, t.tw_ramp);
  return cudaGetLastError();
}

template <int NPHI>
cudaError_t rdft_impl(const Dims& d, const DevTables& t, const float* g, float2* Gh, int batch, cudaStream_t s) {
  using RS = RdftShape<NPHI>;
  if (d.nt % RS::TR) return cudaErrorNotSupported;
  const int win = d.win > 0 ? d.win : d.ntheta;
  const bool narrow = win < d.ntheta;
  if (narrow && (win % 4)) return cudaErrorNotSupported;  // TMA bulk rows: 16-byte multiples
  auto k = narrow ? k_row_rdft<NPHI, true> : k_row_rdft<NPHI, false>;
  if ((reinterpret_cast<uintptr_t>(Gh) & 15) || (d.nt * 8) % 16) return cudaErrorNotSupported;
  CUtensorMap gm, gt;
  cudaError_t e = encode_rowspec_map(&gm, Gh, d.nt, RS::NH, batch, 256);
  if (!e) e = encode_rowspec_map(&gt, Gh, d.nt, RS::NH, batch, 1);
  if (e) return e;
  e = prep(k, RS::SMEM);
  if (e) return e;
  const int per = d.nt / RS::TR, tiles = per * batch;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, RS::G * FftPlan<NPHI, false>::T, RS::SMEM);
  const int slots = d.nsm * (occ > 0 ? occ : 1);
  const int grid = tiles < slots ? tiles : slots;
  k<<<grid, RS::G * FftPlan<NPHI, false>::T, RS::SMEM, s>>>(gm, gt, g, d.nt, per, tiles, t.tw_phi, win, d.win_lo);
  return cudaGetLastError();
}

template <int NPHI>
cudaError_t rdft_p_impl(const Dims& d, const DevTables& t, const float* g, float2* Ph, int batch, cudaStream_t s) {
  using RS = RdftPShape<NPHI>;
  if (!d.pmix || d.ns % RS::KR || !t.ptile || !t.ploc) return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(Ph) & 15) || (reinterpret_cast<uintptr_t>(g) & 15)) return cudaErrorNotSupported;
  auto k = k_row_rdft_p<NPHI>;
  CUtensorMap pm, pt;
  cudaError_t e = encode_rowspec_map(&pm, Ph, d.ns, RS::NH, batch, 256);
  if (!e) e = encode_rowspec_map(&pt, Ph, d.ns, RS::NH, batch, 1);
  if (e) return e;
  e = prep(k, RS::SMEM);
  if (e) return e;
  const int per = d.ns / RS::KR, tiles = per * batch;
  const int grid = tiles < d.nsm ? tiles : d.nsm;
  k<<<grid, RS::G * FftPlan<NPHI, false>::T + 32, RS::SMEM, s>>>(pm, pt, g, d.nt, per, tiles,
                                                                 reinterpret_cast<const int4*>(t.ptile), t.ploc,
                                                                 t.wab, t.tw_phi);
  return cudaGetLastError();
}

template <int L>
cudaError_t conv_impl(const Dims& d, const DevTables& t, const float2* Gh, float2* Yh, int batch, int row_lo,
                      cudaStream_t s, bool pin, const int32_t* rowmap) {
  const int gp = pin ? d.ns : (d.gp > 0 ? d.gp : d.nt);
  const size_t smem = pin ? ((size_t)padded_len(L) + 2 * (size_t)((d.ns + 3) & ~1)) * sizeof(float2) + (size_t)d.nrho * 4
                          : ((size_t)padded_len(L) + ((d.ns + 1) & ~1) + (size_t)gp + 2) * sizeof(float2) +
                                (size_t)d.nrho * 4;
  // nrho <= L/2: the rho column is zero in the upper half and only rows < nrho are kept
  // Khat in TMEM where L is in [4096, 16384]: at most two 256-thread CTAs per SM (256 columns each) or
  // one 512-thread CTA (512 columns), so an allocation never waits; LPBP_K3_TMEM=0 selects the L2 path
  static const bool tmv = [] {
    const char* v = getenv("LPBP_K3_TMEM");
    return v ? atoi(v) != 0 : true;
  }();
  constexpr bool kTmemOk = L >= 4096 && L <= 16384;  // 16384: one 512-thread CTA per SM, 512 columns
  const bool pr = 2 * d.nrho <= L;
  auto k = pr ? k_rho_conv<L, true, false> : k_rho_conv<L, false, false>;
  if constexpr (kTmemOk) {
    if (tmv) k = pr ? k_rho_conv<L, true, true> : k_rho_conv<L, false, true>;
  }
  if (pin) {  // K2p's semi-polar spectra (pruned transforms only: 2 nrho <= L holds for every automatic mesh)
    if (!pr || (d.ns & 1)) return cudaErrorNotSupported;
    k = k_rho_conv<L, true, false, true>;
    if constexpr (kTmemOk) {
      if (tmv) k = k_rho_conv<L, true, true, true>;
    }
  }
  cudaError_t e = prep(k, smem);
  if (e) return e;
  k<<<d.nh, FftPlan<L, false>::T, smem, s>>>(Gh, Yh, batch, d.nt, gp, d.ns, d.nrho, row_lo, d.nrho_pad, d.nh, t.abw,
                                              t.kw, t.khat, t.tw_rho, rowmap, rowmap ? d.row_end : d.nrho_pad);
  return cudaGetLastError();
}

template <int NPHI, int TR, int G>
cudaError_t irdft_impl(const Dims& d, const DevTables& t, const float2* Yh, float* lp, int batch, cudaStream_t s) {
  if (d.nrho_pad % TR) return cudaErrorNotSupported;
  const size_t smem = ((size_t)(NPHI / 2 + 1) * (TR + 1) + (size_t)G * padded_len(NPHI)) * sizeof(float2);
  auto k = k_row_irdft<NPHI, TR, G>;
  cudaError_t e = prep(k, smem);
  if (e) return e;
  k<<<dim3(d.nrho_pad / TR, batch), G * FftPlan<NPHI, true>::T, smem, s>>>(Yh, lp, d.nrho, d.nrho_pad, t.tw_phi);
  return cudaGetLastError();
}
}  // namespace

// Tile shapes per size: (columns or rows per CTA, concurrent FFTs per CTA).
namespace {
template <int M>
cudaError_t ramp_tma_impl(const Dims& d, const DevTables& t, const float* g, float* out, int batch, cudaStream_t s);
}  // namespace

cudaError_t launch_ramp(const Dims& d, const DevTables& t, const float* g, float* out, int batch, cudaStream_t s) {
  if (d.M == 4096) {
    const cudaError_t e = ramp_tma_impl<4096>(d, t, g, out, batch, s);
    if (e != cudaErrorNotSupported) return e;  // nt % 256 != 0 takes the tile kernel below
  }
  switch (d.M) {
    case 512: return ramp_impl<512, 16, 4>(d, t, g, out, batch, s);
    case 1024: return ramp_impl<1024, 16, 2>(d, t, g, out, batch, s);
    case 2048: return ramp_impl<2048, 8, 1>(d, t, g, out, batch, s);
    case 4096: return ramp_impl<4096, 8, 1>(d, t, g, out, batch, s);
    case 8192: return ramp_impl<8192, 8, 1>(d, t, g, out, batch, s);  // nt in (2048, 4096] (one CTA per column pair: 79.9 vs 66.5 us/slice at 3200 x 2048)
    default: return cudaErrorNotSupported;
  }
}
cudaError_t launch_row_rdft(const Dims& d, const DevTables& t, const float* g, float2* Gh, int batch, cudaStream_t s) {
  switch (d.nphi) {
    case 512: return rdft_impl<512>(d, t, g, Gh, batch, s);
    case 1024: return rdft_impl<1024>(d, t, g, Gh, batch, s);
    case 2048: return rdft_impl<2048>(d, t, g, Gh, batch, s);
    case 4096: return rdft_impl<4096>(d, t, g, Gh, batch, s);
    default: return cudaErrorNotSupported;
  }
}
namespace {
bool mixed_enabled();
cudaError_t rdft_mixed_p(const Dims& d, const DevTables& t, const float* g, float2* Ph, int batch, cudaStream_t s);
}  // namespace
bool mixed_p_available(int nphi, int ns, int nrho, int L) {
  return mixed_enabled() && mixed_radix_length(nphi) && !(ns & 1) && 2 * nrho <= L;
}
cudaError_t launch_row_rdft_p(const Dims& d, const DevTables& t, const float* g, float2* Ph, int batch, cudaStream_t s) {
  if (d.generic) return d.pmix == 2 ? rdft_mixed_p(d, t, g, Ph, batch, s) : cudaErrorNotSupported;
  switch (d.nphi) {
    case 512: return rdft_p_impl<512>(d, t, g, Ph, batch, s);
    case 1024: return rdft_p_impl<1024>(d, t, g, Ph, batch, s);
    case 2048: return rdft_p_impl<2048>(d, t, g, Ph, batch, s);
    case 4096: return rdft_p_impl<4096>(d, t, g, Ph, batch, s);
    default: return cudaErrorNotSupported;
  }
}
cudaError_t launch_rho_conv(const Dims& d, const DevTables& t, const float2* Gh, float2* Yh, int batch, int row_lo,
                            cudaStream_t s, bool pin, bool fused_rows) {
  const int32_t* row_need = fused_rows ? (d.ycompact ? t.rowmap_cp : t.rowmap_id) : nullptr;
  switch (d.L) {
    case 512: return conv_impl<512>(d, t, Gh, Yh, batch, row_lo, s, pin, row_need);
    case 1024: return conv_impl<1024>(d, t, Gh, Yh, batch, row_lo, s, pin, row_need);
    case 2048: return conv_impl<2048>(d, t, Gh, Yh, batch, row_lo, s, pin, row_need);
    case 4096: return conv_impl<4096>(d, t, Gh, Yh, batch, row_lo, s, pin, row_need);
    case 8192: return conv_impl<8192>(d, t, Gh, Yh, batch, row_lo, s, pin, row_need);
    case 16384: return conv_impl<16384>(d, t, Gh, Yh, batch, row_lo, s, pin, row_need);
    default: return cudaErrorNotSupported;
  }
}
cudaError_t launch_row_irdft(const Dims& d, const DevTables& t, const float2* Yh, float* lp, int batch, cudaStream_t s) {
  switch (d.nphi) {
    case 512: return irdft_impl<512, 16, 4>(d, t, Yh, lp, batch, s);
    case 1024: return irdft_impl<1024, 16, 2>(d, t, Yh, lp, batch, s);
    case 2048: return irdft_impl<2048, 8, 2>(d, t, Yh, lp, batch, s);
    case 4096: return irdft_impl<4096, 8, 2>(d, t, Yh, lp, batch, s);
    default: return cudaErrorNotSupported;
  }
}
cudaError_t launch_readout(const Dims& d, const DevTables& t, const float* lp, float* img, int batch, cudaStream_t s) {
  const int npix = d.n * d.n;
  k_readout<<<dim3((npix + 1023) / 1024, batch), 256, 0, s>>>(lp, img, d.n, d.nq, d.nrho, d.nphi, t.qidx, t.qw,
                                                            d.out_scale);
  return cudaGetLastError();
}
namespace {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// Spectra Y[b][m][rho] (complex, rho pitch nrho_pad) as floats {2*nrho_pad, nh, batch};
// box {2*rows floats, box_m m, 1}.
cudaError_t encode_spectra_map(CUtensorMap* map, const float2* Y, int nrho_pad, int nh, int batch, int rows,
                               int box_m) {
  auto enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * nrho_pad), (cuuint64_t)nh, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)nrho_pad * 8, (cuuint64_t)nrho_pad * 8 * nh};
  const cuuint32_t box[3] = {(cuuint32_t)(2 * rows), (cuuint32_t)box_m, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(Y), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Row spectra G[b][m][t] (complex, t pitch nt) as a 2-D tensor {2 nt floats, batch * nh rows}; box {8 floats
// (4 complex t), box_m rows}, 32-byte swizzle (K2's staging layout).
cudaError_t encode_rowspec_map(CUtensorMap* map, const float2* G, int nt, int nh, int batch, int box_m) {
  auto enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {(cuuint64_t)(2 * nt), (cuuint64_t)nh * batch};
  const cuuint64_t strides[1] = {(cuuint64_t)nt * 8};
  const cuuint32_t box[2] = {8, (cuuint32_t)box_m};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float2*>(G), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Sinogram batch as a 2-D tensor {ntheta, batch * nt} of fp32, box {8, 256}, 32-byte swizzle.
cudaError_t encode_sino_map(CUtensorMap* map, const float* g, int nt, int ntheta, int batch) {
  auto enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {(cuuint64_t)ntheta, (cuuint64_t)nt * batch};
  const cuuint64_t strides[1] = {(cuuint64_t)ntheta * 4};
  const cuuint32_t box[2] = {8, 256};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(g), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int M>
cudaError_t ramp_tma_impl(const Dims& d, const DevTables& t, const float* g, float* out, int batch, cudaStream_t s) {
  using RS = RampTmaShape<M>;
  if (d.ntheta % RS::TC || d.nt % RS::BOXR || (reinterpret_cast<uintptr_t>(g) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15) || (d.ntheta * 4) % 16)
    return cudaErrorNotSupported;
  CUtensorMap gm, om;
  cudaError_t e = encode_sino_map(&gm, g, d.nt, d.ntheta, batch);
  if (!e) e = encode_sino_map(&om, out, d.nt, d.ntheta, batch);
  if (e) return e;
  const size_t smem = RS::smem(d.nt);
  auto k = k_ramp_tma<M>;
  e = prep(k, smem);
  if (e) return e;
  const int per = d.ntheta / RS::TC, tiles = per * batch;
  const int grid = tiles < d.nsm ? tiles : d.nsm;
  k<<<grid, RS::G * RS::T, smem, s>>>(gm, om, d.nt, per, tiles, t.ramp, t.tw_ramp);
  return cudaGetLastError();
}
}  // namespace

namespace {
template <int M>
cudaError_t ramp_generic_impl(const Dims& d, const DevTables& t, const float* g, float* out, int batch, cudaStream_t s) {
  const size_t smem = (size_t)padded_len(M) * sizeof(float2);
  auto k = k_ramp_generic<M>;
  cudaError_t e = prep(k, smem);
  if (e) return e;
  k<<<dim3((d.ntheta + 1) / 2, batch), FftPlan<M, false>::T, smem, s>>>(g, out, d.nt, d.ntheta, t.ramp, t.tw_ramp);
  return cudaGetLastError();
}
template <int MB>
cudaError_t rdft_generic_impl(const Dims& d, const DevTables& t, const float* g, float2* Gh, int batch,
                              cudaStream_t s) {
  const size_t smem = ((size_t)padded_len(MB) + d.nphi) * sizeof(float2);
  auto k = k_row_rdft_generic<MB>;
  cudaError_t e = prep(k, smem);
  if (e) return e;
  const int win = d.win > 0 ? d.win : d.ntheta, win_lo = d.win > 0 ? d.win_lo : d.ntheta;
  k<<<dim3((d.nt + 1) / 2, batch), FftPlan<MB, false>::T, smem, s>>>(g, Gh, d.nt, d.gp > 0 ? d.gp : d.nt, d.ntheta,
                                                                    win, win_lo, t.chirp,
                                                                    t.bhat_f, t.tw_blue);
  return cudaGetLastError();
}
template <int MB>
cudaError_t irdft_generic_impl(const Dims& d, const DevTables& t, const float2* Yh, float* lp, int batch,
                               cudaStream_t s) {
  const size_t smem = (size_t)padded_len(MB) * sizeof(float2);
  auto k = k_row_irdft_generic<MB>;
  cudaError_t e = prep(k, smem);
  if (e) return e;
  const int grid = d.npairs > 0 ? d.npairs : (d.nrho + 1) / 2;
  k<<<dim3(grid, batch), FftPlan<MB, false>::T, smem, s>>>(Yh, lp, d.nrho, d.nrho_pad, d.ntheta, t.chirp, t.bhat_i,
                                                          t.tw_blue, d.npairs > 0 ? t.pairs : nullptr);
  return cudaGetLastError();
}
}  // namespace

#define LPBP_POW2_SWITCH(N, CALL)                 \
  switch (N) {                                    \
    case 512: return CALL(512);                   \
    case 1024: return CALL(1024);                 \
    case 2048: return CALL(2048);                 \
    case 4096: return CALL(4096);                 \
    case 8192: return CALL(8192);                 \
    case 16384: return CALL(16384);               \
    default: return cudaErrorNotSupported;        \
  }

cudaError_t launch_ramp_generic(const Dims& d, const DevTables& t, const float* g, float* out, int batch,
                                cudaStream_t s) {
#define LPBP_CALL(M) ramp_generic_impl<M>(d, t, g, out, batch, s)
  LPBP_POW2_SWITCH(d.M, LPBP_CALL)
#undef LPBP_CALL
}
namespace {
// (Q, P) instantiations of the mixed-radix row DFTs: Q P = nphi, Q P / 16 threads (whole warps, <= 1024)
#define LPBP_MIXED_SWITCH(NPHI, CALL)               \
  switch (NPHI) {                                   \
    case 3 * 512: return CALL(3, 512);              \
    case 3 * 1024: return CALL(3, 1024);            \
    case 3 * 2048: return CALL(3, 2048);            \
    case 3 * 4096: return CALL(3, 4096);            \
    case 5 * 512: return CALL(5, 512);              \
    case 5 * 1024: return CALL(5, 1024);            \
    case 5 * 2048: return CALL(5, 2048);            \
    case 9 * 512: return CALL(9, 512);              \
    case 9 * 1024: return CALL(9, 1024);            \
    case 15 * 512: return CALL(15, 512);            \
    case 15 * 1024: return CALL(15, 1024);          \
    case 25 * 256: return CALL(25, 256);            \
    case 25 * 512: return CALL(25, 512);            \
    default: return cudaErrorNotSupported;          \
  }
template <int Q, int P>
cudaError_t rdft_mixed_impl(const Dims& d, const float* g, float2* Gh, int batch, cudaStream_t s) {
  using MS = MixedShape<Q, P>;
  auto k = k_row_rdft_mixed<Q, P>;
  cudaError_t e = prep(k, MS::SMEM);
  if (e) return e;
  const int win = d.win > 0 ? d.win : d.ntheta, win_lo = d.win > 0 ? d.win_lo : d.ntheta;
  k<<<dim3((d.nt + 1) / 2, batch), MS::THREADS, MS::SMEM, s>>>(g, Gh, d.nt, d.gp > 0 ? d.gp : d.nt, d.ntheta, win,
                                                              win_lo);
  return cudaGetLastError();
}
template <int Q, int P>
cudaError_t rdft_mixed_p_impl(const Dims& d, const DevTables& t, const float* g, float2* Ph, int batch, cudaStream_t s) {
  using MS = MixedShape<Q, P>;
  if ((d.ns & 1) || (reinterpret_cast<uintptr_t>(Ph) & 15)) return cudaErrorNotSupported;
  auto k = k_row_rdft_mixed_p<Q, P>;
  cudaError_t e = prep(k, MS::SMEM);
  if (e) return e;
  k<<<dim3(d.ns / 2, batch), MS::THREADS, MS::SMEM, s>>>(g, Ph, d.nt, d.ns, d.ntheta, t.ab, t.wab);
  return cudaGetLastError();
}
template <int Q, int P>
cudaError_t irdft_mixed_impl(const Dims& d, const DevTables& t, const float2* Yh, float* lp, int batch, cudaStream_t s) {
  using MS = MixedShape<Q, P>;
  auto k = k_row_irdft_mixed<Q, P>;
  const int nh = d.ntheta + 1, nbox = (nh + 255) / 256;
  if (reinterpret_cast<uintptr_t>(Yh) & 15) return cudaErrorNotSupported;
  CUtensorMap ym;
  cudaError_t e = encode_spectra_map(&ym, Yh, d.nrho_pad, nh, batch, 2, 256);
  if (e) return e;
  const size_t smem = (size_t)nbox * 256 * 16 + MS::SMEM;
  e = prep(k, smem);
  if (e) return e;
  const int grid = d.npairs > 0 ? d.npairs : (d.nrho + 1) / 2;
  k<<<dim3(grid, batch), MS::THREADS, smem, s>>>(ym, lp, d.nrho, d.ntheta, nbox, d.npairs > 0 ? t.pairs : nullptr);
  return cudaGetLastError();
}
cudaError_t rdft_mixed(const Dims& d, const float* g, float2* Gh, int batch, cudaStream_t s) {
#define LPBP_CALL(Q, P) rdft_mixed_impl<Q, P>(d, g, Gh, batch, s)
  LPBP_MIXED_SWITCH(d.nphi, LPBP_CALL)
#undef LPBP_CALL
}
cudaError_t rdft_mixed_p(const Dims& d, const DevTables& t, const float* g, float2* Ph, int batch, cudaStream_t s) {
#define LPBP_CALL(Q, P) rdft_mixed_p_impl<Q, P>(d, t, g, Ph, batch, s)
  LPBP_MIXED_SWITCH(d.nphi, LPBP_CALL)
#undef LPBP_CALL
}
cudaError_t irdft_mixed(const Dims& d, const DevTables& t, const float2* Yh, float* lp, int batch, cudaStream_t s) {
#define LPBP_CALL(Q, P) irdft_mixed_impl<Q, P>(d, t, Yh, lp, batch, s)
  LPBP_MIXED_SWITCH(d.nphi, LPBP_CALL)
#undef LPBP_CALL
}
// LPBP_MIXED=0 keeps the Bluestein kernels for every generic length (A/B measurements, parity)
bool mixed_enabled() {
  static const bool on = [] {
    const char* v = getenv("LPBP_MIXED");
    return v ? atoi(v) != 0 : true;
  }();
  return on;
}
}  // namespace

bool mixed_radix_length(int nphi) {
  switch (nphi) {
    case 3 * 512: case 3 * 1024: case 3 * 2048: case 3 * 4096: case 5 * 512: case 5 * 1024: case 5 * 2048:
    case 9 * 512: case 9 * 1024: case 15 * 512: case 15 * 1024: case 25 * 256: case 25 * 512:
      return true;
    default:
      return false;
  }
}

cudaError_t launch_row_rdft_generic(const Dims& d, const DevTables& t, const float* g, float2* Gh, int batch,
                                    cudaStream_t s) {
  if (mixed_enabled() && mixed_radix_length(d.nphi)) return rdft_mixed(d, g, Gh, batch, s);
#define LPBP_CALL(M) rdft_generic_impl<M>(d, t, g, Gh, batch, s)
  LPBP_POW2_SWITCH(d.MB, LPBP_CALL)
#undef LPBP_CALL
}
cudaError_t launch_row_irdft_generic(const Dims& d, const DevTables& t, const float2* Yh, float* lp, int batch,
                                     cudaStream_t s) {
  if (mixed_enabled() && mixed_radix_length(d.nphi)) return irdft_mixed(d, t, Yh, lp, batch, s);
#define LPBP_CALL(M) irdft_generic_impl<M>(d, t, Yh, lp, batch, s)
  LPBP_POW2_SWITCH(d.MB, LPBP_CALL)
#undef LPBP_CALL
}

int fused_band_rows(int nphi) {
  switch (nphi) {
    case 512: return FusedShape<512>::S;
    case 1024: return FusedShape<1024>::S;
    case 2048: return FusedShape<2048>::S;
    case 4096: return FusedShape<4096>::S;
    case 25 * 256: case 3 * 512: case 5 * 512: case 9 * 512: case 3 * 1024: case 5 * 1024:
      return 2;  // FusedMixedShape::S
    default: return -1;
  }
}

bool fused_mixed_available(const Dims& d) {
  return d.band_rows == 2 && mixed_enabled() && mixed_radix_length(d.nphi);
}

namespace {
template <int NPHI>
cudaError_t fused_impl(const Dims& d, const DevTables& t, const float2* Yh, float* img, int batch, int* counter,
                       cudaStream_t s) {
  using FS = FusedShape<NPHI>;
  if (d.band_rows != FS::S) return cudaErrorInvalidValue;
  auto k = k_irdft_readout<NPHI>;
  cudaError_t e = prep(k, FS::SMEM);
  if (e) return e;
  CUtensorMap map, tail;
  e = encode_spectra_map(&map, Yh, d.nrho_pad, NPHI / 2 + 1, batch, 2, 256);
  if (e) return e;
  e = encode_spectra_map(&tail, Yh, d.nrho_pad, NPHI / 2 + 1, batch, 2, 1);
  if (e) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(int), s);
  if (e) return e;
  const int units = d.nunits * batch;
  int occ = 1;
  constexpr int NTHR = FS::G * FftPlan<NPHI, true>::T + 32;  // FFT groups + the producer warp
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NTHR, FS::SMEM);
  const int slots = d.nsm * (occ > 0 ? occ : 1);
  const int grid = units < slots ? units : slots;
  k<<<grid, NTHR, FS::SMEM, s>>>(map, tail, img, d.nrho, d.n, d.nq, d.row_min, d.nbands, batch,
                                                          counter, t.band_off, d.ycompact ? t.band_row_cp : t.band_row_id,
                                                          reinterpret_cast<const uint2*>(t.units), d.nunits,
                                                          reinterpret_cast<const uint4*>(t.band_entries),
                                                          d.out_scale, t.tw_phi);
  return cudaGetLastError();
}
}  // namespace

namespace {
template <int Q, int P>
cudaError_t fused_mixed_impl(const Dims& d, const DevTables& t, const float2* Yh, float* img, int batch, int* counter,
                             cudaStream_t s) {
  using FS = FusedMixedShape<Q, P>;
  if (d.band_rows != FS::S || (reinterpret_cast<uintptr_t>(Yh) & 15)) return cudaErrorInvalidValue;
  auto k = k_irdft_readout_mixed<Q, P>;
  cudaError_t e = prep(k, FS::SMEM);
  if (e) return e;
  CUtensorMap map;
  e = encode_spectra_map(&map, Yh, d.nrho_pad, FS::NH, batch, 2, 256);
  if (e) return e;
  e = cudaMemsetAsync(counter, 0, sizeof(int), s);
  if (e) return e;
  const int units = d.nunits * batch;
  const int grid = units < d.nsm ? units : d.nsm;
  k<<<grid, FS::NTHR, FS::SMEM, s>>>(map, img, d.nrho, d.n, d.nq, d.row_min, batch, counter, t.band_off,
                                     d.ycompact ? t.band_row_cp : t.band_row_id, reinterpret_cast<const uint2*>(t.units), d.nunits,
                                     reinterpret_cast<const uint4*>(t.band_entries), d.out_scale);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_irdft_readout(const Dims& d, const DevTables& t, const float2* Yh, float* img, int batch,
                                 int* counter, cudaStream_t s) {
  if (fused_mixed_available(d)) {
    switch (d.nphi) {
      case 25 * 256: return fused_mixed_impl<25, 256>(d, t, Yh, img, batch, counter, s);
      case 3 * 512: return fused_mixed_impl<3, 512>(d, t, Yh, img, batch, counter, s);
      case 5 * 512: return fused_mixed_impl<5, 512>(d, t, Yh, img, batch, counter, s);
      case 9 * 512: return fused_mixed_impl<9, 512>(d, t, Yh, img, batch, counter, s);
      case 3 * 1024: return fused_mixed_impl<3, 1024>(d, t, Yh, img, batch, counter, s);
      case 5 * 1024: return fused_mixed_impl<5, 1024>(d, t, Yh, img, batch, counter, s);
      default: return cudaErrorNotSupported;
    }
  }
  switch (d.nphi) {
    case 512: return fused_impl<512>(d, t, Yh, img, batch, counter, s);
    case 1024: return fused_impl<1024>(d, t, Yh, img, batch, counter, s);
    case 2048: return fused_impl<2048>(d, t, Yh, img, batch, counter, s);
    case 4096: return fused_impl<4096>(d, t, Yh, img, batch, counter, s);
    default: return cudaErrorNotSupported;
  }
}

int twiddle_table_len(int N) {
  switch (N) {
    case 128: return TwTable<128>::len;
    case 256: return TwTable<256>::len;
    case 512: return TwTable<512>::len;
    case 1024: return TwTable<1024>::len;
    case 2048: return TwTable<2048>::len;
    case 4096: return TwTable<4096>::len;
    case 8192: return TwTable<8192>::len;
    case 16384: return TwTable<16384>::len;
    default: return -1;
  }
}

cudaError_t launch_init_twiddles(int N, float2* out, cudaStream_t s) {
  const int len = twiddle_table_len(N);
  if (len < 0) return cudaErrorNotSupported;
  const dim3 grid((len + 255) / 256);
  switch (N) {
    case 128: k_init_twiddles<128><<<grid, 256, 0, s>>>(out); break;
    case 256: k_init_twiddles<256><<<grid, 256, 0, s>>>(out); break;
    case 512: k_init_twiddles<512><<<grid, 256, 0, s>>>(out); break;
    case 1024: k_init_twiddles<1024><<<grid, 256, 0, s>>>(out); break;
    case 2048: k_init_twiddles<2048><<<grid, 256, 0, s>>>(out); break;
    case 4096: k_init_twiddles<4096><<<grid, 256, 0, s>>>(out); break;
    case 8192: k_init_twiddles<8192><<<grid, 256, 0, s>>>(out); break;
    case 16384: k_init_twiddles<16384><<<grid, 256, 0, s>>>(out); break;
  }
  return cudaGetLastError();
}

bool sizes_supported(int nt, int ntheta, int L, int M, int MB, bool filter, bool generic) {
  auto pow2in = [](int v, int lo, int hi) { return v >= lo && v <= hi && (v & (v - 1)) == 0; };
  // rho FFT up to 16384 points (nt up to ~5800 at n = nt), ramp embedding up to 8192 (nt <= 4096)
  if (!pow2in(L, 512, 16384)) return false;
  if (filter && !pow2in(M, 512, 8192)) return false;
  // odd nt: row spectra column pitch padded to even; mixed-radix lengths need no Bluestein size
  if (generic) return (pow2in(MB, 512, 16384) || mixed_radix_length(2 * ntheta)) && nt >= 2;
  const int nphi = 2 * ntheta;
  if (!pow2in(nphi, 512, 4096) || nt % 4) return false;
  if (filter && ntheta % 8) return false;
  return true;
}

}  // namespace lpbp
