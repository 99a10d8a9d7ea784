// Device kernels of the BST engine: the reference's frequency-domain
// backprojection (fastbp.bst, bst.py:120-206), fbp's default engine.
//
//   KB1 radial   g -> P[ray][m]   semi-polar unfolding with the Kaiser window,
//                                 length-L real DFTs along s (the +s and -s
//                                 half-rays of one angle packed as re/im of one
//                                 complex FFT), ds / (1/sigma) kernel; also the
//                                 <g, chord> sum for the exact mean (bst.py:173-180)
//   KB2 grid_x   P -> X[x][ky]    bilinear (sigma, theta) gridding onto the padded
//                                 lattice with Hermitian averaging, Nyquist row /
//                                 column zeroed, phase ramps, inverse DFT along x
//                                 keeping the crop; rows ky < big/2 only (the
//                                 spectrum is Hermitian) (grids.py:456-508, bst.py:146-170)
//   KB3 grid_y   X -> img         inverse DFT along y as a real transform (two
//                                 columns packed as re/im), crop, scale and the
//                                 mean offset (subtract_mean mode)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "async.cuh"
#include "bst_kernels.cuh"
#include "fft.cuh"

namespace lpbp {
namespace {

// Barrier of one FFT group of T threads: a named barrier for whole warps, a
// masked __syncwarp when several groups share a warp (bar.sync counts must be
// multiples of 32).
template <int T>
struct GroupBarT {
  int id;
  __device__ __forceinline__ void operator()() const {
    if constexpr (T >= 32) {
      asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(T) : "memory");
    } else {
      const unsigned lane0 = (threadIdx.x & 31u) & ~(unsigned)(T - 1);
      __syncwarp(((1u << T) - 1u) << lane0);
    }
  }
};

// Length-`len` DFT through either the power-of-two FFT (GEN = false, N = len) or
// Bluestein's identity on an N-point circular convolution (GEN = true, N = pow2 >=
// 2 len): forward X[m] = c[m] sum_n x[n] c[n] conj c[m-n], inverse with conjugates,
// c[n] = exp(-i pi n^2 / len) (the generic path of the log-polar engine, kernels.cu).
struct Chirp {
  const float2* c;     // [len]
  const float2* bhat;  // [N] FFT_N of the chirp filter / N
  int len;
};
template <int N, bool INV, bool GEN, bool IN_HALF, bool LAST_SYNC, typename Load, typename Store, typename Sync>
__device__ __forceinline__ void dft(float2* buf, int ti, const float2* tw, const Chirp& ch, Load&& load, Store&& store,
                                    Sync&& sync) {
  if constexpr (!GEN) {
    block_fft<N, INV, LAST_SYNC, false, IN_HALF, 16>(buf, ti, tw, load, store, sync);
  } else {
    auto ld = [&](int idx) -> float2 {
      if (idx >= ch.len) return make_float2(0.f, 0.f);
      const float2 v = load(idx);
      return INV ? cmulc(v, __ldg(ch.c + idx)) : cmul(v, __ldg(ch.c + idx));
    };
    auto mul = [&](int idx, float2 v) -> float2 { return cmul(v, __ldg(ch.bhat + idx)); };
    auto st = [&](int idx, float2 v) {
      if (idx < ch.len) store(idx, INV ? cmulc(v, __ldg(ch.c + idx)) : cmul(v, __ldg(ch.c + idx)));
    };
    block_conv<N, true, 16>(buf, ti, tw, ld, mul, st, sync);  // len <= N/2: half-zero in, low half out
  }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < nw; ++i) s += red[i];
  return s;  // valid in thread 0
}

// ---------------------------------------------------------------------------
// KB1: TC sinogram columns per CTA staged in smem (coalesced float4 loads), G
// FFT groups; column c gives half-rays c (t = +s) and c + ntheta (t = -s).
// ---------------------------------------------------------------------------
// GEN: L is the Bluestein convolution size MB and the DFT length is ch.len; the
// spectrum then goes to a separate zbuf (block_conv has no trailing barrier).
template <int L, int TC, int G, bool IN_HALF, bool GEN>
__global__ void __launch_bounds__(G * FftPlan<L, false>::T, 2)
k_bst_radial(const float* __restrict__ g, float2* __restrict__ P, int nt, int ntheta, int ns, int m_need, int m_pad,
             const int2* __restrict__ tap_base, const float4* __restrict__ tap_w, const float* __restrict__ kern,
             const float2* __restrict__ tw, double* __restrict__ acc, const float4* __restrict__ chord, Chirp ch) {
  constexpr int T = FftPlan<L, false>::T;
  constexpr int TP = TC + 1;
  constexpr int V = TC / 4;
  extern __shared__ __align__(16) float2 smem_b1[];
  float* tile = reinterpret_cast<float*>(smem_b1);  // nt * TP
  float2* bufs = smem_b1 + ((nt * TP + 3) / 4) * 2;
  __shared__ double red[32];
  const int gi = threadIdx.x / T, ti = threadIdx.x % T;
  float2* buf = bufs + gi * padded_len(L);
  float2* zbuf = GEN ? bufs + G * padded_len(L) + gi * padded_len(L / 2) : buf;
  const int Lr = GEN ? ch.len : L;  // DFT length
  const int c0 = blockIdx.x * TC;
  const int nc = min(TC, ntheta - c0);  // ragged last tile
  const int b = blockIdx.y;
  const float* src = g + (size_t)b * nt * ntheta + c0;
  // <g, chord> dt dtheta / 4 (bst.py:173-180) accumulated while the tile streams in: fp32
  // per-thread partials (<= nt TC / blockDim terms), fp64 across the CTA and the batch
  const float dt = 2.f / nt;
  auto chord_w = [&](const float4& cp, float a) {
    return a <= cp.x ? cp.z : (a < cp.y ? cp.z * (cp.y - a) * cp.w : 0.f);
  };
  float part = 0.f;
  if (nc == TC && (ntheta & 3) == 0) {
    static_assert((G * T) % V == 0, "a thread's column quad is fixed");
    const int cq = (threadIdx.x % V) * 4;
    float4 cp[4];
    if (chord) {
#pragma unroll
      for (int k = 0; k < 4; ++k) cp[k] = __ldg(chord + c0 + cq + k);
    }
    for (int e = threadIdx.x; e < nt * V; e += blockDim.x) {
      const int t = e / V;
      const float4 v = __ldg(reinterpret_cast<const float4*>(src + (size_t)t * ntheta + cq));
      float* r = tile + t * TP + cq;
      r[0] = v.x;
      r[1] = v.y;
      r[2] = v.z;
      r[3] = v.w;
      if (chord) {
        const float a = fabsf(-1.f + t * dt);
        part = fmaf(v.x, chord_w(cp[0], a), part);
        part = fmaf(v.y, chord_w(cp[1], a), part);
        part = fmaf(v.z, chord_w(cp[2], a), part);
        part = fmaf(v.w, chord_w(cp[3], a), part);
      }
    }
  } else {
    for (int e = threadIdx.x; e < nt * TC; e += blockDim.x) {
      const int t = e / TC, c = e % TC;
      const float v = c < nc ? __ldg(src + (size_t)t * ntheta + c) : 0.f;
      tile[t * TP + c] = v;
      if (chord && c < nc) part = fmaf(v, chord_w(__ldg(chord + c0 + c), fabsf(-1.f + t * dt)), part);
    }
  }
  if (chord) {
    const double s = block_sum((double)part, red);  // its barriers also publish the tile
    if (threadIdx.x == 0) atomicAdd(acc + 2 * b, s);
  } else {
    __syncthreads();
  }
  for (int round = 0; round < TC / G; ++round) {
    const int c = round * G + gi;
    if (round * G >= nc) break;  // uniform across the CTA
    auto load = [&](int k) -> float2 {  // (+s half-ray, -s half-ray) samples, window folded
      if (!IN_HALF && k >= ns) return make_float2(0.f, 0.f);
      const int2 bb = __ldg(tap_base + k);
      const float4 w = __ldg(tap_w + k);
      const float a = w.x * tile[bb.x * TP + c] + w.y * tile[(bb.x + 1) * TP + c];
      const float m = w.z * tile[bb.y * TP + c] + w.w * tile[(bb.y + 1) * TP + c];
      return make_float2(a, m);
    };
    auto store = [&](int idx, float2 v) { zbuf[pad16(idx)] = v; };
    if constexpr (IN_HALF || GEN) {
      auto load_h = [&](int k) -> float2 { return k < ns ? load(k) : make_float2(0.f, 0.f); };
      dft<L, false, GEN, true, true>(buf, ti, tw, ch, load_h, store, GroupBarT<T>{1 + gi});
    } else {
      dft<L, false, GEN, false, true>(buf, ti, tw, ch, load, store, GroupBarT<T>{1 + gi});
    }
    GroupBarT<T>{1 + gi}();
    // separate the packed spectra: A = (Z[m] + conj Z[-m]) / 2, B = (Z[m] - conj Z[-m]) / 2i
    // ray pair (c, c + ntheta) interleaved: P4[c][m] = (ray c, ray c + ntheta), the gridding's
    // (direct, Hermitian mirror) taps of one angle in one 16-byte load
    // Row ntheta repeats row 0 swapped (ray ntheta, ray 0) so the gridding's j0 + 1 never wraps;
    // row ntheta + 1 and the bins [m_need, m_pad) are zero (read with zero weight, unguarded).
    float4* p4s = reinterpret_cast<float4*>(P) + (size_t)b * (ntheta + 2) * m_pad;
    float4* p4 = p4s + (size_t)(c0 + c) * m_pad;
    const bool wrap_row = c0 + c == 0;
    for (int m = ti; m < m_pad && c < nc; m += T) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m < m_need) {
        const float2 z = zbuf[pad16(m)];
        const float2 w = zbuf[pad16(m == 0 ? 0 : Lr - m)];
        const float k = __ldg(kern + m);
        v = make_float4(0.5f * (z.x + w.x) * k, 0.5f * (z.y - w.y) * k, 0.5f * (z.y + w.y) * k,
                        0.5f * (w.x - z.x) * k);
      }
      p4[m] = v;
      if (wrap_row) {
        p4s[(size_t)ntheta * m_pad + m] = make_float4(v.z, v.w, v.x, v.y);
        p4s[(size_t)(ntheta + 1) * m_pad + m] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    GroupBarT<T>{1 + gi}();
  }
}

// ---------------------------------------------------------------------------
// KB2: rows ky of the padded lattice (TR per CTA, G groups), gridded on the fly
// inside the first FFT pass, inverse DFT along x, crop x in [p0, p0 + n),
// written transposed X[x][ky] (TR consecutive ky per run); accumulates the
// crop mean through cmean (sum over the crop rows of the row's DFT weights).
// ---------------------------------------------------------------------------
// GEN: BIG is the Bluestein convolution size and the padded side is ch.len.
// TMA_OUT: X leaves by 2-D TMA stores (boxes {TR complex, 256 x}, 3-D map {2 HB floats, n, batch}) from
// a [n][TR] staging in TMA's 32-byte swizzle (complex (x, r) at x*TR + (r ^ 2*((x >> 2) & 1))).
template <int BIG, int TR, int G, bool GEN, bool TMA_OUT>
__global__ void __launch_bounds__(G * FftPlan<BIG, true>::T)
k_bst_grid_x(const __grid_constant__ CUtensorMap xmap, const float2* __restrict__ P, float2* __restrict__ X, int nray,
             int nsig, int m_pad, int n, int p0, const uint2* __restrict__ gq, int qpitch, const float2* __restrict__ tau,
             const float2* __restrict__ cmean, const float2* __restrict__ tw, double* __restrict__ acc, Chirp ch) {
  constexpr int T = FftPlan<BIG, true>::T;
  static_assert(!TMA_OUT || TR == 4, "32-byte staging rows");
  const int big = GEN ? ch.len : BIG;
  const int HB = big / 2;
  extern __shared__ __align__(16) float2 smem_b2_raw[];
  float2* smem_b2 = smem_b2_raw + ((1024u - (smem_u32(smem_b2_raw) & 1023u)) & 1023u) / sizeof(float2);
  // [n][TR]; with TMA stores the staging spans whole 256-row boxes (the last box's clipped rows
  // stay inside this CTA's allocation)
  const int nst = TMA_OUT ? (n + 255) / 256 * 256 : n;
  float2* stg = smem_b2;
  float2* buf = stg + (size_t)nst * TR + (threadIdx.x / T) * padded_len(BIG);
  __shared__ double red[32];
  const int gi = threadIdx.x / T, ti = threadIdx.x % T;
  const int ky0 = blockIdx.x * TR;
  const int b = blockIdx.y;
  // [nray/2 + 2][m_pad] float4 ray pairs (ray p, ray p + nray/2); row nray/2 = (ray nray/2, ray 0),
  // row nray/2 + 1 and bins >= nsig zero
  const float4* P4 = reinterpret_cast<const float4*>(P) + (size_t)b * (nray / 2 + 2) * m_pad;
  const int half_ray = nray / 2;
  double mean_part = 0.0;
  for (int rr = 0; rr < TR / G; ++rr) {
    const int r = rr * G + gi;
    const int ky = ky0 + r;
    if (ky >= HB) break;  // uniform within the group
    const float2 ty = __ldg(tau + ky);
    const uint2* gqr = gq + (size_t)ky * qpitch;
    // fp64-built coordinates of (|kfx|, ky); kfx < 0 reflects theta -> pi - theta.  The gridded
    // rows ky >= 0 keep theta in [0, pi], so j0 lies in [0, nray/2] (nray/2 only at theta = pi,
    // where wj = 0) and the pair rows j0, j0 + 1 hold the direct taps in .xy, the Hermitian
    // mirror taps (theta + pi) in .zw.
    auto gq_at = [&](int kx) -> uint2 { return __ldg(gqr + (kx > HB ? big - kx : kx)); };
    struct Tap {
      const float4* q0;
      float wi, wj;
    };
    auto decode = [&](int kx, uint2 e) -> Tap {
      const int i0 = (int)(e.x & 0x1FFFu);  // i0 = nsig - 1 only with wi = 0; bin nsig is zero
      int j0 = (int)(e.y & 0x1FFFu);
      uint32_t qj = e.y >> 13;
      if (kx > HB) {  // fj' = nray/2 - fj
        j0 = half_ray - j0 - (qj != 0u);
        qj = qj ? 524288u - qj : 0u;
      }
      return Tap{P4 + (j0 * m_pad + i0), (float)(e.x >> 13) * (1.f / 524288.f), (float)qj * (1.f / 524288.f)};
    };
    // taps a00, a10 at q0, a01, a11 at q0 + m_pad (theta = pi, j0 = nray/2: the zero row, wj = 0)
    auto finish = [&](int kx, const Tap& t, const float4& a00, const float4& a10, const float4& a01,
                      const float4& a11) -> float2 {
      if (kx == HB || ky == HB) return make_float2(0.f, 0.f);  // Nyquist row / column (bst.py:157-160)
      // G(k) + conj(G(-k)) per tap; the 1/2 is folded into the radial kernel
      const float s00x = a00.x + a00.z, s00y = a00.y - a00.w, s10x = a10.x + a10.z, s10y = a10.y - a10.w;
      const float s01x = a01.x + a01.z, s01y = a01.y - a01.w, s11x = a11.x + a11.z, s11y = a11.y - a11.w;
      const float u0x = fmaf(t.wi, s10x - s00x, s00x), u0y = fmaf(t.wi, s10y - s00y, s00y);
      const float u1x = fmaf(t.wi, s11x - s01x, s01x), u1y = fmaf(t.wi, s11y - s01y, s01y);
      float gx = fmaf(t.wj, u1x - u0x, u0x), gy = fmaf(t.wj, u1y - u0y, u0y);
      if (kx == 0 && ky == 0) {  // numpy pairs the origin bin with itself, not with theta + pi
        gx = 2.f * a00.x;
        gy = 0.f;
      }
      const float2 tx = __ldg(tau + kx);  // the row's tau[ky] is applied at the store
      return make_float2(gx * tx.x - gy * tx.y, gx * tx.y + gy * tx.x);
    };
    auto load = [&](int kx) -> float2 {
      const Tap t = decode(kx, gq_at(kx));
      const float4* q1 = t.q0 + m_pad;
      return finish(kx, t, __ldg(t.q0), __ldg(t.q0 + 1), __ldg(q1), __ldg(q1 + 1));
    };
    float2 rowsum = make_float2(0.f, 0.f);
    auto store = [&](int x, float2 v) {
      const int xc = x - p0;
      if (xc >= 0 && xc < n) {
        v = make_float2(v.x * ty.x - v.y * ty.y, v.x * ty.y + v.y * ty.x);
        stg[(size_t)xc * TR + (TMA_OUT ? (r ^ (((xc >> 2) & 1) << 1)) : r)] = v;
        rowsum.x += v.x;
        rowsum.y += v.y;
      }
    };
    if constexpr (!GEN) {
      // Gather phase ahead of the FFT, free of its live data: this thread's points kx = ti + m T
      // (exactly the indices its first FFT pass reads) in batches of 4 (16 float4 taps in
      // flight, the next batch's table entries prefetched), written to buf[kx]; the FFT then
      // reads them back (same thread) and its first-pass barrier orders the in-place stores.
      constexpr int E = BIG / T, B4 = 4;
      static_assert(E % B4 == 0, "batches of 4 points");
      uint2 gcur[B4];
#pragma unroll
      for (int q = 0; q < B4; ++q) gcur[q] = gq_at(ti + q * T);
#pragma unroll
      for (int m0 = 0; m0 < E; m0 += B4) {
        uint2 gnext[B4];
        if (m0 + B4 < E) {
#pragma unroll
          for (int q = 0; q < B4; ++q) gnext[q] = gq_at(ti + (m0 + B4 + q) * T);
        }
        Tap tp[B4];
        float4 a[B4][4];
#pragma unroll
        for (int q = 0; q < B4; ++q) {
          tp[q] = decode(ti + (m0 + q) * T, gcur[q]);
          const float4* q1 = tp[q].q0 + m_pad;
          a[q][0] = __ldg(tp[q].q0);
          a[q][1] = __ldg(tp[q].q0 + 1);
          a[q][2] = __ldg(q1);
          a[q][3] = __ldg(q1 + 1);
        }
#pragma unroll
        for (int q = 0; q < B4; ++q) {
          const int kx = ti + (m0 + q) * T;
          buf[kx] = finish(kx, tp[q], a[q][0], a[q][1], a[q][2], a[q][3]);
        }
        if (m0 + B4 < E) {
#pragma unroll
          for (int q = 0; q < B4; ++q) gcur[q] = gnext[q];
        }
      }
      auto ld = [&](int kx) -> float2 { return buf[kx]; };
      block_fft<BIG, true, false, true, false, 16>(buf, ti, tw, ld, store, GroupBarT<T>{1 + gi});
    } else {
      dft<BIG, true, GEN, false, false>(buf, ti, tw, ch, load, store, GroupBarT<T>{1 + gi});
    }
    GroupBarT<T>{1 + gi}();  // the next row's first pass overwrites buf
    // crop mean: Re(sum_x X[ky][x] * cmean[ky]), rows 1..BIG/2-1 stand for their conjugate partners too
    const float2 cm = __ldg(cmean + ky);
    const double wgt = ky == 0 ? 1.0 : 2.0;
    mean_part += wgt * ((double)rowsum.x * cm.x - (double)rowsum.y * cm.y);
  }
  const double s = block_sum(mean_part, red);
  if (threadIdx.x == 0) atomicAdd(acc + 2 * b + 1, s);
  __syncthreads();
  if constexpr (TMA_OUT) {
    const int nbox = (n + 255) / 256;  // x past n and ky past HB are clipped by the map
    if (threadIdx.x < 32) {
      fence_proxy_async_smem();  // the transforms' generic stores before this lane's TMA reads
      for (int k = threadIdx.x; k < nbox; k += 32) tma_store_3d(&xmap, 2 * ky0, k * 256, b, stg + (size_t)k * 256 * TR);
      bulk_commit_group();
      bulk_wait_group_read<0>();  // the staging must outlive the reads
    }
  } else {
    float2* Xb = X + (size_t)b * n * HB;
    for (int e = threadIdx.x; e < n * TR; e += blockDim.x) {
      const int xc = e / TR, r = e % TR;
      if (ky0 + r < HB) Xb[(size_t)xc * HB + ky0 + r] = stg[e];
    }
  }
}

// ---------------------------------------------------------------------------
// KB3: TC output columns per CTA (TC/2 packed FFTs over G groups); the column
// pair (x1, x2) is Z[ky] = X[ky][x1] + i X[ky][x2] with Hermitian extension,
// so one inverse FFT gives both real columns.  Crop y in [p0, p0 + n).
// ---------------------------------------------------------------------------
// TMA_OUT: the crop leaves by 2-D TMA stores (boxes {8 columns, 256 rows}, 3-D map {n, n, batch});
// the staging then is [n][8] in TMA's 32-byte swizzle (float (y, c) at y*8 + (c ^ 4*((y >> 2) & 1)))
// instead of the [n][TC + 1] pitch the thread write-out uses.
template <int BIG, int TC, int G, bool GEN, bool TMA_OUT>
__global__ void __launch_bounds__(G * FftPlan<BIG, true>::T)
k_bst_grid_y(const __grid_constant__ CUtensorMap omap, const float2* __restrict__ X, float* __restrict__ img, int n,
             int p0, float s_img, float s_mean, float fbp, int subtract_mean, const double* __restrict__ acc,
             const float2* __restrict__ tw, Chirp ch) {
  constexpr int T = FftPlan<BIG, true>::T;
  static_assert(!TMA_OUT || TC == 8, "32-byte staging rows");
  constexpr int SP = TMA_OUT ? TC : TC + 1;  // staging pitch (floats)
  const int big = GEN ? ch.len : BIG;
  const int HB = big / 2;
  extern __shared__ __align__(16) float2 smem_b3_raw[];
  // 1024-byte aligned (TMA swizzle atoms), offset from the shared symbol to stay in the shared window
  float2* smem_b3 = smem_b3_raw + ((1024u - (smem_u32(smem_b3_raw) & 1023u)) & 1023u) / sizeof(float2);
  const int nst = TMA_OUT ? (n + 255) / 256 * 256 : n;  // whole 256-row TMA boxes (see k_bst_grid_x)
  float* stg = reinterpret_cast<float*>(smem_b3);  // [n][SP]
  float2* buf = smem_b3 + ((size_t)nst * SP + 1) / 2 + (threadIdx.x / T) * padded_len(BIG);
  const int gi = threadIdx.x / T, ti = threadIdx.x % T;
  const int x0 = blockIdx.x * TC;
  const int b = blockIdx.y;
  const float2* Xb = X + (size_t)b * n * HB;
  float offset = 0.f;
  if (subtract_mean) {  // mean_backprojection(g) - mean(img) (bst.py:199-202), in BST image units
    const double mean_bp = acc[2 * b], mean_img = (double)s_mean * acc[2 * b + 1];
    offset = (float)((double)fbp * (mean_bp - mean_img));
  }
  for (int rr = 0; rr < TC / 2 / G; ++rr) {
    const int q = rr * G + gi;  // column pair
    const int xa = x0 + 2 * q, xb = xa + 1;
    const bool hb = xb < n;
    const float2* ca = Xb + (size_t)xa * HB;
    const float2* cb = Xb + (size_t)(hb ? xb : xa) * HB;
    auto load = [&](int ky) -> float2 {
      if (ky == HB) return make_float2(0.f, 0.f);
      const bool hi = ky > HB;
      const int k = hi ? big - ky : ky;
      float2 a = __ldg(ca + k), c = hb ? __ldg(cb + k) : make_float2(0.f, 0.f);
      if (hi) {
        a.y = -a.y;
        c.y = -c.y;
      }
      return make_float2(a.x - c.y, a.y + c.x);  // a + i c
    };
    auto store = [&](int y, float2 v) {
      const int yc = y - p0;
      if (yc >= 0 && yc < n) {
        const float2 o = make_float2(v.x * s_img + offset, v.y * s_img + offset);
        if constexpr (TMA_OUT)
          *reinterpret_cast<float2*>(stg + (size_t)yc * SP + ((2 * q) ^ (((yc >> 2) & 1) << 2))) = o;
        else {
          stg[(size_t)yc * SP + 2 * q] = o.x;
          stg[(size_t)yc * SP + 2 * q + 1] = o.y;
        }
      }
    };
    dft<BIG, true, GEN, false, false>(buf, ti, tw, ch, load, store, GroupBarT<T>{1 + gi});
    GroupBarT<T>{1 + gi}();
  }
  __syncthreads();
  if constexpr (TMA_OUT) {
    const int nbox = (n + 255) / 256;  // rows past n and columns past n are clipped by the map
    if (threadIdx.x < 32) {
      fence_proxy_async_smem();  // the transforms' generic stores before this lane's TMA reads
      for (int k = threadIdx.x; k < nbox; k += 32) tma_store_3d(&omap, x0, k * 256, b, stg + (size_t)k * 256 * SP);
      bulk_commit_group();
      bulk_wait_group_read<0>();  // the staging must outlive the reads
    }
  } else {
    float* ob = img + (size_t)b * n * n;
    const int w = min(TC, n - x0);
    for (int e = threadIdx.x; e < n * TC; e += blockDim.x) {
      const int y = e / TC, c = e % TC;
      if (c < w) ob[(size_t)y * n + x0 + c] = stg[(size_t)y * SP + c];
    }
  }
}

// Images [batch][n][n] fp32 as a 3-D tensor {n, n, batch}; box {8, 256, 1}, 32-byte swizzle (grid_y's staging).
PFN_cuTensorMapEncodeTiled_v12000 tensor_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return enc;
}

bool encode_image_map(CUtensorMap* map, const float* img, int n, int batch) {
  auto enc = tensor_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)n * 4, (cuuint64_t)n * n * 4};
  const cuuint32_t box[3] = {8, 256, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(img), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// X[b][x][ky] (complex, ky pitch hb) as floats {2 hb, n, batch}; box {8 floats = 4 ky, 256 x, 1}, 32-byte swizzle.
bool encode_spectra_x_map(CUtensorMap* map, const float2* X, int hb, int n, int batch) {
  auto enc = tensor_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * hb), (cuuint64_t)n, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)hb * 8, (cuuint64_t)hb * 8 * n};
  const cuuint32_t box[3] = {8, 256, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float2*>(X), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename K>
cudaError_t prep(K k, size_t smem) {
  if (smem > 48 * 1024) return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaSuccess;
}

// N: FFT size (the DFT length L when GEN = false, the Bluestein convolution size otherwise)
template <int N, bool GEN>
cudaError_t radial_impl(const BstDims& d, const BstTables& t, const float* g, float2* P, double* acc, int batch,
                        cudaStream_t s) {
  constexpr int T = FftPlan<N, false>::T;
  constexpr int G = T >= 256 ? 1 : (256 / T > 4 ? 4 : 256 / T);
  constexpr int TC = G >= 4 ? G : 4;
  const size_t smem = (((size_t)d.nt * (TC + 1) + 3) / 4 * 2 + (size_t)G * padded_len(N) +
                       (GEN ? (size_t)G * padded_len(N / 2) : 0)) * sizeof(float2);
  const Chirp ch{t.chirp_L, t.bhat_L, d.L};
  const float2* tw = GEN ? t.tw_mbL : t.tw_L;
  const bool half = 2 * d.ns <= N;
  cudaError_t e;
  if (half || GEN) {
    auto k = k_bst_radial<N, TC, G, true, GEN>;
    if ((e = prep(k, smem))) return e;
    k<<<dim3((d.ntheta + TC - 1) / TC, batch), G * T, smem, s>>>(g, P, d.nt, d.ntheta, d.ns, d.m_need, d.m_pad,
                                                                  t.tap_base, t.tap_w, t.kern, tw, acc,
                                                                  d.subtract_mean ? t.chord : nullptr, ch);
  } else {
    auto k = k_bst_radial<N, TC, G, false, GEN>;
    if ((e = prep(k, smem))) return e;
    k<<<dim3((d.ntheta + TC - 1) / TC, batch), G * T, smem, s>>>(g, P, d.nt, d.ntheta, d.ns, d.m_need, d.m_pad,
                                                                  t.tap_base, t.tap_w, t.kern, tw, acc,
                                                                  d.subtract_mean ? t.chord : nullptr, ch);
  }
  return cudaGetLastError();
}

template <int N, bool GEN>
cudaError_t grid_impl(const BstDims& d, const BstTables& t, const float2* P, float2* X, float* img, double* acc,
                      int batch, cudaStream_t s, cudaEvent_t mid) {
  constexpr int T = FftPlan<N, true>::T;
  constexpr int G = T >= 256 ? (GEN ? 1 : 2) : 4;
  constexpr int TR = 4;
  static_assert(TR % G == 0 || G > TR, "rows per group");
  constexpr int GX = G > TR ? TR : G;
  const Chirp ch{t.chirp_big, t.bhat_big, d.big};
  const float2* tw = GEN ? t.tw_mbbig : t.tw_big;
  const int hb = d.big / 2;
  {
    CUtensorMap xm{};
    const bool tma = (reinterpret_cast<uintptr_t>(X) & 15) == 0 && (hb % 2) == 0 && encode_spectra_x_map(&xm, X, hb, d.n, batch);
    const size_t nst = tma ? ((size_t)d.n + 255) / 256 * 256 : (size_t)d.n;  // whole TMA store boxes
    const size_t smem = 1024 + (nst * TR + (size_t)GX * padded_len(N)) * sizeof(float2);
    auto k = tma ? k_bst_grid_x<N, TR, GX, GEN, true> : k_bst_grid_x<N, TR, GX, GEN, false>;
    cudaError_t e = prep(k, smem);
    if (e) return e;
    k<<<dim3((hb + TR - 1) / TR, batch), GX * T, smem, s>>>(xm, P, X, d.nray, d.m_need, d.m_pad, d.n, d.p0, t.grid_q,
                                                             hb + 1, t.tau, t.cmean, tw, acc, ch);
    if ((e = cudaGetLastError())) return e;
    if (mid) cudaEventRecord(mid, s);  // profiling: between grid_x and grid_y
  }
  {
    constexpr int TC = 8;
    constexpr int GY = G > TC / 2 ? TC / 2 : G;
    CUtensorMap om{};
    const bool tma = (reinterpret_cast<uintptr_t>(img) & 15) == 0 && (d.n % 4) == 0 && encode_image_map(&om, img, d.n, batch);
    const size_t nst = tma ? ((size_t)d.n + 255) / 256 * 256 : (size_t)d.n;  // whole TMA store boxes
    const size_t smem = 1024 + ((nst * (tma ? TC : TC + 1) + 1) / 2 + (size_t)GY * padded_len(N)) * sizeof(float2);
    auto k = tma ? k_bst_grid_y<N, TC, GY, GEN, true> : k_bst_grid_y<N, TC, GY, GEN, false>;
    cudaError_t e = prep(k, smem);
    if (e) return e;
    k<<<dim3((d.n + TC - 1) / TC, batch), GY * T, smem, s>>>(om, X, img, d.n, d.p0, d.s_img, d.s_mean, d.fbp,
                                                            d.subtract_mean, acc, tw, ch);
    return cudaGetLastError();
  }
}

}  // namespace

cudaError_t launch_bst_radial(const BstDims& d, const BstTables& t, const float* g, float2* P, double* acc, int batch,
                              cudaStream_t s) {
  if (d.mb_L > 0) {  // Bluestein (non-power-of-two L)
    switch (d.mb_L) {
      case 512: return radial_impl<512, true>(d, t, g, P, acc, batch, s);
      case 1024: return radial_impl<1024, true>(d, t, g, P, acc, batch, s);
      case 2048: return radial_impl<2048, true>(d, t, g, P, acc, batch, s);
      case 4096: return radial_impl<4096, true>(d, t, g, P, acc, batch, s);
      case 8192: return radial_impl<8192, true>(d, t, g, P, acc, batch, s);
      default: return cudaErrorNotSupported;
    }
  }
  switch (d.L) {
    case 512: return radial_impl<512, false>(d, t, g, P, acc, batch, s);
    case 1024: return radial_impl<1024, false>(d, t, g, P, acc, batch, s);
    case 2048: return radial_impl<2048, false>(d, t, g, P, acc, batch, s);
    case 4096: return radial_impl<4096, false>(d, t, g, P, acc, batch, s);
    case 8192: return radial_impl<8192, false>(d, t, g, P, acc, batch, s);
    default: return cudaErrorNotSupported;
  }
}

cudaError_t launch_bst_grid(const BstDims& d, const BstTables& t, const float2* P, float2* X, float* img, double* acc,
                            int batch, cudaStream_t s, cudaEvent_t mid) {
  if (d.mb_big > 0) {  // Bluestein (padded side not a power of two)
    switch (d.mb_big) {
      case 256: return grid_impl<256, true>(d, t, P, X, img, acc, batch, s, mid);
      case 512: return grid_impl<512, true>(d, t, P, X, img, acc, batch, s, mid);
      case 1024: return grid_impl<1024, true>(d, t, P, X, img, acc, batch, s, mid);
      case 2048: return grid_impl<2048, true>(d, t, P, X, img, acc, batch, s, mid);
      case 4096: return grid_impl<4096, true>(d, t, P, X, img, acc, batch, s, mid);
      case 8192: return grid_impl<8192, true>(d, t, P, X, img, acc, batch, s, mid);
      default: return cudaErrorNotSupported;
    }
  }
  switch (d.big) {
    case 128: return grid_impl<128, false>(d, t, P, X, img, acc, batch, s, mid);
    case 256: return grid_impl<256, false>(d, t, P, X, img, acc, batch, s, mid);
    case 512: return grid_impl<512, false>(d, t, P, X, img, acc, batch, s, mid);
    case 1024: return grid_impl<1024, false>(d, t, P, X, img, acc, batch, s, mid);
    case 2048: return grid_impl<2048, false>(d, t, P, X, img, acc, batch, s, mid);
    case 4096: return grid_impl<4096, false>(d, t, P, X, img, acc, batch, s, mid);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace lpbp
