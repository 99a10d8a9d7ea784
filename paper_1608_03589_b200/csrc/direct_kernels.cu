// Direct pixel-driven backprojector (fastbp reference.py:21-37, the config-4
// accuracy cross-check):
//   b(x) = dtheta * sum_k lerp_t(g[:, k], (x . xi_k + 1) / dt),  zero outside the t range
// (_lerp_profile, grids.py:272-282).  O(n^2 ntheta) lerps per slice.
//
// B200 layout and schedule:
//  * k_direct_pack: the batch is regrouped by 4 slices into angle-major rows of
//    float4 (one entry = the same (t, theta) sample of the group's 4 slices), with
//    PAD zero entries on each side of every row (so every tap of a pixel of
//    [-1, 1]^2 is addressable) and zero slices past the batch.  The angle table
//    (cos, sin) * nt / (2n) is built in fp64 on the device in the same launch.
//  * k_direct: one CTA per (32 x 32 pixel tile, slice group).  For every angle the
//    tile's taps fall in a window of W consecutive entries of that angle's row;
//    stages of A angles arrive by one TMA bulk copy per angle (W * 16 bytes) into a
//    double-buffered shared-memory ring, completing on a per-stage mbarrier.  A
//    thread owns 4 pixels x 4 slices: the coordinate math (one FFMA, a magic-number
//    floor, the weights) is shared by the 4 slices, every tap is one 16-byte shared
//    load, and each lerp is (1 - w) v0 + w v1 as in the reference (two FFMAs).
//    A warp's 32 lanes cover an 8 x 4 pixel block per instruction, so one angle's
//    taps of a warp span <= 10 window entries.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "async.cuh"
#include "direct_kernels.cuh"

namespace lpbp {

namespace {
constexpr int DS = 4;      // slices per group (float4 entries)
constexpr int TILE = 32;   // pixel tile side
constexpr int AMAX = 64;   // angles per stage (upper bound; two per producer lane)
constexpr float MAGIC_HALF = 8388607.5f;  // 2^23 - 0.5: x + MAGIC_HALF rounds x - 0.5 to an integer (x >= 0.5)
constexpr float MAGIC = 8388608.0f;       // 2^23
constexpr int MAGIC_BITS = 0x4B000000;    // __float_as_int(2^23)
}  // namespace

int direct_pad(int nt) { return nt / 4 + 8; }  // >= (sqrt 2 - 1) nt / 2 + 2: every tap of a pixel in [-1,1]^2

DirectGeom direct_geom(int nt, int ntheta, int n, int batch) {
  DirectGeom g{};
  g.nt = nt;
  g.ntheta = ntheta;
  g.n = n;
  g.pad = direct_pad(nt);
  g.ntp = nt + 2 * g.pad;
  g.groups = (batch + DS - 1) / DS;
  // a tile's taps at one angle span <= 62 (|C| + |S|) <= 62 sqrt(2) nt / (2n) entries past its lowest
  // floor; the window starts one entry below that floor and needs one more entry for the upper tap.
  int w = (int)ceil(62.0 * 1.41421356237309515 * nt / (2.0 * n)) + 5;
  w = (w + 1) & ~1;
  g.W = w < g.ntp ? w : g.ntp;
  int a = (3072 / g.W) & ~7;  // ~48 KB of window entries per stage
  g.A = a < 8 ? 8 : (a > AMAX ? AMAX : a);
  g.tab_bytes = (((size_t)ntheta * sizeof(float2)) + 255) & ~(size_t)255;
  g.ws_bytes = g.tab_bytes + (size_t)g.groups * ntheta * g.ntp * sizeof(float4);
  g.smem = (size_t)2 * g.A * g.W * sizeof(float4) + (size_t)2 * g.A * sizeof(float4) + 2 * sizeof(uint64_t);
  return g;
}

// P[grp][k][e] = (g[4 grp + 0][e - pad][k], ..., g[4 grp + 3][e - pad][k]), zero outside.
// Block (32, 8): a 32-angle x 32-entry tile of the group's 4 slices.
__global__ void k_direct_pack(const float* __restrict__ g, float4* __restrict__ P, float2* __restrict__ tab, int nt,
                              int ntheta, int ntp, int pad, int batch, double cscale) {
  __shared__ float tile[DS][TILE][TILE + 1];
  const int k0 = blockIdx.x * TILE, e0 = blockIdx.y * TILE, grp = blockIdx.z;
  const int lane = threadIdx.x;
  if (blockIdx.y == 0 && grp == 0 && threadIdx.y == 0 && k0 + lane < ntheta) {
    double s, c;
    sincospi((double)(k0 + lane) / ntheta, &s, &c);  // theta_k = k pi / ntheta (reference.py:30-36)
    tab[k0 + lane] = make_float2((float)(c * cscale), (float)(s * cscale));
  }
#pragma unroll
  for (int q = 0; q < DS; ++q) {
    const int b = grp * DS + q;
    for (int r = threadIdx.y; r < TILE; r += blockDim.y) {
      const int t = e0 + r - pad, k = k0 + lane;
      float v = 0.f;
      if (b < batch && t >= 0 && t < nt && k < ntheta) v = __ldg(g + ((size_t)b * nt + t) * ntheta + k);
      tile[q][r][lane] = v;
    }
  }
  __syncthreads();
  for (int r = threadIdx.y; r < TILE; r += blockDim.y) {
    const int k = k0 + r, e = e0 + lane;
    if (k < ntheta && e < ntp)
      P[((size_t)grp * ntheta + k) * ntp + e] =
          make_float4(tile[0][lane][r], tile[1][lane][r], tile[2][lane][r], tile[3][lane][r]);
  }
}

__global__ void __launch_bounds__(256, 2)
    k_direct(const float4* __restrict__ P, const float2* __restrict__ tab, float* __restrict__ img, int ntheta, int n,
             int ntp, int pad, int W, int A, int batch, float off, float dtheta) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float4* win = reinterpret_cast<float4*>(smem_raw);            // [2][A][W]
  float4* prm = win + 2 * A * W;                                 // [2][A] (C, S, off - lo, -)
  uint64_t* bar = reinterpret_cast<uint64_t*>(prm + 2 * A);      // [2]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tiles_x = (n + TILE - 1) / TILE;
  const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x, grp = blockIdx.y;
  const float4* Pg = P + (size_t)grp * ntheta * ntp;

  // pixel coordinates in units of half a pixel: x_j = a / n with a = 2j + 1 - n
  const int jx = tx * TILE + (warp & 3) * 8 + (lane & 7);
  const int iy0 = ty * TILE + (warp >> 2) * 16 + (lane >> 3);
  const float a = (float)(2 * min(jx, n - 1) + 1 - n);
  float b[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) b[u] = (float)(2 * min(iy0 + 4 * u, n - 1) + 1 - n);
  // the tile's corner coordinates (clamped to the image) bound every tap's position
  const float a_lo = (float)(2 * (tx * TILE) + 1 - n), a_hi = (float)(2 * min(tx * TILE + TILE - 1, n - 1) + 1 - n);
  const float b_lo = (float)(2 * (ty * TILE) + 1 - n), b_hi = (float)(2 * min(ty * TILE + TILE - 1, n - 1) + 1 - n);

  const int nst = (ntheta + A - 1) / A;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // warp 0 stages the A angles of stage st into ring slot st & 1: each lane places the windows of
  // its (at most two) angles and writes their parameters, then lane 0 arms the barrier with the
  // stage's byte count (its arrival releases the parameter stores) and the lanes issue the copies.
  auto issue = [&](int st) {
    const int k0 = st * A, na = min(A, ntheta - k0), slot = st & 1;
    int lo[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int j = lane + 32 * r;
      lo[r] = 0;
      if (j < na) {
        const float2 cs = __ldg(tab + k0 + j);
        const float fmin = off + fminf(a_lo * cs.x, a_hi * cs.x) + fminf(b_lo * cs.y, b_hi * cs.y);
        lo[r] = max(0, min((int)floorf(fmin) - 1, ntp - W));
        prm[slot * A + j] = make_float4(cs.x, cs.y, off - (float)lo[r], 0.f);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(&bar[slot], (uint32_t)(na * W * sizeof(float4)));
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int j = lane + 32 * r;
      if (j < na)
        tma_bulk_g2s(win + (size_t)(slot * A + j) * W, Pg + (size_t)(k0 + j) * ntp + lo[r],
                     (uint32_t)(W * sizeof(float4)), &bar[slot]);
    }
  };
  if (warp == 0) {
    issue(0);
    if (nst > 1) issue(1);
  }

  float acc[4][DS];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int q = 0; q < DS; ++q) acc[u][q] = 0.f;

  for (int st = 0; st < nst; ++st) {
    const int slot = st & 1, na = min(A, ntheta - st * A);
    mbar_wait(&bar[slot], (uint32_t)((st >> 1) & 1));
    const float4* wslot = win + (size_t)slot * A * W;
    const float4* pslot = prm + slot * A;
#pragma unroll 2
    for (int j = 0; j < na; ++j) {
      const float4 p = pslot[j];
      const float base = fmaf(a, p.x, p.z);
      const float4* row = wslot + j * W;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float f = fmaf(b[u], p.y, base);  // >= 1: position in the window
        const float tr = f + MAGIC_HALF;          // 2^23 + floor(f) (f - 0.5 rounded to nearest)
        const float w1 = f - (tr - MAGIC);        // in [0, 1]
        const float w0 = 1.0f - w1;
        const int i0 = __float_as_int(tr) - MAGIC_BITS;
        const float4 v0 = row[i0], v1 = row[i0 + 1];
        acc[u][0] = fmaf(w1, v1.x, fmaf(w0, v0.x, acc[u][0]));
        acc[u][1] = fmaf(w1, v1.y, fmaf(w0, v0.y, acc[u][1]));
        acc[u][2] = fmaf(w1, v1.z, fmaf(w0, v0.z, acc[u][2]));
        acc[u][3] = fmaf(w1, v1.w, fmaf(w0, v0.w, acc[u][3]));
      }
    }
    __syncthreads();  // every warp is done with ring slot `slot`
    if (warp == 0 && st + 2 < nst) issue(st + 2);
  }

  if (jx < n) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int iy = iy0 + 4 * u;
      if (iy >= n) continue;
#pragma unroll
      for (int q = 0; q < DS; ++q) {
        const int bq = grp * DS + q;
        if (bq < batch) img[((size_t)bq * n + iy) * n + jx] = acc[u][q] * dtheta;
      }
    }
  }
}

cudaError_t launch_direct(const DirectGeom& g, const float* sino, void* ws, float* img, int batch, cudaStream_t s) {
  float2* tab = reinterpret_cast<float2*>(ws);
  float4* P = reinterpret_cast<float4*>(static_cast<unsigned char*>(ws) + g.tab_bytes);
  k_direct_pack<<<dim3((g.ntheta + TILE - 1) / TILE, (g.ntp + TILE - 1) / TILE, g.groups), dim3(32, 8), 0, s>>>(
      sino, P, tab, g.nt, g.ntheta, g.ntp, g.pad, batch, (double)g.nt / (2.0 * g.n));
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  e = cudaFuncSetAttribute(k_direct, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
  if (e) return e;
  const int tiles = ((g.n + TILE - 1) / TILE) * ((g.n + TILE - 1) / TILE);
  // f = a C + b S + nt/2 + pad: the tap position in the padded row (t = -1 at entry pad)
  const float off = 0.5f * (float)g.nt + (float)g.pad;
  const float dtheta = (float)(3.14159265358979323846 / g.ntheta);
  k_direct<<<dim3(tiles, g.groups), 256, g.smem, s>>>(P, tab, img, g.ntheta, g.n, g.ntp, g.pad, g.W, g.A, batch, off,
                                                       dtheta);
  return cudaGetLastError();
}

}  // namespace lpbp
