// Mixed-radix DFTs of length N = Q * P (Q odd and small, P a power of two) for sm_100a.
//
// The phi-axis DFTs have length nphi = 2 ntheta, which is a power of two only for
// power-of-two angle counts; the paper's LNLS datasets have 3200 angles (nphi = 6400 =
// 25 * 256).  Bluestein's identity covers any length at the price of a 16384-point
// circular convolution per 6400-point DFT; this header computes such lengths directly
// by one Cooley-Tukey split (Q-point DFTs in registers, then Q power-of-two FFTs on the
// block_fft engine of fft.cuh):
//
//   n = P n1 + n2,  k = k1 + Q k2   (n1, k1 < Q;  n2, k2 < P)
//   X[k1 + Q k2] = sum_n2 W_P^(n2 k2) [ W_N^(n2 k1) sum_n1 x[P n1 + n2] W_Q^(n1 k1) ]
//
// step A: P DFT-Qs (one per thread, strided input), twiddle W_N^(n2 k1) from the SFU
// after an exact integer phase reduction; step B: Q FFTs of length P, one per group of
// P/16 threads, in place in the group's shared buffer.  DFT-Q is a compile-time
// Cooley-Tukey over the prime factors 3 and 5 with constant twiddles (constexpr sin/cos).
#pragma once
#include <cuda_runtime.h>

#include "fft.cuh"

namespace lpbp {

// ---- constexpr trigonometry (double, |x| reduced to [-pi, pi]; < 1e-15 error) ----------
constexpr double kPiD = 3.14159265358979323846264338327950288;
constexpr double cx_reduce(double x) {
  while (x > kPiD) x -= 2 * kPiD;
  while (x < -kPiD) x += 2 * kPiD;
  return x;
}
constexpr double cx_sin(double x) {
  x = cx_reduce(x);
  double term = x, sum = x;
  for (int k = 1; k < 30; ++k) {
    term *= -x * x / ((2.0 * k) * (2.0 * k + 1.0));
    sum += term;
  }
  return sum;
}
constexpr double cx_cos(double x) {
  x = cx_reduce(x);
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 30; ++k) {
    term *= -x * x / ((2.0 * k - 1.0) * (2.0 * k));
    sum += term;
  }
  return sum;
}

// x * W_Q^(J) (W_Q = exp(-+2 pi i / Q), sign by INV), J compile-time
template <int J, int Q, bool INV>
__device__ __forceinline__ float2 twq(float2 x) {
  constexpr int j = ((J % Q) + Q) % Q;
  if constexpr (j == 0) {
    return x;
  } else {
    constexpr double a = 2.0 * kPiD * (double)j / (double)Q;
    constexpr float c = (float)cx_cos(a);
    constexpr float s = INV ? (float)cx_sin(a) : -(float)cx_sin(a);
    return cmul(x, make_float2(c, s));
  }
}

// ---- small odd DFTs in registers (natural order in and out) ----------------------------
template <int Q>
constexpr int smallest_factor() {
  return Q % 3 == 0 ? 3 : Q % 5 == 0 ? 5 : Q % 7 == 0 ? 7 : Q;
}

template <int Q, bool INV>
struct OddDft {
  static_assert(Q == 1 || smallest_factor<Q>() != Q || Q <= 7, "DFT-Q: factors 3, 5, 7 only");
  __device__ __forceinline__ static void run(float2 (&v)[Q]) {
    if constexpr (Q == 1) {
    } else if constexpr (Q == 3) {
      // X0 = a + b + c;  X1,2 = a - (b + c)/2 -+ i sqrt(3)/2 (b - c)  (forward sign)
      constexpr float h = 0.86602540378443864676f;
      const float2 t = cadd(v[1], v[2]), d = csub(v[1], v[2]);
      const float2 m = v2fma(pk2(t.x, t.y), pk2(-0.5f, -0.5f), pk2(v[0].x, v[0].y));
      v[0] = cadd(v[0], t);
      const float2 r = cscale(make_float2(d.y, -d.x), INV ? -h : h);  // -i h d (forward)
      v[1] = cadd(m, r);
      v[2] = csub(m, r);
    } else if constexpr (Q == 5) {
      constexpr float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
      constexpr float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
      const float2 t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
      const float2 d1 = csub(v[1], v[4]), d2 = csub(v[2], v[3]);
      const float2 x0 = v[0];
      v[0] = cadd(x0, cadd(t1, t2));
      // a1 = x0 + c1 t1 + c2 t2, a2 = x0 + c2 t1 + c1 t2 (FFMA2 with broadcast constants)
      const float2 q = v2fma(pk2(t1.x, t1.y), pk2(c1, c1), pk2(x0.x, x0.y));
      const float2 a1 = v2fma(pk2(t2.x, t2.y), pk2(c2, c2), pk2(q.x, q.y));
      const float2 u = v2fma(pk2(t1.x, t1.y), pk2(c2, c2), pk2(x0.x, x0.y));
      const float2 a2 = v2fma(pk2(t2.x, t2.y), pk2(c1, c1), pk2(u.x, u.y));
      // b1 = s1 d1 + s2 d2, b2 = s2 d1 - s1 d2; X1 = a1 - i b1, X4 = a1 + i b1, X2 = a2 - i b2, X3 = a2 + i b2
      const float2 w1 = v2mul(pk2(d2.x, d2.y), pk2(s2, s2)), w2 = v2mul(pk2(d2.x, d2.y), pk2(-s1, -s1));
      const float2 b1 = v2fma(pk2(d1.x, d1.y), pk2(s1, s1), pk2(w1.x, w1.y));
      const float2 b2 = v2fma(pk2(d1.x, d1.y), pk2(s2, s2), pk2(w2.x, w2.y));
      const float2 ib1 = INV ? make_float2(-b1.y, b1.x) : make_float2(b1.y, -b1.x);  // -+ i b1
      const float2 ib2 = INV ? make_float2(-b2.y, b2.x) : make_float2(b2.y, -b2.x);
      v[1] = cadd(a1, ib1);
      v[4] = csub(a1, ib1);
      v[2] = cadd(a2, ib2);
      v[3] = csub(a2, ib2);
    } else if constexpr (Q == 7 || smallest_factor<Q>() == Q) {
      // direct DFT (prime 7 and anything unfactored): Q^2 constant complex MACs
      float2 out[Q];
      static_for<0, Q>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        float2 acc = v[0];
        static_for<1, Q>([&](auto nc) {
          constexpr int n = decltype(nc)::value;
          acc = cadd(acc, twq<n * k, Q, INV>(v[n]));
        });
        out[k] = acc;
      });
#pragma unroll
      for (int i = 0; i < Q; ++i) v[i] = out[i];
    } else {
      // Q = A B: n = B n1 + n2, k = k1 + A k2
      constexpr int A = smallest_factor<Q>(), B = Q / A;
      float2 y[B][A];
      static_for<0, B>([&](auto n2c) {
        constexpr int n2 = decltype(n2c)::value;
        static_for<0, A>([&](auto n1c) { y[n2][n1c.value] = v[B * n1c.value + n2]; });
        OddDft<A, INV>::run(y[n2]);
        static_for<1, A>([&](auto k1c) {
          constexpr int k1 = decltype(k1c)::value;
          y[n2][k1] = twq<n2 * k1, Q, INV>(y[n2][k1]);
        });
      });
      static_for<0, A>([&](auto k1c) {
        constexpr int k1 = decltype(k1c)::value;
        float2 z[B];
        static_for<0, B>([&](auto n2c) { z[n2c.value] = y[n2c.value][k1]; });
        OddDft<B, INV>::run(z);
        static_for<0, B>([&](auto k2c) { v[k1 + A * k2c.value] = z[k2c.value]; });
      });
    }
  }
};

// ---- the split N = Q P ------------------------------------------------------------------
// Shared layout: Q group buffers of MixedShape::PITCH float2 (padded_len(P) + 1: the odd
// pitch skews the buffers' banks for the strided read-out).
template <int Q, int P>
struct MixedShape {
  static constexpr int N = Q * P;
  static constexpr int TP = FftPlan<P, false>::T;  // threads per length-P FFT
  // whole warps: groups past Q (at most one warp's worth) transform a scratch row nobody reads
  static constexpr int THREADS = (Q * TP + 31) / 32 * 32;
  static constexpr int ROWS = THREADS / TP;
  static constexpr int PITCH = padded_len(P) + 1;
  static constexpr size_t SMEM = (size_t)ROWS * PITCH * sizeof(float2);
  static_assert(THREADS % TP == 0 && THREADS <= 1024, "one CTA, whole FFT groups");
};

// Length-N DFT of load(n) (n in [0, N)) into the group buffers: afterwards X[k1 + Q k2] sits
// at buf[k1 * PITCH + pad16(k2)] (read it with mixed_at).  Every thread of the CTA calls this
// (blockDim.x == MixedShape::THREADS); ends with a CTA barrier.
// Team variant: `team` threads (tid in [0, THREADS)) call this with their own barrier for all of them
// (team_sync) and named barriers from BAR0 for the length-P groups (when a group spans several warps);
// no CTA-wide barrier, so other warps of the CTA (a TMA producer) may run independently.
template <int Q, int P, bool INV, int BAR0, typename Load, typename TeamSync>
__device__ __forceinline__ void block_dft_mixed_team(float2* buf, int tid, Load&& load, TeamSync&& team_sync) {
  using MS = MixedShape<Q, P>;
  constexpr int N = MS::N, TP = MS::TP, PITCH = MS::PITCH;
  constexpr float kStep = (INV ? 6.283185307179586f : -6.283185307179586f) / (float)N;
  // step A: DFT-Q over n1 for each n2, then the inter-step twiddle W_N^(n2 k1)
#pragma unroll 1
  for (int n2 = tid; n2 < P; n2 += MS::THREADS) {
    float2 v[Q];
#pragma unroll
    for (int n1 = 0; n1 < Q; ++n1) v[n1] = load(P * n1 + n2);
    OddDft<Q, INV>::run(v);
    buf[pad16(n2)] = v[0];
    int ph = 0;  // n2 k1 mod N, stepped (n2 < P <= N)
#pragma unroll
    for (int k1 = 1; k1 < Q; ++k1) {
      ph += n2;
      ph = ph >= N ? ph - N : ph;
      const int e = ph > N / 2 ? ph - N : ph;
      float sn, cs;
      __sincosf(kStep * (float)e, &sn, &cs);
      buf[k1 * PITCH + pad16(n2)] = cmul(v[k1], make_float2(cs, sn));
    }
  }
  team_sync();
  // step B: group k1 transforms its row in place (every pass's twiddles from the SFU, SFU_MIN = 1:
  // no table; the inverse plans of 512 / 1024 points start with radix 4, so Ns = 4 passes occur)
  const int g = tid / TP, ti = tid % TP;
  float2* row = buf + g * PITCH;
  auto ld = [&](int idx) -> float2 { return row[pad16(idx)]; };
  auto st = [&](int idx, float2 v) { row[pad16(idx)] = v; };
  // a group's passes exchange data only inside its own row: warp-level barriers for groups of <= 32
  // threads (two 16-thread groups share a warp and its barrier), a named barrier per group otherwise
  auto gsync = [&] {
    if constexpr (TP <= 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(BAR0 + g), "r"(TP) : "memory");
  };
  static_assert(TP <= 32 || BAR0 + MS::ROWS <= 16, "named barriers up to 15");
  block_fft<P, INV, true, true, false, 1>(row, ti, nullptr, ld, st, gsync);
  team_sync();
}

template <int Q, int P, bool INV, typename Load>
__device__ __forceinline__ void block_dft_mixed(float2* buf, Load&& load) {
  block_dft_mixed_team<Q, P, INV, 1>(buf, threadIdx.x, load, [] { __syncthreads(); });
}

// X[k] after block_dft_mixed
template <int Q, int P>
__device__ __forceinline__ float2 mixed_at(const float2* buf, int k) {
  return buf[(k % Q) * MixedShape<Q, P>::PITCH + pad16(k / Q)];
}

}  // namespace lpbp
