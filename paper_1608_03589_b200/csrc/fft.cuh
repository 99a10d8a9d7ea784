// Block-cooperative Stockham FFT building blocks for sm_100a.
//
// A CTA-resident complex FFT of size N is executed by T = N / E threads, each
// holding E complex values in registers.  A pass of radix R (R divides E)
// performs E/R butterflies per thread:
//
//   butterfly j (k = j mod Ns):
//     v[r]  = buf[j + r*N/R]                     (r = 0..R-1)
//     v[r] *= W_{Ns*R}^{+-r*k}                   (inter-pass twiddle)
//     v     = DFT_R(v)                           (registers, constant twiddles)
//     buf[(j/Ns)*Ns*R + k + r*Ns] = v[r]
//
// (Stockham autosort: natural order in, natural order out, Ns = product of the
// radices already applied.)  All values of a pass live in registers between
// its load and its store, so a single shared buffer plus two barriers per pass
// suffices.  Shared addresses are padded by one float2 every 16 elements
// (pad(i) = i + i/16) so the Ns = 1 scatter (stride R) is bank-conflict free.
//
// Twiddles come from a per-size fp32 table tw[i] = exp(-2*pi*i*I/N) built in
// fp64 on the host; the inverse direction uses the conjugate.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>
#include <utility>

namespace lpbp {

// Complex arithmetic on sm_100a packed-fp32 pipes (FADD2 / FMUL2 / FFMA2).  ptxas
// folds lane broadcasts, lane swaps and single-lane negation into the f32x2
// operands, so a complex add is one instruction and a complex multiply two.
__device__ __forceinline__ unsigned long long pk2(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float2 up2(unsigned long long r) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
  return a;
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return up2(r);
}
__device__ __forceinline__ float2 v2mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return up2(r);
}
__device__ __forceinline__ float2 v2fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return up2(r);
}
// a * b = (a.x b.x, a.y b.x) + b.y (-a.y, a.x)
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  const float2 t = v2mul(pk2(a.x, a.y), pk2(b.x, b.x));
  return v2fma(pk2(-a.y, a.x), pk2(b.y, b.y), pk2(t.x, t.y));
}
// a * conj(b) = (a.x b.x, a.y b.x) + b.y (a.y, -a.x)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  const float2 t = v2mul(pk2(a.x, a.y), pk2(b.x, b.x));
  return v2fma(pk2(a.y, -a.x), pk2(b.y, b.y), pk2(t.x, t.y));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return v2mul(pk2(a.x, a.y), pk2(s, s)); }

template <int S>
__host__ __device__ constexpr int padS(int i) { return i + (i >> S); }
__host__ __device__ constexpr int pad16(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_len(int n) { return n + (n >> 4); }

// cos(2*pi*k/32) and sin(2*pi*k/32), k = 0..8 (first octant); the rest by symmetry.
__host__ __device__ constexpr double cos32_oct(int k) {
  return k == 0 ? 1.0
       : k == 1 ? 0.98078528040323044912618223613424
       : k == 2 ? 0.92387953251128675612818318939679
       : k == 3 ? 0.83146961230254523707878837761791
       : k == 4 ? 0.70710678118654752440084436210485
       : k == 5 ? 0.55557023301960222474283081394853
       : k == 6 ? 0.38268343236508977172845998403040
       : k == 7 ? 0.19509032201612826784828486847702
       : 0.0;
}
// cos(2*pi*k/32) for any k (mod 32)
__host__ __device__ constexpr double cos32(int k) {
  k = ((k % 32) + 32) % 32;
  return k <= 8 ? cos32_oct(k) : k <= 16 ? -cos32_oct(16 - k) : k <= 24 ? -cos32_oct(k - 16) : cos32_oct(32 - k);
}
__host__ __device__ constexpr double sin32(int k) { return cos32(k - 8); }

// e + (c + i s) o as two FFMA2: (e.x + c o.x, e.y + s o.x) + o.y (-s, c)
__device__ __forceinline__ float2 cfma_const(float2 e, float2 o, float c, float s) {
  // e + c o + s (-o.y, o.x): both constants enter as broadcast immediates (no register pairs)
  const float2 t = v2fma(pk2(o.x, o.y), pk2(c, c), pk2(e.x, e.y));
  return v2fma(pk2(-o.y, o.x), pk2(s, s), pk2(t.x, t.y));
}
// 2 e - p (one FFMA2): the partner output of a butterfly whose first output is p = e + t
__device__ __forceinline__ float2 ctwice_minus(float2 e, float2 p) {
  return v2fma(pk2(e.x, e.y), pk2(2.f, 2.f), pk2(-p.x, -p.y));
}

// x * exp(s * 2*pi*i*K/R) with s = -1 (forward) or +1 (inverse); K, R compile-time.
template <int K, int R, bool INV>
__device__ __forceinline__ float2 twc(float2 x) {
  constexpr int k = ((K % R) + R) % R;
  if constexpr (k == 0) {
    return x;
  } else if constexpr (4 * k == R) {  // exp(-+i*pi/2) = -+i
    return INV ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);
  } else if constexpr (2 * k == R) {
    return make_float2(-x.x, -x.y);
  } else if constexpr (4 * k == 3 * R) {
    return INV ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);
  } else {
    constexpr int k32 = k * (32 / R);
    constexpr float c = (float)cos32(k32);
    constexpr float s = INV ? (float)sin32(k32) : -(float)sin32(k32);
    return cmul(x, make_float2(c, s));
  }
}

template <int I, int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

// Radix-R DFT in registers, natural order in and out (recursive radix-2 DIT,
// fully unrolled at compile time).  STRIDE/OFF select the subsequence of the
// length-LEN input.  ZU: inputs at index >= LEN/2 are known zero (leaf butterflies
// pairing x[j] with x[j+LEN/2] collapse to copies).  LOW: only outputs < R/2 of
// the top-level transform are needed.
template <int R, bool INV>
struct Dft {
  template <int OFF, int STRIDE, int LEN, bool ZU, bool LOW>
  __device__ __forceinline__ static void run_sub(const float2 (&in)[LEN], float2 (&out)[R]) {
    if constexpr (R == 1) {
      out[0] = in[OFF];
    } else if constexpr (R == 2) {
      const float2 a = in[OFF];
      if constexpr (ZU && OFF + STRIDE >= LEN / 2) {
        out[0] = a;
        out[1] = a;
      } else {
        const float2 b = in[OFF + STRIDE];
        out[0] = cadd(a, b);
        if constexpr (!LOW) out[1] = csub(a, b);
      }
    } else {
      float2 E[R / 2], O[R / 2];
      Dft<R / 2, INV>::template run_sub<OFF, STRIDE * 2, LEN, ZU, false>(in, E);
      Dft<R / 2, INV>::template run_sub<OFF + STRIDE, STRIDE * 2, LEN, ZU, false>(in, O);
      static_for<0, R / 2>([&](auto kc) {
        constexpr int k = decltype(kc)::value;
        if constexpr (k == 0 || 4 * k == R) {  // multiplier 1 or -+i: free
          const float2 t = twc<k, R, INV>(O[k]);
          out[k] = cadd(E[k], t);
          if constexpr (!LOW) out[k + R / 2] = csub(E[k], t);
        } else {  // E + w O as two FFMA2, E - w O = 2E - (E + w O) as one
          constexpr int k32 = k * (32 / R);
          constexpr float c = (float)cos32(k32);
          constexpr float sn = INV ? (float)sin32(k32) : -(float)sin32(k32);
          out[k] = cfma_const(E[k], O[k], c, sn);
          if constexpr (!LOW) out[k + R / 2] = ctwice_minus(E[k], out[k]);
        }
      });
    }
  }
  __device__ __forceinline__ static void run(float2 (&v)[R]) {
    float2 out[R];
    run_sub<0, 1, R, false, false>(v, out);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = out[i];
  }
  // v[R/2..R-1] are zero on entry
  __device__ __forceinline__ static void run_zu(float2 (&v)[R]) {
    float2 out[R];
    run_sub<0, 1, R, true, false>(v, out);
#pragma unroll
    for (int i = 0; i < R; ++i) v[i] = out[i];
  }
  // only v[0..R/2) are produced
  __device__ __forceinline__ static void run_low(float2 (&v)[R]) {
    float2 out[R];
    run_sub<0, 1, R, false, true>(v, out);
#pragma unroll
    for (int i = 0; i < R / 2; ++i) v[i] = out[i];
  }
};

// Multiply v[r] (r = 1..R-1) by the inter-pass twiddle exp(-+2 pi i r k / (Ns R)).
// tw points at this pass's block of the per-size pass table, laid out
// [r-1][k] (k < Ns) so consecutive butterflies read consecutive entries; the
// inverse passes' blocks hold the conjugates.
template <int R, int Ns>
__device__ __forceinline__ void apply_twiddles(float2 (&v)[R], int k, const float2* __restrict__ tw) {
  if constexpr (Ns > 1) {
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(tw + (r - 1) * Ns + k));
  }
}

// Same twiddles generated on the SFU: exact integer phase e = r*k mod (Ns*R),
// folded into (-pi, pi], then MUFU sin/cos (abs error ~4e-7).  Trades the
// twiddle-table loads (L2 latency) for the otherwise idle SFU pipe.
template <int R, int Ns, bool INV>
__device__ __forceinline__ void apply_twiddles_sfu(float2 (&v)[R], int k) {
  if constexpr (Ns > 1) {
    constexpr int M = Ns * R;
    constexpr float kStep = (INV ? 6.283185307179586f : -6.283185307179586f) / (float)M;
#pragma unroll
    for (int r = 1; r < R; ++r) {
      int e = (r * k) & (M - 1);
      e = e > M / 2 ? e - M : e;
      float sn, cs;
      __sincosf(kStep * (float)e, &sn, &cs);
      v[r] = cmul(v[r], make_float2(cs, sn));
    }
  }
}

// SFU twiddles with a radix-4 split r = 4a + b: w^(4a) and w^b (b < 4) come from
// the SFU, the rest is one complex product each (error ~2x a single SFU value).
template <int R, int Ns, bool INV>
__device__ __forceinline__ void apply_twiddles_sfu4(float2 (&v)[R], int k) {
  if constexpr (Ns > 1) {
    constexpr int M = Ns * R;
    constexpr float kStep = (INV ? 6.283185307179586f : -6.283185307179586f) / (float)M;
    auto sfu = [&](int r) {
      int e = (r * k) & (M - 1);
      e = e > M / 2 ? e - M : e;
      float sn, cs;
      __sincosf(kStep * (float)e, &sn, &cs);
      return make_float2(cs, sn);
    };
    float2 wb[4];
#pragma unroll
    for (int b = 1; b < 4 && b < R; ++b) {
      wb[b] = sfu(b);
      v[b] = cmul(v[b], wb[b]);
    }
#pragma unroll
    for (int a = 1; a < R / 4; ++a) {
      const float2 wa = sfu(4 * a);
      v[4 * a] = cmul(v[4 * a], wa);
#pragma unroll
      for (int b = 1; b < 4; ++b) v[4 * a + b] = cmul(v[4 * a + b], cmul(wa, wb[b]));
    }
  }
}

// Pass-0 input element r of butterfly j (index j + r*STRIDE).  A loader may take
// (j, integral_constant<r>) instead of the flat index to specialise on r.
template <int RIDX, int STRIDE, typename Load>
__device__ __forceinline__ float2 load_at(Load& load, int j) {
  if constexpr (std::is_invocable_v<Load&, int, std::integral_constant<int, RIDX>>)
    return load(j, std::integral_constant<int, RIDX>{});
  else
    return load(j + RIDX * STRIDE);
}

// Load the R inputs of butterfly j of a pass from (padded) shared memory.
// Padded addressing: when the stride between a butterfly's elements is a
// multiple of 2^S, pad(base + r*stride) = pad(base) + r*(stride + stride/2^S),
// so every element is one base register plus a compile-time immediate.
template <int N, int R, int S>
__device__ __forceinline__ void pass_load(const float2* buf, int j, float2 (&v)[R]) {
  constexpr int STRIDE = N / R;
  if constexpr (STRIDE % (1 << S) == 0) {
    const float2* b = buf + padS<S>(j);
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = b[r * (STRIDE + (STRIDE >> S))];
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = buf[padS<S>(j + r * STRIDE)];
  }
}
template <int N, int R, int Ns, int S>
__device__ __forceinline__ void pass_store(float2* buf, int j, const float2 (&v)[R]) {
  if constexpr (Ns == 1 && R == (1 << S)) {
    // d = j*R, pad(d + r) = j*(R+1) + r
    float2* b = buf + j * (R + 1);
#pragma unroll
    for (int r = 0; r < R; ++r) b[r] = v[r];
  } else if constexpr (Ns % (1 << S) == 0) {
    float2* b = buf + padS<S>((j / Ns) * Ns * R + (j % Ns));
#pragma unroll
    for (int r = 0; r < R; ++r) b[r * (Ns + (Ns >> S))] = v[r];
  } else {
    const int d = (j / Ns) * Ns * R + (j % Ns);
#pragma unroll
    for (int r = 0; r < R; ++r) buf[padS<S>(d + r * Ns)] = v[r];
  }
}

// One full smem->smem Stockham pass for a group of T threads (ti in [0,T)).
// Caller provides the barrier that separates the previous pass's stores from
// these loads; this function places the barrier between loads and stores.
// SFU_MIN: passes with Ns >= SFU_MIN take SFU twiddles (0 = always the table).
template <int N, int R, int Ns, int T, bool INV, int S, int SFU_MIN = 0, typename Sync>
__device__ __forceinline__ void pass_smem(float2* buf, int ti, const float2* __restrict__ tw, Sync&& sync) {
  constexpr int NB = (N / R) / T;  // butterflies per thread
  static_assert(NB >= 1 && NB * T * R == N, "bad pass shape");
  float2 v[NB][R];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = ti + b * T;
    pass_load<N, R, S>(buf, j, v[b]);
    if constexpr (SFU_MIN > 0 && Ns >= SFU_MIN) apply_twiddles_sfu4<R, Ns, INV>(v[b], j % Ns);
    else apply_twiddles<R, Ns>(v[b], j % Ns, tw);
    Dft<R, INV>::run(v[b]);
  }
  sync();
#pragma unroll
  for (int b = 0; b < NB; ++b) pass_store<N, R, Ns, S>(buf, ti + b * T, v[b]);
}

// Radix plans (forward order; the inverse runs them reversed).  Every plan
// starts with radix 16 so Ns >= 16 for every store after the first pass.
template <int N> struct RadixPlan;
template <> struct RadixPlan<128>   { static constexpr int P = 2; static constexpr int r[3] = {16, 8, 1};  static constexpr int E = 16; };
template <> struct RadixPlan<256>   { static constexpr int P = 2; static constexpr int r[3] = {16, 16, 1}; static constexpr int E = 16; };
template <> struct RadixPlan<512>   { static constexpr int P = 3; static constexpr int r[3] = {16, 8, 4};  static constexpr int E = 16; };
template <> struct RadixPlan<1024>  { static constexpr int P = 3; static constexpr int r[3] = {16, 16, 4}; static constexpr int E = 16; };
template <> struct RadixPlan<2048>  { static constexpr int P = 3; static constexpr int r[3] = {16, 16, 8}; static constexpr int E = 16; };
template <> struct RadixPlan<4096>  { static constexpr int P = 3; static constexpr int r[3] = {16, 16, 16}; static constexpr int E = 16; };
template <> struct RadixPlan<8192>  { static constexpr int P = 3; static constexpr int r[3] = {16, 16, 32}; static constexpr int E = 32; };
template <> struct RadixPlan<16384> { static constexpr int P = 3; static constexpr int r[3] = {16, 32, 32}; static constexpr int E = 32; };

template <int N, bool INV>
struct FftPlan {
  using RP = RadixPlan<N>;
  static constexpr int P = RP::P;
  static constexpr int E = RP::E;
  static constexpr int T = N / E;  // threads per FFT
  static constexpr int radix(int i) { return INV ? RP::r[P - 1 - i] : RP::r[i]; }
  static constexpr int ns(int i) {
    int s = 1;
    for (int q = 0; q < i; ++q) s *= radix(q);
    return s;
  }
  // padding shift for this direction: match the first pass's Ns = 1 scatter stride
  static constexpr int S = radix(0) >= 32 ? 5 : 4;
  // offset (float2 entries) of pass i's twiddle block inside this direction's table
  static constexpr int tw_off(int i) {
    int o = 0;
    for (int q = 1; q < i; ++q) o += (radix(q) - 1) * ns(q);
    return o;
  }
  static constexpr int tw_len = tw_off(P);
};

// Per-size twiddle table: forward passes' blocks, then inverse passes' blocks.
template <int N>
struct TwTable {
  static constexpr int fwd = 0;
  static constexpr int inv = FftPlan<N, false>::tw_len;
  static constexpr int len = FftPlan<N, false>::tw_len + FftPlan<N, true>::tw_len;
};

// Full size-N FFT over a group of T = N/E threads (ti in [0,T)).
//   load(idx)       -> float2 : input element idx (first pass reads it directly)
//   store(idx, val)           : output element idx (last pass writes it directly)
//   sync()                    : barrier covering every thread that shares buf
// LAST_SYNC places a barrier between the last pass's loads and its stores (needed
// when store() writes back into buf); FIRST_SYNC places a sync() barrier between
// pass 0's loads and stores (needed when load() reads buf or a region other
// groups' buffers overlap).
// The caller must guarantee buf is free on entry (no thread still reading it).
// Middle passes go through the padded shared buffer buf (padded_len(N) float2).
// IN_HALF: load(idx) is zero for idx >= N/2 (never called there).
template <int N, bool INV, bool LAST_SYNC, bool FIRST_SYNC = false, bool IN_HALF = false, int SFU_MIN = 0,
          typename Load, typename Store, typename Sync>
__device__ __forceinline__ void block_fft(float2* buf, int ti, const float2* __restrict__ twt,
                                          Load&& load, Store&& store, Sync&& sync) {
  using FP = FftPlan<N, INV>;
  constexpr int T = FP::T;
  constexpr int P = FP::P;
  constexpr int S = FP::S;
  const float2* tw = twt + (INV ? TwTable<N>::inv : TwTable<N>::fwd);
  {  // pass 0: Ns = 1, no twiddles
    constexpr int R = FP::radix(0);
    constexpr int NB = (N / R) / T;
    float2 v[NB][R];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = ti + b * T;
      if constexpr (IN_HALF) {
        static_for<0, R / 2>([&](auto rc) { v[b][rc.value] = load_at<rc.value, N / R>(load, j); });
        Dft<R, INV>::run_zu(v[b]);
      } else {
        static_for<0, R>([&](auto rc) { v[b][rc.value] = load_at<rc.value, N / R>(load, j); });
        Dft<R, INV>::run(v[b]);
      }
    }
    if constexpr (FIRST_SYNC) sync();  // load() reads buf: everyone's pass-0 loads before any store
#pragma unroll
    for (int b = 0; b < NB; ++b) pass_store<N, R, 1, S>(buf, ti + b * T, v[b]);
  }
  sync();
  static_for<1, P - 1>([&](auto ic) {
    constexpr int I = decltype(ic)::value;
    pass_smem<N, FP::radix(I), FP::ns(I), T, INV, S, SFU_MIN>(buf, ti, tw + FP::tw_off(I), sync);
    sync();
  });
  {  // last pass: outputs at j + r*Ns (Ns = N/R, j < Ns)
    constexpr int R = FP::radix(P - 1);
    constexpr int Ns = FP::ns(P - 1);
    constexpr int NB = (N / R) / T;
    static_assert(Ns * R == N, "plan does not multiply to N");
    float2 v[NB][R];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = ti + b * T;
      pass_load<N, R, S>(buf, j, v[b]);
      if constexpr (SFU_MIN > 0 && Ns >= SFU_MIN) apply_twiddles_sfu4<R, Ns, INV>(v[b], j);
      else apply_twiddles<R, Ns>(v[b], j, tw + FP::tw_off(P - 1));
      Dft<R, INV>::run(v[b]);
    }
    if constexpr (LAST_SYNC) sync();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = ti + b * T;
#pragma unroll
      for (int r = 0; r < R; ++r) store(j + r * Ns, v[b][r]);
    }
  }
}

// First-pass input of block_conv: load(idx), or load(integral_constant<e>, idx) where e = b*RL + r is
// the value's compile-time position among the thread's first-pass loads (RL loads per butterfly).
template <int E_IDX, typename Load>
__device__ __forceinline__ float2 load_e(Load& load, int idx) {
  if constexpr (std::is_invocable_v<Load&, std::integral_constant<int, E_IDX>, int>)
    return load(std::integral_constant<int, E_IDX>{}, idx);
  else
    return load(idx);
}

// Pointwise multiply of the fused middle: mul(idx, val), or mul(integral_constant<e>, idx, val) where
// e = b*R + r is the value's compile-time position among the thread's E outputs of the forward
// transform (lets a multiplier keep per-thread operands in registers or TMEM, chunk by chunk).
template <int E_IDX, typename Mul>
__device__ __forceinline__ float2 mul_at(Mul& mul, int idx, float2 v) {
  if constexpr (std::is_invocable_v<Mul&, std::integral_constant<int, E_IDX>, int, float2>)
    return mul(std::integral_constant<int, E_IDX>{}, idx, v);
  else
    return mul(idx, v);
}

// Circular convolution core: y = IFFT_N( mul(FFT_N(x)) ), unnormalised inverse.
// The last forward pass and the first inverse pass share their radix and the
// butterfly->thread map, so the spectrum never touches shared memory: each
// thread multiplies its own outputs (mul(idx, val) -> val) and runs the first
// inverse butterfly in registers.
// PRUNE: load(idx) is zero for idx >= N/2 and store() is only needed for idx < N/2
// (zero-padded linear convolution): first forward pass and last inverse pass
// skip the known-zero inputs / unneeded outputs.
// SFU_MIN: passes with Ns >= SFU_MIN take their twiddles from the SFU instead of the table (0 = never).
template <int N, bool PRUNE = false, int SFU_MIN = 0, typename Load, typename Mul, typename Store, typename Sync>
__device__ __forceinline__ void block_conv(float2* buf, int ti, const float2* __restrict__ twt,
                                           Load&& load, Mul&& mul, Store&& store, Sync&& sync) {
  using F = FftPlan<N, false>;
  using B = FftPlan<N, true>;
  constexpr int T = F::T;
  constexpr int P = F::P;
  static_assert(F::radix(P - 1) == B::radix(0), "fused middle needs matching radices");
  const float2* twf = twt + TwTable<N>::fwd;
  const float2* twi = twt + TwTable<N>::inv;
  {  // forward pass 0
    constexpr int R = F::radix(0);
    constexpr int NB = (N / R) / T;
    constexpr int RL = PRUNE ? R / 2 : R;  // loads per butterfly
    float2 v[NB][R];
    static_for<0, NB>([&](auto bc) {
      constexpr int b = decltype(bc)::value;
      const int j = ti + b * T;
      static_for<0, RL>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        v[b][r] = load_e<b * RL + r>(load, j + r * (N / R));
      });
      if constexpr (PRUNE) Dft<R, false>::run_zu(v[b]);
      else Dft<R, false>::run(v[b]);
    });
#pragma unroll
    for (int b = 0; b < NB; ++b) pass_store<N, R, 1, F::S>(buf, ti + b * T, v[b]);
  }
  sync();
  static_for<1, P - 1>([&](auto ic) {
    constexpr int I = decltype(ic)::value;
    pass_smem<N, F::radix(I), F::ns(I), T, false, F::S, SFU_MIN>(buf, ti, twf + F::tw_off(I), sync);
    sync();
  });
  {  // forward last pass -> pointwise multiply -> inverse pass 0, all in registers
    constexpr int R = F::radix(P - 1);
    constexpr int Ns = F::ns(P - 1);
    constexpr int NB = (N / R) / T;
    float2 v[NB][R];
    static_for<0, NB>([&](auto bc) {
      constexpr int b = decltype(bc)::value;
      const int j = ti + b * T;
      pass_load<N, R, F::S>(buf, j, v[b]);
      if constexpr (SFU_MIN > 0 && Ns >= SFU_MIN) apply_twiddles_sfu4<R, Ns, false>(v[b], j);
      else apply_twiddles<R, Ns>(v[b], j, twf + F::tw_off(P - 1));
      Dft<R, false>::run(v[b]);
      static_for<0, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        v[b][r] = mul_at<b * R + r>(mul, j + r * Ns, v[b][r]);
      });
      Dft<R, true>::run(v[b]);  // inverse pass 0 (Ns = 1: no twiddles)
    });
    sync();
#pragma unroll
    for (int b = 0; b < NB; ++b) pass_store<N, R, 1, B::S>(buf, ti + b * T, v[b]);
  }
  sync();
  static_for<1, P - 1>([&](auto ic) {
    constexpr int I = decltype(ic)::value;
    pass_smem<N, B::radix(I), B::ns(I), T, true, B::S, SFU_MIN>(buf, ti, twi + B::tw_off(I), sync);
    sync();
  });
  {  // inverse last pass
    constexpr int R = B::radix(P - 1);
    constexpr int Ns = B::ns(P - 1);
    constexpr int NB = (N / R) / T;
    float2 v[NB][R];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = ti + b * T;
      pass_load<N, R, B::S>(buf, j, v[b]);
      if constexpr (SFU_MIN > 0 && Ns >= SFU_MIN) apply_twiddles_sfu4<R, Ns, true>(v[b], j);
      else apply_twiddles<R, Ns>(v[b], j, twi + B::tw_off(P - 1));
      if constexpr (PRUNE) Dft<R, true>::run_low(v[b]);
      else Dft<R, true>::run(v[b]);
    }
    constexpr int RO = PRUNE ? R / 2 : R;  // outputs j + r*Ns, r < RO
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = ti + b * T;
#pragma unroll
      for (int r = 0; r < RO; ++r) store(j + r * Ns, v[b][r]);
    }
  }
}

// Fill the pass-twiddle table of size N (TwTable<N>::len entries) in fp64.
template <int N>
__global__ void k_init_twiddles(float2* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= TwTable<N>::len) return;
  auto fill = [&](auto fp, int base, double sgn) {
    using FP = decltype(fp);
    static_for<1, FP::P>([&](auto ic) {
      constexpr int I = decltype(ic)::value;
      constexpr int R = FP::radix(I), Ns = FP::ns(I);
      const int lo = base + FP::tw_off(I), hi = lo + (R - 1) * Ns;
      if (e >= lo && e < hi) {
        const int r = (e - lo) / Ns + 1, k = (e - lo) % Ns;
        double sn, cs;
        sincospi(sgn * 2.0 * (double)(r * k) / (double)(Ns * R), &sn, &cs);
        out[e] = make_float2((float)cs, (float)sn);
      }
    });
  };
  fill(FftPlan<N, false>{}, TwTable<N>::fwd, -1.0);
  fill(FftPlan<N, true>{}, TwTable<N>::inv, +1.0);
}

}  // namespace lpbp
