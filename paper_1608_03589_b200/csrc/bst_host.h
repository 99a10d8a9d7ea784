// Host-side (fp64) geometry and tables of the BST engine, the reference's
// frequency-domain backprojection (fastbp.bst, bst.py:120-206) and fbp's default
// engine (filtering.py:73-98).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "plan_host.h"

namespace lpbp {

struct BstParams {
  int nt, ntheta, n;
  double beta;      // Kaiser window shape (0 = none)
  double zero_pad;  // radial zero padding factor
  int dc_mode;      // 0 = subtract_mean, 1 = kernel_cap
  bool filter;      // fbp: filter_sinogram first, then x 1/(2 pi)
  double lam, cutoff;
};

struct BstHost {
  BstParams p{};
  int ns = 0;       // radial samples per half-ray (2 x nt/2, bst.py:128)
  int nray = 0;     // 2 ntheta half-rays
  int L = 0;        // radial DFT length next_fast_len(max(ceil(2 z (ns-1)), ns))
  int m_need = 0;   // radial bins kept (reach the Nyquist radius of the padded grid)
  int m_pad = 0;    // row pitch of the polar spectrum (multiple of 4)
  int big = 0;      // padded image side DOMAIN_PAD * n
  int p0 = 0;       // crop offset
  double ds = 0, dsigma = 0, dw = 0;
  double out_scale = 0;  // BST_SCALE / (4 d^2) (x FBP_SCALE for fbp)
  // semi-polar taps with the window (and the half weight of s = 0) folded in:
  // positive half-ray at t = +s_k, negative at t = -s_k (grids.py:290-311)
  std::vector<I2> tap_base;  // [ns] (pos base, neg base)
  std::vector<F4> tap_w;     // [ns] (pos w0, pos w1, neg w0, neg w1)
  std::vector<float> kern;   // [m_need] ds * (1/sigma or DC rule) * 1/2 (Hermitian averaging)
  std::vector<F2> tau;       // [big] phase ramp exp(i dw k ((0.5 - p0) dx - 1)), FFT order
  std::vector<F2> cmean;     // [big] sum_{y in crop} exp(2 pi i k y / big) / n^2 (crop mean from a row)
  // chord of the square as a trapezoid in t per angle (subtract_mean): (t1, t2, Lmax * dt * dtheta / 4,
  // 1 / (t2 - t1)) with chord = Lmax for |t| <= t1, linear to 0 at |t| = t2 (radon.py:183-209)
  std::vector<F4> chord_col;  // [ntheta]
  // gridding coordinates of the quadrant kx, ky >= 0 (fp64, grids.py:477-494): qx in [0, big/2],
  // ky in [0, big/2); .x = i0 | q(wi) << 13, .y = j0 | q(wj) << 13, 19-bit fixed-point weights.
  // Points with kfx < 0 reflect theta -> pi - theta in index space.
  int qw_pitch = 0;
  std::vector<uint32_t> grid_q;  // [big/2][qw_pitch][2]
  // fbp: ramp filter on the M-point circular embedding (as the log-polar plan)
  int M = 0, Lr = 0;
  std::vector<float> ramp;
  // generic sizes: Bluestein on pow2 convolutions (0 = the direct power-of-two FFT)
  int mb_L = 0, mb_big = 0;
  std::vector<F2> chirp_L, bhat_L, chirp_big, bhat_big;
  // support (this build): L a power of two in [512, 8192] or 2 L <= 8192 (Bluestein);
  // big a power of two in [128, 4096] or 2 big <= 8192 (Bluestein)
  bool supported = false;
};

// Validates like BstOptions / _radial_spectra (ValueError texts verbatim) and
// builds the tables.  Returns "" on success.
std::string build_bst_host(const BstParams& p, BstHost& h);

}  // namespace lpbp
