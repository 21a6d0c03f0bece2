// codelets.cuh -- register-resident DFT_R codelets for sm_100a, packed fp32x2.
//
// A complex value lives in one float2 register pair (re, im) and every
// butterfly operation is a Blackwell packed instruction:
//   complex add / sub          -> FADD2 (one instruction for re and im)
//   multiply by -i / +i        -> free: FADD2 operand modifiers .LO_HI.NP
//                                 (lane swap + one-lane negate)
//   multiply by a constant w   -> FMUL2 (broadcast w.re) + FFMA2 (swapped x,
//                                 broadcast w.im): 2 instructions
// which halves the issue count of the fp32 scalar formulation.
//
// A codelet computes an R-point DFT (R | 64) of values held in registers,
// natural order in and out, by executing the reference's self-sorting
// Stockham stages (proj/src/formula.cpp:168-197; closed form in SURVEY
// Appendix A) on compile-time indices:
//
//   y[(b*cols + m)*k + c] = sum_a W_r^{b a} * w_s^{a m} * x[(m*r + a)*k + c]
//
// with the remainder radix applied first, exactly like plan_stockham.  After
// full unrolling every index is a constant, so the reference's FusedPKIV /
// Permute gathers become register renaming, its TwiddleMul a multiply by an
// immediate, and its FusedMKIV butterfly straight-line FADD2s.  Multiplies
// by exact +-1 / +-i are elided the way lower_complex.cpp:85-105 elides them.
#pragma once

#include "roots64.cuh"

namespace fftgen_b200 {

#define FFTGEN_FI __device__ __forceinline__

// DIR = -1: forward (exp(-2 pi i jk/N), the reference convention, matrix.cpp:14)
// DIR = +1: inverse (conjugate roots, unnormalised)

FFTGEN_FI float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
FFTGEN_FI float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
FFTGEN_FI float2 cneg(float2 a) { return make_float2(-a.x, -a.y); }

// x * W_4^1: forward -i (re, im) -> (im, -re); inverse +i -> (-im, re)
template <int DIR> FFTGEN_FI float2 mul_w4(float2 a) {
  return DIR < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}

// x * (c + i d): FMUL2 + FFMA2
FFTGEN_FI float2 cmul(float2 x, float c, float d) {
  return __ffma2_rn(make_float2(-x.y, x.x), make_float2(d, d), __fmul2_rn(x, make_float2(c, c)));
}

// x * W_64^e (forward) or conj(W_64^e) (inverse); e is a compile-time
// constant after inlining, so every branch below folds away.
template <int DIR> FFTGEN_FI float2 mul_root64(float2 x, int e) {
  e &= 63;
  if (e == 0) return x;
  if (e == 32) return cneg(x);
  if (e == 16) return mul_w4<DIR>(x);
  if (e == 48) return mul_w4<-DIR>(x);
  const float c = kRoot64Re[e];
  const float d = DIR < 0 ? kRoot64Im[e] : -kRoot64Im[e];
  return cmul(x, c, d);
}

// x * w (runtime twiddle from a forward table); inverse uses conj(w)
template <int DIR> FFTGEN_FI float2 mul_tw(float2 x, float2 w) {
  return cmul(x, w.x, DIR < 0 ? w.y : -w.y);
}

// In-register radix-r butterflies, natural order.
template <int DIR> FFTGEN_FI void dft2(float2 *v) {
  const float2 t = csub(v[0], v[1]);
  v[0] = cadd(v[0], v[1]);
  v[1] = t;
}

template <int DIR> FFTGEN_FI void dft4(float2 *v) {
  const float2 s0 = cadd(v[0], v[2]), d0 = csub(v[0], v[2]);
  const float2 s1 = cadd(v[1], v[3]), d1 = mul_w4<DIR>(csub(v[1], v[3]));
  v[0] = cadd(s0, s1);
  v[2] = csub(s0, s1);
  v[1] = cadd(d0, d1);
  v[3] = csub(d0, d1);
}

template <int DIR> FFTGEN_FI void dft8(float2 *v) {
  float2 e[4] = {v[0], v[2], v[4], v[6]};
  float2 o[4] = {v[1], v[3], v[5], v[7]};
  dft4<DIR>(e);
  dft4<DIR>(o);
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const float2 t = mul_root64<DIR>(o[b], b * 8);  // W_8^b
    v[b] = cadd(e[b], t);
    v[b + 4] = csub(e[b], t);
  }
}

template <int r, int DIR> FFTGEN_FI void dft_small(float2 *v) {
  if constexpr (r == 2) {
    dft2<DIR>(v);
  } else if constexpr (r == 4) {
    dft4<DIR>(v);
  } else {
    static_assert(r == 8, "sub-radix must be 2, 4 or 8");
    dft8<DIR>(v);
  }
}

// Sub-radix sequence (application order) inside an R-point codelet; the
// remainder radix goes first (formula.cpp:184).
template <int R> struct SubRadix;
template <> struct SubRadix<1> { static constexpr int n = 0, r0 = 1, r1 = 1; };
template <> struct SubRadix<2> { static constexpr int n = 1, r0 = 2, r1 = 1; };
template <> struct SubRadix<4> { static constexpr int n = 1, r0 = 4, r1 = 1; };
template <> struct SubRadix<8> { static constexpr int n = 1, r0 = 8, r1 = 1; };
template <> struct SubRadix<16> { static constexpr int n = 2, r0 = 2, r1 = 8; };
template <> struct SubRadix<32> { static constexpr int n = 2, r0 = 4, r1 = 8; };
template <> struct SubRadix<64> { static constexpr int n = 2, r0 = 8, r1 = 8; };

// One Stockham stage over R registers: radix r, cumulative size s.
template <int R, int r, int s, int DIR>
FFTGEN_FI void reg_stage(const float2 *x, float2 *y) {
  constexpr int cols = s / r;
  constexpr int k = R / s;
#pragma unroll
  for (int m = 0; m < cols; ++m) {
#pragma unroll
    for (int c = 0; c < k; ++c) {
      float2 a[r];
#pragma unroll
      for (int q = 0; q < r; ++q)  // w_s^{q m} = W_64^{q m 64 / s}
        a[q] = mul_root64<DIR>(x[(m * r + q) * k + c], (q * m * (64 / s)) & 63);
      dft_small<r, DIR>(a);
#pragma unroll
      for (int b = 0; b < r; ++b) y[(b * cols + m) * k + c] = a[b];
    }
  }
}

// R-point DFT, natural order in/out.
template <int R, int DIR> FFTGEN_FI void reg_fft(float2 *v) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (SubRadix<R>::n == 1) {
    dft_small<R, DIR>(v);
  } else {
    constexpr int r0 = SubRadix<R>::r0, r1 = SubRadix<R>::r1;
    float2 t[R];
    reg_stage<R, r0, r0, DIR>(v, t);
    reg_stage<R, r1, r0 * r1, DIR>(t, v);
  }
}

}  // namespace fftgen_b200
