// codelets.cuh -- register-resident DFT_R codelets for sm_100a.
//
// A codelet computes an R-point DFT (R | 64) of values held in registers,
// natural order in and out.  It executes the reference's self-sorting
// Stockham stages (proj/src/formula.cpp:168-197, closed form in SURVEY
// Appendix A) on compile-time indices:
//
//   y[(b*cols + m)*k + c] = sum_a W_r^{b a} * w_s^{a m} * x[(m*r + a)*k + c]
//
// with the remainder radix applied first, exactly like plan_stockham.  After
// full unrolling every index is a constant, so the gathers / scatters of the
// reference's FusedPKIV / Permute ops become register renaming, its
// TwiddleMul becomes a multiply by an immediate, and its FusedMKIV butterfly
// becomes straight-line adds.  Multiplies by exact 0/+-1/+-i are elided the
// way lower_complex.cpp:85-105 elides them; (+-1 +- i)/sqrt2 uses the
// 2-mul form.
#pragma once

#include "roots64.cuh"

namespace fftgen_b200 {

// DIR = -1: forward (exp(-2 pi i jk/N), the reference convention, matrix.cpp:14)
// DIR = +1: inverse (conjugate roots, unnormalised)

// x *= W_64^e (forward) or conj(W_64^e) (inverse); e is a compile-time
// constant after inlining, so every branch below folds away.
template <int DIR>
__device__ __forceinline__ void mul_root64(float &re, float &im, int e) {
  e &= 63;
  if (e == 0)
    return;
  if (e == 32) {
    re = -re;
    im = -im;
    return;
  }
  // forward: W^16 = -i, W^48 = +i ; inverse swaps them
  const bool minus_i = (e == 16) == (DIR < 0);
  if (e == 16 || e == 48) {
    const float t = re;
    if (minus_i) {  // (re + i im)(-i) = im - i re
      re = im;
      im = -t;
    } else {        // (re + i im)(+i) = -im + i re
      re = -im;
      im = t;
    }
    return;
  }
  const float c = kRoot64Re[e];
  const float d = DIR < 0 ? kRoot64Im[e] : -kRoot64Im[e];
  if ((e & 7) == 0) {
    // |c| == |d| == sqrt(2)/2: (re + i im)(c + i d) with d = +-c
    const float h = c;
    if (d == c) {  // c(1 + i)
      const float t = re - im;
      im = h * (re + im);
      re = h * t;
      return;
    }
    if (d == -c) {  // c(1 - i)
      const float t = re + im;
      im = h * (im - re);
      re = h * t;
      return;
    }
  }
  const float t = re * c - im * d;
  im = fmaf(re, d, im * c);
  re = t;
}

// In-register radix-r butterflies, natural order.
template <int DIR>
__device__ __forceinline__ void dft2(float &ar, float &ai, float &br, float &bi) {
  const float tr = ar - br, ti = ai - bi;
  ar = ar + br;
  ai = ai + bi;
  br = tr;
  bi = ti;
}

template <int DIR>
__device__ __forceinline__ void dft4(float *r, float *i) {
  // X_b = sum_a W4^{ab} x_a ; W4 = -i (forward)
  const float s0r = r[0] + r[2], s0i = i[0] + i[2];
  const float d0r = r[0] - r[2], d0i = i[0] - i[2];
  const float s1r = r[1] + r[3], s1i = i[1] + i[3];
  const float d1r = r[1] - r[3], d1i = i[1] - i[3];
  r[0] = s0r + s1r;
  i[0] = s0i + s1i;
  r[2] = s0r - s1r;
  i[2] = s0i - s1i;
  // W4^1 * d1: forward -i*d1 = (d1i, -d1r); inverse +i*d1 = (-d1i, d1r)
  if (DIR < 0) {
    r[1] = d0r + d1i;
    i[1] = d0i - d1r;
    r[3] = d0r - d1i;
    i[3] = d0i + d1r;
  } else {
    r[1] = d0r - d1i;
    i[1] = d0i + d1r;
    r[3] = d0r + d1i;
    i[3] = d0i - d1r;
  }
}

template <int DIR>
__device__ __forceinline__ void dft8(float *r, float *i) {
  // radix-2 first (even/odd), then DFT4 of each half, then combine
  float er[4] = {r[0], r[2], r[4], r[6]}, ei[4] = {i[0], i[2], i[4], i[6]};
  float orr[4] = {r[1], r[3], r[5], r[7]}, oi[4] = {i[1], i[3], i[5], i[7]};
  dft4<DIR>(er, ei);
  dft4<DIR>(orr, oi);
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    float tr = orr[b], ti = oi[b];
    mul_root64<DIR>(tr, ti, b * 8);  // W_8^b
    r[b] = er[b] + tr;
    i[b] = ei[b] + ti;
    r[b + 4] = er[b] - tr;
    i[b + 4] = ei[b] - ti;
  }
}

template <int r, int DIR>
__device__ __forceinline__ void dft_small(float *re, float *im) {
  if constexpr (r == 2) {
    dft2<DIR>(re[0], im[0], re[1], im[1]);
  } else if constexpr (r == 4) {
    dft4<DIR>(re, im);
  } else {
    static_assert(r == 8, "sub-radix must be 2, 4 or 8");
    dft8<DIR>(re, im);
  }
}

// Sub-radix sequence (application order) used inside an R-point codelet.
// Largest radix 8; the remainder radix goes first (formula.cpp:184).
template <int R> struct SubRadix;
template <> struct SubRadix<1> { static constexpr int n = 0; static constexpr int r[1] = {1}; };
template <> struct SubRadix<2> { static constexpr int n = 1; static constexpr int r[1] = {2}; };
template <> struct SubRadix<4> { static constexpr int n = 1; static constexpr int r[1] = {4}; };
template <> struct SubRadix<8> { static constexpr int n = 1; static constexpr int r[1] = {8}; };
template <> struct SubRadix<16> { static constexpr int n = 2; static constexpr int r[2] = {2, 8}; };
template <> struct SubRadix<32> { static constexpr int n = 2; static constexpr int r[2] = {4, 8}; };
template <> struct SubRadix<64> { static constexpr int n = 2; static constexpr int r[2] = {8, 8}; };

// One Stockham stage over R registers: radix r, cumulative size s.
template <int R, int r, int s, int DIR>
__device__ __forceinline__ void reg_stage(const float *xr, const float *xi, float *yr, float *yi) {
  constexpr int cols = s / r;
  constexpr int k = R / s;
#pragma unroll
  for (int m = 0; m < cols; ++m) {
#pragma unroll
    for (int c = 0; c < k; ++c) {
      float ar[r], ai[r];
#pragma unroll
      for (int a = 0; a < r; ++a) {
        ar[a] = xr[(m * r + a) * k + c];
        ai[a] = xi[(m * r + a) * k + c];
        // w_s^{a m} = W_64^{a m 64 / s}
        mul_root64<DIR>(ar[a], ai[a], (a * m * (64 / s)) & 63);
      }
      dft_small<r, DIR>(ar, ai);
#pragma unroll
      for (int b = 0; b < r; ++b) {
        yr[(b * cols + m) * k + c] = ar[b];
        yi[(b * cols + m) * k + c] = ai[b];
      }
    }
  }
}

// R-point DFT, natural order in/out, values in re[0..R), im[0..R).
template <int R, int DIR>
__device__ __forceinline__ void reg_fft(float *re, float *im) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (SubRadix<R>::n == 1) {
    dft_small<R, DIR>(re, im);
  } else {
    constexpr int r0 = SubRadix<R>::r[0];
    constexpr int r1 = SubRadix<R>::r[1];
    float tr[R], ti[R];
    reg_stage<R, r0, r0, DIR>(re, im, tr, ti);
    reg_stage<R, r1, r0 * r1, DIR>(tr, ti, re, im);
  }
}

}  // namespace fftgen_b200
