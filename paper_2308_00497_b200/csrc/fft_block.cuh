// fft_block.cuh -- K2: batched, shared-memory-resident Stockham FFT (sm_100a).
//
// One CTA owns TPB whole transforms.  The reference's Stockham stage list
// (plan_stockham, proj/src/formula.cpp:168-197) is regrouped into P <= 3
// register passes of radix R_p <= 64; pass p is one Stockham stage of radix
// R_p with cumulative size s_p, cols_p = s_p / R_p, k_p = N / s_p:
//
//   y[(B cols + m) k + c] = DFT_R( x[(m R + A) k + c] * w_s^{A m} )[B]
//
// (a consecutive group of radix-r Stockham stages is exactly one radix-R
// Stockham stage; tests/test_plan.py restates this in numpy).  So
//   * the FusedPKIV / Permute data movement of every stage is folded into the
//     pass's load / store addressing (no permutation pass),
//   * the TwiddleMul of the pass is one multiply by w_s^{A m} from a
//     coalesced [A][m] fp32 table (precomputed in fp64 at plan time, shared by
//     both layouts and both directions),
//   * the FusedMKIV butterflies are the register codelet (codelets.cuh),
//   * HBM is touched exactly once on load (pass 0) and once on store (pass
//     P-1): 16 N bytes per transform, the roofline's algorithmic traffic.
// Between passes the data crosses shared memory once, in split re/im float
// arrays with a padding chosen at compile time (pad_search) so that both
// the writer's and the reader's 32-lane access patterns are conflict-free.
#pragma once

#include <cstdint>

#include "block_geom.hpp"
#include "codelets.cuh"
#include "kernels.hpp"

namespace fftgen_b200 {


template <int LAYOUT> struct GIO;
template <> struct GIO<LAYOUT_INTERLEAVED> {
  static __device__ __forceinline__ void load(const BlockArgs &a, int64_t off, float &re, float &im) {
    const float2 v = __ldcs(reinterpret_cast<const float2 *>(a.in0) + off);
    re = v.x;
    im = v.y;
  }
  static __device__ __forceinline__ void store(const BlockArgs &a, int64_t off, float re, float im) {
    __stcs(reinterpret_cast<float2 *>(a.out0) + off, make_float2(re, im));
  }
};
template <> struct GIO<LAYOUT_SPLIT> {
  static __device__ __forceinline__ void load(const BlockArgs &a, int64_t off, float &re, float &im) {
    re = __ldcs(reinterpret_cast<const float *>(a.in0) + off);
    im = __ldcs(reinterpret_cast<const float *>(a.in1) + off);
  }
  static __device__ __forceinline__ void store(const BlockArgs &a, int64_t off, float re, float im) {
    __stcs(reinterpret_cast<float *>(a.out0) + off, re);
    __stcs(reinterpret_cast<float *>(a.out1) + off, im);
  }
};

template <int N, int p, int DIR>
__device__ __forceinline__ void pass_twiddle(const float2 *__restrict__ tw, int m, int A, float &re, float &im) {
  using G = BlockGeom<N>;
  if (A == 0) return;
  const float2 w = __ldg(tw + G::TW_OFF(p) + A * G::COLS(p) + m);
  const float wi = DIR < 0 ? w.y : -w.y;
  const float t = re * w.x - im * wi;
  im = fmaf(re, wi, im * w.x);
  re = t;
}

template <int N, int p>
__device__ __forceinline__ void smem_write(float *sre, float *sim, int t, const float *re, const float *im) {
  using G = BlockGeom<N>;
  constexpr int R = G::R(p), cols = G::COLS(p), k = G::K(p), J = G::RMAX / R, T = G::T;
  constexpr Pad pd = BoundaryPad<N, p>::value;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int u = t + j * T, m = u / k, c = u % k;
#pragma unroll
    for (int B = 0; B < R; ++B) {
      const int idx = padded((B * cols + m) * k + c, pd);
      sre[idx] = re[j * R + B];
      sim[idx] = im[j * R + B];
    }
  }
}

template <int N, int p, int DIR>
__device__ __forceinline__ void smem_read_pass(const float *sre, const float *sim, int t,
                                               const float2 *__restrict__ tw, float *re, float *im) {
  using G = BlockGeom<N>;
  constexpr int R = G::R(p), k = G::K(p), J = G::RMAX / R, T = G::T;
  constexpr Pad pd = BoundaryPad<N, p - 1>::value;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int u = t + j * T, m = u / k, c = u % k;
#pragma unroll
    for (int A = 0; A < R; ++A) {
      const int idx = padded((m * R + A) * k + c, pd);
      re[j * R + A] = sre[idx];
      im[j * R + A] = sim[idx];
      pass_twiddle<N, p, DIR>(tw, m, A, re[j * R + A], im[j * R + A]);
    }
    reg_fft<R, DIR>(re + j * R, im + j * R);
  }
}

template <int N, int LAYOUT, int DIR>
__global__ void __launch_bounds__(BlockGeom<N>::THREADS)
fft_block_kernel(const BlockArgs args) {
  using G = BlockGeom<N>;
  constexpr int T = G::T, TPB = G::TPB, RM = G::RMAX, P = G::P;
  extern __shared__ float smem[];
  const int tid = threadIdx.x;
  const int f = tid / T;
  const int t = tid - f * T;
  const int64_t b = (int64_t)blockIdx.x * TPB + f;
  const bool live = b < args.batch;
  const int64_t ibase = b * args.idist, obase = b * args.odist;

  float re[RM], im[RM];
  // ---- pass 0: HBM -> registers (coalesced across t), codelet ----------
  {
    constexpr int R = G::R(0), k = G::K(0), J = RM / R;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int c = t + j * T;
#pragma unroll
      for (int A = 0; A < R; ++A) {
        if (live) {
          GIO<LAYOUT>::load(args, ibase + A * k + c, re[j * R + A], im[j * R + A]);
        } else {
          re[j * R + A] = 0.f;
          im[j * R + A] = 0.f;
        }
      }
      reg_fft<R, DIR>(re + j * R, im + j * R);
    }
  }
  if constexpr (P > 1) {
    float *sre = smem + f * (2 * SmemGeom<N>::REGION);
    float *sim = sre + SmemGeom<N>::REGION;
    smem_write<N, 0>(sre, sim, t, re, im);
    __syncthreads();
    smem_read_pass<N, 1, DIR>(sre, sim, t, args.tw, re, im);
    if constexpr (P > 2) {
      __syncthreads();
      smem_write<N, 1>(sre, sim, t, re, im);
      __syncthreads();
      smem_read_pass<N, 2, DIR>(sre, sim, t, args.tw, re, im);
    }
  }
  // ---- last pass: registers -> HBM, k == 1 so lanes over m coalesce -----
  {
    constexpr int q = P - 1;
    constexpr int R = G::R(q), cols = G::COLS(q), k = G::K(q), J = RM / R;
    if (live) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int u = t + j * T, m = u / k, c = u % k;
#pragma unroll
        for (int B = 0; B < R; ++B)
          GIO<LAYOUT>::store(args, obase + (B * cols + m) * k + c, re[j * R + B], im[j * R + B]);
      }
    }
  }
}

}  // namespace fftgen_b200
