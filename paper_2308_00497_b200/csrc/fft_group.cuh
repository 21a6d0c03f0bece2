// fft_group.cuh -- K3: four-step / multi-group Stockham FFT for N > 2^14.
//
// The reference's Stockham stage list (formula.cpp:168-197) is cut into G
// groups (2 <= G <= 4) of consecutive stages; group g is ONE radix-NS_g
// Stockham stage over the whole transform (global s = cols*NS, k = N/s):
//
//   y[(B cols + m) k + c] = DFT_NS( x[(m NS + A) k + c] * w_s^{A m} )[B]
//
// executed by one kernel launch.  This is the reference's Eq.-1 split
// DFT_N = (DFT_N1 (x) I) D^N (I (x) DFT_N2) Pi (formula.hpp:102-106) applied
// recursively, with the stride permutations folded into addressing and the
// twiddle diagonal D folded into pass 0 of the next group.
//
// A CTA owns a tile of TC transforms that are ADJACENT in memory:
//   inner groups (k >= TC): same m, consecutive c  -> columns of stride k
//   last group  (k == 1):   consecutive m          -> contiguous rows
// The tile is staged through shared memory so that every HBM access covers
// TC consecutive elements (TC*8 bytes interleaved, TC*4 per split plane):
//   load:  lanes over c (columns) or over A (rows)
//   store: lanes over c or m -- the transposed store of the last group
// In between, the NS-point sub-FFT runs on the block-kernel machinery
// (registers + padded smem exchange, fft_block.cuh), and the global twiddle
// w_s^{A m} = w_s^{A0 (NS/R0) m} * w_s^{c m} (A = A0 (NS/R0) + c, R0 = the
// sub-FFT's first pass radix) comes from two fp64-exact fp32 tables
// Q[A0][m], P[c][m] built at plan time.
#pragma once

#include <cstdint>

#include "fft_block.cuh"

namespace fftgen_b200 {

template <int L> struct SIO;
template <> struct SIO<LAYOUT_INTERLEAVED> {
  static FFTGEN_FI float2 load(const void *p0, const void *, int64_t off) {
    return __ldcs(reinterpret_cast<const float2 *>(p0) + off);
  }
  static FFTGEN_FI void store(void *p0, void *, int64_t off, float2 v) {
    __stcs(reinterpret_cast<float2 *>(p0) + off, v);
  }
};
template <> struct SIO<LAYOUT_SPLIT> {
  static FFTGEN_FI float2 load(const void *p0, const void *p1, int64_t off) {
    return make_float2(__ldcs(reinterpret_cast<const float *>(p0) + off),
                       __ldcs(reinterpret_cast<const float *>(p1) + off));
  }
  static FFTGEN_FI void store(void *p0, void *p1, int64_t off, float2 v) {
    __stcs(reinterpret_cast<float *>(p0) + off, v.x);
    __stcs(reinterpret_cast<float *>(p1) + off, v.y);
  }
};

template <int NS, int LIN, int LOUT, int DIR, bool ROWS>
__global__ void __launch_bounds__(GroupGeom<NS>::THREADS) fft_group_kernel(const GroupArgs a) {
  using GG = GroupGeom<NS>;
  using G = typename GG::G;
  constexpr int TC = GG::TC, REG = GG::REG, THREADS = GG::THREADS;
  extern __shared__ float4 smem_f4[];
  float2 *stage = reinterpret_cast<float2 *>(smem_f4);
  const int tid = threadIdx.x;

  const int64_t b = blockIdx.x / a.tiles_per_outer;
  const int64_t tt = blockIdx.x - b * a.tiles_per_outer;
  int64_t m0, c0;
  if (ROWS) {
    m0 = tt * TC;
    c0 = 0;
  } else {
    const int64_t u0 = tt * TC;
    m0 = u0 / a.k;
    c0 = u0 - m0 * a.k;
  }
  const int64_t ib = b * a.idist, ob = b * a.odist;

  // ---- cooperative, coalesced tile load (HBM -> smem) --------------------
  // All ITER loads of a thread are issued before the first shared store so
  // each thread keeps ITER independent HBM requests in flight.
  constexpr int ITER = TC * NS / THREADS;
  static_assert(ITER * THREADS == TC * NS, "tile must divide evenly");
  {
    float2 ld[ITER];
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int i = tid + it * THREADS;
      if (ROWS) {  // k == 1: transform f is the contiguous row m0 + f
        const int f = i / NS, A = i % NS;
        ld[it] = SIO<LIN>::load(a.in0, a.in1, ib + (m0 + f) * NS + A);
      } else {     // columns: element A of transform f at (m0 NS + A) k + c0 + f
        const int f = i % TC, A = i / TC;
        ld[it] = SIO<LIN>::load(a.in0, a.in1, ib + (m0 * NS + A) * a.k + c0 + f);
      }
    }
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int i = tid + it * THREADS;
      if (ROWS)
        stage[(i / NS) * REG + i % NS] = ld[it];
      else
        stage[(i % TC) * REG + i / TC] = ld[it];
    }
  }
  __syncthreads();

  // ---- pass 0 with the global twiddle w_s^{A m}, then the local passes ----
  const int f = tid / G::T;
  const int t = tid - f * G::T;
  const int64_t m = ROWS ? m0 + f : m0;
  float2 *sx = stage + f * REG;
  float2 v[G::RMAX];
  {
    constexpr int R = G::R(0), k = G::K(0), J = G::RMAX / R;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int c = t + j * G::T;
      float2 pw = make_float2(1.f, 0.f);
      if (a.cols > 1) pw = __ldg(a.tw_p + c * a.cols + m);
#pragma unroll
      for (int A0 = 0; A0 < R; ++A0) {
        float2 x = sx[A0 * k + c];
        if (a.cols > 1) {
          x = mul_tw<DIR>(x, pw);
          if (A0) x = mul_tw<DIR>(x, __ldg(a.tw_q + A0 * a.cols + m));
        }
        v[j * R + A0] = x;
      }
      reg_fft<R, DIR>(v + j * R);
    }
  }
  __syncthreads();  // staged input consumed; the region becomes the exchange
  if constexpr (G::P == 2) {
    TwPQ<G> pq;
    pq.load(a.tw_local, t);
    smem_write<G, NS, 0>(sx, t, v);
    __syncthreads();
    smem_read_pass1_pq<G, NS, DIR>(sx, t, pq, v);
  } else {
    middle_passes<G, NS, DIR>(sx, t, a.tw_local, v);
  }
  __syncthreads();  // exchange consumed; stage the outputs in natural order
  {
    constexpr int q = G::P - 1;
    constexpr int R = G::R(q), cols = G::COLS(q), k = G::K(q), J = G::RMAX / R;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int u = t + j * G::T, mm = u / k, c = u % k;
#pragma unroll
      for (int B = 0; B < R; ++B) sx[(B * cols + mm) * k + c] = v[j * R + B];
    }
  }
  __syncthreads();

  // ---- cooperative, coalesced tile store (smem -> HBM), lanes over f ------
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int i = tid + it * THREADS;
    const int ff = i % TC, B = i / TC;
    const int64_t off = ROWS ? (int64_t)B * a.cols + m0 + ff : ((int64_t)B * a.cols + m0) * a.k + c0 + ff;
    SIO<LOUT>::store(a.out0, a.out1, ob + off, stage[ff * REG + B]);
  }
}

}  // namespace fftgen_b200
