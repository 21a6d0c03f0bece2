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
// The NS-point sub-FFT is two register passes with one padded shared-memory
// exchange (block_geom.hpp).  HBM is read by pass 0 and written by pass 1
// straight from registers; coalescing comes from the thread mapping, which
// is chosen per side of the exchange:
//   columns: lanes over the tile index f on both sides (TC*8-byte segments)
//   rows:    pass 0 lanes over the row (contiguous loads); pass 1 lanes over
//            f, so the last group's transposed natural-order store covers TC
//            consecutive m per segment.
// The global twiddle w_s^{A m} = w_s^{A0 (NS/R0) m} * w_s^{c m}
// (A = A0 (NS/R0) + c, R0 = the sub-FFT's first pass radix) comes from two
// fp64-exact fp32 tables Q[A0][m], P[c][m] (generated on the device at plan
// time); the lanes of a warp share m, so the Q reads are L1 broadcasts.
// Registers are capped (MIN_BLOCKS) so two 512-thread CTAs stay resident.
#pragma once

#include <cstdint>

#include "fft_block.cuh"

namespace fftgen_b200 {

// Interleaved scratch between groups (LAYOUT_SCRATCH) streams like the user
// buffers: measured on B200, keeping it L2-resident (two-stream chunked
// execution, or both groups in one cooperative launch with per-chunk
// dependencies) kept DRAM traffic at 16 N but lost to the extra launches,
// tails and barriers (2^16: 0.29-0.45 vs 0.46-0.51 of the single-pass roofline).
constexpr int LAYOUT_SCRATCH = 2;

template <int L> struct SIO;
template <> struct SIO<LAYOUT_INTERLEAVED> {
  static FFTGEN_FI float2 load(const void *p0, const void *, int64_t off) {
    return __ldcs(reinterpret_cast<const float2 *>(p0) + off);
  }
  static FFTGEN_FI void store(void *p0, void *, int64_t off, float2 v) {
    __stcs(reinterpret_cast<float2 *>(p0) + off, v);
  }
};
template <> struct SIO<LAYOUT_SCRATCH> {
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

// Barrier among the THREADS compute threads: __syncthreads (BARID 0) or a
// named barrier when a scheduler warp shares the CTA.
template <int BARID, int THREADS> FFTGEN_FI void compute_sync() {
  if constexpr (BARID == 0)
    __syncthreads();
  else
    asm volatile("bar.sync %0, %1;" ::"n"(BARID), "n"(THREADS) : "memory");
}

// One tile of one group: TC adjacent transforms (tile index tt) of the
// transform whose input / output start at element offsets ib / ob.
// Factored pass-1 twiddles for the 2-pass group sub-FFTs of NS >= 2^11: the
// last pass has k == 1, so thread t's butterfly m = t is the same for every
// tile and its 63 twiddles w^{A m} are products Q[a] P[b] of 14 base values
// (TwPQ, the 2-pass K2 scheme) held in registers instead of table loads per
// tile.  Every kernel of a given NS (plain, TMA, plane) uses the same form,
// so their results stay bitwise equal.  Measured on B200 (1 GiB batches):
// 2^21 / 2^22 0.338 / 0.302 -> 0.364 / 0.360 split, 0.363 / 0.329 -> 0.385 /
// 0.396 interleaved; for NS <= 1024 (16 / 32-point pass 1) it was slower
// (2^17 0.450 / 0.471 -> 0.433 / 0.448, 2^23 three-pass 1.13 -> 1.21 ms).
#ifndef FFTGEN_GROUP_PQ
#define FFTGEN_GROUP_PQ 1
#endif
#ifndef FFTGEN_GROUP_PQ_MIN
#define FFTGEN_GROUP_PQ_MIN 2048
#endif
template <class G> constexpr bool group_pq() {
  return FFTGEN_GROUP_PQ && G::P == 2 && G::S(G::P - 1) >= FFTGEN_GROUP_PQ_MIN;
}
template <class G, bool ON = group_pq<G>()> struct GroupTw;
template <class G> struct GroupTw<G, true> {
  TwPQ<G> pq;
  FFTGEN_FI void load(const float2 *__restrict__ tw, int m) { pq.load(tw, m); }
};
template <class G> struct GroupTw<G, false> {
  FFTGEN_FI void load(const float2 *__restrict__, int) {}
};

// Pass-0 global twiddles Q[A0][m] = w_s^{A0 (NS/R0) m} as products of two
// loaded bases, Q[A0 % 8] * Q[8 (A0 / 8)] (14 loads per tile and thread
// instead of R0 - 1 for the 32 / 64-point first passes of NS >= 2^11).
// Every kernel of a given shape uses the same form (results bitwise equal).
// Measured (`scripts/gpu_ab_qpq.sh`): 2^23 interleaved 0.373 -> 0.390, 2^22
// 0.370 / 0.398 -> 0.375 / 0.404, 2^24 interleaved 0.344 -> 0.351.
#ifndef FFTGEN_GROUP_Q_PQ_MIN
#define FFTGEN_GROUP_Q_PQ_MIN 2048
#endif
// (the NS = 4096 rows group of split output ran 2.3x slower with it: excluded)
template <int NS, int R0, bool ROWS, int LOUT> constexpr bool group_q_pq() {
  return NS >= FFTGEN_GROUP_Q_PQ_MIN && R0 >= 16 && !(ROWS && LOUT == LAYOUT_SPLIT && NS >= 4096);
}
template <int R0, bool ON> struct QFact {
  FFTGEN_FI void load(const float2 *, int64_t) {}
  template <int DIR> FFTGEN_FI float2 apply(float2 x, const float2 *__restrict__ qm, int64_t cols, int A0) const {
    return mul_tw<DIR>(x, __ldg(qm + A0 * cols));
  }
};
template <int R0> struct QFact<R0, true> {
  float2 lo[8], hi[R0 / 8];
  FFTGEN_FI void load(const float2 *__restrict__ qm, int64_t cols) {
#pragma unroll
    for (int b = 1; b < 8; ++b) lo[b] = __ldg(qm + b * cols);
#pragma unroll
    for (int a = 1; a < R0 / 8; ++a) hi[a] = __ldg(qm + 8 * a * cols);
  }
  template <int DIR> FFTGEN_FI float2 apply(float2 x, const float2 *__restrict__, int64_t, int A0) const {
    const int a = A0 / 8, b = A0 % 8;
    if (b) x = mul_tw<DIR>(x, lo[b]);
    if (a) x = mul_tw<DIR>(x, hi[a]);
    return x;
  }
};

// Passes 1 .. P-1 of a group sub-FFT whose pass-0 results sit in the padded
// exchange (this column at Xf); lanes run over the tile's columns, thread t
// owns the pass-p butterflies t + j T.
template <class G, int NS, int DIR, int BARID, int THREADS>
FFTGEN_FI void group_passes_rest(float2 *Xf, int t, const float2 *__restrict__ tw, float2 *v) {
  smem_read_pass<G, NS, 1, DIR>(Xf, t, tw, v);
  if constexpr (G::P == 3) {
    compute_sync<BARID, THREADS>();  // pass-1 reads done before the rewrite
    smem_write<G, NS, 1>(Xf, t, v);
    compute_sync<BARID, THREADS>();
    smem_read_pass<G, NS, 2, DIR>(Xf, t, tw, v);
  }
}

template <class G, int NS, int DIR, int BARID, int THREADS, bool ON>
FFTGEN_FI void group_passes_rest(float2 *Xf, int t, const float2 *__restrict__ tw, float2 *v, const GroupTw<G, ON> &gt) {
  if constexpr (ON) {
    smem_read_pass1_pq<G, NS, DIR>(Xf, t, gt.pq, v);
    return;
  }
  group_passes_rest<G, NS, DIR, BARID, THREADS>(Xf, t, tw, v);
}

template <int NS, int LIN, int LOUT, int DIR, bool ROWS, class GG = GroupGeom<NS>, int BARID = 0>
FFTGEN_FI void group_tile(const GroupArgs &a, int64_t ib, int64_t ob, int64_t tt, float2 *smem) {
  using G = typename GG::G;
  constexpr int TC = GG::TC, REG = GG::REG, T = G::T;
  static_assert((G::P == 2 || G::P == 3) && G::K(G::P - 1) == 1 && G::RMAX == G::R(G::P - 1),
                "group sub-FFTs: 2 or 3 register passes, the last one a full-width stage");
  constexpr int R0 = G::R(0), K0 = G::K(0), J0 = G::RMAX / R0;
  constexpr int R1 = G::R(G::P - 1), COLS1 = G::COLS(G::P - 1);  // the last pass
  const int tid = threadIdx.x;
  GroupTw<G> gtw;  // pass-1 twiddle bases of butterfly m = tid / TC (issued early)
  gtw.load(a.tw_local, tid / TC);
  int64_t m0, c0;
  if (ROWS) {
    m0 = tt * TC;
    c0 = 0;
  } else {
    const int64_t u0 = tt * TC;
    m0 = u0 / a.k;
    c0 = u0 - m0 * a.k;
  }

  // ---- pass 0: HBM -> registers, global twiddle, radix-R0 codelets --------
  float2 v[G::RMAX];
  {
    const int f = ROWS ? tid / T : tid % TC;
    const int t = ROWS ? tid % T : tid / TC;
    const int64_t m = ROWS ? m0 + f : m0;
    const bool tw = a.cols > 1;
    // Q[A0][m]: one address per warp (m is shared by the lanes) -> L1 broadcast
    const float2 *qm = a.tw_q + m;
    QFact<R0, group_q_pq<NS, R0, ROWS, LOUT>()> qf;
    if (tw) qf.load(qm, a.cols);
#pragma unroll
    for (int j = 0; j < J0; ++j) {
      const int c = t + j * T;
#pragma unroll
      for (int A0 = 0; A0 < R0; ++A0) {
        const int A = A0 * K0 + c;
        const int64_t off = ROWS ? ib + (m0 + f) * NS + A : ib + (m0 * NS + A) * a.k + c0 + f;
        v[j * R0 + A0] = SIO<LIN>::load(a.in0, a.in1, off);
      }
      if (tw) {
        const float2 pw = __ldg(ROWS ? a.tw_p + m * K0 + c : a.tw_p + c * a.cols + m);
#pragma unroll
        for (int A0 = 0; A0 < R0; ++A0) {
          float2 x = mul_tw<DIR>(v[j * R0 + A0], pw);
          v[j * R0 + A0] = A0 ? qf.template apply<DIR>(x, qm, a.cols, A0) : x;
        }
      }
      reg_fft<R0, DIR>(v + j * R0);
    }
    smem_write<G, NS, 0>(smem + f * REG, t, v);
  }
  compute_sync<BARID, GG::THREADS>();

  // ---- pass 1: smem -> registers (lanes over f), codelet, HBM store ------
  {
    const int f = tid % TC;
    const int t = tid / TC;  // pass-1 butterfly m1 = t (k == 1, J == 1)
    // local pass twiddles w^{A t}: lanes share t -> L1 broadcast loads
    group_passes_rest<G, NS, DIR, BARID, GG::THREADS>(smem + f * REG, t, a.tw_local, v, gtw);
#pragma unroll
    for (int B = 0; B < R1; ++B) {
      const int64_t e = B * COLS1 + t;  // local output index
      const int64_t off = ROWS ? e * a.cols + m0 + f : (e * a.cols + m0) * a.k + c0 + f;
      SIO<LOUT>::store(a.out0, a.out1, ob + off, v[B]);
    }
  }
}

template <int NS, int LIN, int LOUT, int DIR, bool ROWS>
__global__ void __launch_bounds__(GroupGeom<NS>::THREADS, GroupGeom<NS>::MIN_BLOCKS)
fft_group_kernel(const GroupArgs a) {
  extern __shared__ float4 smem_f4[];
  const int64_t b = blockIdx.x / a.tiles_per_outer;
  const int64_t tt = blockIdx.x - b * a.tiles_per_outer;
  group_tile<NS, LIN, LOUT, DIR, ROWS, GroupGeom<NS>, 0>(
      a, b * a.idist, b * a.odist, tt, reinterpret_cast<float2 *>(smem_f4));
}

}  // namespace fftgen_b200
