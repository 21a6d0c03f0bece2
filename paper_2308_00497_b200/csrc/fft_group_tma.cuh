// fft_group_tma.cuh -- K3 group kernel, persistent + TMA tensor-tile variant.
//
// Same tiles, arithmetic and stores as fft_group_kernel (fft_group.cuh), but
// the CTA is persistent and its input tiles arrive by cp.async.bulk.tensor
// into a double-buffered shared stage, two tiles ahead of the one being
// computed, so the HBM reads of a pass never wait on the compute of the tile
// before (the K2 TMA kernel's schedule, fft_block.cuh, applied to the
// four-step groups).  After pass 0 has read a stage's raw tile the same stage
// holds the padded sub-FFT exchange; once pass 1 has read that, the stage is
// refilled.
//
// Raw tile layouts (what the tensor box writes):
//   columns: [A][f]  NS rows of TC adjacent elements (stride k between rows);
//            box {TC elements, <=256 rows} per 256-row chunk of A
//   rows:    [f][A]  TC rows of NS contiguous elements; box {256 floats,
//            NS*2/256 chunks, TC rows}
// split user input (group 0 only) arrives as two planes, re then im.
#pragma once

#include <cstdint>

#include "fft_group.cuh"

namespace fftgen_b200 {

#ifndef FFTGEN_GROUP_TMA_STAGES
#define FFTGEN_GROUP_TMA_STAGES 2
#endif
constexpr int kGroupTmaStages = FFTGEN_GROUP_TMA_STAGES;
// Pass-0 global twiddles of a tile fetched before its stage wait, where
// measured faster (`scripts/gpu_ab_tp.sh`): 2^18 0.427 / 0.422 -> 0.436 /
// 0.434, 2^20 / 2^21 interleaved 0.404 / 0.385 -> 0.413 / 0.392; the split
// NS = 1024 column group with tensor stores (register-bound) loses 0.5 %
// and keeps the loads after the wait.
#ifndef FFTGEN_GROUP_TWPRE
#define FFTGEN_GROUP_TWPRE 1
#endif

// Results staged in a separate output buffer ([e][f], the tile of the store
// box) and written by TMA tensor stores instead of per-lane STGs of
// TC-element segments, where measured faster (B200, 1 GiB batches,
// `scripts/gpu_ab_st.sh`, `gpu_ab_rst.sh`): the NS = 512 rows group (through
// this kernel instead of the plain one: 2^18 / 2^19 split 0.409 / 0.404 ->
// 0.426 / 0.424, interleaved 0.419 / 0.421 -> 0.423 / 0.427) and the NS = 1024
// column group of split input (2^20 / 2^21 split 0.383 / 0.363 -> 0.404 /
// 0.386).  Slower elsewhere: NS = 512 columns (2^17 0.448 -> 0.427), NS = 1024
// rows (2^20 split 0.383 -> 0.378), interleaved NS = 1024 columns (neutral).
#ifndef FFTGEN_GROUP_TMA_STORE
#define FFTGEN_GROUP_TMA_STORE 1
#endif
constexpr bool group_tma_store_rt(int ns, bool rows, int lin) {
  return FFTGEN_GROUP_TMA_STORE && (rows ? (ns == 512 || ns == 1024) : (ns == 1024 && lin == LAYOUT_SPLIT));
}
template <int NS, bool ROWS, int LIN> constexpr bool group_tma_store() { return group_tma_store_rt(NS, ROWS, LIN); }

// STAGES = 2: one CTA per SM, the tile two items ahead is in flight;
// STAGES = 1: two CTAs per SM, each refilling its stage after pass 1.
template <int NS, int STAGES_ = kGroupTmaStages, bool STORE = false> struct GroupTmaGeom {
  using GG = GroupGeom<NS>;
  static constexpr int TC = GG::TC, REG = GG::REG, THREADS = GG::THREADS;
  static constexpr int RAW = TC * NS * 8;  // raw tile bytes
  static constexpr int STAGE = ((TC * REG * 8 > RAW ? TC * REG * 8 : RAW) + 127) / 128 * 128;
  static constexpr int OUT = STORE ? RAW : 0;  // output staging buffer
  // 128 KB tiles (NS >= 2048) fit one stage: the refill overlaps the stores
  static constexpr int STAGES = STAGES_ * STAGE + OUT + 64 > 227 * 1024 ? 1 : STAGES_;
  static constexpr int BYTES = STAGES * STAGE + OUT + 64;
  static constexpr int MIN_BLOCKS = (228 * 1024) / (BYTES + 1024) > 0 ? (228 * 1024) / (BYTES + 1024) : 1;
};

FFTGEN_FI void tma_load_4d(void *dst, const void *tmap, int c0, int c1, int c2, int c3, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

FFTGEN_FI void tma_store_4d(const void *tmap, const void *src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

// store the staged results of a tile ([e][f] boxes of <= 256 rows e; split:
// the re plane, then the im plane); maps from encode_out_maps
template <int NS, int LOUT, bool ROWS>
FFTGEN_FI void group_tma_store(const GroupTmaArgs &ta, const char *out, int64_t b, int64_t m0, int64_t c0) {
  constexpr int TC = GroupTmaGeom<NS>::TC;
  constexpr int CH = NS < 256 ? NS : 256;
  constexpr int W = LOUT == LAYOUT_SPLIT ? 1 : 2;
#pragma unroll
  for (int q = 0; q < NS / CH; ++q) {
    const char *src = out + q * CH * TC * W * 4;
    if constexpr (ROWS) {  // {cols*W floats, NS, batch, 1}
      tma_store_4d(ta.omap[0], src, (int)(m0 * W), q * CH, (int)b, 0);
      if constexpr (LOUT == LAYOUT_SPLIT)
        tma_store_4d(ta.omap[1], src + NS * TC * 4, (int)m0, q * CH, (int)b, 0);
    } else {               // {k*2 floats, cols, NS, batch} (interleaved scratch)
      tma_store_4d(ta.omap[0], src, (int)(c0 * 2), (int)m0, q * CH, (int)b);
    }
  }
}

// issue the raw tile of work item `item` into `stage`
template <int NS, int LIN, bool ROWS>
FFTGEN_FI void group_tma_issue(const GroupTmaArgs &ta, char *stage, uint64_t *bar, int64_t item) {
  using TG = GroupTmaGeom<NS>;
  constexpr int TC = TG::TC;
  const GroupArgs &a = ta.g;
  const int64_t b = item / a.tiles_per_outer, tt = item - b * a.tiles_per_outer;
  mbar_expect_tx(bar, (uint32_t)TG::RAW);
  if constexpr (ROWS) {
    tma_load_4d(stage, ta.tmap[0], 0, 0, (int)(tt * TC), (int)b, bar);
  } else {
    const int64_t u0 = tt * TC, m0 = u0 / a.k, c0 = u0 - m0 * a.k;
    constexpr int CH = NS < 256 ? NS : 256;  // rows per box
    constexpr int W = LIN == LAYOUT_SPLIT ? 1 : 2;
#pragma unroll
    for (int q = 0; q < NS / CH; ++q) {
      tma_load_4d(stage + q * CH * TC * W * 4, ta.tmap[0], (int)(c0 * W), q * CH, (int)m0, (int)b, bar);
      if constexpr (LIN == LAYOUT_SPLIT)
        tma_load_4d(stage + NS * TC * 4 + q * CH * TC * 4, ta.tmap[1], (int)c0, q * CH, (int)m0, (int)b, bar);
    }
  }
}

template <int NS, int LIN, int LOUT, int DIR, bool ROWS>
__global__ void __launch_bounds__(GroupTmaGeom<NS>::THREADS,
                                  (GroupTmaGeom<NS, kGroupTmaStages, group_tma_store<NS, ROWS, LIN>()>::MIN_BLOCKS))
fft_group_tma_kernel(const __grid_constant__ GroupTmaArgs ta) {
  constexpr bool ST = group_tma_store<NS, ROWS, LIN>();
  using TG = GroupTmaGeom<NS, kGroupTmaStages, ST>;
  using G = typename TG::GG::G;
  constexpr int TC = TG::TC, REG = TG::REG, T = G::T;
  constexpr int R0 = G::R(0), K0 = G::K(0), J0 = G::RMAX / R0;
  constexpr int R1 = G::R(G::P - 1), COLS1 = G::COLS(G::P - 1);  // the last pass
  const GroupArgs &a = ta.g;
  extern __shared__ float4 smem_f4[];
  char *smem = reinterpret_cast<char *>(smem_f4);
  constexpr int NST = TG::STAGES;
  char *obuf = smem + NST * TG::STAGE;  // output staging (FFTGEN_GROUP_TMA_STORE)
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + NST * TG::STAGE + TG::OUT);
  const int tid = threadIdx.x;
  const int64_t total = ta.items, stride = gridDim.x;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < NST; ++s)
      if (blockIdx.x + s * stride < total)
        group_tma_issue<NS, LIN, ROWS>(ta, smem + s * TG::STAGE, &bars[s], blockIdx.x + s * stride);
  GroupTw<G> gtw;  // pass-1 twiddle bases of butterfly m = tid / TC, for every tile
  gtw.load(a.tw_local, tid / TC);

  int it = 0;
  for (int64_t item = blockIdx.x; item < total; item += stride, ++it) {
    const int s = NST == 2 ? (it & 1) : 0;
    char *stage = smem + s * TG::STAGE;
    float2 *X = reinterpret_cast<float2 *>(stage);
    const int64_t b = item / a.tiles_per_outer, tt = item - b * a.tiles_per_outer;
    int64_t m0, c0;
    if (ROWS) {
      m0 = tt * TC;
      c0 = 0;
    } else {
      const int64_t u0 = tt * TC;
      m0 = u0 / a.k;
      c0 = u0 - m0 * a.k;
    }
    const int f0 = ROWS ? tid / T : tid % TC;
    const int t0 = ROWS ? tid % T : tid / TC;
    // this tile's pass-0 global twiddles, fetched before the stage wait
    constexpr bool kPre = FFTGEN_GROUP_TWPRE && (ROWS || !ST) && !group_q_pq<NS, R0, ROWS, LOUT>();
    float2 pre_p[kPre ? J0 : 1], pre_q[kPre ? R0 : 1];
    if constexpr (kPre) {
      if (a.cols > 1) {
        const int64_t m = ROWS ? m0 + f0 : m0;
#pragma unroll
        for (int j = 0; j < J0; ++j) {
          const int c = t0 + j * T;
          pre_p[j] = __ldg(ROWS ? a.tw_p + m * K0 + c : a.tw_p + c * a.cols + m);
        }
#pragma unroll
        for (int A0 = 1; A0 < R0; ++A0) pre_q[A0] = __ldg(a.tw_q + m + A0 * a.cols);
      }
    }
    mbar_wait(&bars[s], (NST == 2 ? (it >> 1) : it) & 1);

    // ---- pass 0: raw tile -> registers, global twiddle, radix-R0 codelets ----
    float2 v[G::RMAX];
    {
      const int64_t m = ROWS ? m0 + f0 : m0;
      const bool tw = a.cols > 1;
      const float2 *qm = a.tw_q + m;
      QFact<R0, group_q_pq<NS, R0, ROWS, LOUT>()> qf;
      if (tw) qf.load(qm, a.cols);
#pragma unroll
      for (int j = 0; j < J0; ++j) {
        const int c = t0 + j * T;
#pragma unroll
        for (int A0 = 0; A0 < R0; ++A0) {
          const int A = A0 * K0 + c;
          const int e = ROWS ? f0 * NS + A : A * TC + f0;
          if constexpr (LIN == LAYOUT_SPLIT) {
            const float *sp = reinterpret_cast<const float *>(stage);
            v[j * R0 + A0] = make_float2(sp[e], sp[NS * TC + e]);
          } else {
            v[j * R0 + A0] = X[e];
          }
        }
        if (tw) {
          const float2 pw = kPre ? pre_p[kPre ? j : 0] : __ldg(ROWS ? a.tw_p + m * K0 + c : a.tw_p + c * a.cols + m);
#pragma unroll
          for (int A0 = 0; A0 < R0; ++A0) {
            float2 x = mul_tw<DIR>(v[j * R0 + A0], pw);
            v[j * R0 + A0] = A0 ? (kPre ? mul_tw<DIR>(x, pre_q[kPre ? A0 : 0]) : qf.template apply<DIR>(x, qm, a.cols, A0)) : x;
          }
        }
        reg_fft<R0, DIR>(v + j * R0);
      }
    }
    __syncthreads();  // raw tile consumed: the stage becomes the padded exchange
    smem_write<G, NS, 0>(X + f0 * REG, t0, v);
    __syncthreads();

    // ---- pass 1: exchange -> registers (lanes over f), codelet, HBM store ----
    const int f = tid % TC;
    const int t = tid / TC;
    group_passes_rest<G, NS, DIR, 0, TG::THREADS>(X + f * REG, t, a.tw_local, v, gtw);
    if constexpr (ST)
      if (tid == 0) bulk_wait_read0();  // the previous tile's store has read obuf
    __syncthreads();  // stage free: fetch the tile two items ahead
    if (tid == 0 && item + NST * stride < total) {
      fence_proxy_async();
      group_tma_issue<NS, LIN, ROWS>(ta, stage, &bars[s], item + NST * stride);
    }
    if constexpr (ST) {
    // [e][f] rows of the store box: lanes of a warp write 32 consecutive elements
#pragma unroll
    for (int B = 0; B < R1; ++B) {
      const int e = B * COLS1 + t;
      if constexpr (LOUT == LAYOUT_SPLIT) {
        float *o = reinterpret_cast<float *>(obuf);
        o[e * TC + f] = v[B].x;
        o[NS * TC + e * TC + f] = v[B].y;
      } else {
        reinterpret_cast<float2 *>(obuf)[e * TC + f] = v[B];
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      group_tma_store<NS, LOUT, ROWS>(ta, obuf, b, m0, c0);
      bulk_commit();
    }
    } else {
    (void)obuf;
    const int64_t ob = b * a.odist;
#pragma unroll
    for (int B = 0; B < R1; ++B) {
      const int64_t e = B * COLS1 + t;
      const int64_t off = ROWS ? e * a.cols + m0 + f : (e * a.cols + m0) * a.k + c0 + f;
      SIO<LOUT>::store(a.out0, a.out1, ob + off, v[B]);
    }
    }
  }
  if constexpr (ST)
    if (tid == 0) bulk_wait0();
}

// ---- NS >= 2^11: one raw stage + an fp32 exchange plane --------------------
// The 128 KB tiles of the 2^11 / 2^12 groups leave room for one raw stage
// only; exchanging through the stage itself (fft_group_tma_kernel) delays the
// next tile's TMA load until pass 1 has read the exchange.  Here the exchange
// goes through a separate padded fp32 plane (re, then im: the 2^14 block
// kernel's schedule), so the stage is refilled right after pass 0 and the
// load overlaps the exchange, pass 1 and the stores.
#ifndef FFTGEN_PLANE_MIN_LOG2
#define FFTGEN_PLANE_MIN_LOG2 11
#endif
#ifndef FFTGEN_GROUP_PLANE
#define FFTGEN_GROUP_PLANE 1
#endif

// Plane kernel results by TMA tensor stores, staged through the exchange plane
// in two halves (split: the re plane, then the im plane; interleaved: output
// rows e < NS/2, then the rest) instead of per-lane STGs, where measured
// faster (B200, `scripts/gpu_ab_ps.sh`): every column group and NS = 4096
// rows (2^23 / 2^24 interleaved two-pass 0.334 / 0.310 -> 0.364 / 0.330,
// 2^24 batch 1 0.146 -> 0.137 ms) and NS = 2048 rows of split output (2^21
// split 0.381 -> 0.389); NS = 2048 rows of interleaved output lose (2^21 /
// 2^22 0.385 / 0.396 -> 0.379 / 0.390) and keep the register stores.
#ifndef FFTGEN_PLANE_STORE
#define FFTGEN_PLANE_STORE 1
#endif
constexpr bool group_plane_store_rt(int ns, bool rows, int lout) {
  return FFTGEN_PLANE_STORE && (!rows || ns == 4096 || lout == LAYOUT_SPLIT);
}

// half h of a tile's results, staged in src as [e][f] (<= 256-row boxes)
template <int NS, int LOUT, bool ROWS>
FFTGEN_FI void group_tma_store_half(const GroupTmaArgs &ta, const char *src, int64_t b, int64_t m0, int64_t c0,
                                    int h) {
  constexpr int TC = GroupGeom<NS>::TC;
  constexpr int CH = 256;
  if constexpr (LOUT == LAYOUT_SPLIT) {  // rows only: plane h over all NS rows
#pragma unroll
    for (int q = 0; q < NS / CH; ++q)
      tma_store_4d(ta.omap[h], src + q * CH * TC * 4, (int)m0, q * CH, (int)b, 0);
  } else {
#pragma unroll
    for (int q = 0; q < NS / 2 / CH; ++q) {
      const int e0 = h * (NS / 2) + q * CH;
      if constexpr (ROWS)
        tma_store_4d(ta.omap[0], src + q * CH * TC * 8, (int)(m0 * 2), e0, (int)b, 0);
      else
        tma_store_4d(ta.omap[0], src + q * CH * TC * 8, (int)(c0 * 2), (int)m0, e0, (int)b);
    }
  }
}

// the tile's factored pass-0 twiddle bases fetched before the stage wait
// (`scripts` A/B: 2^22 split 0.371 -> 0.374, 2^24 interleaved 0.342-0.347 ->
// 0.347-0.357, the rest within 0.5 %)
#ifndef FFTGEN_PLANE_TWPRE
#define FFTGEN_PLANE_TWPRE 1
#endif

template <int NS> struct GroupPlaneGeom {
  using GG = GroupGeom<NS>;
  using PL = typename GG::PL;
  using G = typename GG::G;
  static constexpr int TC = GG::TC, THREADS = GG::THREADS;
  static constexpr Pad PAD = BoundaryPad<NS, 0, 4, PL>::value;
  static constexpr int EXP = padded(NS - 1, PAD) + 1;  // plane floats per column
  static constexpr int REGP = GroupRegSearch<NS, TC, PL, 4>::best(EXP | 1);
  static constexpr int RAW = TC * NS * 8;
  static constexpr int PLANE = (TC * REGP * 4 + 127) / 128 * 128;
  static constexpr int BYTES = RAW + PLANE + 64;
  static constexpr bool ENABLED = NS >= (1 << FFTGEN_PLANE_MIN_LOG2) && G::P == 2 && BYTES <= 227 * 1024;
  static constexpr int MIN_BLOCKS = (228 * 1024) / (BYTES + 1024) > 1 ? 2 : 1;
};

template <int NS, int LIN, int LOUT, int DIR, bool ROWS>
__global__ void __launch_bounds__(GroupPlaneGeom<NS>::THREADS, GroupPlaneGeom<NS>::MIN_BLOCKS)
fft_group_plane_kernel(const __grid_constant__ GroupTmaArgs ta) {
  using PG = GroupPlaneGeom<NS>;
  using G = typename PG::G;
  static_assert(PG::ENABLED, "plane-exchange group kernel: NS >= 2^FFTGEN_PLANE_MIN_LOG2, two passes");
  constexpr bool PST = group_plane_store_rt(NS, ROWS, LOUT);
  static_assert(!PST || (PG::PLANE >= NS * PG::TC * 4 && NS / 2 >= 256), "a result half fits the plane");
  static_assert(GroupTmaGeom<NS>::RAW == PG::RAW, "same raw tile as the TMA issue helper");
  constexpr int TC = PG::TC, T = G::T, REGP = PG::REGP;
  constexpr int R0 = G::R(0), K0 = G::K(0), J0 = G::RMAX / R0;
  constexpr int R1 = G::R(1), COLS1 = G::COLS(1);
  const GroupArgs &a = ta.g;
  extern __shared__ float4 smem_f4[];
  char *stage = reinterpret_cast<char *>(smem_f4);
  float *P = reinterpret_cast<float *>(stage + PG::RAW);
  uint64_t *bar = reinterpret_cast<uint64_t *>(stage + PG::RAW + PG::PLANE);
  const int tid = threadIdx.x;
  const int64_t total = ta.items, stride = gridDim.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x < total) group_tma_issue<NS, LIN, ROWS>(ta, stage, bar, blockIdx.x);
  GroupTw<G> gtw;  // pass-1 twiddle bases (fft_group.cuh, FFTGEN_GROUP_PQ)
  gtw.load(a.tw_local, tid / TC);
  int it = 0;
  for (int64_t item = blockIdx.x; item < total; item += stride, ++it) {
    const int64_t b = item / a.tiles_per_outer, tt = item - b * a.tiles_per_outer;
    int64_t m0, c0;
    if (ROWS) {
      m0 = tt * TC;
      c0 = 0;
    } else {
      const int64_t u0 = tt * TC;
      m0 = u0 / a.k;
      c0 = u0 - m0 * a.k;
    }
    const int f0 = ROWS ? tid / T : tid % TC;
    const int t0 = ROWS ? tid % T : tid / TC;
    const int64_t m = ROWS ? m0 + f0 : m0;
    const bool tw = a.cols > 1;
    const float2 *qm = a.tw_q + m;
    QFact<R0, group_q_pq<NS, R0, ROWS, LOUT>()> qf;
    if constexpr (FFTGEN_PLANE_TWPRE)  // this tile's factored twiddle bases before the stage wait
      if (tw) qf.load(qm, a.cols);
    mbar_wait(bar, it & 1);
    // ---- pass 0: raw tile -> registers, global twiddle, radix-R0 codelets ----
    float2 v[G::RMAX];
    {
      if constexpr (!FFTGEN_PLANE_TWPRE)
        if (tw) qf.load(qm, a.cols);
#pragma unroll
      for (int j = 0; j < J0; ++j) {
        const int c = t0 + j * T;
#pragma unroll
        for (int A0 = 0; A0 < R0; ++A0) {
          const int A = A0 * K0 + c;
          const int e = ROWS ? f0 * NS + A : A * TC + f0;
          if constexpr (LIN == LAYOUT_SPLIT) {
            const float *sp = reinterpret_cast<const float *>(stage);
            v[j * R0 + A0] = make_float2(sp[e], sp[NS * TC + e]);
          } else {
            v[j * R0 + A0] = reinterpret_cast<const float2 *>(stage)[e];
          }
        }
        if constexpr (PST)  // the previous tile's second-half store has read the plane
          if (j == 0 && tid == 0) bulk_wait_read0();
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
    }
    __syncthreads();  // raw tile consumed: fetch the next one behind the exchange
    if (tid == 0 && item + stride < total) {
      fence_proxy_async();
      group_tma_issue<NS, LIN, ROWS>(ta, stage, bar, item + stride);
    }
    // ---- exchange through the plane (re, then im) and pass 1 ----------------
    const int f = tid % TC, t = tid / TC;
    plane_write<G, NS, 0, 0>(P + f0 * REGP, t0, v);
    __syncthreads();
    plane_read<G, NS, 1, 0>(P + f * REGP, t, v);
    __syncthreads();
    plane_write<G, NS, 0, 1>(P + f0 * REGP, t0, v);
    __syncthreads();
    plane_read<G, NS, 1, 1>(P + f * REGP, t, v);
    if constexpr (group_pq<G>()) {
#pragma unroll
      for (int A = 1; A < R1; ++A) v[A] = gtw.pq.template apply<DIR>(v[A], A);
      reg_fft<R1, DIR>(v);
    } else {
      pass_compute<G, 1, DIR>(t, a.tw_local, v);
    }
    if constexpr (PST) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        __syncthreads();  // pass-1 plane reads (h = 0) / the first half's store read (h = 1) done
        if constexpr (LOUT == LAYOUT_SPLIT) {
#pragma unroll
          for (int B = 0; B < R1; ++B) P[(B * COLS1 + t) * TC + f] = h ? v[B].y : v[B].x;
        } else {
          float2 *P2 = reinterpret_cast<float2 *>(P);
#pragma unroll
          for (int B = h * (R1 / 2); B < (h + 1) * (R1 / 2); ++B)
            P2[(B * COLS1 + t - h * (NS / 2)) * TC + f] = v[B];
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
          group_tma_store_half<NS, LOUT, ROWS>(ta, reinterpret_cast<const char *>(P), b, m0, c0, h);
          bulk_commit();
          if (h == 0) bulk_wait_read0();
        }
      }
    } else {
      const int64_t ob = b * a.odist;
#pragma unroll
      for (int B = 0; B < R1; ++B) {
        const int64_t e = B * COLS1 + t;
        const int64_t off = ROWS ? e * a.cols + m0 + f : (e * a.cols + m0) * a.k + c0 + f;
        SIO<LOUT>::store(a.out0, a.out1, ob + off, v[B]);
      }
    }
    // the next iteration's plane writes follow its post-pass-0 barrier
  }
  if constexpr (PST)
    if (tid == 0) bulk_wait0();
}

}  // namespace fftgen_b200
