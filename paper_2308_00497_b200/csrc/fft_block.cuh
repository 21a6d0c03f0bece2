// fft_block.cuh -- K2: batched, shared-memory-resident Stockham FFT (sm_100a).
//
// A CTA owns whole transforms.  The reference's Stockham stage list
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
//   * the FusedMKIV butterflies are the packed fp32x2 register codelets
//     (codelets.cuh),
//   * HBM is touched exactly once on load (pass 0) and once on store (pass
//     P-1): 16 N bytes per transform, the roofline's algorithmic traffic.
// Between passes the data crosses shared memory once as float2 with a padding
// chosen at compile time (block_geom.hpp) so writer and reader are
// conflict-free.
//
// Two variants:
//   fft_block_kernel      one CTA per TPB transforms, HBM -> registers directly
//                         (any alignment / dist; all N <= 2^14)
//   fft_block_tma_kernel  persistent; the next group's input is fetched by
//                         cp.async.bulk (TMA) into a double-buffered stage while
//                         the current group computes, so HBM latency is off the
//                         critical path (16-byte aligned data, 256 <= N <= 8192)
#pragma once

#include <cstdint>

#include "block_geom.hpp"
#include "codelets.cuh"
#include "kernels.hpp"

namespace fftgen_b200 {

template <int LAYOUT> struct GIO;
template <> struct GIO<LAYOUT_INTERLEAVED> {
  static FFTGEN_FI float2 load(const BlockArgs &a, int64_t off) {
    return __ldcs(reinterpret_cast<const float2 *>(a.in0) + off);
  }
  static FFTGEN_FI void store(const BlockArgs &a, int64_t off, float2 v) {
    __stcs(reinterpret_cast<float2 *>(a.out0) + off, v);
  }
};
template <> struct GIO<LAYOUT_SPLIT> {
  static FFTGEN_FI float2 load(const BlockArgs &a, int64_t off) {
    return make_float2(__ldcs(reinterpret_cast<const float *>(a.in0) + off),
                       __ldcs(reinterpret_cast<const float *>(a.in1) + off));
  }
  static FFTGEN_FI void store(const BlockArgs &a, int64_t off, float2 v) {
    __stcs(reinterpret_cast<float *>(a.out0) + off, v.x);
    __stcs(reinterpret_cast<float *>(a.out1) + off, v.y);
  }
};

// ---- pass building blocks (G = BlockGeom<N, TP>) -----------------------
#ifndef FFTGEN_K2_TWCACHE
#define FFTGEN_K2_TWCACHE 1
#endif
// also for a factored last pass (2^14: split 0.722 / interleaved 0.714 vs
// 0.667 / 0.695 with one hi * lo product per element)
// 2^14 interleaved: pass-1 bases fetched before the stage wait (0.726 vs
// 0.715; split 0.715 vs 0.724, so split fetches them after the pass-0 write)
#ifndef FFTGEN_TMA1_EARLY_TW
#define FFTGEN_TMA1_EARLY_TW 1
#endif
// 2^14: the last pass computed and stored butterfly by butterfly, so the
// bulk stores of butterfly 0's results drain while butterfly 1 is computed
// (0.768 / 0.777 vs 0.720 / 0.723 for the two-halves epilogue, which waits
// for the first half's store to read the plane before staging the second)
#ifndef FFTGEN_TMA1_SPLITJ
#define FFTGEN_TMA1_SPLITJ 1
#endif
#ifndef FFTGEN_K2_TWCACHE_FACTORED
#define FFTGEN_K2_TWCACHE_FACTORED 1
#endif

// pass 0 from an element accessor: v[j*R + A] = x[A*k + c], c = t + j*T
template <class G, int DIR, class Load>
FFTGEN_FI void pass0(int t, float2 *v, Load &&load) {
  constexpr int R = G::R(0), k = G::K(0), J = G::RMAX / R;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int c = t + j * G::T;
#pragma unroll
    for (int A = 0; A < R; ++A) v[j * R + A] = load(A * k + c);
    reg_fft<R, DIR>(v + j * R);
  }
}

// twiddle w_s^{A m} of pass p (forward sign; mul_tw conjugates for inverse)
template <class G, int p> FFTGEN_FI float2 pass_tw(const float2 *__restrict__ tw, int A, int m) {
  if constexpr (G::TW_FACTORED(p)) {
    const float2 *f = tw + G::TW_FOFF(p);
    const float2 hi = __ldg(f + A * 32 + (m >> 5)), lo = __ldg(f + (G::R(p) + A) * 32 + (m & 31));
    return cmul(hi, lo.x, lo.y);
  } else {
    return __ldg(tw + G::TW_OFF(p) + A * G::COLS(p) + m);
  }
}

template <class G, int N, int p>
FFTGEN_FI void smem_write(float2 *sx, int t, const float2 *v) {
  constexpr int R = G::R(p), cols = G::COLS(p), k = G::K(p), J = G::RMAX / R;
  constexpr Pad pd = BoundaryPad<N, p, 8, typename G::PL>::value;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int u = t + j * G::T, m = u / k, c = u % k;
#pragma unroll
    for (int B = 0; B < R; ++B) sx[padded((B * cols + m) * k + c, pd)] = v[j * R + B];
  }
}

template <class G, int N, int p, int DIR>
FFTGEN_FI void smem_read_pass(const float2 *sx, int t, const float2 *__restrict__ tw, float2 *v) {
  constexpr int R = G::R(p), k = G::K(p), J = G::RMAX / R;
  constexpr Pad pd = BoundaryPad<N, p - 1, 8, typename G::PL>::value;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int u = t + j * G::T, m = u / k, c = u % k;
    v[j * R] = sx[padded((m * R) * k + c, pd)];
#pragma unroll
    for (int A = 1; A < R; ++A) v[j * R + A] = mul_tw<DIR>(sx[padded((m * R + A) * k + c, pd)], pass_tw<G, p>(tw, A, m));
    reg_fft<R, DIR>(v + j * R);
  }
}

// Factored pass twiddles for a 2-pass plan: pass 1 has k == 1 and J == 1, so
// thread t always owns butterfly m = t and needs w_s^{A m} for A < R only.
// With A = a*RLO + b:  w^{A m} = Q[a] * P[b],  P[b] = w^{b m},  Q[a] = w^{RLO a m},
// loaded once per thread from the [A][m] table (RLO-1 + RHI-1 values).
template <class G, int PASS = 1> struct TwPQ {
  static constexpr int R = G::R(PASS);
  static constexpr int RLO = R >= 16 ? 8 : (R >= 4 ? 4 : R);
  static constexpr int RHI = R / RLO;
  float2 p[RLO], q[RHI];
  // (a factored pass table, TW_FACTORED: each base is itself hi * lo)
  FFTGEN_FI void load(const float2 *__restrict__ tw, int m) {
#pragma unroll
    for (int b = 1; b < RLO; ++b) p[b] = pass_tw<G, PASS>(tw, b, m);
#pragma unroll
    for (int a = 1; a < RHI; ++a) q[a] = pass_tw<G, PASS>(tw, a * RLO, m);
  }
  template <int DIR> FFTGEN_FI float2 apply(float2 x, int A) const {
    const int a = A / RLO, b = A % RLO;
    if (b) x = mul_tw<DIR>(x, p[b]);
    if (a) x = mul_tw<DIR>(x, q[a]);
    return x;
  }
};

// Three-pass plans in a persistent kernel: every pass-1 / pass-2 butterfly a
// thread owns (m = (t + j T) / k) is the same for every transform, so their
// twiddles are kept as factored bases in registers for the whole kernel
// (unfactored last-pass tables only; the factored-table pass of 2^14 keeps
// its own scheme).
template <class G> struct TwCache3 {
  static constexpr int J1 = G::RMAX / G::R(1), J2 = G::RMAX / G::R(2);
  TwPQ<G, 1> a[J1];
  TwPQ<G, 2> b[J2];
  FFTGEN_FI void load(const float2 *__restrict__ tw, int t) {
#pragma unroll
    for (int j = 0; j < J1; ++j) a[j].load(tw, (t + j * G::T) / G::K(1));
#pragma unroll
    for (int j = 0; j < J2; ++j) b[j].load(tw, (t + j * G::T) / G::K(2));
  }
};

template <class G, int N, int p, int DIR, class W>
FFTGEN_FI void smem_read_pass_cached(const float2 *sx, int t, const W *w, float2 *v) {
  constexpr int R = G::R(p), k = G::K(p), J = G::RMAX / R;
  constexpr Pad pd = BoundaryPad<N, p - 1, 8, typename G::PL>::value;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int u = t + j * G::T, m = u / k, c = u % k;
    v[j * R] = sx[padded((m * R) * k + c, pd)];
#pragma unroll
    for (int A = 1; A < R; ++A) v[j * R + A] = w[j].template apply<DIR>(sx[padded((m * R + A) * k + c, pd)], A);
    reg_fft<R, DIR>(v + j * R);
  }
}

template <class G> constexpr bool use_twcache3() {
#if FFTGEN_K2_TWCACHE
  return G::P == 3 && (FFTGEN_K2_TWCACHE_FACTORED || !G::TW_FACTORED(2));
#else
  return false;
#endif
}

template <class G, int N, int DIR>
FFTGEN_FI void middle_passes_cached(float2 *sx, int t, const TwCache3<G> &tc, float2 *v) {
  smem_write<G, N, 0>(sx, t, v);
  __syncthreads();
  smem_read_pass_cached<G, N, 1, DIR>(sx, t, tc.a, v);
  __syncthreads();
  smem_write<G, N, 1>(sx, t, v);
  __syncthreads();
  smem_read_pass_cached<G, N, 2, DIR>(sx, t, tc.b, v);
}

template <class G, int N, int DIR>
FFTGEN_FI void smem_read_pass1_pq(const float2 *sx, int t, const TwPQ<G> &w, float2 *v) {
  constexpr int R = G::R(1);
  constexpr Pad pd = BoundaryPad<N, 0, 8, typename G::PL>::value;
  static_assert(G::P == 2 && G::K(1) == 1 && G::RMAX == R, "factored twiddles need a 2-pass plan");
#pragma unroll
  for (int A = 0; A < R; ++A) v[A] = w.template apply<DIR>(sx[padded(t * R + A, pd)], A);
  reg_fft<R, DIR>(v);
}

// last pass: k == 1 so lanes over m are coalesced in HBM
template <class G, int LAYOUT>
FFTGEN_FI void store_last(const BlockArgs &a, int64_t obase, int t, const float2 *v) {
  constexpr int q = G::P - 1;
  constexpr int R = G::R(q), cols = G::COLS(q), k = G::K(q), J = G::RMAX / R;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int u = t + j * G::T, m = u / k, c = u % k;
#pragma unroll
    for (int B = 0; B < R; ++B) GIO<LAYOUT>::store(a, obase + (B * cols + m) * k + c, v[j * R + B]);
  }
}

// passes 1..P-1 through the exchange buffer sx
template <class G, int N, int DIR>
FFTGEN_FI void middle_passes(float2 *sx, int t, const float2 *__restrict__ tw, float2 *v) {
  if constexpr (G::P > 1) {
    smem_write<G, N, 0>(sx, t, v);
    __syncthreads();
    smem_read_pass<G, N, 1, DIR>(sx, t, tw, v);
    if constexpr (G::P > 2) {
      __syncthreads();
      smem_write<G, N, 1>(sx, t, v);
      __syncthreads();
      smem_read_pass<G, N, 2, DIR>(sx, t, tw, v);
    }
    if constexpr (G::P > 3) {
      __syncthreads();
      smem_write<G, N, 2>(sx, t, v);
      __syncthreads();
      smem_read_pass<G, N, 3, DIR>(sx, t, tw, v);
    }
  }
}

// ---- variant 1: direct ---------------------------------------------------
template <int N, int LAYOUT, int DIR, class PL = BlockPlan<N>>
__global__ void __launch_bounds__(BlockGeom<N, 0, PL>::THREADS) fft_block_kernel(const BlockArgs args) {
  using G = BlockGeom<N, 0, PL>;
  extern __shared__ float4 smem_f4[];
  const int tid = threadIdx.x;
  const int f = tid / G::T;
  const int t = tid - f * G::T;
  const int64_t b = (int64_t)blockIdx.x * G::TPB + f;
  const bool live = b < args.batch;
  const int64_t ibase = b * args.idist;

  float2 v[G::RMAX];
  pass0<G, DIR>(t, v, [&](int e) { return live ? GIO<LAYOUT>::load(args, ibase + e) : make_float2(0.f, 0.f); });
  float2 *sx = reinterpret_cast<float2 *>(smem_f4) + f * SmemGeom<N, PL>::REGION;
  if constexpr (G::P == 2) {
    TwPQ<G> pq;
    pq.load(args.tw, t);
    smem_write<G, N, 0>(sx, t, v);
    __syncthreads();
    smem_read_pass1_pq<G, N, DIR>(sx, t, pq, v);
  } else if constexpr (use_twcache3<G>()) {  // same arithmetic as the TMA kernel
    TwCache3<G> tc3;
    tc3.load(args.tw, t);
    middle_passes_cached<G, N, DIR>(sx, t, tc3, v);
  } else {
    middle_passes<G, N, DIR>(sx, t, args.tw, v);
  }
  if (live) store_last<G, LAYOUT>(args, b * args.odist, t, v);
}

// ---- variant 2: persistent, TMA double-buffered --------------------------
FFTGEN_FI uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

FFTGEN_FI void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
FFTGEN_FI void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
FFTGEN_FI void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// 1-D bulk copy global -> shared (TMA), completion counted on `bar`
FFTGEN_FI void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
FFTGEN_FI void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Raw stage layout of transform f of a group.  Packed (dist == N, the
// group's transforms are one contiguous run): interleaved at f * 8N, split re
// at f * 4N and im at TP * 4N + f * 4N, so one bulk copy per plane moves the
// whole group; otherwise transform f sits in its slot at f * SLOT.
template <int N, int LAYOUT, class PL = BlockPlan<N>> struct RawAt {
  using TG = TmaGeom<N, PL>;
  static FFTGEN_FI char *re(char *stage, int f, bool packed) {
    return stage + (packed ? f * (LAYOUT == LAYOUT_SPLIT ? 4 * N : 8 * N) : f * TG::SLOT);
  }
  static FFTGEN_FI char *im(char *stage, int f, bool packed) {  // split only
    return packed ? stage + TG::TP * 4 * N + f * 4 * N : stage + f * TG::SLOT + 4 * N;
  }
};

template <int N, int LAYOUT, class PL = BlockPlan<N>>
FFTGEN_FI void tma_issue(const BlockArgs &a, char *stage, uint64_t *bar, int64_t group) {
  using TG = TmaGeom<N, PL>;
  const int64_t b0 = group * TG::TP;
  const int cnt = (int)(a.batch - b0 < TG::TP ? a.batch - b0 : TG::TP);
  constexpr uint32_t plane = LAYOUT == LAYOUT_SPLIT ? 4 * N : 8 * N;
  mbar_expect_tx(bar, (uint32_t)cnt * 8 * N);
  if (a.idist == N) {  // packed: one copy per plane for the whole group
    if (LAYOUT == LAYOUT_SPLIT) {
      bulk_g2s(stage, reinterpret_cast<const float *>(a.in0) + b0 * N, cnt * plane, bar);
      bulk_g2s(RawAt<N, LAYOUT, PL>::im(stage, 0, true), reinterpret_cast<const float *>(a.in1) + b0 * N,
               cnt * plane, bar);
    } else {
      bulk_g2s(stage, reinterpret_cast<const float2 *>(a.in0) + b0 * N, cnt * plane, bar);
    }
    return;
  }
  for (int f = 0; f < cnt; ++f) {
    char *dst = stage + f * TG::SLOT;
    const int64_t b = b0 + f;
    if (LAYOUT == LAYOUT_SPLIT) {
      bulk_g2s(dst, reinterpret_cast<const float *>(a.in0) + b * a.idist, plane, bar);
      bulk_g2s(dst + plane, reinterpret_cast<const float *>(a.in1) + b * a.idist, plane, bar);
    } else {
      bulk_g2s(dst, reinterpret_cast<const float2 *>(a.in0) + b * a.idist, plane, bar);
    }
  }
}

// 1-D bulk copy shared -> global (TMA store), tracked by the bulk group
FFTGEN_FI void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
FFTGEN_FI void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
FFTGEN_FI void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
FFTGEN_FI void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Stage the last pass's outputs in the raw layout (RawAt) for a bulk store.
template <class G, int N, int LAYOUT>
FFTGEN_FI void smem_write_out(char *stage, int f, bool packed, int t, const float2 *v) {
  using RA = RawAt<N, LAYOUT, typename G::PL>;
  constexpr int q = G::P - 1;
  constexpr int R = G::R(q), cols = G::COLS(q), k = G::K(q), J = G::RMAX / R;
  char *re = RA::re(stage, f, packed);
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int u = t + j * G::T, m = u / k, c = u % k;
#pragma unroll
    for (int B = 0; B < R; ++B) {
      const int e = (B * cols + m) * k + c;
      if constexpr (LAYOUT == LAYOUT_SPLIT) {
        reinterpret_cast<float *>(re)[e] = v[j * R + B].x;
        reinterpret_cast<float *>(RA::im(stage, f, packed))[e] = v[j * R + B].y;
      } else {
        reinterpret_cast<float2 *>(re)[e] = v[j * R + B];
      }
    }
  }
}

template <int N, int LAYOUT, class PL = BlockPlan<N>>
FFTGEN_FI void tma_store(const BlockArgs &a, char *stage, int64_t group) {
  using TG = TmaGeom<N, PL>;
  const int64_t b0 = group * TG::TP;
  const int cnt = (int)(a.batch - b0 < TG::TP ? a.batch - b0 : TG::TP);
  constexpr uint32_t plane = LAYOUT == LAYOUT_SPLIT ? 4 * N : 8 * N;
  if (a.odist == N) {  // packed
    if (LAYOUT == LAYOUT_SPLIT) {
      bulk_s2g(reinterpret_cast<float *>(a.out0) + b0 * N, stage, cnt * plane);
      bulk_s2g(reinterpret_cast<float *>(a.out1) + b0 * N, RawAt<N, LAYOUT, PL>::im(stage, 0, true), cnt * plane);
    } else {
      bulk_s2g(reinterpret_cast<float2 *>(a.out0) + b0 * N, stage, cnt * plane);
    }
    bulk_commit();
    return;
  }
  for (int f = 0; f < cnt; ++f) {
    char *src = stage + f * TG::SLOT;
    const int64_t b = b0 + f;
    if (LAYOUT == LAYOUT_SPLIT) {
      bulk_s2g(reinterpret_cast<float *>(a.out0) + b * a.odist, src, plane);
      bulk_s2g(reinterpret_cast<float *>(a.out1) + b * a.odist, src + plane, plane);
    } else {
      bulk_s2g(reinterpret_cast<float2 *>(a.out0) + b * a.odist, src, plane);
    }
  }
  bulk_commit();
}

// STORE_TMA: outputs go smem -> HBM by cp.async.bulk (needs 16-byte aligned
// output rows) instead of per-thread coalesced st.global.
template <int N, int LAYOUT, int DIR, bool STORE_TMA, class PL = BlockPlan<N>>
__global__ void __launch_bounds__(TmaGeom<N, PL>::THREADS) fft_block_tma_kernel(const BlockArgs args) {
  using TG = TmaGeom<N, PL>;
  using G = typename TG::G;
  static_assert(TG::STAGES >= 1 && TG::STAGES <= 4, "1-4 stages");
  constexpr int NST = TG::STAGES;
  extern __shared__ float4 smem_f4[];
  char *smem = reinterpret_cast<char *>(smem_f4);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + TG::STAGES * TG::STAGE_BYTES);
  const int tid = threadIdx.x;
  const int f = tid / G::T;
  const int t = tid - f * G::T;
  const int64_t groups = (args.batch + TG::TP - 1) / TG::TP;
  const int64_t stride = gridDim.x;
  const bool packed_in = args.idist == N, packed_out = args.odist == N;

  if (tid == 0) {
    for (int s = 0; s < TG::STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < TG::STAGES; ++s) {
      const int64_t g = blockIdx.x + s * stride;
      if (g < groups) tma_issue<N, LAYOUT, PL>(args, smem + s * TG::STAGE_BYTES, &bars[s], g);
    }
  }
  // 2-pass plans: this thread's pass-1 twiddle bases live in registers;
  // 3-pass plans (2^13): those of passes 1 and 2 (TwCache3)
  TwPQ<G> pq;
  if constexpr (G::P == 2) pq.load(args.tw, t);
  constexpr bool kCache3 = use_twcache3<G>();
  TwCache3<G> tc3;
  if constexpr (kCache3) tc3.load(args.tw, t);

  int it = 0;
  for (int64_t g = blockIdx.x; g < groups; g += stride, ++it) {
    const int s = it % NST;
    char *stage = smem + s * TG::STAGE_BYTES;
    char *slot = stage + f * TG::SLOT;
    mbar_wait(&bars[s], (it / NST) & 1);

    float2 v[G::RMAX];
    if constexpr (LAYOUT == LAYOUT_SPLIT) {
      const float *re = reinterpret_cast<const float *>(RawAt<N, LAYOUT, PL>::re(stage, f, packed_in));
      const float *im = reinterpret_cast<const float *>(RawAt<N, LAYOUT, PL>::im(stage, f, packed_in));
      pass0<G, DIR>(t, v, [&](int e) { return make_float2(re[e], im[e]); });
    } else {
      const float2 *x = reinterpret_cast<const float2 *>(RawAt<N, LAYOUT, PL>::re(stage, f, packed_in));
      pass0<G, DIR>(t, v, [&](int e) { return x[e]; });
    }
    __syncthreads();  // raw stage fully consumed; reuse it as the exchange
    if (NST >= 2 && STORE_TMA && tid == 0 && it >= 1) {
      // the previous stage held group it-1, bulk-stored at the end of the last
      // iteration: refill it with group it-1+NST once that store has drained
      // shared memory (pass 0 above overlapped the drain)
      const int64_t gn = g + (NST - 1) * stride;
      if (gn < groups) {
        const int sp = (it - 1) % NST;
        bulk_wait_read0();
        tma_issue<N, LAYOUT, PL>(args, smem + sp * TG::STAGE_BYTES, &bars[sp], gn);
      }
    }
    float2 *sx = reinterpret_cast<float2 *>(slot);
    if constexpr (G::P == 2) {
      smem_write<G, N, 0>(sx, t, v);
      __syncthreads();
      smem_read_pass1_pq<G, N, DIR>(sx, t, pq, v);
    } else if constexpr (kCache3) {
      middle_passes_cached<G, N, DIR>(sx, t, tc3, v);
    } else {
      middle_passes<G, N, DIR>(sx, t, args.tw, v);
    }
    __syncthreads();  // exchange fully consumed
    const int64_t b = g * TG::TP + f;
    if constexpr (STORE_TMA) {
      smem_write_out<G, N, LAYOUT>(stage, f, packed_out, t, v);
      fence_proxy_async();  // make generic-proxy writes visible to the bulk copy
      __syncthreads();
      if (tid == 0) {
        tma_store<N, LAYOUT, PL>(args, stage, g);
        if (NST == 1 && g + stride < groups) {  // refill once the store has read the stage
          bulk_wait_read0();
          tma_issue<N, LAYOUT, PL>(args, stage, &bars[0], g + stride);
        }
      }
      (void)b;
    } else {
      if (tid == 0) {
        const int64_t gn = g + TG::STAGES * stride;
        if (gn < groups) {
          fence_proxy_async();
          tma_issue<N, LAYOUT, PL>(args, stage, &bars[s], gn);
        }
      }
      if (b < args.batch) store_last<G, LAYOUT>(args, b * args.odist, t, v);
    }
  }
  if (STORE_TMA && tid == 0) bulk_wait0();
}

// ---- variant 3: single-stage TMA + plane-wise exchange (N = 2^14) --------
// One CTA (512 threads) per SM.  The raw stage is refilled with the next
// transform right after pass 0 has read it; passes 1-2 exchange through a
// single padded fp32 plane, re then im (BoundaryPad<N, p, 4> keeps the
// 32-bit writer and reader patterns conflict-free).
template <class G, int N, int p, int COMP>
FFTGEN_FI void plane_write(float *X, int t, const float2 *v) {
  constexpr int R = G::R(p), cols = G::COLS(p), k = G::K(p), J = G::RMAX / R;
  constexpr Pad pd = BoundaryPad<N, p, 4, typename G::PL>::value;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int u = t + j * G::T, m = u / k, c = u % k;
#pragma unroll
    for (int B = 0; B < R; ++B) X[padded((B * cols + m) * k + c, pd)] = COMP ? v[j * R + B].y : v[j * R + B].x;
  }
}

template <class G, int N, int p, int COMP>  // reader of pass p (pad of boundary p-1)
FFTGEN_FI void plane_read(const float *X, int t, float2 *v) {
  constexpr int R = G::R(p), k = G::K(p), J = G::RMAX / R;
  constexpr Pad pd = BoundaryPad<N, p - 1, 4, typename G::PL>::value;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int u = t + j * G::T, m = u / k, c = u % k;
#pragma unroll
    for (int A = 0; A < R; ++A) {
      const float x = X[padded((m * R + A) * k + c, pd)];
      if (COMP)
        v[j * R + A].y = x;
      else
        v[j * R + A].x = x;
    }
  }
}

template <class G, int p, int DIR>
FFTGEN_FI void pass_compute(int t, const float2 *__restrict__ tw, float2 *v) {
  constexpr int R = G::R(p), k = G::K(p), J = G::RMAX / R;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int u = t + j * G::T, m = u / k;
#pragma unroll
    for (int A = 1; A < R; ++A) v[j * R + A] = mul_tw<DIR>(v[j * R + A], pass_tw<G, p>(tw, A, m));
    reg_fft<R, DIR>(v + j * R);
  }
}

template <class G, int p, int DIR, class W>
FFTGEN_FI void pass_compute_cached(int t, const W *w, float2 *v) {
  constexpr int R = G::R(p), J = G::RMAX / R;
#pragma unroll
  for (int j = 0; j < J; ++j) {
#pragma unroll
    for (int A = 1; A < R; ++A) v[j * R + A] = w[j].template apply<DIR>(v[j * R + A], A);
    reg_fft<R, DIR>(v + j * R);
  }
}

template <class G, int N, int p>
FFTGEN_FI void plane_exchange(float *X, int t, float2 *v) {
  plane_write<G, N, p - 1, 0>(X, t, v);
  __syncthreads();
  plane_read<G, N, p, 0>(X, t, v);
  __syncthreads();
  plane_write<G, N, p - 1, 1>(X, t, v);
  __syncthreads();
  plane_read<G, N, p, 1>(X, t, v);
}

template <class G, int N, int p, int DIR>
FFTGEN_FI void plane_exchange_pass(float *X, int t, const float2 *__restrict__ tw, float2 *v) {
  plane_write<G, N, p - 1, 0>(X, t, v);
  __syncthreads();
  plane_read<G, N, p, 0>(X, t, v);  // overwrites .x only; old .y still in place
  __syncthreads();
  plane_write<G, N, p - 1, 1>(X, t, v);
  __syncthreads();
  plane_read<G, N, p, 1>(X, t, v);
  pass_compute<G, p, DIR>(t, tw, v);
}

// Stage half of the last pass's outputs in the plane X for a bulk store:
// split -> plane COMP (re or im, N floats); interleaved -> output half COMP
// (k == 1 in the last pass, so element (B*cols + m) is in half B / (R/2):
// the register index alone picks the half, N/2 float2 = one plane).
template <class G, int N, int LAYOUT, int COMP>
FFTGEN_FI void plane_write_out(float *X, int t, const float2 *v) {
  constexpr int q = G::P - 1;
  constexpr int R = G::R(q), cols = G::COLS(q), J = G::RMAX / R;
  static_assert(G::K(q) == 1, "last pass writes natural order");
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int m = t + j * G::T;
    if constexpr (LAYOUT == LAYOUT_SPLIT) {
#pragma unroll
      for (int B = 0; B < R; ++B) X[B * cols + m] = COMP ? v[j * R + B].y : v[j * R + B].x;
    } else {
      float2 *X2 = reinterpret_cast<float2 *>(X);
#pragma unroll
      for (int B = COMP * (R / 2); B < (COMP + 1) * (R / 2); ++B) X2[(B - COMP * (R / 2)) * cols + m] = v[j * R + B];
    }
  }
}

// Exchange 1 runs as float2 through the raw stage (+ the head of X) and the
// next transform's load is issued after it (both exchanges plane-wise with the
// load issued right after pass 0 measured 0.57 / 0.58 vs 0.67 / 0.70).
template <int N, int LAYOUT, int DIR, bool STORE_TMA>
__global__ void __launch_bounds__(Tma1Geom<N>::THREADS, Tma1Geom<N>::MIN_BLOCKS) fft_block_tma1_kernel(const BlockArgs args) {
  using TG = Tma1Geom<N>;
  using G = typename TG::G;
  static_assert(G::TPB == 1 && G::P == 3, "single-stage variant is for one 3-pass transform per CTA");
  static_assert(TG::PLANE >= 4 * N, "the plane holds half an output transform");
  extern __shared__ float4 smem_f4[];
  char *stage = reinterpret_cast<char *>(smem_f4);
  float *X = reinterpret_cast<float *>(stage + TG::RAW);
  uint64_t *bar = reinterpret_cast<uint64_t *>(stage + TG::RAW + TG::PLANE);
  const int t = threadIdx.x;
  constexpr bool kCache = use_twcache3<G>();
  constexpr bool kEarly = kCache && FFTGEN_TMA1_EARLY_TW && LAYOUT == LAYOUT_INTERLEAVED;
  constexpr bool kSplitJ = kCache && STORE_TMA && FFTGEN_TMA1_SPLITJ;
  constexpr uint32_t plane = LAYOUT == LAYOUT_SPLIT ? 4 * N : 8 * N;
  auto issue = [&](int64_t b) {
    mbar_expect_tx(bar, 8 * N);
    if (LAYOUT == LAYOUT_SPLIT) {
      bulk_g2s(stage, reinterpret_cast<const float *>(args.in0) + b * args.idist, plane, bar);
      bulk_g2s(stage + plane, reinterpret_cast<const float *>(args.in1) + b * args.idist, plane, bar);
    } else {
      bulk_g2s(stage, reinterpret_cast<const float2 *>(args.in0) + b * args.idist, plane, bar);
    }
  };
  // one half of the output (split: one plane) from X to HBM
  auto store_half = [&](int64_t b, int h) {
    if (LAYOUT == LAYOUT_SPLIT)
      bulk_s2g(reinterpret_cast<float *>(h ? args.out1 : args.out0) + b * args.odist, X, 4 * N);
    else
      bulk_s2g(reinterpret_cast<float2 *>(args.out0) + b * args.odist + h * (N / 2), X, 4 * N);
    bulk_commit();
  };
  if (t == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0 && blockIdx.x < args.batch) issue(blockIdx.x);
  int it = 0;
  for (int64_t b = blockIdx.x; b < args.batch; b += gridDim.x, ++it) {
    TwCache3<G> tc1;
    if constexpr (kEarly) {
#pragma unroll
      for (int j = 0; j < TwCache3<G>::J1; ++j) tc1.a[j].load(args.tw, (t + j * G::T) / G::K(1));
    }
    mbar_wait(bar, it & 1);
    float2 v[G::RMAX];
    if constexpr (LAYOUT == LAYOUT_SPLIT) {
      const float *re = reinterpret_cast<const float *>(stage), *im = re + N;
      pass0<G, DIR>(t, v, [&](int e) { return make_float2(re[e], im[e]); });
    } else {
      const float2 *x = reinterpret_cast<const float2 *>(stage);
      pass0<G, DIR>(t, v, [&](int e) { return x[e]; });
    }
    // the previous transform's last bulk store has read X before it is rewritten
    if (STORE_TMA && t == 0) bulk_wait_read0();
    __syncthreads();  // stage consumed
    {
      static_assert(BoundaryPad<N, 0, 8, typename G::PL>::region * 8 <= TG::RAW + TG::PLANE, "exchange 1 fits");
      float2 *sx = reinterpret_cast<float2 *>(stage);
      smem_write<G, N, 0>(sx, t, v);
      if constexpr (kCache) {
        TwCache3<G> &tc = tc1;
        if constexpr (!kEarly) {
#pragma unroll
          for (int j = 0; j < TwCache3<G>::J1; ++j) tc.a[j].load(args.tw, (t + j * G::T) / G::K(1));
        }
        __syncthreads();
        smem_read_pass_cached<G, N, 1, DIR>(sx, t, tc.a, v);
      } else {
        __syncthreads();
        smem_read_pass<G, N, 1, DIR>(sx, t, args.tw, v);
      }
      __syncthreads();  // stage free: fetch the next transform behind pass 2
      if (t == 0 && b + gridDim.x < args.batch) {
        fence_proxy_async();
        issue(b + gridDim.x);
      }
    }
    if constexpr (kCache) {
      TwCache3<G> tc;
#pragma unroll
      for (int j = 0; j < TwCache3<G>::J2; ++j) tc.b[j].load(args.tw, (t + j * G::T) / G::K(2));
      plane_exchange<G, N, 2>(X, t, v);
      if constexpr (kSplitJ) {
        // last pass butterfly by butterfly: the results of butterfly 0 leave
        // (bulk stores of [B][t] rows) while butterfly 1 is computed
        constexpr int R = G::R(2), T = G::T, COLS = G::COLS(2);
        static_assert(G::RMAX / R == 2 && G::K(2) == 1, "two last-pass butterflies per thread");
        __syncthreads();  // pass-2 reads of X done
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
          for (int A = 1; A < R; ++A) v[j * R + A] = tc.b[j].template apply<DIR>(v[j * R + A], A);
          reg_fft<R, DIR>(v + j * R);
          if (j == 1) {
            if (t == 0) bulk_wait_read0();  // butterfly 0's results have left X
            __syncthreads();
          }
#pragma unroll
          for (int B = 0; B < R; ++B) {
            if constexpr (LAYOUT == LAYOUT_SPLIT) {
              X[B * T + t] = v[j * R + B].x;
              X[R * T + B * T + t] = v[j * R + B].y;
            } else {
              reinterpret_cast<float2 *>(X)[B * T + t] = v[j * R + B];
            }
          }
          fence_proxy_async();
          __syncthreads();
          if (t == 0) {
#pragma unroll 1
            for (int B = 0; B < R; ++B) {
              const int64_t e = b * args.odist + B * COLS + j * T;
              if constexpr (LAYOUT == LAYOUT_SPLIT) {
                bulk_s2g(reinterpret_cast<float *>(args.out0) + e, X + B * T, T * 4);
                bulk_s2g(reinterpret_cast<float *>(args.out1) + e, X + R * T + B * T, T * 4);
              } else {
                bulk_s2g(reinterpret_cast<float2 *>(args.out0) + e, reinterpret_cast<const float2 *>(X) + B * T, T * 8);
              }
            }
            bulk_commit();
          }
        }
        continue;
      }
      pass_compute_cached<G, 2, DIR>(t, tc.b, v);
    } else {
      plane_exchange_pass<G, N, 2, DIR>(X, t, args.tw, v);
    }
    if constexpr (STORE_TMA) {
      __syncthreads();  // pass-2 reads of X done
      plane_write_out<G, N, LAYOUT, 0>(X, t, v);
      fence_proxy_async();
      __syncthreads();
      if (t == 0) {
        store_half(b, 0);
        bulk_wait_read0();
      }
      __syncthreads();
      plane_write_out<G, N, LAYOUT, 1>(X, t, v);
      fence_proxy_async();
      __syncthreads();
      if (t == 0) store_half(b, 1);
    } else {
      store_last<G, LAYOUT>(args, b * args.odist, t, v);
      __syncthreads();  // X is rewritten by the next iteration
    }
  }
  if (STORE_TMA && t == 0) bulk_wait0();
}

}  // namespace fftgen_b200
