// fft_cluster.cuh -- K5: single-HBM-pass FFT with one transform per
// thread-block cluster, N = NS0 * NS1 in 2^14 .. 2^17 (too large for one CTA's
// shared memory).
//
// The transform is the reference's Stockham stage list (formula.cpp:168-197)
// regrouped into two radix-NS stages -- the Eq.-1 four-step of
// formula.hpp:102-106 with the stride permutations folded into addressing:
//
//   group 0 (s = NS0, cols = 1, k = NS1):  y[B NS1 + c] = DFT_NS0( x[A NS1 + c] )[B]
//   group 1 (s = N, cols = NS0, k = 1):    X[B NS0 + m] = DFT_NS1( y[m NS1 + A] w_N^{A m} )[B]
//
// executed by ONE cluster of C CTAs instead of two kernel launches with an HBM
// intermediate.  CTA r of the cluster owns
//   group 0: the TC0 = NS1 / C adjacent columns c in [r TC0, (r+1) TC0)
//            (one TMA tensor box of NS0 row segments x TC0 elements),
//   group 1: the TC1 = NS0 / C adjacent rows m in [r TC1, (r+1) TC1)
//            (natural-order output, TC1-element segments stored from registers).
// The intermediate y never leaves the chip: group-0 results go straight into
// the shared memory of the CTA that owns their row with st.async, whose bytes
// complete a transaction count on the owner's mbarrier.  HBM therefore sees
// exactly 16 N bytes per transform -- the single-pass roofline -- where the
// two-launch K3 path moves 32 N.
//
// The kernel is persistent (grid = co-resident clusters x C) with two shared
// buffers per CTA:
//   S: raw group-0 tile (TMA destination), then the padded group-0 exchange;
//      refilled with the NEXT transform's tile as soon as group-0 pass 1 has
//      read it, so HBM reads overlap the exchange, group 1 and the stores.
//   X: receive rows (st.async destination), then the padded group-1 exchange.
// Per transform:
//   1. wait S full (mbarrier, TMA bytes); group-0 pass 0 from S, codelets,
//      padded write to S; pass 1: local twiddles, codelets; issue next TMA.
//   2. cluster barrier wait (every CTA has finished reading its X of the
//      previous transform), st.async of the group-0 outputs into the owners' X.
//   3. wait X full (mbarrier, N / C * 8 bytes from the whole cluster).
//   4. group-1 pass 0 from X with w_N^{A m} (fp64-exact device tables),
//      codelets, padded rewrite of X; pass 1, codelets, HBM store.
//   5. cluster barrier arrive (X free for the next transform).
#pragma once

#include <cstdint>

#include "fft_group.cuh"

namespace fftgen_b200 {

// group 0, pass 0 of transform t+1 runs between the sends of transform t and
// the wait for its rows (1), or after transform t's stores (0); 2 = per
// layout as measured at 2^15: split 0.464 vs 0.458, interleaved 0.484 vs 0.491
#ifndef FFTGEN_K5_PIPE
#define FFTGEN_K5_PIPE 2
#endif
// group-1 results leave as one TMA tensor box per CTA (staged in X) instead
// of register stores (1), or not (0); 2 = per layout as measured at 2^15:
// split 0.486 vs 0.463, interleaved 0.485 vs 0.490
#ifndef FFTGEN_K5_TMA_STORE
#define FFTGEN_K5_TMA_STORE 2
#endif

template <int NS0, int NS1, int C> struct ClusterGeom {
  static constexpr int N = NS0 * NS1;
  static constexpr int TC0 = NS1 / C;  // group-0 columns per CTA
  static constexpr int TC1 = NS0 / C;  // group-1 rows per CTA
  using G0 = BlockGeom<NS0, TC0>;
  using G1 = BlockGeom<NS1, TC1>;
  static constexpr int T0 = G0::T, T1 = G1::T;
  // a group whose tile needs fewer threads leaves the rest idle for that group
  static constexpr int THREADS0 = G0::THREADS, THREADS1 = G1::THREADS;
  static constexpr int THREADS = THREADS0 > THREADS1 ? THREADS0 : THREADS1;
  static_assert(THREADS <= 1024 && THREADS0 % 32 == 0 && THREADS1 % 32 == 0, "CTA shape");
  static_assert(G0::P == 2 && G1::P == 2 && G0::K(1) == 1 && G1::K(1) == 1, "2-pass sub-FFTs");
  // padded per-column stride of the sub-FFT exchanges (odd: lanes over f hit distinct banks)
  static constexpr int EX0 = SmemGeom<NS0>::BASE > NS0 ? SmemGeom<NS0>::BASE : NS0;
  static constexpr int EX1 = SmemGeom<NS1>::BASE > NS1 ? SmemGeom<NS1>::BASE : NS1;
  static constexpr int REG0 = EX0 | 1, REG1 = EX1 | 1;
  // receive rows: a half-warp of the group-1 reader covers 16 / T1 rows when
  // T1 < 16, so shift consecutive rows by T1 bank pairs
  static constexpr int RS = T1 < 16 ? NS1 + T1 : NS1;
  static constexpr int amax(int a, int b) { return a > b ? a : b; }
  static constexpr int TILE = N / C;                                   // elements per CTA
  static constexpr int SLEN = (amax(TILE, TC0 * REG0) + 15) / 16 * 16;  // float2
  static constexpr int XLEN = (amax(TC1 * RS, TC1 * REG1) + 15) / 16 * 16;
  static constexpr int BYTES = (SLEN + XLEN) * 8 + 64;                  // + 2 mbarriers
  static constexpr int XBYTES = TC1 * NS1 * 8;                          // st.async bytes per transform
  static_assert(BYTES <= 227 * 1024, "fits one SM");
  // CTAs per SM the shared memory allows (228 KB per SM, 1 KB reserved per CTA)
  static constexpr int MIN_BLOCKS = (228 * 1024) / (BYTES + 1024) > 0 ? (228 * 1024) / (BYTES + 1024) : 1;
  static_assert((TC0 * 4) % 16 == 0 && NS0 <= 256 && TC0 * 2 <= 256, "TMA box limits");
};

FFTGEN_FI uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
FFTGEN_FI uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
FFTGEN_FI uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// shared::cta address -> shared::cluster address of the same offset in CTA `rank`
FFTGEN_FI uint32_t dsmem_map(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// remote store whose 8 bytes complete a transaction on the owner's mbarrier
FFTGEN_FI void st_async(uint32_t caddr, float2 v, uint32_t cbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(caddr),
               "f"(v.x), "f"(v.y), "r"(cbar)
               : "memory");
}
FFTGEN_FI void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
FFTGEN_FI void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
FFTGEN_FI void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

// 3-D tensor TMA: box {TC0 elements, NS0 rows, 1 transform} -> smem
FFTGEN_FI void tma_load_3d(void *dst, const void *tmap, int c0, int c1, int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// 3-D tensor TMA store: smem box -> global (bulk group)
FFTGEN_FI void tma_store_3d(const void *tmap, const void *src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(tmap),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

// group-0 tile of transform b -> S (rows [A][f]; split: re plane then im plane)
template <class CG, int LIN>
FFTGEN_FI void cluster_tile_issue(const ClusterArgs &a, char *S, uint64_t *bar, int64_t b, int r) {
  mbar_expect_tx(bar, (uint32_t)CG::TILE * 8u);
  if constexpr (LIN == LAYOUT_SPLIT) {
    tma_load_3d(S, a.tmap[0], r * CG::TC0, 0, (int)b, bar);
    tma_load_3d(S + CG::TILE * 4, a.tmap[1], r * CG::TC0, 0, (int)b, bar);
  } else {
    tma_load_3d(S, a.tmap[0], 2 * r * CG::TC0, 0, (int)b, bar);
  }
}

template <int NS0, int NS1, int C, int LIN, int LOUT, int DIR>
__global__ void __launch_bounds__(ClusterGeom<NS0, NS1, C>::THREADS, ClusterGeom<NS0, NS1, C>::MIN_BLOCKS) fft_cluster_kernel(const __grid_constant__ ClusterArgs a) {
  using CG = ClusterGeom<NS0, NS1, C>;
  using G0 = typename CG::G0;
  using G1 = typename CG::G1;
  extern __shared__ float4 smem_f4[];
  float2 *S = reinterpret_cast<float2 *>(smem_f4);
  float2 *X = S + CG::SLEN;
  uint64_t *bars = reinterpret_cast<uint64_t *>(X + CG::XLEN);  // [0] S full, [1] X full
  const int tid = threadIdx.x;
  const int r = (int)cluster_ctarank();
  const int64_t stride = nclusters_x();
  const int64_t b0 = cluster_id_x();

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();  // peers' mbarriers exist before any st.async targets them
  if (tid == 0 && b0 < a.batch) cluster_tile_issue<CG, LIN>(a, reinterpret_cast<char *>(S), &bars[0], b0, r);

  constexpr int R00 = G0::R(0), K00 = G0::K(0), J00 = G0::RMAX / R00;
  constexpr int R01 = G0::R(1), COLS01 = G0::COLS(1);
  constexpr int R10 = G1::R(0), K10 = G1::K(0), J10 = G1::RMAX / R10;
  constexpr int R11 = G1::R(1), COLS11 = G1::COLS(1);
  const uint32_t xbar_local = smem_u32(&bars[1]);
  const uint32_t xs_local = smem_u32(X);

  constexpr bool PIPE = FFTGEN_K5_PIPE == 2 ? LIN == LAYOUT_SPLIT : FFTGEN_K5_PIPE != 0;
  constexpr bool TSTORE = FFTGEN_K5_TMA_STORE == 2 ? LOUT == LAYOUT_SPLIT : FFTGEN_K5_TMA_STORE != 0;
  const int f0 = tid % CG::TC0, t0 = tid / CG::TC0;
  // group 0, pass 0 of the tile in S (the it-th arrival): raw rows [A][f] ->
  // registers -> codelets -> padded exchange in S
  auto g0_front = [&](int it_tile) {
    float2 w[G0::RMAX];
    mbar_wait(&bars[0], it_tile & 1);
    if (tid < CG::THREADS0) {
#pragma unroll
      for (int j = 0; j < J00; ++j) {
        const int c = t0 + j * CG::T0;
#pragma unroll
        for (int A0 = 0; A0 < R00; ++A0) {
          const int e = (A0 * K00 + c) * CG::TC0 + f0;
          if constexpr (LIN == LAYOUT_SPLIT) {
            const float *sp = reinterpret_cast<const float *>(S);
            w[j * R00 + A0] = make_float2(sp[e], sp[CG::TILE + e]);
          } else {
            w[j * R00 + A0] = S[e];
          }
        }
        reg_fft<R00, DIR>(w + j * R00);
      }
    }
    __syncthreads();  // raw tile consumed: S becomes the padded exchange
    if (tid < CG::THREADS0) smem_write<G0, NS0, 0>(S + f0 * CG::REG0, t0, w);
  };

  // pass-1 twiddle bases of both group sub-FFTs (fft_group.cuh, FFTGEN_GROUP_PQ):
  // this thread's butterflies t0 / tid / TC1 are the same for every transform
  GroupTw<G0> gtw0;
  if (tid < CG::THREADS0) gtw0.load(a.tw_local0, t0);
  GroupTw<G1> gtw1;
  if (tid < CG::THREADS1) gtw1.load(a.tw_local1, tid / CG::TC1);
  int it = 0;
  if (b0 < a.batch) g0_front(0);
  for (int64_t b = b0; b < a.batch; b += stride, ++it) {
    const int64_t ob = b * a.odist;
    float2 v[G0::RMAX > G1::RMAX ? G0::RMAX : G1::RMAX];
    // ---- group 0, pass 1: padded exchange in S -> registers ---------------
    __syncthreads();
    if (tid < CG::THREADS0) group_passes_rest<G0, NS0, DIR, 0, 0>(S + f0 * CG::REG0, t0, a.tw_local0, v, gtw0);
    __syncthreads();  // S free: fetch the next transform's tile behind the rest of this one
    if (tid == 0 && b + stride < a.batch) {
      fence_proxy_async();
      cluster_tile_issue<CG, LIN>(a, reinterpret_cast<char *>(S), &bars[0], b + stride, r);
    }
    // ---- exchange: group-0 output e of column r TC0 + f0 is y[e NS1 + c] -----
    if (tid == 0) mbar_expect_tx(&bars[1], CG::XBYTES);
    if (it > 0) cluster_wait();  // every peer has finished reading its X
    if (tid < CG::THREADS0) {
      const uint32_t col = 8u * (uint32_t)(r * CG::TC0 + f0);
#pragma unroll
      for (int B = 0; B < R01; ++B) {
        const int e = B * COLS01 + t0;
        const uint32_t owner = (uint32_t)(e / CG::TC1);
        st_async(dsmem_map(xs_local + col + 8u * (uint32_t)((e % CG::TC1) * CG::RS), owner), v[B],
                 dsmem_map(xbar_local, owner));
      }
    }
    // group 0, pass 0 of the next transform while the peers' rows arrive
    if (PIPE && b + stride < a.batch) g0_front(it + 1);
    // ---- group 1, pass 0: X rows -> registers, twiddle w_N^{A m} -------------
    mbar_wait(&bars[1], it & 1);
    const int f1 = tid / CG::T1, t1 = tid % CG::T1;
    if (tid < CG::THREADS1) {
      const int m = r * CG::TC1 + f1;
      const float2 *rowp = X + f1 * CG::RS;
      const float2 *qm = a.tw_q + m;
#pragma unroll
      for (int j = 0; j < J10; ++j) {
        const int c = t1 + j * CG::T1;
#pragma unroll
        for (int A0 = 0; A0 < R10; ++A0) v[j * R10 + A0] = rowp[A0 * K10 + c];
        const float2 pw = __ldg(a.tw_p + m * K10 + c);  // [m][c]: the rows group's P table
#pragma unroll
        for (int A0 = 0; A0 < R10; ++A0) {
          const float2 x = mul_tw<DIR>(v[j * R10 + A0], pw);
          v[j * R10 + A0] = A0 ? mul_tw<DIR>(x, __ldg(qm + A0 * NS0)) : x;
        }
        reg_fft<R10, DIR>(v + j * R10);
      }
    }
    __syncthreads();  // all rows read: X becomes the padded exchange
    if (tid < CG::THREADS1) smem_write<G1, NS1, 0>(X + f1 * CG::REG1, t1, v);
    __syncthreads();
    const int f = tid % CG::TC1, t = tid / CG::TC1;
    if (tid < CG::THREADS1) group_passes_rest<G1, NS1, DIR, 0, 0>(X + f * CG::REG1, t, a.tw_local1, v, gtw1);
    if constexpr (TSTORE) {
      // output rows e of this CTA's TC1 columns m: box [e][f] in X, one tensor store
      static_assert(NS1 * CG::TC1 <= CG::XLEN, "the output box fits X");
      __syncthreads();  // every pass-1 read of X done
      if (tid < CG::THREADS1) {
#pragma unroll
        for (int B = 0; B < R11; ++B) {
          const int e = B * COLS11 + t;
          if constexpr (LOUT == LAYOUT_SPLIT) {
            float *xf = reinterpret_cast<float *>(X);
            xf[e * CG::TC1 + f] = v[B].x;
            xf[NS1 * CG::TC1 + e * CG::TC1 + f] = v[B].y;
          } else {
            X[e * CG::TC1 + f] = v[B];
          }
        }
      }
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        constexpr int W = LOUT == LAYOUT_SPLIT ? 1 : 2;
        tma_store_3d(a.omap[0], X, r * CG::TC1 * W, 0, (int)b);
        if constexpr (LOUT == LAYOUT_SPLIT)
          tma_store_3d(a.omap[1], reinterpret_cast<const float *>(X) + NS1 * CG::TC1, r * CG::TC1, 0, (int)b);
        bulk_commit();
        bulk_wait_read0();  // X is read before the peers may refill it
      }
      (void)ob;
    } else if (tid < CG::THREADS1) {
      const int64_t m = (int64_t)r * CG::TC1 + f;
#pragma unroll
      for (int B = 0; B < R11; ++B)
        SIO<LOUT>::store(a.out0, a.out1, ob + (int64_t)(B * COLS11 + t) * NS0 + m, v[B]);
    }
    // every X read of this thread is done: X is free
    cluster_arrive_relaxed();
    if (!PIPE && b + stride < a.batch) g0_front(it + 1);
  }
  if (it > 0) cluster_wait();  // complete the last barrier phase before exit
  if (TSTORE && tid == 0) bulk_wait0();
}

}  // namespace fftgen_b200
