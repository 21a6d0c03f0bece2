// fft_split.cuh -- K7: N = C * 2^14 (2^15, 2^16) in ONE HBM pass as a radix-C
// decimation-in-frequency step across a C-CTA thread-block cluster, then one
// 2^14-point transform per CTA with the single-stage schedule of
// fft_block_tma1_kernel (fft_block.cuh).
//
// With M = N / C, n = n' + p M (n' < M, p < C) and output index C j + q:
//
//   X[C j + q] = sum_{n'} w_M^{n' j} z_q(n'),
//   z_q(n')    = w_N^{n' q} sum_p x[n' + p M] w_C^{p q}
//
// i.e. the reference's DFT_N = (DFT_M (x) I_C)-style factorisation of
// formula.hpp:102-106 (Eq. 1) taken with the radix-C factor first: the C-point
// butterflies DFT_C (x) I_M, the twiddle diagonal D^N, and C independent
// M-point transforms whose outputs interleave with stride C (the stride
// permutation folded into the store addressing).
//
// CTA r of the cluster loads the slice n' in [r M/C, (r+1) M/C) of all C
// segments (C bulk copies per plane), computes the C outputs z_q(n') of each
// of its butterflies and sends z_q(n') to CTA q with st.async (8 bytes per
// element, completing on CTA q's mbarrier).  CTA q then owns z_q, a natural-
// order 2^14-point input in its stage buffer, and runs the three-pass
// transform: pass 0 from the stage, exchange 1 through the stage, the next
// transform's raw slice issued into the stage, exchange 2 through a separate
// fp32 plane, and stores to out[C j + q].  HBM sees 16 N bytes per transform.
//
// Per transform and CTA: one split cluster barrier (arrive after the raw slice
// is read -- the stage may then be overwritten by the peers' z -- and wait
// before sending z), one z mbarrier (M * 8 bytes from the whole cluster), one
// raw mbarrier (TMA bytes).
#pragma once

#include <cstdint>

#include "fft_block.cuh"
#include "fft_cluster.cuh"

namespace fftgen_b200 {

template <int C> struct SplitGeom {
  static constexpr int M = 16384;  // points per CTA
  using TG = Tma1Geom<M>;
  using G = typename TG::G;
  static constexpr int THREADS = TG::THREADS;
  static constexpr int SLICE = M / C;          // butterflies per CTA
  static constexpr int NPT = SLICE / THREADS;  // butterflies per thread
  static_assert(SLICE % THREADS == 0 && NPT * C <= G::RMAX, "radix-C step fits the sub-FFT registers");
  static_assert(G::P == 3 && G::TPB == 1, "three-pass 2^14 sub-FFT");
  static constexpr int BYTES = TG::BYTES;  // stage + plane + mbarriers
};

FFTGEN_FI void cluster_arrive_release() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
FFTGEN_FI void cluster_wait_acquire() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

template <int C, int LAYOUT, int DIR>
__global__ void __launch_bounds__(SplitGeom<C>::THREADS, 1) fft_split_kernel(const __grid_constant__ SplitArgs a) {
  using SG = SplitGeom<C>;
  using TG = typename SG::TG;
  using G = typename SG::G;
  constexpr int M = SG::M, SLICE = SG::SLICE, NPT = SG::NPT, TH = SG::THREADS;
  extern __shared__ float4 smem_f4[];
  char *stage = reinterpret_cast<char *>(smem_f4);
  float *X = reinterpret_cast<float *>(stage + TG::RAW);
  uint64_t *bars = reinterpret_cast<uint64_t *>(stage + TG::RAW + TG::PLANE);  // [0] raw, [1] z
  const int t = threadIdx.x;
  const int r = (int)cluster_ctarank();
  const int64_t stride = nclusters_x();
  const int64_t b0 = cluster_id_x();

  // raw slice n' in [r SLICE, (r+1) SLICE) of the C segments -> stage [p][n'] (split: re planes, then im)
  auto issue = [&](int64_t b) {
    mbar_expect_tx(&bars[0], (uint32_t)M * 8u);
#pragma unroll
    for (int p = 0; p < C; ++p) {
      const int64_t off = b * a.idist + (int64_t)p * M + (int64_t)r * SLICE;
      if constexpr (LAYOUT == LAYOUT_SPLIT) {
        bulk_g2s(stage + p * SLICE * 4, reinterpret_cast<const float *>(a.in0) + off, SLICE * 4, &bars[0]);
        bulk_g2s(stage + M * 4 + p * SLICE * 4, reinterpret_cast<const float *>(a.in1) + off, SLICE * 4, &bars[0]);
      } else {
        bulk_g2s(stage + p * SLICE * 8, reinterpret_cast<const float2 *>(a.in0) + off, SLICE * 8, &bars[0]);
      }
    }
  };

  if (t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();  // peers' z mbarriers exist before any st.async targets them
  if (t == 0 && b0 < a.batch) issue(b0);
  const uint32_t zbar_local = smem_u32(&bars[1]);
  const uint32_t stage_local = smem_u32(stage);

  int it = 0;
  for (int64_t b = b0; b < a.batch; b += stride, ++it) {
    float2 v[G::RMAX];
    // ---- radix-C butterflies of this CTA's slice ------------------------------
    mbar_wait(&bars[0], it & 1);
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const int nl = t + i * TH;
#pragma unroll
      for (int p = 0; p < C; ++p) {
        if constexpr (LAYOUT == LAYOUT_SPLIT) {
          const float *sp = reinterpret_cast<const float *>(stage);
          v[i * C + p] = make_float2(sp[p * SLICE + nl], sp[M + p * SLICE + nl]);
        } else {
          v[i * C + p] = reinterpret_cast<const float2 *>(stage)[p * SLICE + nl];
        }
      }
    }
    if (t == 0) mbar_expect_tx(&bars[1], (uint32_t)M * 8u);  // before any peer may send z
    cluster_arrive_release();                                 // raw slice read: the stage may be overwritten
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const int n = r * SLICE + t + i * TH;
      reg_fft<C, DIR>(v + i * C);
#pragma unroll
      for (int q = 1; q < C; ++q) v[i * C + q] = mul_tw<DIR>(v[i * C + q], __ldg(a.tw_n + n * q));
    }
    cluster_wait_acquire();  // every CTA of the cluster has read its raw slice
#pragma unroll
    for (int q = 0; q < C; ++q) {
      const uint32_t zq = dsmem_map(stage_local, (uint32_t)q), barq = dsmem_map(zbar_local, (uint32_t)q);
#pragma unroll
      for (int i = 0; i < NPT; ++i) st_async(zq + 8u * (uint32_t)(r * SLICE + t + i * TH), v[i * C + q], barq);
    }

    // ---- 2^14-point transform of z_r (natural order in the stage) -------------
    mbar_wait(&bars[1], it & 1);
    pass0<G, DIR>(t, v, [&](int e) { return reinterpret_cast<const float2 *>(stage)[e]; });
    __syncthreads();  // z consumed: the stage becomes exchange 1
    float2 *sx = reinterpret_cast<float2 *>(stage);
    smem_write<G, M, 0>(sx, t, v);
    __syncthreads();
    smem_read_pass<G, M, 1, DIR>(sx, t, a.tw, v);
    __syncthreads();  // stage free: the next transform's raw slice behind exchange 2
    if (t == 0 && b + stride < a.batch) {
      fence_proxy_async();
      issue(b + stride);
    }
    plane_exchange_pass<G, M, 2, DIR>(X, t, a.tw, v);
    {
      constexpr int q = G::P - 1;
      constexpr int R = G::R(q), cols = G::COLS(q), J = G::RMAX / R;
      static_assert(G::K(q) == 1, "last pass writes natural order");
      const int64_t ob = b * a.odist + r;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int m = t + j * G::T;
#pragma unroll
        for (int B = 0; B < R; ++B) {
          const int64_t o = ob + (int64_t)C * (B * cols + m);
          if constexpr (LAYOUT == LAYOUT_SPLIT) {
            __stcs(reinterpret_cast<float *>(a.out0) + o, v[j * R + B].x);
            __stcs(reinterpret_cast<float *>(a.out1) + o, v[j * R + B].y);
          } else {
            __stcs(reinterpret_cast<float2 *>(a.out0) + o, v[j * R + B]);
          }
        }
      }
    }
    __syncthreads();  // plane reads done before the next transform's exchange 1 reaches its head
  }
  cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
}

}  // namespace fftgen_b200
