// dist.cu -- device stages of the distributed four-step (config C5).
//
// One N-point transform, block-distributed over P ranks (rank r holds
// x[r M : (r+1) M], M = N/P).  With n = a + M r (a < M, r < P) and
// k = k_b + P k_a, the reference's two-factor split (formula.cpp:160-165,
// Eq. 1 with K = P, M = N/P) reads
//
//   X[k_b + P k_a] = sum_a w_M^{a k_a} * ( w_N^{a k_b} * sum_r x[a + M r] w_P^{r k_b} )
//
// and runs as three all-to-alls of CONTIGUOUS equal chunks (L1 = N/P^2
// elements each) around three local passes, so no exchange needs a separate
// pack or transpose copy:
//
//   exchange 1  the user's block as-is: rank q receives R1[r][j] = x[r M + q L1 + j]
//   butterfly   (this file) Y[k_b][j] = w_N^{(q L1 + j) k_b} * DFT_P(R1[.][j])[k_b]
//               -- the P-point DFT_P (x) I_L1 butterfly and the twiddle
//               diagonal D^N of Eq. 1 in one pass; row k_b IS the chunk
//               for rank k_b (the pack is the store order)
//   exchange 2  rank q' receives R2[q][j] = Y_q[q'][j], i.e. a = q L1 + j in
//               natural order: the M-point input of the local transform
//   local       the single-GPU sm_100a plan of size M (K2 / K5 / K3)
//   exchange 3  chunk s of Z = Z[s L1 : (s+1) L1] goes to rank s
//   unpack      (this file) out[P j + q'] = R3[q'][j]: the stride-P
//               interleave of the last stride permutation Pi^N_P
//               (formula.cpp:216-224), the one data movement the contiguous
//               exchanges cannot absorb (the P sources of an output block
//               interleave at element granularity)
//
// Both kernels stream 16-byte vectors (two complex elements per thread and
// chunk); the twiddle w_N^e (e < N) is the product of two fp64-exact fp32
// tables T_lo[e mod 2^h] * T_hi[e >> h], h = ceil(log2 N / 2) -- 2^15
// entries each (256 KB, L2-resident) at N = 2^30.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "codelets.cuh"
#include "kernels.hpp"

namespace fftgen_b200 {

namespace {

FFTGEN_FI float2 cprod(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}

template <int P, int DIR>
__global__ void __launch_bounds__(256) dist_butterfly_kernel(const float2 *__restrict__ in, float2 *__restrict__ out,
                                                             int64_t l1, int64_t a0, const float2 *__restrict__ tlo,
                                                             const float2 *__restrict__ thi, int h, int64_t nmask) {
  const int64_t step = 2 * (int64_t)gridDim.x * blockDim.x;
  const int64_t lomask = (int64_t(1) << h) - 1;
  for (int64_t j = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); j < l1; j += step) {
    float2 v0[P], v1[P];
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const float4 t = __ldcs(reinterpret_cast<const float4 *>(in + r * l1 + j));
      v0[r] = make_float2(t.x, t.y);
      v1[r] = make_float2(t.z, t.w);
    }
    reg_fft<P, DIR>(v0);
    reg_fft<P, DIR>(v1);
    const int64_t a = a0 + j;
#pragma unroll
    for (int kb = 1; kb < P; ++kb) {
      const int64_t e0 = (a * kb) & nmask, e1 = ((a + 1) * kb) & nmask;
      v0[kb] = mul_tw<DIR>(v0[kb], cprod(__ldg(tlo + (e0 & lomask)), __ldg(thi + (e0 >> h))));
      v1[kb] = mul_tw<DIR>(v1[kb], cprod(__ldg(tlo + (e1 & lomask)), __ldg(thi + (e1 >> h))));
    }
#pragma unroll
    for (int kb = 0; kb < P; ++kb)
      __stcs(reinterpret_cast<float4 *>(out + kb * l1 + j), make_float4(v0[kb].x, v0[kb].y, v1[kb].x, v1[kb].y));
  }
}

template <int P>
__global__ void __launch_bounds__(256) dist_unpack_kernel(const float2 *__restrict__ in, float2 *__restrict__ out,
                                                          int64_t l1) {
  const int64_t step = 2 * (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); j < l1; j += step) {
    float4 t[P];
#pragma unroll
    for (int q = 0; q < P; ++q) t[q] = __ldcs(reinterpret_cast<const float4 *>(in + q * l1 + j));
    // out[P j + q] = element j of chunk q, out[P (j+1) + q] = element j+1
    float4 *o = reinterpret_cast<float4 *>(out + P * j);
    if constexpr (P == 1) {
      __stcs(o, t[0]);
    } else {
#pragma unroll
      for (int q = 0; q < P; q += 2) {
        __stcs(o + q / 2, make_float4(t[q].x, t[q].y, t[q + 1].x, t[q + 1].y));
        __stcs(o + (P + q) / 2, make_float4(t[q].z, t[q].w, t[q + 1].z, t[q + 1].w));
      }
    }
  }
}

// ---- peer-memory variants: the exchanges fused into the kernels -----------
// With every rank's blocks mapped into this process (CUDA IPC / symmetric
// memory over NVLink; or plain device buffers when the ranks are emulated on
// one GPU), exchange 1 becomes the butterfly's loads (chunk q of each rank's
// input block, read over NVLink), exchange 2 its stores (row k_b straight
// into slot q of rank k_b's receive block), and exchange 3 + unpack one pull
// kernel: no NCCL kernels, no staging copies -- each element crosses NVLink
// once per exchange, inside the compute kernel.
struct PeerPtrs {
  const float2 *p[16];
};
struct PeerOut {
  float2 *p[16];
};

template <int P, int DIR>
__global__ void __launch_bounds__(256) dist_butterfly_peer_kernel(PeerPtrs src, PeerOut dst, int64_t l1, int64_t a0,
                                                                  const float2 *__restrict__ tlo,
                                                                  const float2 *__restrict__ thi, int h, int64_t nmask) {
  const int64_t step = 2 * (int64_t)gridDim.x * blockDim.x;
  const int64_t lomask = (int64_t(1) << h) - 1;
  for (int64_t j = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); j < l1; j += step) {
    float2 v0[P], v1[P];
#pragma unroll
    for (int r = 0; r < P; ++r) {  // chunk q (offset a0) of rank r's block
      const float4 t = __ldcs(reinterpret_cast<const float4 *>(src.p[r] + a0 + j));
      v0[r] = make_float2(t.x, t.y);
      v1[r] = make_float2(t.z, t.w);
    }
    reg_fft<P, DIR>(v0);
    reg_fft<P, DIR>(v1);
    const int64_t a = a0 + j;
#pragma unroll
    for (int kb = 1; kb < P; ++kb) {
      const int64_t e0 = (a * kb) & nmask, e1 = ((a + 1) * kb) & nmask;
      v0[kb] = mul_tw<DIR>(v0[kb], cprod(__ldg(tlo + (e0 & lomask)), __ldg(thi + (e0 >> h))));
      v1[kb] = mul_tw<DIR>(v1[kb], cprod(__ldg(tlo + (e1 & lomask)), __ldg(thi + (e1 >> h))));
    }
#pragma unroll
    for (int kb = 0; kb < P; ++kb)  // slot q of rank k_b's receive block
      __stcs(reinterpret_cast<float4 *>(dst.p[kb] + a0 + j), make_float4(v0[kb].x, v0[kb].y, v1[kb].x, v1[kb].y));
  }
}

template <int P>
__global__ void __launch_bounds__(256) dist_unpack_peer_kernel(PeerPtrs src, float2 *__restrict__ out, int64_t l1,
                                                               int64_t s0) {
  const int64_t step = 2 * (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); j < l1; j += step) {
    float4 t[P];
#pragma unroll
    for (int q = 0; q < P; ++q) t[q] = __ldcs(reinterpret_cast<const float4 *>(src.p[q] + s0 + j));
    float4 *o = reinterpret_cast<float4 *>(out + P * j);
    if constexpr (P == 1) {
      __stcs(o, t[0]);
    } else {
#pragma unroll
      for (int q = 0; q < P; q += 2) {
        __stcs(o + q / 2, make_float4(t[q].x, t[q].y, t[q + 1].x, t[q + 1].y));
        __stcs(o + (P + q) / 2, make_float4(t[q].z, t[q].w, t[q + 1].z, t[q + 1].w));
      }
    }
  }
}

// out[i] = w_n^{(i step) mod n}: fp64 sincospi of an exact argument, exact at
// quadrant multiples (unit_root, matrix.cpp:14-35), rounded once to fp32
__global__ void gen_pow_kernel(float2 *__restrict__ out, int64_t count, int64_t step, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = (int64_t)(((unsigned __int128)i * (unsigned __int128)step) % (unsigned __int128)n);
    float2 w;
    if ((4 * e) % n == 0) {
      const int q = (int)(4 * e / n);
      w = q == 0 ? make_float2(1.f, 0.f) : q == 1 ? make_float2(0.f, -1.f) : q == 2 ? make_float2(-1.f, 0.f)
                                                                                     : make_float2(0.f, 1.f);
    } else {
      double sn, cs;
      sincospi(-2.0 * (double)e / (double)n, &sn, &cs);
      w = make_float2((float)cs, (float)sn);
    }
    out[i] = w;
  }
}

unsigned stream_grid(int64_t work_items) {
  // two elements per thread, 256 threads: up to 16 CTAs per SM of 148
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work_items + 511) / 512, 148 * 16));
}

template <int DIR>
cudaError_t butterfly_dispatch(int p, const float2 *in, float2 *out, int64_t l1, int64_t a0, const float2 *tlo,
                               const float2 *thi, int h, int64_t nmask, cudaStream_t s) {
  const unsigned g = stream_grid(l1);
  switch (p) {
  case 1: dist_butterfly_kernel<1, DIR><<<g, 256, 0, s>>>(in, out, l1, a0, tlo, thi, h, nmask); break;
  case 2: dist_butterfly_kernel<2, DIR><<<g, 256, 0, s>>>(in, out, l1, a0, tlo, thi, h, nmask); break;
  case 4: dist_butterfly_kernel<4, DIR><<<g, 256, 0, s>>>(in, out, l1, a0, tlo, thi, h, nmask); break;
  case 8: dist_butterfly_kernel<8, DIR><<<g, 256, 0, s>>>(in, out, l1, a0, tlo, thi, h, nmask); break;
  case 16: dist_butterfly_kernel<16, DIR><<<g, 256, 0, s>>>(in, out, l1, a0, tlo, thi, h, nmask); break;
  default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int DIR>
cudaError_t butterfly_peer_dispatch(int p, const PeerPtrs &src, const PeerOut &dst, int64_t l1, int64_t a0,
                                    const float2 *tlo, const float2 *thi, int h, int64_t nmask, cudaStream_t s) {
  const unsigned g = stream_grid(l1);
  switch (p) {
  case 1: dist_butterfly_peer_kernel<1, DIR><<<g, 256, 0, s>>>(src, dst, l1, a0, tlo, thi, h, nmask); break;
  case 2: dist_butterfly_peer_kernel<2, DIR><<<g, 256, 0, s>>>(src, dst, l1, a0, tlo, thi, h, nmask); break;
  case 4: dist_butterfly_peer_kernel<4, DIR><<<g, 256, 0, s>>>(src, dst, l1, a0, tlo, thi, h, nmask); break;
  case 8: dist_butterfly_peer_kernel<8, DIR><<<g, 256, 0, s>>>(src, dst, l1, a0, tlo, thi, h, nmask); break;
  case 16: dist_butterfly_peer_kernel<16, DIR><<<g, 256, 0, s>>>(src, dst, l1, a0, tlo, thi, h, nmask); break;
  default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

bool dist_world_supported(int p) { return p == 1 || p == 2 || p == 4 || p == 8 || p == 16; }

cudaError_t dist_butterfly_peers(int p, int dir, const float2 *const *src, float2 *const *dst, int64_t l1,
                                 int64_t a0, const float2 *tlo, const float2 *thi, int h, int log2n, cudaStream_t s) {
  if (p < 1 || p > 16) return cudaErrorInvalidValue;
  PeerPtrs sp{};
  PeerOut dp{};
  for (int r = 0; r < p; ++r) {
    sp.p[r] = src[r];
    dp.p[r] = dst[r];
  }
  const int64_t nmask = (int64_t(1) << log2n) - 1;
  return dir < 0 ? butterfly_peer_dispatch<-1>(p, sp, dp, l1, a0, tlo, thi, h, nmask, s)
                 : butterfly_peer_dispatch<1>(p, sp, dp, l1, a0, tlo, thi, h, nmask, s);
}

cudaError_t dist_unpack_peers(int p, const float2 *const *src, float2 *out, int64_t l1, int64_t s0, cudaStream_t s) {
  if (p < 1 || p > 16) return cudaErrorInvalidValue;
  PeerPtrs sp{};
  for (int r = 0; r < p; ++r) sp.p[r] = src[r];
  const unsigned g = stream_grid(l1);
  switch (p) {
  case 1: dist_unpack_peer_kernel<1><<<g, 256, 0, s>>>(sp, out, l1, s0); break;
  case 2: dist_unpack_peer_kernel<2><<<g, 256, 0, s>>>(sp, out, l1, s0); break;
  case 4: dist_unpack_peer_kernel<4><<<g, 256, 0, s>>>(sp, out, l1, s0); break;
  case 8: dist_unpack_peer_kernel<8><<<g, 256, 0, s>>>(sp, out, l1, s0); break;
  case 16: dist_unpack_peer_kernel<16><<<g, 256, 0, s>>>(sp, out, l1, s0); break;
  default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t dist_gen_tables(float2 *tlo, float2 *thi, int log2n, int h, cudaStream_t s) {
  const int64_t n = int64_t(1) << log2n, nlo = int64_t(1) << h, nhi = n >> h;
  gen_pow_kernel<<<stream_grid(2 * nlo), 256, 0, s>>>(tlo, nlo, 1, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gen_pow_kernel<<<stream_grid(2 * nhi), 256, 0, s>>>(thi, nhi, nlo, n);
  return cudaGetLastError();
}

cudaError_t dist_butterfly(int p, int dir, const float2 *in, float2 *out, int64_t l1, int64_t a0, const float2 *tlo,
                           const float2 *thi, int h, int log2n, cudaStream_t s) {
  const int64_t nmask = (int64_t(1) << log2n) - 1;
  return dir < 0 ? butterfly_dispatch<-1>(p, in, out, l1, a0, tlo, thi, h, nmask, s)
                 : butterfly_dispatch<1>(p, in, out, l1, a0, tlo, thi, h, nmask, s);
}

cudaError_t dist_unpack(int p, const float2 *in, float2 *out, int64_t l1, cudaStream_t s) {
  const unsigned g = stream_grid(l1);
  switch (p) {
  case 1: dist_unpack_kernel<1><<<g, 256, 0, s>>>(in, out, l1); break;
  case 2: dist_unpack_kernel<2><<<g, 256, 0, s>>>(in, out, l1); break;
  case 4: dist_unpack_kernel<4><<<g, 256, 0, s>>>(in, out, l1); break;
  case 8: dist_unpack_kernel<8><<<g, 256, 0, s>>>(in, out, l1); break;
  case 16: dist_unpack_kernel<16><<<g, 256, 0, s>>>(in, out, l1); break;
  default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ---- seeded_input (verify.cpp:55-78) on the device ------------------------
// The reference draws splitmix64 sequentially from state = seed; draw k
// (1-based) sees state seed + k*gamma, so element j of transform b is
//   re = 2 u(mix(s + (2j+1) gamma)) - 1,  im = 2 u(mix(s + (2j+2) gamma)) - 1,
// s = seed0 + b, u(bits) = (bits >> 11) 2^-53 -- computed in fp64 like the
// reference and rounded once to fp32 (bit-identical to the host generator's
// values cast to float).
namespace {
__device__ __forceinline__ uint64_t splitmix_finalize(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ float seeded_value(uint64_t state) {
  return (float)(2.0 * ((double)(splitmix_finalize(state) >> 11) * 0x1.0p-53) - 1.0);
}

template <bool SPLIT>
__global__ void __launch_bounds__(256) seeded_input_kernel(void *out0, void *out1, int64_t n, int64_t batch,
                                                           uint64_t seed0, int64_t dist) {
  constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
  const int64_t total = n * batch;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / n, j = i - b * n;
    const uint64_t s = seed0 + (uint64_t)b;
    const float re = seeded_value(s + (uint64_t)(2 * j + 1) * kGamma);
    const float im = seeded_value(s + (uint64_t)(2 * j + 2) * kGamma);
    if constexpr (SPLIT) {
      reinterpret_cast<float *>(out0)[b * dist + j] = re;
      reinterpret_cast<float *>(out1)[b * dist + j] = im;
    } else {
      reinterpret_cast<float2 *>(out0)[b * dist + j] = make_float2(re, im);
    }
  }
}
}  // namespace

cudaError_t seeded_input(bool split, void *out0, void *out1, int64_t n, int64_t batch, uint64_t seed0, int64_t dist,
                         cudaStream_t s) {
  const int64_t total = n * batch;
  if (total <= 0) return cudaSuccess;
  const unsigned g = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (split)
    seeded_input_kernel<true><<<g, 256, 0, s>>>(out0, out1, n, batch, seed0, dist);
  else
    seeded_input_kernel<false><<<g, 256, 0, s>>>(out0, out1, n, batch, seed0, dist);
  return cudaGetLastError();
}

}  // namespace fftgen_b200
