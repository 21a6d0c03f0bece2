// fft_rows.cu -- K2r: N = 8 .. 64, one transform per thread.
//
// For the smallest sizes the whole DFT_N is one register codelet (reg_fft<N>,
// codelets.cuh: the reference's Stockham stages on compile-time indices), so
// no exchange is needed at all; what limits the shared-memory block kernel
// there is HBM access granularity: its pass-0 lanes read 4- / 8-byte
// elements (split N = 32: 0.50 of HBM).  Here a CTA of THREADS threads owns
// THREADS consecutive transforms and moves them as whole rows:
//   1. cp.async 16-byte chunks, lanes over consecutive chunks of the
//      CTA's rows (fully coalesced, no register staging), into padded rows
//      (pitch ROWF + 4 floats: an odd number of 16-byte chunks, so the
//      per-thread row reads below are conflict-free);
//   2. thread t reads row t (LDS.128), runs the codelet, writes the row back;
//   3. coalesced 16-byte streaming stores of the rows.
// Split rows come from the re and im planes separately (two padded planes).
#include <cuda_runtime.h>

#include <algorithm>

#include "codelets.cuh"
#include "kernels.hpp"

namespace fftgen_b200 {

// transforms per CTA (measured, 1 GiB batches: N = 64 with 64 threads 0.93 /
// 1.02 split / interleaved vs 0.88 / 1.00 with 128 and 0.72 / 0.69 with 256;
// smaller N the same at 64 and 128).  One tile per CTA: persistent CTAs
// looping over tiles (grid capped at 4 / 16 CTAs per SM) measured slower
// (N = 8 split 0.79 / 0.71, N = 32 split 0.90 / 0.93 vs 0.88 / 1.05).

template <int N, int LAYOUT> struct RowsGeom {
  static constexpr int THREADS = N >= 64 ? 64 : 128;
  static constexpr int W = LAYOUT == LAYOUT_SPLIT ? 1 : 2;   // floats per element of a plane
  static constexpr int PLANES = LAYOUT == LAYOUT_SPLIT ? 2 : 1;
  static constexpr int ROWF = N * W;                         // floats per row and plane
  static constexpr int CPR = ROWF / 4;                       // 16-byte chunks per row
  static constexpr int PITCH = ROWF + 4;
  static constexpr int BYTES = PLANES * THREADS * PITCH * 4;
  static_assert(CPR >= 2 && (PITCH / 4) % 2 == 1, "odd 16-byte pitch");
};

FFTGEN_FI void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

template <int N, int LAYOUT, int DIR>
__global__ void __launch_bounds__(RowsGeom<N, LAYOUT>::THREADS) fft_rows_kernel(const BlockArgs a) {
  using RG = RowsGeom<N, LAYOUT>;
  constexpr int T = RG::THREADS, CPR = RG::CPR, PITCH = RG::PITCH, W = RG::W;
  extern __shared__ float4 smem_f4[];
  float *S = reinterpret_cast<float *>(smem_f4);
  const int tid = threadIdx.x;
  const int64_t b0 = (int64_t)blockIdx.x * T;
  const int rows = (int)std::min<int64_t>(T, a.batch - b0);

  // 1. rows -> padded shared rows (chunk q: row q / CPR, chunk q % CPR)
#pragma unroll
  for (int pl = 0; pl < RG::PLANES; ++pl) {
    const float *src = reinterpret_cast<const float *>(pl ? a.in1 : a.in0);
#pragma unroll
    for (int k = 0; k < CPR; ++k) {
      const int q = tid + k * T, r = q / CPR, c = q - r * CPR;
      if (r < rows) cp_async16(S + (pl * T + r) * PITCH + 4 * c, src + ((b0 + r) * a.idist) * W + 4 * c);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();

  // 2. row tid: the whole transform in registers
  float2 v[N];
  float *row0 = S + tid * PITCH;
#pragma unroll
  for (int c = 0; c < CPR; ++c) {
    const float4 x = *reinterpret_cast<const float4 *>(row0 + 4 * c);
    if constexpr (LAYOUT == LAYOUT_SPLIT) {
      const float4 y = *reinterpret_cast<const float4 *>(row0 + T * PITCH + 4 * c);
      v[4 * c] = make_float2(x.x, y.x);
      v[4 * c + 1] = make_float2(x.y, y.y);
      v[4 * c + 2] = make_float2(x.z, y.z);
      v[4 * c + 3] = make_float2(x.w, y.w);
    } else {
      v[2 * c] = make_float2(x.x, x.y);
      v[2 * c + 1] = make_float2(x.z, x.w);
    }
  }
  reg_fft<N, DIR>(v);
#pragma unroll
  for (int c = 0; c < CPR; ++c) {
    if constexpr (LAYOUT == LAYOUT_SPLIT) {
      *reinterpret_cast<float4 *>(row0 + 4 * c) = make_float4(v[4 * c].x, v[4 * c + 1].x, v[4 * c + 2].x, v[4 * c + 3].x);
      *reinterpret_cast<float4 *>(row0 + T * PITCH + 4 * c) =
          make_float4(v[4 * c].y, v[4 * c + 1].y, v[4 * c + 2].y, v[4 * c + 3].y);
    } else {
      *reinterpret_cast<float4 *>(row0 + 4 * c) = make_float4(v[2 * c].x, v[2 * c].y, v[2 * c + 1].x, v[2 * c + 1].y);
    }
  }
  __syncthreads();

  // 3. padded rows -> HBM, coalesced streaming stores
#pragma unroll
  for (int pl = 0; pl < RG::PLANES; ++pl) {
    float *dst = reinterpret_cast<float *>(pl ? a.out1 : a.out0);
#pragma unroll
    for (int k = 0; k < CPR; ++k) {
      const int q = tid + k * T, r = q / CPR, c = q - r * CPR;
      if (r < rows)
        __stcs(reinterpret_cast<float4 *>(dst + ((b0 + r) * a.odist) * W + 4 * c),
               *reinterpret_cast<const float4 *>(S + (pl * T + r) * PITCH + 4 * c));
    }
  }
}

namespace {
template <int N, int LAYOUT, int DIR> cudaError_t rows_launch_t(const BlockArgs &a, cudaStream_t s) {
  using RG = RowsGeom<N, LAYOUT>;
  const int64_t grid = (a.batch + RG::THREADS - 1) / RG::THREADS;
  if (grid <= 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  fft_rows_kernel<N, LAYOUT, DIR><<<(unsigned)grid, RG::THREADS, RG::BYTES, s>>>(a);
  return cudaGetLastError();
}
template <int N> cudaError_t rows_launch_n(int layout, int dir, const BlockArgs &a, cudaStream_t s) {
  if (layout == LAYOUT_SPLIT)
    return dir < 0 ? rows_launch_t<N, LAYOUT_SPLIT, -1>(a, s) : rows_launch_t<N, LAYOUT_SPLIT, 1>(a, s);
  return dir < 0 ? rows_launch_t<N, LAYOUT_INTERLEAVED, -1>(a, s) : rows_launch_t<N, LAYOUT_INTERLEAVED, 1>(a, s);
}
template <int N> cudaError_t rows_prepare_n() {
  cudaError_t e;
  const int bs = RowsGeom<N, LAYOUT_SPLIT>::BYTES, bi = RowsGeom<N, LAYOUT_INTERLEAVED>::BYTES;
  if ((e = cudaFuncSetAttribute(fft_rows_kernel<N, LAYOUT_SPLIT, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bs)))
    return e;
  if ((e = cudaFuncSetAttribute(fft_rows_kernel<N, LAYOUT_SPLIT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bs)))
    return e;
  if ((e = cudaFuncSetAttribute(fft_rows_kernel<N, LAYOUT_INTERLEAVED, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                bi)))
    return e;
  return cudaFuncSetAttribute(fft_rows_kernel<N, LAYOUT_INTERLEAVED, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bi);
}
}  // namespace

bool rows_enabled(int log2n) { return log2n >= 3 && log2n <= 6; }

cudaError_t rows_prepare(int log2n) {
  switch (log2n) {
  case 3: return rows_prepare_n<8>();
  case 4: return rows_prepare_n<16>();
  case 5: return rows_prepare_n<32>();
  case 6: return rows_prepare_n<64>();
  default: return cudaErrorInvalidValue;
  }
}

cudaError_t rows_launch(int log2n, int layout, int dir, const BlockArgs &a, cudaStream_t s) {
  switch (log2n) {
  case 3: return rows_launch_n<8>(layout, dir, a, s);
  case 4: return rows_launch_n<16>(layout, dir, a, s);
  case 5: return rows_launch_n<32>(layout, dir, a, s);
  case 6: return rows_launch_n<64>(layout, dir, a, s);
  default: return cudaErrorInvalidValue;
  }
}

void rows_geom(int log2n, int layout, int64_t *threads, int64_t *smem) {
  const int T = log2n >= 6 ? 64 : 128;
  *threads = T;
  const int n = 1 << log2n, w = layout == LAYOUT_SPLIT ? 1 : 2, planes = layout == LAYOUT_SPLIT ? 2 : 1;
  *smem = (int64_t)planes * T * (n * w + 4) * 4;
}

}  // namespace fftgen_b200
