// block_instances.cuh -- instantiates the K2 block kernels for every
// N = 2^0 .. 2^14 at one (LAYOUT, DIR); included by block_<l>_<d>.cu so the
// four variants compile in parallel.
#pragma once
#include <cuda_runtime.h>

#include "fft_block.cuh"

namespace fftgen_b200 {

template <int N, int LAYOUT, int DIR>
cudaError_t block_launch_n(const BlockArgs &a, cudaStream_t s) {
  using G = BlockGeom<N>;
  const int64_t grid = (a.batch + G::TPB - 1) / G::TPB;
  constexpr int smem = SmemGeom<N>::BYTES;
  if (grid <= 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  fft_block_kernel<N, LAYOUT, DIR><<<(unsigned)grid, G::THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

template <int N, int LAYOUT, int DIR>
cudaError_t block_prepare_n(int *tma_blocks_per_sm) {
  constexpr int smem = SmemGeom<N>::BYTES;
  cudaError_t e = cudaSuccess;
  if (smem > 48 * 1024)
    e = cudaFuncSetAttribute(fft_block_kernel<N, LAYOUT, DIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  *tma_blocks_per_sm = 0;
  if constexpr (Tma1Geom<N>::ENABLED) {
    constexpr int tsmem = Tma1Geom<N>::BYTES;
    for (auto fn : {fft_block_tma1_kernel<N, LAYOUT, DIR, false>, fft_block_tma1_kernel<N, LAYOUT, DIR, true>}) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);
      if (e != cudaSuccess) return e;
    }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        tma_blocks_per_sm, fft_block_tma1_kernel<N, LAYOUT, DIR, true>, Tma1Geom<N>::THREADS, tsmem);
  } else if constexpr (TmaGeom<N>::ENABLED) {
    constexpr int tsmem = TmaGeom<N>::BYTES;
    e = cudaFuncSetAttribute(fft_block_tma_kernel<N, LAYOUT, DIR, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(fft_block_tma_kernel<N, LAYOUT, DIR, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, tsmem);
    if (e != cudaSuccess) return e;
    int b0 = 0, b1 = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b0, fft_block_tma_kernel<N, LAYOUT, DIR, false>,
                                                      TmaGeom<N>::THREADS, tsmem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, fft_block_tma_kernel<N, LAYOUT, DIR, true>,
                                                      TmaGeom<N>::THREADS, tsmem);
    *tma_blocks_per_sm = b0 < b1 ? b0 : b1;
  }
  return e;
}

template <int N, int LAYOUT, int DIR>
cudaError_t block_tma_launch_n(const BlockArgs &a, int grid, int flags, cudaStream_t s) {
  const bool store_tma = flags & BLOCK_TMA_STORE;
  if constexpr (Tma1Geom<N>::ENABLED) {
    if (grid <= 0 || a.batch <= 0) return cudaSuccess;
    constexpr int th = Tma1Geom<N>::THREADS, sm = Tma1Geom<N>::BYTES;
    if (store_tma) fft_block_tma1_kernel<N, LAYOUT, DIR, true><<<grid, th, sm, s>>>(a);
    else fft_block_tma1_kernel<N, LAYOUT, DIR, false><<<grid, th, sm, s>>>(a);
    return cudaGetLastError();
  } else if constexpr (TmaGeom<N>::ENABLED) {
    if (grid <= 0 || a.batch <= 0) return cudaSuccess;
    if (store_tma)
      fft_block_tma_kernel<N, LAYOUT, DIR, true><<<grid, TmaGeom<N>::THREADS, TmaGeom<N>::BYTES, s>>>(a);
    else
      fft_block_tma_kernel<N, LAYOUT, DIR, false><<<grid, TmaGeom<N>::THREADS, TmaGeom<N>::BYTES, s>>>(a);
    return cudaGetLastError();
  } else {
    return cudaErrorNotSupported;
  }
}

// direct kernel under a pass-radix cap (CapPlanGeom): only the (N, CAP)
// pairs whose plan differs from the default are instantiated
template <int N, int LAYOUT, int DIR, int CAP>
cudaError_t block_cap_launch_n(const BlockArgs &a, cudaStream_t s) {
  if constexpr (CapPlanGeom<N, CAP>::DISTINCT) {
    using PL = typename CapPlanGeom<N, CAP>::type;
    using G = BlockGeom<N, 0, PL>;
    const int64_t grid = (a.batch + G::TPB - 1) / G::TPB;
    constexpr int smem = SmemGeom<N, PL>::BYTES;
    if (grid <= 0) return cudaSuccess;
    if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    fft_block_kernel<N, LAYOUT, DIR, PL><<<(unsigned)grid, G::THREADS, smem, s>>>(a);
    return cudaGetLastError();
  } else {
    return cudaErrorInvalidValue;
  }
}

// (the persistent TMA kernel with these plans measured slower than both the
// direct kernel and the default TMA plans -- DESIGN.md section 6 -- so the
// capped plans run on the direct kernel only)
template <int N, int LAYOUT, int DIR, int CAP>
cudaError_t block_cap_prepare_n() {
  if constexpr (CapPlanGeom<N, CAP>::DISTINCT) {
    using PL = typename CapPlanGeom<N, CAP>::type;
    constexpr int smem = SmemGeom<N, PL>::BYTES;
    if (smem > 48 * 1024)
      return cudaFuncSetAttribute(fft_block_kernel<N, LAYOUT, DIR, PL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  smem);
    return cudaSuccess;
  } else {
    return cudaErrorInvalidValue;
  }
}

#define FFTGEN_CAP_SWITCH(FN, LAYOUT, DIR, CAP, ...)             \
  switch (log2n) {                                               \
  case 7: return FN<128, LAYOUT, DIR, CAP>(__VA_ARGS__);         \
  case 8: return FN<256, LAYOUT, DIR, CAP>(__VA_ARGS__);         \
  case 9: return FN<512, LAYOUT, DIR, CAP>(__VA_ARGS__);         \
  case 10: return FN<1024, LAYOUT, DIR, CAP>(__VA_ARGS__);       \
  case 11: return FN<2048, LAYOUT, DIR, CAP>(__VA_ARGS__);       \
  case 12: return FN<4096, LAYOUT, DIR, CAP>(__VA_ARGS__);       \
  case 13: return FN<8192, LAYOUT, DIR, CAP>(__VA_ARGS__);       \
  case 14: return FN<16384, LAYOUT, DIR, CAP>(__VA_ARGS__);      \
  default: return cudaErrorInvalidValue;                         \
  }

#define FFTGEN_BLOCK_SWITCH(FN, LAYOUT, DIR, ...)          \
  switch (log2n) {                                         \
  case 0: return FN<1, LAYOUT, DIR>(__VA_ARGS__);          \
  case 1: return FN<2, LAYOUT, DIR>(__VA_ARGS__);          \
  case 2: return FN<4, LAYOUT, DIR>(__VA_ARGS__);          \
  case 3: return FN<8, LAYOUT, DIR>(__VA_ARGS__);          \
  case 4: return FN<16, LAYOUT, DIR>(__VA_ARGS__);         \
  case 5: return FN<32, LAYOUT, DIR>(__VA_ARGS__);         \
  case 6: return FN<64, LAYOUT, DIR>(__VA_ARGS__);         \
  case 7: return FN<128, LAYOUT, DIR>(__VA_ARGS__);        \
  case 8: return FN<256, LAYOUT, DIR>(__VA_ARGS__);        \
  case 9: return FN<512, LAYOUT, DIR>(__VA_ARGS__);        \
  case 10: return FN<1024, LAYOUT, DIR>(__VA_ARGS__);      \
  case 11: return FN<2048, LAYOUT, DIR>(__VA_ARGS__);      \
  case 12: return FN<4096, LAYOUT, DIR>(__VA_ARGS__);      \
  case 13: return FN<8192, LAYOUT, DIR>(__VA_ARGS__);      \
  case 14: return FN<16384, LAYOUT, DIR>(__VA_ARGS__);     \
  default: return cudaErrorInvalidValue;                   \
  }

#define FFTGEN_BLOCK_INSTANCES(SUFFIX, LAYOUT, DIR)                                           \
  cudaError_t block_launch_##SUFFIX(int log2n, const BlockArgs &a, cudaStream_t s) {          \
    FFTGEN_BLOCK_SWITCH(block_launch_n, LAYOUT, DIR, a, s)                                    \
  }                                                                                           \
  cudaError_t block_prepare_##SUFFIX(int log2n, int *tma_blocks_per_sm) {                     \
    FFTGEN_BLOCK_SWITCH(block_prepare_n, LAYOUT, DIR, tma_blocks_per_sm)                      \
  }                                                                                           \
  cudaError_t block_tma_launch_##SUFFIX(int log2n, const BlockArgs &a, int grid, int flags, \
                                        cudaStream_t s) {                                     \
    FFTGEN_BLOCK_SWITCH(block_tma_launch_n, LAYOUT, DIR, a, grid, flags, s)               \
  }                                                                                           \
  cudaError_t block_cap_launch_##SUFFIX(int log2n, int cap, const BlockArgs &a, cudaStream_t s) { \
    switch (cap) {                                                                            \
    case 8: FFTGEN_CAP_SWITCH(block_cap_launch_n, LAYOUT, DIR, 8, a, s)                       \
    case 16: FFTGEN_CAP_SWITCH(block_cap_launch_n, LAYOUT, DIR, 16, a, s)                     \
    case 32: FFTGEN_CAP_SWITCH(block_cap_launch_n, LAYOUT, DIR, 32, a, s)                     \
    default: return cudaErrorInvalidValue;                                                    \
    }                                                                                         \
  }                                                                                           \
  cudaError_t block_cap_prepare_##SUFFIX(int log2n, int cap) {                                \
    switch (cap) {                                                                            \
    case 8: FFTGEN_CAP_SWITCH(block_cap_prepare_n, LAYOUT, DIR, 8)                            \
    case 16: FFTGEN_CAP_SWITCH(block_cap_prepare_n, LAYOUT, DIR, 16)                          \
    case 32: FFTGEN_CAP_SWITCH(block_cap_prepare_n, LAYOUT, DIR, 32)                          \
    default: return cudaErrorInvalidValue;                                                    \
    }                                                                                         \
  }

}  // namespace fftgen_b200
