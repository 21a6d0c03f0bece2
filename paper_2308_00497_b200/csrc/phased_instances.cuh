// phased_instances.cuh -- instances and cooperative launches of the K6 phased
// kernel (fft_phased.cuh) for the 2-group splits 2^15 .. 2^20.
#pragma once
#include <cuda_runtime.h>

#include "fft_phased.cuh"

namespace fftgen_b200 {

// variant 1: TMA tiles (fft_phased_kernel); 2: plain tiles (fft_stream_kernel)
template <int NS0, int NS1, int L, int DIR>
cudaError_t phased_launch_t(const PhasedArgs &pa, int grid, cudaStream_t s) {
  void *args[] = {const_cast<PhasedArgs *>(&pa)};
  if (pa.variant == 2)
    return cudaLaunchCooperativeKernel((const void *)fft_stream_kernel<NS0, NS1, L, L, DIR>, dim3(grid),
                                       dim3(StreamGeom<NS0, NS1>::THREADS), args, StreamGeom<NS0, NS1>::SMEM, s);
  return cudaLaunchCooperativeKernel((const void *)fft_phased_kernel<NS0, NS1, L, L, DIR>, dim3(grid),
                                     dim3(PhasedGeom<NS0, NS1>::THREADS), args, PhasedGeom<NS0, NS1>::SMEM, s);
}

template <int NS0, int NS1, int L, int DIR> cudaError_t phased_prepare_t(int *bps, int variant) {
  cudaError_t e;
  int n = 0;
  if (variant == 2) {
    auto k = fft_stream_kernel<NS0, NS1, L, L, DIR>;
    using SG = StreamGeom<NS0, NS1>;
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SG::SMEM);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, SG::THREADS, SG::SMEM);
  } else {
    auto k = fft_phased_kernel<NS0, NS1, L, L, DIR>;
    using PG = PhasedGeom<NS0, NS1>;
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PG::SMEM);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, PG::THREADS, PG::SMEM);
  }
  if (n < *bps) *bps = n;
  return e;
}

template <int NS0, int NS1, int DIR>
cudaError_t phased_launch_l(int layout, const PhasedArgs &pa, int grid, cudaStream_t s) {
  return layout == LAYOUT_SPLIT ? phased_launch_t<NS0, NS1, LAYOUT_SPLIT, DIR>(pa, grid, s)
                                : phased_launch_t<NS0, NS1, LAYOUT_INTERLEAVED, DIR>(pa, grid, s);
}
template <int NS0, int NS1, int DIR> cudaError_t phased_prepare_l(int *bps, int variant) {
  cudaError_t e = phased_prepare_t<NS0, NS1, LAYOUT_SPLIT, DIR>(bps, variant);
  return e != cudaSuccess ? e : phased_prepare_t<NS0, NS1, LAYOUT_INTERLEAVED, DIR>(bps, variant);
}

#define FFTGEN_PHASED_SHAPES(X)                                                                        \
  X(7, 8, 128, 256) X(8, 8, 256, 256) X(8, 9, 256, 512) X(9, 8, 512, 256) X(9, 9, 512, 512) X(9, 10, 512, 1024) \
  X(10, 10, 1024, 1024)

template <int DIR>
cudaError_t phased_launch_dir(int l0, int l1, int layout, const PhasedArgs &pa, int grid, cudaStream_t s) {
  switch (l0 * 16 + l1) {
#define FFTGEN_PH_LAUNCH(A, B, NA, NB) \
  case A * 16 + B: return phased_launch_l<NA, NB, DIR>(layout, pa, grid, s);
    FFTGEN_PHASED_SHAPES(FFTGEN_PH_LAUNCH)
#undef FFTGEN_PH_LAUNCH
  default: return cudaErrorInvalidValue;
  }
}
template <int DIR> cudaError_t phased_prepare_dir(int l0, int l1, int *bps, int variant) {
  switch (l0 * 16 + l1) {
#define FFTGEN_PH_PREPARE(A, B, NA, NB) \
  case A * 16 + B: return phased_prepare_l<NA, NB, DIR>(bps, variant);
    FFTGEN_PHASED_SHAPES(FFTGEN_PH_PREPARE)
#undef FFTGEN_PH_PREPARE
  default: return cudaErrorInvalidValue;
  }
}

#define FFTGEN_PHASED_INSTANCES(SUFFIX, DIR)                                                           \
  cudaError_t phased_launch_##SUFFIX(int l0, int l1, int layout, const PhasedArgs &pa, int grid,       \
                                     cudaStream_t s) {                                                \
    return phased_launch_dir<DIR>(l0, l1, layout, pa, grid, s);                                       \
  }                                                                                                   \
  cudaError_t phased_prepare_##SUFFIX(int l0, int l1, int *bps, int variant) {                         \
    return phased_prepare_dir<DIR>(l0, l1, bps, variant);                                             \
  }

}  // namespace fftgen_b200
