// phased_instances.cuh -- instances and cooperative launches of the K6 phased
// kernel (fft_phased.cuh) for the 2-group splits 2^15 .. 2^20.
#pragma once
#include <cuda_runtime.h>

#include "fft_phased.cuh"

namespace fftgen_b200 {

template <int NS0, int NS1, int L, int DIR>
cudaError_t phased_launch_t(const PhasedArgs &pa, int grid, cudaStream_t s) {
  using PG = PhasedGeom<NS0, NS1>;
  void *args[] = {const_cast<PhasedArgs *>(&pa)};
  return cudaLaunchCooperativeKernel((const void *)fft_phased_kernel<NS0, NS1, L, L, DIR>, dim3(grid),
                                     dim3(PG::THREADS), args, PG::SMEM, s);
}

template <int NS0, int NS1, int L, int DIR> cudaError_t phased_prepare_t(int *bps) {
  using PG = PhasedGeom<NS0, NS1>;
  auto k = fft_phased_kernel<NS0, NS1, L, L, DIR>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PG::SMEM);
  int n = 0;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, PG::THREADS, PG::SMEM);
  if (n < *bps) *bps = n;
  return e;
}

template <int NS0, int NS1, int DIR>
cudaError_t phased_launch_l(int layout, const PhasedArgs &pa, int grid, cudaStream_t s) {
  return layout == LAYOUT_SPLIT ? phased_launch_t<NS0, NS1, LAYOUT_SPLIT, DIR>(pa, grid, s)
                                : phased_launch_t<NS0, NS1, LAYOUT_INTERLEAVED, DIR>(pa, grid, s);
}
template <int NS0, int NS1, int DIR> cudaError_t phased_prepare_l(int *bps) {
  cudaError_t e = phased_prepare_t<NS0, NS1, LAYOUT_SPLIT, DIR>(bps);
  return e != cudaSuccess ? e : phased_prepare_t<NS0, NS1, LAYOUT_INTERLEAVED, DIR>(bps);
}

#define FFTGEN_PHASED_SHAPES(X)                                                                        \
  X(7, 8, 128, 256) X(8, 8, 256, 256) X(8, 9, 256, 512) X(9, 9, 512, 512) X(9, 10, 512, 1024)        \
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
template <int DIR> cudaError_t phased_prepare_dir(int l0, int l1, int *bps) {
  switch (l0 * 16 + l1) {
#define FFTGEN_PH_PREPARE(A, B, NA, NB) \
  case A * 16 + B: return phased_prepare_l<NA, NB, DIR>(bps);
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
  cudaError_t phased_prepare_##SUFFIX(int l0, int l1, int *bps) { return phased_prepare_dir<DIR>(l0, l1, bps); }

}  // namespace fftgen_b200
