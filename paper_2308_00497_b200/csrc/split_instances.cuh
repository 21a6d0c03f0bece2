// split_instances.cuh -- instances and cluster launches of the K7 kernel
// (fft_split.cuh) for N = 2^15 (C = 2) and 2^16 (C = 4) at one direction.
#pragma once
#include <cuda_runtime.h>

#include "fft_split.cuh"

namespace fftgen_b200 {

template <int C, int L, int DIR> cudaLaunchConfig_t split_config(int clusters, cudaStream_t s, cudaLaunchAttribute *attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * C));
  cfg.blockDim = dim3(SplitGeom<C>::THREADS);
  cfg.dynamicSmemBytes = SplitGeom<C>::BYTES;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

template <int C, int L, int DIR> cudaError_t split_launch_t(const SplitArgs &a, int max_clusters, cudaStream_t s) {
  if (a.batch <= 0) return cudaSuccess;
  const int clusters = (int)(a.batch < max_clusters ? a.batch : max_clusters);
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = split_config<C, L, DIR>(clusters, s, attr);
  return cudaLaunchKernelEx(&cfg, fft_split_kernel<C, L, DIR>, a);
}

template <int C, int L, int DIR> cudaError_t split_prepare_t(int *max_clusters) {
  auto k = fft_split_kernel<C, L, DIR>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SplitGeom<C>::BYTES);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = split_config<C, L, DIR>(1, 0, attr);
  int n = 0;
  e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
  *max_clusters = n;
  return e;
}

template <int C, int DIR> cudaError_t split_launch_c(int layout, const SplitArgs &a, int mc, cudaStream_t s) {
  return layout == LAYOUT_SPLIT ? split_launch_t<C, LAYOUT_SPLIT, DIR>(a, mc, s)
                                : split_launch_t<C, LAYOUT_INTERLEAVED, DIR>(a, mc, s);
}
template <int C, int DIR> cudaError_t split_prepare_c(int *max_clusters) {
  int m0 = 0, m1 = 0;
  cudaError_t e = split_prepare_t<C, LAYOUT_SPLIT, DIR>(&m0);
  if (e == cudaSuccess) e = split_prepare_t<C, LAYOUT_INTERLEAVED, DIR>(&m1);
  *max_clusters = m0 < m1 ? m0 : m1;
  return e;
}

}  // namespace fftgen_b200

#define FFTGEN_SPLIT_INSTANCES(SUFFIX, DIR)                                                               \
  cudaError_t split_launch_##SUFFIX(int log2n, int layout, const SplitArgs &a, int mc, cudaStream_t s) {  \
    switch (log2n) {                                                                                      \
    case 15: return split_launch_c<2, DIR>(layout, a, mc, s);                                             \
    case 16: return split_launch_c<4, DIR>(layout, a, mc, s);                                             \
    default: return cudaErrorInvalidValue;                                                                \
    }                                                                                                     \
  }                                                                                                       \
  cudaError_t split_prepare_##SUFFIX(int log2n, int *mc) {                                                \
    switch (log2n) {                                                                                      \
    case 15: return split_prepare_c<2, DIR>(mc);                                                          \
    case 16: return split_prepare_c<4, DIR>(mc);                                                          \
    default: return cudaErrorInvalidValue;                                                                \
    }                                                                                                     \
  }
