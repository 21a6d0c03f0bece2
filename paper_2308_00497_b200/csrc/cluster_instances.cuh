// cluster_instances.cuh -- instances and cluster launches of the K5
// single-pass cluster kernel (fft_cluster.cuh).
#pragma once
#include <cuda_runtime.h>

#include "fft_cluster.cuh"

namespace fftgen_b200 {

template <int NS0, int NS1, int C, int L, int DIR>
cudaLaunchConfig_t cluster_config(int clusters, cudaStream_t s, cudaLaunchAttribute *attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * C));
  cfg.blockDim = dim3(ClusterGeom<NS0, NS1, C>::THREADS);
  cfg.dynamicSmemBytes = ClusterGeom<NS0, NS1, C>::BYTES;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

// persistent: min(batch, max_clusters) clusters loop over the batch
template <int NS0, int NS1, int C, int L, int DIR>
cudaError_t cluster_launch_t(const ClusterArgs &a, int64_t batch, int max_clusters, cudaStream_t s) {
  if (batch <= 0) return cudaSuccess;
  const int clusters = (int)(batch < max_clusters ? batch : max_clusters);
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = cluster_config<NS0, NS1, C, L, DIR>(clusters, s, attr);
  return cudaLaunchKernelEx(&cfg, fft_cluster_kernel<NS0, NS1, C, L, L, DIR>, a);
}

// kernel attributes; *max_clusters = co-resident clusters of this shape
template <int NS0, int NS1, int C, int L, int DIR> cudaError_t cluster_prepare_t(int *max_clusters) {
  auto k = fft_cluster_kernel<NS0, NS1, C, L, L, DIR>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ClusterGeom<NS0, NS1, C>::BYTES);
  if (e == cudaSuccess && C > 8) e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = cluster_config<NS0, NS1, C, L, DIR>(1, 0, attr);
  int n = 0;
  e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
  *max_clusters = n;
  return e;
}

template <int NS0, int NS1, int C, int DIR>
cudaError_t cluster_launch_l(int layout, const ClusterArgs &a, int64_t batch, int max_clusters, cudaStream_t s) {
  return layout == LAYOUT_SPLIT ? cluster_launch_t<NS0, NS1, C, LAYOUT_SPLIT, DIR>(a, batch, max_clusters, s)
                                : cluster_launch_t<NS0, NS1, C, LAYOUT_INTERLEAVED, DIR>(a, batch, max_clusters, s);
}
template <int NS0, int NS1, int C, int DIR> cudaError_t cluster_prepare_l(int *max_clusters) {
  int m0 = 0, m1 = 0;
  cudaError_t e = cluster_prepare_t<NS0, NS1, C, LAYOUT_SPLIT, DIR>(&m0);
  if (e == cudaSuccess) e = cluster_prepare_t<NS0, NS1, C, LAYOUT_INTERLEAVED, DIR>(&m1);
  *max_clusters = m0 < m1 ? m0 : m1;
  return e;
}

// (log2 NS0, log2 NS1, NS0, NS1, C).  The shape key is (l0, l1, C); C > 8
// is a non-portable cluster size.
#define FFTGEN_CLUSTER_SHAPES(X)                                                                          \
  X(7, 7, 128, 128, 2) X(7, 7, 128, 128, 4) X(7, 8, 128, 256, 4) X(7, 8, 128, 256, 8) X(8, 8, 256, 256, 8) \
  X(8, 8, 256, 256, 16)
#define FFTGEN_CLUSTER_KEY(A, B, C) ((A) * 4096 + (B) * 64 + (C))

template <int DIR> cudaError_t cluster_launch_dir(int l0, int l1, int c, int layout, const ClusterArgs &a,
                                                  int64_t batch, int max_clusters, cudaStream_t s) {
  switch (FFTGEN_CLUSTER_KEY(l0, l1, c)) {
#define FFTGEN_CL_LAUNCH(A, B, NA, NB, C) \
  case FFTGEN_CLUSTER_KEY(A, B, C): return cluster_launch_l<NA, NB, C, DIR>(layout, a, batch, max_clusters, s);
    FFTGEN_CLUSTER_SHAPES(FFTGEN_CL_LAUNCH)
#undef FFTGEN_CL_LAUNCH
  default: return cudaErrorInvalidValue;
  }
}
template <int DIR> cudaError_t cluster_prepare_dir(int l0, int l1, int c, int *max_clusters) {
  switch (FFTGEN_CLUSTER_KEY(l0, l1, c)) {
#define FFTGEN_CL_PREPARE(A, B, NA, NB, C) \
  case FFTGEN_CLUSTER_KEY(A, B, C): return cluster_prepare_l<NA, NB, C, DIR>(max_clusters);
    FFTGEN_CLUSTER_SHAPES(FFTGEN_CL_PREPARE)
#undef FFTGEN_CL_PREPARE
  default: return cudaErrorInvalidValue;
  }
}

#define FFTGEN_CLUSTER_INSTANCES(SUFFIX, DIR)                                                                \
  cudaError_t cluster_launch_##SUFFIX(int l0, int l1, int c, int layout, const ClusterArgs &a, int64_t batch, \
                                      int max_clusters, cudaStream_t s) {                                   \
    return cluster_launch_dir<DIR>(l0, l1, c, layout, a, batch, max_clusters, s);                           \
  }                                                                                                         \
  cudaError_t cluster_prepare_##SUFFIX(int l0, int l1, int c, int *max_clusters) {                          \
    return cluster_prepare_dir<DIR>(l0, l1, c, max_clusters);                                               \
  }

}  // namespace fftgen_b200
