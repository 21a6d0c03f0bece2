// group_instances.cuh -- instantiates the K3 group kernel (fft_group.cuh)
// for NS = 2^7 .. 2^12 and the (input layout, output layout, rows) shapes a
// multi-group plan uses: first group (user -> interleaved scratch, columns),
// middle groups (scratch -> scratch, columns), last group (scratch -> user,
// rows with the transposed store).
#pragma once
#include <cuda_runtime.h>

#include "fft_group.cuh"
#include "fft_group_tma.cuh"

namespace fftgen_b200 {

template <int NS, int LIN, int LOUT, int DIR, bool ROWS>
cudaError_t group_launch_t(const GroupArgs &a, int64_t grid, cudaStream_t s) {
  if (grid <= 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  fft_group_kernel<NS, LIN, LOUT, DIR, ROWS><<<(unsigned)grid, GroupGeom<NS>::THREADS, GroupGeom<NS>::BYTES, s>>>(a);
  return cudaGetLastError();
}

template <int NS, int LIN, int LOUT, int DIR, bool ROWS>
cudaError_t group_prepare_t() {
  return cudaFuncSetAttribute(fft_group_kernel<NS, LIN, LOUT, DIR, ROWS>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, GroupGeom<NS>::BYTES);
}

// shape: 0 = (interleaved -> scratch, columns), 1 = (split -> scratch, columns),
//        2 = (scratch -> interleaved, rows),     3 = (scratch -> split, rows),
//        4 = (scratch -> scratch, columns)
template <int NS, int DIR>
cudaError_t group_launch_ns(int shape, const GroupArgs &a, int64_t grid, cudaStream_t s) {
  switch (shape) {
  case 0: return group_launch_t<NS, LAYOUT_INTERLEAVED, LAYOUT_SCRATCH, DIR, false>(a, grid, s);
  case 1: return group_launch_t<NS, LAYOUT_SPLIT, LAYOUT_SCRATCH, DIR, false>(a, grid, s);
  case 2: return group_launch_t<NS, LAYOUT_SCRATCH, LAYOUT_INTERLEAVED, DIR, true>(a, grid, s);
  case 3: return group_launch_t<NS, LAYOUT_SCRATCH, LAYOUT_SPLIT, DIR, true>(a, grid, s);
  case 4: return group_launch_t<NS, LAYOUT_SCRATCH, LAYOUT_SCRATCH, DIR, false>(a, grid, s);
  default: return cudaErrorInvalidValue;
  }
}

template <int NS, int DIR>
cudaError_t group_prepare_ns() {
  cudaError_t e;
  if ((e = group_prepare_t<NS, LAYOUT_INTERLEAVED, LAYOUT_SCRATCH, DIR, false>()) != cudaSuccess) return e;
  if ((e = group_prepare_t<NS, LAYOUT_SPLIT, LAYOUT_SCRATCH, DIR, false>()) != cudaSuccess) return e;
  if ((e = group_prepare_t<NS, LAYOUT_SCRATCH, LAYOUT_INTERLEAVED, DIR, true>()) != cudaSuccess) return e;
  if ((e = group_prepare_t<NS, LAYOUT_SCRATCH, LAYOUT_SPLIT, DIR, true>()) != cudaSuccess) return e;
  return group_prepare_t<NS, LAYOUT_SCRATCH, LAYOUT_SCRATCH, DIR, false>();
}

// NS >= 2^FFTGEN_PLANE_MIN_LOG2: the TMA-tile variant is the plane-exchange
// kernel (next tile fetched right after pass 0); -DFFTGEN_GROUP_PLANE=0 keeps
// the stage-exchange one
template <int NS> constexpr bool use_plane() { return FFTGEN_GROUP_PLANE && GroupPlaneGeom<NS>::ENABLED; }

template <int NS, int LIN, int LOUT, int DIR, bool ROWS>
cudaError_t group_tma_launch_t(const GroupTmaArgs &ta, int grid, cudaStream_t s) {
  if (grid <= 0) return cudaSuccess;
  if constexpr (use_plane<NS>())
    fft_group_plane_kernel<NS, LIN, LOUT, DIR, ROWS>
        <<<grid, GroupPlaneGeom<NS>::THREADS, GroupPlaneGeom<NS>::BYTES, s>>>(ta);
  else
    fft_group_tma_kernel<NS, LIN, LOUT, DIR, ROWS>
        <<<grid, GroupTmaGeom<NS>::THREADS, GroupTmaGeom<NS, kGroupTmaStages, group_tma_store<NS, ROWS, LIN>()>::BYTES, s>>>(ta);
  return cudaGetLastError();
}

template <class K> cudaError_t prepare_kernel(K k, int threads, int bytes, int *bps) {
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  int n = 0;
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, threads, bytes);
  if (n < *bps) *bps = n;
  return e;
}

template <int NS, int LIN, int LOUT, int DIR, bool ROWS> cudaError_t group_tma_prepare_t(int *bps) {
  if constexpr (use_plane<NS>())
    return prepare_kernel(fft_group_plane_kernel<NS, LIN, LOUT, DIR, ROWS>, GroupPlaneGeom<NS>::THREADS,
                          GroupPlaneGeom<NS>::BYTES, bps);
  else
    return prepare_kernel(fft_group_tma_kernel<NS, LIN, LOUT, DIR, ROWS>, GroupTmaGeom<NS>::THREADS,
                          GroupTmaGeom<NS, kGroupTmaStages, group_tma_store<NS, ROWS, LIN>()>::BYTES, bps);
}

template <int NS, int DIR>
cudaError_t group_tma_launch_ns(int shape, const GroupTmaArgs &ta, int grid, cudaStream_t s) {
  switch (shape) {
  case 0: return group_tma_launch_t<NS, LAYOUT_INTERLEAVED, LAYOUT_SCRATCH, DIR, false>(ta, grid, s);
  case 1: return group_tma_launch_t<NS, LAYOUT_SPLIT, LAYOUT_SCRATCH, DIR, false>(ta, grid, s);
  case 2: return group_tma_launch_t<NS, LAYOUT_SCRATCH, LAYOUT_INTERLEAVED, DIR, true>(ta, grid, s);
  case 3: return group_tma_launch_t<NS, LAYOUT_SCRATCH, LAYOUT_SPLIT, DIR, true>(ta, grid, s);
  case 4: return group_tma_launch_t<NS, LAYOUT_SCRATCH, LAYOUT_SCRATCH, DIR, false>(ta, grid, s);
  default: return cudaErrorInvalidValue;
  }
}

template <int NS, int DIR> cudaError_t group_tma_prepare_ns(int *bps) {
  cudaError_t e;
  if ((e = group_tma_prepare_t<NS, LAYOUT_INTERLEAVED, LAYOUT_SCRATCH, DIR, false>(bps)) != cudaSuccess) return e;
  if ((e = group_tma_prepare_t<NS, LAYOUT_SPLIT, LAYOUT_SCRATCH, DIR, false>(bps)) != cudaSuccess) return e;
  if ((e = group_tma_prepare_t<NS, LAYOUT_SCRATCH, LAYOUT_INTERLEAVED, DIR, true>(bps)) != cudaSuccess) return e;
  if ((e = group_tma_prepare_t<NS, LAYOUT_SCRATCH, LAYOUT_SPLIT, DIR, true>(bps)) != cudaSuccess) return e;
  return group_tma_prepare_t<NS, LAYOUT_SCRATCH, LAYOUT_SCRATCH, DIR, false>(bps);
}

#define FFTGEN_GROUP_INSTANCES(SUFFIX, DIR)                                                          \
  cudaError_t group_launch_##SUFFIX(int log2ns, int shape, const GroupArgs &a, int64_t grid,        \
                                    cudaStream_t s) {                                               \
    switch (log2ns) {                                                                               \
    case 7: return group_launch_ns<128, DIR>(shape, a, grid, s);                                    \
    case 8: return group_launch_ns<256, DIR>(shape, a, grid, s);                                    \
    case 9: return group_launch_ns<512, DIR>(shape, a, grid, s);                                    \
    case 10: return group_launch_ns<1024, DIR>(shape, a, grid, s);                                  \
    case 11: return group_launch_ns<2048, DIR>(shape, a, grid, s);                                  \
    case 12: return group_launch_ns<4096, DIR>(shape, a, grid, s);                                  \
    default: return cudaErrorInvalidValue;                                                          \
    }                                                                                               \
  }                                                                                                 \
  cudaError_t group_prepare_##SUFFIX(int log2ns) {                                                  \
    switch (log2ns) {                                                                               \
    case 7: return group_prepare_ns<128, DIR>();                                                    \
    case 8: return group_prepare_ns<256, DIR>();                                                    \
    case 9: return group_prepare_ns<512, DIR>();                                                    \
    case 10: return group_prepare_ns<1024, DIR>();                                                  \
    case 11: return group_prepare_ns<2048, DIR>();                                                  \
    case 12: return group_prepare_ns<4096, DIR>();                                                  \
    default: return cudaErrorInvalidValue;                                                          \
    }                                                                                               \
  }                                                                                                 \
  cudaError_t group_tma_launch_##SUFFIX(int log2ns, int shape, const GroupTmaArgs &ta, int grid,    \
                                        cudaStream_t s) {                                           \
    switch (log2ns) {                                                                               \
    case 7: return group_tma_launch_ns<128, DIR>(shape, ta, grid, s);                               \
    case 8: return group_tma_launch_ns<256, DIR>(shape, ta, grid, s);                               \
    case 9: return group_tma_launch_ns<512, DIR>(shape, ta, grid, s);                               \
    case 10: return group_tma_launch_ns<1024, DIR>(shape, ta, grid, s);                             \
    case 11: return group_tma_launch_ns<2048, DIR>(shape, ta, grid, s);                             \
    case 12: return group_tma_launch_ns<4096, DIR>(shape, ta, grid, s);                             \
    default: return cudaErrorInvalidValue;                                                          \
    }                                                                                               \
  }                                                                                                 \
  cudaError_t group_tma_prepare_##SUFFIX(int log2ns, int *bps) {                                    \
    switch (log2ns) {                                                                               \
    case 7: return group_tma_prepare_ns<128, DIR>(bps);                                             \
    case 8: return group_tma_prepare_ns<256, DIR>(bps);                                             \
    case 9: return group_tma_prepare_ns<512, DIR>(bps);                                             \
    case 10: return group_tma_prepare_ns<1024, DIR>(bps);                                           \
    case 11: return group_tma_prepare_ns<2048, DIR>(bps);                                           \
    case 12: return group_tma_prepare_ns<4096, DIR>(bps);                                           \
    default: return cudaErrorInvalidValue;                                                          \
    }                                                                                               \
  }

}  // namespace fftgen_b200
