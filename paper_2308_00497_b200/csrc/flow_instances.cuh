// flow_instances.cuh -- instances of the K3 dataflow kernel (fft_group.cuh)
// for the 2-group splits whose groups share one CTA shape.
#pragma once
#include <cuda_runtime.h>

#include "fft_group.cuh"

namespace fftgen_b200 {

template <int NS0, int NS1> using FlowShape = FlowGeom<NS0, NS1>;

template <int NS0, int NS1, int DIR>
cudaError_t flow_launch_t(int layout, const FlowArgs &f, int grid, cudaStream_t s) {
  using FS = FlowShape<NS0, NS1>;
  if (layout == LAYOUT_SPLIT)
    fft_flow_kernel<NS0, NS1, LAYOUT_SPLIT, LAYOUT_SPLIT, DIR><<<grid, FS::THREADS, FS::SMEM, s>>>(f);
  else
    fft_flow_kernel<NS0, NS1, LAYOUT_INTERLEAVED, LAYOUT_INTERLEAVED, DIR><<<grid, FS::THREADS, FS::SMEM, s>>>(f);
  return cudaGetLastError();
}

template <int NS0, int NS1, int DIR>
cudaError_t flow_prepare_t(int *bps) {
  using FS = FlowShape<NS0, NS1>;
  auto k0 = fft_flow_kernel<NS0, NS1, LAYOUT_SPLIT, LAYOUT_SPLIT, DIR>;
  auto k1 = fft_flow_kernel<NS0, NS1, LAYOUT_INTERLEAVED, LAYOUT_INTERLEAVED, DIR>;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, FS::SMEM)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, FS::SMEM)) != cudaSuccess) return e;
  int b0 = 0, b1 = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b0, k0, FS::THREADS, FS::SMEM)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k1, FS::THREADS, FS::SMEM)) != cudaSuccess) return e;
  *bps = b0 < b1 ? b0 : b1;
  return cudaSuccess;
}

#define FFTGEN_FLOW_SWITCH(FN, DIR, ...)                              \
  switch (l0 * 16 + l1) {                                            \
  case 7 * 16 + 7: return FN<128, 128, DIR>(__VA_ARGS__);            \
  case 7 * 16 + 8: return FN<128, 256, DIR>(__VA_ARGS__);            \
  case 8 * 16 + 8: return FN<256, 256, DIR>(__VA_ARGS__);            \
  case 8 * 16 + 9: return FN<256, 512, DIR>(__VA_ARGS__);            \
  case 9 * 16 + 9: return FN<512, 512, DIR>(__VA_ARGS__);            \
  case 9 * 16 + 10: return FN<512, 1024, DIR>(__VA_ARGS__);         \
  case 10 * 16 + 10: return FN<1024, 1024, DIR>(__VA_ARGS__);        \
  default: return cudaErrorInvalidValue;                             \
  }

#define FFTGEN_FLOW_INSTANCES(SUFFIX, DIR)                                                              \
  cudaError_t flow_launch_##SUFFIX(int l0, int l1, int layout, const FlowArgs &f, int grid, cudaStream_t s) { \
    FFTGEN_FLOW_SWITCH(flow_launch_t, DIR, layout, f, grid, s)                                          \
  }                                                                                                     \
  cudaError_t flow_prepare_##SUFFIX(int l0, int l1, int *bps) { FFTGEN_FLOW_SWITCH(flow_prepare_t, DIR, bps) }

}  // namespace fftgen_b200
