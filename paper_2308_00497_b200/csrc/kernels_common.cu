// kernels_common.cu -- K2 pass geometry for the host plan builder, launch
// dispatch across the (layout, direction) instance files, and the fp64 <->
// fp32 conversion kernels used by fftgen_interpret_f64.
#include <cuda_runtime.h>

#include "fft_block.cuh"
#include "kernels.hpp"
#include "plan.hpp"

namespace fftgen_b200 {

cudaError_t block_launch_i_f(int, const BlockArgs &, cudaStream_t);
cudaError_t block_launch_i_b(int, const BlockArgs &, cudaStream_t);
cudaError_t block_launch_s_f(int, const BlockArgs &, cudaStream_t);
cudaError_t block_launch_s_b(int, const BlockArgs &, cudaStream_t);
cudaError_t block_prepare_i_f(int);
cudaError_t block_prepare_i_b(int);
cudaError_t block_prepare_s_f(int);
cudaError_t block_prepare_s_b(int);

cudaError_t block_launch(int log2n, int layout, int dir, const BlockArgs &a, cudaStream_t s) {
  if (layout == LAYOUT_INTERLEAVED)
    return dir < 0 ? block_launch_i_f(log2n, a, s) : block_launch_i_b(log2n, a, s);
  return dir < 0 ? block_launch_s_f(log2n, a, s) : block_launch_s_b(log2n, a, s);
}

cudaError_t block_prepare(int log2n) {
  cudaError_t e;
  if ((e = block_prepare_i_f(log2n)) != cudaSuccess) return e;
  if ((e = block_prepare_i_b(log2n)) != cudaSuccess) return e;
  if ((e = block_prepare_s_f(log2n)) != cudaSuccess) return e;
  return block_prepare_s_b(log2n);
}

// ---- fp64 <-> fp32 for the interpret() drop-in ---------------------------
__global__ void f64_to_f32_kernel(const double *__restrict__ in, float *__restrict__ out, int64_t count) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < count; i += (int64_t)gridDim.x * blockDim.x) out[i] = (float)in[i];
}
__global__ void f32_to_f64_kernel(const float *__restrict__ in, double *__restrict__ out, int64_t count) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < count; i += (int64_t)gridDim.x * blockDim.x) out[i] = (double)in[i];
}

cudaError_t convert_f64_to_f32(const double *in, float *out, int64_t count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 16);
  f64_to_f32_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, out, count);
  return cudaGetLastError();
}
cudaError_t convert_f32_to_f64(const float *in, double *out, int64_t count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 16);
  f32_to_f64_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, out, count);
  return cudaGetLastError();
}

// N = 1 identity transform as a device copy (plan_stockham(1) = DFT_1).
__global__ void copy_kernel(const float *__restrict__ in, float *__restrict__ out, int64_t count,
                            int64_t istride, int64_t ostride, int width) {
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = i0; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / width, w = i % width;
    out[b * ostride + w] = in[b * istride + w];
  }
}
cudaError_t strided_copy(const float *in, float *out, int64_t rows, int width, int64_t istride,
                         int64_t ostride, cudaStream_t s) {
  const int64_t count = rows * width;
  if (count <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 16);
  copy_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, out, count, istride, ostride, width);
  return cudaGetLastError();
}

}  // namespace fftgen_b200
