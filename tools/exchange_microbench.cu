// Development microbenchmark (not part of the library): the K2 / K3 pass
// exchange of a 32 x 32 complex tile held by one warp (lane l owns column l:
// v[B] = y[B][l]; after the exchange lane l owns row l: v[A] = y[l][A]),
// done two ways:
//   smem : 32 STS.64 into a padded per-warp region, __syncwarp, 32 LDS.64
//          (the kernels' scheme, conflict-free with a 33-element row stride)
//   shfl : the 5-stage __shfl_xor_sync recursive block transpose
//          (16 register pairs per stage, 32 SHFL.32 + selects per stage)
// Every warp repeats the exchange ITERS times with a dependent FMA between
// rounds; the kernel time gives exchanges per second per SM.  Both variants
// are checked to produce the transpose.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exchange_microbench tools/exchange_microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int ITERS = 256;

__device__ __forceinline__ void xch_smem(float2 *v, float2 *region, int lane) {
#pragma unroll
  for (int b = 0; b < 32; ++b) region[b * 33 + lane] = v[b];
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 32; ++a) v[a] = region[lane * 33 + a];
  __syncwarp();
}

__device__ __forceinline__ void xch_shfl(float2 *v, int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool hi = lane & s;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i & s) continue;
      // lanes without bit s keep v[i] and trade v[i|s]; lanes with it keep v[i|s] and trade v[i]
      float2 send = hi ? v[i] : v[i | s];
      float2 got;
      got.x = __shfl_xor_sync(0xffffffffu, send.x, s);
      got.y = __shfl_xor_sync(0xffffffffu, send.y, s);
      if (hi)
        v[i] = got;
      else
        v[i | s] = got;
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) bench_kernel(float2 *out, int check) {
  extern __shared__ float2 smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2 *region = smem + warp * 32 * 33;
  float2 v[32];
#pragma unroll
  for (int b = 0; b < 32; ++b) v[b] = make_float2(float(b * 32 + lane), float(blockIdx.x));
  if (check) {
    if (MODE == 0)
      xch_smem(v, region, lane);
    else
      xch_shfl(v, lane);
    // y[B][l] = B * 32 + l, so lane l must now hold y[l][a] = l * 32 + a
#pragma unroll
    for (int a = 0; a < 32; ++a)
      if (v[a].x != float(lane * 32 + a)) out[0].x = 1.0f;
    return;
  }
  for (int it = 0; it < ITERS; ++it) {
    if (MODE == 0)
      xch_smem(v, region, lane);
    else
      xch_shfl(v, lane);
#pragma unroll
    for (int a = 0; a < 32; ++a) v[a].x = fmaf(v[a].x, 1.0000001f, v[a].y);
  }
  float acc = 0.f;
#pragma unroll
  for (int a = 0; a < 32; ++a) acc += v[a].x;
  if (acc == 12345.678f) out[1].x = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float2 *out;
  cudaMalloc(&out, 2 * sizeof(float2));
  const int smem = 8 * 32 * 33 * sizeof(float2);
  cudaFuncSetAttribute(bench_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(bench_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char *names[2] = {"smem", "shfl"};
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(out, 0, 2 * sizeof(float2));
    if (mode == 0)
      bench_kernel<0><<<1, 256, smem>>>(out, 1);
    else
      bench_kernel<1><<<1, 256, smem>>>(out, 1);
    float2 h;
    cudaMemcpy(&h, out, sizeof(h), cudaMemcpyDeviceToHost);
    const int blocks = sms * 8;  // 64 warps worth per SM requested; residency decides
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0)
        bench_kernel<0><<<blocks, 256, smem>>>(out, 0);
      else
        bench_kernel<1><<<blocks, 256, smem>>>(out, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double xch = double(blocks) * 8 * ITERS;  // warp exchanges of 32x32 complex
    const double bytes = xch * 32 * 32 * 8;          // tile bytes exchanged
    std::printf("{\"mode\": \"%s\", \"transpose_ok\": %s, \"ms\": %.4f, \"warp_exchanges_per_us_per_sm\": %.3f, "
                "\"tile_bytes_per_s\": %.4g, \"cycles_per_exchange_per_sm\": %.1f}\n",
                names[mode], h.x == 0.0f ? "true" : "false", ms, xch / (ms * 1e3) / sms, bytes / (ms * 1e-3),
                (ms * 1e-3) * 1.9e9 * sms / xch);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
