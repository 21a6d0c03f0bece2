// kernels.hpp -- host-visible launch entry points of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fftgen_b200 {

enum { LAYOUT_INTERLEAVED = 0, LAYOUT_SPLIT = 1 };

// Arguments of the K2 block kernel (fft_block.cuh).
struct BlockArgs {
  const void *in0;
  const void *in1;     // split: imaginary plane
  void *out0;
  void *out1;
  int64_t idist;       // elements between consecutive transforms (input)
  int64_t odist;
  int64_t batch;
  const float2 *tw;    // concatenated [A][m] pass tables, w_s^{A m} (forward)
};

// K2: one CTA per TPB whole transforms, N = 2^log2n <= 2^14.
cudaError_t block_launch(int log2n, int layout, int dir, const BlockArgs &a, cudaStream_t s);
cudaError_t block_prepare(int log2n, int *tma_blocks_per_sm);
// persistent TMA-pipelined variant (fft_block_tma_kernel); grid = CTAs
cudaError_t block_tma_launch(int log2n, int layout, int dir, const BlockArgs &a, int grid, bool store_tma,
                             cudaStream_t s);
bool block_tma_enabled(int log2n);
int block_tma_transforms_per_cta(int log2n);
void block_tma_geom(int log2n, int64_t *threads, int64_t *tp, int64_t *smem);
void block_launch_geom(int log2n, int64_t *threads, int64_t *tpb, int64_t *smem);

// Arguments of the K3 group kernel (fft_group.cuh): one radix-NS Stockham
// stage of the whole transform with global (cols, k).
struct GroupArgs {
  const void *in0;
  const void *in1;
  void *out0;
  void *out1;
  int64_t cols, k;         // global Stockham parameters of the group
  int64_t idist, odist;    // elements between consecutive transforms
  int64_t tiles_per_outer; // CTAs per transform
  const float2 *tw_local;  // NS-point block-plan pass tables
  const float2 *tw_q;      // [A0][m] = w_s^{A0 (NS/R0) m}   (cols > 1)
  const float2 *tw_p;      // [c][m]  = w_s^{c m}
};

// Both groups of a 2-group plan in one persistent launch (fft_flow_kernel):
// group-0 output goes to slot b % ring_slots of an L2-resident ring.
struct FlowArgs {
  GroupArgs g0, g1;        // g0: user in -> ring; g1: ring -> user out
  int64_t n, batch, lag, ring_slots, tiles0, tiles1;
  unsigned long long *work;  // work-item counter (zeroed per launch)
  int *done0, *done1;        // per-slot completed tiles of group 0 / group 1
};
bool flow_supported(int log2ns0, int log2ns1);
cudaError_t flow_prepare(int log2ns0, int log2ns1, int *blocks_per_sm, int *smem_bytes);
cudaError_t flow_launch(int log2ns0, int log2ns1, int layout, int dir, const FlowArgs &f, int grid, cudaStream_t s);

// shape: 0 interleaved->scratch columns, 1 split->scratch columns,
//        2 scratch->interleaved rows,     3 scratch->split rows, 4 scratch->scratch columns
cudaError_t group_launch(int log2ns, int shape, int dir, const GroupArgs &a, int64_t batch, cudaStream_t s);
cudaError_t group_prepare(int log2ns);
void group_geom(int log2ns, int64_t *threads, int64_t *tc, int64_t *smem, int64_t *r0);

// K4: out[x*cols + m] = w_s^{x*row_scale*m}, fp64-accurate, rounded to fp32
cudaError_t gen_twiddles(float2 *out, int64_t rows, int64_t cols, int64_t row_scale, int64_t s, cudaStream_t st);

// distributed four-step twiddle diagonal on a local (rows x cols, ld) block
cudaError_t twiddle_block(float2 *data, int64_t rows, int64_t cols, int64_t ld, int64_t row_offset,
                          int64_t col_offset, int64_t n, int dir, cudaStream_t s);

cudaError_t convert_f64_to_f32(const double *in, float *out, int64_t count, cudaStream_t s);
cudaError_t convert_f32_to_f64(const float *in, double *out, int64_t count, cudaStream_t s);
cudaError_t strided_copy(const float *in, float *out, int64_t rows, int width, int64_t istride,
                         int64_t ostride, cudaStream_t s);

}  // namespace fftgen_b200
