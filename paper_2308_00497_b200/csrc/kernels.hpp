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
// K2r (fft_rows.cu): N = 8 .. 64, one transform per thread, coalesced 16-byte
// row moves; needs 16-byte aligned planes and dist
bool rows_enabled(int log2n);
cudaError_t rows_prepare(int log2n);
cudaError_t rows_launch(int log2n, int layout, int dir, const BlockArgs &a, cudaStream_t s);
void rows_geom(int log2n, int layout, int64_t *threads, int64_t *smem);
cudaError_t block_prepare(int log2n, int *tma_blocks_per_sm);
// K2 direct kernel under a pass-radix cap (8 / 16 / 32; CapPlanGeom) for the
// sizes whose capped plan differs from the default
cudaError_t block_cap_launch(int log2n, int cap, int layout, int dir, const BlockArgs &a, cudaStream_t s);
cudaError_t block_cap_prepare(int log2n, int cap);
// persistent TMA-pipelined variant (fft_block_tma_kernel); grid = CTAs;
// flags: BLOCK_TMA_STORE (bulk-store epilogue)
constexpr int BLOCK_TMA_STORE = 1;
cudaError_t block_tma_launch(int log2n, int layout, int dir, const BlockArgs &a, int grid, int flags,
                             cudaStream_t s);
bool block_tma_enabled(int log2n);
bool block_tma1(int log2n);  // the size runs the single-stage fft_block_tma1_kernel
int block_tma_transforms_per_cta(int log2n);
void block_tma_geom(int log2n, int64_t *threads, int64_t *tp, int64_t *smem);
void block_launch_geom(int log2n, int64_t *threads, int64_t *tpb, int64_t *smem, int cap = 0);

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
  const float2 *tw_p;      // [c][m] = w_s^{c m}; [m][c] for the rows group (k == 1)
};

// shape: 0 interleaved->scratch columns, 1 split->scratch columns,
//        2 scratch->interleaved rows,     3 scratch->split rows, 4 scratch->scratch columns
cudaError_t group_launch(int log2ns, int shape, int dir, const GroupArgs &a, int64_t batch, cudaStream_t s);
cudaError_t group_prepare(int log2ns);

// Persistent TMA variant of the group kernel (fft_group_tma.cuh): tensor maps
// of the input planes (re / interleaved, im), the group's args and the number
// of (transform, tile) work items.
struct GroupTmaArgs {
  alignas(64) unsigned char tmap[2][128];
  alignas(64) unsigned char omap[2][128];  // output maps (FFTGEN_GROUP_TMA_STORE)
  GroupArgs g;
  int64_t items;
};
// *blocks_per_sm: resident CTAs per SM of the slowest shape of this NS
cudaError_t group_tma_prepare(int log2ns, int *blocks_per_sm);
// encode ta.tmap for ta.g's input; false if the input is not TMA-addressable
bool group_tma_encode(int log2ns, int shape, int64_t batch, GroupTmaArgs &ta);
// whether the TMA variant of this group shape stores its results by TMA tensor stores
bool group_tma_stores(int log2ns, int shape);
// tensor maps of a's input planes for tiles of tc transforms (shape as group_launch)
bool encode_tile_maps(const GroupArgs &a, int log2ns, int shape, int64_t batch, int64_t tc,
                      unsigned char (*tmap)[128]);
cudaError_t group_tma_launch(int log2ns, int shape, int dir, const GroupTmaArgs &ta, int grid, cudaStream_t s);
void group_geom(int log2ns, int64_t *threads, int64_t *tc, int64_t *smem, int64_t *r0);
// whether the NS-point group's TMA variant is the plane-exchange kernel
bool group_plane(int log2ns);

// K5: one transform per thread-block cluster, N = NS0 * NS1 (2^14 .. 2^17),
// intermediate exchanged through distributed shared memory (fft_cluster.cuh).
struct ClusterArgs {
  // TMA tensor maps (CUtensorMap, 128 B each) of the input planes viewed as
  // [batch][NS0][NS1] (re / interleaved, im): group-0 tiles are 2-D boxes
  alignas(64) unsigned char tmap[2][128];
  // output planes viewed as [batch][NS1][NS0]: group-1 results leave as
  // boxes {TC1 columns, NS1 rows} (FFTGEN_K5_TMA_STORE)
  alignas(64) unsigned char omap[2][128];
  const void *in0, *in1;
  void *out0, *out1;
  int64_t idist, odist;
  int64_t batch;
  const float2 *tw_local0;  // NS0-point block-plan pass table
  const float2 *tw_local1;  // NS1-point block-plan pass table
  const float2 *tw_q;       // group 1: [A0][m] = w_N^{A0 (NS1/R0) m}
  const float2 *tw_p;       // group 1 (rows): [m][c] = w_N^{c m}
};
// default cluster size C of the (NS0, NS1) split for a layout, 0 = none
int cluster_default_size(int log2ns0, int log2ns1, int layout);
// *max_clusters: co-resident clusters (the persistent grid)
cudaError_t cluster_prepare(int log2ns0, int log2ns1, int csize, int *max_clusters);
cudaError_t cluster_launch(int log2ns0, int log2ns1, int csize, int layout, int dir, const ClusterArgs &a,
                           int64_t batch, int max_clusters, cudaStream_t s);
// threads / dynamic smem of a compiled (NS0, NS1, C) shape; 0 if not compiled
void cluster_geom(int log2ns0, int log2ns1, int csize, int64_t *threads, int64_t *smem);
// encode a.tmap for a.in0 / a.in1 (16-byte aligned planes, idist * element a multiple of 16)
cudaError_t cluster_encode_maps(int log2ns0, int log2ns1, int csize, int layout, ClusterArgs &a);

// K4: out[x*cols + m] = w_s^{x*row_scale*m}, fp64-accurate, rounded to fp32
cudaError_t gen_twiddles(float2 *out, int64_t rows, int64_t cols, int64_t row_scale, int64_t s, cudaStream_t st);

// distributed four-step twiddle diagonal on a local (rows x cols, ld) block
cudaError_t twiddle_block(float2 *data, int64_t rows, int64_t cols, int64_t ld, int64_t row_offset,
                          int64_t col_offset, int64_t n, int dir, cudaStream_t s);

// distributed four-step stages (dist.cu): P-point butterfly + D^N twiddle over
// P chunks of l1 elements (a0 = rank * l1), and the stride-P output interleave
bool dist_world_supported(int p);
cudaError_t dist_gen_tables(float2 *tlo, float2 *thi, int log2n, int h, cudaStream_t s);
cudaError_t dist_butterfly(int p, int dir, const float2 *in, float2 *out, int64_t l1, int64_t a0, const float2 *tlo,
                           const float2 *thi, int h, int log2n, cudaStream_t s);
cudaError_t dist_unpack(int p, const float2 *in, float2 *out, int64_t l1, cudaStream_t s);
// peer-memory variants (exchanges fused into the loads / stores): src / dst
// hold the P ranks' block base pointers
cudaError_t dist_butterfly_peers(int p, int dir, const float2 *const *src, float2 *const *dst, int64_t l1,
                                 int64_t a0, const float2 *tlo, const float2 *thi, int h, int log2n, cudaStream_t s);
cudaError_t dist_unpack_peers(int p, const float2 *const *src, float2 *out, int64_t l1, int64_t s0, cudaStream_t s);

// seeded_input (verify.cpp:55-78) for transforms b < batch, seed seed0 + b, fp32
cudaError_t seeded_input(bool split, void *out0, void *out1, int64_t n, int64_t batch, uint64_t seed0, int64_t dist,
                         cudaStream_t s);

cudaError_t convert_f64_to_f32(const double *in, float *out, int64_t count, cudaStream_t s);
cudaError_t convert_f32_to_f64(const float *in, double *out, int64_t count, cudaStream_t s);
cudaError_t strided_copy(const float *in, float *out, int64_t rows, int width, int64_t istride,
                         int64_t ostride, cudaStream_t s);

}  // namespace fftgen_b200
