// kernels_common.cu -- K2 pass geometry for the host plan builder, launch
// dispatch across the (layout, direction) instance files, and the fp64 <->
// fp32 conversion kernels used by fftgen_interpret_f64.
#include <cuda_runtime.h>

#include <algorithm>

#include "fft_block.cuh"
#include "kernels.hpp"
#include "plan.hpp"

namespace fftgen_b200 {

cudaError_t block_launch_i_f(int, const BlockArgs &, cudaStream_t);
cudaError_t block_launch_i_b(int, const BlockArgs &, cudaStream_t);
cudaError_t block_launch_s_f(int, const BlockArgs &, cudaStream_t);
cudaError_t block_launch_s_b(int, const BlockArgs &, cudaStream_t);
cudaError_t block_prepare_i_f(int, int *);
cudaError_t block_prepare_i_b(int, int *);
cudaError_t block_prepare_s_f(int, int *);
cudaError_t block_prepare_s_b(int, int *);
cudaError_t block_tma_launch_i_f(int, const BlockArgs &, int, int, cudaStream_t);
cudaError_t block_tma_launch_i_b(int, const BlockArgs &, int, int, cudaStream_t);
cudaError_t block_tma_launch_s_f(int, const BlockArgs &, int, int, cudaStream_t);
cudaError_t block_tma_launch_s_b(int, const BlockArgs &, int, int, cudaStream_t);

cudaError_t block_cap_launch_i_f(int, int, const BlockArgs &, cudaStream_t);
cudaError_t block_cap_launch_i_b(int, int, const BlockArgs &, cudaStream_t);
cudaError_t block_cap_launch_s_f(int, int, const BlockArgs &, cudaStream_t);
cudaError_t block_cap_launch_s_b(int, int, const BlockArgs &, cudaStream_t);
cudaError_t block_cap_prepare_i_f(int, int);
cudaError_t block_cap_prepare_i_b(int, int);
cudaError_t block_cap_prepare_s_f(int, int);
cudaError_t block_cap_prepare_s_b(int, int);

cudaError_t block_cap_launch(int log2n, int cap, int layout, int dir, const BlockArgs &a, cudaStream_t s) {
  if (layout == LAYOUT_INTERLEAVED)
    return dir < 0 ? block_cap_launch_i_f(log2n, cap, a, s) : block_cap_launch_i_b(log2n, cap, a, s);
  return dir < 0 ? block_cap_launch_s_f(log2n, cap, a, s) : block_cap_launch_s_b(log2n, cap, a, s);
}

cudaError_t block_cap_prepare(int log2n, int cap) {
  cudaError_t e;
  if ((e = block_cap_prepare_i_f(log2n, cap)) != cudaSuccess) return e;
  if ((e = block_cap_prepare_i_b(log2n, cap)) != cudaSuccess) return e;
  if ((e = block_cap_prepare_s_f(log2n, cap)) != cudaSuccess) return e;
  return block_cap_prepare_s_b(log2n, cap);
}

cudaError_t block_launch(int log2n, int layout, int dir, const BlockArgs &a, cudaStream_t s) {
  if (layout == LAYOUT_INTERLEAVED)
    return dir < 0 ? block_launch_i_f(log2n, a, s) : block_launch_i_b(log2n, a, s);
  return dir < 0 ? block_launch_s_f(log2n, a, s) : block_launch_s_b(log2n, a, s);
}

cudaError_t block_tma_launch(int log2n, int layout, int dir, const BlockArgs &a, int grid, int flags,
                             cudaStream_t s) {
  if (layout == LAYOUT_INTERLEAVED)
    return dir < 0 ? block_tma_launch_i_f(log2n, a, grid, flags, s)
                   : block_tma_launch_i_b(log2n, a, grid, flags, s);
  return dir < 0 ? block_tma_launch_s_f(log2n, a, grid, flags, s)
                 : block_tma_launch_s_b(log2n, a, grid, flags, s);
}

// Sets the smem attributes of all four (layout, direction) instances and
// returns the TMA variant's resident CTAs per SM (min over instances; 0 if
// the size has no TMA variant).
cudaError_t block_prepare(int log2n, int *tma_blocks_per_sm) {
  cudaError_t e;
  int b[4] = {0, 0, 0, 0};
  if ((e = block_prepare_i_f(log2n, &b[0])) != cudaSuccess) return e;
  if ((e = block_prepare_i_b(log2n, &b[1])) != cudaSuccess) return e;
  if ((e = block_prepare_s_f(log2n, &b[2])) != cudaSuccess) return e;
  if ((e = block_prepare_s_b(log2n, &b[3])) != cudaSuccess) return e;
  *tma_blocks_per_sm = std::min(std::min(b[0], b[1]), std::min(b[2], b[3]));
  return cudaSuccess;
}

namespace {
// persistent TMA variants exist for 256 <= N <= 2^14; N = 64 / 128 run the
// direct kernel (measured on B200: TMA 0.76-0.90 vs direct 0.79-0.99)
template <int N> bool tma_enabled_n() { return Tma1Geom<N>::ENABLED || (TmaGeom<N>::ENABLED && N >= 256); }
template <int N> void tma_geom_n(int64_t *threads, int64_t *tp, int64_t *smem) {
  if constexpr (Tma1Geom<N>::ENABLED) {
    *threads = Tma1Geom<N>::THREADS, *tp = 1, *smem = Tma1Geom<N>::BYTES;
  } else if constexpr (TmaGeom<N>::ENABLED) {
    *threads = TmaGeom<N>::THREADS, *tp = TmaGeom<N>::TP, *smem = TmaGeom<N>::BYTES;
  } else {
    *threads = *tp = *smem = 0;
  }
}
}  // namespace

bool block_tma_enabled(int log2n) {
  switch (log2n) {
  case 6: return tma_enabled_n<64>();
  case 7: return tma_enabled_n<128>();
  case 8: return tma_enabled_n<256>();
  case 9: return tma_enabled_n<512>();
  case 10: return tma_enabled_n<1024>();
  case 11: return tma_enabled_n<2048>();
  case 12: return tma_enabled_n<4096>();
  case 13: return tma_enabled_n<8192>();
  case 14: return tma_enabled_n<16384>();
  default: return false;
  }
}

bool block_tma1(int log2n) {
  switch (log2n) {
  case 13: return Tma1Geom<8192>::ENABLED;
  case 14: return Tma1Geom<16384>::ENABLED;
  default: return false;
  }
}

void block_tma_geom(int log2n, int64_t *threads, int64_t *tp, int64_t *smem) {
  *threads = *tp = *smem = 0;
  switch (log2n) {
  case 6: return tma_geom_n<64>(threads, tp, smem);
  case 7: return tma_geom_n<128>(threads, tp, smem);
  case 8: return tma_geom_n<256>(threads, tp, smem);
  case 9: return tma_geom_n<512>(threads, tp, smem);
  case 10: return tma_geom_n<1024>(threads, tp, smem);
  case 11: return tma_geom_n<2048>(threads, tp, smem);
  case 12: return tma_geom_n<4096>(threads, tp, smem);
  case 13: return tma_geom_n<8192>(threads, tp, smem);
  case 14: return tma_geom_n<16384>(threads, tp, smem);
  default: return;
  }
}

int block_tma_transforms_per_cta(int log2n) {
  int64_t th, tp, sm;
  block_tma_geom(log2n, &th, &tp, &sm);
  return (int)tp;
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

// ---- K3 group kernels ------------------------------------------------------
#include "fft_group.cuh"
#include "fft_group_tma.cuh"

namespace fftgen_b200 {

cudaError_t group_launch_f(int, int, const GroupArgs &, int64_t, cudaStream_t);
cudaError_t group_launch_b(int, int, const GroupArgs &, int64_t, cudaStream_t);
cudaError_t group_prepare_f(int);
cudaError_t group_prepare_b(int);

cudaError_t group_launch(int log2ns, int shape, int dir, const GroupArgs &a, int64_t batch, cudaStream_t s) {
  const int64_t grid = batch * a.tiles_per_outer;
  return dir < 0 ? group_launch_f(log2ns, shape, a, grid, s) : group_launch_b(log2ns, shape, a, grid, s);
}

cudaError_t group_prepare(int log2ns) {
  cudaError_t e = group_prepare_f(log2ns);
  return e != cudaSuccess ? e : group_prepare_b(log2ns);
}

cudaError_t group_tma_launch_f(int, int, const GroupTmaArgs &, int, cudaStream_t);
cudaError_t group_tma_launch_b(int, int, const GroupTmaArgs &, int, cudaStream_t);
cudaError_t group_tma_prepare_f(int, int *);
cudaError_t group_tma_prepare_b(int, int *);

cudaError_t group_tma_prepare(int log2ns, int *bps) {
  *bps = 1 << 30;
  cudaError_t e = group_tma_prepare_f(log2ns, bps);
  return e != cudaSuccess ? e : group_tma_prepare_b(log2ns, bps);
}

bool group_plane(int log2ns) {
  switch (log2ns) {
  case 10: return FFTGEN_GROUP_PLANE && GroupPlaneGeom<1024>::ENABLED;
  case 11: return FFTGEN_GROUP_PLANE && GroupPlaneGeom<2048>::ENABLED;
  case 12: return FFTGEN_GROUP_PLANE && GroupPlaneGeom<4096>::ENABLED;
  default: return false;
  }
}

cudaError_t group_tma_launch(int log2ns, int shape, int dir, const GroupTmaArgs &ta, int grid, cudaStream_t s) {
  return dir < 0 ? group_tma_launch_f(log2ns, shape, ta, grid, s) : group_tma_launch_b(log2ns, shape, ta, grid, s);
}

}  // namespace fftgen_b200

// ---- K4: device twiddle-table generation -----------------------------------
namespace fftgen_b200 {

// out[x * cols + m] = w_s^{x * row_scale * m}, computed in fp64 (sincospi of an
// exact argument, exact at quadrant multiples like unit_root, matrix.cpp:14-35)
// and rounded once to fp32.
__global__ void gen_twiddles_kernel(float2 *__restrict__ out, int64_t rows, int64_t cols, int64_t row_scale,
                                    int64_t s) {
  const int64_t total = rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = i / cols, m = i - x * cols;
    const int64_t e = (x * row_scale % s) * m % s;
    float2 w;
    if ((4 * e) % s == 0) {
      const int q = (int)(4 * e / s);
      w = q == 0 ? make_float2(1.f, 0.f) : q == 1 ? make_float2(0.f, -1.f) : q == 2 ? make_float2(-1.f, 0.f)
                                                                                     : make_float2(0.f, 1.f);
    } else {
      double sn, cs;
      sincospi(-2.0 * (double)e / (double)s, &sn, &cs);
      w = make_float2((float)cs, (float)sn);
    }
    out[i] = w;
  }
}

cudaError_t gen_twiddles(float2 *out, int64_t rows, int64_t cols, int64_t row_scale, int64_t s, cudaStream_t st) {
  const int64_t total = rows * cols;
  if (total <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 32);
  gen_twiddles_kernel<<<(unsigned)blocks, 256, 0, st>>>(out, rows, cols, row_scale, s);
  return cudaGetLastError();
}

}  // namespace fftgen_b200

// ---- distributed four-step: twiddle diagonal on a local block --------------
namespace fftgen_b200 {

// data[r * ld + c] *= w_n^{(row_offset + r) (col_offset + c)}  (conj for DIR > 0)
__global__ void twiddle_block_kernel(float2 *__restrict__ data, int64_t rows, int64_t cols, int64_t ld,
                                     int64_t row_offset, int64_t col_offset, int64_t n, int dir) {
  const int64_t total = rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const unsigned __int128 prod = (unsigned __int128)(row_offset + r) * (unsigned __int128)(col_offset + c);
    const int64_t e = (int64_t)(prod % (unsigned __int128)n);
    float wr, wi;
    if ((4 * e) % n == 0) {
      const int q = (int)(4 * e / n);
      wr = q == 0 ? 1.f : (q == 2 ? -1.f : 0.f);
      wi = q == 1 ? -1.f : (q == 3 ? 1.f : 0.f);
    } else {
      double sn, cs;
      sincospi(-2.0 * (double)e / (double)n, &sn, &cs);
      wr = (float)cs;
      wi = (float)sn;
    }
    if (dir > 0) wi = -wi;
    float2 *p = data + r * ld + c;
    const float2 x = *p;
    *p = make_float2(x.x * wr - x.y * wi, fmaf(x.x, wi, x.y * wr));
  }
}

cudaError_t twiddle_block(float2 *data, int64_t rows, int64_t cols, int64_t ld, int64_t row_offset,
                          int64_t col_offset, int64_t n, int dir, cudaStream_t s) {
  const int64_t total = rows * cols;
  if (total <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 32);
  twiddle_block_kernel<<<(unsigned)blocks, 256, 0, s>>>(data, rows, cols, ld, row_offset, col_offset, n, dir);
  return cudaGetLastError();
}

}  // namespace fftgen_b200

// ---- K5 cluster dispatch -----------------------------------------------------
#include <cuda.h>
#include <cudaTypedefs.h>

#include "cluster_instances.cuh"

namespace fftgen_b200 {

cudaError_t cluster_launch_f(int, int, int, int, const ClusterArgs &, int64_t, int, cudaStream_t);
cudaError_t cluster_launch_b(int, int, int, int, const ClusterArgs &, int64_t, int, cudaStream_t);
cudaError_t cluster_prepare_f(int, int, int, int *);
cudaError_t cluster_prepare_b(int, int, int, int *);

// Default cluster size per (l0, l1, layout), 0 = the two-launch K3 path.
// Measured on B200 (scripts/sweep.py, 1 GiB batches, TFLOP/s K5 vs K3):
//   2^15 C=8: split 13.8 vs 12.5, interleaved 14.5 vs 12.3
//   2^16 C=16: split 12.9 vs 12.6, interleaved 13.7 vs 14.4 (K3 with the TMA
//              first group: split 0.764 ms vs 0.835 ms for K5)
//   2^17 C=16: split 10.4 vs 12.0, interleaved 10.7 vs 13.2 (shape dropped: 2^17 now splits 2^9 x 2^8)
// 2^14 C=4: 14.6 vs 17.0 for the K2 block kernel (shape dropped).
int cluster_default_size(int l0, int l1, int /*layout*/) {
  switch (l0 * 16 + l1) {
  case 7 * 16 + 8: return 8;
  case 8 * 16 + 8: return 0;
  default: return 0;
  }
}

void cluster_geom(int l0, int l1, int c, int64_t *threads, int64_t *smem) {
  *threads = *smem = 0;
  switch (FFTGEN_CLUSTER_KEY(l0, l1, c)) {
#define FFTGEN_CG(A, B, NA, NB, C)                       \
  case FFTGEN_CLUSTER_KEY(A, B, C):                      \
    *threads = ClusterGeom<NA, NB, C>::THREADS;           \
    *smem = ClusterGeom<NA, NB, C>::BYTES;                \
    break;
    FFTGEN_CLUSTER_SHAPES(FFTGEN_CG)
#undef FFTGEN_CG
  default: break;
  }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
}  // namespace

cudaError_t cluster_encode_maps(int l0, int l1, int csize, int layout, ClusterArgs &a) {
  int64_t threads, smem;
  cluster_geom(l0, l1, csize, &threads, &smem);
  if (threads == 0) return cudaErrorInvalidValue;
  auto enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  const int64_t ns0 = int64_t(1) << l0, ns1 = int64_t(1) << l1, tc0 = ns1 / csize;
  const bool split = layout == LAYOUT_SPLIT;
  const int64_t w = split ? 1 : 2;  // floats per element of a plane
  // dims (innermost first): floats of a row, rows, transforms
  cuuint64_t dims[3] = {(cuuint64_t)(ns1 * w), (cuuint64_t)ns0, (cuuint64_t)a.batch};
  cuuint64_t strides[2] = {(cuuint64_t)(ns1 * w * 4), (cuuint64_t)(a.idist * w * 4)};
  cuuint32_t box[3] = {(cuuint32_t)(tc0 * w), (cuuint32_t)ns0, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const void *planes[2] = {a.in0, split ? a.in1 : a.in0};
  for (int i = 0; i < (split ? 2 : 1); ++i) {
    CUresult r = enc(reinterpret_cast<CUtensorMap *>(a.tmap[i]), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                     const_cast<void *>(planes[i]), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  // outputs: rows e of NS0 elements, boxes {TC1 columns, NS1 rows}
  const int64_t tc1 = ns0 / csize;
  cuuint64_t odims[3] = {(cuuint64_t)(ns0 * w), (cuuint64_t)ns1, (cuuint64_t)a.batch};
  cuuint64_t ostrides[2] = {(cuuint64_t)(ns0 * w * 4), (cuuint64_t)(a.odist * w * 4)};
  cuuint32_t obox[3] = {(cuuint32_t)(tc1 * w), (cuuint32_t)ns1, 1};
  void *oplanes[2] = {a.out0, split ? a.out1 : a.out0};
  for (int i = 0; i < (split ? 2 : 1); ++i) {
    CUresult r = enc(reinterpret_cast<CUtensorMap *>(a.omap[i]), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, oplanes[i],
                     odims, ostrides, obox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

cudaError_t cluster_prepare(int l0, int l1, int c, int *max_clusters) {
  int a = 0, b = 0;
  cudaError_t e = cluster_prepare_f(l0, l1, c, &a);
  if (e == cudaSuccess) e = cluster_prepare_b(l0, l1, c, &b);
  *max_clusters = a < b ? a : b;
  return e;
}

cudaError_t cluster_launch(int l0, int l1, int c, int layout, int dir, const ClusterArgs &a, int64_t batch,
                           int max_clusters, cudaStream_t s) {
  return dir < 0 ? cluster_launch_f(l0, l1, c, layout, a, batch, max_clusters, s)
                 : cluster_launch_b(l0, l1, c, layout, a, batch, max_clusters, s);
}

}  // namespace fftgen_b200

namespace fftgen_b200 {

bool encode_tile_maps(const GroupArgs &a, int log2ns, int shape, int64_t batch, int64_t tc,
                      unsigned char (*tmap)[128]) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const int64_t ns = int64_t(1) << log2ns;
  const bool rows = shape == 2 || shape == 3;
  const bool split_in = shape == 1;
  const int64_t w = split_in ? 1 : 2;  // floats per element of an input plane
  const void *planes[2] = {a.in0, split_in ? a.in1 : a.in0};
  const int nplanes = split_in ? 2 : 1;
  for (int i = 0; i < nplanes; ++i)
    if ((uintptr_t)planes[i] % 16 != 0) return false;
  if ((a.idist * w * 4) % 16 != 0) return false;
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
  if (rows) {  // [batch][cols rows][NS*2 floats] as {CH floats, chunks, rows, batch}
    const int64_t ch = std::min<int64_t>(ns * 2, 256), nch = ns * 2 / ch;
    dims[0] = ch; dims[1] = nch; dims[2] = a.cols; dims[3] = batch;
    strides[0] = ch * 4; strides[1] = ns * 8; strides[2] = a.idist * 8;
    box[0] = ch; box[1] = nch; box[2] = tc; box[3] = 1;
  } else {     // [batch][cols][NS][k] as {k*w floats, NS, cols, batch}
    if ((a.k * w * 4) % 16 != 0) return false;
    dims[0] = a.k * w; dims[1] = ns; dims[2] = a.cols; dims[3] = batch;
    strides[0] = a.k * w * 4; strides[1] = ns * a.k * w * 4; strides[2] = a.idist * w * 4;
    box[0] = tc * w; box[1] = std::min<int64_t>(ns, 256); box[2] = 1; box[3] = 1;
  }
  for (int i = 0; i < nplanes; ++i) {
    CUresult r = enc(reinterpret_cast<CUtensorMap *>(tmap[i]), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                     const_cast<void *>(planes[i]), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
  }
  return true;
}

// tensor maps of a's output for the staged tile stores of fft_group_tma_kernel
// (FFTGEN_GROUP_TMA_STORE): rows (last group) {cols*w floats, NS, batch, 1},
// columns (interleaved scratch) {k*2 floats, cols, NS, batch}
bool encode_out_maps(const GroupArgs &a, int log2ns, int shape, int64_t batch, int64_t tc,
                     unsigned char (*omap)[128]) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const int64_t ns = int64_t(1) << log2ns, ch = std::min<int64_t>(ns, 256);
  const bool rows = shape == 2 || shape == 3;
  const bool split_out = shape == 3;
  const int64_t w = split_out ? 1 : 2;
  void *planes[2] = {a.out0, split_out ? a.out1 : a.out0};
  const int nplanes = split_out ? 2 : 1;
  for (int i = 0; i < nplanes; ++i)
    if ((uintptr_t)planes[i] % 16 != 0) return false;
  if ((a.odist * w * 4) % 16 != 0) return false;
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4], estr[4] = {1, 1, 1, 1};
  if (rows) {
    if ((a.cols * w * 4) % 16 != 0) return false;
    dims[0] = a.cols * w; dims[1] = ns; dims[2] = batch; dims[3] = 1;
    strides[0] = a.cols * w * 4; strides[1] = a.odist * w * 4; strides[2] = a.odist * w * 4 * batch;
    box[0] = tc * w; box[1] = ch; box[2] = 1; box[3] = 1;
  } else {
    if ((a.k * 2 * 4) % 16 != 0) return false;
    dims[0] = a.k * 2; dims[1] = a.cols; dims[2] = ns; dims[3] = batch;
    strides[0] = a.k * 8; strides[1] = a.cols * a.k * 8; strides[2] = a.odist * 8;
    box[0] = tc * 2; box[1] = 1; box[2] = ch; box[3] = 1;
  }
  for (int i = 0; i < nplanes; ++i) {
    CUresult r = enc(reinterpret_cast<CUtensorMap *>(omap[i]), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, planes[i], dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
  }
  return true;
}

bool group_tma_stores(int log2ns, int shape) {
  const bool rows = shape == 2 || shape == 3;
  const int lin = shape == 0 ? LAYOUT_INTERLEAVED : (shape == 1 ? LAYOUT_SPLIT : LAYOUT_SCRATCH);
  const int lout = shape == 2 ? LAYOUT_INTERLEAVED : (shape == 3 ? LAYOUT_SPLIT : LAYOUT_SCRATCH);
  return group_plane(log2ns) ? group_plane_store_rt(1 << log2ns, rows, lout) : group_tma_store_rt(1 << log2ns, rows, lin);
}

bool group_tma_encode(int log2ns, int shape, int64_t batch, GroupTmaArgs &ta) {
  int64_t threads, tc, smem, r0;
  group_geom(log2ns, &threads, &tc, &smem, &r0);
  if (!encode_tile_maps(ta.g, log2ns, shape, batch, tc, ta.tmap)) return false;
  // the plane kernel (NS >= 2^11) stores from registers
  if (group_tma_stores(log2ns, shape)) return encode_out_maps(ta.g, log2ns, shape, batch, tc, ta.omap);
  return true;
}

}  // namespace fftgen_b200

