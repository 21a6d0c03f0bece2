/* include/fftgen_b200.h -- the drop-in C ABI of the B200 FFT hot path.
 *
 * Replaces the reference's plan -> execute path (arxiv 2308.00497,
 * /root/reference/proj):
 *
 *   reference                                          here
 *   ---------------------------------------------     -------------------------------
 *   PipelineConfig            include/fftgen/driver.hpp:26-35   fftgen_config
 *   compile_pipeline()        include/fftgen/driver.hpp:44-45   fftgen_plan_create()
 *   CompiledPipeline          include/fftgen/driver.hpp:37-42   fftgen_plan (opaque)
 *   interpret()               include/fftgen/exec.hpp:26-27     fftgen_execute() (device buffers)
 *                                                               fftgen_execute_host() (host fp32)
 *                                                               fftgen_interpret_f64() (ComplexBuffer storage)
 *   emitted C ABI fft()       src/emit_c.cpp:88                 fftgen_interpret_f64()
 *   print_pipeline()          include/fftgen/rewrite.hpp:91-92  fftgen_plan_pipeline_text()
 *   fftgen::Error hierarchy   include/fftgen/error.hpp:16-71    fftgen_status codes
 *
 * Extensions the north star requires: a batch count, an inverse direction,
 * fp32 storage, two complex layouts with caller-owned device pointers and a
 * CUDA stream.  Plain pointers and integers only; no torch / C++ types.
 *
 * Semantics:
 *   forward  X[j] = sum_k x[k] exp(-2 pi i jk/N)   (unit_root, matrix.cpp:14-35)
 *   inverse  X[j] = sum_k x[k] exp(+2 pi i jk/N)   unnormalised (FFTW/cuFFT convention)
 *   interleaved: transform b, element e at ((float2*)in0)[b*dist + e]
 *   split:       re at in0[b*dist + e], im at in1[b*dist + e]
 *                (dist = n: planar arrays; the reference ComplexBuffer's
 *                 [re n | im n] block per transform is in1 = in0 + n, dist = 2n)
 *   out-of-place, or exactly in place (out0 == in0, out1 == in1); partially
 *   overlapping input and output ranges are rejected with FFTGEN_ERR_EXEC.
 *   Kernels are enqueued on the caller's stream; the plan owns its twiddle
 *   tables and scratch, all allocated at plan creation (an execute never
 *   allocates, so executes can be captured in CUDA graphs).  Plan creation
 *   and destruction are thread-safe; a plan may be executed concurrently from
 *   several host threads on different streams only when its executes use no
 *   scratch: block (N <= 2^14) plans, and cluster plans (2^15) on 16-byte
 *   aligned data with dist * element size a multiple of 16 (unaligned data
 *   takes the two-launch path through the plan's bounded fallback scratch).
 */
#ifndef FFTGEN_B200_H
#define FFTGEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFTGEN_B200_ABI_VERSION 3

typedef struct fftgen_plan fftgen_plan;

/* Status codes.  fftgen_b200.hpp maps them back onto the reference's exception
 * classes (error.hpp:16-71): PLAN -> PlanError, DIMENSION -> DimensionError,
 * FUSE -> FuseError, LOWER -> LowerError, BOUNDS -> BoundsError, GPUMAP ->
 * GpuMapError, EXEC/CUDA/NOMEM -> ExecError, INVALID -> DimensionError. */
typedef enum {
  FFTGEN_OK = 0,
  FFTGEN_ERR_PLAN = 1,      /* non-power-of-two n, bad radix, size cap      (PlanError) */
  FFTGEN_ERR_DIMENSION = 2, /* sizes / dist / batch do not line up          (DimensionError) */
  FFTGEN_ERR_EXEC = 3,      /* bad layout / direction / pointer at execute  (ExecError) */
  FFTGEN_ERR_FUSE = 4,      /* radix above the kernel cap 64                (FuseError) */
  FFTGEN_ERR_INVALID = 5,   /* NULL handle or config                        */
  FFTGEN_ERR_CUDA = 6,      /* CUDA runtime failure (device, launch)        */
  FFTGEN_ERR_NOMEM = 7,     /* device allocation failed                     */
  FFTGEN_ERR_LOWER = 8,     /* rejected schedule option (vector width,
                               tile size)                                   (LowerError) */
  FFTGEN_ERR_BOUNDS = 9,    /* a buffer is shorter than the plan's access
                               range (batch, dist)                          (BoundsError) */
  FFTGEN_ERR_GPUMAP = 10    /* no sm_100a launch geometry for the plan on
                               this device (kernel attributes, occupancy)   (GpuMapError) */
} fftgen_status;

enum { FFTGEN_LAYOUT_INTERLEAVED = 0, FFTGEN_LAYOUT_SPLIT = 1 };     /* ComplexLayout, loopir.hpp:187 */
enum { FFTGEN_ALG_COOLEY_TUKEY = 0, FFTGEN_ALG_STOCKHAM = 1 };       /* Algorithm, driver.hpp:21 */
enum { FFTGEN_FORWARD = -1, FFTGEN_INVERSE = 1 };
enum { FFTGEN_VEC_NONE = 0, FFTGEN_VEC_INNER = 1, FFTGEN_VEC_OUTER = 2 };  /* VecMode, driver.hpp:23 */
enum { FFTGEN_TILE_NONE = 0, FFTGEN_TILE_EXACT = 1, FFTGEN_TILE_CACHE = 2 }; /* TilePolicy, loopir.hpp:240-248 */

/* Kernel-selection tuning bits (fftgen_config.tuning).  0 selects the
 * measured-fastest kernels; the bits reproduce the
 * alternatives for A/B measurement and for the bitwise-equality tests. */
enum {
  FFTGEN_TUNE_NO_TMA = 1,        /* N <= 2^14: the direct block kernel; four-step groups: plain tiles */
  FFTGEN_TUNE_NO_TMA_STORE = 2,  /* block kernels: register stores instead of bulk stores */
  FFTGEN_TUNE_GROUP_TMA_ALL = 4, /* every four-step group as the persistent TMA-tile kernel */
  FFTGEN_TUNE_GROUPS_1024 = 8,   /* four-step groups of at most 2^10 points (three passes from 2^21) */
  FFTGEN_TUNE_TWO_PASS = 16      /* two four-step groups up to 2^24 (NS = 2^11 / 2^12 tiles) */
};

typedef struct {
  int64_t n;          /* transform size, power of two >= 1                    (PipelineConfig.n) */
  int32_t algorithm;  /* FFTGEN_ALG_*; selects the reference op list that
                         introspection reports (default Cooley-Tukey, like
                         PipelineConfig.algorithm); execution always uses the
                         self-sorting Stockham passes                         */
  int32_t radix;      /* power of two >= 2 (PipelineConfig.radix, default 2)   */
  int32_t layout;     /* FFTGEN_LAYOUT_*                                  (PipelineConfig.layout) */
  int32_t device;     /* CUDA device ordinal                                   */
  int64_t batch;      /* transforms per execute, >= 1                          */
  /* The reference's CPU loop-IR schedule (PipelineConfig.vec / vector_width /
   * interleaved_opt / tile, driver.hpp:26-35).  Validated like
   * vectorize() / tile() (transforms.cpp: LowerError for a vector width that
   * is not a power of two <= 64 or a non-positive tile size) and otherwise
   * result-neutral: the reference guarantees vectorized, tiled and scalar
   * programs agree bitwise, and the sm_100a passes have their own schedule. */
  int32_t vec;             /* FFTGEN_VEC_*                    (default NONE) */
  int32_t vector_width;    /* lanes                           (default 8)    */
  int32_t interleaved_opt; /* 0 / 1                           (default 0)    */
  int32_t tile_kind;       /* FFTGEN_TILE_*                   (default NONE) */
  int64_t tile_value;      /* tile size or cache byte budget                 */
  /* Kernel selection (B200 extension, not in the reference) */
  uint32_t tuning;         /* FFTGEN_TUNE_* bits, 0 = measured defaults      */
  int32_t cluster_size;    /* single-pass cluster kernel for N = 2^15 / 2^16:
                              0 = measured default, -1 = never (two launches),
                              or a compiled size (4, 8, 16)                  */
  int32_t host_chunk_mb;   /* fftgen_execute_host chunk (in + out per slot),
                              0 = 128 MiB                                    */
  int32_t pass_radix;      /* radix hint for the sm_100a register passes of
                              N <= 2^14: 0 = the measured default plan (radix 8
                              at 2^7 .. 2^9, radix <= 64 elsewhere); 8, 16, 32
                              = passes of at most that radix in the
                              reference's Stockham shape (remainder radix
                              first) where that takes <= 3 passes and differs
                              from the radix-64 plan (N = 2^7 .. 2^12); 64 =
                              the radix-<=64 two / three-pass plans (with the
                              TMA kernels).  Four-step sizes ignore it.      */
} fftgen_config;

/* Fills the PipelineConfig defaults (driver.hpp:26-35) plus batch=1, device=0. */
void fftgen_config_init(fftgen_config *cfg);

/* Plan creation (compile_pipeline).  Validates like plan_cooley_tukey /
 * plan_stockham (formula.cpp:150-197): PlanError for a non-power-of-two n or a
 * radix that is not a power of two >= 2, FuseError for radix > 64 when n > 64.
 * Builds the execution passes and uploads the fp64-accurate fp32 twiddle
 * tables to `device`. */
fftgen_status fftgen_plan_create(fftgen_plan **out, const fftgen_config *cfg);
fftgen_status fftgen_plan_destroy(fftgen_plan *plan);

/* Execute on device buffers (the hot path).  `dist` is in complex elements
 * for interleaved and in floats for split; dist >= n.  `stream` is a
 * cudaStream_t (NULL = legacy default stream). */
fftgen_status fftgen_execute(const fftgen_plan *plan, int direction,
                             const void *in0, const void *in1,
                             void *out0, void *out1, int64_t dist, void *stream);

/* Execute on HOST fp32 buffers with the same addressing as fftgen_execute.
 * Host->device copies, kernels and device->host copies are pipelined in
 * chunks over two streams; pinned host memory gives full PCIe bandwidth.
 * Blocks until the result is in `out`. */
fftgen_status fftgen_execute_host(const fftgen_plan *plan, int direction,
                                  const float *in0, const float *in1,
                                  float *out0, float *out1, int64_t dist);

/* interpret() drop-in on the reference's own storage: `batch` consecutive
 * ComplexBuffers of 2n doubles each in the plan's layout (interleaved:
 * (re,im) pairs; split: [re n | im n]).  Values are rounded to fp32 on the
 * device, transformed in fp32 and widened back.  Also the batched analogue of
 * the emitted `void fft(const double *in, double *out, long n)`. */
fftgen_status fftgen_interpret_f64(const fftgen_plan *plan, int direction,
                                   const double *in, double *out);

/* Distributed four-step helper (the twiddle diagonal D^N of Eq. 1,
 * formula.hpp:44-49, applied to one rank's block): for an interleaved fp32
 * block of `rows` x `cols` complex values with leading dimension `ld`,
 *   data[r*ld + c] *= w_n^{(row_offset + r) * (col_offset + c)}
 * (w_n = exp(-2 pi i / n); conjugated for FFTGEN_INVERSE), twiddles
 * computed in fp64 on the device, exact at quadrant multiples. */
fftgen_status fftgen_twiddle_multiply(int direction, void *data, int64_t rows, int64_t cols, int64_t ld,
                                      int64_t row_offset, int64_t col_offset, int64_t n, void *stream);

/* ---- distributed four-step: ONE n-point transform over `world` ranks ----
 * (config C5; the reference's two-factor split formula.cpp:160-165
 * with K = world, M = n/world).  Interleaved fp32 complex only.  Rank r holds
 * x[r M : (r+1) M] and ends with X[r M : (r+1) M] (natural order).  Every
 * exchange is an all-to-all of `world` CONTIGUOUS chunks of n/world^2
 * elements (chunk q of the send buffer goes to rank q and lands as chunk r of
 * its receive buffer: ncclSend/ncclRecv in a group, all_to_all_single):
 *
 *   exchange(in -> w0); butterfly(w0 -> w1); exchange(w1 -> w0);
 *   local(w0 -> w1);    exchange(w1 -> w0);  unpack(w0 -> out)
 *
 * The P-point butterfly applies the twiddle diagonal D^N and stores in the
 * per-peer chunk order (no pack copy); the local stage is the single-GPU
 * plan of size n/world; unpack is the final stride-`world` interleave.
 * Buffers are n/world elements, 16-byte aligned, pairwise disjoint. */
typedef struct fftgen_dist_plan fftgen_dist_plan;
/* PlanError: n not a power of two or n/world > 2^30; DimensionError: world not
 * 1/2/4/8/16, rank outside [0, world), or n < 2*world^2. */
fftgen_status fftgen_dist_plan_create(fftgen_dist_plan **out, int64_t n, int world, int rank, int device);
fftgen_status fftgen_dist_plan_destroy(fftgen_dist_plan *plan);
fftgen_status fftgen_dist_butterfly(const fftgen_dist_plan *plan, int direction, const void *recv, void *send,
                                    void *stream);
fftgen_status fftgen_dist_local(const fftgen_dist_plan *plan, int direction, const void *in, void *out,
                                void *stream);
fftgen_status fftgen_dist_unpack(const fftgen_dist_plan *plan, const void *recv, void *out, void *stream);
/* All-to-all callback: `world` chunks of chunk_bytes, send -> recv, enqueued
 * on (or ordered after) `stream`; returns 0 on success. */
typedef int (*fftgen_exchange_fn)(void *ctx, const void *send, void *recv, size_t chunk_bytes, void *stream);
/* The whole pipeline above on one rank with the caller's exchange. */
fftgen_status fftgen_dist_execute(const fftgen_dist_plan *plan, int direction, const void *in, void *out,
                                  void *work0, void *work1, fftgen_exchange_fn exchange, void *ctx, void *stream);
/* Cyclic (transposed) output order: exchange, butterfly,
 * exchange, local plan only -- out[j] = X[rank + world*j] for j < n/world,
 * two exchanges instead of three and no unpack.  `work1` is not used. */
fftgen_status fftgen_dist_execute_cyclic(const fftgen_dist_plan *plan, int direction, const void *in, void *out,
                                         void *work0, void *work1, fftgen_exchange_fn exchange, void *ctx,
                                         void *stream);
/* Peer-memory transport: every rank's blocks are mapped into this process
 * (CUDA IPC / symmetric memory over NVLink, or plain device buffers when the
 * ranks are emulated on one GPU) and the exchanges run inside the kernels:
 *   butterfly_peers: reads chunk `rank` of every rank's input block
 *     (in_blocks[r], exchange 1 as loads) and writes row k_b into slot `rank`
 *     of rank k_b's receive block (recv_blocks[k_b], exchange 2 as stores);
 *   local (fftgen_dist_local) on the rank's own receive block -> z;
 *   unpack_peers: reads slot `rank` of every rank's z block (z_blocks[q'],
 *     exchange 3 as loads) into the rank's natural-order output.
 * Tables hold `world` device pointers; the caller orders the stages across
 * ranks (a barrier between them when the ranks are separate processes). */
fftgen_status fftgen_dist_butterfly_peers(const fftgen_dist_plan *plan, int direction, const void *const *in_blocks,
                                          void *const *recv_blocks, void *stream);
fftgen_status fftgen_dist_unpack_peers(const fftgen_dist_plan *plan, const void *const *z_blocks, void *out,
                                       void *stream);
/* Elements per exchange chunk (n/world^2) and the rank's block (n/world). */
int64_t fftgen_dist_chunk_elems(const fftgen_dist_plan *plan);
int64_t fftgen_dist_block_elems(const fftgen_dist_plan *plan);
/* The local n/world-point plan (for describe / launch accounting). */
const fftgen_plan *fftgen_dist_local_plan(const fftgen_dist_plan *plan);

/* The reference's synthetic input seeded_input(n, seed) (verify.cpp:55-78:
 * splitmix64, re/im uniform in [-1, 1)) generated on `device` for `batch`
 * transforms, transform b with seed seed0 + b, rounded once to fp32 (bitwise
 * the host generator's values cast to float), written in `layout` with the
 * fftgen_execute addressing (out1 = im plane for split). */
fftgen_status fftgen_seeded_input(int layout, int64_t n, int64_t batch, uint64_t seed0, void *out0, void *out1,
                                  int64_t dist, int device, void *stream);

const char *fftgen_error_string(fftgen_status status);
/* Detail message of the most recent failure on the calling thread. */
const char *fftgen_last_error(void);
int fftgen_abi_version(void);

/* ---- introspection (parity of plan indices) -------------------------- */
/* Reference Stockham stage radices in application order (formula.cpp:182-195).
 * Returns the count; copies at most cap entries. */
int fftgen_plan_radices(const fftgen_plan *plan, int64_t *radices, int cap);
/* The reference's fused operator list for (n, algorithm, radix)
 * (rewrite.cpp:94-184), one op per entry: desc = {kind, p0, p1, p2} with kind
 * 0 FusedMKIV(m, copies) 1 FusedIKMV(n, copies) 2 FusedPKIV(m, total, k)
 * 3 TwiddleMul(len) 4 Permute(m, total). */
int fftgen_plan_num_ops(const fftgen_plan *plan);
fftgen_status fftgen_plan_op(const fftgen_plan *plan, int idx, int64_t desc[4]);
/* Source-index map of a data-movement op (y[o] = x[map[o]]), or the w_s
 * exponent of every coefficient of a TwiddleMul (with *s_out = s). */
fftgen_status fftgen_plan_op_map(const fftgen_plan *plan, int idx, int64_t *map, int64_t *s_out);
/* print_pipeline() text of the op list (rewrite.cpp:275-296). */
fftgen_status fftgen_plan_pipeline_text(const fftgen_plan *plan, char *buf, size_t cap);
/* The sm_100a execution: passes (radix R, cols, k) and launches. */
int fftgen_plan_num_passes(const fftgen_plan *plan);
fftgen_status fftgen_plan_pass(const fftgen_plan *plan, int idx, int64_t desc[4]);
fftgen_status fftgen_plan_describe(const fftgen_plan *plan, char *buf, size_t cap);
/* Host-only program texts for a config (no device touched; validates like
 * fftgen_plan_create: PlanError / FuseError / LowerError):
 *   FFTGEN_TEXT_FORMULA   print_formula of plan_cooley_tukey / plan_stockham
 *                         (formula.cpp:104-197), byte-identical to the reference
 *   FFTGEN_TEXT_PIPELINE  print_pipeline of the fused op list (rewrite.cpp:275-296)
 *   FFTGEN_TEXT_LOOPS     the sm_100a pass / group program as loop nests
 *   FFTGEN_TEXT_RADICES   the Stockham radices, application order */
enum { FFTGEN_TEXT_FORMULA = 0, FFTGEN_TEXT_PIPELINE = 1, FFTGEN_TEXT_LOOPS = 2, FFTGEN_TEXT_RADICES = 3 };
fftgen_status fftgen_program_text(const fftgen_config *cfg, int what, char *buf, size_t cap);
/* The device-generated twiddle tables of four-step group `group` (K4; parity
 * introspection): which 0 = Q[A0][m] = w_s^{A0 (NS/R0) m} (R0 x cols), which 1
 * = P = w_s^{c m} ([c][m] for column groups, [m][c] for the rows group),
 * copied to `out` as (re, im) float pairs, at most `cap` elements.  Returns the
 * table's element count, 0 for a group without a table (cols == 1), -1 on a
 * bad argument. */
int64_t fftgen_plan_group_twiddles(const fftgen_plan *plan, int group, int which, float *out, int64_t cap);
/* Kernel launches one fftgen_execute issues (for launch accounting). */
int fftgen_plan_launches(const fftgen_plan *plan);
size_t fftgen_plan_scratch_bytes(const fftgen_plan *plan);

#ifdef __cplusplus
}
#endif
#endif /* FFTGEN_B200_H */
