// plan.hpp -- host-side plan builder (C++), the B200 replacement for the
// reference's compile_pipeline (proj/src/driver.cpp:11-34).
//
// It restates, for introspection and index parity, the reference planners
// and sparse fusion (formula.cpp:150-197, rewrite.cpp:46-184) as a compact
// operator list, and derives from N the sm_100a execution: either one
// shared-memory-resident kernel (K2, N <= 2^14) or a four-step of two such
// kernels (K3, 2^15 <= N <= 2^28).  Twiddles are generated in fp64 with the
// reference's unit_root formula (matrix.cpp:14-35) and rounded to fp32 once,
// at plan time.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace fftgen_b200 {

// Mirrors of the reference's error classes (error.hpp:16-71); the C ABI maps
// them to fftgen_status codes and fftgen.hpp maps the codes back.
struct PlanError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DimensionError : std::runtime_error { using std::runtime_error::runtime_error; };
struct FuseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ExecError : std::runtime_error { using std::runtime_error::runtime_error; };
struct LowerError : std::runtime_error { using std::runtime_error::runtime_error; };

// Sets the calling thread's fftgen_last_error() text (capi.cpp).
void set_last_error(const std::string &msg);

// The reference's CPU schedule options (PipelineConfig.vec / vector_width /
// tile), validated like vectorize() / tile() (transforms.cpp:85-95, 351-354).
void check_schedule(int vec, int64_t vector_width, int tile_kind, int64_t tile_value);

enum OpKind { OP_MKIV = 0, OP_IKMV = 1, OP_PKIV = 2, OP_TWIDDLE = 3, OP_PERMUTE = 4 };

// One fused operator in the reference's application order (rewrite.hpp:24-52).
// TwiddleMul coefficients are described, not stored: coefficient i is
// unit_root(tw_total, kk*mm) with b = (i mod tw_total*tw_repeat) / tw_repeat,
// kk = b / tw_block, mm = b mod tw_block.
struct RefOp {
  int kind;
  int64_t p0, p1, p2;
  int64_t tw_total, tw_block, tw_repeat;
};

// exp(-2 pi i t / n) in fp64, exact at quadrant multiples (matrix.cpp:14-35).
void unit_root(int64_t n, int64_t t, double *re, double *im);

std::vector<int64_t> stockham_radices(int64_t n, int64_t radix);
std::vector<RefOp> fuse_ops(int64_t n, int algorithm, int64_t radix);
std::string pipeline_text(const std::vector<RefOp> &ops, int64_t n);
// print_formula(plan_cooley_tukey / plan_stockham (n, radix)) (formula.cpp:104-197)
std::string formula_text(int64_t n, int algorithm, int64_t radix);
void op_map(const RefOp &op, int64_t n, int64_t *map, int64_t *s_out);

// One execution pass: a radix-R Stockham stage over the whole transform.
struct PassDesc {
  int64_t R, cols, k, s;
};

enum Strategy { STRAT_IDENTITY = 0, STRAT_BLOCK = 1, STRAT_FOURSTEP = 2 };

// One K3 group (fft_group.cuh): a radix-NS Stockham stage of the whole
// transform with global (cols, k); `rows` for the last group (k == 1).
struct GroupDesc {
  int log2ns = 0;
  int64_t ns = 0, cols = 0, k = 0, s = 0;
  int64_t r0 = 0;           // first pass radix of the NS-point sub-FFT
  int64_t tc = 0;           // transforms per CTA tile
  bool rows = false;
  int64_t local_off = 0;    // float2 offset of the NS-point pass tables
  int64_t q_off = 0, p_off = 0;  // float2 offsets of Q[A0][m], P[c][m] (cols > 1)
};

struct ExecPlan {
  int64_t n = 0;
  int block_cap = 0;  // K2: pass-radix cap in effect (0 = the default plan)
  Strategy strategy = STRAT_BLOCK;
  int log2n = 0;
  std::vector<PassDesc> passes;
  // host copies of the fp32 twiddle tables (uploaded by the C ABI)
  std::vector<float> tw_block;   // K2 pass tables of the single kernel / per-NS group tables
  // K3: groups and the device-generated Q/P table size (float2 count)
  std::vector<GroupDesc> groups;
  int64_t tw_group_len = 0;
  int scratch_buffers = 0;       // intermediate N-element buffers per transform
};

// The group split of log2 N used by the four-step path (2..4 groups of
// 2^7..2^12 points).
enum SplitMode { SPLIT_DEFAULT = 0, SPLIT_GROUPS_1024 = 1, SPLIT_TWO_PASS = 2 };
// layout: 0 interleaved, 1 split (the default split depends on it at 2^23)
std::vector<int> group_split(int log2n, int mode = SPLIT_DEFAULT, int layout = 0);
// whether a group runs the persistent TMA-tile kernel by default (measured)
bool group_prefers_tma(int log2ns, bool first, bool rows, int64_t cols = 0);
void group_geom(int log2ns, int64_t *threads, int64_t *tc, int64_t *smem, int64_t *r0);

ExecPlan build_exec_plan(int64_t n, int split_mode = SPLIT_DEFAULT, int pass_radix = 0, int layout = 0);
// the sm_100a pass / group program as loop nests (the --emit loops text)
std::string program_text(int64_t n, int split_mode = SPLIT_DEFAULT, int pass_radix = 0, int layout = 0);

// K2 pass structure of an N-point block kernel (defined in kernels_common.cu
// from the compile-time BlockPlan), and its [A][m] twiddle table in floats.
// cap: the pass-radix hint (0 = default; 8 / 16 / 32 select the capped plan
// where block_cap_distinct says it differs from the default)
int block_num_passes(int log2n, int cap = 0);
void block_pass(int log2n, int p, int64_t *R, int64_t *cols, int64_t *k, int cap = 0);
std::vector<float> block_twiddles(int log2n, int cap = 0);
bool block_cap_distinct(int log2n, int cap);
std::vector<float> group_twiddles(int log2ns);

}  // namespace fftgen_b200
