// include/fftgen_b200.hpp -- C++ host API over the C ABI (include/fftgen_b200.h).
//
// Source-compatible with the reference's public plan -> execute API in
// proj/include/fftgen (driver.hpp, exec.hpp, error.hpp and the ComplexBuffer /
// TilePolicy types of loopir.hpp): the same names, fields, argument meaning
// and exception classes, so code written against
//
//   CompiledPipeline c = compile_pipeline(config);
//   ComplexBuffer y = interpret(c.final_ir, ComplexBuffer::from_vector(x, layout), opts);
//
// compiles unchanged against this header (the reference's own
// tests/test_exec.cpp known-answer cases do: tests/cpp/refshim +
// tests/test_cpp_api.py) and runs the sm_100a kernels.
//
//   reference (file:line)                          here
//   Error / ParseError / DimensionError /          same classes (error.hpp:16-71)
//     PlanError / FuseError / LowerError /
//     ExecError / BoundsError / GpuMapError
//   Algorithm, VecMode (driver.hpp:21-23)          same enums
//   ComplexLayout, TilePolicy (loopir.hpp:187,240) same
//   PipelineConfig (driver.hpp:26-35)              same fields + batch, device, tuning
//   CompiledPipeline {formula, fused, complex_ir,  same members (driver.hpp:37-42); the
//     final_ir} (driver.hpp:37-42)                 LoopProgram is the device plan handle
//   compile_pipeline (driver.hpp:44-45)            same; validates like the reference
//   algorithm_name / layout_name / vec_mode_name   same (driver.hpp:47-52)
//   ExecOptions {threads} (exec.hpp:16-21)         same + direction (the reference is forward-only)
//   interpret(LoopProgram, ComplexBuffer,          same (exec.hpp:26-27): fp64 storage in/out,
//     ExecOptions) (exec.hpp:26-27)                fp32 on the GPU; ExecError on a length or
//                                                  layout mismatch (interpret.cpp:46-63)
//   ComplexBuffer (loopir.hpp:215-228)             same storage contract
//
// plus device-pointer execution (CompiledPipeline::execute) with a direction
// and a CUDA stream, and a batched interpret.  Header-only; no CUDA headers.
#ifndef FFTGEN_B200_HPP
#define FFTGEN_B200_HPP

#include <algorithm>
#include <complex>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "fftgen_b200.h"

namespace fftgen {

using cplx = std::complex<double>;

// ---- error.hpp:16-71 ---------------------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string &msg) : std::runtime_error(msg) {}
};
class ParseError : public Error {  // malformed formula text, 1-based position
 public:
  ParseError(const std::string &msg, int line, int column)
      : Error(std::to_string(line) + ":" + std::to_string(column) + ": " + msg), line(line), column(column) {}
  int line;
  int column;
};
class DimensionError : public Error {
 public:
  using Error::Error;
};
class PlanError : public Error {
 public:
  using Error::Error;
};
class FuseError : public Error {
 public:
  using Error::Error;
};
class LowerError : public Error {
 public:
  using Error::Error;
};
class ExecError : public Error {
 public:
  using Error::Error;
};
class BoundsError : public Error {
 public:
  using Error::Error;
};
class GpuMapError : public Error {
 public:
  using Error::Error;
};

// ---- driver.hpp:21-35, loopir.hpp:187 / 240-248 -------------------------------
enum class Algorithm { CooleyTukey, Stockham };
enum class VecMode { None, Inner, Outer };
enum class ComplexLayout { Interleaved, Split };
enum class Direction { Forward = FFTGEN_FORWARD, Inverse = FFTGEN_INVERSE };

struct TilePolicy {
  enum Kind { ExactSize, CacheVolume } kind = ExactSize;
  int64_t value = 0;  // tile size or byte budget
  static TilePolicy exact(int64_t t) { return {ExactSize, t}; }
  static TilePolicy cache(int64_t bytes = 32 * 1024) { return {CacheVolume, bytes}; }
};

struct PipelineConfig {
  int64_t n = 0;
  Algorithm algorithm = Algorithm::CooleyTukey;
  int64_t radix = 2;
  ComplexLayout layout = ComplexLayout::Interleaved;
  // the reference's CPU loop-IR schedule: validated like vectorize() / tile()
  // (LowerError), result-neutral on the GPU (the reference guarantees
  // scheduled and scalar programs agree bitwise)
  VecMode vec = VecMode::None;
  int64_t vector_width = 8;
  bool interleaved_opt = false;
  std::optional<TilePolicy> tile;
  // B200 extensions
  int64_t batch = 1;      // transforms per execute
  int device = 0;         // CUDA device ordinal
  uint32_t tuning = 0;    // FFTGEN_TUNE_* kernel-selection bits (0 = measured defaults)
  int pass_radix = 0;     // radix hint for the register passes (fftgen_config.pass_radix)
};

inline std::string algorithm_name(Algorithm a) { return a == Algorithm::CooleyTukey ? "cooley-tukey" : "stockham"; }
inline std::string layout_name(ComplexLayout l) { return l == ComplexLayout::Interleaved ? "interleaved" : "split"; }
// "none", "inner", "outer", "inner-opt", "outer-opt" (driver.cpp:44-51)
inline std::string vec_mode_name(const PipelineConfig &config) {
  if (config.vec == VecMode::None) return "none";
  return std::string(config.vec == VecMode::Inner ? "inner" : "outer") + (config.interleaved_opt ? "-opt" : "");
}

// Maps a C-ABI status onto the reference's exception classes.
inline void check(fftgen_status st) {
  if (st == FFTGEN_OK) return;
  const std::string msg = std::string(fftgen_error_string(st)) + ": " + fftgen_last_error();
  switch (st) {
  case FFTGEN_ERR_PLAN: throw PlanError(msg);
  case FFTGEN_ERR_FUSE: throw FuseError(msg);
  case FFTGEN_ERR_DIMENSION:
  case FFTGEN_ERR_INVALID: throw DimensionError(msg);
  case FFTGEN_ERR_LOWER: throw LowerError(msg);
  case FFTGEN_ERR_BOUNDS: throw BoundsError(msg);
  case FFTGEN_ERR_GPUMAP: throw GpuMapError(msg);
  default: throw ExecError(msg);
  }
}

// Flat float64 storage for n complex values under a layout (loopir.hpp:215-228):
// interleaved keeps value j at (2j, 2j+1); split keeps reals in [0, n) and
// imaginaries in [n, 2n).
struct ComplexBuffer {
  std::vector<double> data;
  ComplexLayout layout = ComplexLayout::Interleaved;
  int64_t logical_len = 0;

  static ComplexBuffer zeros(int64_t n, ComplexLayout layout) {
    ComplexBuffer b;
    b.data.assign(2 * n, 0.0);
    b.layout = layout;
    b.logical_len = n;
    return b;
  }
  static ComplexBuffer from_vector(const std::vector<cplx> &v, ComplexLayout layout) {
    ComplexBuffer b = zeros(static_cast<int64_t>(v.size()), layout);
    for (int64_t j = 0; j < b.logical_len; ++j) b.set(j, v[j]);
    return b;
  }
  cplx get(int64_t j) const {
    return layout == ComplexLayout::Interleaved ? cplx{data[2 * j], data[2 * j + 1]}
                                                : cplx{data[j], data[logical_len + j]};
  }
  void set(int64_t j, cplx v) {
    if (layout == ComplexLayout::Interleaved) {
      data[2 * j] = v.real();
      data[2 * j + 1] = v.imag();
    } else {
      data[j] = v.real();
      data[logical_len + j] = v.imag();
    }
  }
  std::vector<cplx> to_vector() const {
    std::vector<cplx> v(logical_len);
    for (int64_t j = 0; j < logical_len; ++j) v[j] = get(j);
    return v;
  }
  ComplexBuffer relayout(ComplexLayout target) const {
    if (target == layout) return *this;
    ComplexBuffer out = zeros(logical_len, target);
    for (int64_t j = 0; j < logical_len; ++j) out.set(j, get(j));
    return out;
  }
};

// ---- the compiled program ------------------------------------------------------
// One fused operator of the reference's list (rewrite.hpp:24-52, application
// order): kind 0 FusedMKIV(m, copies) 1 FusedIKMV(n, copies) 2 FusedPKIV(m,
// total, k) 3 TwiddleMul(len) 4 Permute(m, total).
struct FusedOp {
  int kind = 0;
  int64_t p0 = 0, p1 = 0, p2 = 0;
};
struct FuseResult {
  std::vector<FusedOp> ops;
};
// The factorisation the plan was built from (formula.hpp): plan_stockham /
// plan_cooley_tukey of (n, radix).
struct Formula {
  int64_t n = 0;
  Algorithm algorithm = Algorithm::CooleyTukey;
  int64_t radix = 2;
};
using FormulaPtr = std::shared_ptr<const Formula>;

// LoopProgram (loopir.hpp:151-208) on the B200 is the device program: the
// sm_100a pass / group schedule, the fp32 twiddle tables on the device and
// the plan's scratch, owned through a shared handle (cheap to copy).
class LoopProgram {
 public:
  LoopProgram() = default;
  LoopProgram(std::shared_ptr<fftgen_plan> plan, int64_t n, ComplexLayout layout, int64_t batch)
      : plan_(std::move(plan)), n_(n), layout_(layout), batch_(batch) {}
  fftgen_plan *handle() const { return plan_.get(); }
  int64_t size() const { return n_; }
  int64_t batch() const { return batch_; }
  ComplexLayout layout() const { return layout_; }
  explicit operator bool() const { return plan_ != nullptr; }

  // Device buffers; dist in complex elements (interleaved) or floats (split).
  void execute(Direction dir, const void *in0, const void *in1, void *out0, void *out1, int64_t dist,
               void *stream = nullptr) const {
    check(fftgen_execute(need(), static_cast<int>(dir), in0, in1, out0, out1, dist, stream));
  }
  // Host fp32 buffers, pipelined through the device.
  void execute_host(Direction dir, const float *in0, const float *in1, float *out0, float *out1,
                    int64_t dist) const {
    check(fftgen_execute_host(need(), static_cast<int>(dir), in0, in1, out0, out1, dist));
  }
  std::string describe() const { return text(fftgen_plan_describe); }
  std::string pipeline_text() const { return text(fftgen_plan_pipeline_text); }
  int launches() const { return fftgen_plan_launches(need()); }

 private:
  fftgen_plan *need() const {
    if (!plan_) throw ExecError("empty LoopProgram: compile a pipeline first");
    return plan_.get();
  }
  std::string text(fftgen_status (*fn)(const fftgen_plan *, char *, size_t)) const {
    std::vector<char> buf(1 << 16);
    while (fn(need(), buf.data(), buf.size()) != FFTGEN_OK) {
      if (buf.size() > (size_t(1) << 28)) check(FFTGEN_ERR_DIMENSION);
      buf.resize(buf.size() * 4);
    }
    return std::string(buf.data());
  }
  std::shared_ptr<fftgen_plan> plan_;
  int64_t n_ = 0;
  ComplexLayout layout_ = ComplexLayout::Interleaved;
  int64_t batch_ = 0;
};

// CompiledPipeline (driver.hpp:37-42): the same four members; complex_ir and
// final_ir are the same device program (the B200 lowering has no separate
// pre-layout form), plus convenience forwarding to final_ir.
struct CompiledPipeline {
  FormulaPtr formula;
  FuseResult fused;
  LoopProgram complex_ir;
  LoopProgram final_ir;
  PipelineConfig config_;

  const PipelineConfig &config() const { return config_; }
  fftgen_plan *handle() const { return final_ir.handle(); }
  void execute(Direction dir, const void *in0, const void *in1, void *out0, void *out1, int64_t dist,
               void *stream = nullptr) const {
    final_ir.execute(dir, in0, in1, out0, out1, dist, stream);
  }
  void execute_host(Direction dir, const float *in0, const float *in1, float *out0, float *out1,
                    int64_t dist) const {
    final_ir.execute_host(dir, in0, in1, out0, out1, dist);
  }
  std::vector<int64_t> radices() const {
    std::vector<int64_t> r(64);
    r.resize(fftgen_plan_radices(handle(), r.data(), 64));
    return r;
  }
  std::string pipeline_text() const { return final_ir.pipeline_text(); }
  std::string describe() const { return final_ir.describe(); }
  int launches() const { return final_ir.launches(); }
};

// compile_pipeline (driver.cpp:11-34): plan -> fuse -> [tile / vectorize
// validation] -> the sm_100a program; PlanError / FuseError / LowerError /
// DimensionError like the reference, GpuMapError when the device cannot run it.
inline CompiledPipeline compile_pipeline(const PipelineConfig &config) {
  fftgen_config c;
  fftgen_config_init(&c);
  c.n = config.n;
  c.algorithm = config.algorithm == Algorithm::Stockham ? FFTGEN_ALG_STOCKHAM : FFTGEN_ALG_COOLEY_TUKEY;
  if (config.radix < 0 || config.radix > (int64_t(1) << 30))
    throw PlanError("radix must be a power of two >= 2, got " + std::to_string(config.radix));
  c.radix = static_cast<int32_t>(config.radix);
  c.layout = config.layout == ComplexLayout::Split ? FFTGEN_LAYOUT_SPLIT : FFTGEN_LAYOUT_INTERLEAVED;
  c.vec = config.vec == VecMode::Inner ? FFTGEN_VEC_INNER : (config.vec == VecMode::Outer ? FFTGEN_VEC_OUTER
                                                                                          : FFTGEN_VEC_NONE);
  if (config.vector_width > (int64_t(1) << 30) || config.vector_width < -(int64_t(1) << 30))
    throw LowerError("vector width capped at 64 lanes");
  c.vector_width = static_cast<int32_t>(config.vector_width);
  c.interleaved_opt = config.interleaved_opt ? 1 : 0;
  if (config.tile) {
    c.tile_kind = config.tile->kind == TilePolicy::ExactSize ? FFTGEN_TILE_EXACT : FFTGEN_TILE_CACHE;
    c.tile_value = config.tile->value;
  }
  c.batch = config.batch;
  c.device = config.device;
  c.tuning = config.tuning;
  c.pass_radix = config.pass_radix;
  fftgen_plan *p = nullptr;
  check(fftgen_plan_create(&p, &c));
  std::shared_ptr<fftgen_plan> plan(p, [](fftgen_plan *q) { fftgen_plan_destroy(q); });
  CompiledPipeline out;
  out.config_ = config;
  out.formula = std::make_shared<const Formula>(Formula{config.n, config.algorithm, config.radix});
  const int nops = fftgen_plan_num_ops(p);
  for (int i = 0; i < nops; ++i) {
    int64_t d[4];
    check(fftgen_plan_op(p, i, d));
    out.fused.ops.push_back(FusedOp{static_cast<int>(d[0]), d[1], d[2], d[3]});
  }
  out.final_ir = LoopProgram(plan, config.n, config.layout, config.batch);
  out.complex_ir = out.final_ir;
  return out;
}

// ---- exec.hpp:16-27 ----------------------------------------------------------
struct ExecOptions {
  int threads = 1;  // the reference's host workers; the GPU program ignores it (results never depend on it)
  Direction direction = Direction::Forward;  // B200 extension: the reference has no inverse
};

namespace detail {
inline void check_input(const LoopProgram &prog, const ComplexBuffer &b) {
  if (b.logical_len != prog.size())
    throw ExecError("input length " + std::to_string(b.logical_len) + " does not match pipeline size " +
                    std::to_string(prog.size()));
  if (b.layout != prog.layout())
    throw ExecError("input layout does not match the layout the program was lowered for");
  if (static_cast<int64_t>(b.data.size()) != 2 * b.logical_len)
    throw ExecError("buffer storage holds " + std::to_string(b.data.size()) + " doubles, expected " +
                    std::to_string(2 * b.logical_len));
}
}  // namespace detail

// interpret over `batch` buffers at once (one per transform of the plan).
inline std::vector<ComplexBuffer> interpret(const LoopProgram &prog, const std::vector<ComplexBuffer> &inputs,
                                            const ExecOptions &opts = {}) {
  if (!prog) throw ExecError("empty LoopProgram: compile a pipeline first");
  if (static_cast<int64_t>(inputs.size()) != prog.batch())
    throw ExecError("got " + std::to_string(inputs.size()) + " buffers for a plan of batch " +
                    std::to_string(prog.batch()));
  const int64_t n = prog.size();
  std::vector<double> flat;
  flat.reserve(2 * n * prog.batch());
  for (const ComplexBuffer &b : inputs) {
    detail::check_input(prog, b);
    flat.insert(flat.end(), b.data.begin(), b.data.end());
  }
  std::vector<double> out(flat.size());
  check(fftgen_interpret_f64(prog.handle(), static_cast<int>(opts.direction), flat.data(), out.data()));
  std::vector<ComplexBuffer> res(inputs.size());
  for (size_t i = 0; i < inputs.size(); ++i) {
    res[i] = ComplexBuffer::zeros(n, prog.layout());
    std::copy(out.begin() + i * 2 * n, out.begin() + (i + 1) * 2 * n, res[i].data.begin());
  }
  return res;
}

// interpret (exec.hpp:26-27): out-of-place, the result by value.
inline ComplexBuffer interpret(const LoopProgram &prog, const ComplexBuffer &input, const ExecOptions &opts = {}) {
  return interpret(prog, std::vector<ComplexBuffer>{input}, opts).front();
}

// Direction-first forms over a CompiledPipeline (the round-1 API).
inline std::vector<ComplexBuffer> interpret(const CompiledPipeline &prog, const std::vector<ComplexBuffer> &inputs,
                                            Direction dir = Direction::Forward) {
  ExecOptions o;
  o.direction = dir;
  return interpret(prog.final_ir, inputs, o);
}
inline ComplexBuffer interpret(const CompiledPipeline &prog, const ComplexBuffer &input,
                               Direction dir = Direction::Forward) {
  ExecOptions o;
  o.direction = dir;
  return interpret(prog.final_ir, input, o);
}

// ---- the distributed four-step of one transform over `world` ranks ----------
// (fftgen_dist_*).  Device blocks of block_elems()
// interleaved fp32 complex values; the exchange is the caller's all-to-all of
// `world` contiguous chunks of chunk_bytes (NCCL grouped send/recv), any
// callable `int(const void *send, void *recv, size_t chunk_bytes, void *stream)`
// returning 0 on success.
class DistributedPlan {
 public:
  DistributedPlan(int64_t n, int world, int rank, int device = 0) {
    fftgen_dist_plan *p = nullptr;
    check(fftgen_dist_plan_create(&p, n, world, rank, device));
    plan_.reset(p, [](fftgen_dist_plan *q) { fftgen_dist_plan_destroy(q); });
  }
  int64_t block_elems() const { return fftgen_dist_block_elems(plan_.get()); }
  int64_t chunk_elems() const { return fftgen_dist_chunk_elems(plan_.get()); }
  fftgen_dist_plan *handle() const { return plan_.get(); }

  template <class Exchange>
  void execute(Direction dir, const void *in, void *out, void *work0, void *work1, Exchange &&exchange,
               void *stream = nullptr) const {
    struct Ctx {
      Exchange *f;
    } ctx{&exchange};
    auto tramp = [](void *c, const void *send, void *recv, size_t bytes, void *s) -> int {
      return (*static_cast<Ctx *>(c)->f)(send, recv, bytes, s);
    };
    check(fftgen_dist_execute(plan_.get(), static_cast<int>(dir), in, out, work0, work1, tramp, &ctx, stream));
  }
  // cyclic output order: out[j] = X[rank + world*j], two exchanges
  template <class Exchange>
  void execute_cyclic(Direction dir, const void *in, void *out, void *work0, Exchange &&exchange,
                      void *stream = nullptr) const {
    struct Ctx {
      Exchange *f;
    } ctx{&exchange};
    auto tramp = [](void *c, const void *send, void *recv, size_t bytes, void *s) -> int {
      return (*static_cast<Ctx *>(c)->f)(send, recv, bytes, s);
    };
    check(fftgen_dist_execute_cyclic(plan_.get(), static_cast<int>(dir), in, out, work0, nullptr, tramp, &ctx,
                                     stream));
  }
  // the stages one by one (the exchanges in between are the caller's)
  void butterfly(Direction dir, const void *recv, void *send, void *stream = nullptr) const {
    check(fftgen_dist_butterfly(plan_.get(), static_cast<int>(dir), recv, send, stream));
  }
  void local(Direction dir, const void *in, void *out, void *stream = nullptr) const {
    check(fftgen_dist_local(plan_.get(), static_cast<int>(dir), in, out, stream));
  }
  void unpack(const void *recv, void *out, void *stream = nullptr) const {
    check(fftgen_dist_unpack(plan_.get(), recv, out, stream));
  }
  // peer-memory transport: every rank's blocks mapped into this process
  void butterfly_peers(Direction dir, const std::vector<const void *> &in_blocks,
                       const std::vector<void *> &recv_blocks, void *stream = nullptr) const {
    check(fftgen_dist_butterfly_peers(plan_.get(), static_cast<int>(dir), in_blocks.data(), recv_blocks.data(),
                                      stream));
  }
  void unpack_peers(const std::vector<const void *> &z_blocks, void *out, void *stream = nullptr) const {
    check(fftgen_dist_unpack_peers(plan_.get(), z_blocks.data(), out, stream));
  }

 private:
  std::shared_ptr<fftgen_dist_plan> plan_;
};

}  // namespace fftgen

#endif  // FFTGEN_B200_HPP
