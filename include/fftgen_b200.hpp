// include/fftgen_b200.hpp -- C++ host API over the C ABI (include/fftgen_b200.h).
//
// A drop-in for the reference's plan -> execute API in proj/include/fftgen:
// the same names, argument meaning and error behaviour, so a caller of the
// reference switches by including this header instead of
// fftgen/driver.hpp + fftgen/exec.hpp + fftgen/error.hpp and linking
// libfftgen_b200.so.
//
//   reference                                       here
//   Error / PlanError / DimensionError / FuseError  same classes (error.hpp:16-71)
//     / ExecError
//   Algorithm, ComplexLayout                        same enums (driver.hpp:21, loopir.hpp:187)
//   PipelineConfig {n, algorithm, radix, layout}    same fields + batch, device (driver.hpp:26-35)
//   CompiledPipeline compile_pipeline(config)       same (driver.hpp:44-45); owns the device plan
//   ComplexBuffer {data, layout, logical_len}       same storage contract (loopir.hpp:215-228)
//   ComplexBuffer interpret(program, input)         same (exec.hpp:26-27), on the GPU; an
//                                                   overload takes a batch of buffers
//   print_pipeline(ops)                             CompiledPipeline::pipeline_text()
//   algorithm_name / layout_name                    same (driver.hpp:47-49)
//
// plus device-pointer execution (CompiledPipeline::execute) with a direction
// and a CUDA stream.  Header-only; no CUDA headers are required.
#ifndef FFTGEN_B200_HPP
#define FFTGEN_B200_HPP

#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fftgen_b200.h"

namespace fftgen {

using cplx = std::complex<double>;

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string &msg) : std::runtime_error(msg) {}
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
class ExecError : public Error {
 public:
  using Error::Error;
};

enum class Algorithm { CooleyTukey, Stockham };
enum class ComplexLayout { Interleaved, Split };
enum class Direction { Forward = FFTGEN_FORWARD, Inverse = FFTGEN_INVERSE };

struct PipelineConfig {
  int64_t n = 0;
  Algorithm algorithm = Algorithm::CooleyTukey;
  int64_t radix = 2;
  ComplexLayout layout = ComplexLayout::Interleaved;
  int64_t batch = 1;  // transforms per execute
  int device = 0;     // CUDA device ordinal
};

inline std::string algorithm_name(Algorithm a) { return a == Algorithm::CooleyTukey ? "cooley-tukey" : "stockham"; }
inline std::string layout_name(ComplexLayout l) { return l == ComplexLayout::Interleaved ? "interleaved" : "split"; }

// Maps a C-ABI status onto the reference's exception classes.
inline void check(fftgen_status st) {
  if (st == FFTGEN_OK) return;
  const std::string msg = std::string(fftgen_error_string(st)) + ": " + fftgen_last_error();
  switch (st) {
  case FFTGEN_ERR_PLAN: throw PlanError(msg);
  case FFTGEN_ERR_FUSE: throw FuseError(msg);
  case FFTGEN_ERR_DIMENSION:
  case FFTGEN_ERR_INVALID: throw DimensionError(msg);
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

// The compiled plan (CompiledPipeline analogue): radix stages, fused op list,
// sm_100a passes and the device twiddle tables.  Cheap to copy (shared).
class CompiledPipeline {
 public:
  explicit CompiledPipeline(const PipelineConfig &cfg) : cfg_(cfg) {
    fftgen_config c;
    fftgen_config_init(&c);
    c.n = cfg.n;
    c.algorithm = cfg.algorithm == Algorithm::Stockham ? FFTGEN_ALG_STOCKHAM : FFTGEN_ALG_COOLEY_TUKEY;
    c.radix = static_cast<int32_t>(cfg.radix);
    c.layout = cfg.layout == ComplexLayout::Split ? FFTGEN_LAYOUT_SPLIT : FFTGEN_LAYOUT_INTERLEAVED;
    c.batch = cfg.batch;
    c.device = cfg.device;
    fftgen_plan *p = nullptr;
    check(fftgen_plan_create(&p, &c));
    plan_.reset(p, [](fftgen_plan *q) { fftgen_plan_destroy(q); });
  }

  const PipelineConfig &config() const { return cfg_; }
  fftgen_plan *handle() const { return plan_.get(); }

  // Device buffers; dist in complex elements (interleaved) or floats (split).
  void execute(Direction dir, const void *in0, const void *in1, void *out0, void *out1, int64_t dist,
               void *stream = nullptr) const {
    check(fftgen_execute(plan_.get(), static_cast<int>(dir), in0, in1, out0, out1, dist, stream));
  }
  // Host fp32 buffers, pipelined through the device.
  void execute_host(Direction dir, const float *in0, const float *in1, float *out0, float *out1,
                    int64_t dist) const {
    check(fftgen_execute_host(plan_.get(), static_cast<int>(dir), in0, in1, out0, out1, dist));
  }

  std::vector<int64_t> radices() const {
    std::vector<int64_t> r(64);
    r.resize(fftgen_plan_radices(plan_.get(), r.data(), 64));
    return r;
  }
  std::string pipeline_text() const { return text(fftgen_plan_pipeline_text); }
  std::string describe() const { return text(fftgen_plan_describe); }
  int launches() const { return fftgen_plan_launches(plan_.get()); }

 private:
  std::string text(fftgen_status (*fn)(const fftgen_plan *, char *, size_t)) const {
    std::vector<char> buf(1 << 16);
    while (fn(plan_.get(), buf.data(), buf.size()) != FFTGEN_OK) {
      if (buf.size() > (size_t(1) << 28)) check(FFTGEN_ERR_DIMENSION);
      buf.resize(buf.size() * 4);
    }
    return std::string(buf.data());
  }
  PipelineConfig cfg_;
  std::shared_ptr<fftgen_plan> plan_;
};

inline CompiledPipeline compile_pipeline(const PipelineConfig &config) { return CompiledPipeline(config); }

// interpret(): one ComplexBuffer per transform, layouts must match the plan
// (interpret.cpp:46-63 raises ExecError on a length or layout mismatch).
inline std::vector<ComplexBuffer> interpret(const CompiledPipeline &prog, const std::vector<ComplexBuffer> &inputs,
                                            Direction dir = Direction::Forward) {
  const PipelineConfig &cfg = prog.config();
  if (static_cast<int64_t>(inputs.size()) != cfg.batch)
    throw ExecError("got " + std::to_string(inputs.size()) + " buffers for a plan of batch " +
                    std::to_string(cfg.batch));
  std::vector<double> flat;
  flat.reserve(2 * cfg.n * cfg.batch);
  for (const ComplexBuffer &b : inputs) {
    if (b.logical_len != cfg.n)
      throw ExecError("input length " + std::to_string(b.logical_len) + " does not match pipeline size " +
                      std::to_string(cfg.n));
    if (b.layout != cfg.layout)
      throw ExecError("input layout does not match the layout the program was lowered for");
    flat.insert(flat.end(), b.data.begin(), b.data.end());
  }
  std::vector<double> out(flat.size());
  check(fftgen_interpret_f64(prog.handle(), static_cast<int>(dir), flat.data(), out.data()));
  std::vector<ComplexBuffer> res(inputs.size());
  for (size_t i = 0; i < inputs.size(); ++i) {
    res[i] = ComplexBuffer::zeros(cfg.n, cfg.layout);
    std::copy(out.begin() + i * 2 * cfg.n, out.begin() + (i + 1) * 2 * cfg.n, res[i].data.begin());
  }
  return res;
}

inline ComplexBuffer interpret(const CompiledPipeline &prog, const ComplexBuffer &input,
                               Direction dir = Direction::Forward) {
  return interpret(prog, std::vector<ComplexBuffer>{input}, dir).front();
}

}  // namespace fftgen

#endif  // FFTGEN_B200_HPP
