// tests/cpp/refshim/fftgen/exec.hpp -- "fftgen/exec.hpp" mapped onto the B200
// C++ API (test infrastructure).
//
// interpret / ExecOptions / ComplexBuffer are the product's
// (include/fftgen_b200.hpp).  The reference's CPU ahead-of-time path
// (emit_c, emit_c.cpp) and its intermediate passes (plan_cooley_tukey ->
// fuse -> bufferize -> lower_complex) have no B200 counterpart -- the
// device program replaces them, SURVEY 8(a) a12/a15/a16 -- so the emit test
// cases of test_exec.cpp are compiled but not run (tests/test_cpp_api.py
// selects the known-answer cases); these declarations only let the file
// compile unchanged and raise if reached.
#pragma once
#include <string>
#include <vector>

#include "fftgen_b200.hpp"

namespace fftgen {
inline std::string emit_c(const LoopProgram &, const std::string &) {
  throw LowerError("emit_c: the B200 program is a device plan, not scalar C (out of scope)");
}
inline FormulaPtr plan_cooley_tukey(int64_t n, int64_t radix) {
  return std::make_shared<const Formula>(Formula{n, Algorithm::CooleyTukey, radix});
}
inline FuseResult fuse(const Formula &) { throw LowerError("fuse: host-only reference pass (out of scope)"); }
inline LoopProgram bufferize(const std::vector<FusedOp> &, int64_t) {
  throw LowerError("bufferize: host-only reference pass (out of scope)");
}
inline LoopProgram lower_complex(const LoopProgram &, ComplexLayout) {
  throw LowerError("lower_complex: host-only reference pass (out of scope)");
}
}  // namespace fftgen
