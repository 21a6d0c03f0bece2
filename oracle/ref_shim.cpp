// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never on the product path).
//
// A thin extern "C" harness over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libfftgen_ref.so).  Nothing here re-implements the reference:
// every entry point forwards to the reference's own public API so the test
// suite, the golden-fixture generator and bench.py's CPU baseline can call it
// through ctypes.
//
//   compile_pipeline     proj/src/driver.cpp:11-34
//   interpret            proj/src/interpret.cpp:275-281
//   seeded_input         proj/src/verify.cpp:69-78
//   dft_oracle           proj/src/verify.cpp:19-37
//   unit_root            proj/src/matrix.cpp:14-35
//   fuse / apply_op      proj/src/rewrite.cpp:175-241
//   print_pipeline       proj/src/rewrite.cpp:275-296
//   emit_c               proj/src/emit_c.cpp:155
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
// arm may load this library.

#include <atomic>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "fftgen/driver.hpp"
#include "fftgen/exec.hpp"
#include "fftgen/formula.hpp"
#include "fftgen/rewrite.hpp"
#include "fftgen/verify.hpp"

using namespace fftgen;

namespace {

thread_local std::string g_err;

using Key = std::tuple<int64_t, int, int64_t, int>;

std::mutex g_mu;
std::map<Key, std::shared_ptr<const CompiledPipeline>> g_cache;

std::shared_ptr<const CompiledPipeline> compiled(int64_t n, int alg,
                                                 int64_t radix, int layout) {
  const Key key{n, alg, radix, layout};
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end())
      return it->second;
  }
  PipelineConfig cfg;
  cfg.n = n;
  cfg.algorithm = alg == 1 ? Algorithm::Stockham : Algorithm::CooleyTukey;
  cfg.radix = radix;
  cfg.layout = layout == 1 ? ComplexLayout::Split : ComplexLayout::Interleaved;
  auto p = std::make_shared<const CompiledPipeline>(compile_pipeline(cfg));
  std::lock_guard<std::mutex> lk(g_mu);
  g_cache[key] = p;
  return p;
}

FuseResult fused(int64_t n, int alg, int64_t radix) {
  FormulaPtr f = alg == 1 ? plan_stockham(n, radix) : plan_cooley_tukey(n, radix);
  return fuse(*f);
}

template <class F> int guarded(F &&f) {
  try {
    return f();
  } catch (const PlanError &e) {
    g_err = e.what();
    return 1;
  } catch (const DimensionError &e) {
    g_err = e.what();
    return 2;
  } catch (const ExecError &e) {
    g_err = e.what();
    return 3;
  } catch (const Error &e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception &e) {
    g_err = e.what();
    return 5;
  }
}

int copy_text(const std::string &s, char *buf, int64_t cap) {
  if (buf && cap > 0) {
    const int64_t k = std::min<int64_t>(cap - 1, (int64_t)s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return 0;
}

} // namespace

extern "C" {

const char *ref_last_error(void) { return g_err.c_str(); }

// seeded_input(n, seed) as 2n interleaved doubles.
int ref_seeded_input(int64_t n, uint64_t seed, double *out) {
  return guarded([&] {
    const auto x = seeded_input(n, seed);
    for (int64_t j = 0; j < n; ++j) {
      out[2 * j] = x[j].real();
      out[2 * j + 1] = x[j].imag();
    }
    return 0;
  });
}

int ref_unit_root(int64_t n, int64_t t, double *out2) {
  const cplx w = unit_root(n, t);
  out2[0] = w.real();
  out2[1] = w.imag();
  return 0;
}

// Brute-force O(N^2) oracle; interleaved in/out.
int ref_dft_oracle(int64_t n, const double *in, double *out) {
  return guarded([&] {
    std::vector<cplx> x(n);
    for (int64_t j = 0; j < n; ++j)
      x[j] = {in[2 * j], in[2 * j + 1]};
    const auto y = dft_oracle(x);
    for (int64_t j = 0; j < n; ++j) {
      out[2 * j] = y[j].real();
      out[2 * j + 1] = y[j].imag();
    }
    return 0;
  });
}

// compile_pipeline + interpret over `batch` transforms of 2n doubles each in
// the program's layout (the reference ComplexBuffer storage), split across
// `threads` workers, one whole transform per call (interpret() builds a
// private Machine per call, so concurrent calls are safe -- SURVEY 8b).
int ref_forward_batch(int64_t n, int alg, int64_t radix, int layout,
                      int64_t batch, const double *in, double *out,
                      int threads) {
  return guarded([&] {
    auto prog = compiled(n, alg, radix, layout);
    const ComplexLayout lay =
        layout == 1 ? ComplexLayout::Split : ComplexLayout::Interleaved;
    std::atomic<int64_t> next{0};
    std::atomic<int> failed{0};
    std::string first_err;
    std::mutex err_mu;
    auto worker = [&] {
      ComplexBuffer buf = ComplexBuffer::zeros(n, lay);
      for (;;) {
        const int64_t b = next.fetch_add(1);
        if (b >= batch || failed.load())
          return;
        try {
          std::memcpy(buf.data.data(), in + b * 2 * n, sizeof(double) * 2 * n);
          const ComplexBuffer y = interpret(prog->final_ir, buf);
          std::memcpy(out + b * 2 * n, y.data.data(), sizeof(double) * 2 * n);
        } catch (const std::exception &e) {
          std::lock_guard<std::mutex> lk(err_mu);
          first_err = e.what();
          failed = 1;
        }
      }
    };
    if (threads <= 1) {
      worker();
    } else {
      std::vector<std::thread> pool;
      for (int t = 0; t < threads; ++t)
        pool.emplace_back(worker);
      for (auto &th : pool)
        th.join();
    }
    if (failed)
      throw ExecError(first_err);
    return 0;
  });
}

int ref_forward(int64_t n, int alg, int64_t radix, int layout, const double *in,
                double *out) {
  return ref_forward_batch(n, alg, radix, layout, 1, in, out, 1);
}

// Compile only (plan creation cost), for timing / error-behaviour tests.
int ref_compile(int64_t n, int alg, int64_t radix, int layout) {
  return guarded([&] {
    compiled(n, alg, radix, layout);
    return 0;
  });
}

int ref_formula_text(int64_t n, int alg, int64_t radix, char *buf, int64_t cap) {
  return guarded([&] {
    FormulaPtr f = alg == 1 ? plan_stockham(n, radix) : plan_cooley_tukey(n, radix);
    return copy_text(print_formula(*f), buf, cap);
  });
}

int ref_pipeline_text(int64_t n, int alg, int64_t radix, char *buf, int64_t cap) {
  return guarded([&] {
    const auto r = fused(n, alg, radix);
    return copy_text(print_pipeline(r.ops), buf, cap);
  });
}

int ref_num_ops(int64_t n, int alg, int64_t radix) {
  int64_t count = -1;
  const int rc = guarded([&] {
    count = (int64_t)fused(n, alg, radix).ops.size();
    return 0;
  });
  return rc ? -1 : (int)count;
}

// desc = {kind, p0, p1, p2}; kind 0 MKIV(m, copies) 1 IKMV(n, copies)
// 2 PKIV(m, total, k) 3 TwiddleMul(len) 4 Permute(m, total) 5 Dense(dim).
int ref_op_desc(int64_t n, int alg, int64_t radix, int idx, int64_t *desc) {
  return guarded([&] {
    const auto r = fused(n, alg, radix);
    const FusedOp &op = r.ops.at(idx);
    desc[1] = desc[2] = desc[3] = 0;
    if (auto *x = std::get_if<FusedMkiv>(&op)) {
      desc[0] = 0; desc[1] = x->kernel.rows; desc[2] = x->copies;
    } else if (auto *x = std::get_if<FusedIkmv>(&op)) {
      desc[0] = 1; desc[1] = x->kernel.rows; desc[2] = x->copies;
    } else if (auto *x = std::get_if<FusedPkiv>(&op)) {
      desc[0] = 2; desc[1] = x->perm_m; desc[2] = x->perm_total; desc[3] = x->block_k;
    } else if (auto *x = std::get_if<TwiddleMul>(&op)) {
      desc[0] = 3; desc[1] = (int64_t)x->coeffs.size();
    } else if (auto *x = std::get_if<Permute>(&op)) {
      desc[0] = 4; desc[1] = x->perm_m; desc[2] = x->perm_total;
    } else {
      desc[0] = 5; desc[1] = std::get<DenseApply>(op).matrix.rows;
    }
    return 0;
  });
}

// Index map of a data-movement op, extracted the way SURVEY Appendix A says:
// apply_op on x[i] = (i, 0); y[o].real() is the source index of output o.
int ref_op_index_map(int64_t n, int alg, int64_t radix, int idx, int64_t *map) {
  return guarded([&] {
    const auto r = fused(n, alg, radix);
    std::vector<cplx> x(n);
    for (int64_t i = 0; i < n; ++i)
      x[i] = {(double)i, 0.0};
    const auto y = apply_op(r.ops.at(idx), x);
    for (int64_t o = 0; o < n; ++o)
      map[o] = (int64_t)y[o].real();
    return 0;
  });
}

// Twiddle op coefficients (raw doubles, interleaved) and their exponents of
// w_s recovered by exact equality against unit_root(s, e), e in [0, s).
// exps[i] = -1 if no exact match exists.
int ref_op_twiddle(int64_t n, int alg, int64_t radix, int idx, int64_t s,
                   int64_t *exps, double *coeffs) {
  return guarded([&] {
    const auto r = fused(n, alg, radix);
    const auto *tw = std::get_if<TwiddleMul>(&r.ops.at(idx));
    if (!tw)
      throw DimensionError("op is not a TwiddleMul");
    std::map<std::pair<double, double>, int64_t> table;
    for (int64_t e = s - 1; e >= 0; --e) {
      const cplx w = unit_root(s, e);
      table[{w.real(), w.imag()}] = e;
    }
    for (size_t i = 0; i < tw->coeffs.size(); ++i) {
      const cplx c = tw->coeffs[i];
      if (coeffs) {
        coeffs[2 * i] = c.real();
        coeffs[2 * i + 1] = c.imag();
      }
      auto it = table.find({c.real(), c.imag()});
      exps[i] = it == table.end() ? -1 : it->second;
    }
    return 0;
  });
}

// emit_c text of the lowered program (reference AoT path). Returns the text
// length through *len; copies up to cap-1 bytes into buf when buf != NULL.
int ref_emit_c(int64_t n, int alg, int64_t radix, int layout, const char *fn,
               char *buf, int64_t cap, int64_t *len) {
  return guarded([&] {
    auto prog = compiled(n, alg, radix, layout);
    const std::string text = emit_c(prog->final_ir, fn);
    *len = (int64_t)text.size();
    return copy_text(text, buf, cap);
  });
}

// mflops(n, seconds) and error_metric, for bench/verify parity.
double ref_mflops(int64_t n, double seconds) { return mflops(n, seconds); }

double ref_error_metric(int64_t n, const double *a, const double *b) {
  std::vector<cplx> va(n), vb(n);
  for (int64_t j = 0; j < n; ++j) {
    va[j] = {a[2 * j], a[2 * j + 1]};
    vb[j] = {b[2 * j], b[2 * j + 1]};
  }
  return error_metric(va, vb);
}

} // extern "C"
