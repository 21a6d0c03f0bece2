// tests/cpp/api_test.cpp -- the reference's own exec/verify known-answer
// tests (proj/tests/test_exec.cpp, test_verify.cpp), restated against the
// B200 C++ API (include/fftgen_b200.hpp) with a plain assert harness (no
// doctest in this image).  Checked against the pinned C oracle
// (oracle/fftgen_oracle.c).
//
//   api_test cpu   -- no GPU: header semantics + plan validation errors
//   api_test gpu   -- full: known answers, oracle parity, error behaviour
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../oracle/fftgen_oracle.h"
#include "fftgen_b200.hpp"

using namespace fftgen;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    ++g_checks;                                                             \
    if (!(cond)) {                                                          \
      ++g_fail;                                                             \
      std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                       \
  } while (0)

template <class E, class F> static bool throws(F &&f) {
  try {
    f();
  } catch (const E &) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static std::vector<cplx> seeded(int64_t n, uint64_t seed) {
  std::vector<double> d(2 * n);
  orc_seeded_input(n, seed, d.data());
  std::vector<cplx> v(n);
  for (int64_t j = 0; j < n; ++j) v[j] = {(double)(float)d[2 * j], (double)(float)d[2 * j + 1]};
  return v;
}

static double rel_l2(const std::vector<cplx> &a, const std::vector<cplx> &b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += std::norm(a[i] - b[i]);
    den += std::norm(b[i]);
  }
  return std::sqrt(num / den);
}

static std::vector<cplx> run_config(const PipelineConfig &cfg, const std::vector<cplx> &x,
                                    Direction dir = Direction::Forward) {
  auto prog = compile_pipeline(cfg);
  return interpret(prog, ComplexBuffer::from_vector(x, cfg.layout), dir).to_vector();
}

static void cpu_tests() {
  // ComplexBuffer storage contract (loopir.hpp:215-228, test_loopir.cpp:158-188)
  auto b = ComplexBuffer::from_vector({{1, 2}, {3, 4}}, ComplexLayout::Split);
  CHECK(b.data == std::vector<double>({1, 3, 2, 4}));
  CHECK(b.relayout(ComplexLayout::Interleaved).data == std::vector<double>({1, 2, 3, 4}));
  CHECK(b.relayout(ComplexLayout::Interleaved).relayout(ComplexLayout::Split).data == b.data);
  // PipelineConfig defaults (driver.hpp:26-35)
  PipelineConfig c;
  CHECK(c.algorithm == Algorithm::CooleyTukey && c.radix == 2 && c.layout == ComplexLayout::Interleaved);
  CHECK(algorithm_name(Algorithm::Stockham) == "stockham" && layout_name(ComplexLayout::Split) == "split");
  // planner validation happens before any device is touched (formula.cpp:150-160)
  c.n = 12;
  CHECK(throws<PlanError>([&] { compile_pipeline(c); }));
  c.n = 16;
  c.radix = 3;
  CHECK(throws<PlanError>([&] { compile_pipeline(c); }));
  c.radix = 128;
  c.n = 256;
  CHECK(throws<FuseError>([&] { compile_pipeline(c); }));
  c.radix = 2;
  c.batch = 0;
  CHECK(throws<DimensionError>([&] { compile_pipeline(c); }));
}

static void gpu_tests() {
  // transform of a delta is the all-ones vector (test_exec.cpp:81-91)
  {
    PipelineConfig c;
    c.n = 4;
    auto out = run_config(c, {{1, 0}, {0, 0}, {0, 0}, {0, 0}});
    for (auto &v : out) CHECK(v == cplx(1.0, 0.0));
  }
  // size-2 transform of (1, 2) (test_exec.cpp:93-99)
  {
    PipelineConfig c;
    c.n = 2;
    auto out = run_config(c, {{1, 0}, {2, 0}});
    CHECK(out[0] == cplx(3, 0) && out[1] == cplx(-1, 0));
  }
  // size-8 pipeline matches the brute-force oracle (test_exec.cpp:101-111)
  for (Algorithm alg : {Algorithm::CooleyTukey, Algorithm::Stockham}) {
    PipelineConfig c;
    c.n = 8;
    c.algorithm = alg;
    auto x = seeded(8, 77);
    std::vector<double> xi(16), X(16);
    for (int j = 0; j < 8; ++j) {
      xi[2 * j] = x[j].real();
      xi[2 * j + 1] = x[j].imag();
    }
    orc_dft_oracle(8, xi.data(), X.data());
    auto got = run_config(c, x);
    std::vector<double> g(16);
    for (int j = 0; j < 8; ++j) {
      g[2 * j] = got[j].real();
      g[2 * j + 1] = got[j].imag();
    }
    CHECK(orc_error_metric(8, g.data(), X.data()) < 1e-7);
  }
  // interpretation is pure (test_exec.cpp:113-126): bitwise repeatable
  {
    PipelineConfig c;
    c.n = 4096;
    c.layout = ComplexLayout::Split;
    auto x = seeded(4096, 13);
    auto a = run_config(c, x), b = run_config(c, x);
    CHECK(a == b);
  }
  // oracle parity, both layouts, forward and inverse, several sizes
  for (int64_t n : {16, 1024, 4096, 16384, 65536, 1 << 20}) {
    for (ComplexLayout lay : {ComplexLayout::Interleaved, ComplexLayout::Split}) {
      for (Direction d : {Direction::Forward, Direction::Inverse}) {
        PipelineConfig c;
        c.n = n;
        c.layout = lay;
        c.algorithm = Algorithm::Stockham;
        auto x = seeded(n, 3);
        std::vector<double> xi(2 * n), want(2 * n);
        for (int64_t j = 0; j < n; ++j) {
          xi[2 * j] = x[j].real();
          xi[2 * j + 1] = x[j].imag();
        }
        if (d == Direction::Forward)
          orc_forward_batch(n, 1, 4, 1, xi.data(), want.data(), 4);
        else
          orc_inverse_batch(n, 1, 4, 1, xi.data(), want.data(), 4);
        std::vector<cplx> w(n);
        for (int64_t j = 0; j < n; ++j) w[j] = {want[2 * j], want[2 * j + 1]};
        const double err = rel_l2(run_config(c, x, d), w);
        CHECK(err < 1e-5 * std::log2((double)n));
        if (!(err < 3e-6)) std::fprintf(stderr, "n=%lld err=%g\n", (long long)n, err);
      }
    }
  }
  // batched interpret and layout mismatch -> ExecError (interpret.cpp:59-61)
  {
    PipelineConfig c;
    c.n = 64;
    c.batch = 3;
    auto prog = compile_pipeline(c);
    std::vector<ComplexBuffer> in;
    for (int b = 0; b < 3; ++b) in.push_back(ComplexBuffer::from_vector(seeded(64, 1 + b), c.layout));
    auto out = interpret(prog, in);
    CHECK(out.size() == 3 && out[2].logical_len == 64);
    in[1] = in[1].relayout(ComplexLayout::Split);
    CHECK(throws<ExecError>([&] { interpret(prog, in); }));
    CHECK(throws<ExecError>([&] { interpret(prog, ComplexBuffer::zeros(64, c.layout)); }));  // batch mismatch
    CHECK(prog.radices() == std::vector<int64_t>({2, 2, 2, 2, 2, 2}));
    CHECK(prog.pipeline_text().rfind("Permute(m=2, total=64)", 0) == 0);
    CHECK(throws<ExecError>([&] { prog.execute(Direction::Forward, nullptr, nullptr, nullptr, nullptr, 64); }));
  }
}

// fftgen::DistributedPlan: the distributed four-step through the C++ API
// with an exchange callable (world 1: the all-to-all is a device copy), and
// its argument validation.
extern "C" int cudaMalloc(void **, size_t);
extern "C" int cudaFree(void *);
extern "C" int cudaMemcpy(void *, const void *, size_t, int);
extern "C" int cudaMemcpyAsync(void *, const void *, size_t, int, void *);
extern "C" int cudaDeviceSynchronize();
extern "C" int cudaMemset(void *, int, size_t);

static void dist_tests() {
  CHECK(throws<DimensionError>([] { DistributedPlan(1 << 12, 3, 0); }));
  CHECK(throws<PlanError>([] { DistributedPlan(3000, 2, 0); }));
  const int64_t n = 1 << 16;
  DistributedPlan dp(n, 1, 0);
  CHECK(dp.block_elems() == n && dp.chunk_elems() == n);
  std::vector<double> d(2 * n);
  orc_seeded_input(n, 11, d.data());
  std::vector<float> h(2 * n);
  for (int64_t i = 0; i < 2 * n; ++i) h[i] = (float)d[i];
  void *x = nullptr, *y = nullptr, *w0 = nullptr, *w1 = nullptr;
  cudaMalloc(&x, 8 * n);
  cudaMalloc(&y, 8 * n);
  cudaMalloc(&w0, 8 * n);
  cudaMalloc(&w1, 8 * n);
  cudaMemcpy(x, h.data(), 8 * n, 1);
  int calls = 0;
  dp.execute(Direction::Forward, x, y, w0, w1, [&](const void *s, void *r, size_t bytes, void *st) {
    ++calls;
    return cudaMemcpyAsync(r, s, bytes, 3, st);
  });
  cudaDeviceSynchronize();
  std::vector<float> out(2 * n);
  cudaMemcpy(out.data(), y, 8 * n, 2);
  std::vector<double> in64(2 * n), want(2 * n);
  for (int64_t i = 0; i < 2 * n; ++i) in64[i] = h[i];
  orc_forward_batch(n, 1, 4, 1, in64.data(), want.data(), 4);
  std::vector<cplx> got(n), w(n);
  for (int64_t j = 0; j < n; ++j) got[j] = {out[2 * j], out[2 * j + 1]}, w[j] = {want[2 * j], want[2 * j + 1]};
  CHECK(calls == 3);
  CHECK(rel_l2(got, w) < 3e-6);
  // cyclic output order (world 1: the natural order) with two exchanges
  calls = 0;
  cudaMemset(y, 0, 8 * n);
  dp.execute_cyclic(Direction::Forward, x, y, w0, [&](const void *s, void *r, size_t bytes, void *st) {
    ++calls;
    return cudaMemcpyAsync(r, s, bytes, 3, st);
  });
  cudaDeviceSynchronize();
  std::vector<float> outc(2 * n);
  cudaMemcpy(outc.data(), y, 8 * n, 2);
  CHECK(calls == 2 && outc == out);
  // a failing exchange surfaces as ExecError
  CHECK(throws<ExecError>([&] { dp.execute(Direction::Forward, x, y, w0, w1, [](const void *, void *, size_t, void *) { return 7; }); }));
  CHECK(throws<ExecError>([&] { dp.butterfly(Direction::Forward, x, x); }));  // out of place only
  cudaFree(x);
  cudaFree(y);
  cudaFree(w0);
  cudaFree(w1);
}

int main(int argc, char **argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  cpu_tests();
  if (mode == "gpu") {
    gpu_tests();
    dist_tests();
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
