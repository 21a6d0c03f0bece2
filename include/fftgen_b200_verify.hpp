// include/fftgen_b200_verify.hpp -- the reference's verification API
// (proj/include/fftgen/verify.hpp, proj/src/verify.cpp:19-181) for host C++
// callers of include/fftgen_b200.hpp: the synthetic input generator every
// benchmark and parity check uses, the O(N^2) fp64 DFT oracle, the error
// metric, the FLOP-rate normalisation, bench() with its CSV row and the
// run_verification() configuration sweep -- the same names and semantics,
// executing through interpret() on the GPU.  Header-only, host only; the
// device-side generator is fftgen_seeded_input (include/fftgen_b200.h).
#ifndef FFTGEN_B200_VERIFY_HPP
#define FFTGEN_B200_VERIFY_HPP

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "fftgen_b200.hpp"

namespace fftgen {

namespace detail {
inline uint64_t splitmix64(uint64_t &state) {
  state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline double unit_double(uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }
}  // namespace detail

// re/im uniform in [-1, 1): draw 2j and 2j+1 of splitmix64 from state = seed
// (verify.cpp:55-78)
inline std::vector<cplx> seeded_input(int64_t n, uint64_t seed) {
  uint64_t state = seed;
  std::vector<cplx> x(n);
  for (int64_t j = 0; j < n; ++j) {
    const double re = 2.0 * detail::unit_double(detail::splitmix64(state)) - 1.0;
    const double im = 2.0 * detail::unit_double(detail::splitmix64(state)) - 1.0;
    x[j] = {re, im};
  }
  return x;
}

// exp(-2 pi i t / n), exact at quadrant multiples (matrix.cpp:14-35)
inline cplx unit_root(int64_t n, int64_t t) {
  t %= n;
  if (t < 0) t += n;
  if (4 * t % n == 0) {
    static const double qr[4] = {1.0, 0.0, -1.0, 0.0}, qi[4] = {0.0, -1.0, 0.0, 1.0};
    return {qr[4 * t / n], qi[4 * t / n]};
  }
  const double angle = -2.0 * M_PI * static_cast<double>(t) / static_cast<double>(n);
  return {std::cos(angle), std::sin(angle)};
}

// X[j] = sum_k x[k] w_N^{jk}: one root table, exponents reduced mod N, real
// and imaginary parts accumulated separately left to right (verify.cpp:19-37)
inline std::vector<cplx> dft_oracle(const std::vector<cplx> &x) {
  const int64_t n = static_cast<int64_t>(x.size());
  std::vector<cplx> roots(n);
  for (int64_t t = 0; t < n; ++t) roots[t] = unit_root(n, t);
  std::vector<cplx> y(n);
  for (int64_t j = 0; j < n; ++j) {
    double re = 0.0, im = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const cplx w = roots[(j * k) % n];
      re += w.real() * x[k].real() - w.imag() * x[k].imag();
      im += w.real() * x[k].imag() + w.imag() * x[k].real();
    }
    y[j] = {re, im};
  }
  return y;
}

// max_j |a[j] - b[j]| / N (verify.cpp:39-46)
inline double error_metric(const std::vector<cplx> &a, const std::vector<cplx> &b) {
  if (a.size() != b.size()) throw DimensionError("error_metric: vectors differ in length");
  double worst = 0.0;
  for (size_t i = 0; i < a.size(); ++i) worst = std::max(worst, std::abs(a[i] - b[i]));
  return worst / static_cast<double>(a.size());
}

// 5 N log2 N / seconds / 1e6 (verify.cpp:48-51)
inline double mflops(int64_t n, double seconds) {
  return 5.0 * static_cast<double>(n) * std::log2(static_cast<double>(n)) / seconds / 1e6;
}

// "n=<n> alg=<algorithm> radix=<r> layout=<layout> vec=<mode>" (verify.cpp:119-125)
inline std::string describe_config(const PipelineConfig &c) {
  return "n=" + std::to_string(c.n) + " alg=" + algorithm_name(c.algorithm) + " radix=" + std::to_string(c.radix) +
         " layout=" + layout_name(c.layout) + " vec=" + vec_mode_name(c);
}

struct BenchResult {
  PipelineConfig config;
  int64_t repeats = 0;
  double mean_seconds = 0.0;
  double rate_mflops = 0.0;
  uint64_t seed = 0;
};

// Compiles the configuration and times `repeats` interpret() calls over one
// fixed seeded input: the reference's end-to-end rate (verify.cpp:80-100),
// host buffers in and out of the GPU program on every call.
inline BenchResult bench(const PipelineConfig &config, int64_t repeats = 1000, uint64_t seed = 1) {
  const CompiledPipeline compiled = compile_pipeline(config);
  const ComplexBuffer input = ComplexBuffer::from_vector(seeded_input(config.n, seed), config.layout);
  using clock = std::chrono::steady_clock;
  const auto begin = clock::now();
  for (int64_t r = 0; r < repeats; ++r) interpret(compiled.final_ir, input);
  const auto end = clock::now();
  BenchResult res;
  res.config = config;
  res.repeats = repeats;
  res.mean_seconds = std::chrono::duration<double>(end - begin).count() / static_cast<double>(repeats);
  res.rate_mflops = mflops(config.n, res.mean_seconds);
  res.seed = seed;
  return res;
}

inline std::string bench_csv_header() {
  return "n,algorithm,radix,layout,vector_mode,repeats,mean_seconds,mflops,seed";
}

// verify.cpp:106-117: %.9e seconds, %.6f MFLOP/s, seed last
inline std::string bench_csv_row(const BenchResult &r) {
  char secs[64], rate[64];
  std::snprintf(secs, sizeof secs, "%.9e", r.mean_seconds);
  std::snprintf(rate, sizeof rate, "%.6f", r.rate_mflops);
  return std::to_string(r.config.n) + "," + algorithm_name(r.config.algorithm) + "," +
         std::to_string(r.config.radix) + "," + layout_name(r.config.layout) + "," + vec_mode_name(r.config) + "," +
         std::to_string(r.repeats) + "," + secs + "," + rate + "," + std::to_string(r.seed);
}

struct VerifyCase {
  PipelineConfig config;
  double max_error = 0.0;
  bool pass = false;
};

// The configuration matrix of verify.cpp:127-181 -- both algorithms, radices
// {2, 4, 16} that divide n, both layouts, vector modes none / inner / outer
// (+ the -opt variants for interleaved) -- each against the oracle on
// `inputs` seeded vectors; pass = error_metric < 1e-7.
inline std::vector<VerifyCase> run_verification(const std::vector<int64_t> &sizes, int inputs = 5) {
  std::vector<VerifyCase> cases;
  std::map<std::pair<int64_t, uint64_t>, std::vector<cplx>> want;
  for (int64_t n : sizes) {
    for (int t = 0; t < inputs; ++t) {
      const uint64_t seed = 1 + static_cast<uint64_t>(t);
      if (!want.count({n, seed})) want[{n, seed}] = dft_oracle(seeded_input(n, seed));
    }
    for (Algorithm alg : {Algorithm::CooleyTukey, Algorithm::Stockham})
      for (int64_t radix : {2, 4, 16}) {
        if (radix > n || n % radix != 0) continue;
        for (ComplexLayout layout : {ComplexLayout::Interleaved, ComplexLayout::Split}) {
          std::vector<std::pair<VecMode, bool>> modes = {
              {VecMode::None, false}, {VecMode::Inner, false}, {VecMode::Outer, false}};
          if (layout == ComplexLayout::Interleaved) {
            modes.push_back({VecMode::Inner, true});
            modes.push_back({VecMode::Outer, true});
          }
          for (const auto &[vec, opt] : modes) {
            PipelineConfig config;
            config.n = n;
            config.algorithm = alg;
            config.radix = radix;
            config.layout = layout;
            config.vec = vec;
            config.interleaved_opt = opt;
            const CompiledPipeline compiled = compile_pipeline(config);
            VerifyCase vc;
            vc.config = config;
            for (int t = 0; t < inputs; ++t) {
              const uint64_t seed = 1 + static_cast<uint64_t>(t);
              const ComplexBuffer out =
                  interpret(compiled.final_ir, ComplexBuffer::from_vector(seeded_input(n, seed), layout));
              vc.max_error = std::max(vc.max_error, error_metric(out.to_vector(), want[{n, seed}]));
            }
            vc.pass = vc.max_error < 1e-7;
            cases.push_back(std::move(vc));
          }
        }
      }
  }
  return cases;
}

}  // namespace fftgen

#endif  // FFTGEN_B200_VERIFY_HPP
