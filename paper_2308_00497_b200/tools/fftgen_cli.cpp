// fftgen_cli.cpp -- command-line front end of the B200 path, mirroring the
// reference CLI (proj/tools/main.cpp:127-259):
//
//   fftgen-b200 compile --size N [--algorithm A] [--radix R] [--layout L] --emit ir|kernels|radices
//   fftgen-b200 run     --size N [...] (--random SEED | --input FILE) [--inverse]
//   fftgen-b200 verify  [--sizes 16..4096|a,b,c] [--inputs 5]
//   fftgen-b200 bench   --sizes ... --csv PATH [--batch B] [--repeats R] [--layout L] [--inverse]
//
// Exit codes: 0 success, 1 failed verification or runtime error, 2 usage
// error (main.cpp:250-258).  `verify` runs the reference's configuration
// matrix (verify.cpp:127-181: both algorithms, radices {2,4,16}, both
// layouts; vectorisation modes do not exist on this path) on the GPU against
// an fp64 brute-force DFT (the dft_oracle formula, verify.cpp:19-37) with the
// reference's gate max|a-b|/N < 1e-7 (verify.cpp:173).  `bench` writes the
// reference CSV schema (verify.cpp:102-117) plus GPU columns.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "fftgen_b200.hpp"

using namespace fftgen;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

// seeded_input (verify.cpp:55-78): splitmix64, re/im uniform in [-1, 1)
std::vector<cplx> seeded_input(int64_t n, uint64_t seed) {
  uint64_t state = seed;
  auto next = [&]() {
    state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  std::vector<cplx> x(n);
  for (int64_t j = 0; j < n; ++j) {
    const double re = 2.0 * static_cast<double>(next() >> 11) * 0x1.0p-53 - 1.0;
    const double im = 2.0 * static_cast<double>(next() >> 11) * 0x1.0p-53 - 1.0;
    x[j] = {re, im};
  }
  return x;
}

// unit_root (matrix.cpp:14-35) and the O(N^2) double-sum DFT (verify.cpp:19-37)
cplx unit_root(int64_t n, int64_t t) {
  t %= n;
  if (t < 0) t += n;
  if (4 * t % n == 0) {
    static const cplx q[4] = {{1, 0}, {0, -1}, {-1, 0}, {0, 1}};
    return q[4 * t / n];
  }
  const double a = -2.0 * M_PI * static_cast<double>(t) / static_cast<double>(n);
  return {std::cos(a), std::sin(a)};
}

std::vector<cplx> dft(const std::vector<cplx> &x) {
  const int64_t n = static_cast<int64_t>(x.size());
  std::vector<cplx> roots(n), out(n);
  for (int64_t t = 0; t < n; ++t) roots[t] = unit_root(n, t);
  for (int64_t j = 0; j < n; ++j) {
    double re = 0, im = 0;
    for (int64_t k = 0; k < n; ++k) {
      const cplx w = roots[(j * k) % n];
      re += w.real() * x[k].real() - w.imag() * x[k].imag();
      im += w.real() * x[k].imag() + w.imag() * x[k].real();
    }
    out[j] = {re, im};
  }
  return out;
}

double error_metric(const std::vector<cplx> &a, const std::vector<cplx> &b) {
  double worst = 0;
  for (size_t j = 0; j < a.size(); ++j) worst = std::max(worst, std::abs(a[j] - b[j]));
  return worst / static_cast<double>(a.size());
}

struct Args {
  std::vector<std::string> v;
  size_t i = 0;
  bool has(const char *flag) const {
    for (const auto &s : v)
      if (s == flag) return true;
    return false;
  }
  std::string get(const char *flag, const std::string &def = "", bool required = false) const {
    for (size_t k = 0; k + 1 < v.size(); ++k)
      if (v[k] == flag) return v[k + 1];
    if (required) throw UsageError(std::string("missing ") + flag);
    return def;
  }
};

std::vector<int64_t> parse_sizes(const std::string &text) {
  std::vector<int64_t> sizes;
  const auto dots = text.find("..");
  if (dots != std::string::npos) {
    const int64_t lo = std::stoll(text.substr(0, dots)), hi = std::stoll(text.substr(dots + 2));
    if (!is_pow2(lo) || !is_pow2(hi) || lo > hi) throw UsageError("--sizes range must be powers of two A..B");
    for (int64_t n = lo; n <= hi; n *= 2) sizes.push_back(n);
    return sizes;
  }
  std::stringstream ss(text);
  std::string item;
  while (std::getline(ss, item, ',')) sizes.push_back(std::stoll(item));
  for (int64_t n : sizes)
    if (!is_pow2(n)) throw UsageError("sizes must be powers of two");
  if (sizes.empty()) throw UsageError("no sizes given");
  return sizes;
}

PipelineConfig config_from(const Args &a) {
  PipelineConfig c;
  c.n = std::stoll(a.get("--size", "0", true));
  const std::string alg = a.get("--algorithm", "cooley-tukey");
  if (alg != "cooley-tukey" && alg != "stockham") throw UsageError("--algorithm cooley-tukey|stockham");
  c.algorithm = alg == "stockham" ? Algorithm::Stockham : Algorithm::CooleyTukey;
  c.radix = std::stoll(a.get("--radix", "2"));
  const std::string lay = a.get("--layout", "interleaved");
  if (lay != "interleaved" && lay != "split") throw UsageError("--layout interleaved|split");
  c.layout = lay == "split" ? ComplexLayout::Split : ComplexLayout::Interleaved;
  c.batch = std::stoll(a.get("--batch", "1"));
  return c;
}

std::string describe(const PipelineConfig &c) {  // describe_config (verify.cpp:119-125)
  std::ostringstream o;
  o << "n=" << c.n << " alg=" << algorithm_name(c.algorithm) << " radix=" << c.radix
    << " layout=" << layout_name(c.layout) << " vec=none";
  return o.str();
}

int cmd_compile(const Args &a) {
  const PipelineConfig c = config_from(a);
  const std::string emit = a.get("--emit", "", true);
  auto prog = compile_pipeline(c);
  if (emit == "ir") {
    std::cout << prog.pipeline_text();
  } else if (emit == "kernels") {
    std::cout << prog.describe();
  } else if (emit == "radices") {
    for (int64_t r : prog.radices()) std::cout << r << " ";
    std::cout << "\n";
  } else {
    throw UsageError("--emit ir|kernels|radices");
  }
  return 0;
}

int cmd_run(const Args &a) {
  PipelineConfig c = config_from(a);
  c.batch = 1;
  std::vector<cplx> x;
  if (a.has("--random")) {
    x = seeded_input(c.n, std::stoull(a.get("--random")));
  } else if (a.has("--input")) {
    std::ifstream in(a.get("--input"));
    if (!in) throw Error("cannot open input file " + a.get("--input"));
    double re, im;
    while (in >> re >> im) x.emplace_back(re, im);
    if ((int64_t)x.size() != c.n)
      throw Error("input file holds " + std::to_string(x.size()) + " values, expected " + std::to_string(c.n));
  } else {
    throw UsageError("run: need --input FILE or --random SEED");
  }
  auto prog = compile_pipeline(c);
  const auto out = interpret(prog, ComplexBuffer::from_vector(x, c.layout),
                             a.has("--inverse") ? Direction::Inverse : Direction::Forward);
  for (int64_t j = 0; j < out.logical_len; ++j) std::printf("%.17g %.17g\n", out.get(j).real(), out.get(j).imag());
  return 0;
}

int cmd_verify(const Args &a) {
  const auto sizes = parse_sizes(a.get("--sizes", "16..4096"));
  const int inputs = std::stoi(a.get("--inputs", "5"));
  int cases = 0, failures = 0;
  for (int64_t n : sizes) {
    std::vector<std::vector<cplx>> xs, want;
    for (int t = 0; t < inputs; ++t) {
      xs.push_back(seeded_input(n, 1 + t));
      want.push_back(dft(xs.back()));
    }
    for (Algorithm alg : {Algorithm::CooleyTukey, Algorithm::Stockham})
      for (int64_t radix : {2, 4, 16}) {
        if (radix > n || n % radix != 0) continue;
        for (ComplexLayout lay : {ComplexLayout::Interleaved, ComplexLayout::Split}) {
          PipelineConfig c;
          c.n = n;
          c.algorithm = alg;
          c.radix = radix;
          c.layout = lay;
          c.batch = inputs;
          auto prog = compile_pipeline(c);
          std::vector<ComplexBuffer> in;
          for (const auto &x : xs) in.push_back(ComplexBuffer::from_vector(x, lay));
          const auto out = interpret(prog, in);
          double err = 0;
          for (int t = 0; t < inputs; ++t) err = std::max(err, error_metric(out[t].to_vector(), want[t]));
          const bool pass = err < 1e-7;
          std::printf("%s %s err=%.3e\n", pass ? "PASS" : "FAIL", describe(c).c_str(), err);
          ++cases;
          failures += !pass;
        }
      }
  }
  std::printf("%d configurations, %d failed\n", cases, failures);
  return failures == 0 ? 0 : 1;
}

int cmd_bench(const Args &a) {
  const auto sizes = parse_sizes(a.get("--sizes", "", true));
  const std::string csv_path = a.get("--csv", "", true);
  const int64_t repeats = std::stoll(a.get("--repeats", "100"));
  const int64_t batch_bytes = std::stoll(a.get("--batch-bytes", std::to_string(int64_t(1) << 30)));
  const Direction dir = a.has("--inverse") ? Direction::Inverse : Direction::Forward;
  std::ofstream csv(csv_path);
  if (!csv) throw Error("cannot open " + csv_path + " for writing");
  // reference schema (verify.cpp:106-117), then the GPU columns
  csv << "n,algorithm,radix,layout,vector_mode,repeats,mean_seconds,mflops,seed,"
         "gpus,batch,direction,gflops,gbs,roofline_frac\n";
  const double peak_gbs = std::atof(a.get("--peak-gbs", "6549.1").c_str());
  for (int64_t n : sizes) {
    PipelineConfig c;
    c.n = n;
    c.algorithm = Algorithm::Stockham;
    c.radix = std::stoll(a.get("--radix", "2"));
    c.layout = a.get("--layout", "split") == "split" ? ComplexLayout::Split : ComplexLayout::Interleaved;
    c.batch = a.has("--batch") ? std::stoll(a.get("--batch")) : std::max<int64_t>(1, batch_bytes / (8 * n));
    auto prog = compile_pipeline(c);
    const size_t floats = 2 * (size_t)n * (size_t)c.batch;
    float *in = nullptr, *out = nullptr;
    if (cudaMalloc(&in, floats * 4) != cudaSuccess || cudaMalloc(&out, floats * 4) != cudaSuccess)
      throw ExecError("device allocation failed");
    std::vector<float> host(floats);
    for (size_t i = 0; i < floats; ++i) host[i] = (float)((i * 2654435761u) % 2001) / 1000.0f - 1.0f;
    cudaMemcpy(in, host.data(), floats * 4, cudaMemcpyHostToDevice);
    const bool split = c.layout == ComplexLayout::Split;
    const float *i1 = split ? in + (size_t)n * c.batch : nullptr;
    float *o1 = split ? out + (size_t)n * c.batch : nullptr;
    for (int w = 0; w < 3; ++w) prog.execute(dir, in, i1, out, o1, n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int64_t r = 0; r < repeats; ++r) prog.execute(dir, in, i1, out, o1, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mean = ms / 1e3 / repeats;
    const double flops = 5.0 * n * std::log2((double)n) * c.batch;
    const double gbs = 16.0 * n * c.batch / mean / 1e9;
    char row[512];
    std::snprintf(row, sizeof row, "%lld,stockham,%lld,%s,none,%lld,%.9e,%.6f,1,1,%lld,%s,%.3f,%.1f,%.4f",
                  (long long)n, (long long)c.radix, layout_name(c.layout).c_str(), (long long)repeats, mean,
                  flops / mean / 1e6, (long long)c.batch, dir == Direction::Forward ? "forward" : "inverse",
                  flops / mean / 1e9, gbs, gbs / peak_gbs);
    csv << row << "\n";
    std::printf("%s batch=%lld mean=%.3es rate=%.1f gflops %.0f GB/s\n", describe(c).c_str(), (long long)c.batch,
                mean, flops / mean / 1e9, gbs);
    cudaFree(in);
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return 0;
}

}  // namespace

int main(int argc, char **argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s compile|run|verify|bench [options]\n", argv[0]);
    return 2;
  }
  Args a;
  for (int i = 2; i < argc; ++i) a.v.push_back(argv[i]);
  const std::string cmd = argv[1];
  try {
    if (cmd == "compile") return cmd_compile(a);
    if (cmd == "run") return cmd_run(a);
    if (cmd == "verify") return cmd_verify(a);
    if (cmd == "bench") return cmd_bench(a);
    throw UsageError("unknown subcommand " + cmd);
  } catch (const UsageError &e) {
    std::fprintf(stderr, "usage error: %s\n", e.what());
    return 2;
  } catch (const std::invalid_argument &e) {
    std::fprintf(stderr, "usage error: bad number (%s)\n", e.what());
    return 2;
  } catch (const Error &e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
