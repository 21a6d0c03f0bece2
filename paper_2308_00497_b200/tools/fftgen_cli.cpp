// fftgen_cli.cpp -- command-line front end of the B200 path, mirroring the
// reference CLI (proj/tools/main.cpp:28-259) flag for flag:
//
//   fftgen-b200 compile --size N [stage flags] --emit formula|ir|loops|kernels|c
//   fftgen-b200 run     --size N [stage flags] (--random SEED | --input FILE) [--inverse]
//   fftgen-b200 verify  [--sizes 16..4096|a,b,c] [--inputs 5]
//   fftgen-b200 bench   --sizes ... --csv PATH [stage flags] [--repeats R]
//                       [--device [--batch B] [--inverse] [--peak-gbs G]]
//
// stage flags (StageFlags, main.cpp:28-85): --algorithm cooley-tukey|stockham,
// --radix R, --layout interleaved|split, --vectorize none|inner|outer,
// --vector-width W, --interleaved-opt, --tile-size T | --tile-cache BYTES; and
// the B200 radix hint --pass-radix 8|16|32 (register passes of at most that radix).
//
// Exit codes: 0 success, 1 failed verification or runtime error (an
// fftgen::Error), 2 usage error (main.cpp:250-258).  `verify` is the
// reference's run_verification matrix (verify.cpp:127-181) through the GPU
// program; `bench` writes the reference CSV (verify.cpp:80-117: interpret()
// timing, the reference's end-to-end rate); `bench --device` times batched
// executes on device-resident data and adds the GPU columns.  `--emit c`
// (the reference's scalar C emitter) has no B200 counterpart: LowerError.
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
#include "fftgen_b200_verify.hpp"

using namespace fftgen;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

struct Args {
  std::vector<std::string> v;
  size_t i = 0;
  bool has(const char *flag) const {
    for (const auto &s : v)
      if (s == flag) return true;
    return false;
  }
  std::string get(const char *flag, const std::string &def = "", bool required = false) const {
    for (size_t k = 0; k < v.size(); ++k)
      if (v[k] == flag) {
        if (k + 1 >= v.size() || v[k + 1].rfind("--", 0) == 0)
          throw UsageError(std::string(flag) + " needs a value");
        return v[k + 1];
      }
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

// StageFlags::to_config (main.cpp:62-85): shape errors are usage errors
PipelineConfig config_from(const Args &a, bool with_size = true) {
  PipelineConfig c;
  if (with_size) {
    c.n = std::stoll(a.get("--size", "0", true));
    if (!is_pow2(c.n)) throw UsageError("--size must be a power of two");
  }
  const std::string alg = a.get("--algorithm", "cooley-tukey");
  if (alg != "cooley-tukey" && alg != "stockham") throw UsageError("--algorithm cooley-tukey|stockham");
  c.algorithm = alg == "stockham" ? Algorithm::Stockham : Algorithm::CooleyTukey;
  c.radix = std::stoll(a.get("--radix", "2"));
  if (!is_pow2(c.radix) || c.radix < 2) throw UsageError("--radix must be a power of two >= 2");
  const std::string lay = a.get("--layout", "interleaved");
  if (lay != "interleaved" && lay != "split") throw UsageError("--layout interleaved|split");
  c.layout = lay == "split" ? ComplexLayout::Split : ComplexLayout::Interleaved;
  const std::string vec = a.get("--vectorize", "none");
  if (vec != "none" && vec != "inner" && vec != "outer") throw UsageError("--vectorize none|inner|outer");
  c.vec = vec == "none" ? VecMode::None : (vec == "inner" ? VecMode::Inner : VecMode::Outer);
  c.vector_width = std::stoll(a.get("--vector-width", "8"));
  c.interleaved_opt = a.has("--interleaved-opt");
  if (c.interleaved_opt && c.layout == ComplexLayout::Split)
    throw UsageError("--interleaved-opt only applies to the interleaved layout");
  if (a.has("--tile-size") && a.has("--tile-cache")) throw UsageError("--tile-size excludes --tile-cache");
  const int64_t ts = std::stoll(a.get("--tile-size", "0")), tcache = std::stoll(a.get("--tile-cache", "0"));
  if (ts > 0) c.tile = TilePolicy::exact(ts);
  else if (tcache > 0) c.tile = TilePolicy::cache(tcache);
  c.batch = std::stoll(a.get("--batch", "1"));
  c.pass_radix = std::stoi(a.get("--pass-radix", "0"));  // B200 extension: radix hint for the register passes
  return c;
}

fftgen_config c_config(const PipelineConfig &c) {
  fftgen_config f;
  fftgen_config_init(&f);
  f.n = c.n;
  f.algorithm = c.algorithm == Algorithm::Stockham ? FFTGEN_ALG_STOCKHAM : FFTGEN_ALG_COOLEY_TUKEY;
  f.radix = static_cast<int32_t>(c.radix);
  f.layout = c.layout == ComplexLayout::Split ? FFTGEN_LAYOUT_SPLIT : FFTGEN_LAYOUT_INTERLEAVED;
  f.vec = c.vec == VecMode::Inner ? FFTGEN_VEC_INNER : (c.vec == VecMode::Outer ? FFTGEN_VEC_OUTER : FFTGEN_VEC_NONE);
  f.vector_width = static_cast<int32_t>(c.vector_width);
  f.interleaved_opt = c.interleaved_opt;
  f.pass_radix = c.pass_radix;
  if (c.tile) {
    f.tile_kind = c.tile->kind == TilePolicy::ExactSize ? FFTGEN_TILE_EXACT : FFTGEN_TILE_CACHE;
    f.tile_value = c.tile->value;
  }
  return f;
}

// host-only texts (no device): formula, ir, loops, radices
std::string program_text(const PipelineConfig &c, int what) {
  const fftgen_config f = c_config(c);
  std::vector<char> buf(1 << 16);
  fftgen_status st;
  while ((st = fftgen_program_text(&f, what, buf.data(), buf.size())) == FFTGEN_ERR_DIMENSION &&
         buf.size() < (size_t(1) << 28))
    buf.resize(buf.size() * 4);
  check(st);
  return std::string(buf.data());
}

// cmd_compile (main.cpp:127-148)
int cmd_compile(const Args &a) {
  const std::string emit = a.get("--emit", "", true);
  if (emit != "formula" && emit != "ir" && emit != "loops" && emit != "kernels" && emit != "c" && emit != "radices")
    throw UsageError("--emit formula|ir|loops|kernels|c");
  if (emit == "c" && a.get("--vectorize", "none") != "none")
    throw UsageError("--emit c is scalar only; use --vectorize none");
  const PipelineConfig c = config_from(a);
  if (emit == "formula") {
    std::cout << program_text(c, FFTGEN_TEXT_FORMULA);
  } else if (emit == "ir") {
    std::cout << program_text(c, FFTGEN_TEXT_PIPELINE);
  } else if (emit == "loops") {
    std::cout << program_text(c, FFTGEN_TEXT_LOOPS);
  } else if (emit == "radices") {
    std::cout << program_text(c, FFTGEN_TEXT_RADICES);
  } else if (emit == "kernels") {
    std::cout << compile_pipeline(c).describe();
  } else {
    program_text(c, FFTGEN_TEXT_PIPELINE);  // the config's own errors first
    throw LowerError("LowerError: --emit c: the B200 program is a device plan, not a scalar C translation unit");
  }
  return 0;
}

// cmd_run (main.cpp:150-165): prints "%.17g %.17g" per output element
int cmd_run(const Args &a) {
  if (!a.has("--random") && !a.has("--input")) throw UsageError("run: need --input FILE or --random SEED");
  if (a.has("--random") && a.has("--input")) throw UsageError("--random excludes --input");
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

// cmd_verify (main.cpp:167-179): run_verification through the GPU program
int cmd_verify(const Args &a) {
  const auto sizes = parse_sizes(a.get("--sizes", "16..4096"));
  const int inputs = std::stoi(a.get("--inputs", "5"));
  const auto cases = run_verification(sizes, inputs);
  int failures = 0;
  for (const VerifyCase &vc : cases) {
    std::printf("%s %s err=%.3e\n", vc.pass ? "PASS" : "FAIL", describe_config(vc.config).c_str(), vc.max_error);
    failures += !vc.pass;
  }
  std::printf("%zu configurations, %d failed\n", cases.size(), failures);
  return failures == 0 ? 0 : 1;
}

// cmd_bench (main.cpp:181-197): the reference CSV of bench() per size
int cmd_bench_reference(const Args &a) {
  const auto sizes = parse_sizes(a.get("--sizes", "", true));
  const std::string csv_path = a.get("--csv", "", true);
  const int64_t repeats = std::stoll(a.get("--repeats", "1000"));
  PipelineConfig flags = config_from(a, false);
  std::ofstream csv(csv_path);
  if (!csv) throw Error("cannot open " + csv_path + " for writing");
  csv << bench_csv_header() << "\n";
  for (int64_t n : sizes) {
    flags.n = n;
    const BenchResult r = bench(flags, repeats);
    csv << bench_csv_row(r) << "\n";
    std::printf("%s mean=%.3es rate=%.1f mflops\n", describe_config(r.config).c_str(), r.mean_seconds,
                r.rate_mflops);
  }
  return 0;
}

// bench --device: batched executes on device-resident data, CUDA-event timed
int cmd_bench(const Args &a) {
  if (!a.has("--device")) return cmd_bench_reference(a);
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
    std::printf("%s batch=%lld mean=%.3es rate=%.1f gflops %.0f GB/s\n", describe_config(c).c_str(), (long long)c.batch,
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
    // every value option must carry a value wherever it appears (CLI11 semantics)
    static const char *kValueFlags[] = {"--size", "--algorithm", "--radix", "--layout", "--vectorize",
                                        "--vector-width", "--tile-size", "--tile-cache", "--emit", "--input",
                                        "--random", "--sizes", "--inputs", "--repeats", "--csv", "--batch",
                                        "--batch-bytes", "--peak-gbs", "--pass-radix"};
    for (size_t k = 0; k < a.v.size(); ++k)
      for (const char *f : kValueFlags)
        if (a.v[k] == f && (k + 1 >= a.v.size() || a.v[k + 1].rfind("--", 0) == 0))
          throw UsageError(std::string(f) + " needs a value");
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
