// tests/cpp/plan_tool.cpp -- CPU driver over the product's host plan builder
// (paper_2308_00497_b200/csrc/plan.cpp + geom.cpp).  Used by tests/test_plan.py
// to check plan indices against the reference's goldens without a GPU.
//   plan_tool text N ALG RADIX      print_pipeline text
//   plan_tool maps N ALG RADIX      per data-movement / twiddle op: idx kind s values...
//   plan_tool formula N ALG RADIX   print_formula text of the planner
//   plan_tool loops N               the sm_100a pass / group program
//   plan_tool radices N RADIX       Stockham radices, application order
//   plan_tool passes N [PASS_RADIX [LAYOUT]] sm_100a passes: R cols k s
//   plan_tool twiddles N            K2 pass twiddle table (hex floats)
// Exit codes: 0 ok, 1 PlanError, 2 DimensionError, 4 FuseError.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "plan.hpp"

using namespace fftgen_b200;

int main(int argc, char **argv) {
  if (argc < 3) return 2;
  const std::string cmd = argv[1];
  const int64_t n = std::atoll(argv[2]);
  try {
    if (cmd == "text" || cmd == "maps") {
      const int alg = std::atoi(argv[3]);
      const int64_t radix = std::atoll(argv[4]);
      const auto ops = fuse_ops(n, alg, radix);
      if (cmd == "text") {
        std::fputs(pipeline_text(ops, n).c_str(), stdout);
        return 0;
      }
      std::vector<int64_t> map(n);
      for (size_t i = 0; i < ops.size(); ++i) {
        if (ops[i].kind == OP_MKIV || ops[i].kind == OP_IKMV) continue;
        int64_t s = 0;
        op_map(ops[i], n, map.data(), &s);
        std::printf("%zu %d %lld", i, ops[i].kind, (long long)s);
        for (int64_t v : map) std::printf(" %lld", (long long)v);
        std::printf("\n");
      }
    } else if (cmd == "formula") {
      std::printf("%s\n", formula_text(n, std::atoi(argv[3]), std::atoll(argv[4])).c_str());
    } else if (cmd == "loops") {
      std::fputs(program_text(n).c_str(), stdout);
    } else if (cmd == "radices") {
      for (int64_t r : stockham_radices(n, std::atoll(argv[3]))) std::printf("%lld ", (long long)r);
      std::printf("\n");
    } else if (cmd == "passes") {
      const ExecPlan p = build_exec_plan(n, SPLIT_DEFAULT, argc > 3 ? std::atoi(argv[3]) : 0, argc > 4 ? std::atoi(argv[4]) : 0);
      for (const auto &d : p.passes)
        std::printf("%lld %lld %lld %lld\n", (long long)d.R, (long long)d.cols, (long long)d.k, (long long)d.s);
    } else if (cmd == "twiddles") {
      const ExecPlan p = build_exec_plan(n);
      for (float v : p.tw_block) std::printf("%a ", (double)v);
      std::printf("\n");
    }
  } catch (const PlanError &e) {
    std::fprintf(stderr, "PlanError: %s\n", e.what());
    return 1;
  } catch (const DimensionError &e) {
    std::fprintf(stderr, "DimensionError: %s\n", e.what());
    return 2;
  } catch (const FuseError &e) {
    std::fprintf(stderr, "FuseError: %s\n", e.what());
    return 4;
  }
  return 0;
}
