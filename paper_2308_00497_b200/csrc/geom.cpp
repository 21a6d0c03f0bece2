// geom.cpp -- host queries of the K2 pass geometry (block_geom.hpp) and the
// fp64-accurate fp32 pass twiddle tables.  Host-only; no CUDA needed.
#include <string>
#include <vector>

#include "block_geom.hpp"
#include "plan.hpp"

namespace fftgen_b200 {

namespace {
template <int N, class PL = BlockPlan<N>> struct GeomQuery {
  using G = BlockGeom<N, 0, PL>;
  static int passes() { return G::P; }
  static void pass(int p, int64_t *R, int64_t *cols, int64_t *k) {
    *R = G::R(p);
    *cols = G::COLS(p);
    *k = G::K(p);
  }
  static void launch(int64_t *threads, int64_t *tpb, int64_t *smem) {
    *threads = G::THREADS;
    *tpb = G::TPB;
    *smem = SmemGeom<N, PL>::BYTES;
  }
};
// the plan a (N, pass-radix cap) pair runs: the capped plan when it differs
// from the default (CapPlanGeom::DISTINCT), else the default
template <int N, class F> decltype(auto) with_plan(int cap, F &&f) {
  if (cap == 8 && CapPlanGeom<N, 8>::DISTINCT) return f(GeomQuery<N, typename CapPlanGeom<N, 8>::type>{});
  if (cap == 16 && CapPlanGeom<N, 16>::DISTINCT) return f(GeomQuery<N, typename CapPlanGeom<N, 16>::type>{});
  if (cap == 32 && CapPlanGeom<N, 32>::DISTINCT) return f(GeomQuery<N, typename CapPlanGeom<N, 32>::type>{});
  return f(GeomQuery<N>{});
}
template <int N> bool cap_distinct(int cap) {
  return (cap == 8 && CapPlanGeom<N, 8>::DISTINCT) || (cap == 16 && CapPlanGeom<N, 16>::DISTINCT) ||
         (cap == 32 && CapPlanGeom<N, 32>::DISTINCT);
}
#define FFTGEN_GEOM_CASE(L, NN, BODY) \
  case L: return with_plan<NN>(cap, [&](auto q) { using Q = decltype(q); BODY; });
#define FFTGEN_GEOM_SWITCH(BODY)                                                                             \
  switch (log2n) {                                                                                           \
    FFTGEN_GEOM_CASE(0, 1, BODY) FFTGEN_GEOM_CASE(1, 2, BODY) FFTGEN_GEOM_CASE(2, 4, BODY)                   \
    FFTGEN_GEOM_CASE(3, 8, BODY) FFTGEN_GEOM_CASE(4, 16, BODY) FFTGEN_GEOM_CASE(5, 32, BODY)                 \
    FFTGEN_GEOM_CASE(6, 64, BODY) FFTGEN_GEOM_CASE(7, 128, BODY) FFTGEN_GEOM_CASE(8, 256, BODY)              \
    FFTGEN_GEOM_CASE(9, 512, BODY) FFTGEN_GEOM_CASE(10, 1024, BODY) FFTGEN_GEOM_CASE(11, 2048, BODY)         \
    FFTGEN_GEOM_CASE(12, 4096, BODY) FFTGEN_GEOM_CASE(13, 8192, BODY) FFTGEN_GEOM_CASE(14, 16384, BODY)      \
  default: throw PlanError("no block kernel for 2^" + std::to_string(log2n));                               \
  }
}  // namespace

int block_num_passes(int log2n, int cap) { FFTGEN_GEOM_SWITCH(return Q::passes()) }

void block_pass(int log2n, int p, int64_t *R, int64_t *cols, int64_t *k, int cap) {
  FFTGEN_GEOM_SWITCH(Q::pass(p, R, cols, k))
}

void block_launch_geom(int log2n, int64_t *threads, int64_t *tpb, int64_t *smem, int cap) {
  FFTGEN_GEOM_SWITCH(Q::launch(threads, tpb, smem))
}

bool block_cap_distinct(int log2n, int cap) {
  switch (log2n) {
  case 7: return cap_distinct<128>(cap);
  case 8: return cap_distinct<256>(cap);
  case 9: return cap_distinct<512>(cap);
  case 10: return cap_distinct<1024>(cap);
  case 11: return cap_distinct<2048>(cap);
  case 12: return cap_distinct<4096>(cap);
  case 13: return cap_distinct<8192>(cap);
  case 14: return cap_distinct<16384>(cap);
  default: return false;
  }
}

// [A][m] tables of w_s^{A m} for passes 1..P-1, fp64 -> fp32 (forward sign).
std::vector<float> block_twiddles(int log2n, int cap) {
  std::vector<float> out;
  auto push = [&](int64_t s, int64_t e) {
    double re, im;
    unit_root(s, e, &re, &im);
    out.push_back(static_cast<float>(re));
    out.push_back(static_cast<float>(im));
  };
  const int np = block_num_passes(log2n, cap);
  for (int p = 1; p < np; ++p) {
    int64_t R, cols, k;
    block_pass(log2n, p, &R, &cols, &k, cap);
    for (int64_t A = 0; A < R; ++A)
      for (int64_t m = 0; m < cols; ++m) push(R * cols, A * m);
  }
  // factor tables of the passes with >= 1024 columns (BlockGeom::TW_FACTORED):
  // [A][h] = w_s^{A 32 h}, then [A][l] = w_s^{A l}, h, l < 32
  for (int p = 1; p < np; ++p) {
    int64_t R, cols, k;
    block_pass(log2n, p, &R, &cols, &k, cap);
    if (cols < FFTGEN_TW_FACTOR_COLS) continue;
    for (int64_t A = 0; A < R; ++A)
      for (int64_t h = 0; h < 32; ++h) push(R * cols, A * 32 * h);
    for (int64_t A = 0; A < R; ++A)
      for (int64_t l = 0; l < 32; ++l) push(R * cols, A * l);
  }
  return out;
}

// the same [A][m] tables for a K3 group's NS-point sub-FFT plan (GroupPlan)
std::vector<float> group_twiddles(int log2ns) {
  std::vector<float> out;
  auto emit = [&](auto geom) {
    using G = decltype(geom);
    for (int p = 1; p < G::P; ++p) {
      const int64_t R = G::R(p), cols = G::COLS(p), s = R * cols;
      for (int64_t A = 0; A < R; ++A)
        for (int64_t m = 0; m < cols; ++m) {
          double re, im;
          unit_root(s, A * m, &re, &im);
          out.push_back(static_cast<float>(re));
          out.push_back(static_cast<float>(im));
        }
    }
  };
  switch (log2ns) {
  case 7: emit(BlockGeom<128, 0, GroupPlan<128>>{}); break;
  case 8: emit(BlockGeom<256, 0, GroupPlan<256>>{}); break;
  case 9: emit(BlockGeom<512, 0, GroupPlan<512>>{}); break;
  case 10: emit(BlockGeom<1024, 0, GroupPlan<1024>>{}); break;
  case 11: emit(BlockGeom<2048, 0, GroupPlan<2048>>{}); break;
  case 12: emit(BlockGeom<4096, 0, GroupPlan<4096>>{}); break;
  default: throw PlanError("no group kernel for 2^" + std::to_string(log2ns));
  }
  return out;
}

void group_geom(int log2ns, int64_t *threads, int64_t *tc, int64_t *smem, int64_t *r0) {
  switch (log2ns) {
#define FFTGEN_GG(L, NN)               \
  case L:                              \
    *threads = GroupGeom<NN>::THREADS; \
    *tc = GroupGeom<NN>::TC;           \
    *smem = GroupGeom<NN>::BYTES;      \
    *r0 = GroupGeom<NN>::R0;           \
    return;
    FFTGEN_GG(7, 128) FFTGEN_GG(8, 256) FFTGEN_GG(9, 512) FFTGEN_GG(10, 1024) FFTGEN_GG(11, 2048)
    FFTGEN_GG(12, 4096)
#undef FFTGEN_GG
  default:
    *threads = *tc = *smem = *r0 = 0;
  }
}

}  // namespace fftgen_b200
