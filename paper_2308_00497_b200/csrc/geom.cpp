// geom.cpp -- host queries of the K2 pass geometry (block_geom.hpp) and the
// fp64-accurate fp32 pass twiddle tables.  Host-only; no CUDA needed.
#include <string>
#include <vector>

#include "block_geom.hpp"
#include "plan.hpp"

namespace fftgen_b200 {

namespace {
template <int N> struct GeomQuery {
  static int passes() { return BlockGeom<N>::P; }
  static void pass(int p, int64_t *R, int64_t *cols, int64_t *k) {
    *R = BlockGeom<N>::R(p);
    *cols = BlockGeom<N>::COLS(p);
    *k = BlockGeom<N>::K(p);
  }
  static void launch(int64_t *threads, int64_t *tpb, int64_t *smem) {
    *threads = BlockGeom<N>::THREADS;
    *tpb = BlockGeom<N>::TPB;
    *smem = SmemGeom<N>::BYTES;
  }
};
#define FFTGEN_GEOM_SWITCH(EXPR)                 \
  switch (log2n) {                               \
  case 0: { using Q = GeomQuery<1>; EXPR; }      \
  case 1: { using Q = GeomQuery<2>; EXPR; }      \
  case 2: { using Q = GeomQuery<4>; EXPR; }      \
  case 3: { using Q = GeomQuery<8>; EXPR; }      \
  case 4: { using Q = GeomQuery<16>; EXPR; }     \
  case 5: { using Q = GeomQuery<32>; EXPR; }     \
  case 6: { using Q = GeomQuery<64>; EXPR; }     \
  case 7: { using Q = GeomQuery<128>; EXPR; }    \
  case 8: { using Q = GeomQuery<256>; EXPR; }    \
  case 9: { using Q = GeomQuery<512>; EXPR; }    \
  case 10: { using Q = GeomQuery<1024>; EXPR; }  \
  case 11: { using Q = GeomQuery<2048>; EXPR; }  \
  case 12: { using Q = GeomQuery<4096>; EXPR; }  \
  case 13: { using Q = GeomQuery<8192>; EXPR; }  \
  case 14: { using Q = GeomQuery<16384>; EXPR; } \
  default: throw PlanError("no block kernel for 2^" + std::to_string(log2n)); \
  }
}  // namespace

int block_num_passes(int log2n) { FFTGEN_GEOM_SWITCH(return Q::passes()) }

void block_pass(int log2n, int p, int64_t *R, int64_t *cols, int64_t *k) {
  FFTGEN_GEOM_SWITCH(Q::pass(p, R, cols, k); return)
}

void block_launch_geom(int log2n, int64_t *threads, int64_t *tpb, int64_t *smem) {
  FFTGEN_GEOM_SWITCH(Q::launch(threads, tpb, smem); return)
}

// [A][m] tables of w_s^{A m} for passes 1..P-1, fp64 -> fp32 (forward sign).
std::vector<float> block_twiddles(int log2n) {
  std::vector<float> out;
  auto push = [&](int64_t s, int64_t e) {
    double re, im;
    unit_root(s, e, &re, &im);
    out.push_back(static_cast<float>(re));
    out.push_back(static_cast<float>(im));
  };
  const int np = block_num_passes(log2n);
  for (int p = 1; p < np; ++p) {
    int64_t R, cols, k;
    block_pass(log2n, p, &R, &cols, &k);
    for (int64_t A = 0; A < R; ++A)
      for (int64_t m = 0; m < cols; ++m) push(R * cols, A * m);
  }
  // factor tables of the passes with >= 1024 columns (BlockGeom::TW_FACTORED):
  // [A][h] = w_s^{A 32 h}, then [A][l] = w_s^{A l}, h, l < 32
  for (int p = 1; p < np; ++p) {
    int64_t R, cols, k;
    block_pass(log2n, p, &R, &cols, &k);
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
