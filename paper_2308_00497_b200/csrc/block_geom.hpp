// block_geom.hpp -- compile-time geometry of the K2 block kernel, shared by
// the CUDA kernels (fft_block.cuh) and the host plan builder (geom.cpp).
// Pure constexpr C++17; compiles with g++ and nvcc alike.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define FFTGEN_HD __host__ __device__
#else
#define FFTGEN_HD
#endif

namespace fftgen_b200 {

// -------------------------------------------------------------------------
// Pass plans: radices per pass for each N handled by one CTA.
template <int NP, int R0, int R1, int R2> struct PlanT {
  static constexpr int P = NP;
  FFTGEN_HD static constexpr int r(int p) { return p == 0 ? R0 : (p == 1 ? R1 : R2); }
};
template <int N> struct BlockPlan;
template <> struct BlockPlan<1> : PlanT<1, 1, 1, 1> {};
template <> struct BlockPlan<2> : PlanT<1, 2, 1, 1> {};
template <> struct BlockPlan<4> : PlanT<1, 4, 1, 1> {};
template <> struct BlockPlan<8> : PlanT<1, 8, 1, 1> {};
template <> struct BlockPlan<16> : PlanT<1, 16, 1, 1> {};
template <> struct BlockPlan<32> : PlanT<1, 32, 1, 1> {};
template <> struct BlockPlan<64> : PlanT<1, 64, 1, 1> {};
template <> struct BlockPlan<128> : PlanT<2, 8, 16, 1> {};
template <> struct BlockPlan<256> : PlanT<2, 16, 16, 1> {};
template <> struct BlockPlan<512> : PlanT<2, 16, 32, 1> {};
template <> struct BlockPlan<1024> : PlanT<2, 32, 32, 1> {};
template <> struct BlockPlan<2048> : PlanT<2, 32, 64, 1> {};
template <> struct BlockPlan<4096> : PlanT<2, 64, 64, 1> {};
template <> struct BlockPlan<8192> : PlanT<3, 32, 16, 16> {};
template <> struct BlockPlan<16384> : PlanT<3, 32, 32, 16> {};

template <int N> struct BlockGeom {
  using PL = BlockPlan<N>;
  static constexpr int P = PL::P;
  static constexpr int RMAX = PL::r(0) > PL::r(1) ? (PL::r(0) > PL::r(2) ? PL::r(0) : PL::r(2))
                                                  : (PL::r(1) > PL::r(2) ? PL::r(1) : PL::r(2));
  static constexpr int T = N / RMAX;                           // threads per transform
  static constexpr int TPB = T >= 128 ? 1 : 128 / T;           // transforms per CTA
  static constexpr int THREADS = T * TPB;
  FFTGEN_HD static constexpr int R(int p) { return PL::r(p); }
  FFTGEN_HD static constexpr int S(int p) {          // cumulative size after pass p
    int s = 1;
    for (int q = 0; q <= p; ++q) s *= PL::r(q);
    return s;
  }
  FFTGEN_HD static constexpr int COLS(int p) { return S(p) / PL::r(p); }
  FFTGEN_HD static constexpr int K(int p) { return N / S(p); }
  // offset of pass p's [A][m] twiddle table (p >= 1) inside the plan table
  FFTGEN_HD static constexpr int TW_OFF(int p) {
    int o = 0;
    for (int q = 1; q < p; ++q) o += PL::r(q) * COLS(q);
    return o;
  }
  static constexpr int TW_LEN = P > 1 ? TW_OFF(P) : 0;
};

// -------------------------------------------------------------------------
// Shared-memory padding: padded(i) = i + K * (i / PP).  Chosen per pass
// boundary at compile time by simulating warp 0's writer (pass p) and reader
// (pass p+1) addresses and minimising the worst bank-conflict degree.
struct Pad {
  int PP;
  int K;
};
FFTGEN_HD constexpr int padded(int i, Pad pd) { return pd.K ? i + pd.K * (i / pd.PP) : i; }

template <int N> struct PadSearch {
  using G = BlockGeom<N>;
  // worst conflict over the writer of pass p and the reader of pass p+1.
  // Lanes of one access touch distinct elements, so the degree is the
  // largest per-bank count.  Representative registers x and butterflies j
  // suffice: the patterns are affine in both.
  static constexpr int cost(int p, Pad pd) {
    const int T = G::T;
    int worst = 0;
    for (int side = 0; side < 2; ++side) {
      const int q = p + side;
      const int R = G::R(q), cols = G::COLS(q), k = G::K(q), J = G::RMAX / G::R(q);
      const int xs[4] = {0, 1, R / 2, R - 1};
      const int js[2] = {0, J - 1};
      for (int jj = 0; jj < 2; ++jj)
        for (int xx = 0; xx < 4; ++xx) {
          const int j = js[jj], x = xs[xx];
          int cnt[32] = {};
          for (int l = 0; l < 32; ++l) {
            const int t = l % T, f = l / T;  // T < 32: other transforms
            const int u = t + j * T, m = u / k, c = u % k;
            const int idx = side == 0 ? (x * cols + m) * k + c : (m * R + x) * k + c;
            const int b = (padded(idx, pd) + f * (padded(N - 1, pd) + 1)) & 31;
            cnt[b]++;
            worst = cnt[b] > worst ? cnt[b] : worst;
          }
        }
    }
    return worst;
  }
  static constexpr Pad best(int p) {
    Pad bestp{32, 0};
    int bc = 1 << 30, bo = 1 << 30;
    for (int PP = 32; PP <= N; PP *= 2)
      for (int K = 0; K <= 32; K = K ? K * 2 : 1) {
        const Pad pd{PP, K};
        const int c = cost(p, pd);
        const int o = K * (N / PP);
        if (c < bc || (c == bc && o < bo)) {
          bc = c;
          bo = o;
          bestp = pd;
        }
      }
    return bestp;
  }
};

template <int N, int p> struct BoundaryPad {
  static constexpr Pad value = BlockGeom<N>::P > 1 ? PadSearch<N>::best(p) : Pad{32, 0};
  static constexpr int region = padded(N - 1, value) + 1;
};

template <int N> struct SmemGeom {
  using G = BlockGeom<N>;
  static constexpr int r0 = BoundaryPad<N, 0>::region;
  static constexpr int r1 = G::P > 2 ? BoundaryPad<N, 1>::region : 0;
  static constexpr int REGION = G::P > 1 ? (r0 > r1 ? r0 : r1) : 0;  // floats per re/im plane
  static constexpr int BYTES = G::TPB * REGION * 2 * 4;
};

// -------------------------------------------------------------------------


}  // namespace fftgen_b200
