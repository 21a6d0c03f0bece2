// block_geom.hpp -- compile-time geometry of the K2 block kernels, shared by
// the CUDA kernels (fft_block.cuh) and the host plan builder (geom.cpp).
// Pure constexpr C++17; compiles with g++ and nvcc alike.
#pragma once

#include <cstdint>
#include <type_traits>

#ifdef __CUDACC__
#define FFTGEN_HD __host__ __device__
#else
#define FFTGEN_HD
#endif

namespace fftgen_b200 {

// -------------------------------------------------------------------------
// Pass plans: radices per pass for each N handled by one CTA.  Any grouping
// of the reference's radix-2 Stockham stage list is a valid regrouping; the
// register radix is capped at 64 (128 registers of float2 data per thread).
template <int NP, int R0, int R1, int R2, int R3 = 1> struct PlanT {
  static constexpr int P = NP;
  FFTGEN_HD static constexpr int r(int p) { return p == 0 ? R0 : (p == 1 ? R1 : (p == 2 ? R2 : R3)); }
};
template <int N> struct BlockPlan;
template <> struct BlockPlan<1> : PlanT<1, 1, 1, 1> {};
template <> struct BlockPlan<2> : PlanT<1, 2, 1, 1> {};
template <> struct BlockPlan<4> : PlanT<1, 4, 1, 1> {};
template <> struct BlockPlan<8> : PlanT<1, 8, 1, 1> {};
template <> struct BlockPlan<16> : PlanT<2, 4, 4, 1> {};
template <> struct BlockPlan<32> : PlanT<2, 4, 8, 1> {};
// 64 as two radix-8 passes: eight lanes per transform keep loads coalesced
// (one thread per radix-64 transform strided lanes 512 B apart: 0.16 / 0.30)
template <> struct BlockPlan<64> : PlanT<2, 8, 8, 1> {};
template <> struct BlockPlan<128> : PlanT<2, 8, 16, 1> {};
template <> struct BlockPlan<256> : PlanT<2, 16, 16, 1> {};
template <> struct BlockPlan<512> : PlanT<2, 16, 32, 1> {};
template <> struct BlockPlan<1024> : PlanT<2, 32, 32, 1> {};
template <> struct BlockPlan<2048> : PlanT<2, 32, 64, 1> {};
template <> struct BlockPlan<4096> : PlanT<2, 64, 64, 1> {};
template <> struct BlockPlan<8192> : PlanT<3, 32, 16, 16> {};
template <> struct BlockPlan<16384> : PlanT<3, 32, 32, 16> {};

// Pass plans under a register-radix cap (the radix hint,
// fftgen_config.pass_radix = 8 / 16 / 32): the default plan when its radices
// already fit the cap, else the reference's own Stockham shape for that
// radix -- the remainder radix first, then CAP-point passes (plan_stockham,
// formula.cpp:182-195) -- when that needs at most three register passes;
// otherwise the default (a hint never fails a plan).
constexpr int clog2(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}
template <class PL> constexpr int plan_rmax() {
  int m = 1;
  for (int p = 0; p < PL::P; ++p) m = PL::r(p) > m ? PL::r(p) : m;
  return m;
}
template <int N, int CAP> struct CapPlanGeom {
  static constexpr int L = clog2(N), C = clog2(CAP);
  static constexpr bool DEFAULT_FITS = plan_rmax<BlockPlan<N>>() <= CAP;
  static constexpr int NP = L == 0 ? 1 : (L + C - 1) / C;
  static constexpr bool DISTINCT = !DEFAULT_FITS && NP <= 4;
  static constexpr int R0 = N >> (C * (NP - 1));
  using Cap = PlanT<NP, R0, (NP >= 2 ? CAP : 1), (NP >= 3 ? CAP : 1), (NP >= 4 ? CAP : 1)>;
  using type = std::conditional_t<DISTINCT, Cap, BlockPlan<N>>;
};

// Plans of the K3 group sub-FFTs: the block plan of the same size.  (Three
// 8/16-point register passes for NS = 512 / 1024 measured slower on B200:
// 2^18 0.31 vs 0.41, 2^20 0.29 vs 0.37 of the single-pass roofline.)
// (NS = 2^11 / 2^12 as three 16-point passes on 1024-thread tiles measured
// slower too.)
template <int N> struct GroupPlan : BlockPlan<N> {};
#define FFTGEN_GROUP_MAXT_HUGE 512

// TP = transforms per CTA.  0 -> the direct kernel's default (128 threads).
#ifndef FFTGEN_TW_FACTOR_COLS
#define FFTGEN_TW_FACTOR_COLS 1024
#endif
template <int N, int TP_ = 0, class PL_ = BlockPlan<N>> struct BlockGeom {
  using PL = PL_;
  static constexpr int P = PL::P;
  static constexpr int RMAX = plan_rmax<PL>();
  static constexpr int T = N / RMAX;  // threads per transform
  static constexpr int TPB = TP_ ? TP_ : (T >= 128 ? 1 : 128 / T);
  static constexpr int THREADS = T * TPB;
  FFTGEN_HD static constexpr int R(int p) { return PL::r(p); }
  FFTGEN_HD static constexpr int S(int p) {  // cumulative size after pass p
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
  // A pass whose [A][m] table has >= 1024 columns (the last pass of N = 2^14:
  // 128 KB, beyond what L1 keeps next to a 199 KB shared-memory carve-out)
  // reads w_s^{A m} = w_s^{A 32 (m >> 5)} * w_s^{A (m & 31)} from two
  // 32-column tables appended after the pass tables (TW_LEN): 8 KB in L1.
  FFTGEN_HD static constexpr bool TW_FACTORED(int p) { return p >= 1 && COLS(p) >= FFTGEN_TW_FACTOR_COLS; }
  FFTGEN_HD static constexpr int TW_FOFF(int p) {  // factor tables of pass p
    int o = TW_LEN;
    for (int q = 1; q < p; ++q)
      if (TW_FACTORED(q)) o += 2 * 32 * PL::r(q);
    return o;
  }
};

// -------------------------------------------------------------------------
// Shared-memory exchange buffers hold float2 (re, im) elements, accessed with
// 64-bit LDS/STS: a warp access is served as two half-warp wavefronts, each
// conflict-free when its 16 lanes hit 16 distinct 8-byte bank pairs.
// padded(i) = i + K * (i / PP) is chosen per pass boundary at compile time by
// simulating warp 0's writer (pass p) and reader (pass p+1) addresses and
// minimising the wavefront count (ideal: 2 per access).
struct Pad {
  int PP;
  int K;
};
FFTGEN_HD constexpr int padded(int i, Pad pd) { return pd.K ? i + pd.K * (i / pd.PP) : i; }

// ELEM = element bytes: 8 (float2 exchange) or 4 (one re/im plane).
template <int N, int ELEM = 8, class PL = BlockPlan<N>> struct PadSearch {
  using G = BlockGeom<N, 0, PL>;
  static constexpr int WAVE = 128 / ELEM;  // lanes served per shared-memory wavefront
  // Representative registers x and butterflies j suffice: the access
  // patterns are affine in both.
  // stride: float2 between the transforms of a CTA (<= 0: padded(N - 1) + 1)
  static constexpr int cost(int p, Pad pd, int stride = 0) {
    const int T = G::T;
    const int S = stride > 0 ? stride : padded(N - 1, pd) + 1;
    int worst = 0;
    for (int side = 0; side < 2; ++side) {
      const int q = p + side;
      const int R = G::R(q), cols = G::COLS(q), k = G::K(q), J = G::RMAX / G::R(q);
      const int xs[4] = {0, 1, R / 2, R - 1};
      const int js[2] = {0, J - 1};
      for (int jj = 0; jj < 2; ++jj)
        for (int xx = 0; xx < 4; ++xx) {
          const int j = js[jj], x = xs[xx];
          int wavefronts = 0;
          for (int half = 0; half < 32 / WAVE; ++half) {
            int cnt[32] = {};
            int deg = 0;
            for (int l = WAVE * half; l < WAVE * half + WAVE; ++l) {
              const int t = l % T, f = l / T;  // T < 32: other transforms
              const int u = t + j * T, m = u / k, c = u % k;
              const int idx = side == 0 ? (x * cols + m) * k + c : (m * R + x) * k + c;
              const int b = (padded(idx, pd) + f * S) % WAVE;
              cnt[b]++;
              deg = cnt[b] > deg ? cnt[b] : deg;
            }
            wavefronts += deg;
          }
          worst = wavefronts > worst ? wavefronts : worst;
        }
    }
    return worst;
  }
  static constexpr Pad best(int p) {
    Pad bestp{16, 0};
    int bc = 1 << 30, bo = 1 << 30;
    for (int PP = 16; PP <= N; PP *= 2)
      for (int K = 0; K <= 16; K = K ? K * 2 : 1) {
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

template <int N, int p, int ELEM = 8, class PL = BlockPlan<N>> struct BoundaryPad {
  static constexpr Pad value = BlockGeom<N, 0, PL>::P > 1 ? PadSearch<N, ELEM, PL>::best(p) : Pad{16, 0};
  static constexpr int region = padded(N - 1, value) + 1;
  static constexpr int wavefronts = BlockGeom<N, 0, PL>::P > 1 ? PadSearch<N, ELEM, PL>::cost(p, value) : 0;
};

// When a half-warp spans several transforms (T < 16 threads per transform),
// the transform stride itself decides which bank pairs they share: search
// the smallest extra stride F in [0, 16) that minimises the worst simulated
// access of every pass boundary (N = 64: 8-way -> conflict-free).
template <int N, class PL> struct StrideSearch {
  using G = BlockGeom<N, 0, PL>;
  template <int p> static constexpr int boundary_cost(int stride) {
    if constexpr (p + 1 < G::P) return PadSearch<N, 8, PL>::cost(p, BoundaryPad<N, p, 8, PL>::value, stride);
    else return 0;
  }
  static constexpr int worst(int stride) {
    const int c0 = boundary_cost<0>(stride), c1 = boundary_cost<1>(stride), c2 = boundary_cost<2>(stride);
    const int c01 = c0 > c1 ? c0 : c1;
    return c01 > c2 ? c01 : c2;
  }
  static constexpr int best(int base) {
    int bf = 0, bw = worst(base);
    for (int F = 1; F < 16; ++F)
      if (worst(base + F) < bw) bw = worst(base + F), bf = F;
    return bf;
  }
};

template <int N, class PL = BlockPlan<N>> struct SmemGeom {
  using G = BlockGeom<N, 0, PL>;
  static constexpr int r0 = BoundaryPad<N, 0, 8, PL>::region;
  static constexpr int r1 = G::P > 2 ? BoundaryPad<N, 1, 8, PL>::region : 0;
  static constexpr int r2 = G::P > 3 ? BoundaryPad<N, 2, 8, PL>::region : 0;
  static constexpr int r01 = r0 > r1 ? r0 : r1;
  static constexpr int BASE = G::P > 1 ? (r01 > r2 ? r01 : r2) : 0;
  static constexpr int REGION = (G::P > 1 && G::T < 16) ? BASE + StrideSearch<N, PL>::best(BASE) : BASE;  // float2 per transform
  static constexpr int BYTES = G::TPB * REGION * 8;
};

// -------------------------------------------------------------------------
// TMA-pipelined persistent variant: each CTA loops over groups of TP
// transforms; the raw input of group i+1 is fetched by cp.async.bulk into one
// of STAGES stage buffers while group i is computed.  After pass 0 has read a
// stage's raw data, the same stage buffer holds the padded exchange.
// Geometry, measured on B200 (scripts/ab_libs.sh, 1 GiB batches): a 64 KB
// group per stage (TP = 64 KB / 8N transforms, one packed bulk copy per
// plane) and two stages per CTA run at 0.94-1.00 of the measured HBM peak
// for N = 256 .. 2048 (256: 0.94 / 1.00 split / interleaved vs 0.85 / 0.92
// with 16 KB groups; 512: 0.95 / 1.00 vs 0.86 / 0.90; 1024: 0.98 / 0.98 vs
// 0.88 / 0.89; 2048: 0.98 / 0.98 vs 0.86 / 0.87) -- the group's TMA copies
// are large and the compute of one group covers the next one's load.  N =
// 4096 keeps one transform per CTA, single-buffered, six warps more per SM
// (0.95-0.97; 2 x 2 transforms: 0.95), and 8192 is one transform per stage.
template <int N, class PL = BlockPlan<N>> struct TmaGeom {
  static constexpr bool ENABLED = N >= 64 && N <= 8192;
  static constexpr int T = BlockGeom<N, 0, PL>::T;
  static constexpr int tp_bytes = (65536 / (8 * N)) > 0 ? 65536 / (8 * N) : 1;
  static constexpr int TP = N == 4096 ? 1 : tp_bytes;
  using G = BlockGeom<N, TP, PL>;
  static constexpr int THREADS = G::THREADS;
  // (three stages: 2^13 0.69 vs 0.86, 2^10 0.88 vs 0.98; single-buffered
  // 2^13: 0.77 / 0.81 vs 0.86 / 0.86)
  static constexpr int STAGES = N == 4096 ? 1 : 2;
  static constexpr int RAW = 8 * N;                                   // bytes per transform
  static constexpr int XCH = 8 * SmemGeom<N, PL>::REGION;             // padded exchange bytes
  static constexpr int SLOT = ((RAW > XCH ? RAW : XCH) + 127) / 128 * 128;
  static constexpr int STAGE_BYTES = TP * SLOT;
  static constexpr int BYTES = STAGES * STAGE_BYTES + 128;            // + mbarriers
};

// -------------------------------------------------------------------------
// Single-stage TMA variant for the largest smem-resident size (N = 2^14): one
// raw input stage (8N bytes) plus one padded fp32 plane.  Pass 0 reads the
// stage, exchange 1 runs as float2 through the stage (+ the head of the
// plane), the next transform's cp.async.bulk is issued into the stage, and
// exchange 2 goes through the plane (re, then im) behind it.  Measured on
// B200 (1 GiB batches, bulk-store epilogue, factored last-pass twiddles):
// 0.67 / 0.70 of HBM (split / interleaved) vs 0.50 / 0.54 for the direct
// kernel (at 2^13: 0.80 / 0.82 vs 0.86 / 0.86 for the double-buffered TMA
// kernel, so 2^13 keeps that one).
template <int N> struct Tma1Geom {
  static constexpr bool ENABLED = N == 16384;
  using G = BlockGeom<N>;
  static constexpr int THREADS = G::THREADS;
  static constexpr int RAW = 8 * N;
  static constexpr int r0 = BoundaryPad<N, 0, 4>::region;
  static constexpr int r1 = BoundaryPad<N, 1, 4>::region;
  static constexpr int PLANE = ((r0 > r1 ? r0 : r1) * 4 + 127) / 128 * 128;
  static constexpr int BYTES = RAW + PLANE + 128;
  static constexpr int MIN_BLOCKS = (228 * 1024) / (BYTES + 1024) > 0 ? (228 * 1024) / (BYTES + 1024) : 1;
};

// -------------------------------------------------------------------------
// K3 group kernel tile: TC adjacent transforms of size NS per CTA (32-64 KB
// of float2 in shared memory, <= 512 threads); odd per-transform stride REG so
// lanes walking over the tile index f hit distinct bank pairs.
// MAXT caps the threads per CTA.  Tile bytes per NS, measured on B200
// (scripts/gpu_ab.sh): 16-point-codelet groups (NS <= 256) run best as 32 KB
// tiles of 256 threads, four CTAs per SM (2^16 interleaved two-launch 0.50 vs
// 0.44 of the single-pass roofline with 64 KB tiles); 32-point groups
// (NS >= 512) need 64 KB tiles to keep 64-byte column segments (2^20: 0.35
// vs 0.21 with 32 KB).
#ifndef FFTGEN_GROUP_TILE_SMALL
#define FFTGEN_GROUP_TILE_SMALL 32768
#endif
#ifndef FFTGEN_GROUP_TILE_LARGE
#define FFTGEN_GROUP_TILE_LARGE 65536
#endif
// NS = 2^11 / 2^12 groups (the 2-pass plans of 2^21 .. 2^24) keep 128 KB
// tiles -- 8 / 4 columns of 64 / 32 bytes -- one CTA of 256 threads per SM
// with the full register file for the 64-point codelets.
#ifndef FFTGEN_GROUP_TILE_HUGE
#define FFTGEN_GROUP_TILE_HUGE 131072
#endif
// Transform stride REG of a group tile's exchange (float2 between the TC
// transforms): lanes walk the tile index f fastest on the column-mapped
// sides (f = l % TC, t = l / TC), and the first-pass writer of the rows group
// walks t (f = l / T).  With TC >= 16 any odd stride puts a half-warp's 16
// transforms on distinct bank pairs; with TC = 4 / 8 (the NS = 2^11 / 2^12
// tiles) a half-warp mixes f and t, so the stride is searched here by
// simulating every pass boundary's accesses like PadSearch (ideal: 2
// wavefronts per warp access).
template <int NS, int TC, class PL, int ELEM = 8> struct GroupRegSearch {
  using G = BlockGeom<NS, 0, PL>;
  static constexpr int WAVE = 128 / ELEM;  // lanes one shared-memory wavefront serves
  static constexpr Pad PAD0 = BoundaryPad<NS, 0, ELEM, PL>::value;
  static constexpr Pad PAD1 = G::P > 2 ? BoundaryPad<NS, 1, ELEM, PL>::value : Pad{16, 0};
  static constexpr int side_cost(int p, int side, bool rows_map, int reg) {
    const int T = G::T, q = p + side;
    const int R = G::R(q), cols = G::COLS(q), k = G::K(q), J = G::RMAX / G::R(q);
    const Pad pd = p == 0 ? PAD0 : PAD1;
    const int xs[4] = {0, 1, R / 2, R - 1};
    const int js[2] = {0, J - 1};
    int worst = 0;
    for (int jj = 0; jj < 2; ++jj)
      for (int xx = 0; xx < 4; ++xx) {
        int wavefronts = 0;
        for (int half = 0; half < 32 / WAVE; ++half) {
          int cnt[32] = {};
          int deg = 0;
          for (int l = WAVE * half; l < WAVE * half + WAVE; ++l) {
            const int f = rows_map ? l / T : l % TC, t = rows_map ? l % T : l / TC;
            if (f >= TC || t >= T) continue;
            const int u = t + js[jj] * T, m = u / k, c = u % k, x = xs[xx];
            const int idx = side == 0 ? (x * cols + m) * k + c : (m * R + x) * k + c;
            const int b = (padded(idx, pd) + f * reg) % WAVE;
            cnt[b]++;
            deg = cnt[b] > deg ? cnt[b] : deg;
          }
          wavefronts += deg;
        }
        worst = wavefronts > worst ? wavefronts : worst;
      }
    return worst;
  }
  static constexpr int cost(int reg) {
    int worst = 0;
    for (int p = 0; p + 1 < G::P; ++p) {
      int w = side_cost(p, 0, false, reg);
      if (p == 0) {
        const int wr = side_cost(p, 0, true, reg);
        w = wr > w ? wr : w;
      }
      const int r = side_cost(p, 1, false, reg);
      w = r > w ? r : w;
      worst = w > worst ? w : worst;
    }
    return worst;
  }
  static constexpr int best(int base) {  // base: the odd default; move only when strictly better
    int br = base, bc = cost(base);
    for (int r = base + 1; r < base + 32; ++r)
      if (cost(r) < bc) bc = cost(r), br = r;
    return br;
  }
};

template <int NS, int MAXT = (NS >= 2048 ? FFTGEN_GROUP_MAXT_HUGE : 512)> struct GroupGeom {
  using PL = GroupPlan<NS>;
  static constexpr int T = BlockGeom<NS, 0, PL>::T;
  static constexpr int TILE_BYTES =
      NS <= 256 ? FFTGEN_GROUP_TILE_SMALL : (NS <= 1024 ? FFTGEN_GROUP_TILE_LARGE : FFTGEN_GROUP_TILE_HUGE);
  static constexpr int TC_BYTES = TILE_BYTES / (8 * NS);                // transforms per tile
  static constexpr int TC = TC_BYTES * T > MAXT ? MAXT / T : TC_BYTES;  // <= MAXT threads
  using G = BlockGeom<NS, TC, PL>;
  static constexpr int THREADS = G::THREADS;
  static constexpr int EX = SmemGeom<NS, PL>::BASE > NS ? SmemGeom<NS, PL>::BASE : NS;
  // float2 stride between the tile's transforms: odd (lanes over f hit
  // distinct bank pairs) unless the simulated accesses find a better one
  static constexpr int REG = GroupRegSearch<NS, TC, PL>::best(EX | 1);
  static constexpr int REG_WAVEFRONTS = GroupRegSearch<NS, TC, PL>::cost(REG);
  static constexpr int REG_WAVEFRONTS_ODD = GroupRegSearch<NS, TC, PL>::cost(EX | 1);
  static constexpr int BYTES = TC * REG * 8;
  // resident CTAs the register budget must allow: 16-point codelets fit 64
  // registers, 32-point ones (NS >= 512) need 128
  static constexpr int MIN_BLOCKS =
      NS >= 2048 ? (TILE_BYTES > 65536 ? 1 : 2) : (G::RMAX > 16 ? 2 : (THREADS >= 512 ? 2 : (THREADS >= 256 ? 4 : 3)));
  static constexpr int R0 = G::R(0);
  static constexpr int K0 = NS / R0;
};

}  // namespace fftgen_b200
