// plan.cpp -- host plan builder (see plan.hpp).
#include "plan.hpp"

#include <cmath>
#include <sstream>

namespace fftgen_b200 {

namespace {
bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }
int ilog2(int64_t n) {
  int l = 0;
  while ((int64_t(1) << l) < n) ++l;
  return l;
}
void check_sizes(int64_t n, int64_t radix) {
  if (!is_pow2(n))
    throw PlanError("size must be a power of two, got " + std::to_string(n));
  if (radix < 2 || !is_pow2(radix))
    throw PlanError("radix must be a power of two >= 2, got " + std::to_string(radix));
}
void check_kernel_cap(int64_t size) {  // FuseOptions::kernel_cap (rewrite.hpp:66)
  if (size > 64)
    throw FuseError("DFT kernel of size " + std::to_string(size) +
                    " exceeds the kernel cap 64; plan it into smaller factors first");
}
RefOp mk(int kind, int64_t a, int64_t b = 0, int64_t c = 0) { return RefOp{kind, a, b, c, 0, 0, 0}; }
RefOp tw(int64_t total, int64_t block, int64_t repeat) {
  return RefOp{OP_TWIDDLE, 0, 0, 0, total, block, repeat};
}
}  // namespace

void unit_root(int64_t n, int64_t t, double *re, double *im) {
  t %= n;
  if (t < 0) t += n;
  if (4 * t % n == 0) {
    static const double qr[4] = {1.0, 0.0, -1.0, 0.0}, qi[4] = {0.0, -1.0, 0.0, 1.0};
    *re = qr[4 * t / n];
    *im = qi[4 * t / n];
    return;
  }
  const double angle = -2.0 * M_PI * static_cast<double>(t) / static_cast<double>(n);
  *re = std::cos(angle);
  *im = std::sin(angle);
}

// plan_stockham's radix sequence in application order (formula.cpp:168-197):
// r = min(radix, remaining) is pushed from the largest s down, so the
// remainder radix is applied first.
std::vector<int64_t> stockham_radices(int64_t n, int64_t radix) {
  check_sizes(n, radix);
  std::vector<int64_t> push;
  for (int64_t remaining = n; remaining > 1;) {
    const int64_t r = radix < remaining ? radix : remaining;
    push.push_back(r);
    remaining /= r;
  }
  return std::vector<int64_t>(push.rbegin(), push.rend());
}

namespace {
// I_C (x) B = Pi^N_C (B (x) I_C) Pi^N_M  (emit_lifted, rewrite.cpp:60-75)
void emit_lifted(std::vector<RefOp> &ops, int64_t copies, int64_t b_dim, RefOp lifted) {
  if (copies == 1) {
    ops.push_back(lifted);
    return;
  }
  const int64_t n = copies * b_dim;
  ops.push_back(mk(OP_PERMUTE, b_dim, n));
  ops.push_back(lifted);
  ops.push_back(mk(OP_PERMUTE, copies, n));
}

// Fuser::walk over plan_cooley_tukey(n_sub, radix) under I_copies
// (formula.cpp:150-166, rewrite.cpp:94-170): factors apply right to left.
void ct_walk(std::vector<RefOp> &ops, int64_t n_sub, int64_t radix, int64_t copies) {
  if (n_sub <= radix) {
    if (n_sub == 1) return;
    check_kernel_cap(n_sub);
    ops.push_back(mk(OP_IKMV, n_sub, copies));
    return;
  }
  const int64_t k = radix, m = n_sub / radix;
  if (copies == 1)
    ops.push_back(mk(OP_PERMUTE, k, n_sub));
  else
    emit_lifted(ops, copies, n_sub, mk(OP_PKIV, k, n_sub, copies));
  ct_walk(ops, m, radix, copies * k);
  ops.push_back(tw(n_sub, m, 1));
  check_kernel_cap(k);
  emit_lifted(ops, copies, k * m, mk(OP_MKIV, k, m * copies));
}
}  // namespace

std::vector<RefOp> fuse_ops(int64_t n, int algorithm, int64_t radix) {
  check_sizes(n, radix);
  std::vector<RefOp> ops;
  if (algorithm == 0) {
    ct_walk(ops, n, radix, 1);
    return ops;
  }
  if (n == 1) return ops;
  const auto rs = stockham_radices(n, radix);
  int64_t s = 1;
  for (size_t t = 0; t < rs.size(); ++t) {
    const int64_t r = rs[t];
    s *= r;
    const int64_t k = n / s;
    check_kernel_cap(r);
    if (t > 0) {
      // (Pi^s_r (x) I_k) then (D^s_{s/r} (x) I_k)   (formula.cpp:186-190)
      ops.push_back(k == 1 ? mk(OP_PERMUTE, r, s) : mk(OP_PKIV, r, s, k));
      ops.push_back(tw(s, s / r, k));
    }
    ops.push_back(n / r == 1 ? mk(OP_IKMV, r, 1) : mk(OP_MKIV, r, n / r));
  }
  return ops;
}

namespace {
// plan_cooley_tukey(n, radix) (formula.cpp:150-166) printed by print_formula
// (formula.cpp:104-146): compose factors joined by " . ", Kronecker factors
// inside a composition parenthesised, a composition in atom position too.
std::string ct_formula(int64_t n, int64_t radix, bool atom) {
  if (n <= radix) return "DFT " + std::to_string(n);
  const int64_t k = radix, m = n / k;
  const std::string body = "(DFT " + std::to_string(k) + " kron I " + std::to_string(m) + ") . D " +
                           std::to_string(n) + " " + std::to_string(m) + " . (I " + std::to_string(k) + " kron " +
                           ct_formula(m, radix, true) + ") . Pi " + std::to_string(n) + " " + std::to_string(k);
  return atom ? "(" + body + ")" : body;
}
}  // namespace

std::string formula_text(int64_t n, int algorithm, int64_t radix) {
  check_sizes(n, radix);
  if (algorithm == 0) return ct_formula(n, radix, false);
  // plan_stockham(n, radix) (formula.cpp:168-197): per stage, outermost
  // (largest s) first, DFT_r (x) I_{n/r}, then (D^s_{s/r} (x) I_k) and
  // (Pi^s_r (x) I_k) unless s == r
  if (n == 1) return "DFT 1";
  std::vector<std::string> f;
  for (int64_t remaining = n; remaining > 1;) {
    const int64_t r = radix < remaining ? radix : remaining;
    const int64_t s = remaining, k = n / s;
    const std::string rs = std::to_string(r), ss = std::to_string(s), ks = std::to_string(k);
    f.push_back(n / r == 1 ? "DFT " + rs : "(DFT " + rs + " kron I " + std::to_string(n / r) + ")");
    if (s > r) {
      const std::string d = "D " + ss + " " + std::to_string(s / r);
      f.push_back(k == 1 ? d : "(" + d + " kron I " + ks + ")");
      f.push_back("(Pi " + ss + " " + rs + " kron I " + ks + ")");
    }
    remaining /= r;
  }
  std::string out;  // a single factor (n <= radix) prints bare: compose() returns it

  for (size_t i = 0; i < f.size(); ++i) out += (i ? " . " : "") + f[i];
  return out;
}

std::string program_text(int64_t n, int split_mode, int pass_radix, int layout) {
  // the sm_100a execution plan as loop nests: one Stockham stage of radix R
  // per register pass (K2) or per four-step group launch (K3)
  const ExecPlan p = build_exec_plan(n, split_mode, pass_radix, layout);
  std::ostringstream out;
  if (p.strategy == STRAT_IDENTITY) {
    out << "copy: y[0] = x[0]\n";
    return out.str();
  }
  const bool four = p.strategy == STRAT_FOURSTEP;
  out << (four ? "four-step: " : "block: ") << p.passes.size() << (four ? " group launches" : " register passes")
      << " over N = " << n << "\n";
  for (size_t i = 0; i < p.passes.size(); ++i) {
    const PassDesc &d = p.passes[i];
    const bool first = i == 0, last = i + 1 == p.passes.size();
    out << (four ? "group " : "pass ") << i << ": for m < " << d.cols << ", c < " << d.k << ", B < " << d.R
        << ":  y[(B*" << d.cols << " + m)*" << d.k << " + c] = sum_A W_" << d.R << "^(B A) * "
        << (d.cols > 1 ? "w_" + std::to_string(d.s) + "^(A m) * " : std::string())
        << "x[(m*" << d.R << " + A)*" << d.k << " + c]"
        << "   [" << (first ? "HBM" : (four ? "HBM scratch" : "smem")) << " -> "
        << (last ? "HBM" : (four ? "HBM scratch" : "smem")) << "]\n";
  }
  return out.str();
}

std::string pipeline_text(const std::vector<RefOp> &ops, int64_t n) {
  std::ostringstream out;  // print_pipeline format (rewrite.cpp:275-296)
  for (const RefOp &op : ops) {
    switch (op.kind) {
    case OP_MKIV: out << "FusedMKIV(m=" << op.p0 << ", copies=" << op.p1 << ")\n"; break;
    case OP_IKMV: out << "FusedIKMV(n=" << op.p0 << ", copies=" << op.p1 << ")\n"; break;
    case OP_PKIV:
      out << "FusedPKIV(m=" << op.p0 << ", total=" << op.p1 << ", k=" << op.p2 << ")\n";
      break;
    case OP_TWIDDLE: out << "TwiddleMul(len=" << n << ")\n"; break;
    default: out << "Permute(m=" << op.p0 << ", total=" << op.p1 << ")\n"; break;
    }
  }
  return out.str();
}

void op_map(const RefOp &op, int64_t n, int64_t *map, int64_t *s_out) {
  if (s_out) *s_out = 0;
  if (op.kind == OP_PKIV) {  // y[k(i cols + j) + c] = x[k(j p + i) + c]  (rewrite.cpp:217-226)
    const int64_t p = op.p0, cols = op.p1 / op.p0, k = op.p2;
    for (int64_t i = 0; i < p; ++i)
      for (int64_t j = 0; j < cols; ++j)
        for (int64_t c = 0; c < k; ++c) map[k * (i * cols + j) + c] = k * (j * p + i) + c;
  } else if (op.kind == OP_PERMUTE) {  // y[i cols + j] = x[j p + i]  (rewrite.cpp:232-239)
    const int64_t p = op.p0, cols = op.p1 / op.p0;
    for (int64_t i = 0; i < p; ++i)
      for (int64_t j = 0; j < cols; ++j) map[i * cols + j] = j * p + i;
  } else if (op.kind == OP_TWIDDLE) {
    const int64_t period = op.tw_total * op.tw_repeat;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t b = (i % period) / op.tw_repeat;
      map[i] = ((b / op.tw_block) * (b % op.tw_block)) % op.tw_total;
    }
    if (s_out) *s_out = op.tw_total;
  } else {
    throw DimensionError("op is a butterfly, not a data-movement or twiddle op");
  }
}

void check_schedule(int vec, int64_t vector_width, int tile_kind, int64_t tile_value) {
  if (tile_kind < 0 || tile_kind > 2) throw LowerError("unknown tile policy " + std::to_string(tile_kind));
  if (tile_kind != 0 && tile_value <= 0)  // tile_nest (transforms.cpp:85-95)
    throw LowerError(std::string(tile_kind == 1 ? "tile size" : "cache volume") + " must be positive, got " +
                     std::to_string(tile_value));
  if (vec < 0 || vec > 2) throw LowerError("unknown vector mode " + std::to_string(vec));
  if (vec != 0) {  // vectorize (transforms.cpp:349-354)
    if (!is_pow2(vector_width))
      throw LowerError("vector width must be a power of two, got " + std::to_string(vector_width));
    if (vector_width > 64) throw LowerError("vector width capped at 64 lanes");
  }
}

ExecPlan build_exec_plan(int64_t n, int split_mode, int pass_radix, int layout) {
  if (!is_pow2(n)) throw PlanError("size must be a power of two, got " + std::to_string(n));
  ExecPlan p;
  p.n = n;
  p.log2n = ilog2(n);
  if (n == 1) {
    p.strategy = STRAT_IDENTITY;
    return p;
  }
  if (pass_radix != 0 && pass_radix != 8 && pass_radix != 16 && pass_radix != 32 && pass_radix != 64)
    throw PlanError("pass radix hint must be 0, 8, 16, 32 or 64, got " + std::to_string(pass_radix));
  if (p.log2n <= 14) {
    p.strategy = STRAT_BLOCK;
    // measured default: 2^7 .. 2^9 as radix-8 three-pass plans on the direct
    // kernel (1 GiB batches, split / interleaved fraction of HBM: 2^7 0.90 /
    // 1.05 vs 0.85 / 1.01, 2^8 0.99 / 1.05 vs 0.92 / 1.00 (TMA), 2^9 0.98 /
    // 1.04 vs 0.93 / 1.00 (TMA)); interleaved 2^10 / 2^11 as radix-16
    // three-pass plans on the direct kernel (1.05 / 1.01 vs 0.98 / 0.98 TMA;
    // split stays on TMA: 0.96 / 0.95 vs 0.98 / 0.98); pass_radix 64 selects
    // the two-pass plans
    const int dcap = p.log2n >= 7 && p.log2n <= 9 ? 8 : ((p.log2n == 10 || p.log2n == 11) && layout == 0 ? 16 : 0);
    const int cap = pass_radix == 0 ? dcap : (pass_radix == 64 ? 0 : pass_radix);
    p.block_cap = block_cap_distinct(p.log2n, cap) ? cap : 0;
    const int np = block_num_passes(p.log2n, p.block_cap);
    for (int q = 0; q < np; ++q) {
      PassDesc d{};
      block_pass(p.log2n, q, &d.R, &d.cols, &d.k, p.block_cap);
      d.s = d.R * d.cols;
      p.passes.push_back(d);
    }
    p.tw_block = block_twiddles(p.log2n, p.block_cap);
    return p;
  }
  if (p.log2n > 30)
    throw PlanError("size 2^" + std::to_string(p.log2n) + " exceeds the single-GPU limit 2^30");
  // K3 four-step: groups of consecutive Stockham stages, each one kernel
  p.strategy = STRAT_FOURSTEP;
  const std::vector<int> split = group_split(p.log2n, split_mode, layout);
  int64_t s = 1;
  std::vector<int> seen_local;
  for (size_t g = 0; g < split.size(); ++g) {
    GroupDesc d;
    d.log2ns = split[g];
    d.ns = int64_t(1) << d.log2ns;
    d.cols = s;
    s *= d.ns;
    d.s = s;
    d.k = n / s;
    d.rows = g + 1 == split.size();
    int64_t threads, smem;
    group_geom(d.log2ns, &threads, &d.tc, &smem, &d.r0);
    if (d.tc == 0) throw PlanError("no group kernel for 2^" + std::to_string(d.log2ns));
    // local NS-point pass tables, shared by groups of the same NS
    bool found = false;
    for (const GroupDesc &e : p.groups)
      if (e.log2ns == d.log2ns) {
        d.local_off = e.local_off;
        found = true;
      }
    if (!found) {
      d.local_off = (int64_t)p.tw_block.size() / 2;
      const auto t = group_twiddles(d.log2ns);
      p.tw_block.insert(p.tw_block.end(), t.begin(), t.end());
    }
    if (d.cols > 1) {
      d.q_off = p.tw_group_len;
      p.tw_group_len += d.r0 * d.cols;
      d.p_off = p.tw_group_len;
      p.tw_group_len += (d.ns / d.r0) * d.cols;
    }
    p.passes.push_back(PassDesc{d.ns, d.cols, d.k, d.s});
    p.groups.push_back(d);
  }
  p.scratch_buffers = split.size() >= 3 ? 2 : 1;
  return p;
}

std::vector<int> group_split(int log2n, int mode, int layout) {
  // 2 groups up to 2^22 (NS <= 2^11), 3 groups up to 2^28, 4 groups up to
  // 2^30; sizes as even as possible.  mode SPLIT_GROUPS_1024: NS <= 2^10 (2
  // groups up to 2^20); SPLIT_TWO_PASS: 2 groups up to 2^24 (NS <= 2^12, 32 N
  // bytes of HBM traffic instead of 48 N).  Measured on B200 (1 GiB batches,
  // split / interleaved ms): 2^21 10+11 1.05 / 1.00 vs 7+7+7 1.17 / 1.14;
  // 2^22 11+11 1.23 / 1.16 vs 7+7+8 1.15 / 1.08; 2^24 12+12 1.95 / 1.54 vs
  // 8+8+8 1.15 / 1.07 (the 128 KB NS = 4096 tiles leave one CTA per SM).
  // With the plane-exchange TMA kernel for NS >= 2^11 (round 2): 2^22 11+11
  // 1.09 / 1.00 vs 7+7+8 1.13 / 1.10; 2^23 11+12 1.37 / 1.13 vs 1.14 / 1.07
  // and 2^24 12+12 1.58 / 1.27 vs 1.14 / 1.08 stay three-pass.
  // Earlier:
  // 2^28 as 9+9+10 3.43 ms vs 7+7+7+7 3.65 ms; 2^30 as 10+10+10 19.3 ms vs
  // 7+7+8+8 14.3 ms (1024-point columns at a 2^20 stride leave DRAM only
  // 64-byte segments).
  // (+ factored pass-1 twiddles for NS >= 2^11: interleaved 2^23 11+12 0.94
  // vs 1.07 ms per GiB three-pass, 2^24 12+12 1.06 vs 1.06 (batch 8) and
  // 0.146 vs 0.149 ms (batch 1); split 2^23 / 2^24 1.28 / 1.48 vs 1.13 /
  // 1.14 -- the NS = 4096 tiles move 16-byte plane segments -- keep three)
  // (+ TMA tensor stores from the plane kernel: split 2^23 11+12 1.07 vs 1.13
  // ms per GiB -> two; 2^24 1.22 vs 1.15 -> three)
  const int two = mode == SPLIT_GROUPS_1024 ? 20 : (mode == SPLIT_TWO_PASS ? 24 : (layout == 0 ? 24 : 23));
  const int g = log2n <= two ? 2 : (log2n <= 28 ? 3 : 4);
  std::vector<int> out(g, log2n / g);
  // One 2^9 group among 2^8 ones goes first, where the TMA column kernel runs
  // it (measured on B200: 2^17 0.45 / 0.47 vs 0.42 / 0.45, 2^25 0.29 / 0.30 vs
  // 0.27 / 0.28 split / interleaved); otherwise the larger groups go last
  // (2^19 as 10+9: 0.36 vs 0.38).
  const bool large_first = log2n / g == 8 && log2n % g == 1;
  for (int i = 0; i < log2n % g; ++i) out[large_first ? i : g - 1 - i] += 1;
  // Two-group splits chosen from the per-launch rates (B200, ncu launch lists
  // profiles/r2al_k3_launches.txt: rows groups of few points and column
  // groups of many run fastest) and confirmed by sweeps
  // (`scripts/gpu_ab_order.sh`, `gpu_ab_splits.sh`, `gpu_ab_splits2.sh`):
  //   2^18 10+8 (both layouts)  0.460 / 0.458 vs 0.438 / 0.438 for 9+9
  //   2^19 11+8 interleaved     0.470 vs 0.428 (9+10);  split 10+9 0.452 vs 0.415
  //   2^20 12+8 interleaved     0.420 vs 0.411 (10+10); split keeps 10+10
  //   2^21 11+10 interleaved    0.414 vs 0.396 (10+11); split keeps 10+11
  //   2^23 12+11 split          0.316 vs 0.312 (11+12)
  // Rows groups of 128 points lose everywhere (2^16..2^19 as 9+7 .. 12+7).
  if (mode == SPLIT_DEFAULT && g == 2) {
    const bool il = layout == 0;
    int a = 0;
    if (log2n == 18) a = 10;
    else if (log2n == 19) a = il ? 11 : 10;
    else if (log2n == 20 && il) a = 12;
    else if (log2n == 21 && il) a = 11;
    else if (log2n == 23 && !il) a = 12;
    if (a) out = {a, log2n - a};
  }
  // three / four-group plans (`scripts/gpu_ab_splits3.sh`, batch 1): small
  // groups first, the largest last -- 2^26 8+8+10 0.27 / 0.24 vs 0.245 /
  // 0.226 (9+9+8), 2^27 interleaved 8+8+11 0.271 vs 0.251 (9+9+9; split keeps
  // it: 0.238 vs 0.250), 2^28 8+9+11 0.246 / 0.217 vs 0.237 / 0.202
  // (9+9+10), 2^29 interleaved 8+9+12 5.48 vs 6.01 ms (7+7+7+8; split keeps
  // the four groups: 6.73 / 6.51 vs 6.32 ms for 8+9+12 / 8+10+11), 2^30
  // interleaved 8+11+11 12.0 vs 12.3 ms (7+7+8+8; split keeps the four
  // groups: 14.9 vs 13.0 ms); 2^25 keeps 9+8+8 (8+8+9 / 7+8+10 lose 4-10 %)
  if (mode == SPLIT_DEFAULT) {
    const bool il = layout == 0;
    if (log2n == 26) out = {8, 8, 10};
    else if (log2n == 27 && il) out = {8, 8, 11};
    else if (log2n == 28) out = {8, 9, 11};
    else if (log2n == 29 && il) out = {8, 9, 12};
    else if (log2n == 30 && il) out = {8, 11, 11};
  }
  return out;
}

// TMA tiles for first-group columns at NS >= 2^9 and for every NS >= 2^11
// group (the plane-exchange kernel: 2^21 rows 0.339 / 0.363 vs 0.335 / 0.351
// with the plain rows kernel, 2^22 1.09 / 1.00 vs 1.12 / 1.04 ms per GiB)
#ifndef FFTGEN_PLANE_MIN_LOG2
#define FFTGEN_PLANE_MIN_LOG2 11
#endif
bool group_prefers_tma(int log2ns, bool first, bool rows, int64_t cols) {
  // rows: the 2^9 groups and the 2^10 group of 2^19 (cols 512) through the TMA
  // kernel with staged tensor stores (fft_group_tma.cuh); the 2^10 rows of
  // 2^20 stay on the plain kernel (0.383 vs 0.378)
  const bool rows_tma = rows && (log2ns == 9 || (log2ns == 10 && cols <= 512));
  return (!rows && first && log2ns >= 9) || rows_tma || log2ns >= FFTGEN_PLANE_MIN_LOG2;
}

}  // namespace fftgen_b200
