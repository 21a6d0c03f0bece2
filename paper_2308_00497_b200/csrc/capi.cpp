// capi.cpp -- implementation of the C ABI declared in include/fftgen_b200.h.
//
// Host C++ only: validation (mirroring the reference's PlanError /
// DimensionError / ExecError behaviour), plan construction, twiddle upload,
// launch of the sm_100a kernels, and the chunked host<->device pipeline of
// the host-buffer entry points.  No CPU fallback exists: without a usable
// CUDA device every execute fails with FFTGEN_ERR_CUDA.
#include "fftgen_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.hpp"
#include "plan.hpp"

using namespace fftgen_b200;

namespace {
thread_local std::string g_last_error;

fftgen_status fail(fftgen_status st, const std::string &msg) {
  g_last_error = msg;
  return st;
}

fftgen_status cuda_fail(cudaError_t e, const char *what) {
  return fail(FFTGEN_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// NVTX range around each public execute (header-only NVTX3: a no-op unless a
// profiler such as nsys / ncu --nvtx is attached)
struct NvtxRange {
  explicit NvtxRange(const fftgen_plan *p, const char *what);
  ~NvtxRange() { nvtxRangePop(); }
};

struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class F> fftgen_status guarded(F &&f) {
  try {
    return f();
  } catch (const PlanError &e) {
    return fail(FFTGEN_ERR_PLAN, e.what());
  } catch (const FuseError &e) {
    return fail(FFTGEN_ERR_FUSE, e.what());
  } catch (const DimensionError &e) {
    return fail(FFTGEN_ERR_DIMENSION, e.what());
  } catch (const ExecError &e) {
    return fail(FFTGEN_ERR_EXEC, e.what());
  } catch (const LowerError &e) {
    return fail(FFTGEN_ERR_LOWER, e.what());
  } catch (const std::bad_alloc &) {
    return fail(FFTGEN_ERR_NOMEM, "host allocation failed");
  } catch (const std::exception &e) {
    return fail(FFTGEN_ERR_EXEC, e.what());
  }
}
}  // namespace

void fftgen_b200::set_last_error(const std::string &msg) { g_last_error = msg; }

struct fftgen_plan {
  fftgen_config cfg{};
  ExecPlan ex;
  std::vector<int64_t> radices;
  std::vector<RefOp> ops;
  float2 *d_tw = nullptr;
  // K3 four-step: device-generated group twiddles and intermediate buffers
  float2 *d_twg = nullptr;
  float2 *d_scratch = nullptr;
  // cluster plans: a bounded two-launch scratch (allocated with the plan) for
  // data the TMA tiles cannot address (unaligned), used chunk by chunk
  float2 *d_fallback = nullptr;
  size_t scratch_bytes = 0, fallback_bytes = 0;
  int64_t fallback_chunk = 0;  // transforms per two-launch chunk
  // K3 groups: persistent TMA variant (resident CTAs per group, 0 = off)
  std::vector<int> group_tma_grid;
  // K5: 2-group plans run as one cluster per transform (DSMEM intermediate)
  bool use_cluster = false;
  int max_clusters = 0, cluster_size = 0;
  // host-buffer pipeline scratch (lazily allocated, guarded by mu)
  std::mutex mu;
  void *d_stage = nullptr;
  size_t stage_bytes = 0;
  // host pipeline: chunk i uses slot / stream i % kHostSlots, so the H2D copy
  // of one chunk overlaps the kernels and the D2H copy of the previous one
  static constexpr int kHostSlots = 2;
  cudaStream_t streams[kHostSlots] = {};
  // persistent TMA variant: resident CTAs on the device (0 = unavailable)
  int tma_grid = 0;
  bool use_tma = true;
  bool use_tma_store = true;
  bool use_rows = false;  // K2r row kernel (N = 8 .. 64)
};

NvtxRange::NvtxRange(const fftgen_plan *p, const char *what) {
  char msg[96];
  std::snprintf(msg, sizeof msg, "%s n=%lld batch=%lld", what, (long long)p->cfg.n, (long long)p->cfg.batch);
  nvtxRangePushA(msg);
}

namespace {

// Do the strided ranges {a + b*step + [0, width)} and {c + b*step + [0, width)},
// b in [0, count), share a byte?  (Both sides use the plan's dist.)
bool strided_overlap(uintptr_t a, uintptr_t c, int64_t step, int64_t width, int64_t count) {
  const int64_t d = (int64_t)(c - a);  // wraps like the pointers do
  const int64_t span = (count - 1) * step;
  if (d >= span + width || -d >= span + width) return false;  // disjoint extents
  // b2 - b1 = j in (-count, count): is |d + j step| < width for some j?
  const int64_t j0 = step > 0 ? -d / step : 0;
  for (int64_t j = j0 - 1; j <= j0 + 1; ++j)
    if (j > -count && j < count) {
      const int64_t r = d + j * step;
      if (r < width && -r < width) return true;
    }
  return false;
}

fftgen_status validate_exec(const fftgen_plan *p, int direction, const void *in0, const void *in1,
                            const void *out0, const void *out1, int64_t dist) {
  if (!p) return fail(FFTGEN_ERR_INVALID, "NULL plan");
  if (direction != FFTGEN_FORWARD && direction != FFTGEN_INVERSE)
    return fail(FFTGEN_ERR_EXEC, "direction must be FFTGEN_FORWARD (-1) or FFTGEN_INVERSE (+1)");
  if (!in0 || !out0) return fail(FFTGEN_ERR_EXEC, "NULL data pointer");
  const bool split = p->cfg.layout == FFTGEN_LAYOUT_SPLIT;
  if (split && (!in1 || !out1))
    return fail(FFTGEN_ERR_EXEC, "split layout needs both re (in0/out0) and im (in1/out1) pointers");
  if (dist < p->cfg.n)
    return fail(FFTGEN_ERR_DIMENSION, "dist " + std::to_string(dist) + " is smaller than n " +
                                          std::to_string(p->cfg.n));
  // element alignment: float2 for interleaved, float for split
  const uintptr_t al = split ? 4 : 8;
  for (const void *q : {in0, in1, out0, out1})
    if (q && (uintptr_t)q % al != 0)
      return fail(FFTGEN_ERR_EXEC, "data pointer not aligned to its " + std::to_string(al) + "-byte element");
  // exactly in place (out_i == in_i) is supported; any other shared byte
  // between an output plane and an input or the other output plane is not
  const int64_t esz = split ? 4 : 8, step = dist * esz, width = p->cfg.n * esz, cnt = p->cfg.batch;
  const void *ins[2] = {in0, split ? in1 : nullptr}, *outs[2] = {out0, split ? out1 : nullptr};
  for (int o = 0; o < 2; ++o) {
    if (!outs[o]) continue;
    for (int i = 0; i < 2; ++i)
      if (ins[i] && !(i == o && ins[i] == outs[o]) &&
          strided_overlap((uintptr_t)ins[i], (uintptr_t)outs[o], step, width, cnt))
        return fail(FFTGEN_ERR_EXEC, "output plane " + std::to_string(o) + " partially overlaps input plane " +
                                         std::to_string(i) + " (only exactly in-place execution is supported)");
    if (o == 1 && strided_overlap((uintptr_t)outs[0], (uintptr_t)outs[1], step, width, cnt))
      return fail(FFTGEN_ERR_EXEC, "the re and im output planes overlap");
  }
  return FFTGEN_OK;
}

// One K3 group launch: the first group reads the user layout, the last writes
// it, intermediates are interleaved scratch.
GroupArgs make_group_args(const fftgen_plan *p, int g, const void *in0, const void *in1, void *out0, void *out1,
                          int64_t idist, int64_t odist) {
  const GroupDesc &d = p->ex.groups[g];
  GroupArgs a{};
  a.in0 = in0;
  a.in1 = in1;
  a.out0 = out0;
  a.out1 = out1;
  a.cols = d.cols;
  a.k = d.k;
  a.idist = idist;
  a.odist = odist;
  a.tiles_per_outer = (d.cols * d.k) / d.tc;
  a.tw_local = p->d_tw + d.local_off;
  a.tw_q = d.cols > 1 ? p->d_twg + d.q_off : nullptr;
  a.tw_p = d.cols > 1 ? p->d_twg + d.p_off : nullptr;
  return a;
}

// l2: the intermediate is an L2-resident chunk slot (2-group plans)
cudaError_t launch_group(const fftgen_plan *p, int g, int direction, const void *in0, const void *in1,
                         void *out0, void *out1, int64_t idist, int64_t odist, int64_t batch, cudaStream_t s,
                         bool l2 = false) {
  const GroupDesc &d = p->ex.groups[g];
  const bool first = g == 0, last = g + 1 == (int)p->ex.groups.size();
  const bool split = p->cfg.layout == FFTGEN_LAYOUT_SPLIT;
  const GroupArgs a = make_group_args(p, g, in0, in1, out0, out1, idist, odist);
  const int shape = l2 ? (last ? (split ? 8 : 7) : (split ? 6 : 5))
                      : (last ? (split ? 3 : 2) : (first ? (split ? 1 : 0) : 4));
  if (!l2 && g < (int)p->group_tma_grid.size() && p->group_tma_grid[g] > 0) {
    GroupTmaArgs ta{};
    ta.g = a;
    ta.items = batch * a.tiles_per_outer;
    if (group_tma_encode(d.log2ns, shape, batch, ta)) {
      const int grid = (int)std::min<int64_t>(ta.items, p->group_tma_grid[g]);
      return group_tma_launch(d.log2ns, shape, direction, ta, grid, s);
    }
  }
  return group_launch(d.log2ns, shape, direction, a, batch, s);
}

cudaError_t run_groups(const fftgen_plan *p, int direction, const void *in0, const void *in1, void *out0,
                       void *out1, int64_t dist, int64_t batch, float2 *scratch, size_t per, cudaStream_t s);

// Enqueue one execute over `batch` transforms on stream s (device pointers).
cudaError_t enqueue(const fftgen_plan *p, int direction, const void *in0, const void *in1, void *out0,
                    void *out1, int64_t dist, int64_t batch, cudaStream_t s) {
  const int64_t n = p->cfg.n;
  const int layout = p->cfg.layout;
  switch (p->ex.strategy) {
  case STRAT_IDENTITY: {
    if (layout == FFTGEN_LAYOUT_INTERLEAVED)
      return strided_copy((const float *)in0, (float *)out0, batch, 2, 2 * dist, 2 * dist, s);
    cudaError_t e = strided_copy((const float *)in0, (float *)out0, batch, 1, dist, dist, s);
    if (e != cudaSuccess) return e;
    return strided_copy((const float *)in1, (float *)out1, batch, 1, dist, dist, s);
  }
  case STRAT_BLOCK: {
    BlockArgs a{};
    a.in0 = in0;
    a.in1 = in1;
    a.out0 = out0;
    a.out1 = out1;
    a.idist = dist;
    a.odist = dist;
    a.batch = batch;
    a.tw = p->d_tw;
    (void)n;
    // cp.async.bulk needs 16-byte aligned sources and 16-byte multiples
    const int64_t esz = layout == FFTGEN_LAYOUT_SPLIT ? 4 : 8;
    const bool aligned = ((uintptr_t)in0 % 16 == 0) && (!in1 || (uintptr_t)in1 % 16 == 0) &&
                         (dist * esz) % 16 == 0;
    const bool out_aligned = ((uintptr_t)out0 % 16 == 0) && (!out1 || (uintptr_t)out1 % 16 == 0);
    if (p->use_rows && aligned && out_aligned) return rows_launch(p->ex.log2n, layout, direction, a, s);
    if (p->use_tma && p->tma_grid > 0 && aligned) {
      const int64_t tp = block_tma_transforms_per_cta(p->ex.log2n);
      const int grid = (int)std::min<int64_t>((batch + tp - 1) / tp, p->tma_grid);
      const int flags = p->use_tma_store && out_aligned ? BLOCK_TMA_STORE : 0;
      return block_tma_launch(p->ex.log2n, layout, direction, a, grid, flags, s);
    }
    if (p->ex.block_cap) return block_cap_launch(p->ex.log2n, p->ex.block_cap, layout, direction, a, s);
    return block_launch(p->ex.log2n, layout, direction, a, s);
  }
  case STRAT_FOURSTEP: {
    const auto &gs = p->ex.groups;
    const bool split = layout == FFTGEN_LAYOUT_SPLIT;
    const int64_t esz = split ? 4 : 8;
    const bool rows_aligned = ((uintptr_t)in0 % 16 == 0) && (!in1 || (uintptr_t)in1 % 16 == 0) &&
                              (dist * esz) % 16 == 0;
    const bool out_aligned = ((uintptr_t)out0 % 16 == 0) && (!out1 || (uintptr_t)out1 % 16 == 0);
    if (p->use_cluster && rows_aligned && out_aligned) {
      // persistent clusters, one transform per cluster at a time; group-0
      // tiles arrive as TMA tensor boxes, the intermediate moves through DSMEM
      ClusterArgs c{};
      c.in0 = in0;
      c.in1 = in1;
      c.out0 = out0;
      c.out1 = out1;
      c.idist = dist;
      c.odist = dist;
      c.batch = batch;
      c.tw_local0 = p->d_tw + gs[0].local_off;
      c.tw_local1 = p->d_tw + gs[1].local_off;
      c.tw_q = p->d_twg + gs[1].q_off;
      c.tw_p = p->d_twg + gs[1].p_off;
      // a tensor map the driver rejects takes the two-launch path below
      if (cluster_encode_maps(gs[0].log2ns, gs[1].log2ns, p->cluster_size, layout, c) == cudaSuccess)
        return cluster_launch(gs[0].log2ns, gs[1].log2ns, p->cluster_size, layout, direction, c, batch,
                              p->max_clusters, s);
    }
    // two-launch (K3) path; cluster plans run it chunk by chunk through
    // their bounded fallback scratch (no allocation at execute time)
    float2 *scratch = p->use_cluster ? p->d_fallback : p->d_scratch;
    const int64_t chunk = p->use_cluster ? p->fallback_chunk : batch;
    const int64_t esz_in = split ? 1 : 2;  // floats per element of a user plane
    for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
      const int64_t cnt = std::min(chunk, batch - b0);
      const int64_t off = b0 * dist * esz_in;  // float offset of the chunk in the user planes
      const float *i0 = (const float *)in0 + off, *i1 = in1 ? (const float *)in1 + off : nullptr;
      float *o0 = (float *)out0 + off, *o1 = out1 ? (float *)out1 + off : nullptr;
      cudaError_t e = run_groups(p, direction, i0, i1, o0, o1, dist, cnt, scratch, (size_t)chunk * (size_t)n, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  default:
    return cudaErrorNotSupported;
  }
}

// The K3 group launches of one chunk of `batch` transforms; the groups
// ping-pong through interleaved scratch buffers of `per` float2 each:
// in -> S0 [-> S1 -> S0 ...] -> out.
cudaError_t run_groups(const fftgen_plan *p, int direction, const void *in0, const void *in1, void *out0,
                       void *out1, int64_t dist, int64_t batch, float2 *scratch, size_t per, cudaStream_t s) {
  const auto &gs = p->ex.groups;
  const int64_t n = p->cfg.n;
  for (size_t g = 0; g < gs.size(); ++g) {
    const bool first = g == 0, last = g + 1 == gs.size();
    float2 *src = first ? nullptr : scratch + ((g - 1) % p->ex.scratch_buffers) * per;
    float2 *dst = last ? nullptr : scratch + (g % p->ex.scratch_buffers) * per;
    cudaError_t e = launch_group(p, (int)g, direction, first ? in0 : src, first ? in1 : nullptr, last ? out0 : dst,
                                 last ? out1 : nullptr, first ? dist : n, last ? dist : n, batch, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

size_t elem_bytes(const fftgen_plan *p) { return 8; }  // fp32 complex, either layout

// Chunked host pipeline: `stage(chunk_first, count, slot_ptr, stream)`.
template <class F>
fftgen_status host_pipeline(fftgen_plan *p, size_t slot_bytes_per_transform, F &&stage) {
  const int64_t batch = p->cfg.batch;
  constexpr int K = fftgen_plan::kHostSlots;
  // 128 MiB per chunk and slot (in + out), the first and last four chunks
  // ramping 1/16 .. 1/2 of that so the pipeline fills and drains quickly.
  // Measured on B200 at N=4096 split (4 GiB of PCIe traffic per execute,
  // scripts/gpu_e2e_ab.sh): 128 MiB + ramp 4: 347-349 GFLOP/s; 64 MiB: 342-344;
  // 256 MiB: 345; 512 MiB + ramp 6: 330; 4 slots x 32 MiB: 50.2 vs 47.8 ms.
  // fftgen_config.host_chunk_mb overrides the chunk.
  const int64_t target = int64_t(p->cfg.host_chunk_mb > 0 ? p->cfg.host_chunk_mb : 128) << 20;
  int64_t chunk = std::max<int64_t>(1, target / (int64_t)slot_bytes_per_transform);
  chunk = std::min(chunk, batch);
  // ramp: the first chunks are 1/2^RAMP, 1/2^(RAMP-1), ... of a full chunk, so
  // the pipeline fills (H2D of chunk 0 alone) and drains sooner
  constexpr int ramp = 4;
  const size_t slot = (size_t)chunk * slot_bytes_per_transform;
  cudaError_t e;
  if (p->stage_bytes < K * slot) {
    if (p->d_stage) cudaFree(p->d_stage);
    p->d_stage = nullptr;
    p->stage_bytes = 0;
    if ((e = cudaMalloc(&p->d_stage, K * slot)) != cudaSuccess)
      return fail(FFTGEN_ERR_NOMEM, std::string("staging buffers: ") + cudaGetErrorString(e));
    p->stage_bytes = K * slot;
  }
  for (auto &s : p->streams)
    if (!s && (e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
  int i = 0;
  for (int64_t b0 = 0, cnt = 0; b0 < batch; b0 += cnt, ++i) {
    const int64_t want = i < ramp ? std::max<int64_t>(1, chunk >> (ramp - i)) : chunk;
    const int64_t left = batch - b0;
    // ramp down symmetrically: the last chunks shrink like the first ones grew
    int64_t tail = want;
    for (int r = 1; r <= ramp && left <= (chunk >> r) * 2 && (chunk >> r) > 0; ++r) tail = chunk >> r;
    cnt = std::min(std::min(want, tail), left);
    char *slot_ptr = (char *)p->d_stage + (i % K) * slot;
    // four-step plans share one scratch buffer (the two-launch scratch, or a
    // cluster plan's fallback for unaligned chunks): keep their chunks
    // stream-ordered; aligned cluster chunks use no scratch
    const int sid = (p->ex.strategy == STRAT_FOURSTEP && !p->use_cluster) ? 0 : (i % K);
    if ((e = stage(b0, cnt, slot_ptr, p->streams[sid])) != cudaSuccess) {
      // drain what was already enqueued: no copy may still touch the
      // caller's host buffers once this call has returned
      for (auto &st : p->streams) cudaStreamSynchronize(st);
      return cuda_fail(e, "host pipeline");
    }
  }
  fftgen_status st = FFTGEN_OK;
  for (auto &s : p->streams)
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess && st == FFTGEN_OK) st = cuda_fail(e, "cudaStreamSynchronize");
  return st;
}

fftgen_status copy_text(const std::string &s, char *buf, size_t cap) {
  if (!buf || cap == 0) return fail(FFTGEN_ERR_INVALID, "NULL buffer");
  const size_t k = std::min(cap - 1, s.size());
  std::memcpy(buf, s.data(), k);
  buf[k] = 0;
  return s.size() < cap ? FFTGEN_OK : fail(FFTGEN_ERR_DIMENSION, "buffer too small");
}

}  // namespace

extern "C" {

void fftgen_config_init(fftgen_config *cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof *cfg);
  cfg->n = 0;
  cfg->algorithm = FFTGEN_ALG_COOLEY_TUKEY;  // PipelineConfig defaults (driver.hpp:26-35)
  cfg->radix = 2;
  cfg->layout = FFTGEN_LAYOUT_INTERLEAVED;
  cfg->vec = FFTGEN_VEC_NONE;
  cfg->vector_width = 8;
  cfg->interleaved_opt = 0;
  cfg->tile_kind = FFTGEN_TILE_NONE;
  cfg->device = 0;
  cfg->batch = 1;
}

int fftgen_abi_version(void) { return FFTGEN_B200_ABI_VERSION; }

const char *fftgen_error_string(fftgen_status s) {
  switch (s) {
  case FFTGEN_OK: return "ok";
  case FFTGEN_ERR_PLAN: return "PlanError";
  case FFTGEN_ERR_DIMENSION: return "DimensionError";
  case FFTGEN_ERR_EXEC: return "ExecError";
  case FFTGEN_ERR_FUSE: return "FuseError";
  case FFTGEN_ERR_INVALID: return "invalid argument";
  case FFTGEN_ERR_CUDA: return "CUDA error";
  case FFTGEN_ERR_NOMEM: return "out of device memory";
  case FFTGEN_ERR_LOWER: return "LowerError";
  case FFTGEN_ERR_BOUNDS: return "BoundsError";
  case FFTGEN_ERR_GPUMAP: return "GpuMapError";
  }
  return "unknown status";
}

const char *fftgen_last_error(void) { return g_last_error.c_str(); }

fftgen_status fftgen_plan_create(fftgen_plan **out, const fftgen_config *cfg) {
  if (!out || !cfg) return fail(FFTGEN_ERR_INVALID, "NULL plan pointer or config");
  *out = nullptr;
  return guarded([&]() -> fftgen_status {
    if (cfg->layout != FFTGEN_LAYOUT_INTERLEAVED && cfg->layout != FFTGEN_LAYOUT_SPLIT)
      throw ExecError("unknown complex layout " + std::to_string(cfg->layout));
    if (cfg->algorithm != FFTGEN_ALG_COOLEY_TUKEY && cfg->algorithm != FFTGEN_ALG_STOCKHAM)
      throw PlanError("unknown algorithm " + std::to_string(cfg->algorithm));
    if (cfg->batch < 1) throw DimensionError("batch must be >= 1, got " + std::to_string(cfg->batch));
    // same validation order as compile_pipeline: plan_* -> fuse -> tile -> vectorize
    auto ops = fuse_ops(cfg->n, cfg->algorithm, cfg->radix);
    auto radices = stockham_radices(cfg->n, cfg->radix);
    check_schedule(cfg->vec, cfg->vector_width, cfg->tile_kind, cfg->tile_value);
    ExecPlan ex = build_exec_plan(cfg->n,
                                  (cfg->tuning & FFTGEN_TUNE_GROUPS_1024)
                                      ? SPLIT_GROUPS_1024
                                      : ((cfg->tuning & FFTGEN_TUNE_TWO_PASS) ? SPLIT_TWO_PASS : SPLIT_DEFAULT),
                                  cfg->pass_radix, cfg->layout);

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (cfg->device < 0 || cfg->device >= ndev)
      return fail(FFTGEN_ERR_CUDA, "device " + std::to_string(cfg->device) + " not present (" +
                                       std::to_string(ndev) + " visible)");
    DeviceGuard g(cfg->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    int sms = 0;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device)) != cudaSuccess)
      return cuda_fail(e, "device attributes");

    auto *p = new fftgen_plan();
    p->cfg = *cfg;
    p->ex = std::move(ex);
    p->ops = std::move(ops);
    p->radices = std::move(radices);
    auto bail = [&](fftgen_status st, const std::string &msg) {
      fftgen_plan_destroy(p);
      return fail(st, msg);
    };
    const uint32_t tune = cfg->tuning;
    if (p->ex.strategy == STRAT_BLOCK) {
      int per_sm = 0;
      if ((e = block_prepare(p->ex.log2n, &per_sm)) != cudaSuccess)
        return bail(FFTGEN_ERR_GPUMAP, std::string("block kernel attributes: ") + cudaGetErrorString(e));
      p->tma_grid = block_tma_enabled(p->ex.log2n) ? per_sm * sms : 0;
      if (p->ex.block_cap) {  // the radix hint's plan runs on the direct kernel (measured fastest for it)
        if ((e = block_cap_prepare(p->ex.log2n, p->ex.block_cap)) != cudaSuccess)
          return bail(FFTGEN_ERR_GPUMAP, std::string("capped block kernel attributes: ") + cudaGetErrorString(e));
        p->tma_grid = 0;
      }
      p->use_tma = !(tune & FFTGEN_TUNE_NO_TMA);
      p->use_tma_store = !(tune & FFTGEN_TUNE_NO_TMA_STORE);
      // N = 8 .. 64: the row kernel (FFTGEN_TUNE_NO_TMA keeps the direct kernel)
      if (rows_enabled(p->ex.log2n) && !p->ex.block_cap && p->use_tma) {
        if ((e = rows_prepare(p->ex.log2n)) != cudaSuccess)
          return bail(FFTGEN_ERR_GPUMAP, std::string("row kernel attributes: ") + cudaGetErrorString(e));
        p->use_rows = true;
      }
    }
    cudaStream_t ps = nullptr;  // private stream for the plan's own uploads
    if ((e = cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking)) != cudaSuccess)
      return bail(FFTGEN_ERR_CUDA, std::string("stream creation: ") + cudaGetErrorString(e));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{ps};
    if (p->ex.strategy == STRAT_FOURSTEP) {
      for (const GroupDesc &d : p->ex.groups)
        if ((e = group_prepare(d.log2ns)) != cudaSuccess)
          return bail(FFTGEN_ERR_GPUMAP, std::string("group kernel attributes: ") + cudaGetErrorString(e));
      // Persistent TMA group kernels where they measured faster (B200,
      // scripts/gpu_ab.sh, 32 KB tiles for NS <= 256): first-group columns at
      // NS >= 512, whose 64 KB tiles leave one CTA of 256 threads per SM without
      // a prefetch (2^18 split 0.40 vs 0.35, 2^20 0.35 vs 0.32 of the single-pass
      // roofline); the 4-CTA 32 KB plain tiles win below (2^16 split 0.43 vs
      // 0.41) and for rows.  FFTGEN_TUNE_NO_TMA / _GROUP_TMA_ALL force none / all.
      for (size_t gi = 0; gi < p->ex.groups.size(); ++gi) {
        const GroupDesc &d = p->ex.groups[gi];
        const bool want = !(tune & FFTGEN_TUNE_NO_TMA) &&
                          ((tune & FFTGEN_TUNE_GROUP_TMA_ALL) || group_prefers_tma(d.log2ns, gi == 0, d.rows, d.cols));
        int bps = 0;
        if (want && (e = group_tma_prepare(d.log2ns, &bps)) != cudaSuccess)
          return bail(FFTGEN_ERR_GPUMAP, std::string("group TMA kernel attributes: ") + cudaGetErrorString(e));
        p->group_tma_grid.push_back(want ? bps * sms : 0);
      }
      // K4: Q[A0][m] = w_s^{A0 (NS/R0) m}, P[c][m] = w_s^{c m}, generated on the device in fp64
      if (p->ex.tw_group_len > 0) {
        if ((e = cudaMalloc(&p->d_twg, p->ex.tw_group_len * sizeof(float2))) != cudaSuccess)
          return bail(FFTGEN_ERR_NOMEM, std::string("group twiddles: ") + cudaGetErrorString(e));
        for (const GroupDesc &d : p->ex.groups) {
          if (d.cols <= 1) continue;
          // P is [c][m] for column groups (lanes share m) and [m][c] for the
          // rows group (lanes walk c within a row: coalesced twiddle loads)
          if ((e = gen_twiddles(p->d_twg + d.q_off, d.r0, d.cols, d.ns / d.r0, d.s, ps)) != cudaSuccess ||
              (e = d.rows ? gen_twiddles(p->d_twg + d.p_off, d.cols, d.ns / d.r0, 1, d.s, ps)
                          : gen_twiddles(p->d_twg + d.p_off, d.ns / d.r0, d.cols, 1, d.s, ps)) != cudaSuccess)
            return bail(FFTGEN_ERR_CUDA, std::string("twiddle generation: ") + cudaGetErrorString(e));
        }
      }
      const auto &gs = p->ex.groups;
      // K5 where measured faster than K3 (cluster_default_size); config
      // cluster_size forces a compiled (NS0, NS1, C) shape or (-1) never
      int csize = gs.size() == 2 ? cluster_default_size(gs[0].log2ns, gs[1].log2ns, cfg->layout) : 0;
      if (cfg->cluster_size < 0) {
        csize = 0;
      } else if (cfg->cluster_size > 0) {
        int64_t t = 0, sm = 0;
        if (gs.size() == 2) cluster_geom(gs[0].log2ns, gs[1].log2ns, cfg->cluster_size, &t, &sm);
        if (t == 0)
          return bail(FFTGEN_ERR_GPUMAP, "no cluster kernel of size " + std::to_string(cfg->cluster_size) +
                                             " for n = " + std::to_string(cfg->n));
        csize = cfg->cluster_size;
      }
      if (csize > 0) {
        p->cluster_size = csize;
        if ((e = cluster_prepare(gs[0].log2ns, gs[1].log2ns, csize, &p->max_clusters)) != cudaSuccess)
          return bail(FFTGEN_ERR_GPUMAP, std::string("cluster kernel attributes: ") + cudaGetErrorString(e));
        p->use_cluster = p->max_clusters > 0;
      }
      p->scratch_bytes = p->use_cluster ? 0
                                        : (size_t)p->ex.scratch_buffers * (size_t)cfg->batch * (size_t)cfg->n *
                                              sizeof(float2);
      if (p->scratch_bytes > 0 && (e = cudaMalloc(&p->d_scratch, p->scratch_bytes)) != cudaSuccess)
        return bail(FFTGEN_ERR_NOMEM, "four-step scratch (" + std::to_string(p->scratch_bytes) +
                                          " bytes): " + cudaGetErrorString(e));
      if (p->use_cluster) {
        // data the TMA tiles cannot address (not 16-byte aligned) runs the
        // two-launch path in chunks through <= 64 MiB of plan-owned scratch
        const int64_t per_transform = p->ex.scratch_buffers * cfg->n * (int64_t)sizeof(float2);
        p->fallback_chunk = std::max<int64_t>(1, std::min<int64_t>(cfg->batch, (int64_t(64) << 20) / per_transform));
        p->fallback_bytes = (size_t)p->fallback_chunk * (size_t)per_transform;
        if ((e = cudaMalloc(&p->d_fallback, p->fallback_bytes)) != cudaSuccess)
          return bail(FFTGEN_ERR_NOMEM, "cluster fallback scratch: " + std::string(cudaGetErrorString(e)));
      }
    }
    const auto &tw = p->ex.tw_block;
    if (!tw.empty()) {
      if ((e = cudaMalloc(&p->d_tw, tw.size() * sizeof(float))) != cudaSuccess)
        return bail(FFTGEN_ERR_NOMEM, std::string("twiddle table: ") + cudaGetErrorString(e));
      if ((e = cudaMemcpyAsync(p->d_tw, tw.data(), tw.size() * sizeof(float), cudaMemcpyHostToDevice, ps)) !=
          cudaSuccess)
        return bail(FFTGEN_ERR_CUDA, std::string("twiddle upload: ") + cudaGetErrorString(e));
    }
    // the tables are complete before any stream can use the plan; only the
    // plan's own stream is waited on (no device-wide synchronisation)
    if ((e = cudaStreamSynchronize(ps)) != cudaSuccess)
      return bail(FFTGEN_ERR_CUDA, std::string("plan creation: ") + cudaGetErrorString(e));
    *out = p;
    return FFTGEN_OK;
  });
}

fftgen_status fftgen_plan_destroy(fftgen_plan *p) {
  if (!p) return FFTGEN_OK;
  {
    DeviceGuard g(p->cfg.device);
    if (p->d_tw) cudaFree(p->d_tw);
    if (p->d_twg) cudaFree(p->d_twg);
    if (p->d_scratch) cudaFree(p->d_scratch);
    if (p->d_fallback) cudaFree(p->d_fallback);
    if (p->d_stage) cudaFree(p->d_stage);
    for (auto &s : p->streams)
      if (s) cudaStreamDestroy(s);
  }
  delete p;
  return FFTGEN_OK;
}


fftgen_status fftgen_execute(const fftgen_plan *p, int direction, const void *in0, const void *in1,
                             void *out0, void *out1, int64_t dist, void *stream) {
  fftgen_status st = validate_exec(p, direction, in0, in1, out0, out1, dist);
  if (st != FFTGEN_OK) return st;
  NvtxRange range(p, "fftgen_execute");
  DeviceGuard g(p->cfg.device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  cudaError_t e = enqueue(p, direction, in0, in1, out0, out1, dist, p->cfg.batch, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return FFTGEN_OK;
}

fftgen_status fftgen_execute_host(const fftgen_plan *cp, int direction, const float *in0, const float *in1,
                                  float *out0, float *out1, int64_t dist) {
  fftgen_status st = validate_exec(cp, direction, in0, in1, out0, out1, dist);
  if (st != FFTGEN_OK) return st;
  auto *p = const_cast<fftgen_plan *>(cp);
  std::lock_guard<std::mutex> lk(p->mu);
  NvtxRange range(p, "fftgen_execute_host");
  DeviceGuard g(p->cfg.device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  const int64_t n = p->cfg.n;
  const bool split = p->cfg.layout == FFTGEN_LAYOUT_SPLIT;
  const size_t per = 2 * (size_t)n * elem_bytes(p);  // device in + out, packed (dist = n)
  return host_pipeline(p, per, [&](int64_t b0, int64_t cnt, char *slot, cudaStream_t s) {
    cudaError_t e;
    float *din = (float *)slot;
    float *dout = din + 2 * n * cnt;
    const size_t w = (split ? 1 : 2) * n * sizeof(float), hp = (split ? 1 : 2) * dist * sizeof(float);
    const float *h0 = in0 + b0 * dist * (split ? 1 : 2);
    if ((e = cudaMemcpy2DAsync(din, w, h0, hp, w, cnt, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
    float *din1 = nullptr, *dout1 = nullptr;
    if (split) {
      din1 = din + n * cnt;
      dout1 = dout + n * cnt;
      if ((e = cudaMemcpy2DAsync(din1, w, in1 + b0 * dist, hp, w, cnt, cudaMemcpyHostToDevice, s)) != cudaSuccess)
        return e;
    }
    if ((e = enqueue(p, direction, din, din1, dout, dout1, n, cnt, s)) != cudaSuccess) return e;
    float *ho0 = out0 + b0 * dist * (split ? 1 : 2);
    if ((e = cudaMemcpy2DAsync(ho0, hp, dout, w, w, cnt, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if (split && (e = cudaMemcpy2DAsync(out1 + b0 * dist, hp, dout1, w, w, cnt, cudaMemcpyDeviceToHost, s)) !=
                     cudaSuccess)
      return e;
    return cudaSuccess;
  });
}

fftgen_status fftgen_interpret_f64(const fftgen_plan *cp, int direction, const double *in, double *out) {
  if (!cp) return fail(FFTGEN_ERR_INVALID, "NULL plan");
  if (!in || !out) return fail(FFTGEN_ERR_EXEC, "NULL data pointer");
  if (direction != FFTGEN_FORWARD && direction != FFTGEN_INVERSE)
    return fail(FFTGEN_ERR_EXEC, "direction must be FFTGEN_FORWARD (-1) or FFTGEN_INVERSE (+1)");
  auto *p = const_cast<fftgen_plan *>(cp);
  std::lock_guard<std::mutex> lk(p->mu);
  DeviceGuard g(p->cfg.device);
  if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
  const int64_t n = p->cfg.n;
  const bool split = p->cfg.layout == FFTGEN_LAYOUT_SPLIT;
  // per transform: 2n doubles in, 2n floats in, 2n floats out, 2n doubles out
  const size_t per = 2 * (size_t)n * (8 + 4 + 4 + 8);
  return host_pipeline(p, per, [&](int64_t b0, int64_t cnt, char *slot, cudaStream_t s) {
    cudaError_t e;
    const int64_t cntf = 2 * n * cnt;
    double *d64in = (double *)slot;
    float *f32in = (float *)(d64in + cntf);
    float *f32out = f32in + cntf;
    double *d64out = (double *)(f32out + cntf);
    if ((e = cudaMemcpyAsync(d64in, in + b0 * 2 * n, cntf * sizeof(double), cudaMemcpyHostToDevice, s)) !=
        cudaSuccess)
      return e;
    if (p->ex.strategy == STRAT_IDENTITY)  // DFT_1: no arithmetic, so no fp32 rounding either
      return cudaMemcpyAsync(out + b0 * 2 * n, d64in, cntf * sizeof(double), cudaMemcpyDeviceToHost, s);
    if ((e = convert_f64_to_f32(d64in, f32in, cntf, s)) != cudaSuccess) return e;
    if (split)  // reference ComplexBuffer split storage: [re n | im n] per transform
      e = enqueue(p, direction, f32in, f32in + n, f32out, f32out + n, 2 * n, cnt, s);
    else
      e = enqueue(p, direction, f32in, nullptr, f32out, nullptr, n, cnt, s);
    if (e != cudaSuccess) return e;
    if ((e = convert_f32_to_f64(f32out, d64out, cntf, s)) != cudaSuccess) return e;
    return cudaMemcpyAsync(out + b0 * 2 * n, d64out, cntf * sizeof(double), cudaMemcpyDeviceToHost, s);
  });
}

// ---- introspection -------------------------------------------------------
int fftgen_plan_radices(const fftgen_plan *p, int64_t *radices, int cap) {
  if (!p) return -1;
  const int cnt = (int)p->radices.size();
  for (int i = 0; i < cnt && i < cap && radices; ++i) radices[i] = p->radices[i];
  return cnt;
}

int fftgen_plan_num_ops(const fftgen_plan *p) { return p ? (int)p->ops.size() : -1; }

fftgen_status fftgen_plan_op(const fftgen_plan *p, int idx, int64_t desc[4]) {
  if (!p || !desc) return fail(FFTGEN_ERR_INVALID, "NULL argument");
  if (idx < 0 || idx >= (int)p->ops.size()) return fail(FFTGEN_ERR_DIMENSION, "op index out of range");
  const RefOp &op = p->ops[idx];
  desc[0] = op.kind;
  desc[1] = op.kind == OP_TWIDDLE ? p->cfg.n : op.p0;
  desc[2] = op.kind == OP_TWIDDLE ? 0 : op.p1;
  desc[3] = op.kind == OP_TWIDDLE ? 0 : op.p2;
  return FFTGEN_OK;
}

fftgen_status fftgen_plan_op_map(const fftgen_plan *p, int idx, int64_t *map, int64_t *s_out) {
  if (!p || !map) return fail(FFTGEN_ERR_INVALID, "NULL argument");
  if (idx < 0 || idx >= (int)p->ops.size()) return fail(FFTGEN_ERR_DIMENSION, "op index out of range");
  return guarded([&]() -> fftgen_status {
    op_map(p->ops[idx], p->cfg.n, map, s_out);
    return FFTGEN_OK;
  });
}


fftgen_status fftgen_plan_pipeline_text(const fftgen_plan *p, char *buf, size_t cap) {
  if (!p) return fail(FFTGEN_ERR_INVALID, "NULL plan");
  return copy_text(pipeline_text(p->ops, p->cfg.n), buf, cap);
}

fftgen_status fftgen_program_text(const fftgen_config *cfg, int what, char *buf, size_t cap) {
  if (!cfg) return fail(FFTGEN_ERR_INVALID, "NULL config");
  std::string text;
  fftgen_status st = guarded([&]() -> fftgen_status {
    if (cfg->algorithm != FFTGEN_ALG_COOLEY_TUKEY && cfg->algorithm != FFTGEN_ALG_STOCKHAM)
      throw PlanError("unknown algorithm " + std::to_string(cfg->algorithm));
    const auto ops = fuse_ops(cfg->n, cfg->algorithm, cfg->radix);  // the plan_create validation order
    check_schedule(cfg->vec, cfg->vector_width, cfg->tile_kind, cfg->tile_value);
    switch (what) {
    case FFTGEN_TEXT_FORMULA: text = formula_text(cfg->n, cfg->algorithm, cfg->radix) + "\n"; break;
    case FFTGEN_TEXT_PIPELINE: text = pipeline_text(ops, cfg->n); break;
    case FFTGEN_TEXT_LOOPS:
      text = program_text(cfg->n,
                          (cfg->tuning & FFTGEN_TUNE_GROUPS_1024)
                              ? SPLIT_GROUPS_1024
                              : ((cfg->tuning & FFTGEN_TUNE_TWO_PASS) ? SPLIT_TWO_PASS : SPLIT_DEFAULT),
                          cfg->pass_radix, cfg->layout);
      break;
    case FFTGEN_TEXT_RADICES: {
      std::ostringstream o;
      for (int64_t r : stockham_radices(cfg->n, cfg->radix)) o << r << " ";
      text = o.str() + "\n";
      break;
    }
    default: throw DimensionError("unknown program text kind " + std::to_string(what));
    }
    return FFTGEN_OK;
  });
  return st != FFTGEN_OK ? st : copy_text(text, buf, cap);
}

int64_t fftgen_plan_group_twiddles(const fftgen_plan *p, int group, int which, float *out, int64_t cap) {
  if (!p || p->ex.strategy != STRAT_FOURSTEP || group < 0 || group >= (int)p->ex.groups.size() ||
      (which != 0 && which != 1) || cap < 0 || (cap > 0 && !out)) {
    fail(FFTGEN_ERR_INVALID, "bad plan, group or table");
    return -1;
  }
  const GroupDesc &d = p->ex.groups[group];
  if (d.cols <= 1) return 0;
  const int64_t count = which == 0 ? d.r0 * d.cols : (d.ns / d.r0) * d.cols;
  const int64_t m = std::min(count, cap);
  if (m > 0) {
    DeviceGuard g(p->cfg.device);
    const float2 *src = p->d_twg + (which == 0 ? d.q_off : d.p_off);
    if (cudaMemcpy(out, src, (size_t)m * sizeof(float2), cudaMemcpyDeviceToHost) != cudaSuccess) {
      fail(FFTGEN_ERR_CUDA, "twiddle table copy");
      return -1;
    }
  }
  return count;
}

int fftgen_plan_num_passes(const fftgen_plan *p) { return p ? (int)p->ex.passes.size() : -1; }

fftgen_status fftgen_plan_pass(const fftgen_plan *p, int idx, int64_t desc[4]) {
  if (!p || !desc) return fail(FFTGEN_ERR_INVALID, "NULL argument");
  if (idx < 0 || idx >= (int)p->ex.passes.size()) return fail(FFTGEN_ERR_DIMENSION, "pass index out of range");
  const PassDesc &d = p->ex.passes[idx];
  desc[0] = d.R;
  desc[1] = d.cols;
  desc[2] = d.k;
  desc[3] = d.s;
  return FFTGEN_OK;
}

int fftgen_plan_launches(const fftgen_plan *p) {
  if (!p) return -1;
  switch (p->ex.strategy) {
  case STRAT_IDENTITY: return p->cfg.layout == FFTGEN_LAYOUT_SPLIT ? 2 : 1;
  case STRAT_BLOCK: return 1;
  default: return p->use_cluster ? 1 : (int)p->ex.groups.size();
  }
}

size_t fftgen_plan_scratch_bytes(const fftgen_plan *p) { return p ? p->scratch_bytes + p->fallback_bytes : 0; }

fftgen_status fftgen_plan_describe(const fftgen_plan *p, char *buf, size_t cap) {
  if (!p) return fail(FFTGEN_ERR_INVALID, "NULL plan");
  std::ostringstream o;
  o << "n=" << p->cfg.n << " batch=" << p->cfg.batch
    << " layout=" << (p->cfg.layout == FFTGEN_LAYOUT_SPLIT ? "split" : "interleaved")
    << " device=" << p->cfg.device << "\n";
  o << "reference stages (radix " << p->cfg.radix << "):";
  for (auto r : p->radices) o << " " << r;
  o << "\n";
  if (p->ex.strategy == STRAT_BLOCK) {
    int64_t threads, tpb, smem;
    if (p->use_rows) {
      rows_geom(p->ex.log2n, p->cfg.layout, &threads, &smem);
      o << "kernel fft_rows_kernel<" << p->cfg.n << "> grid[" << (p->cfg.batch + threads - 1) / threads << "] block["
        << threads << "] smem=" << smem << "B transforms/CTA=" << threads
        << " (one transform per thread: DFT_" << p->cfg.n
        << " as one register codelet over the passes below; coalesced 16-byte row moves; direct kernel if"
           " unaligned)\n";
    } else if (p->use_tma && p->tma_grid > 0) {
      block_tma_geom(p->ex.log2n, &threads, &tpb, &smem);
      const int64_t groups = (p->cfg.batch + tpb - 1) / tpb;
      const bool single = block_tma1(p->ex.log2n);
      o << "kernel fft_block_tma" << (single ? "1" : "") << "_kernel<" << p->cfg.n << "> grid["
        << std::min<int64_t>(groups, p->tma_grid) << "] block[" << threads << "] smem=" << smem
        << "B transforms/group=" << tpb
        << (single ? " (persistent, cp.async.bulk single stage + plane exchange; direct kernel if unaligned)\n"
                   : " (persistent, cp.async.bulk double-buffered; direct kernel if unaligned)\n");
    } else {
      block_launch_geom(p->ex.log2n, &threads, &tpb, &smem, p->ex.block_cap);
      o << "kernel fft_block_kernel<" << p->cfg.n << "> grid[" << (p->cfg.batch + tpb - 1) / tpb << "] block["
        << threads << "] smem=" << smem << "B transforms/CTA=" << tpb;
      if (p->ex.block_cap) o << " (pass radix hint " << p->ex.block_cap << ")";
      o << "\n";
    }
    for (size_t i = 0; i < p->ex.passes.size(); ++i) {
      const auto &d = p->ex.passes[i];
      o << "  pass " << i << ": radix " << d.R << " s=" << d.s << " cols=" << d.cols << " k=" << d.k
        << (i == 0 ? " (HBM load)" : " (smem)") << (i + 1 == p->ex.passes.size() ? " (HBM store)" : "") << "\n";
    }
  } else if (p->ex.strategy == STRAT_FOURSTEP) {
    if (p->use_cluster) {
      int64_t threads, smem;
      const int64_t csize = p->cluster_size;
      cluster_geom(p->ex.groups[0].log2ns, p->ex.groups[1].log2ns, p->cluster_size, &threads, &smem);
      o << "cluster: 1 fft_cluster_kernel<" << p->ex.groups[0].ns << "," << p->ex.groups[1].ns << "," << csize
        << "> launch grid[" << p->cfg.batch * csize << "] cluster[" << csize << "] block[" << threads
        << "] smem=" << smem << "B co-resident clusters=" << p->max_clusters
        << " (persistent; one transform per cluster, intermediate in DSMEM, no scratch)\n";
    } else
      o << "four-step: " << p->ex.groups.size() << " fft_group_kernel launches, scratch " << p->scratch_bytes
        << " B\n";
    for (size_t i = 0; i < p->ex.groups.size(); ++i) {
      const GroupDesc &d = p->ex.groups[i];
      int64_t threads, tc, smem, r0;
      group_geom(d.log2ns, &threads, &tc, &smem, &r0);
      const bool tma = i < p->group_tma_grid.size() && p->group_tma_grid[i] > 0;
      const bool last = i + 1 == p->ex.groups.size(), split = p->cfg.layout == FFTGEN_LAYOUT_SPLIT;
      const int shape = last ? (split ? 3 : 2) : (i == 0 ? (split ? 1 : 0) : 4);
      const bool stores = tma && group_tma_stores(d.log2ns, shape);
      o << "  group " << i << ": "
        << (tma ? (group_plane(d.log2ns) ? "fft_group_plane_kernel<" : "fft_group_tma_kernel<") : "fft_group_kernel<")
        << d.ns
        << "> radix "
        << d.ns << " s=" << d.s
        << " cols=" << d.cols << " k=" << d.k << (d.rows ? " rows (transposed store)" : " columns")
        << " grid[" << p->cfg.batch * (d.cols * d.k / tc) << "] block[" << threads << "] smem=" << smem
        << "B tile=" << tc
        << (tma ? (group_plane(d.log2ns) ? " (persistent, TMA tensor tile + fp32 exchange plane, next tile fetched after pass 0; "
                                    "plain kernel if unaligned)"
                                  : " (persistent, TMA tensor tiles double-buffered; plain kernel if unaligned)")
                : "")
        << (stores ? " results by TMA tensor stores" : "") << "\n";
    }
  } else if (p->ex.strategy == STRAT_IDENTITY) {
    o << "identity copy\n";
  }
  return copy_text(o.str(), buf, cap);
}

}  // extern "C"

extern "C" fftgen_status fftgen_twiddle_multiply(int direction, void *data, int64_t rows, int64_t cols, int64_t ld,
                                                 int64_t row_offset, int64_t col_offset, int64_t n, void *stream) {
  if (direction != FFTGEN_FORWARD && direction != FFTGEN_INVERSE)
    return fail(FFTGEN_ERR_EXEC, "direction must be FFTGEN_FORWARD (-1) or FFTGEN_INVERSE (+1)");
  if (!data) return fail(FFTGEN_ERR_EXEC, "NULL data pointer");
  if (rows < 0 || cols < 0 || ld < cols || n < 1 || row_offset < 0 || col_offset < 0)
    return fail(FFTGEN_ERR_DIMENSION, "bad twiddle block geometry");
  cudaError_t e = twiddle_block((float2 *)data, rows, cols, ld, row_offset, col_offset, n, direction,
                                (cudaStream_t)stream);
  return e == cudaSuccess ? FFTGEN_OK : cuda_fail(e, "twiddle kernel");
}
