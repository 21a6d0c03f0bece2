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
  } catch (const std::bad_alloc &) {
    return fail(FFTGEN_ERR_NOMEM, "host allocation failed");
  } catch (const std::exception &e) {
    return fail(FFTGEN_ERR_EXEC, e.what());
  }
}
}  // namespace

struct fftgen_plan {
  fftgen_config cfg{};
  ExecPlan ex;
  std::vector<int64_t> radices;
  std::vector<RefOp> ops;
  float2 *d_tw = nullptr;
  // K3 four-step: device-generated group twiddles and intermediate buffers
  float2 *d_twg = nullptr;
  float2 *d_tws = nullptr;  // K7: 2^14 block-plan tables, then w_N^e for e < N
  float2 *d_scratch = nullptr;
  float2 *d_fallback = nullptr;  // full-batch scratch of cluster / phased plans, on first unaligned execute
  size_t scratch_bytes = 0;
  // K5: 2-group plans run as one cluster per transform (DSMEM intermediate)
  // K3 groups: persistent TMA variant (resident CTAs per group, 0 = off)
  std::vector<int> group_tma_grid;
  bool use_cluster = false;
  bool use_split = false;  // K7 split-cluster kernel (fft_split.cuh)
  int split_clusters = 0;
  int64_t split_twn_off = 0;  // float2 offset of the w_N table in d_tws
  // K6: 2-group plans in one cooperative launch, intermediate in two L2 slots
  bool use_phased = false;
  int phased_grid = 0, phased_variant = 0;
  int64_t phased_lag = 1, phased_slots = 3;
  int64_t phased_chunk = 0;
  int *d_done = nullptr;  // per-chunk completed tiles of group 0 and group 1
  int max_clusters = 0, cluster_size = 0;
  std::mutex scratch_mu;  // lazy two-launch scratch of cluster plans (unaligned data)
  // L2-resident chunked execution of 2-group plans (0 = off)
  int64_t chunk = 0;
  cudaStream_t xs[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_a[2] = {nullptr, nullptr}, ev_b[2] = {nullptr, nullptr},
              ev_join[2] = {nullptr, nullptr};
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
  bool tma1_plane_ex1 = false;  // FFTGEN_TMA1_EX1=0
};

NvtxRange::NvtxRange(const fftgen_plan *p, const char *what) {
  char msg[96];
  std::snprintf(msg, sizeof msg, "%s n=%lld batch=%lld", what, (long long)p->cfg.n, (long long)p->cfg.batch);
  nvtxRangePushA(msg);
}

namespace {

fftgen_status validate_exec(const fftgen_plan *p, int direction, const void *in0, const void *in1,
                            const void *out0, const void *out1, int64_t dist) {
  if (!p) return fail(FFTGEN_ERR_INVALID, "NULL plan");
  if (direction != FFTGEN_FORWARD && direction != FFTGEN_INVERSE)
    return fail(FFTGEN_ERR_EXEC, "direction must be FFTGEN_FORWARD (-1) or FFTGEN_INVERSE (+1)");
  if (!in0 || !out0) return fail(FFTGEN_ERR_EXEC, "NULL data pointer");
  if (p->cfg.layout == FFTGEN_LAYOUT_SPLIT && (!in1 || !out1))
    return fail(FFTGEN_ERR_EXEC, "split layout needs both re (in0/out0) and im (in1/out1) pointers");
  if (dist < p->cfg.n)
    return fail(FFTGEN_ERR_DIMENSION, "dist " + std::to_string(dist) + " is smaller than n " +
                                          std::to_string(p->cfg.n));
  // element alignment: float2 for interleaved, float for split
  const uintptr_t al = p->cfg.layout == FFTGEN_LAYOUT_SPLIT ? 4 : 8;
  for (const void *q : {in0, in1, out0, out1})
    if (q && (uintptr_t)q % al != 0)
      return fail(FFTGEN_ERR_EXEC, "data pointer not aligned to its " + std::to_string(al) + "-byte element");
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
    if (p->use_tma && p->tma_grid > 0 && aligned) {
      const int64_t tp = block_tma_transforms_per_cta(p->ex.log2n);
      const int64_t groups = (batch + tp - 1) / tp;
      const int grid = (int)std::min<int64_t>(groups, p->tma_grid);
      return block_tma_launch(p->ex.log2n, layout, direction, a, grid,
                              (p->use_tma_store && out_aligned ? BLOCK_TMA_STORE : 0) |
                                  (p->tma1_plane_ex1 ? BLOCK_TMA1_PLANE_EX1 : 0),
                              s);
    }
    return block_launch(p->ex.log2n, layout, direction, a, s);
  }
  case STRAT_FOURSTEP: {
    const auto &gs = p->ex.groups;
    const bool split = layout == FFTGEN_LAYOUT_SPLIT;
    const int64_t esz = split ? 4 : 8;
    const bool rows_aligned = ((uintptr_t)in0 % 16 == 0) && (!in1 || (uintptr_t)in1 % 16 == 0) &&
                              (dist * esz) % 16 == 0;
    if (p->use_split && rows_aligned) {
      // radix-C DIF step across a C-CTA cluster + one 2^14-point transform per CTA
      SplitArgs sa{};
      sa.in0 = in0;
      sa.in1 = in1;
      sa.out0 = out0;
      sa.out1 = out1;
      sa.idist = dist;
      sa.odist = dist;
      sa.batch = batch;
      sa.tw = p->d_tws;
      sa.tw_n = p->d_tws + p->split_twn_off;
      return split_launch(p->ex.log2n, layout, direction, sa, p->split_clusters, s);
    }
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
    if (p->use_phased) {
      // one cooperative launch; chunks stream through two L2-resident slots
      PhasedArgs pa{};
      pa.g0 = make_group_args(p, 0, in0, in1, p->d_scratch, nullptr, dist, n);
      pa.g1 = make_group_args(p, 1, p->d_scratch, nullptr, out0, out1, n, dist);
      pa.batch = batch;
      pa.chunk = std::min<int64_t>(p->phased_chunk, batch);
      pa.done = p->d_done;
      pa.variant = p->phased_variant;
      pa.lag = p->phased_lag;
      pa.slots = p->phased_slots;
      int64_t threads, smem, t0, t1;
      phased_geom(gs[0].log2ns, gs[1].log2ns, p->phased_variant, &threads, &smem, &t0, &t1);
      const int64_t nchunks = (batch + pa.chunk - 1) / pa.chunk;
      if (p->phased_variant == 2 ||
          (encode_tile_maps(pa.g0, gs[0].log2ns, split ? 1 : 0, batch, gs[1].ns / t0, pa.tmap0) &&
           encode_tile_maps(pa.g1, gs[1].log2ns, 2, p->phased_slots * pa.chunk, gs[0].ns / t1,
                            reinterpret_cast<unsigned char(*)[128]>(pa.tmap1)))) {
        cudaError_t e = cudaMemsetAsync(p->d_done, 0, 2 * nchunks * sizeof(int), s);
        if (e != cudaSuccess) return e;
        const int grid = (int)std::min<int64_t>(p->phased_grid, batch * (t0 + t1));
        return phased_launch(gs[0].log2ns, gs[1].log2ns, layout, direction, pa, grid, s);
      }
    }
    if (gs.size() == 2 && p->chunk > 0 && batch >= 2 * p->chunk) {
      // L2-resident chunking: group 0 of chunk c on xs[0], group 1 on xs[1];
      // the intermediate of a chunk (<= 2 slots live) is read back from L2.
      cudaError_t e;
      if ((e = cudaEventRecord(p->ev_fork, s)) != cudaSuccess) return e;
      for (auto &x : p->xs)
        if ((e = cudaStreamWaitEvent(x, p->ev_fork, 0)) != cudaSuccess) return e;
      const int64_t esz = split ? 1 : 2;  // floats per element of a user plane
      int64_t c = 0;
      for (int64_t b0 = 0; b0 < batch; b0 += p->chunk, ++c) {
        const int64_t cnt = std::min<int64_t>(p->chunk, batch - b0);
        const int slot = (int)(c & 1);
        float2 *buf = p->d_scratch + (size_t)slot * p->chunk * n;
        if (c >= 2 && (e = cudaStreamWaitEvent(p->xs[0], p->ev_b[slot], 0)) != cudaSuccess) return e;
        const float *i0 = (const float *)in0 + b0 * dist * esz;
        const float *i1 = in1 ? (const float *)in1 + b0 * dist : nullptr;
        if ((e = launch_group(p, 0, direction, i0, i1, buf, nullptr, dist, n, cnt, p->xs[0], true)) != cudaSuccess)
          return e;
        if ((e = cudaEventRecord(p->ev_a[slot], p->xs[0])) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(p->xs[1], p->ev_a[slot], 0)) != cudaSuccess) return e;
        float *o0 = (float *)out0 + b0 * dist * esz;
        float *o1 = out1 ? (float *)out1 + b0 * dist : nullptr;
        if ((e = launch_group(p, 1, direction, buf, nullptr, o0, o1, n, dist, cnt, p->xs[1], true)) != cudaSuccess)
          return e;
        if ((e = cudaEventRecord(p->ev_b[slot], p->xs[1])) != cudaSuccess) return e;
      }
      for (int i = 0; i < 2; ++i) {
        if ((e = cudaEventRecord(p->ev_join[i], p->xs[i])) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(s, p->ev_join[i], 0)) != cudaSuccess) return e;
      }
      return cudaSuccess;
    }
    float2 *scratch = p->d_scratch;
    if (p->use_cluster || p->use_phased || p->use_split) {
      // TMA tiles need 16-byte aligned rows: unaligned data takes the
      // two-launch path, whose full-batch scratch is allocated on first use
      auto *mp = const_cast<fftgen_plan *>(p);
      std::lock_guard<std::mutex> lk(mp->scratch_mu);
      const size_t need = (size_t)p->ex.scratch_buffers * (size_t)p->cfg.batch * (size_t)n * sizeof(float2);
      if (!mp->d_fallback) {
        cudaError_t e = cudaMalloc(&mp->d_fallback, need);
        if (e != cudaSuccess) return e;
      }
      scratch = mp->d_fallback;
    }
    // groups ping-pong through interleaved scratch: in -> S0 [-> S1 -> S0 ...] -> out
    const size_t per = (size_t)p->cfg.batch * (size_t)n;  // float2 per scratch buffer
    for (size_t g = 0; g < gs.size(); ++g) {
      const bool first = g == 0, last = g + 1 == gs.size();
      float2 *src = first ? nullptr : scratch + ((g - 1) % p->ex.scratch_buffers) * per;
      float2 *dst = last ? nullptr : scratch + (g % p->ex.scratch_buffers) * per;
      cudaError_t e = launch_group(p, (int)g, direction, first ? in0 : src, first ? in1 : nullptr,
                                   last ? out0 : dst, last ? out1 : nullptr, first ? dist : n, last ? dist : n,
                                   batch, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  default:
    return cudaErrorNotSupported;
  }
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
  // FFTGEN_HOST_CHUNK_MB / FFTGEN_HOST_RAMP override.
  int64_t target = int64_t(128) << 20;
  if (const char *env = std::getenv("FFTGEN_HOST_CHUNK_MB")) target = std::max<int64_t>(1, std::atoll(env)) << 20;
  int64_t chunk = std::max<int64_t>(1, target / (int64_t)slot_bytes_per_transform);
  chunk = std::min(chunk, batch);
  // ramp: the first chunks are 1/2^RAMP, 1/2^(RAMP-1), ... of a full chunk, so
  // the pipeline fills (H2D of chunk 0 alone) and drains sooner
  int ramp = 4;
  if (const char *env = std::getenv("FFTGEN_HOST_RAMP")) ramp = std::max(0, std::min(6, std::atoi(env)));
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
    // two-launch four-step plans share one scratch buffer: keep their chunks
    // stream-ordered (the K5 cluster path has no scratch)
    const int sid = (p->ex.strategy == STRAT_FOURSTEP && !p->use_cluster && !p->use_split) ? 0 : (i % K);
    if ((e = stage(b0, cnt, slot_ptr, p->streams[sid])) != cudaSuccess) return cuda_fail(e, "host pipeline");
  }
  for (auto &s : p->streams)
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  return FFTGEN_OK;
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
    // same validation order as compile_pipeline -> plan_* -> fuse
    auto ops = fuse_ops(cfg->n, cfg->algorithm, cfg->radix);
    auto radices = stockham_radices(cfg->n, cfg->radix);
    const char *c14 = std::getenv("FFTGEN_CLUSTER14");
    ExecPlan ex = build_exec_plan(cfg->n, c14 && c14[0] != '0');

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (cfg->device < 0 || cfg->device >= ndev)
      return fail(FFTGEN_ERR_CUDA, "device " + std::to_string(cfg->device) + " not present (" +
                                       std::to_string(ndev) + " visible)");
    DeviceGuard g(cfg->device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");

    auto *p = new fftgen_plan();
    p->cfg = *cfg;
    p->ex = std::move(ex);
    p->ops = std::move(ops);
    p->radices = std::move(radices);
    if (p->ex.strategy == STRAT_BLOCK) {
      int per_sm = 0, sms = 0;
      if ((e = block_prepare(p->ex.log2n, &per_sm)) != cudaSuccess ||
          (e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device)) != cudaSuccess) {
        delete p;
        return cuda_fail(e, "kernel attributes");
      }
      p->tma_grid = block_tma_enabled(p->ex.log2n) ? per_sm * sms : 0;
      if (const char *env = std::getenv("FFTGEN_DISABLE_TMA")) p->use_tma = env[0] == '0';
      if (const char *env = std::getenv("FFTGEN_DISABLE_TMA_STORE")) p->use_tma_store = env[0] == '0';
      if (const char *env = std::getenv("FFTGEN_TMA1_EX1")) p->tma1_plane_ex1 = env[0] == '0';
    }
    auto bail = [&](fftgen_status st, const std::string &msg) {
      fftgen_plan_destroy(p);
      return fail(st, msg);
    };
    if (p->ex.strategy == STRAT_FOURSTEP) {
      for (const GroupDesc &d : p->ex.groups)
        if ((e = group_prepare(d.log2ns)) != cudaSuccess)
          return bail(FFTGEN_ERR_CUDA, std::string("group kernel attributes: ") + cudaGetErrorString(e));
      // Persistent TMA group kernels where they measured faster (B200,
      // scripts/gpu_ab.sh, 32 KB tiles for NS <= 256): first-group columns at
      // NS >= 512, whose 64 KB tiles leave one CTA of 256 threads per SM without
      // a prefetch (2^18 split 0.40 vs 0.35, 2^20 0.35 vs 0.32 of the single-pass
      // roofline); the 4-CTA 32 KB plain tiles win below (2^16 split 0.43 vs
      // 0.41) and for rows.  FFTGEN_GROUP_TMA=0 / 1 forces none / all.
      const char *gt = std::getenv("FFTGEN_GROUP_TMA");
      const int force = gt ? (gt[0] == '0' ? 0 : 1) : -1;
      if (force != 0) {
        int sms = 0;
        if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device)) != cudaSuccess)
          return bail(FFTGEN_ERR_CUDA, "device attributes");
        for (size_t g = 0; g < p->ex.groups.size(); ++g) {
          const GroupDesc &d = p->ex.groups[g];
          const bool first = g == 0;
          const bool want = force == 1 || (!d.rows && first && d.log2ns >= 9);
          int bps = 0;
          if (want && (e = group_tma_prepare(d.log2ns, &bps)) != cudaSuccess)
            return bail(FFTGEN_ERR_CUDA, std::string("group TMA kernel attributes: ") + cudaGetErrorString(e));
          p->group_tma_grid.push_back(want ? bps * sms : 0);
        }
      }
      // K4: Q[A0][m] = w_s^{A0 (NS/R0) m}, P[c][m] = w_s^{c m}, generated on the device in fp64
      if (p->ex.tw_group_len > 0) {
        if ((e = cudaMalloc(&p->d_twg, p->ex.tw_group_len * sizeof(float2))) != cudaSuccess)
          return bail(FFTGEN_ERR_NOMEM, std::string("group twiddles: ") + cudaGetErrorString(e));
        for (const GroupDesc &d : p->ex.groups) {
          if (d.cols <= 1) continue;
          // P is [c][m] for column groups (lanes share m) and [m][c] for the
          // rows group (lanes walk c within a row: coalesced twiddle loads)
          if ((e = gen_twiddles(p->d_twg + d.q_off, d.r0, d.cols, d.ns / d.r0, d.s, 0)) != cudaSuccess ||
              (e = d.rows ? gen_twiddles(p->d_twg + d.p_off, d.cols, d.ns / d.r0, 1, d.s, 0)
                          : gen_twiddles(p->d_twg + d.p_off, d.ns / d.r0, d.cols, 1, d.s, 0)) != cudaSuccess)
            return bail(FFTGEN_ERR_CUDA, std::string("twiddle generation: ") + cudaGetErrorString(e));
        }
      }
      if (p->ex.groups.size() == 2) {
        // opt-in: chunk of intermediate per slot; two slots live in L2
        int64_t chunk_bytes = 0;
        if (const char *env = std::getenv("FFTGEN_L2_CHUNK_BYTES")) chunk_bytes = std::atoll(env);
        const int64_t per_tf = cfg->n * (int64_t)sizeof(float2);
        p->chunk = chunk_bytes > 0 ? std::max<int64_t>(1, chunk_bytes / per_tf) : 0;
        if (p->chunk > 0 && cfg->batch >= 2 * p->chunk) {
          for (auto &x : p->xs)
            if ((e = cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking)) != cudaSuccess)
              return bail(FFTGEN_ERR_CUDA, "stream creation");
          cudaEvent_t *evs[] = {&p->ev_fork, &p->ev_a[0], &p->ev_a[1], &p->ev_b[0], &p->ev_b[1],
                                &p->ev_join[0], &p->ev_join[1]};
          for (cudaEvent_t *ev : evs)
            if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess)
              return bail(FFTGEN_ERR_CUDA, "event creation");
        } else {
          p->chunk = 0;
        }
      }
      const auto &gs = p->ex.groups;
      const char *no_cluster = std::getenv("FFTGEN_DISABLE_CLUSTER");
      // K5 where measured faster than K3 (cluster_default_size); FFTGEN_CLUSTER_SIZE=C
      // forces any compiled (NS0, NS1, C) shape
      int csize = gs.size() == 2 ? cluster_default_size(gs[0].log2ns, gs[1].log2ns, cfg->layout) : 0;
      if (const char *env = std::getenv("FFTGEN_CLUSTER_SIZE"); env && gs.size() == 2) {
        int64_t t = 0, sm = 0;
        cluster_geom(gs[0].log2ns, gs[1].log2ns, std::atoi(env), &t, &sm);
        if (t > 0) csize = std::atoi(env);
      }
      if (csize > 0 && !(no_cluster && no_cluster[0] != '0')) {
        p->cluster_size = csize;
        if ((e = cluster_prepare(gs[0].log2ns, gs[1].log2ns, csize, &p->max_clusters)) != cudaSuccess)
          return bail(FFTGEN_ERR_CUDA, std::string("cluster kernel attributes: ") + cudaGetErrorString(e));
        p->use_cluster = p->max_clusters > 0;
      }
      // K7 split-cluster kernel (FFTGEN_SPLIT=1): 2^15 / 2^16 in one HBM pass
      const char *sp = std::getenv("FFTGEN_SPLIT");
      if (sp && sp[0] == '1' && split_supported(p->ex.log2n)) {
        if ((e = split_prepare(p->ex.log2n, &p->split_clusters)) != cudaSuccess)
          return bail(FFTGEN_ERR_CUDA, std::string("split kernel attributes: ") + cudaGetErrorString(e));
        if (p->split_clusters > 0) {
          std::vector<float> t = block_twiddles(14);
          p->split_twn_off = (int64_t)t.size() / 2;
          for (int64_t i = 0; i < cfg->n; ++i) {
            double re, im;
            unit_root(cfg->n, i, &re, &im);
            t.push_back(static_cast<float>(re));
            t.push_back(static_cast<float>(im));
          }
          if ((e = cudaMalloc(&p->d_tws, t.size() * sizeof(float))) != cudaSuccess)
            return bail(FFTGEN_ERR_NOMEM, std::string("split twiddles: ") + cudaGetErrorString(e));
          if ((e = cudaMemcpy(p->d_tws, t.data(), t.size() * sizeof(float), cudaMemcpyHostToDevice)) != cudaSuccess)
            return bail(FFTGEN_ERR_CUDA, std::string("split twiddle upload: ") + cudaGetErrorString(e));
          p->use_split = true;
          p->use_cluster = false;
        }
      }
      // K6 phased kernel (opt-in, FFTGEN_PHASED=1).  Measured on B200 it keeps
      // DRAM bytes at exactly 16 N per transform (the intermediate never leaves
      // L2), but runs below the two-launch K3 path: 2^16 0.29 vs 0.43, 2^18
      // 0.28 vs 0.41, 2^20 0.25 vs 0.35 of the single-pass roofline.  K3's
      // passes are bound by the per-tile processing rate of one 16-warp CTA per
      // SM (3.5 us per 64 KB tile at 2^16), not by HBM, so halving the HBM
      // bytes of a tile does not shorten it.
      const char *ph = std::getenv("FFTGEN_PHASED");
      if (gs.size() == 2 && !p->use_cluster && !p->use_split && phased_supported(gs[0].log2ns, gs[1].log2ns) && ph &&
          (ph[0] == '1' || ph[0] == '2')) {
        int bps = 0, sms = 0;
        p->phased_variant = ph[0] - '0';
        if ((e = phased_prepare(gs[0].log2ns, gs[1].log2ns, p->phased_variant, &bps)) != cudaSuccess ||
            (e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device)) != cudaSuccess)
          return bail(FFTGEN_ERR_CUDA, std::string("phased kernel attributes: ") + cudaGetErrorString(e));
        if (bps > 0) {
          int64_t slot_mb = 16;
          if (const char *env = std::getenv("FFTGEN_PHASE_SLOT_MB")) slot_mb = std::max<int64_t>(1, std::atoll(env));
          p->phased_chunk = std::min<int64_t>(cfg->batch, std::max<int64_t>(1, (slot_mb << 20) / (cfg->n * 8)));
          if (const char *env = std::getenv("FFTGEN_PHASE_LAG")) p->phased_lag = std::max<int64_t>(1, std::atoll(env));
          p->phased_slots = p->phased_lag + 2;
          p->phased_grid = bps * sms;
          p->use_phased = true;
          p->chunk = 0;
          const int64_t nchunks = (cfg->batch + p->phased_chunk - 1) / p->phased_chunk;
          if ((e = cudaMalloc(&p->d_done, 2 * nchunks * sizeof(int))) != cudaSuccess)
            return bail(FFTGEN_ERR_NOMEM, "chunk counters");
        }
      }
      p->scratch_bytes = (p->use_cluster || p->use_split) ? 0
                         : p->use_phased ? (size_t)p->phased_slots * (size_t)p->phased_chunk * (size_t)cfg->n * sizeof(float2)
                                         : (size_t)p->ex.scratch_buffers * (size_t)cfg->batch * (size_t)cfg->n *
                                           sizeof(float2);
      if (p->scratch_bytes > 0 && (e = cudaMalloc(&p->d_scratch, p->scratch_bytes)) != cudaSuccess)
        return bail(FFTGEN_ERR_NOMEM, "four-step scratch (" + std::to_string(p->scratch_bytes) +
                                          " bytes): " + cudaGetErrorString(e));
    }
    const auto &tw = p->ex.tw_block;
    if (!tw.empty()) {
      if ((e = cudaMalloc(&p->d_tw, tw.size() * sizeof(float))) != cudaSuccess)
        return bail(FFTGEN_ERR_NOMEM, std::string("twiddle table: ") + cudaGetErrorString(e));
      if ((e = cudaMemcpy(p->d_tw, tw.data(), tw.size() * sizeof(float), cudaMemcpyHostToDevice)) != cudaSuccess)
        return bail(FFTGEN_ERR_CUDA, std::string("twiddle upload: ") + cudaGetErrorString(e));
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess)
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
    if (p->d_tws) cudaFree(p->d_tws);
    if (p->d_scratch) cudaFree(p->d_scratch);
    if (p->d_done) cudaFree(p->d_done);
    if (p->d_fallback) cudaFree(p->d_fallback);
    for (auto &x : p->xs)
      if (x) cudaStreamDestroy(x);
    for (cudaEvent_t ev : {p->ev_fork, p->ev_a[0], p->ev_a[1], p->ev_b[0], p->ev_b[1], p->ev_join[0], p->ev_join[1]})
      if (ev) cudaEventDestroy(ev);
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
  default: return (p->use_cluster || p->use_phased || p->use_split) ? 1 : (int)p->ex.groups.size();
  }
}

size_t fftgen_plan_scratch_bytes(const fftgen_plan *p) { return p ? p->scratch_bytes : 0; }

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
    if (p->use_tma && p->tma_grid > 0) {
      block_tma_geom(p->ex.log2n, &threads, &tpb, &smem);
      const int64_t groups = (p->cfg.batch + tpb - 1) / tpb;
      const bool single = block_tma1(p->ex.log2n);
      o << "kernel fft_block_tma" << (single ? "1" : "") << "_kernel<" << p->cfg.n << "> grid["
        << std::min<int64_t>(groups, p->tma_grid) << "] block[" << threads << "] smem=" << smem
        << "B transforms/group=" << tpb
        << (single ? " (persistent, cp.async.bulk single stage + plane exchange; direct kernel if unaligned)\n"
                   : " (persistent, cp.async.bulk double-buffered; direct kernel if unaligned)\n");
    } else {
      block_launch_geom(p->ex.log2n, &threads, &tpb, &smem);
      o << "kernel fft_block_kernel<" << p->cfg.n << "> grid[" << (p->cfg.batch + tpb - 1) / tpb << "] block["
        << threads << "] smem=" << smem << "B transforms/CTA=" << tpb << "\n";
    }
    for (size_t i = 0; i < p->ex.passes.size(); ++i) {
      const auto &d = p->ex.passes[i];
      o << "  pass " << i << ": radix " << d.R << " s=" << d.s << " cols=" << d.cols << " k=" << d.k
        << (i == 0 ? " (HBM load)" : " (smem)") << (i + 1 == p->ex.passes.size() ? " (HBM store)" : "") << "\n";
    }
  } else if (p->ex.strategy == STRAT_FOURSTEP) {
    if (p->use_split) {
      int64_t threads, smem, csize;
      split_geom(p->ex.log2n, &threads, &smem, &csize);
      o << "split: 1 fft_split_kernel<" << csize << "> launch grid["
        << std::min<int64_t>(p->cfg.batch, p->split_clusters) * csize << "] cluster[" << csize << "] block["
        << threads << "] smem=" << smem << "B co-resident clusters=" << p->split_clusters
        << " (persistent; radix-" << csize << " DIF step through DSMEM, one 2^14-point transform per CTA, "
        << "stride-" << csize << " stores, no scratch; two-launch path if unaligned)\n";
    } else if (p->use_cluster) {
      int64_t threads, smem;
      const int64_t csize = p->cluster_size;
      cluster_geom(p->ex.groups[0].log2ns, p->ex.groups[1].log2ns, p->cluster_size, &threads, &smem);
      o << "cluster: 1 fft_cluster_kernel<" << p->ex.groups[0].ns << "," << p->ex.groups[1].ns << "," << csize
        << "> launch grid[" << p->cfg.batch * csize << "] cluster[" << csize << "] block[" << threads
        << "] smem=" << smem << "B co-resident clusters=" << p->max_clusters
        << " (persistent; one transform per cluster, intermediate in DSMEM, no scratch)\n";
    } else if (p->use_phased) {
      int64_t threads, smem, t0, t1;
      phased_geom(p->ex.groups[0].log2ns, p->ex.groups[1].log2ns, p->phased_variant, &threads, &smem, &t0, &t1);
      o << "phased: 1 " << (p->phased_variant == 2 ? "fft_stream_kernel<" : "fft_phased_kernel<") << p->ex.groups[0].ns << "," << p->ex.groups[1].ns
        << "> cooperative launch grid[" << p->phased_grid << "] block[" << threads << "] smem=" << smem
        << "B chunk=" << p->phased_chunk << " transforms, lag " << p->phased_lag << ", " << p->phased_slots
        << " L2 slots = " << p->scratch_bytes
        << " B (both groups streamed through L2 with per-chunk dependencies, TMA tiles, intermediate "
           "discarded after use)\n";
    } else
      o << "four-step: " << p->ex.groups.size() << " fft_group_kernel launches, scratch " << p->scratch_bytes
        << " B\n";
    for (size_t i = 0; i < p->ex.groups.size(); ++i) {
      const GroupDesc &d = p->ex.groups[i];
      int64_t threads, tc, smem, r0;
      group_geom(d.log2ns, &threads, &tc, &smem, &r0);
      const bool tma = i < p->group_tma_grid.size() && p->group_tma_grid[i] > 0;
      o << "  group " << i << ": " << (tma ? "fft_group_tma_kernel<" : "fft_group_kernel<") << d.ns << "> radix "
        << d.ns << " s=" << d.s
        << " cols=" << d.cols << " k=" << d.k << (d.rows ? " rows (transposed store)" : " columns")
        << " grid[" << p->cfg.batch * (d.cols * d.k / tc) << "] block[" << threads << "] smem=" << smem
        << "B tile=" << tc
        << (tma ? " (persistent, TMA tensor tiles double-buffered; plain kernel if unaligned)" : "") << "\n";
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
