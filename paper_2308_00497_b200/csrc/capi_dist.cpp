// capi_dist.cpp -- C ABI of the distributed four-step (include/fftgen_b200.h,
// "distributed four-step"; device stages in dist.cu) and of the device-side
// seeded_input generator.
//
// A fftgen_dist_plan is one rank's share of an n-point transform over `world`
// ranks: the P-point butterfly's twiddle tables (rank-independent), the
// rank's offset a0 = rank * n / world^2 into the twiddle diagonal, and the
// single-GPU plan of the local n/world-point transform.  The exchanges are
// the caller's (NCCL grouped send/recv, torch all_to_all_single, or a device
// copy when several ranks are emulated on one GPU); fftgen_dist_execute runs
// the whole pipeline with an exchange callback.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "fftgen_b200.h"
#include "kernels.hpp"
#include "plan.hpp"

using namespace fftgen_b200;

struct fftgen_dist_plan {
  int64_t n = 0, m = 0, l1 = 0;
  int world = 1, rank = 0, device = 0, log2n = 0, h = 0;
  fftgen_plan *local = nullptr;
  float2 *d_tlo = nullptr, *d_thi = nullptr;
};

namespace {
// the message fftgen_last_error() returns (thread-local, kept by capi.cpp)
fftgen_status dfail(fftgen_status st, const std::string &msg) {
  set_last_error(msg);
  return st;
}
fftgen_status dcuda(cudaError_t e, const char *what) {
  return dfail(FFTGEN_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool is_pow2(int64_t v) { return v >= 1 && (v & (v - 1)) == 0; }
int ilog2(int64_t v) {
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

struct Guard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit Guard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// both buffers hold the rank's block of m elements, 16-byte aligned, disjoint
fftgen_status check_pair(const fftgen_dist_plan *p, const void *in, const void *out) {
  if (!p) return dfail(FFTGEN_ERR_INVALID, "NULL plan");
  if (!in || !out) return dfail(FFTGEN_ERR_EXEC, "NULL data pointer");
  if ((uintptr_t)in % 16 || (uintptr_t)out % 16)
    return dfail(FFTGEN_ERR_EXEC, "distributed buffers must be 16-byte aligned");
  const uintptr_t a = (uintptr_t)in, b = (uintptr_t)out, bytes = (uintptr_t)p->m * 8;
  if (a < b + bytes && b < a + bytes) return dfail(FFTGEN_ERR_EXEC, "distributed stages are out of place");
  return FFTGEN_OK;
}
}  // namespace

extern "C" {

fftgen_status fftgen_dist_plan_create(fftgen_dist_plan **out, int64_t n, int world, int rank, int device) {
  if (!out) return dfail(FFTGEN_ERR_INVALID, "NULL plan pointer");
  *out = nullptr;
  if (!is_pow2(n)) return dfail(FFTGEN_ERR_PLAN, "size must be a power of two, got " + std::to_string(n));
  if (!dist_world_supported(world))
    return dfail(FFTGEN_ERR_DIMENSION, "world size must be 1, 2, 4, 8 or 16, got " + std::to_string(world));
  if (rank < 0 || rank >= world)
    return dfail(FFTGEN_ERR_DIMENSION, "rank " + std::to_string(rank) + " outside world " + std::to_string(world));
  if (n < 2 * (int64_t)world * world)
    return dfail(FFTGEN_ERR_DIMENSION, "n must be at least 2 * world^2 = " + std::to_string(2 * world * world));
  if (n / world > (int64_t(1) << 30))
    return dfail(FFTGEN_ERR_PLAN, "the local transform n/world exceeds the single-GPU limit 2^30");
  auto *p = new fftgen_dist_plan();
  p->n = n;
  p->world = world;
  p->rank = rank;
  p->device = device;
  p->m = n / world;
  p->l1 = p->m / world;
  p->log2n = ilog2(n);
  p->h = (p->log2n + 1) / 2;
  fftgen_config c;
  fftgen_config_init(&c);
  c.n = p->m;
  c.algorithm = FFTGEN_ALG_STOCKHAM;
  c.radix = 4;
  c.layout = FFTGEN_LAYOUT_INTERLEAVED;
  c.device = device;
  c.batch = 1;
  fftgen_status st = fftgen_plan_create(&p->local, &c);
  if (st != FFTGEN_OK) {
    delete p;
    return st;
  }
  Guard g(device);
  cudaError_t e = g.err;
  const int64_t nlo = int64_t(1) << p->h, nhi = n >> p->h;
  cudaStream_t s = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&p->d_tlo, nlo * sizeof(float2));
  if (e == cudaSuccess) e = cudaMalloc(&p->d_thi, nhi * sizeof(float2));
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = dist_gen_tables(p->d_tlo, p->d_thi, p->log2n, p->h, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (s) cudaStreamDestroy(s);
  if (e != cudaSuccess) {
    fftgen_dist_plan_destroy(p);
    return dcuda(e, "distributed plan tables");
  }
  *out = p;
  return FFTGEN_OK;
}

fftgen_status fftgen_dist_plan_destroy(fftgen_dist_plan *p) {
  if (!p) return FFTGEN_OK;
  {
    Guard g(p->device);
    if (p->d_tlo) cudaFree(p->d_tlo);
    if (p->d_thi) cudaFree(p->d_thi);
  }
  fftgen_plan_destroy(p->local);
  delete p;
  return FFTGEN_OK;
}

fftgen_status fftgen_dist_butterfly(const fftgen_dist_plan *p, int direction, const void *recv, void *send,
                                    void *stream) {
  fftgen_status st = check_pair(p, recv, send);
  if (st != FFTGEN_OK) return st;
  if (direction != FFTGEN_FORWARD && direction != FFTGEN_INVERSE)
    return dfail(FFTGEN_ERR_EXEC, "direction must be FFTGEN_FORWARD (-1) or FFTGEN_INVERSE (+1)");
  Guard g(p->device);
  if (g.err != cudaSuccess) return dcuda(g.err, "cudaSetDevice");
  cudaError_t e = dist_butterfly(p->world, direction, (const float2 *)recv, (float2 *)send, p->l1,
                                 (int64_t)p->rank * p->l1, p->d_tlo, p->d_thi, p->h, p->log2n, (cudaStream_t)stream);
  return e == cudaSuccess ? FFTGEN_OK : dcuda(e, "distributed butterfly");
}

fftgen_status fftgen_dist_local(const fftgen_dist_plan *p, int direction, const void *in, void *out, void *stream) {
  fftgen_status st = check_pair(p, in, out);
  if (st != FFTGEN_OK) return st;
  return fftgen_execute(p->local, direction, in, nullptr, out, nullptr, p->m, stream);
}

fftgen_status fftgen_dist_unpack(const fftgen_dist_plan *p, const void *recv, void *out, void *stream) {
  fftgen_status st = check_pair(p, recv, out);
  if (st != FFTGEN_OK) return st;
  Guard g(p->device);
  if (g.err != cudaSuccess) return dcuda(g.err, "cudaSetDevice");
  cudaError_t e = dist_unpack(p->world, (const float2 *)recv, (float2 *)out, p->l1, (cudaStream_t)stream);
  return e == cudaSuccess ? FFTGEN_OK : dcuda(e, "distributed unpack");
}

// pointer tables of the P ranks' blocks, 16-byte aligned, disjoint from out
static fftgen_status check_peers(const fftgen_dist_plan *p, const void *const *peers, const char *what) {
  if (!p) return dfail(FFTGEN_ERR_INVALID, "NULL plan");
  if (!peers) return dfail(FFTGEN_ERR_EXEC, std::string("NULL ") + what + " pointer table");
  for (int r = 0; r < p->world; ++r) {
    if (!peers[r]) return dfail(FFTGEN_ERR_EXEC, std::string(what) + " block of rank " + std::to_string(r) + " is NULL");
    if ((uintptr_t)peers[r] % 16) return dfail(FFTGEN_ERR_EXEC, "distributed buffers must be 16-byte aligned");
  }
  return FFTGEN_OK;
}

fftgen_status fftgen_dist_butterfly_peers(const fftgen_dist_plan *p, int direction, const void *const *in_blocks,
                                          void *const *recv_blocks, void *stream) {
  fftgen_status st;
  if ((st = check_peers(p, in_blocks, "input")) != FFTGEN_OK ||
      (st = check_peers(p, (const void *const *)recv_blocks, "receive")) != FFTGEN_OK)
    return st;
  // every receive block is written while other ranks still read every input
  // block: the two sets must not share a byte
  const uintptr_t bytes = (uintptr_t)p->m * 8;
  for (int r = 0; r < p->world; ++r)
    for (int s = 0; s < p->world; ++s) {
      const uintptr_t a = (uintptr_t)in_blocks[r], b = (uintptr_t)recv_blocks[s];
      if (a < b + bytes && b < a + bytes)
        return dfail(FFTGEN_ERR_EXEC, "receive block of rank " + std::to_string(s) + " overlaps the input block of rank " +
                                          std::to_string(r));
    }
  if (direction != FFTGEN_FORWARD && direction != FFTGEN_INVERSE)
    return dfail(FFTGEN_ERR_EXEC, "direction must be FFTGEN_FORWARD (-1) or FFTGEN_INVERSE (+1)");
  Guard g(p->device);
  if (g.err != cudaSuccess) return dcuda(g.err, "cudaSetDevice");
  cudaError_t e = dist_butterfly_peers(p->world, direction, (const float2 *const *)in_blocks,
                                       (float2 *const *)recv_blocks, p->l1, (int64_t)p->rank * p->l1, p->d_tlo,
                                       p->d_thi, p->h, p->log2n, (cudaStream_t)stream);
  return e == cudaSuccess ? FFTGEN_OK : dcuda(e, "distributed peer butterfly");
}

fftgen_status fftgen_dist_unpack_peers(const fftgen_dist_plan *p, const void *const *z_blocks, void *out,
                                       void *stream) {
  fftgen_status st = check_peers(p, z_blocks, "local-result");
  if (st != FFTGEN_OK) return st;
  if (!out || (uintptr_t)out % 16) return dfail(FFTGEN_ERR_EXEC, "output block NULL or not 16-byte aligned");
  for (int r = 0; r < p->world; ++r) {
    const uintptr_t a = (uintptr_t)z_blocks[r], b = (uintptr_t)out, bytes = (uintptr_t)p->m * 8;
    if (a < b + bytes && b < a + bytes) return dfail(FFTGEN_ERR_EXEC, "distributed stages are out of place");
  }
  Guard g(p->device);
  if (g.err != cudaSuccess) return dcuda(g.err, "cudaSetDevice");
  cudaError_t e = dist_unpack_peers(p->world, (const float2 *const *)z_blocks, (float2 *)out, p->l1,
                                    (int64_t)p->rank * p->l1, (cudaStream_t)stream);
  return e == cudaSuccess ? FFTGEN_OK : dcuda(e, "distributed peer unpack");
}

fftgen_status fftgen_dist_execute(const fftgen_dist_plan *p, int direction, const void *in, void *out, void *w0,
                                  void *w1, fftgen_exchange_fn exchange, void *ctx, void *stream) {
  if (!p) return dfail(FFTGEN_ERR_INVALID, "NULL plan");
  if (!exchange) return dfail(FFTGEN_ERR_INVALID, "NULL exchange callback");
  fftgen_status st;
  if ((st = check_pair(p, in, w0)) != FFTGEN_OK || (st = check_pair(p, w0, w1)) != FFTGEN_OK ||
      (st = check_pair(p, w0, out)) != FFTGEN_OK || (st = check_pair(p, w1, out)) != FFTGEN_OK)
    return st;
  const size_t chunk = (size_t)p->l1 * 8;
  auto xchg = [&](const void *s, void *r) -> fftgen_status {
    const int rc = exchange(ctx, s, r, chunk, stream);
    return rc == 0 ? FFTGEN_OK : dfail(FFTGEN_ERR_EXEC, "exchange callback failed with " + std::to_string(rc));
  };
  if ((st = xchg(in, w0)) != FFTGEN_OK) return st;
  if ((st = fftgen_dist_butterfly(p, direction, w0, w1, stream)) != FFTGEN_OK) return st;
  if ((st = xchg(w1, w0)) != FFTGEN_OK) return st;
  if ((st = fftgen_dist_local(p, direction, w0, w1, stream)) != FFTGEN_OK) return st;
  if ((st = xchg(w1, w0)) != FFTGEN_OK) return st;
  return fftgen_dist_unpack(p, w0, out, stream);
}

fftgen_status fftgen_dist_execute_cyclic(const fftgen_dist_plan *p, int direction, const void *in, void *out,
                                         void *w0, void *w1, fftgen_exchange_fn exchange, void *ctx, void *stream) {
  (void)w1;
  if (!p) return dfail(FFTGEN_ERR_INVALID, "NULL plan");
  if (!exchange) return dfail(FFTGEN_ERR_INVALID, "NULL exchange callback");
  fftgen_status st;
  if ((st = check_pair(p, in, w0)) != FFTGEN_OK || (st = check_pair(p, w0, out)) != FFTGEN_OK ||
      (st = check_pair(p, in, out)) != FFTGEN_OK)
    return st;
  const size_t chunk = (size_t)p->l1 * 8;
  auto xchg = [&](const void *s, void *r) -> fftgen_status {
    const int rc = exchange(ctx, s, r, chunk, stream);
    return rc == 0 ? FFTGEN_OK : dfail(FFTGEN_ERR_EXEC, "exchange callback failed with " + std::to_string(rc));
  };
  // the butterfly writes `out` (free until the local plan), which the second
  // exchange moves back into w0 for the local plan
  if ((st = xchg(in, w0)) != FFTGEN_OK) return st;
  if ((st = fftgen_dist_butterfly(p, direction, w0, out, stream)) != FFTGEN_OK) return st;
  if ((st = xchg(out, w0)) != FFTGEN_OK) return st;
  return fftgen_dist_local(p, direction, w0, out, stream);
}

fftgen_status fftgen_seeded_input(int layout, int64_t n, int64_t batch, uint64_t seed0, void *out0, void *out1,
                                  int64_t dist, int device, void *stream) {
  const bool split = layout == FFTGEN_LAYOUT_SPLIT;
  if (layout != FFTGEN_LAYOUT_INTERLEAVED && !split)
    return dfail(FFTGEN_ERR_EXEC, "unknown complex layout " + std::to_string(layout));
  if (n < 1 || batch < 0 || dist < n) return dfail(FFTGEN_ERR_DIMENSION, "bad seeded_input geometry");
  if (!out0 || (split && !out1)) return dfail(FFTGEN_ERR_EXEC, "NULL data pointer");
  const uintptr_t al = split ? 4 : 8;
  if ((uintptr_t)out0 % al || (split && (uintptr_t)out1 % al))
    return dfail(FFTGEN_ERR_EXEC, "data pointer not aligned to its " + std::to_string(al) + "-byte element");
  Guard g(device);
  if (g.err != cudaSuccess) return dcuda(g.err, "cudaSetDevice");
  cudaError_t e = seeded_input(split, out0, out1, n, batch, seed0, dist, (cudaStream_t)stream);
  return e == cudaSuccess ? FFTGEN_OK : dcuda(e, "seeded_input kernel");
}

int64_t fftgen_dist_chunk_elems(const fftgen_dist_plan *p) { return p ? p->l1 : -1; }
int64_t fftgen_dist_block_elems(const fftgen_dist_plan *p) { return p ? p->m : -1; }
const fftgen_plan *fftgen_dist_local_plan(const fftgen_dist_plan *p) { return p ? p->local : nullptr; }

}  // extern "C"
