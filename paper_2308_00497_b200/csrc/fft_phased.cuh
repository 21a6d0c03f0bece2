// fft_phased.cuh -- K6: both groups of a 2-group four-step plan in one
// persistent cooperative launch, with the intermediate held in L2.
//
// The batch is cut into chunks of `chunk` transforms whose intermediate (one
// "slot", chunk * N * 8 bytes) stays in L2; pa.slots = 3 slots rotate.
// All tiles of the launch form one global sequence
//     G0(0) | G0(1) G1(0) | G0(2) G1(1) | ... | G1(last)
// (G0(c): the column tiles of group 0 for chunk c, user input -> slot c%3;
//  G1(c): the row tiles of group 1 for chunk c, slot c%3 -> user output),
// dealt round-robin to the resident CTAs, each of which walks its share in
// order.  Dependencies are counted per chunk (release / acquire at gpu scope):
//   G1(c) tiles need every G0(c) tile stored,
//   G0(c) tiles need every G1(c-3) tile read (same slot; three slots keep
//   that dependency a whole segment behind the two-item TMA prefetch),
// and always point to earlier items of the sequence, so the walk cannot
// deadlock (a CTA waits only for an item at the front of its own queue, after
// it has published everything before it).
// Tiles arrive by TMA tensor boxes into a double-buffered stage two items
// ahead (a not-yet-ready item is fetched when it reaches the front of the
// queue instead), like fft_group_tma_kernel.  The intermediate is written
// with st.global.cg (write-back into L2), read back by TMA and dropped with
// discard.global.L2, so its dirty lines are never written back: HBM sees the
// input read and the output write only -- 16 N bytes per transform, the
// single-pass roofline -- while each group keeps the K3 tile arithmetic
// (bitwise equal to the two-launch path).
#pragma once

#include <cstdint>

#include "fft_group_tma.cuh"

namespace fftgen_b200 {

template <int NS0, int NS1> struct PhasedGeom {
  static constexpr int MAXT =
      GroupGeom<NS0>::THREADS < GroupGeom<NS1>::THREADS ? GroupGeom<NS0>::THREADS : GroupGeom<NS1>::THREADS;
  using GG0 = GroupGeom<NS0, MAXT>;
  using GG1 = GroupGeom<NS1, MAXT>;
  static_assert(GG0::THREADS == GG1::THREADS, "both groups share the CTA shape");
  static constexpr int THREADS = GG0::THREADS;
  static constexpr int RAW0 = GG0::TC * NS0 * 8, RAW1 = GG1::TC * NS1 * 8;  // tile bytes
  static constexpr int amax(int a, int b) { return a > b ? a : b; }
  static constexpr int STAGE =
      (amax(amax(RAW0, GG0::TC * GG0::REG * 8), amax(RAW1, GG1::TC * GG1::REG * 8)) + 127) / 128 * 128;
  static constexpr int SMEM = 2 * STAGE + 64;
  static constexpr int MIN_BLOCKS = (228 * 1024) / (SMEM + 1024) > 0 ? (228 * 1024) / (SMEM + 1024) : 1;
  static constexpr int TILES0 = NS1 / GG0::TC;  // group 0: cols 1, k NS1
  static constexpr int TILES1 = NS0 / GG1::TC;  // group 1: cols NS0, k 1
};

FFTGEN_FI int ld_acquire_gpu_s32(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
FFTGEN_FI void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

struct StreamItem {
  int grp;        // 0 or 1
  int64_t c, bl;  // chunk, transform within the chunk
  int64_t tt;     // tile within the transform
};

// Segment c of the sequence holds G0(c) (c < nchunks) then G1(c - lag)
// (0 <= c - lag < nchunks).  P(c) = tiles before segment c, monotone, so the
// segment of item t is found by bisection.
template <class PG>
FFTGEN_FI int64_t stream_prefix(int64_t c, const PhasedArgs &pa, int64_t nchunks) {
  auto done_tf = [&](int64_t m) {  // transforms in the first m chunks
    m = m < 0 ? 0 : (m > nchunks ? nchunks : m);
    const int64_t v = m * pa.chunk;
    return v < pa.batch ? v : pa.batch;
  };
  return PG::TILES0 * done_tf(c) + PG::TILES1 * done_tf(c - pa.lag);
}

template <class PG>
FFTGEN_FI StreamItem stream_decode(int64_t t, const PhasedArgs &pa, int64_t nchunks) {
  int64_t lo = 0, hi = nchunks + pa.lag;  // P(lo) <= t < P(hi)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (stream_prefix<PG>(mid, pa, nchunks) <= t)
      lo = mid;
    else
      hi = mid;
  }
  const int64_t c = lo, r = t - stream_prefix<PG>(c, pa, nchunks);
  auto cnt = [&](int64_t k) { return k + 1 < nchunks ? pa.chunk : pa.batch - k * pa.chunk; };
  const int64_t n0 = c < nchunks ? cnt(c) * PG::TILES0 : 0;
  StreamItem it{};
  int64_t j;
  if (r < n0)
    it.grp = 0, it.c = c, j = r;
  else
    it.grp = 1, it.c = c - pa.lag, j = r - n0;
  const int64_t T = it.grp ? PG::TILES1 : PG::TILES0;
  it.bl = j / T;
  it.tt = j - it.bl * T;
  return it;
}

// G1(c) needs every G0(c) tile stored; G0(c) needs every G1(c - slots) tile
// read (the slot it overwrites)
template <class PG>
FFTGEN_FI bool stream_ready(const PhasedArgs &pa, const StreamItem &it, int64_t nchunks) {
  auto cnt = [&](int64_t c) { return c + 1 < nchunks ? pa.chunk : pa.batch - c * pa.chunk; };
  if (it.grp == 1) return ld_acquire_gpu_s32(pa.done + it.c) >= (int)(cnt(it.c) * PG::TILES0);
  if (it.c >= pa.slots)
    return ld_acquire_gpu_s32(pa.done + nchunks + it.c - pa.slots) >= (int)(cnt(it.c - pa.slots) * PG::TILES1);
  return true;
}

template <class PG, int NS0, int NS1, int LIN>
FFTGEN_FI void stream_issue(const PhasedArgs &pa, const StreamItem &it, char *stage, uint64_t *bar) {
  fence_proxy_async_global();  // generic writes of the producers -> async-proxy (TMA) reads
  if (it.grp == 0) {
    constexpr int TC = PG::GG0::TC, CH = NS0 < 256 ? NS0 : 256, W = LIN == LAYOUT_SPLIT ? 1 : 2;
    const int b = (int)(it.c * pa.chunk + it.bl), c0 = (int)(it.tt * TC);
    mbar_expect_tx(bar, (uint32_t)PG::RAW0);
#pragma unroll
    for (int q = 0; q < NS0 / CH; ++q) {
      tma_load_4d(stage + q * CH * TC * W * 4, pa.tmap0[0], c0 * W, q * CH, 0, b, bar);
      if constexpr (LIN == LAYOUT_SPLIT)
        tma_load_4d(stage + NS0 * TC * 4 + q * CH * TC * 4, pa.tmap0[1], c0, q * CH, 0, b, bar);
    }
  } else {
    constexpr int TC = PG::GG1::TC;
    mbar_expect_tx(bar, (uint32_t)PG::RAW1);
    tma_load_4d(stage, pa.tmap1, 0, 0, (int)(it.tt * TC), (int)((it.c % pa.slots) * pa.chunk + it.bl), bar);
  }
}

template <int NS0, int NS1, int LIN, int LOUT, int DIR>
__global__ void __launch_bounds__(PhasedGeom<NS0, NS1>::THREADS, PhasedGeom<NS0, NS1>::MIN_BLOCKS)
fft_phased_kernel(const __grid_constant__ PhasedArgs pa) {
  using PG = PhasedGeom<NS0, NS1>;
  constexpr int64_t N = (int64_t)NS0 * NS1;
  extern __shared__ float4 smem_f4[];
  char *smem = reinterpret_cast<char *>(smem_f4);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + 2 * PG::STAGE);
  // in the dynamic region: static shared memory would shift the TMA stages
  // off their 128-byte alignment
  int *issued = reinterpret_cast<int *>(bars + 2);
  const int tid = threadIdx.x;
  const int64_t nchunks = (pa.batch + pa.chunk - 1) / pa.chunk;
  const int64_t total = pa.batch * (PG::TILES0 + PG::TILES1), stride = gridDim.x;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < 2; ++s) {
      const int64_t t = blockIdx.x + s * stride;
      issued[s] = 0;
      if (t < total) {
        const StreamItem it = stream_decode<PG>(t, pa, nchunks);
        if (stream_ready<PG>(pa, it, nchunks)) {
          stream_issue<PG, NS0, NS1, LIN>(pa, it, smem + s * PG::STAGE, &bars[s]);
          issued[s] = 1;
        }
      }
    }
  }
  __syncthreads();

  int k = 0;
  for (int64_t t = blockIdx.x; t < total; t += stride, ++k) {
    const int s = k & 1;
    char *stage = smem + s * PG::STAGE;
    const StreamItem it = stream_decode<PG>(t, pa, nchunks);
    if (tid == 0 && !issued[s]) {  // front of the queue: everything before it is published
      while (!stream_ready<PG>(pa, it, nchunks)) __nanosleep(64);
      stream_issue<PG, NS0, NS1, LIN>(pa, it, stage, &bars[s]);
      issued[s] = 1;
    }
    mbar_wait(&bars[s], (k >> 1) & 1);
    if (it.grp == 0) {
      const int64_t c0 = it.tt * PG::GG0::TC;
      GroupArgs a = pa.g0;
      tile_from_stage<NS0, LIN, LAYOUT_L2, DIR, false, typename PG::GG0>(a, stage, (it.c % pa.slots) * pa.chunk * N + it.bl * N,
                                                                          0, c0);
    } else {
      // the TMA has read the slot's lines: drop them without write-back
      const int64_t m0 = it.tt * PG::GG1::TC;
      const char *lines = reinterpret_cast<const char *>(
          reinterpret_cast<const float2 *>(pa.g1.in0) + ((it.c % pa.slots) * pa.chunk + it.bl) * N + m0 * NS1);
      for (int l = tid; l < PG::RAW1 / 128; l += PG::THREADS)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(lines + l * 128) : "memory");
      tile_from_stage<NS1, LAYOUT_L2, LOUT, DIR, true, typename PG::GG1>(
          pa.g1, stage, (it.c * pa.chunk + it.bl) * pa.g1.odist, m0, 0);
    }
    __syncthreads();  // stage fully read, this tile's stores and discards issued
    if (tid == 0) {
      fence_proxy_async_global();
      __threadfence();
      atomicAdd(pa.done + (it.grp ? nchunks : 0) + it.c, 1);
      issued[s] = 0;
      const int64_t tn = t + 2 * stride;
      if (tn < total) {
        const StreamItem nx = stream_decode<PG>(tn, pa, nchunks);
        if (stream_ready<PG>(pa, nx, nchunks)) {
          stream_issue<PG, NS0, NS1, LIN>(pa, nx, stage, &bars[s]);
          issued[s] = 1;
        }
      }
    }
    __syncthreads();  // issued[] visible
  }
}


// ---- K6b: the same stream of tiles with the plain group tiles --------------
//
// Geometry of fft_group_kernel (32 KB tiles of 256 threads for NS <= 256, up to
// four CTAs per SM, loads straight to registers), and dependencies published
// once per CTA and group-chunk instead of once per tile: a CTA adds its tile
// count for (group, chunk) when its walk moves on to the next group-chunk,
// after one fence, and waits for the next group-chunk's dependency only after
// that -- so it never waits with an unpublished tile of its own, and the walk
// stays deadlock-free under the co-residency of the cooperative launch.
template <int NS0, int NS1> struct StreamGeom {
  using PG = PhasedGeom<NS0, NS1>;
  using GG0 = typename PG::GG0;
  using GG1 = typename PG::GG1;
  static constexpr int THREADS = PG::THREADS;
  static constexpr int SMEM = GG0::BYTES > GG1::BYTES ? GG0::BYTES : GG1::BYTES;
  static constexpr int MIN_BLOCKS = GG0::MIN_BLOCKS < GG1::MIN_BLOCKS ? GG0::MIN_BLOCKS : GG1::MIN_BLOCKS;
  static constexpr int TILES0 = PG::TILES0, TILES1 = PG::TILES1;
};

template <int NS0, int NS1, int LIN, int LOUT, int DIR>
__global__ void __launch_bounds__(StreamGeom<NS0, NS1>::THREADS, StreamGeom<NS0, NS1>::MIN_BLOCKS)
fft_stream_kernel(const __grid_constant__ PhasedArgs pa) {
  using SG = StreamGeom<NS0, NS1>;
  using PG = typename SG::PG;
  constexpr int64_t N = (int64_t)NS0 * NS1;
  extern __shared__ float4 smem_f4[];
  float2 *smem = reinterpret_cast<float2 *>(smem_f4);
  const int tid = threadIdx.x;
  const int64_t nchunks = (pa.batch + pa.chunk - 1) / pa.chunk;
  const int64_t total = pa.batch * (PG::TILES0 + PG::TILES1), stride = gridDim.x;
  int64_t cur = -1;  // current group-chunk key: grp * nchunks + c
  int mine = 0;      // tiles of `cur` done by this CTA
  auto publish = [&]() {
    __syncthreads();  // every thread's stores of `cur` precede the release
    if (tid == 0 && cur >= 0 && mine > 0) {
      __threadfence();
      atomicAdd(pa.done + cur, mine);
    }
    mine = 0;
  };
  for (int64_t t = blockIdx.x; t < total; t += stride) {
    const StreamItem it = stream_decode<PG>(t, pa, nchunks);
    const int64_t key = it.grp * nchunks + it.c;
    if (key != cur) {
      publish();
      cur = key;
      if (tid == 0)
        while (!stream_ready<PG>(pa, it, nchunks)) __nanosleep(64);
      __syncthreads();
    }
    if (it.grp == 0) {
      const int64_t ob = (it.c % pa.slots) * pa.chunk * N + it.bl * N;
      group_tile<NS0, LIN, LAYOUT_L2, DIR, false, typename SG::GG0>(pa.g0, (it.c * pa.chunk + it.bl) * pa.g0.idist,
                                                                    ob, it.tt, smem);
    } else {
      const int64_t ib = (it.c % pa.slots) * pa.chunk * N + it.bl * N;
      group_tile<NS1, LAYOUT_L2, LOUT, DIR, true, typename SG::GG1, 0, true>(
          pa.g1, ib, (it.c * pa.chunk + it.bl) * pa.g1.odist, it.tt, smem);
    }
    ++mine;
    __syncthreads();  // the next tile rewrites the exchange buffer
  }
  publish();
}
}  // namespace fftgen_b200
