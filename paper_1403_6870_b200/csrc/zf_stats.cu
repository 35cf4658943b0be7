// zf_stats.cu -- validation reductions (production mode checks) and the
// generate-and-reduce kernel (the reference's aggregate / bench loop,
// _kernels.py:306-393 and :703-922, fused with quality.py:92-106 sums).
//
// Determinism: the grid is a pure function of n (not of the device's
// occupancy), every lane folds its samples in a fixed order, and each block
// reduces its lanes with a fixed shuffle tree into one partial row of
// [x, x^2, x^3, x^4, x^5] sums; the host adds the rows with an exact (fsum)
// summation.  Integer counts are order-free.
#include <cuda_runtime.h>

#include <algorithm>

#include "zf_internal.h"
#include "zf_tile.cuh"

namespace zf {
namespace {

#ifndef ZF_STAT_BLOCKS
#define ZF_STAT_BLOCKS (148 * 8)
#endif
constexpr uint32_t kMaxStatBlocks = ZF_STAT_BLOCKS;
constexpr int kMaxBins = 4096;

// Block scratch; the histogram (nbins + 2 u32) follows it in dynamic shared
// memory only when enabled, so moment-only reductions keep full occupancy.
struct StatsShared {
  double thresh[8];
  double warp_sums[kWarps][5];
};
// the per-warp queues (and their 16-byte round scratch) follow it
static_assert(sizeof(StatsShared) % 16 == 0, "queue alignment");

template <bool EXTRA, bool MOMENTS>
__device__ void init_sink(StatsSinkT<EXTRA, MOMENTS>& k, StatsShared* sh, unsigned int* hist,
                          const zf_stats_cfg& cfg) {
  if (cfg.nbins)  // hist has nbins + 2 slots only when the histogram is enabled
    for (int i = threadIdx.x; i < cfg.nbins + 2; i += blockDim.x) hist[i] = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q)  // static indices: the param struct stays out of local memory
    if (threadIdx.x == q) sh->thresh[q] = cfg.thresh[q];
  k.hist = hist;
  k.lo = cfg.hist_lo;
  k.inv_w = cfg.nbins ? (double)cfg.nbins / (cfg.hist_hi - cfg.hist_lo) : 0.0;
  k.nbins = cfg.nbins;
  k.nthresh = cfg.nthresh;
  k.abs_t = cfg.abs_thresh != 0;
  k.t = sh->thresh;
  k.tmin = __longlong_as_double(0x7ff0000000000000ll);
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (q < cfg.nthresh) k.tmin = fmin(k.tmin, cfg.thresh[q]);
}

template <bool EXTRA, bool MOMENTS>
__device__ void flush_sink(const StatsSinkT<EXTRA, MOMENTS>& k, StatsShared* sh,
                           const unsigned int* hist,
                           const zf_stats_cfg& cfg, double* __restrict__ partials,
                           unsigned long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int q = 0; q < 5; ++q) {
    double v = k.s[q];
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0) sh->warp_sums[wid][q] = v;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (!EXTRA || q >= cfg.nthresh) break;
    unsigned long long v = k.thr[q];
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0 && v) atomicAdd(counts + cfg.nbins + 2 + q, v);
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double acc = 0.0;
    for (int w = 0; w < kWarps; ++w) acc += sh->warp_sums[w][threadIdx.x];
    partials[(uint64_t)blockIdx.x * 5 + threadIdx.x] = acc;
  }
  if (cfg.nbins)
    for (int i = threadIdx.x; i < cfg.nbins + 2; i += blockDim.x)
      if (hist[i]) atomicAdd(counts + i, (unsigned long long)hist[i]);
}

// Sum-only flush: lanes -> warps (shuffle tree) -> block row [sum, 0, 0, 0, 0].
__device__ void flush_sum(double v, StatsShared* sh, double* __restrict__ partials) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  if (lane == 0) sh->warp_sums[wid][0] = v;
  __syncthreads();
  if (threadIdx.x < 5) {
    double acc = 0.0;
    if (threadIdx.x == 0)
      for (int w = 0; w < kWarps; ++w) acc += sh->warp_sums[w][0];
    partials[(uint64_t)blockIdx.x * 5 + threadIdx.x] = acc;
  }
}

// Tail-only flush: threshold counts (atomics), zero partial rows.
__device__ void flush_tail(const TailSink& k, const zf_stats_cfg& cfg,
                           double* __restrict__ partials, unsigned long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q >= cfg.nthresh) break;
    unsigned long long v = k.thr[q];
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0 && v) atomicAdd(counts + cfg.nbins + 2 + q, v);
  }
  if (threadIdx.x < 5) partials[(uint64_t)blockIdx.x * 5 + threadIdx.x] = 0.0;
}

// MODE 0: the aggregate (moments == 1, no histogram, no thresholds);
// 1: moments x^1..x^5 only; 2: moments + histogram + threshold counts;
// 3: histogram / threshold counts without moments (moments == 0);
// 4: threshold counts above every fast-path value (see TailSink).
template <int DIST, int MODE>
__global__ void __launch_bounds__(kThreads)
    fill_stats_kernel(const DevTables* __restrict__ gt, uint64_t seed, uint64_t ctr_base,
                      uint64_t n, zf_stats_cfg cfg, double* __restrict__ partials,
                      unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kPacks = kPacksOf<DIST>;
  DevPack* sp = reinterpret_cast<DevPack*>(smem_raw);
  StatsShared* sh = reinterpret_cast<StatsShared*>(smem_raw + kPacks * sizeof(DevPack));
  uint32_t* queues = reinterpret_cast<uint32_t*>(sh + 1);
  uint32_t* queue = queues + (threadIdx.x >> 5) * kQueueWords;
  unsigned int* hist = queues + kWarps * kQueueWords;
  stage_block(sp, primary_pack<DIST>(gt), kPacks * (int)sizeof(DevPack));
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  const int lane = threadIdx.x & 31;
  LaneCounts lc;
  if constexpr (MODE == 0) {
    __syncthreads();
    SumSink sink;
    // the aggregate pairs tiles (the next grid-stride tile: +2-4.5 %)
    run_tiles<DIST, false, 3, SumSink, kTrad<DIST> ? 1 : 2>(sp[0], sp[kPacks - 1], seed, ctr_base, sink,
                                                     n, warp0, nwarps, queue, lane, lc);
    flush_sum(sink.s, sh, partials);
  } else if constexpr (MODE == 4) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (threadIdx.x == q) sh->thresh[q] = cfg.thresh[q];
    TailSink sink;
    sink.nthresh = cfg.nthresh;
    sink.abs_t = cfg.abs_thresh != 0;
    sink.t = sh->thresh;
    __syncthreads();
    run_tiles<DIST, false, 3>(sp[0], sp[kPacks - 1], seed, ctr_base, sink, n, warp0, nwarps,
                              queue, lane, lc);
    flush_tail(sink, cfg, partials, counts);
  } else {
    StatsSinkT<MODE == 2 || MODE == 3, MODE != 3> sink;
    init_sink(sink, sh, hist, cfg);
    __syncthreads();
    run_tiles<DIST, false, 3>(sp[0], sp[kPacks - 1], seed, ctr_base, sink, n, warp0, nwarps,
                              queue, lane, lc);
    __syncthreads();
    flush_sink(sink, sh, hist, cfg, partials, counts);
  }
}

// Buffer statistics: 16-byte loads, grid-stride over vector slots.
template <typename T, bool EXTRA>
__global__ void __launch_bounds__(kThreads)
    stats_kernel(const T* __restrict__ x, uint64_t n, zf_stats_cfg cfg,
                 double* __restrict__ partials, unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  StatsShared* sh = reinterpret_cast<StatsShared*>(smem_raw);
  unsigned int* hist = reinterpret_cast<unsigned int*>(sh + 1);
  StatsSinkT<EXTRA> sink;
  init_sink(sink, sh, hist, cfg);
  __syncthreads();
  using Vec = typename VecOf<T>::T;
  constexpr int V = VecOf<T>::V;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t head = std::min<uint64_t>(n, (16 - (reinterpret_cast<uintptr_t>(x) & 15)) % 16 / sizeof(T));
  if (tid < head) sink.add((double)x[tid]);
  const T* xa = x + head;
  const uint64_t nv = (n - head) / V;
  const Vec* xv = reinterpret_cast<const Vec*>(xa);
#pragma unroll 4
  for (uint64_t i = tid; i < nv; i += stride) {
    const Vec w = __ldcs(xv + i);
    const T* e = reinterpret_cast<const T*>(&w);
#pragma unroll
    for (int j = 0; j < V; ++j) sink.add((double)e[j]);
  }
  for (uint64_t i = head + nv * V + tid; i < n; i += stride) sink.add((double)x[i]);
  __syncthreads();
  flush_sink(sink, sh, hist, cfg, partials, counts);
}

int check_cfg(const zf_stats_cfg* cfg) {
  if (!cfg) return ZF_EINVAL;
  if (cfg->nbins < 0 || cfg->nbins > kMaxBins || cfg->nthresh < 0 || cfg->nthresh > 8)
    return ZF_EINVAL;
  if (cfg->nbins && !(cfg->hist_hi > cfg->hist_lo)) return ZF_EINVAL;
  if (cfg->moments < 0 || cfg->moments > 5) return ZF_EINVAL;
  return ZF_OK;
}

bool extra(const zf_stats_cfg* cfg) { return cfg->nbins != 0 || cfg->nthresh != 0; }
bool sum_only(const zf_stats_cfg* cfg) { return cfg->moments == 1 && !extra(cfg); }

// Every threshold at or above the largest fast-path magnitude of the
// (modified) table: fast x = u * sx[i + 1], i < lmax, |u| <= 2^64 (exp) or
// 2^63 (normal), so |x| <= max sx * 2^64 (2^63) exactly (power-of-two scale).
bool tail_only(const zf_tables* t, int dist, const zf_stats_cfg* cfg) {
  if (cfg->nbins != 0 || cfg->nthresh == 0 || t->kind != kKindModified) return false;
  if (dist != ZF_EXP && dist != ZF_NORMAL) return false;
  const DevPack& p = dist == ZF_EXP ? t->host.ex : t->host.hn;
  double m = 0.0;
  for (int i = 1; i <= p.lmax; ++i) m = std::max(m, p.sx[i]);
  const double fast_max = m * (dist == ZF_EXP ? 0x1p64 : 0x1p63);
  for (int q = 0; q < cfg->nthresh; ++q)
    if (!(cfg->thresh[q] >= fast_max)) return false;
  return true;
}

size_t hist_bytes(const zf_stats_cfg* cfg) {
  return cfg->nbins ? ((size_t)(cfg->nbins + 2) * sizeof(unsigned int) + 15) / 16 * 16 : 0;
}


template <int DIST>
int launch_fill_stats_dist(const zf_tables* t, uint64_t seed, uint64_t ctr_base, uint64_t n,
                           const zf_stats_cfg* cfg, double* partials, unsigned long long* counts,
                           cudaStream_t s) {
  constexpr int kPacks = kPacksOf<DIST>;
  const uint32_t grid = stats_blocks(n);
  const int mode = sum_only(cfg)                    ? 0
                   : cfg->moments != 0               ? (extra(cfg) ? 2 : 1)
                   : tail_only(t, DIST, cfg)         ? 4
                                                     : 3;
  const size_t smem = kPacks * sizeof(DevPack) + sizeof(StatsShared) +
                      (size_t)kWarps * kQueueWords * sizeof(uint32_t) + hist_bytes(cfg);
  auto kern = mode == 0   ? fill_stats_kernel<DIST, 0>
              : mode == 1 ? fill_stats_kernel<DIST, 1>
              : mode == 2 ? fill_stats_kernel<DIST, 2>
              : mode == 3 ? fill_stats_kernel<DIST, 3>
                          : fill_stats_kernel<DIST, 4>;
  ZF_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, kThreads, smem, s>>>(t->dev, seed, ctr_base, n, *cfg, partials, counts);
  return cuda_status(cudaGetLastError());
}

}  // namespace

uint32_t stats_blocks(uint64_t n) {
  const uint64_t want = (n + (uint64_t)kTile * kWarps - 1) / ((uint64_t)kTile * kWarps);
  return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(want, kMaxStatBlocks));
}

int launch_fill_stats(const zf_tables* t, int dist, uint64_t seed, uint64_t ctr_base, uint64_t n,
                      const zf_stats_cfg* cfg, double* partials, unsigned long long* counts,
                      cudaStream_t s) {
  ZF_TRY_STATUS(check_cfg(cfg));
  ZF_TRY_STATUS(check_kind(t, dist));
  if (dist == ZF_EXP)
    return launch_fill_stats_dist<ZF_EXP>(t, seed, ctr_base, n, cfg, partials, counts, s);
  if (dist == ZF_NORMAL)
    return launch_fill_stats_dist<ZF_NORMAL>(t, seed, ctr_base, n, cfg, partials, counts, s);
  if (dist == ZF_TRAD_EXP)
    return launch_fill_stats_dist<ZF_TRAD_EXP>(t, seed, ctr_base, n, cfg, partials, counts, s);
  if (dist == ZF_TRAD_NORMAL)
    return launch_fill_stats_dist<ZF_TRAD_NORMAL>(t, seed, ctr_base, n, cfg, partials, counts, s);
  return ZF_EDIST;
}

int launch_stats(int dtype, const void* x, uint64_t n, const zf_stats_cfg* cfg, double* partials,
                 unsigned long long* counts, cudaStream_t s) {
  ZF_TRY_STATUS(check_cfg(cfg));
  const uint32_t grid = stats_blocks(n);
  const size_t smem = sizeof(StatsShared) + hist_bytes(cfg);
  const bool ex = extra(cfg);
  if (dtype == ZF_F64)
    (ex ? stats_kernel<double, true> : stats_kernel<double, false>)<<<grid, kThreads, smem, s>>>(
        static_cast<const double*>(x), n, *cfg, partials, counts);
  else if (dtype == ZF_F32)
    (ex ? stats_kernel<float, true> : stats_kernel<float, false>)<<<grid, kThreads, smem, s>>>(
        static_cast<const float*>(x), n, *cfg, partials, counts);
  else
    return ZF_EDIST;
  return cuda_status(cudaGetLastError());
}

}  // namespace zf

#if defined(ZF_CHECKS) && ZF_CHECKS
// debug builds: the first failed ZF_CHECK of this file's kernels (0 = none); resets it
extern "C" unsigned int zf_debug_check_line_stats(void) {
  unsigned int v = 0, z = 0;
  cudaMemcpyFromSymbol(&v, zf::zf_check_line, sizeof v);
  cudaMemcpyToSymbol(zf::zf_check_line, &z, sizeof z);
  return v;
}
#endif
