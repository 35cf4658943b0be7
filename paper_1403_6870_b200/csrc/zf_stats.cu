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

constexpr uint32_t kMaxStatBlocks = 148 * 8;
constexpr int kMaxBins = 4096;

struct StatsShared {
  double thresh[8];
  unsigned int hist[kMaxBins + 2];
  double warp_sums[kWarps][5];
};

__device__ void init_sink(StatsSink& k, StatsShared* sh, const zf_stats_cfg& cfg) {
  for (int i = threadIdx.x; i < cfg.nbins + 2; i += blockDim.x) sh->hist[i] = 0;
  if (threadIdx.x < 8) sh->thresh[threadIdx.x] = cfg.thresh[threadIdx.x];
  k.hist = sh->hist;
  k.lo = cfg.hist_lo;
  k.inv_w = cfg.nbins ? (double)cfg.nbins / (cfg.hist_hi - cfg.hist_lo) : 0.0;
  k.nbins = cfg.nbins;
  k.nthresh = cfg.nthresh;
  k.abs_t = cfg.abs_thresh != 0;
  k.t = sh->thresh;
}

__device__ void flush_sink(const StatsSink& k, StatsShared* sh, const zf_stats_cfg& cfg,
                           double* __restrict__ partials, unsigned long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int q = 0; q < 5; ++q) {
    double v = k.s[q];
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (lane == 0) sh->warp_sums[wid][q] = v;
  }
  for (int q = 0; q < cfg.nthresh; ++q) {
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
  for (int i = threadIdx.x; i < cfg.nbins + 2; i += blockDim.x)
    if (sh->hist[i]) atomicAdd(counts + i, (unsigned long long)sh->hist[i]);
}

template <int DIST>
__global__ void __launch_bounds__(kThreads)
    fill_stats_kernel(const DevTables* __restrict__ gt, uint64_t seed, uint64_t ctr_base,
                      uint64_t n, zf_stats_cfg cfg, double* __restrict__ partials,
                      unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kPacks = DIST == ZF_NORMAL ? 2 : 1;
  DevPack* sp = reinterpret_cast<DevPack*>(smem_raw);
  StatsShared* sh = reinterpret_cast<StatsShared*>(smem_raw + kPacks * sizeof(DevPack));
  uint32_t* queue = reinterpret_cast<uint32_t*>(sh + 1) + (threadIdx.x >> 5) * kQueueCap;
  stage_block(sp, DIST == ZF_NORMAL ? (const void*)&gt->hn : (const void*)&gt->ex,
              kPacks * (int)sizeof(DevPack));
  StatsSink sink;
  init_sink(sink, sh, cfg);
  __syncthreads();
  LaneCounts lc;
  const int lane = threadIdx.x & 31;
  run_tiles<DIST, false, 3>(sp[0], sp[kPacks - 1], seed, ctr_base, sink, n,
                         (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5),
                         (uint64_t)gridDim.x * kWarps, queue, lane, lc);
  __syncthreads();
  flush_sink(sink, sh, cfg, partials, counts);
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    stats_kernel(const T* __restrict__ x, uint64_t n, zf_stats_cfg cfg,
                 double* __restrict__ partials, unsigned long long* __restrict__ counts) {
  __shared__ StatsShared sh;
  StatsSink sink;
  init_sink(sink, &sh, cfg);
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    sink.add((double)x[i]);
  __syncthreads();
  flush_sink(sink, &sh, cfg, partials, counts);
}

int check_cfg(const zf_stats_cfg* cfg) {
  if (!cfg) return ZF_EINVAL;
  if (cfg->nbins < 0 || cfg->nbins > kMaxBins || cfg->nthresh < 0 || cfg->nthresh > 8)
    return ZF_EINVAL;
  if (cfg->nbins && !(cfg->hist_hi > cfg->hist_lo)) return ZF_EINVAL;
  return ZF_OK;
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
  const uint32_t grid = stats_blocks(n);
  const size_t queue = (size_t)kWarps * kQueueCap * sizeof(uint32_t);
  if (dist == ZF_EXP) {
    const size_t smem = sizeof(DevPack) + sizeof(StatsShared) + queue;
    ZF_TRY(cudaFuncSetAttribute(fill_stats_kernel<ZF_EXP>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fill_stats_kernel<ZF_EXP><<<grid, kThreads, smem, s>>>(t->dev, seed, ctr_base, n, *cfg,
                                                           partials, counts);
  } else if (dist == ZF_NORMAL) {
    const size_t smem = 2 * sizeof(DevPack) + sizeof(StatsShared) + queue;
    ZF_TRY(cudaFuncSetAttribute(fill_stats_kernel<ZF_NORMAL>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fill_stats_kernel<ZF_NORMAL><<<grid, kThreads, smem, s>>>(t->dev, seed, ctr_base, n, *cfg,
                                                              partials, counts);
  } else {
    return ZF_EDIST;
  }
  return cuda_status(cudaGetLastError());
}

int launch_stats(int dtype, const void* x, uint64_t n, const zf_stats_cfg* cfg, double* partials,
                 unsigned long long* counts, cudaStream_t s) {
  ZF_TRY_STATUS(check_cfg(cfg));
  const uint32_t grid = stats_blocks(n);
  if (dtype == ZF_F64)
    stats_kernel<double><<<grid, kThreads, 0, s>>>(static_cast<const double*>(x), n, *cfg,
                                                   partials, counts);
  else if (dtype == ZF_F32)
    stats_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<const float*>(x), n, *cfg, partials,
                                                  counts);
  else
    return ZF_EDIST;
  return cuda_status(cudaGetLastError());
}

}  // namespace zf
