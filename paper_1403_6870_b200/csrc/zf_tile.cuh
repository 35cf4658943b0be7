// zf_tile.cuh -- the production warp tile, shared by the fill, batch and
// generate-and-reduce kernels.  A "sink" decides what happens to each value:
// StoreSink writes it to HBM (128-bit vector stores in pass 1), StatsSink folds
// it into per-lane moment sums / histogram / threshold counts without storing.
#pragma once
#include <cuda_runtime.h>

#include "zf_device.cuh"

namespace zf {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPerLane = 16;
constexpr int kTile = 32 * kPerLane;  // samples per warp tile

template <typename OutT>
struct VecOf;
template <>
struct VecOf<double> {
  static constexpr int V = 2;
  using T = double2;
  __device__ static T make(const double* v) { return make_double2(v[0], v[1]); }
};
template <>
struct VecOf<float> {
  static constexpr int V = 4;
  using T = float4;
  __device__ static T make(const float* v) { return make_float4(v[0], v[1], v[2], v[3]); }
};

struct LaneCounts {
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
};

template <typename OutT, bool VEC>
struct StoreSink {
  using Out = OutT;
  static constexpr int V = VecOf<OutT>::V;
  OutT* __restrict__ out;
  // pass 1: V consecutive values at k (exceptional ones are placeholders,
  // overwritten in pass 2 while the line is still in L2)
  __device__ __forceinline__ void put_vec(uint64_t k, const OutT* v, uint32_t /*exc_bits*/) {
    if constexpr (VEC) {
      *reinterpret_cast<typename VecOf<OutT>::T*>(out + k) = VecOf<OutT>::make(v);
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) out[k + e] = v[e];
    }
  }
  __device__ __forceinline__ void put(uint64_t k, OutT v, bool /*exc*/) { out[k] = v; }
};

// Validation statistics: raw power sums x^1..x^5 (quality.py:92-106), an
// equal-width histogram with under/overflow bins and threshold counts.
struct StatsSink {
  using Out = double;
  static constexpr int V = 2;
  double s[5] = {0, 0, 0, 0, 0};
  unsigned long long thr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned int* hist;  // smem, nbins + 2
  double lo, inv_w;
  int nbins, nthresh;
  bool abs_t;
  const double* t;  // thresholds (smem)
  __device__ __forceinline__ void add(double x) {
    double p = x;
    s[0] += p;
    p *= x;
    s[1] += p;
    p *= x;
    s[2] += p;
    p *= x;
    s[3] += p;
    p *= x;
    s[4] += p;
    const double a = abs_t ? fabs(x) : x;
    for (int q = 0; q < nthresh; ++q) thr[q] += a > t[q];
    if (nbins) {
      const double f = (x - lo) * inv_w;
      int b = f < 0.0 ? -1 : (f >= (double)nbins ? nbins : (int)f);
      atomicAdd(hist + (b + 1), 1u);
    }
  }
  __device__ __forceinline__ void put_vec(uint64_t, const double* v, uint32_t exc_bits) {
#pragma unroll
    for (int e = 0; e < V; ++e)
      if (!((exc_bits >> e) & 1)) add(v[e]);
  }
  __device__ __forceinline__ void put(uint64_t, double v, bool exc) {
    if (!exc) add(v);
  }
};

// Pass 1 of one warp tile: samples [base, min(base + kTile, n)) of the
// counter stream (seed, ctr_base).  Every lane computes the fast-path value of
// its 16 samples and hands V of them at a time to the sink; returns the lane's
// mask of exceptional samples (bit it*V + e  <->  offset it*32*V + lane*V + e).
template <int DIST, bool COUNTED, class Sink>
__device__ __forceinline__ uint32_t fast_pass(const DevPack& P, uint64_t seed, uint64_t ctr_base,
                                              Sink& sink, uint64_t n, uint64_t base, int lane,
                                              LaneCounts& lc) {
  using OutT = typename Sink::Out;
  constexpr int V = Sink::V;
  constexpr int kIters = kPerLane / V;
  constexpr uint64_t kIterStride = (uint64_t)(32 * V) * kGamma;  // mod 2^64
  const uint32_t lmax = (uint32_t)P.lmax;
  const double* sx = P.sx;
  const uint64_t k_lane = base + (uint64_t)lane * V;
  const uint64_t st0 = seed + (ctr_base + k_lane + 1) * kGamma;
  uint32_t mask = 0;
  if (base + kTile <= n) {
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
      const uint64_t st = st0 + (uint64_t)it * kIterStride;
      OutT v[V];
      uint32_t bits = 0;
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const uint64_t u = mix13(st + (uint64_t)e * kGamma);
        bits |= (uint32_t)(((uint32_t)u & 0xFFu) >= lmax) << e;
        v[e] = to_out<OutT>(fast_value<DIST>(sx, u));
      }
      mask |= bits << (it * V);
      sink.put_vec(k_lane + (uint64_t)it * 32 * V, v, bits);
    }
    if (COUNTED) {
      const unsigned fast = kPerLane - __popc(mask);
      lc.c[0] += fast;
      lc.c[1] += fast;
    }
  } else {
    // ragged last tile: identical words, bounds-checked element stores
    unsigned valid = 0;
#pragma unroll
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const uint64_t k = k_lane + (uint64_t)it * 32 * V + e;
        if (k < n) {
          const uint64_t u = mix13(st0 + (uint64_t)it * kIterStride + (uint64_t)e * kGamma);
          const bool exc = ((uint32_t)u & 0xFFu) >= lmax;
          mask |= (uint32_t)exc << (it * V + e);
          sink.put(k, to_out<OutT>(fast_value<DIST>(sx, u)), exc);
          ++valid;
        }
      }
    }
    if (COUNTED) {
      const unsigned fast = valid - __popc(mask);
      lc.c[0] += fast;
      lc.c[1] += fast;
    }
  }
  return mask;
}

// Pass 2 body for one exceptional sample k: the full draw on its secondary
// counter stream, written through the sink.
template <int DIST, bool COUNTED, class Sink>
__device__ __forceinline__ void resolve_one(const DevPack& P, const DevPack& E, uint64_t seed,
                                            uint64_t ctr_base, Sink& sink, uint64_t k,
                                            LaneCounts& lc) {
  using OutT = typename Sink::Out;
  const uint64_t K = ctr_base + k;
  const uint64_t u = mix13(seed + (K + 1) * kGamma);
  CtrStream s{seed + (kExcBase + (K << kExcShift)) * kGamma};
  double v;
  if (COUNTED) {
    Count c;
    v = draw<DIST>(P, E, u, s, c);
#pragma unroll
    for (int q = 0; q < 6; ++q) lc.c[q] += c.c[q];
  } else {
    NoCount c;
    v = draw<DIST>(P, E, u, s, c);
  }
  sink.put(k, to_out<OutT>(v), false);
}

// Exclusive warp prefix of `mine`; returns it and sets *total (warp-uniform).
__device__ __forceinline__ int warp_excl_scan(int mine, int lane, int* total) {
  int incl = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  *total = __shfl_sync(0xffffffffu, incl, 31);
  return incl - mine;
}

template <int V>
__device__ __forceinline__ uint32_t mask_bit_offset(int b, int lane) {
  return (uint32_t)((b / V) * 32 * V + lane * V + (b % V));
}

// One warp tile with immediate pass 2 (used where consecutive tiles belong to
// different requests, i.e. the batch kernel).  queue: kTile u32 per warp.
template <int DIST, bool COUNTED, class Sink>
__device__ __forceinline__ void fill_tile(const DevPack& P, const DevPack& E, uint64_t seed,
                                          uint64_t ctr_base, Sink& sink, uint64_t n,
                                          uint64_t base, uint32_t* queue, int lane,
                                          LaneCounts& lc) {
  const uint32_t mask = fast_pass<DIST, COUNTED>(P, seed, ctr_base, sink, n, base, lane, lc);
  int total;
  int slot = warp_excl_scan(__popc(mask), lane, &total);
  if (total == 0) return;  // warp-uniform
  for (uint32_t m = mask; m; m &= m - 1)
    queue[slot++] = mask_bit_offset<Sink::V>(__ffs(m) - 1, lane);
  __syncwarp();
  for (int j = lane; j < total; j += 32)
    resolve_one<DIST, COUNTED>(P, E, seed, ctr_base, sink, base + queue[j], lc);
  __syncwarp();
}

// Queue capacity per warp for the cross-tile deferral: < 32 leftovers plus a
// full tile of exceptions always fit, so no overflow path is needed.
constexpr int kQueueCap = 32 + kTile;

// A warp's whole share of a fill: tiles first_tile, first_tile + stride, ...
// Exceptional samples are queued across tiles (entry = tile iteration << 9 |
// offset) and resolved only in full rounds of 32 -- one per lane -- so pass 2
// runs with every lane busy instead of once per tile with a few.
template <int DIST, bool COUNTED, class Sink>
__device__ __forceinline__ void run_tiles(const DevPack& P, const DevPack& E, uint64_t seed,
                                          uint64_t ctr_base, Sink& sink, uint64_t n,
                                          uint64_t first_tile, uint64_t stride, uint32_t* q,
                                          int lane, LaneCounts& lc) {
  static_assert(kTile == 512, "entry packing assumes 9 offset bits");
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  int qn = 0;  // warp-uniform queue length
  auto k_of = [&](uint32_t e) -> uint64_t {
    return (first_tile + (uint64_t)(e >> 9) * stride) * kTile + (e & 511u);
  };
  uint32_t iter = 0;
  for (uint64_t tile = first_tile; tile < ntiles; tile += stride, ++iter) {
    const uint32_t mask =
        fast_pass<DIST, COUNTED>(P, seed, ctr_base, sink, n, tile * kTile, lane, lc);
    int total;
    int slot = qn + warp_excl_scan(__popc(mask), lane, &total);
    if (total == 0) continue;
    for (uint32_t m = mask; m; m &= m - 1)
      q[slot++] = (iter << 9) | mask_bit_offset<Sink::V>(__ffs(m) - 1, lane);
    qn += total;
    __syncwarp();
    if (qn < 32) continue;
    int done = 0;
    for (; qn - done >= 32; done += 32)
      resolve_one<DIST, COUNTED>(P, E, seed, ctr_base, sink, k_of(q[done + lane]), lc);
    __syncwarp();
    for (int j = lane; j < qn - done; j += 32) q[j] = q[j + done];
    qn -= done;
    __syncwarp();
  }
  if (lane < qn) resolve_one<DIST, COUNTED>(P, E, seed, ctr_base, sink, k_of(q[lane]), lc);
  __syncwarp();
}

__device__ __forceinline__ void flush_counts(const LaneCounts& lc,
                                             unsigned long long* __restrict__ counters) {
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    unsigned long long v = lc.c[q];
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(counters + q, v);
  }
}

}  // namespace zf
