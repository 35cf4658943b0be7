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

// One warp tile: samples [base, min(base + kTile, n)) of the counter stream
// (seed, ctr_base); pass 1 = fast path for all, pass 2 = compacted exceptions.
template <int DIST, bool COUNTED, class Sink>
__device__ __forceinline__ void fill_tile(const DevPack& P, const DevPack& E, uint64_t seed,
                                          uint64_t ctr_base, Sink& sink, uint64_t n,
                                          uint64_t base, uint16_t* queue, int lane,
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

  // ---- pass 2: compact the exceptional samples of the whole warp ----------
  const int mine = __popc(mask);
  int incl = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (total == 0) return;  // warp-uniform
  int slot = incl - mine;
  for (uint32_t m = mask; m; m &= m - 1) {
    const int b = __ffs(m) - 1;
    queue[slot++] = (uint16_t)((b / V) * 32 * V + lane * V + (b % V));
  }
  __syncwarp();
  for (int j0 = 0; j0 < total; j0 += 32) {
    const int j = j0 + lane;
    if (j < total) {
      const uint64_t k = base + queue[j];
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
  }
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
