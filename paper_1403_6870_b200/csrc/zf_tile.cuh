// zf_tile.cuh -- the production warp tile, shared by the fill, batch and
// generate-and-reduce kernels.
//
// A warp walks "tiles" of kTile consecutive samples (kPerLane per lane).
//   pass 1  every lane computes the fast-path value of its samples (one
//           counter-stream word, LDS.64, I2F, DMUL) and hands V of them at a time
//           to the sink; exceptional samples (byte >= L_max, ~1.2-1.6 %) only
//           set a bit in the lane's mask.
//   pass 2  the warp compacts the masked samples into a per-warp smem queue
//           that persists across tiles and resolves them in full rounds of 32
//           (one sample per lane) once 32 are queued.  Callers may run pass 1
//           on 2 (or 4) tiles before one round of this bookkeeping
//           (run_tiles<..., NT>: the lane masks side by side in one mask).
// A "sink" decides what happens to each value: StoreSink writes it to HBM
// (128-bit vector stores in pass 1, 8-byte patches in pass 2 to lines that are
// still L2-resident), StatsSink folds it into moment sums / histogram /
// threshold counts without storing anything.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "zf_device.cuh"

namespace zf {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
// CTA size of the production fill kernel (a warp count that is not a power of
// two lets more 84-88-register warps fit on an SM)
#ifndef ZF_FILL_THREADS
#define ZF_FILL_THREADS 256
#endif
constexpr int kFillThreads = ZF_FILL_THREADS;
constexpr int kFillWarps = kFillThreads / 32;
#ifndef ZF_PER_LANE
#define ZF_PER_LANE 16
#endif
constexpr int kPerLane = ZF_PER_LANE;  // samples per lane per tile (<= 32: mask bits)
constexpr int kTile = 32 * kPerLane;   // samples per warp tile
constexpr int kTileBits = kTile == 512 ? 9 : kTile == 1024 ? 10 : 8;
constexpr int kPerLaneBits = kTileBits - 5;
static_assert((1 << kTileBits) == kTile, "tile must be 256, 512 or 1024 samples");
#ifndef ZF_PASS1_UNROLL
#define ZF_PASS1_UNROLL 8
#endif
constexpr int kPass1Unroll = ZF_PASS1_UNROLL;

// Rounds compute the alias-pick and first-attempt words side by side.
#ifndef ZF_HOIST
#define ZF_HOIST 1
#endif
// Tables staged by two bulk copies: pass 1 waits only for the scale array.
// Normal rounds: each lane's first two box attempts side by side before the
// cooperative iterations (+1 % normal fill, 713 vs 706 G/s at 2^28).
#ifndef ZF_SPEC2
#define ZF_SPEC2 1
#endif
#ifndef ZF_ASYNC_STAGE
#define ZF_ASYNC_STAGE 1
#endif
// Normal rounds: a tail sample's first Marsaglia attempt from the words the
// box attempt already computed (see resolve_round_normal).
#ifndef ZF_TAILFAST
#define ZF_TAILFAST 1
#endif

#ifndef ZF_QUEUE_CAP
#define ZF_QUEUE_CAP 128
#endif
constexpr int kQueueCap = ZF_QUEUE_CAP;
// Normal rounds of 32 use warp-cooperative box attempts (resolve_round_normal);
// ZF_COOP=0 builds the plain recursive rounds for A/B runs.
#ifndef ZF_COOP
#define ZF_COOP 1
#endif
// per-warp shared words: the queue, then 32 x 16 B of round scratch
constexpr int kQueueWords = kQueueCap + (ZF_COOP ? 128 : 0);
// Paired tiles (run_tiles<..., PAIR = true>): the queue bookkeeping runs once
// per pair of tiles, the two 16-bit lane masks side by side in one 32-bit
// mask -- 1.6 % fewer instructions, +2-3 % for the modified fp64 fills and the
// sum-only aggregate, and +2 % at the board's power cap.  The
// callers choose: it costs the traditional kernels and the fp32 normal fill
// (a longer pass-1 body in the I-cache) and does not help the batch kernel.
// ZF_PAIR=0 builds every kernel unpaired (A/B).
#ifndef ZF_PAIR
#define ZF_PAIR 1
#endif
// paired normal kernels: the second queue entry of a lane by a predicated
// store as well (with 32 samples per lane mask, 83 % of pairs have a lane
// holding two: 770 -> 775 G/s at 2^32)
#ifndef ZF_SECOND_STORE
#define ZF_SECOND_STORE 1
#endif
static_assert(kPerLane == 16 || !ZF_PAIR, "paired tiles need 16-bit lane masks");

// ZF_CHECKS=1 (debug builds, tests/test_gpu_checked.py): device-side bounds and
// protocol checks -- queue slots inside the queue, round-scratch indices
// inside the warp's 32 records, every store inside the output, the staged
// pack complete before a round reads it.  A failed check records its source
// line in zf_check_line (one per translation unit, read back by
// zf_debug_check_line_*) and the kernel carries on.
#if defined(ZF_CHECKS) && ZF_CHECKS
static __device__ unsigned int zf_check_line;
#define ZF_CHECK(cond)                                  \
  do {                                                  \
    if (!(cond)) atomicCAS(&zf_check_line, 0u, __LINE__); \
  } while (0)
#else
#define ZF_CHECK(cond) \
  do {                 \
  } while (0)
#endif

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

// mask |= bit if d is NaN (setp.nan on the fp64 pipe + a predicated add)
__device__ __forceinline__ void or_if_nan(uint32_t& mask, double d, uint32_t bit) {
  asm("{\n\t.reg .pred p;\n\tsetp.nan.f64 p, %1, %1;\n\t@p or.b32 %0, %0, %2;\n\t}"
      : "+r"(mask)
      : "d"(d), "r"(bit));
}

template <typename OutT, bool VEC>
struct StoreSink {
  using Out = OutT;
  static constexpr int V = VecOf<OutT>::V;
  OutT* __restrict__ out;
#if defined(ZF_CHECKS) && ZF_CHECKS
  uint64_t n_check = ~0ull;  // stores must stay below it
#endif
  // pass 1: V consecutive values at k (exceptional ones are NaN placeholders,
  // overwritten in pass 2 while the line is still in L2)
  __device__ __forceinline__ void put_vec(uint64_t k, const OutT* v, uint32_t /*exc_bits*/) {
#if defined(ZF_CHECKS) && ZF_CHECKS
    ZF_CHECK(k + V <= n_check);
#endif
    if constexpr (VEC) {
      *reinterpret_cast<typename VecOf<OutT>::T*>(out + k) = VecOf<OutT>::make(v);
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) out[k + e] = v[e];
    }
  }
  __device__ __forceinline__ void put(uint64_t k, OutT v, bool /*exc*/) {
#if defined(ZF_CHECKS) && ZF_CHECKS
    ZF_CHECK(k < n_check);
#endif
    out[k] = v;
  }
  __device__ __forceinline__ void flag(uint32_t& mask, double d, uint32_t bit) {
    or_if_nan(mask, d, bit);
  }
};

// Generate-and-aggregate (the reference's aggregate / bench loop): one running
// fp64 sum per lane.  The NaN test that flags an exceptional sample also
// predicates the add, so the fast path pays one DADD and no integer work.
struct SumSink {
  using Out = double;
  static constexpr int V = 2;
  double s = 0.0;
  __device__ __forceinline__ void flag(uint32_t& mask, double d, uint32_t bit) {
    asm("{\n\t.reg .pred p;\n\tsetp.nan.f64 p, %2, %2;\n\t@p or.b32 %0, %0, %3;"
        "\n\t@!p add.rn.f64 %1, %1, %2;\n\t}"
        : "+r"(mask), "+d"(s)
        : "d"(d), "r"(bit));
  }
  __device__ __forceinline__ void put_vec(uint64_t, const double*, uint32_t) {}
  __device__ __forceinline__ void put(uint64_t, double v, bool exc) {
    if (!exc) s = __dadd_rn(s, v);
  }
};

// Validation statistics: raw power sums x^1..x^5 (quality.py:92-106), an
// equal-width histogram with under/overflow bins and threshold counts.
// EXTRA = false: moments only (no histogram / thresholds); MOMENTS = false:
// histogram / thresholds only.
template <bool EXTRA, bool MOMENTS = true>
struct StatsSinkT {
  using Out = double;
  static constexpr int V = 2;
  double s[5] = {0, 0, 0, 0, 0};
  unsigned long long thr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned int* hist;  // smem, nbins + 2
  double lo, inv_w, tmin;  // tmin: smallest threshold (+inf if none)
  int nbins, nthresh;
  bool abs_t;
  const double* t;  // thresholds (smem)
  __device__ __forceinline__ void add(double x) {
    if constexpr (MOMENTS) {
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
    }
    if constexpr (EXTRA) {
      const double a = abs_t ? fabs(x) : x;
      if (a > tmin) {  // tail counts: almost every sample is below all thresholds
#pragma unroll
        for (int q = 0; q < 8; ++q)  // fixed trip count keeps thr[] in registers
          if (q < nthresh) thr[q] += a > t[q];
      }
      if (nbins) {
        const double f = (x - lo) * inv_w;
        int b = f < 0.0 ? -1 : (f >= (double)nbins ? nbins : (int)f);
        atomicAdd(hist + (b + 1), 1u);
      }
    }
  }
  __device__ __forceinline__ void put_vec(uint64_t, const double* v, uint32_t exc_bits) {
#pragma unroll
    for (int e = 0; e < V; ++e)
      if (!((exc_bits >> e) & 1)) add(v[e]);  // bits above V are ignored
  }
  __device__ __forceinline__ void put(uint64_t, double v, bool exc) {
    if (!exc) add(v);
  }
  __device__ __forceinline__ void flag(uint32_t& mask, double d, uint32_t bit) {
    or_if_nan(mask, d, bit);
  }
};
using StatsSink = StatsSinkT<true>;

// Tail counts only, for thresholds no fast-path value can exceed (every one
// at or above the table's largest fast-path magnitude, e.g. |x| > 5, 6, 7 and
// x > X[1] in config 5): pass 1 only flags exceptional samples, and just the
// values that come out of the rounds (and the ragged last tile) are compared.
struct TailSink {
  using Out = double;
  static constexpr int V = 2;
  // per-lane counts: a lane sees < 2^32 samples (2^44 / the stats grid's threads)
  uint32_t thr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int nthresh;
  bool abs_t;
  const double* t;  // thresholds (smem)
  __device__ __forceinline__ void flag(uint32_t& mask, double d, uint32_t bit) {
    or_if_nan(mask, d, bit);
  }
  __device__ __forceinline__ void put_vec(uint64_t, const double*, uint32_t) {}
  __device__ __forceinline__ void put(uint64_t, double x, bool exc) {
    if (exc) return;
    const double a = abs_t ? fabs(x) : x;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < nthresh) thr[q] += a > t[q];
  }
};


// Pass 1 of one warp tile: samples [base, min(base + kTile, n)) of the counter
// stream (seed, ctr_base).  Returns the lane's mask of exceptional samples
// (bit it*V + e  <->  offset it*32*V + lane*V + e).
template <int DIST, bool COUNTED, class Sink>
__device__ __forceinline__ uint32_t fast_pass(const DevPack& P, uint64_t seed, uint64_t ctr_base,
                                              Sink& sink, uint64_t n, uint64_t base, int lane,
                                              LaneCounts& lc) {
  using OutT = typename Sink::Out;
  constexpr int V = Sink::V;
  constexpr int kIters = kPerLane / V;
  constexpr uint64_t kIterStride = (uint64_t)(32 * V) * kGamma;  // mod 2^64
  const double* sx = P.sx;
  const uint64_t k_lane = base + (uint64_t)lane * V;
  const uint64_t st0 = seed + (ctr_base + k_lane + 1) * kGamma;
  uint32_t mask = 0;
  if (base + kTile <= n) {
#pragma unroll kPass1Unroll
    for (int it = 0; it < kIters; ++it) {
      const uint64_t st = st0 + (uint64_t)it * kIterStride;
      OutT v[V];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        // sx[i+1] is NaN for every byte i >= L_max (see fill_devpack), so the
        // fast value itself flags an exceptional sample: a DSETP on the fp64
        // pipe instead of integer compare/select work on the busy ALU pipe.
#if defined(ZF_DEBUG_P1)  // energy isolation builds (run with ZF_PASS2=9): drop one stage
        // 1: no word function (the counter itself)  2: no table lookup
        // 3: no conversion + multiply (word bits stored)  4: constant stores only
        const uint64_t z = st + (uint64_t)e * kGamma;
        const uint64_t w = ZF_DEBUG_P1 == 1 || ZF_DEBUG_P1 == 4 ? z : ctr_word(z);
        double d;
        if (ZF_DEBUG_P1 == 2)
          d = __dmul_rn(__ll2double_rn((long long)w), 0x1p-63);
        else if (ZF_DEBUG_P1 == 3)
          d = __longlong_as_double((long long)(w & 0x3fffffffffffffffull)) + sx[(w & 0xFF) + 1];
        else if (ZF_DEBUG_P1 == 4)
          d = (double)e;
        else
          d = fast_value<DIST>(sx, w);
#else
        const uint64_t w = ctr_word(st + (uint64_t)e * kGamma);
        double d = fast_value<DIST>(sx, w);
#endif
        if constexpr (kTrad<DIST>)  // traditional: integer fast-accept test
          d = trad_fast<DIST>(P.kk, w) ? d : __longlong_as_double(0x7ff8000000000000ll);
        sink.flag(mask, d, 1u << (it * V + e));
        v[e] = to_out<OutT>(d);
      }
      sink.put_vec(k_lane + (uint64_t)it * 32 * V, v, mask >> (it * V));
    }
    if (COUNTED) {
      const unsigned fast = kPerLane - __popc(mask);
      lc.c[0] += fast;
      lc.c[1] += fast;
    }
  } else {
    // ragged last tile: identical words, bounds-checked element stores
    unsigned valid = 0;
#pragma unroll 1
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const uint64_t k = k_lane + (uint64_t)it * 32 * V + e;
        if (k < n) {
          const uint64_t u = ctr_word(st0 + (uint64_t)it * kIterStride + (uint64_t)e * kGamma);
          const double d = fast_value<DIST>(sx, u);
          // modified tables: the NaN sentinel of sx (pass 1 may run before the
          // rest of the pack -- lmax included -- has been staged); traditional
          // tables are staged whole before pass 1
          const bool exc = kTrad<DIST> ? exc_word<DIST>(P, u) : isnan(d);
          mask |= (uint32_t)exc << (it * V + e);
          sink.put(k, to_out<OutT>(d), exc);
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

// Pass 2 body for one exceptional sample k: the full recursive draw on its
// secondary counter stream, written through the sink.
template <int DIST, bool COUNTED, class Sink>
__device__ __forceinline__ void resolve_one(const DevPack& P, const DevPack& E, uint64_t seed,
                                            uint64_t ctr_base, Sink& sink, uint64_t k,
                                            LaneCounts& lc) {
  using OutT = typename Sink::Out;
#if defined(ZF_DEBUG_P2) && ZF_DEBUG_P2 == 2  // cost isolation: store without drawing
  sink.put(k, to_out<OutT>(0.0), false);
  return;
#endif
  const uint64_t K = ctr_base + k;
#if ZF_HOIST
  if constexpr (DIST == ZF_EXP && !COUNTED) {
    sink.put(k, to_out<OutT>(exp_draw_ctr(P, seed + (kExcBase + (K << kExcShift)) * kGamma)),
             false);
    return;
  }
#endif
  // k is exceptional: the modified exponential draw only needs to know that
  // (its first word's bits are never read again), the normal one needs the
  // sign bit, the traditional ones the whole word
  const uint64_t u = DIST == ZF_EXP ? 0xFFull : ctr_word(seed + (K + 1) * kGamma);
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
#if defined(ZF_DEBUG_P2) && ZF_DEBUG_P2 == 1  // cost isolation: draw without storing
  if (v == 12345.0) sink.put(k, to_out<OutT>(v), false);
  return;
#endif
  sink.put(k, to_out<OutT>(v), false);
}

// kSlotLanes[r]: bits 0, r, 2r, ... below 32 (the lanes serving slot 0 of r)
__constant__ const uint32_t kSlotLanes[33] = {
    0u,          0xFFFFFFFFu, 0x55555555u, 0x49249249u, 0x11111111u, 0x42108421u, 0x41041041u,
    0x10204081u, 0x01010101u, 0x08040201u, 0x40100401u, 0x00400801u, 0x01001001u, 0x04002001u,
    0x10004001u, 0x40008001u, 0x00010001u, 0x00020001u, 0x00040001u, 0x00080001u, 0x00100001u,
    0x00200001u, 0x00400001u, 0x00800001u, 0x01000001u, 0x02000001u, 0x04000001u, 0x08000001u,
    0x10000001u, 0x20000001u, 0x40000001u, 0x80000001u, 0x00000001u};
// A full round of 32 normal draws (one queued sample k per lane) with
// warp-cooperative box attempts.  Every lane first makes its own sample's
// alias pick and first box attempt, as the sequential loop does.  Then, while
// r samples are unresolved, lane L works on unresolved sample L mod r and
// evaluates its attempt number next + L / r: the words of attempt a of sample
// K sit at fixed positions 3 + 2a, 4 + 2a of K's secondary counter stream, so
// any lane can evaluate any attempt.  A sample takes its accepted attempt with
// the lowest index (the lowest accepting lane of its slot) -- exactly the one
// the sequential loop would stop at -- and otherwise advances `next` by the
// number of lanes that served it.  Owners publish (stream base, j, next) in
// `own` (32 x 16 B of per-warp shared scratch); a round takes ~2-3 iterations
// where the one-sample-per-lane loop waits ~5.4 for its slowest lane.
template <class Sink>
__device__ __forceinline__ void resolve_round_normal(const DevPack& P, const DevPack& E,
                                                     uint64_t seed, uint64_t ctr_base, Sink& sink,
                                                     uint64_t k, int lane, uint32_t* own) {
  // (own must be 16-byte aligned: kQueueCap words past a 16-byte aligned queue)
  using OutT = typename Sink::Out;
  const uint64_t K = ctr_base + k;
  const uint64_t u = ctr_word(seed + (K + 1) * kGamma);  // the sign word
  const uint64_t sbase = seed + (kExcBase + (K << kExcShift)) * kGamma;
  double val;
  bool done;
#if ZF_HOIST
  // the alias pick's and the first box attempt's words are independent
  // counter positions: compute them side by side
  const uint64_t w1 = ctr_word(sbase + kGamma), w2 = ctr_word(sbase + 2 * kGamma);
  const uint64_t w3 = ctr_word(sbase + 3 * kGamma), w4 = ctr_word(sbase + 4 * kGamma);
#if ZF_SPEC2
  // and the second attempt's (positions 5, 6): with ~58 % acceptance per box
  // attempt, 18 % of the lanes are left for the cooperative iterations
  const uint64_t w5 = ctr_word(sbase + 5 * kGamma), w6 = ctr_word(sbase + 6 * kGamma);
#endif
  const int j = alias_from(P, w1, w2);
  uint32_t next = 1;  // this lane's sample: attempts 0 .. next-1 all rejected
  if (j == 0) {
#if ZF_TAILFAST
    // Marsaglia's first attempt from words 3 and 4 (already computed for the
    // box attempt) when both embedded exponential draws take their fast path
    // -- the common case, the same arithmetic as normal_tail; anything else
    // (an exceptional byte: NaN, or a rejection) runs the full loop
    const double e1 = fast_value<ZF_EXP>(E.sx, w3), e2 = fast_value<ZF_EXP>(E.sx, w4);
    const double x = __ddiv_rn(e1, P.tailx);
    if (__dadd_rn(e2, e2) > __dmul_rn(x, x)) {
      val = __dadd_rn(P.tailx, x);
    } else
#endif
    {
      NoCount c;
      CtrStream s{sbase + 2 * kGamma};
      val = normal_tail(P, E, s, c);
    }
    done = true;
  } else {
    done = normal_box_words(P, j, w3, w4, val);
#if ZF_SPEC2
    double x1;
    const bool a1 = normal_box_words(P, j, w5, w6, x1);
    if (!done && a1) {
      val = x1;
      done = true;
    }
    next = 2;
#endif
  }
#else
  uint32_t next = 1;  // this lane's sample: attempts 0 .. next-1 all rejected
  CtrStream s{sbase};
  const int j = alias_pick(P, s);
  if (j == 0) {
    NoCount c;
    val = normal_tail(P, E, s, c);
    done = true;
  } else {
    done = normal_box_attempt(P, j, s, val);
  }
#endif
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t un = __ballot_sync(0xffffffffu, !done); un;
       un = __ballot_sync(0xffffffffu, !done)) {
    const int r = __popc(un);
    const int rank = __popc(un & lt);  // my slot if unresolved
    // owners publish (stream base, slot j, next attempt) at their rank
    ZF_CHECK(r >= 1 && r <= 32 && rank < 32);
    if (!done)
      reinterpret_cast<uint4*>(own)[rank] =
          make_uint4((uint32_t)sbase, (uint32_t)(sbase >> 32), (uint32_t)j, next);
    __syncwarp();
    // lane / r and lane % r without an integer division: (lane + 0.5) / r is
    // at least 1/64 away from an integer, far above the reciprocal's error
    const int qd = __float2int_rz(__fmul_rn((float)lane + 0.5f, __frcp_rn((float)r)));
    ZF_CHECK(lane - qd * r >= 0 && lane - qd * r < r);
    const uint4 st4 = reinterpret_cast<const uint4*>(own)[lane - qd * r];
    __syncwarp();
    const uint64_t sb = ((uint64_t)st4.y << 32) | st4.x;
    const int jo = (int)st4.z;
    const uint32_t a = st4.w + (uint32_t)qd;
    CtrStream t{sb + (uint64_t)(2 + 2 * a) * kGamma};
    double x;
    const bool acc = normal_box_attempt(P, jo, t, x);
    const uint32_t A = __ballot_sync(0xffffffffu, acc);
    // lanes serving slot `rank`: rank, rank + r, rank + 2r, ...
    const uint32_t mine = kSlotLanes[r] << rank;
    const uint32_t hits = done ? 0u : (A & mine);
    const int w = hits ? __ffs(hits) - 1 : lane;
    const double xw = __shfl_sync(0xffffffffu, x, w);
    if (hits) {
      val = xw;
      done = true;
    } else if (!done) {
      next += (uint32_t)__popc(mine);
    }
  }
  sink.put(k, to_out<OutT>((long long)u < 0 ? -val : val), false);
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

// The same prefix from bit-plane ballots: counts are tiny (a lane holds ~0.19
// exceptional samples per tile), so planes 0 and 1 decide it unless some lane
// has 4 or more, which falls back to the shuffle scan.  No dependent shuffle
// chain after pass 1: three independent ballots and a few popcounts.
__device__ __forceinline__ int warp_excl_count(int mine, int lane, int* total) {
  const uint32_t b0 = __ballot_sync(0xffffffffu, mine & 1);
  const uint32_t b1 = __ballot_sync(0xffffffffu, mine & 2);
  const uint32_t big = __ballot_sync(0xffffffffu, mine >= 4);
  if (big) return warp_excl_scan(mine, lane, total);
  const uint32_t lt = (1u << lane) - 1u;
  *total = __popc(b0) + 2 * __popc(b1);
  return __popc(b0 & lt) + 2 * __popc(b1 & lt);
}

// The same from the lane masks themselves: when no lane holds two or more
// exceptional samples (~60 % of 512-sample tiles) one ballot of "any" decides
// the prefix; otherwise the bit-plane count above.
__device__ __forceinline__ int warp_excl_mask(uint32_t mask, int lane, int* total,
                                              bool* multi_any = nullptr) {
  const uint32_t multi = __ballot_sync(0xffffffffu, (mask & (mask - 1u)) != 0u);
  if (multi_any) *multi_any = multi != 0u;
  if (multi) return warp_excl_count(__popc(mask), lane, total);
  const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
  *total = __popc(any);
  return __popc(any & ((1u << lane) - 1u));
}
__device__ __forceinline__ int warp_excl_mask(uint64_t mask, int lane, int* total,
                                              bool* multi_any = nullptr) {
  const uint32_t multi = __ballot_sync(0xffffffffu, (mask & (mask - 1u)) != 0u);
  if (multi_any) *multi_any = multi != 0u;
  if (multi) return warp_excl_count(__popcll(mask), lane, total);
  const uint32_t any = __ballot_sync(0xffffffffu, mask != 0u);
  *total = __popc(any);
  return __popc(any & ((1u << lane) - 1u));
}

// x without its highest set bit; 0 for x == 0 (the shift count is masked so
// it stays defined when __clz(0) == 32)
__device__ __forceinline__ uint32_t drop_top(uint32_t x) {
  return x & ~(0x80000000u >> (__clz(x) & 31));
}

template <int V>
__device__ __forceinline__ uint32_t mask_bit_offset(int b, int lane) {
  return (uint32_t)((b / V) * 32 * V + lane * V + (b % V));
}

// Per-warp queue words: < 32 leftovers + the exceptions of one tile (~15 on
// average for 1024 samples); a tile that would overflow is resolved in place.
// Small on purpose: shared memory, not registers, limits CTAs per SM.

// Pass-2 policies (template parameter P2 of run_tiles), all bit-identical:
//   3  rounds of exactly 32 recursive draws as soon as 32 are queued
//   9  DEBUG ONLY: pass 1 alone, exceptions left as NaN (cost isolation)
// (Round-1 experiments with uniform speculative rounds, lane-refilling box
// engines, a resumable state machine and warp specialisation were all
// bit-identical but slower on B200: their extra registers and code cost the
// fast path more than they saved.)
// A warp's whole share of a fill: tiles first_tile, first_tile + stride, ...
// lane-mask helpers for the 32-bit (one or two tiles) and 64-bit (four tiles)
// masks of run_tiles
__device__ __forceinline__ int mask_top(uint32_t m) { return 31 - __clz(m); }
__device__ __forceinline__ int mask_top(uint64_t m) { return 63 - __clzll((long long)m); }
__device__ __forceinline__ uint64_t drop_top(uint64_t x) {
  return x & ~(0x8000000000000000ull >> (__clzll((long long)x) & 63));
}
__device__ __forceinline__ int mask_popc(uint32_t m) { return __popc(m); }
__device__ __forceinline__ int mask_popc(uint64_t m) { return __popcll(m); }

template <int DIST, bool COUNTED, int P2, class Sink, int NT_ = 1>
__device__ __forceinline__ void run_tiles(const DevPack& P, const DevPack& E, uint64_t seed,
                                          uint64_t ctr_base, Sink& sink, uint64_t n,
                                          uint64_t first_tile, uint64_t stride, uint32_t* q,
                                          int lane, LaneCounts& lc,
                                          const uint64_t* late = nullptr,
                                          uint64_t pair_off = 0) {
  static_assert(P2 == 3 || P2 == 9, "unknown pass-2 policy");
  // tiles per queue bookkeeping (1, 2 or 4; ZF_PAIR=0 forces 1)
  constexpr int NT = ZF_PAIR ? NT_ : 1;
  static_assert(NT == 1 || NT == 2 || NT == 4, "1, 2 or 4 tiles per bookkeeping");
  constexpr bool PAIR = NT > 1;
  using Mask = typename std::conditional<NT == 4, uint64_t, uint32_t>::type;
  constexpr int kEntBits = kPerLaneBits + (NT == 4 ? 2 : NT == 2 ? 1 : 0);  // mask-bit field
  // paired bookkeeping: the loop visits tiles first_tile + i * step, each with
  // its partner tile + off (pair_off = 0: the partner is the next grid-stride
  // tile, off = stride and step = 2 * stride; the fill kernel passes
  // adjacent pairs, off = 1 with a doubled first tile and stride)
  const uint64_t off = pair_off ? pair_off : stride;
  const uint64_t step = (PAIR && !pair_off) ? NT * stride : stride;
  // `late`: mbarrier (phase 0) of the table arrays only the rounds read
  bool tables_ready = late == nullptr;
  auto need_tables = [&]() {
    if (!tables_ready) {
      mbar_wait(late, 0);
      tables_ready = true;
    }
    ZF_CHECK(P.nslots == P.lmax + 1 && E.nslots == E.lmax + 1);  // the whole pack landed
  };
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  // queue entry = loop iteration << (kEntBits + 5) | lane << kEntBits | mask
  // bit (bit >= 16: the pair's second tile): the enqueue loop (a few lanes
  // active) only ORs the bit in; the full-warp rounds decode the sample offset
  auto k_of = [&](uint32_t e) -> uint64_t {
    const uint32_t b = e & ((1u << kEntBits) - 1u);
    const uint32_t o = mask_bit_offset<Sink::V>((int)(b & (kPerLane - 1u)),
                                                (int)((e >> kEntBits) & 31u));
    const uint64_t t = first_tile + (uint64_t)(e >> (kEntBits + 5)) * step +
                       (PAIR ? (uint64_t)(b >> kPerLaneBits) * off : 0);
    return t * kTile + o;
  };
  if constexpr (P2 == 9) {
    for (uint64_t tile = first_tile; tile < ntiles; tile += step) {
#pragma unroll
      for (int h = 0; h < NT; ++h)
        if (h == 0 || tile + h * off < ntiles)
          fast_pass<DIST, COUNTED>(P, seed, ctr_base, sink, n, (tile + h * off) * kTile, lane, lc);
    }
    return;
  } else {
    int qn = 0;  // warp-uniform queue length
    uint32_t iter = 0;
    const uint32_t qs = (uint32_t)__cvta_generic_to_shared(q);
    for (uint64_t tile = first_tile; tile < ntiles; tile += step, ++iter) {
      Mask mask = fast_pass<DIST, COUNTED>(P, seed, ctr_base, sink, n, tile * kTile, lane, lc);
#pragma unroll
      for (int h = 1; h < NT; ++h)
        if (tile + h * off < ntiles)
          mask |= (Mask)fast_pass<DIST, COUNTED>(P, seed, ctr_base, sink, n,
                                                 (tile + h * off) * kTile, lane, lc)
                  << (16 * h);
      int total;
      bool multi;  // some lane holds two or more exceptions
      int slot = qn + warp_excl_mask(mask, lane, &total, &multi);
#if defined(ZF_CHECKS) && ZF_CHECKS
      const int first_slot = slot;  // this lane's entries: [first_slot, + popc(mask))
#endif
#if defined(ZF_DEBUG_Q) && ZF_DEBUG_Q == 1  // cost isolation: scan only
      if (total == 12345) q[lane] = slot;
      continue;
#endif
      if (total == 0) continue;
      if (qn + total > kQueueCap) {
        // (practically never: ~100 exceptions in one tile, expected ~15) resolve
        // this tile's exceptions in place, each lane walking its own mask
        need_tables();
        for (Mask m = mask; m; m &= m - 1) {
          const int b = mask_top(m ^ (m & (m - 1)));  // lowest set bit
          resolve_one<DIST, COUNTED>(
              P, E, seed, ctr_base, sink,
              (tile + (uint64_t)(b >> kPerLaneBits) * off) * kTile +
                  mask_bit_offset<Sink::V>(b & (kPerLane - 1), lane),
              lc);
        }
        __syncwarp();
        continue;
      }
      const uint32_t tag = (iter << (kEntBits + 5)) | ((uint32_t)lane << kEntBits);
      {
        // every lane's highest entry with one predicated shared store (no
        // divergent block); the loop runs only when some lane holds two or
        // more (~40 % of tiles) and then only for the rest of the bits
        const int hb = mask_top(mask);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
                     "@p st.shared.u32 [%0], %1;\n\t}"
                     ::"r"(qs + 4u * (uint32_t)slot), "r"(tag | (uint32_t)hb),
                     "r"((uint32_t)(mask != 0))
                     : "memory");
        if (multi) {
          if constexpr (DIST == ZF_EXP || (ZF_SECOND_STORE && PAIR)) {
          // exponential (1.56 % exceptional: a lane holds two in ~57 % of
          // tiles) and paired normal kernels: the second entry is predicated
          // as well and the loop runs only for lanes with three or more.
          // (The unpaired normal kernel loses 6 % with it: +4 registers and
          // a worse layout.)
          const Mask m2 = drop_top(mask);
          const int hb2 = mask_top(m2);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
                       "@p st.shared.u32 [%0], %1;\n\t}"
                       ::"r"(qs + 4u * (uint32_t)(slot + 1)), "r"(tag | (uint32_t)hb2),
                       "r"((uint32_t)(m2 != 0))
                       : "memory");
          if (__ballot_sync(0xffffffffu, (m2 & (m2 - 1u)) != 0u)) {
            slot += 2;
            for (Mask m = drop_top(m2); m;) {
              const int b = mask_top(m);
              m ^= (Mask)1 << b;
              ZF_CHECK(slot < kQueueCap);
            q[slot++] = tag | (uint32_t)b;
            }
          }
          } else {
          ++slot;
          for (Mask m = drop_top(mask); m;) {
            const int b = mask_top(m);
            m ^= (Mask)1 << b;
            ZF_CHECK(slot < kQueueCap);
            q[slot++] = tag | (uint32_t)b;
          }
          }
        }
      }
      qn += total;
#if defined(ZF_CHECKS) && ZF_CHECKS
      ZF_CHECK(qn <= kQueueCap && first_slot + mask_popc(mask) <= qn);
#endif
      __syncwarp();
#if defined(ZF_DEBUG_Q) && ZF_DEBUG_Q == 2  // cost isolation: scan + enqueue, no rounds
      if (qn >= 32) qn = 0;
      continue;
#endif
      if (qn < 32) continue;
      need_tables();
      int done = 0;
      for (; qn - done >= 32; done += 32)
      {
        if constexpr (ZF_COOP && DIST == ZF_NORMAL && !COUNTED) {
          const uint32_t tag = q[done + lane];
          __syncwarp();
          resolve_round_normal(P, E, seed, ctr_base, sink, k_of(tag), lane, q + kQueueCap);
        } else {
          resolve_one<DIST, COUNTED>(P, E, seed, ctr_base, sink, k_of(q[done + lane]), lc);
        }
      }
      __syncwarp();
      for (int j = lane; j < qn - done; j += 32) q[j] = q[j + done];
      qn -= done;
      __syncwarp();
    }
    if (qn) need_tables();
    if (lane < qn) resolve_one<DIST, COUNTED>(P, E, seed, ctr_base, sink, k_of(q[lane]), lc);
    __syncwarp();
  }
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
