// zf_replay.cu -- oracle mode: the reference's sequential word stream, resolved
// in parallel; plus device generation of the reference's word streams.
//
// The reference consumes ONE word stream with a variable number of words per
// draw (fill_exp, _kernels.py:226-260; replay source :83-88).  Position p of
// the stream starts a one-word draw when its low byte is < L_max, unless p lies
// inside an earlier exceptional draw.  Pipeline over a window of L logical
// positions (word p = words[(cursor + p) % nwords]):
//
//   A  classify + compact   E = sorted positions whose byte >= L_max   (~1.6 %)
//   B  exceptional draws    full draw body from every e in E, in parallel:
//                           length, value, path record, counter deltas
//   C  resolve              e is a real start iff no earlier *real* draw covers
//                           it.  "Heads" (not covered by any earlier candidate,
//                           from an exclusive max-scan of e + len) are real;
//                           between heads a thread walks its short cluster.
//   D  mark + rank          interior words of real draws are not starts; an
//                           exclusive scan of start flags gives output ranks
//   E  emit                 out[rank] = fast value or the exceptional value
//
// If the window is too short for n draws, the host doubles L and reruns.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <type_traits>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "zf_internal.h"

namespace zf {
namespace {

constexpr int kRT = 256;              // threads per block
#ifndef ZF_RI
#define ZF_RI 8
#endif
constexpr int kRI = ZF_RI;            // items per thread
constexpr int kRB = kRT * kRI;        // positions per block
constexpr uint32_t kIncomplete = 0xFFFFFFFFu;

struct Window {
  const uint64_t* w;
  uint64_t nwords, cursor, L;
  __device__ __forceinline__ uint64_t word(uint64_t p) const {
    uint64_t idx = cursor + p;
    if (idx >= nwords) idx %= nwords;
    return __ldg(reinterpret_cast<const unsigned long long*>(w) + idx);
  }
};

// ---- block-wide exclusive scans (256 threads) -------------------------------
template <typename T, class Op>
__device__ __forceinline__ T block_exclusive(T v, T identity, Op op, T* smem_warp, T* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl = op(incl, y);
  }
  if (lane == 31) smem_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    T x = lane < nw ? smem_warp[lane] : identity;
    T xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, xi, d);
      if (lane >= d) xi = op(xi, y);
    }
    if (lane < nw) smem_warp[lane] = xi;  // inclusive per warp
  }
  __syncthreads();
  const T warp_prefix = wid ? smem_warp[wid - 1] : identity;
  const T up = __shfl_up_sync(0xffffffffu, incl, 1);  // all 32 lanes must execute it
  T res = op(warp_prefix, lane ? up : identity);
  if (total) *total = smem_warp[nw - 1];
  __syncthreads();
  return res;
}

struct Add {
  template <typename T>
  __host__ __device__ T operator()(T a, T b) const { return a + b; }
};
struct Max {
  template <typename T>
  __host__ __device__ T operator()(T a, T b) const { return a > b ? a : b; }
};

// ---- warp-striped position layout --------------------------------------------
// Block b covers positions [b*kRB, (b+1)*kRB); warp w the span of 32*kRI
// positions starting at b*kRB + w*32*kRI, item j of lane l being position
// span + 32*j + l: every load is a coalesced row, order is position order, and
// prefix counts come from ballots.
constexpr int kWarpSpan = 32 * kRI;

__device__ __forceinline__ uint64_t striped_pos(int j) {
  return (uint64_t)blockIdx.x * kRB + (uint64_t)(threadIdx.x >> 5) * kWarpSpan + 32 * j +
         (threadIdx.x & 31);
}

// This thread's kRI striped words (0 past the window).  Windows that do not
// wrap (every sequential-generator fill) take a branch-free path so all kRI
// loads are in flight together; wrapping replay lists use the modulo.
__device__ __forceinline__ void load_striped(const Window& win, uint64_t w[kRI]) {
  const unsigned long long* base = reinterpret_cast<const unsigned long long*>(win.w);
  if (win.cursor + win.L <= win.nwords) {
#pragma unroll
    for (int j = 0; j < kRI; ++j) {
      const uint64_t p = striped_pos(j);
      w[j] = p < win.L ? __ldg(base + win.cursor + p) : 0;
    }
  } else {  // unrolled too: a dynamic index would put w[] in local memory
#pragma unroll
    for (int j = 0; j < kRI; ++j) {
      const uint64_t p = striped_pos(j);
      w[j] = p < win.L ? win.word(p) : 0;
    }
  }
}

// the same for two counts at once (one pair of barriers)
__device__ __forceinline__ void warp_base2(uint32_t ta, uint32_t tb, uint2* smem, uint32_t* ba,
                                           uint32_t* bb) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) smem[wid] = make_uint2(ta, tb);
  __syncthreads();
  uint32_t a = 0, b = 0;
#pragma unroll
  for (int w = 0; w < kRT / 32; ++w) {
    const uint2 t = smem[w];
    a += w < wid ? t.x : 0;
    b += w < wid ? t.y : 0;
  }
  *ba = a;
  *bb = b;
  __syncthreads();
}

// exclusive prefix of per-warp totals over the block's warps (+ block total)
__device__ __forceinline__ uint32_t warp_base(uint32_t warp_total, uint32_t* smem,
                                              uint32_t* block_total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) smem[wid] = warp_total;
  __syncthreads();
  uint32_t base = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kRT / 32; ++w) {
    const uint32_t t = smem[w];
    base += w < wid ? t : 0;
    tot += t;
  }
  if (block_total) *block_total = tot;
  __syncthreads();
  return base;
}

// ---- A: classify / compact ---------------------------------------------------
template <int DIST>
__global__ void __launch_bounds__(kRT)
    rp_count_exc(Window win, const DevPack* __restrict__ P, uint32_t* __restrict__ bcnt) {
  __shared__ uint32_t wb[kRT / 32];
  // all kRI loads in flight before the first ballot (a ballot per load would
  // serialise them: ~3 TB/s instead of the HBM rate)
  uint64_t w[kRI];
  load_striped(win, w);
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kRI; ++j)
    c += __popc(__ballot_sync(0xffffffffu, striped_pos(j) < win.L && exc_word<DIST>(*P, w[j])));
  uint32_t tot;
  warp_base(c, wb, &tot);
  if (threadIdx.x == 0) bcnt[blockIdx.x] = tot;
}

template <int DIST>
__global__ void __launch_bounds__(kRT)
    rp_compact_exc(Window win, const DevPack* __restrict__ P, const uint32_t* __restrict__ boff,
                   uint32_t* __restrict__ E, uint32_t cap) {
  __shared__ uint32_t wb[kRT / 32];
  const uint32_t lt = (1u << (threadIdx.x & 31)) - 1u;
  uint64_t w[kRI];
  load_striped(win, w);
  uint32_t b[kRI];
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kRI; ++j) {
    b[j] = __ballot_sync(0xffffffffu, striped_pos(j) < win.L && exc_word<DIST>(*P, w[j]));
    c += __popc(b[j]);
  }
  uint32_t o = boff[blockIdx.x] + warp_base(c, wb, nullptr);
#pragma unroll
  for (int j = 0; j < kRI; ++j) {
    if ((b[j] >> (threadIdx.x & 31)) & 1) {
      const uint32_t e = o + __popc(b[j] & lt);
      if (e < cap) E[e] = (uint32_t)striped_pos(j);  // (the host sized E for a bound)
    }
    o += __popc(b[j]);
  }
}

// ---- B: exceptional draws ------------------------------------------------------
struct ExcOut {
  uint32_t* len;
  double* val;
  uint32_t* meta;  // layer | path << 8 | attempts << 16
  uint32_t* cnt;   // [m][6]
};

template <int DIST>
__global__ void __launch_bounds__(kRT)
    rp_draw_exc(const DevTables* __restrict__ gt, Window win, const uint32_t* __restrict__ E,
                const uint32_t* __restrict__ pm, ExcOut o) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kPacks = kPacksOf<DIST>;
  DevPack* sp = reinterpret_cast<DevPack*>(smem_raw);
  stage_block(sp, primary_pack<DIST>(gt), kPacks * (int)sizeof(DevPack));
  __syncthreads();
  const uint32_t i = blockIdx.x * kRT + threadIdx.x;
  if (i >= *pm) return;
  const uint64_t p = E[i];
  BufStream s{win.w, win.nwords, win.cursor, p + 1, win.L, 0, false};
  const uint64_t u = win.word(p);
  Count c;
  const double v = draw<DIST>(sp[0], sp[kPacks - 1], u, s, c);
  o.len[i] = s.over ? kIncomplete : 1u + s.count;
  o.val[i] = v;
  o.meta[i] = (uint32_t)(u & 0xFF) | ((uint32_t)c.path << 8) | ((uint32_t)c.attempts << 16);
#pragma unroll
  for (int q = 0; q < 6; ++q) o.cnt[(uint64_t)i * 6 + q] = c.c[q];
}

// ---- C: resolve real starts ------------------------------------------------------
__device__ __forceinline__ uint64_t reach_of(const uint32_t* E, const uint32_t* len, uint32_t i) {
  const uint32_t l = len[i];
  return l == kIncomplete ? ~0ull : (uint64_t)E[i] + l;
}

__global__ void rp_reach_max(const uint32_t* __restrict__ E, const uint32_t* __restrict__ len,
                             const uint32_t* __restrict__ pm, uint64_t* __restrict__ bmax) {
  __shared__ uint64_t wb[32];
  const uint32_t m = *pm;
  const uint64_t i0 = (uint64_t)blockIdx.x * kRB + (uint64_t)threadIdx.x * kRI;
  uint64_t mx = 0;
  for (int j = 0; j < kRI; ++j)
    if (i0 + j < m) mx = max(mx, reach_of(E, len, (uint32_t)(i0 + j)));
  uint64_t tot;
  block_exclusive<uint64_t>(mx, 0ull, Max(), wb, &tot);
  if (threadIdx.x == 0) bmax[blockIdx.x] = tot;
}

__global__ void rp_heads(const uint32_t* __restrict__ E, const uint32_t* __restrict__ len,
                         const uint32_t* __restrict__ pm, const uint64_t* __restrict__ bpre,
                         uint8_t* __restrict__ head) {
  __shared__ uint64_t wb[32];
  const uint32_t m = *pm;
  const uint64_t i0 = (uint64_t)blockIdx.x * kRB + (uint64_t)threadIdx.x * kRI;
  uint64_t mx = 0;
  for (int j = 0; j < kRI; ++j)
    if (i0 + j < m) mx = max(mx, reach_of(E, len, (uint32_t)(i0 + j)));
  uint64_t run = max(bpre[blockIdx.x], block_exclusive<uint64_t>(mx, 0ull, Max(), wb, nullptr));
  for (int j = 0; j < kRI; ++j) {
    const uint64_t i = i0 + j;
    if (i >= m) break;
    head[i] = run <= E[i];
    run = max(run, reach_of(E, len, (uint32_t)i));
  }
}

constexpr int kWalkChunk = 16;

__global__ void rp_walk(const uint32_t* __restrict__ E, const uint32_t* __restrict__ len,
                        const uint8_t* __restrict__ head, const uint32_t* __restrict__ pm,
                        uint8_t* __restrict__ real) {
  const uint32_t m = *pm;
  const uint64_t beg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kWalkChunk;
  if (beg >= m) return;
  const uint64_t end = std::min<uint64_t>(beg + kWalkChunk, m);
  uint64_t i = beg;
  while (i < end && !head[i]) ++i;  // leading non-heads belong to the previous walker
  if (i == end) return;
  uint64_t cursor = 0;
  for (; i < m && (i < end || !head[i]); ++i) {
    const uint8_t r = E[i] >= cursor;
    real[i] = r;
    if (r) cursor = reach_of(E, len, (uint32_t)i);
  }
}

// ---- D: interior counts --------------------------------------------------------
// count the interior words of every real draw per emit block (real draws never
// overlap, so the counts are exact) and record, for every block a draw enters
// from an earlier block, how many of its leading positions it covers (`spill`;
// the emit kernel marks the rest of its block's interior words itself)
__global__ void rp_mark(const uint32_t* __restrict__ E, const uint32_t* __restrict__ len,
                        const uint8_t* __restrict__ real, const uint32_t* __restrict__ pm,
                        uint64_t L, uint32_t* __restrict__ block_int,
                        uint32_t* __restrict__ spill) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *pm || !real[i]) return;
  const uint64_t p = E[i];
  const uint64_t stop = len[i] == kIncomplete ? L : std::min<uint64_t>(p + len[i], L);
  for (uint64_t q = p + 1; q < stop;) {
    const uint64_t b = q / kRB, e = std::min<uint64_t>(stop, (b + 1) * kRB);
    atomicAdd(block_int + b, (uint32_t)(e - q));
    if (q == b * kRB) spill[b] = (uint32_t)(e - q);  // entered from an earlier block
    q = e;
  }
}

// Stages C and D in one CTA for short exceptional lists (m <= kSmallResolve,
// e.g. config 1's ~17 k): the reach prefix-max, heads, cluster walks and
// interior counts without four launches and two scans.  Also zeroes the
// per-block counts it accumulates into.
constexpr uint32_t kSmallResolve = 1u << 17;
__global__ void __launch_bounds__(1024)
    rp_resolve_small(const uint32_t* __restrict__ E, const uint32_t* __restrict__ len,
                     const uint32_t* __restrict__ pm, uint64_t L, uint8_t* __restrict__ real,
                     uint32_t* __restrict__ block_int, uint32_t* __restrict__ spill, uint32_t nb) {
  __shared__ uint64_t wb[32];
  __shared__ uint32_t headbits[kSmallResolve / 32];
  const uint32_t m = min(*pm, kSmallResolve);
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
    block_int[b] = 0;
    spill[b] = 0;
  }
  for (uint32_t w = threadIdx.x; w < (m + 31) / 32; w += blockDim.x) headbits[w] = 0;
  const uint32_t per = (m + blockDim.x - 1) / blockDim.x;
  const uint32_t beg = min(m, threadIdx.x * per), end = min(m, beg + per);
  uint64_t mx = 0;
  for (uint32_t i = beg; i < end; ++i) mx = max(mx, reach_of(E, len, i));
  // (block_exclusive synchronises, so the zeroing above is complete after it)
  uint64_t run = block_exclusive<uint64_t>(mx, 0ull, Max(), wb, nullptr);
  for (uint32_t i = beg; i < end; ++i) {  // heads: not covered by an earlier candidate
    if (run <= E[i]) atomicOr(&headbits[i >> 5], 1u << (i & 31));
    run = max(run, reach_of(E, len, i));
  }
  __syncthreads();
  auto head = [&](uint32_t i) { return (headbits[i >> 5] >> (i & 31)) & 1u; };
  // walks: a thread walks every cluster whose head lies in its range, into the
  // next thread's range if the cluster runs on
  {
    uint32_t i = beg;
    while (i < end && !head(i)) ++i;  // leading non-heads belong to an earlier walker
    // (a range without a head starts no walk: stepping on from `end` with an
    // empty cursor would race the earlier walker's flags with wrong ones)
    const bool walks = i < end;
    uint64_t cursor = 0;
    for (; walks && i < m && (i < end || !head(i)); ++i) {
      const uint8_t r = E[i] >= cursor;
      real[i] = r;
      if (r) cursor = reach_of(E, len, i);
    }
  }
  __syncthreads();
  for (uint32_t i = beg; i < end; ++i) {  // interior counts per emit block (rp_mark)
    if (!real[i]) continue;
    const uint64_t p = E[i];
    const uint64_t stop = len[i] == kIncomplete ? L : std::min<uint64_t>(p + len[i], L);
    for (uint64_t q = p + 1; q < stop;) {
      const uint64_t b = q / kRB, e = std::min<uint64_t>(stop, (b + 1) * kRB);
      atomicAdd(block_int + b, (uint32_t)(e - q));
      if (q == b * kRB) spill[b] = (uint32_t)(e - q);
      q = e;
    }
  }
}

// start positions per emit block = block length - interior words
__global__ void rp_block_starts(const uint32_t* __restrict__ block_int, uint32_t nb, uint64_t L,
                                uint32_t* __restrict__ starts) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const uint64_t len = std::min<uint64_t>(L, (uint64_t)(b + 1) * kRB) - (uint64_t)b * kRB;
  starts[b] = (uint32_t)(len - block_int[b]);
}


// ---- E: emit -------------------------------------------------------------------------
struct EmitArgs {
  const uint32_t* E;             // exceptional positions (sorted)
  const uint8_t* real;           // real[i]: E[i] starts a draw
  const uint32_t* pm;            // m (device)
  const uint32_t* spill;         // leading positions of a block covered by an earlier draw
  uint32_t nseg;                 // boff_exc entries (segments or blocks)
  const uint32_t* boff_exc;
  const uint32_t* boff_start;
  const uint32_t* len;
  const double* val;
  const uint32_t* meta;
  const uint32_t* cnt;
  uint64_t n;
  zf_path_rec* recs;
  unsigned long long* counters;  // internal [6]
  unsigned long long* consumed;  // internal scalar: words consumed + 1 (0: n not reached)
  uint32_t boff_stride;          // boff_exc entries per emit block (1, or 2 with segments)
};

#ifndef ZF_EMIT_MINB
#define ZF_EMIT_MINB 8  // 32 registers (a few bytes of stack): occupancy hides the load latency
#endif
// FULL = false: plain fills (no path records, no counters) -- the default
// oracle-mode call; its per-position code keeps no counter or record state.
// Positions are 32-bit (windows are < 2^32 positions, run_generated/replay_typed).
template <int DIST, typename OutT, bool FULL>
__global__ void __launch_bounds__(kRT, FULL ? 4 : ZF_EMIT_MINB)
    rp_emit(const DevTables* __restrict__ gt, Window win, EmitArgs a, OutT* __restrict__ out) {
  __shared__ uint2 wb[kRT / 32];
  const DevPack* P = primary_pack<DIST>(gt);
  const double* sx = P->sx;  // 2 KB, L1-resident: no per-block staging barrier
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t L32 = (uint32_t)win.L;
  const uint32_t p0 = (uint32_t)striped_pos(0);  // this thread's item j is p0 + 32 j
  // the block's offsets do not depend on the words: in flight with them
  const uint32_t boff_e = __ldg(a.boff_exc + (uint64_t)blockIdx.x * a.boff_stride);
  const uint32_t boff_s = __ldg(a.boff_start + blockIdx.x);
  const uint64_t nxt = (uint64_t)(blockIdx.x + 1) * a.boff_stride;
  // (m may be clamped to the bound the arrays were sized for: that pass is
  // flagged and redone, so entries past it are only ever skipped here)
  const uint32_t m = __ldg(a.pm);
  const uint32_t e_end = min(nxt < a.nseg ? __ldg(a.boff_exc + nxt) : m, m);
  const uint32_t spill = __ldg(a.spill + blockIdx.x);
  // this thread's first entry of the block's slice, in flight with the words
  const uint32_t i0 = boff_e + threadIdx.x;
  const bool has0 = i0 < e_end;
  const uint8_t real0 = has0 ? __ldg(a.real + i0) : 0;
  const uint32_t p_0 = has0 ? __ldg(a.E + i0) : 0, l_0 = has0 ? __ldg(a.len + i0) : 0;
  uint64_t wds[kRI];
  load_striped(win, wds);
  // interior words of this block as a 2048-bit map: the real draws that start
  // in it (its slice of E) and the one an earlier block's draw spills in
  __shared__ uint32_t imap[kRB / 32];
  const uint32_t b0 = blockIdx.x * (uint32_t)kRB;
  if (threadIdx.x < kRB / 32) {
    const uint32_t lo = threadIdx.x * 32u;  // word w covers positions b0 + [32w, 32w + 32)
    imap[threadIdx.x] = spill >= lo + 32u ? 0xFFFFFFFFu : spill > lo ? (1u << (spill - lo)) - 1u : 0u;
  }
  __syncthreads();
  for (uint32_t i = i0; i < e_end; i += kRT) {
    const bool first = i == i0;
    if (!(first ? real0 : __ldg(a.real + i))) continue;
    const uint32_t p = first ? p_0 : __ldg(a.E + i), l = first ? l_0 : __ldg(a.len + i);
    const uint32_t stop = l == kIncomplete ? L32 : min(p + l, L32);
    for (uint32_t q = p + 1 - b0, qe = min(stop - b0, (uint32_t)kRB); q < qe;) {
      // the run [q, qe) word by word
      const uint32_t w = q >> 5, hi = min(qe, (w + 1) * 32u);
      const uint32_t bits = (hi - q == 32 ? 0xFFFFFFFFu : ((1u << (hi - q)) - 1u)) << (q & 31);
      atomicOr(&imap[w], bits);
      q = hi;
    }
  }
  __syncthreads();
  // item j of this warp is the 32 positions of bitmap word wid * kRI + j (lane
  // = bit), so the warp's start ballot is that word complemented: one
  // broadcast LDS per item, no per-lane bit extraction
  const uint32_t wid = threadIdx.x >> 5;
  const uint32_t pw0 = b0 + wid * (uint32_t)kWarpSpan;
  // (the start ballot is re-read in the emit loop rather than kept: the plain
  // kernel runs at 32 registers)
  auto start_bits = [&](int j) -> uint32_t {
    const uint32_t pw = pw0 + 32u * j;  // first position of the item's 32
    // in-window lanes: the low min(L - pw, 32) bits, branch-free
    const uint32_t dd = pw >= L32 ? 0u : min(L32 - pw, 32u);
    return ~imap[wid * kRI + j] & __funnelshift_lc(0xFFFFFFFFu, 0u, dd);
  };
  uint32_t be[kRI];
  uint32_t ce = 0, cs = 0;
  [[maybe_unused]] const uint32_t lmx = (uint32_t)P->lmax;
#pragma unroll
  for (int j = 0; j < kRI; ++j) {
    const bool in = pw0 + 32u * j + lane < L32;
    bool exc;
    if constexpr (kTrad<DIST>)
      exc = exc_word<DIST>(*P, wds[j]);
    else
      exc = ((uint32_t)wds[j] & 0xFFu) >= lmx;
    be[j] = __ballot_sync(0xffffffffu, in && exc);
    ce += __popc(be[j]);
    cs += __popc(start_bits(j));
  }
  uint32_t eidx, rank;
  warp_base2(ce, cs, wb, &eidx, &rank);
  eidx += boff_e;
  rank += boff_s;
  const uint32_t n32 = (uint32_t)a.n;  // n < 2^31
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < kRI; ++j) {
    const uint32_t bs = start_bits(j);
    const bool is_ex = (be[j] >> lane) & 1, is_st = (bs >> lane) & 1;
    const uint32_t e_i = eidx + __popc(be[j] & lt), r_i = rank + __popc(bs & lt);
    if (is_st && r_i < n32 && !(is_ex && e_i >= m)) {
      const uint32_t p = p0 + 32u * j;
      double v;
      uint32_t nw = 1;
      if (is_ex) {
        nw = a.len[e_i];
        v = a.val[e_i];
      } else {
        v = __dmul_rn(kSigned<DIST> ? __ll2double_rn((long long)wds[j])
                                    : __ull2double_rn(wds[j]),
                      __ldg(sx + (wds[j] & 0xFF) + 1));
      }
      if (nw != kIncomplete) {
        out[r_i] = to_out<OutT>(v);
        if constexpr (FULL) {
          uint32_t meta;
          if (is_ex) {
            meta = a.meta[e_i];
            if (a.counters)
              for (int q = 0; q < 6; ++q) c[q] += a.cnt[(uint64_t)e_i * 6 + q];
          } else {
            meta = ((uint32_t)wds[j] & 0xFF) | (ZF_PATH_FAST << 8);
            c[0] += 1;
            c[1] += 1;
          }
          if (a.recs) {
            zf_path_rec r;
            r.start = p;
            r.nwords = nw;
            r.layer = (uint8_t)(meta & 0xFF);
            r.path = (uint8_t)((meta >> 8) & 0xFF);
            r.attempts = (uint16_t)(meta >> 16);
            a.recs[r_i] = r;
          }
        }
        if (r_i + 1 == n32) *a.consumed = (unsigned long long)p + nw + 1;  // 0: not reached
      }
    }
    eidx += __popc(be[j]);
    rank += __popc(bs);
  }
  if (FULL && a.counters) {  // counted fills only: 6 atomics per warp on 6 addresses
    for (int q = 0; q < 6; ++q) {
      unsigned long long v = c[q];
      for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
      if ((threadIdx.x & 31) == 0 && v) atomicAdd(a.counters + q, v);
    }
  }
}

__global__ void add_counters(const unsigned long long* __restrict__ src,
                             unsigned long long* __restrict__ dst) {
  if (threadIdx.x < 6) dst[threadIdx.x] += src[threadIdx.x];
}

// ---- word generation ---------------------------------------------------------------
// CTR = false: splitmix64 words (gid 1); true: the production counter stream's
// primary words ctr_word(seed + (K + 1) * gamma)
template <bool CTR>
__global__ void words_weyl(uint64_t state, uint64_t n, uint64_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = CTR ? ctr_word(state + (i + 1) * kGamma) : mix13(state + (i + 1) * kGamma);
}

__device__ __forceinline__ void xo_step(uint64_t s[4]) {
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
}

#ifndef ZF_XO_BLOCK
#define ZF_XO_BLOCK 1024
#endif
// block parents for the device xoshiro jump (xo_jump_block)
#ifndef ZF_XO_PARENT
#define ZF_XO_PARENT 1
#endif
constexpr int kXoBlock = ZF_XO_BLOCK;  // words per thread
constexpr int kXoBits = 8;      // jump-table radix 256: <= 3 polynomials for 2^24 threads
constexpr int kXoRadix = 1 << kXoBits;
constexpr int kXoLevels = 5;    // base-256 digits of the thread index (2^40 threads)

// Short windows use 64-word blocks: 16x the threads, so the per-thread jump
// (a latency-bound chain of up to 3 x 256 generator steps) and the sequential
// block walk both shrink -- 1.1 M words took 46 us with 1024-word blocks.
constexpr int kXoBlockShort = 64;
constexpr uint64_t kXoShortMax = 1ull << 22;  // windows up to this many words

// the jump table for blocks of B words, built once per B on the host and kept
// on every device that used it (40 KB each)
const uint64_t* jump_table_device(int B = kXoBlock) {
  static std::mutex mu;
  static std::vector<uint64_t> host[2];
  static std::vector<uint64_t*> per_device[2] = {std::vector<uint64_t*>(64, nullptr),
                                                 std::vector<uint64_t*>(64, nullptr)};
  const int which = B == kXoBlock ? 0 : 1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (host[which].empty()) {
    host[which].assign((size_t)kXoLevels * (kXoRadix - 1) * 4, 0);
    xoshiro_radix_polys((uint64_t)B, kXoBits, kXoLevels, host[which].data());
  }
  if (!per_device[which][dev]) {
    uint64_t* d = nullptr;
    const size_t bytes = host[which].size() * sizeof(uint64_t);
    if (cudaMalloc(&d, bytes) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, host[which].data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(d);
      return nullptr;
    }
    per_device[which][dev] = d;
  }
  return per_device[which][dev];
}


// state <- (poly)(T) state: 256 generator steps, the xor of the states at the
// poly's set coefficients (branch-free, so lanes with different polys stay
// converged)
__device__ __forceinline__ void xo_apply(const unsigned long long* __restrict__ poly,
                                         uint64_t s[4]) {
  uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll 1
  for (int w = 0; w < 4; ++w) {
    uint64_t bits = __ldg(poly + w);
#pragma unroll 8
    for (int b = 0; b < 64; ++b) {
      const uint64_t m = 0ull - (bits & 1);
      acc[0] ^= s[0] & m;
      acc[1] ^= s[1] & m;
      acc[2] ^= s[2] & m;
      acc[3] ^= s[3] & m;
      bits >>= 1;
      xo_step(s);
    }
  }
  s[0] = acc[0];
  s[1] = acc[1];
  s[2] = acc[2];
  s[3] = acc[3];
}

// start state of thread t's block: s0 jumped by t * kXoBlock words
__device__ __forceinline__ void xo_jump_to(const uint64_t* __restrict__ table, uint64_t t,
                                           uint64_t s[4], int first_level = 0) {
  const unsigned long long* pp = reinterpret_cast<const unsigned long long*>(table);
  for (int r = first_level; r < kXoLevels && (t >> (kXoBits * r)) != 0; ++r) {
    const int d = (int)((t >> (kXoBits * r)) & (kXoRadix - 1));
    if (d) xo_apply(pp + ((size_t)r * (kXoRadix - 1) + d - 1) * 4, s);
  }
}

// The same for every thread of a block of consecutive t (blockDim.x divides
// 256): thread 0 jumps to the block's parent (t with its base-256 digit 0
// cleared, all higher digits) and shares it; every thread then applies only its
// own digit 0 -- one polynomial application per thread instead of one per
// nonzero digit (2-3 for windows of 2^26 words).  Includes a __syncthreads.
__device__ __forceinline__ void xo_jump_block(const uint64_t* __restrict__ table, uint64_t t,
                                              ulonglong4 s0, uint64_t s[4]) {
  __shared__ uint64_t parent[4];
  if (threadIdx.x == 0) {
    uint64_t p[4] = {s0.x, s0.y, s0.z, s0.w};
    xo_jump_to(table, t & ~(uint64_t)(kXoRadix - 1), p, 1);
    parent[0] = p[0];
    parent[1] = p[1];
    parent[2] = p[2];
    parent[3] = p[3];
  }
  __syncthreads();
  s[0] = parent[0];
  s[1] = parent[1];
  s[2] = parent[2];
  s[3] = parent[3];
  const int d = (int)(t & (kXoRadix - 1));
  if (d) xo_apply(reinterpret_cast<const unsigned long long*>(table) + (size_t)(d - 1) * 4, s);
}

// thread t owns words [t*B, (t+1)*B): start state = T^(t*B) s0, one jump
// polynomial x^(d*256^r*B) per nonzero base-256 digit d of t; output staged
// through a 32x32 smem tile per warp so stores are coalesced rows.
template <int B>
__global__ void __launch_bounds__(128)
    words_xoshiro(ulonglong4 s0, const uint64_t* __restrict__ polys, uint64_t n,
                  uint64_t* __restrict__ out) {
  __shared__ uint64_t tile[4][32][33];
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t s[4] = {s0.x, s0.y, s0.z, s0.w};
#if ZF_XO_PARENT
  xo_jump_block(polys, t, s0, s);
#else
  xo_jump_to(polys, t, s);
#endif
  const uint64_t warp_first = t - lane;  // thread index of lane 0
  for (int c = 0; c < B; c += 32) {
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      tile[wid][lane][j] = ((s[0] + s[3]) << 23 | (s[0] + s[3]) >> 41) + s[0];
      xo_step(s);
    }
    __syncwarp();
    for (int r = 0; r < 32; ++r) {  // row r = lane r's 32 consecutive words
      const uint64_t idx = (warp_first + r) * B + c + lane;
      if (idx < n) out[idx] = tile[wid][r][lane];
    }
    __syncwarp();
  }
}

// ---- generated windows: words + classification in one pass ----------------------
// For the reference's own generators (gid 0/1) the window is produced on the
// device anyway; the kernel that writes it also flags the exceptional words of
// each thread's 1024-word segment into per-segment slots, so the replay
// pipeline skips its two classification passes over the window.

struct XoGen {
  uint64_t s[4];
  __device__ __forceinline__ uint64_t next() {
    const uint64_t r = ((s[0] + s[3]) << 23 | (s[0] + s[3]) >> 41) + s[0];
    xo_step(s);
    return r;
  }
};
struct SmGen {
  uint64_t st;
  __device__ __forceinline__ uint64_t next() {
    st += kGamma;
    return mix13(st);
  }
};

constexpr int kClsCap = 64;  // exceptional slots per segment (expected ~16)
static_assert(kRB % kXoBlock == 0, "emit blocks cover whole segments");

template <int DIST, int GID>
__global__ void __launch_bounds__(128)
    words_cls(ulonglong4 s0, const uint64_t* __restrict__ polys, uint64_t n,
              uint64_t* __restrict__ out, const DevPack* __restrict__ P,
              uint32_t* __restrict__ slots, uint32_t* __restrict__ slot_cnt,
              unsigned int* __restrict__ overflow) {
  __shared__ uint64_t tile[4][32][33];
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  using G = typename std::conditional<GID == ZF_GEN_XOSHIRO256PP, XoGen, SmGen>::type;
  G g;
  if constexpr (GID == ZF_GEN_XOSHIRO256PP) {
#if ZF_XO_PARENT
    xo_jump_block(polys, t, s0, g.s);
#else
    g = XoGen{{s0.x, s0.y, s0.z, s0.w}};
    xo_jump_to(polys, t, g.s);
#endif
  } else {
    g = SmGen{s0.x + t * (uint64_t)kXoBlock * kGamma};
  }
  const uint64_t warp_first = t - lane;
  const uint64_t p0 = t * kXoBlock;
  const uint32_t lmax = (uint32_t)__ldg(&P->lmax);  // hoisted: one load per thread
  uint32_t* const my_slots = slots + t * kClsCap;
  uint32_t k = 0;
  auto exc_of = [&](uint64_t w) -> bool {
    return kTrad<DIST> ? exc_word<DIST>(*P, w) : ((uint32_t)w & 0xFFu) >= lmax;
  };
  if ((warp_first + 32) * kXoBlock <= n) {
    // the whole warp's segments lie inside the window (every warp but the
    // last): no per-word bounds, the slot store predicated (an overflowing
    // segment keeps writing its last slot; the flag below reports it)
    for (int c = 0; c < kXoBlock; c += 32) {
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const uint64_t w = g.next();
        tile[wid][lane][j] = w;
        if (exc_of(w)) my_slots[min(k, (uint32_t)kClsCap - 1)] = (uint32_t)(p0 + c + j);
        k += exc_of(w);
      }
      __syncwarp();
      uint64_t* o = out + warp_first * kXoBlock + c + lane;
#pragma unroll 8
      for (int r = 0; r < 32; ++r) o[(uint64_t)r * kXoBlock] = tile[wid][r][lane];
      __syncwarp();
    }
  } else {
    for (int c = 0; c < kXoBlock; c += 32) {
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        const uint64_t w = g.next();
        tile[wid][lane][j] = w;
        const uint64_t p = p0 + c + j;
        if (exc_of(w) && p < n) {
          if (k < kClsCap) my_slots[k] = (uint32_t)p;
          ++k;
        }
      }
      __syncwarp();
      for (int r = 0; r < 32; ++r) {
        const uint64_t idx = (warp_first + r) * kXoBlock + c + lane;
        if (idx < n) out[idx] = tile[wid][r][lane];
      }
      __syncwarp();
    }
  }
  if (p0 < n) {
    slot_cnt[t] = k < kClsCap ? k : kClsCap;
    if (k > kClsCap) atomicOr(overflow, 1u);
  }
}

__global__ void cls_compact(const uint32_t* __restrict__ slot_cnt, const uint32_t* __restrict__ coff,
                            uint64_t T, const uint32_t* __restrict__ slots,
                            uint32_t* __restrict__ E, uint32_t cap) {
  const uint64_t slot = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t t = slot / kClsCap, k = slot % kClsCap;
  if (t < T && k < slot_cnt[t] && coff[t] + k < cap) E[coff[t] + k] = slots[slot];
}

// m above the bound the host sized the exceptional arrays for: clamp it (the
// window is redone with exact sizes) and flag it
__global__ void clamp_m(uint32_t* __restrict__ pm, uint32_t cap, unsigned int* __restrict__ flags) {
  if (*pm > cap) {
    *pm = cap;
    atomicOr(flags, 2u);
  }
}

// the segment-slot overflow of words_cls as a flag of this window
__global__ void copy_flag(const unsigned int* __restrict__ src, unsigned int* __restrict__ flags) {
  if (*src) atomicOr(flags, 1u);
}

// pre-classified window (words_cls): slots per segment + overflow flag
struct PreClass {
  const uint32_t* slots;
  const uint32_t* slot_cnt;
  uint64_t T;
  const unsigned int* overflow;
};

// ZF_DEBUG=1: synchronise and report after every pipeline stage (stderr)
static bool debug_on() {
  static const bool on = getenv("ZF_DEBUG") != nullptr;
  return on;
}
static void dbg(const char* what, cudaStream_t s) {
  if (!debug_on()) return;
  static auto last = std::chrono::steady_clock::now();
  cudaError_t e = cudaStreamSynchronize(s);
  const auto now = std::chrono::steady_clock::now();
  fprintf(stderr, "[zf] %-16s %-10s %8.3f ms\n", what, cudaGetErrorString(e),
          std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

struct Workspace {
  std::vector<void*> ptrs;
  cudaStream_t s;
  explicit Workspace(cudaStream_t st) : s(st) {}
  template <typename T>
  cudaError_t alloc(T** p, uint64_t count) {
    void* v = nullptr;
    cudaError_t e = cudaMallocAsync(&v, std::max<uint64_t>(count, 1) * sizeof(T), s);
    if (e == cudaSuccess) ptrs.push_back(v);
    *p = static_cast<T*>(v);
    return e;
  }
  ~Workspace() {
    for (void* p : ptrs) cudaFreeAsync(p, s);
  }
};

// exclusive device scan (CUB) of n entries; *total (device, nullable) gets the
// reduction of all n (= out[n-1] op in[n-1])
template <typename T>
__global__ void scan_total(const T* __restrict__ in, const T* __restrict__ out, uint64_t n,
                           bool max_op, T* __restrict__ total) {
  const T a = out[n - 1], b = in[n - 1];
  *total = max_op ? (a > b ? a : b) : a + b;
}

template <typename T, class Op>
int device_scan(Workspace& ws, const T* in, T* out, uint64_t n, Op op, T init, T* total,
                cudaStream_t s) {
  if (n == 0) return ZF_OK;
  size_t bytes = 0;
  ZF_TRY(cub::DeviceScan::ExclusiveScan(nullptr, bytes, in, out, op, init, (int64_t)n, s));
  unsigned char* tmp = nullptr;
  ZF_TRY(ws.alloc(&tmp, bytes));
  ZF_TRY(cub::DeviceScan::ExclusiveScan(tmp, bytes, in, out, op, init, (int64_t)n, s));
  if (total) scan_total<T><<<1, 1, 0, s>>>(in, out, n, std::is_same<Op, Max>::value, total);
  return cuda_status(cudaGetLastError());
}

// One window.  Normally no host synchronisation until the end: the exceptional
// arrays are sized for a bound on their count m (random streams have ~1.6 % of
// positions exceptional, the bound is 6.25 % + 4096) and every kernel reads m
// from the device.  A window whose m exceeds the bound, or whose generator
// segments overflowed their slots, is flagged and redone with exact sizes
// (`exact`: one synchronisation to read m).
// Exclusive scan of a short array (<= kSmallScan entries) by one 1024-thread
// block: one launch where CUB takes two plus a total kernel.  Fused extras:
// STARTS -- the input is the per-block interior count and the scanned value
// is the block's start count (block length - interior words); the total is
// written to *total, and if cap != 0 clamped to cap with flag bit 2.
constexpr uint32_t kSmallScan = 1u << 13;  // one SM: longer arrays go to CUB
template <typename T, class Op, bool STARTS>
__global__ void __launch_bounds__(1024)
    scan_small(const T* __restrict__ in, T* __restrict__ out, uint32_t n, T init, Op op,
               T* __restrict__ total, uint32_t cap, unsigned int* __restrict__ flags, uint64_t L) {
  __shared__ T wb[32];
  const uint32_t per = (n + 1023) / 1024;
  const uint32_t b = threadIdx.x * per, e = min(n, b + per);
  auto val = [&](uint32_t i) -> T {
    if constexpr (STARTS) {
      const uint64_t len = std::min<uint64_t>(L, (uint64_t)(i + 1) * kRB) - (uint64_t)i * kRB;
      return (T)(len - in[i]);
    } else {
      return in[i];
    }
  };
  T loc = init;
  for (uint32_t i = b; i < e; ++i) loc = op(loc, val(i));
  T tot;
  T run = op(init, block_exclusive<T>(loc, init, op, wb, &tot));
  for (uint32_t i = b; i < e; ++i) {
    const T v = val(i);
    out[i] = run;
    run = op(run, v);
  }
  if (threadIdx.x == 0 && total) {
    T t = op(init, tot);
    if (cap && t > (T)cap) {
      t = (T)cap;
      atomicOr(flags, 2u);
    }
    *total = t;
  }
}

// exclusive scan of n entries, reduction into *total (nullable); cap != 0
// clamps the total (flag bit 2), STARTS as in scan_small
template <typename T, class Op, bool STARTS = false>
int scan_n(Workspace& ws, const T* in, T* out, uint64_t n, Op op, T init, T* total,
           cudaStream_t s, uint32_t cap = 0, unsigned int* flags = nullptr, uint64_t L = 0,
           T* tmp_in = nullptr) {
  if (n == 0) return ZF_OK;
  if (n <= kSmallScan) {
    scan_small<T, Op, STARTS><<<1, 1024, 0, s>>>(in, out, (uint32_t)n, init, op, total, cap,
                                                  flags, L);
    return cuda_status(cudaGetLastError());
  }
  const T* src = in;
  if constexpr (STARTS) {  // large windows: the start counts first, then CUB
    rp_block_starts<<<(uint32_t)((n + 255) / 256), 256, 0, s>>>(in, (uint32_t)n, L, tmp_in);
    src = tmp_in;
  }
  ZF_TRY_STATUS(device_scan<T>(ws, src, out, n, op, init, total, s));
  if (cap) clamp_m<<<1, 1, 0, s>>>(reinterpret_cast<uint32_t*>(total), cap, flags);
  return cuda_status(cudaGetLastError());
}

template <int DIST, typename OutT>
int replay_window(const zf_tables* t, const Window& win, void* out, uint64_t n, zf_path_rec* recs,
                  int64_t* counters, uint64_t* consumed_host, bool* retry, cudaStream_t s,
                  const PreClass* pre = nullptr, bool exact = false) {
  *retry = false;
  if (debug_on()) fprintf(stderr, "[zf] replay_window L=%llu nwords=%llu cursor=%llu n=%llu%s\n",
                          (unsigned long long)win.L, (unsigned long long)win.nwords,
                          (unsigned long long)win.cursor, (unsigned long long)n,
                          exact ? " (exact)" : "");
  const DevPack* dP = primary_pack<DIST>(t->dev);  // device address
  const uint64_t L = win.L;
  const uint32_t nb = (uint32_t)((L + kRB - 1) / kRB);
  Workspace ws(s);
  uint32_t *bcnt, *boff, *E, *bcnt2, *boff2, *spill;
  // [0] exceptional count m (u32), [1] flags (u32) | [2] consumed, [3..8] counters
  unsigned long long* scal;
  ZF_TRY(ws.alloc(&bcnt, nb));
  ZF_TRY(ws.alloc(&spill, nb));
  ZF_TRY(ws.alloc(&boff, nb));
  ZF_TRY(ws.alloc(&bcnt2, nb));
  ZF_TRY(ws.alloc(&boff2, nb));
  ZF_TRY(ws.alloc(&scal, 16));
  uint32_t* dm = reinterpret_cast<uint32_t*>(scal);
  unsigned int* dflags = reinterpret_cast<unsigned int*>(scal) + 1;
  ZF_TRY(cudaMemsetAsync(scal, 0, 16 * sizeof(unsigned long long), s));
  // exceptional positions: from the generator's slots, or two passes here
  uint32_t* coff = nullptr;
  const bool use_pre = pre != nullptr && !exact;
  const uint32_t boff_stride = use_pre ? (uint32_t)(kRB / kXoBlock) : 1u;
  // the bound the exceptional arrays are sized for (exact: m itself)
  uint32_t cap = exact ? 0u : (uint32_t)std::min<uint64_t>(L, L / 16 + 4096);
  if (use_pre) {
    ZF_TRY(ws.alloc(&coff, pre->T));
    ZF_TRY_STATUS(scan_n<uint32_t>(ws, pre->slot_cnt, coff, pre->T, Add(), 0u, dm, s, cap, dflags));
    copy_flag<<<1, 1, 0, s>>>(pre->overflow, dflags);
  } else {
    rp_count_exc<DIST><<<nb, kRT, 0, s>>>(win, dP, bcnt);
    dbg("rp_count_exc", s);
    ZF_TRY_STATUS(scan_n<uint32_t>(ws, bcnt, boff, nb, Add(), 0u, dm, s, cap, dflags));
    dbg("scan_exc", s);
  }
  if (exact) {
    ZF_TRY(cudaMemcpyAsync(&cap, dm, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    ZF_TRY(cudaStreamSynchronize(s));
  }
  ExcOut eo;
  uint8_t *head, *real;
  uint64_t *bmax, *bpre;
  const uint32_t nbE = (cap + kRB - 1) / kRB;
  ZF_TRY(ws.alloc(&E, cap));
  ZF_TRY(ws.alloc(&eo.len, cap));
  ZF_TRY(ws.alloc(&eo.val, cap));
  ZF_TRY(ws.alloc(&eo.meta, cap));
  ZF_TRY(ws.alloc(&eo.cnt, (uint64_t)cap * 6));
  ZF_TRY(ws.alloc(&head, cap));
  ZF_TRY(ws.alloc(&real, cap));
  ZF_TRY(ws.alloc(&bmax, nbE));
  ZF_TRY(ws.alloc(&bpre, nbE));
  if (use_pre) {
    const uint64_t slots = pre->T * kClsCap;
    cls_compact<<<(uint32_t)((slots + 255) / 256), 256, 0, s>>>(pre->slot_cnt, coff, pre->T,
                                                                pre->slots, E, cap);
  } else {
    rp_compact_exc<DIST><<<nb, kRT, 0, s>>>(win, dP, boff, E, cap);
  }
  dbg("compact", s);
  const bool small_resolve = cap <= kSmallResolve;
  if (cap) {
    constexpr int kPacks = kPacksOf<DIST>;
    const size_t smem = kPacks * sizeof(DevPack);
    ZF_TRY(cudaFuncSetAttribute(rp_draw_exc<DIST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
    rp_draw_exc<DIST><<<(cap + kRT - 1) / kRT, kRT, smem, s>>>(t->dev, win, E, dm, eo);
    dbg("rp_draw_exc<DIST>", s);
  }
  if (small_resolve) {
    rp_resolve_small<<<1, 1024, 0, s>>>(E, eo.len, dm, L, real, bcnt, spill, nb);
    dbg("rp_resolve_small", s);
  } else {
    rp_reach_max<<<nbE, kRT, 0, s>>>(E, eo.len, dm, bmax);
    dbg("rp_reach_max", s);
    ZF_TRY_STATUS(scan_n<uint64_t>(ws, bmax, bpre, nbE, Max(), 0ull, nullptr, s));
    rp_heads<<<nbE, kRT, 0, s>>>(E, eo.len, dm, bpre, head);
    dbg("rp_heads", s);
    // (rp_walk writes real[i] for every i < m: entry 0 is always a head)
    const uint64_t walkers = (cap + kWalkChunk - 1) / kWalkChunk;
    rp_walk<<<(uint32_t)((walkers + kRT - 1) / kRT), kRT, 0, s>>>(E, eo.len, head, dm, real);
    dbg("rp_walk", s);
    ZF_TRY(cudaMemsetAsync(bcnt, 0, nb * sizeof(uint32_t), s));  // reused: interior per block
    ZF_TRY(cudaMemsetAsync(spill, 0, nb * sizeof(uint32_t), s));
    rp_mark<<<(cap + kRT - 1) / kRT, kRT, 0, s>>>(E, eo.len, real, dm, L, bcnt, spill);
    dbg("rp_mark", s);
  }
  ZF_TRY_STATUS((scan_n<uint32_t, Add, true>(ws, bcnt, boff2, nb, Add(), 0u, nullptr, s, 0,
                                             nullptr, L, bcnt2)));
  dbg("block starts", s);
  EmitArgs a{E, real, dm, spill, use_pre ? (uint32_t)pre->T : nb, use_pre ? coff : boff, boff2,
             eo.len, eo.val, eo.meta, eo.cnt, n, recs, counters ? scal + 3 : nullptr, scal + 2,
             boff_stride};
  if (recs || counters)
    rp_emit<DIST, OutT, true><<<nb, kRT, 0, s>>>(t->dev, win, a, static_cast<OutT*>(out));
  else
    rp_emit<DIST, OutT, false><<<nb, kRT, 0, s>>>(t->dev, win, a, static_cast<OutT*>(out));
  dbg("rp_emit", s);
  ZF_TRY(cudaGetLastError());
  unsigned long long res[3] = {0, 0, 0};  // m | flags, consumed
  ZF_TRY(cudaMemcpyAsync(res, scal, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  ZF_TRY(cudaStreamSynchronize(s));
  if (res[0] >> 32) {
    // a segment overflowed its slots or m exceeded the bound: the results of
    // this pass are void (the output is rewritten)
    if (exact) return ZF_ERANGE;  // (unreachable: exact passes set no flags)
    return replay_window<DIST, OutT>(t, win, out, n, recs, counters, consumed_host, retry, s, pre,
                                     true);
  }
  if (res[2] == 0) {  // the window holds fewer than n draws
    *retry = true;
    return ZF_OK;
  }
  const unsigned long long consumed = res[2] - 1;
  if (counters) add_counters<<<1, 32, 0, s>>>(scal + 3, reinterpret_cast<unsigned long long*>(counters));
  *consumed_host = consumed;
  return cuda_status(cudaGetLastError());
}

template <int DIST, typename OutT>
int replay_typed(const zf_tables* t, const uint64_t* words, uint64_t nwords, uint64_t cursor,
                 int wrap, void* out, uint64_t n, zf_path_rec* recs, int64_t* counters,
                 uint64_t* consumed, cudaStream_t s) {
  // A window of 2n + 2^20 words is never needed by a random stream (draws take
  // ~1.06 words on average); a replay list whose draws cycle forever (possible
  // with short wrapping lists -- the reference would loop without end) is
  // reported as ZF_ERANGE instead of growing the window towards 2^32.
  const uint64_t sane = 2 * n + (1ull << 20);
  const uint64_t cap = std::min<uint64_t>(
      sane, wrap ? (1ull << 32) - kRB : nwords - std::min(cursor, nwords));
  uint64_t L = std::min<uint64_t>(cap, n + n / 8 + 4096);
  for (;;) {
    if (L == 0) return ZF_ESHORT;
    Window win{words, nwords, wrap ? cursor % nwords : cursor, L};
    bool retry = false;
    ZF_TRY_STATUS((replay_window<DIST, OutT>(t, win, out, n, recs, counters, consumed, &retry, s)));
    if (!retry) return ZF_OK;
    if (L >= cap) return (wrap || cap == sane) ? ZF_ERANGE : ZF_ESHORT;
    L = std::min<uint64_t>(cap, 2 * L);
  }
}

// one window of L generated words (gid 0/1), classified while generated
template <int DIST, typename OutT>
int generated_window(const zf_tables* t, int gid, const uint64_t st[4], uint64_t L, void* out,
                     uint64_t n, zf_path_rec* recs, int64_t* counters, uint64_t* consumed,
                     cudaStream_t s) {
  Workspace ws(s);
  const uint64_t T = (L + kXoBlock - 1) / kXoBlock;
  uint64_t* words;
  uint32_t *slots, *slot_cnt;
  unsigned int* overflow;
  ZF_TRY(ws.alloc(&words, L));
  ZF_TRY(ws.alloc(&slots, T * kClsCap));
  ZF_TRY(ws.alloc(&slot_cnt, T));
  ZF_TRY(ws.alloc(&overflow, 1));
  ZF_TRY(cudaMemsetAsync(overflow, 0, sizeof(unsigned int), s));
  const uint64_t* dpolys = nullptr;
  if (gid == ZF_GEN_XOSHIRO256PP) {
    if (T - 1 >= (1ull << (kXoBits * kXoLevels))) return ZF_ERANGE;
    dpolys = jump_table_device();
    if (!dpolys) return ZF_EDEVICE;
  }
  const ulonglong4 s0 = make_ulonglong4(st[0], st[1], st[2], st[3]);
  const uint64_t blocks = (T + 127) / 128;
  const DevPack* dP = primary_pack<DIST>(t->dev);
  if (gid == ZF_GEN_XOSHIRO256PP)
    words_cls<DIST, ZF_GEN_XOSHIRO256PP><<<(uint32_t)blocks, 128, 0, s>>>(
        s0, dpolys, L, words, dP, slots, slot_cnt, overflow);
  else
    words_cls<DIST, ZF_GEN_SPLITMIX64><<<(uint32_t)blocks, 128, 0, s>>>(
        s0, dpolys, L, words, dP, slots, slot_cnt, overflow);
  ZF_TRY(cudaGetLastError());
  Window win{words, L, 0, L};
  PreClass pre{slots, slot_cnt, T, overflow};
  bool retry = false;
  ZF_TRY_STATUS((replay_window<DIST, OutT>(t, win, out, n, recs, counters, consumed, &retry, s,
                                           &pre)));
  return retry ? ZF_ESHORT : ZF_OK;
}

}  // namespace

int run_generated(const zf_tables* t, int dist, int dtype, int gid, const uint64_t st[4],
                  uint64_t L, void* out, uint64_t n, zf_path_rec* recs, int64_t* counters,
                  uint64_t* consumed, cudaStream_t s) {
  *consumed = 0;
  if (n == 0) return ZF_OK;
  if (!out) return ZF_EINVAL;
  if (n >= (1ull << 31) || L >= (1ull << 32) - kRB) return ZF_ERANGE;
  if (gid != ZF_GEN_XOSHIRO256PP && gid != ZF_GEN_SPLITMIX64) return ZF_EDIST;
  ZF_TRY_STATUS(check_kind(t, dist));
#define ZF_GEN(D, O) return generated_window<D, O>(t, gid, st, L, out, n, recs, counters, consumed, s)
  if (dist == ZF_EXP && dtype == ZF_F64) ZF_GEN(ZF_EXP, double);
  if (dist == ZF_EXP && dtype == ZF_F32) ZF_GEN(ZF_EXP, float);
  if (dist == ZF_NORMAL && dtype == ZF_F64) ZF_GEN(ZF_NORMAL, double);
  if (dist == ZF_NORMAL && dtype == ZF_F32) ZF_GEN(ZF_NORMAL, float);
  if (dist == ZF_TRAD_EXP && dtype == ZF_F64) ZF_GEN(ZF_TRAD_EXP, double);
  if (dist == ZF_TRAD_EXP && dtype == ZF_F32) ZF_GEN(ZF_TRAD_EXP, float);
  if (dist == ZF_TRAD_NORMAL && dtype == ZF_F64) ZF_GEN(ZF_TRAD_NORMAL, double);
  if (dist == ZF_TRAD_NORMAL && dtype == ZF_F32) ZF_GEN(ZF_TRAD_NORMAL, float);
#undef ZF_GEN
  return ZF_EDIST;
}

int run_replay(const zf_tables* t, int dist, int dtype, const uint64_t* words, uint64_t nwords,
               uint64_t cursor, int wrap, void* out, uint64_t n, zf_path_rec* recs,
               int64_t* counters, uint64_t* consumed, cudaStream_t s) {
  *consumed = 0;
  if (n == 0) return ZF_OK;
  if (!words || nwords == 0 || !out) return ZF_EINVAL;
  if (n >= (1ull << 31)) return ZF_ERANGE;
  ZF_TRY_STATUS(check_kind(t, dist));
  if (dist == ZF_EXP && dtype == ZF_F64)
    return replay_typed<ZF_EXP, double>(t, words, nwords, cursor, wrap, out, n, recs, counters,
                                        consumed, s);
  if (dist == ZF_EXP && dtype == ZF_F32)
    return replay_typed<ZF_EXP, float>(t, words, nwords, cursor, wrap, out, n, recs, counters,
                                       consumed, s);
  if (dist == ZF_NORMAL && dtype == ZF_F64)
    return replay_typed<ZF_NORMAL, double>(t, words, nwords, cursor, wrap, out, n, recs,
                                           counters, consumed, s);
  if (dist == ZF_NORMAL && dtype == ZF_F32)
    return replay_typed<ZF_NORMAL, float>(t, words, nwords, cursor, wrap, out, n, recs, counters,
                                          consumed, s);
  if (dist == ZF_TRAD_EXP && dtype == ZF_F64)
    return replay_typed<ZF_TRAD_EXP, double>(t, words, nwords, cursor, wrap, out, n, recs,
                                             counters, consumed, s);
  if (dist == ZF_TRAD_EXP && dtype == ZF_F32)
    return replay_typed<ZF_TRAD_EXP, float>(t, words, nwords, cursor, wrap, out, n, recs,
                                            counters, consumed, s);
  if (dist == ZF_TRAD_NORMAL && dtype == ZF_F64)
    return replay_typed<ZF_TRAD_NORMAL, double>(t, words, nwords, cursor, wrap, out, n, recs,
                                                counters, consumed, s);
  if (dist == ZF_TRAD_NORMAL && dtype == ZF_F32)
    return replay_typed<ZF_TRAD_NORMAL, float>(t, words, nwords, cursor, wrap, out, n, recs,
                                               counters, consumed, s);
  return ZF_EDIST;
}

int launch_words(int gid, const uint64_t* state, uint64_t n, uint64_t* out, cudaStream_t s) {
  if (n == 0) return ZF_OK;
  if (gid == ZF_GEN_SPLITMIX64 || gid == ZF_GEN_CTR) {
    // ctr words are the primary counter stream from sample position state[1]
    const uint64_t st = gid == ZF_GEN_CTR ? state[0] + state[1] * kGamma : state[0];
    const uint32_t grid = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    if (gid == ZF_GEN_CTR)
      words_weyl<true><<<grid, 256, 0, s>>>(st, n, out);
    else
      words_weyl<false><<<grid, 256, 0, s>>>(st, n, out);
    return cuda_status(cudaGetLastError());
  }
  if (gid != ZF_GEN_XOSHIRO256PP) return ZF_EDIST;
  const bool shrt = n <= kXoShortMax;
  const int B = shrt ? kXoBlockShort : kXoBlock;
  const uint64_t threads = (n + B - 1) / B;
  if (threads - 1 >= (1ull << (kXoBits * kXoLevels))) return ZF_ERANGE;
  const uint64_t* dpolys = jump_table_device(B);
  if (!dpolys) return ZF_EDEVICE;
  const ulonglong4 s0 = make_ulonglong4(state[0], state[1], state[2], state[3]);
  // round the grid to whole warps so every warp's smem tile is full
  const uint64_t blocks = (threads + 127) / 128;
  if (shrt)
    words_xoshiro<kXoBlockShort><<<(uint32_t)blocks, 128, 0, s>>>(s0, dpolys, n, out);
  else
    words_xoshiro<kXoBlock><<<(uint32_t)blocks, 128, 0, s>>>(s0, dpolys, n, out);
  return cuda_status(cudaGetLastError());
}

}  // namespace zf
