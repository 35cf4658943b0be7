// zf_device.cuh -- device-side building blocks shared by every sm_100a kernel.
//
// * splitmix64 word function (the reference's gid-1 generator, _kernels.py:77-82)
//   used as a counter-based source: word c of seed s is mix13(s + (c+1)*gamma),
//   so any position is reachable in O(1) ("counter-based skip-ahead").
// * the shared-memory table pack (layout of _packs.py:31-60, padded to 256 slots)
// * the modified-ziggurat draw bodies, templated on the word stream so the
//   production kernel (counter stream) and the oracle-mode replay pipeline run
//   literally the same arithmetic (_kernels.py:128-181 exp, :406-495 normal).
//
// Arithmetic follows SURVEY.md section 7.4 exactly: explicit __dmul_rn /
// __dadd_rn / __dsub_rn / __ddiv_rn so nvcc cannot contract into DFMA, Python's
// left-to-right association, __ull2double_rn / __ll2double_rn conversions,
// __double2ll_rz truncation for the alias index.  exp() is only compared.
#pragma once
#include <cstdint>

#include "zigfast_b200.h"

namespace zf {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kM1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kM2 = 0x94D049BB133111EBull;
// Secondary (exceptional) words of global sample K live at splitmix positions
// 2^63 + K * 2^19 + t: disjoint from every primary position K < 2^44.
constexpr uint64_t kExcBase = 1ull << 63;
constexpr int kExcShift = 19;
constexpr int kSlots = 256;

__host__ __device__ __forceinline__ uint64_t mix13(uint64_t z) {
  z = (z ^ (z >> 30)) * kM1;
  z = (z ^ (z >> 27)) * kM2;
  return z ^ (z >> 31);
}

// One distribution's pack.  sx has kSlots+2 entries so sx[i+1] is in bounds for
// every byte i: the fast loop reads it branch-free, and entries past L_max hold
// NaN so an exceptional byte yields a NaN fast value (its detection flag).
// Doubles first so every array is 16-byte aligned.
struct alignas(16) DevPack {
  double sx[kSlots + 2];
  double xlo[kSlots];
  double xw[kSlots];
  double flo[kSlots];
  double fh[kSlots];
  double prob[kSlots];
  double eps;
  double tailx;
  int32_t alias[kSlots];
  int32_t lmax;
  int32_t nslots;
  int32_t pad_[2];
};

// Normal kernels need the half-normal pack and the exponential pack (for the
// Marsaglia tail); they are stored back to back so one copy stages both.
struct alignas(16) DevTables {
  DevPack hn;
  DevPack ex;
};

static_assert(sizeof(DevPack) % 16 == 0, "DevPack must be int4-copyable");

__device__ __forceinline__ double u01(uint64_t u) {
  return __dmul_rn(__ull2double_rn(u), 0x1p-64);
}

// ---------------------------------------------------------------------------
// word streams
// ---------------------------------------------------------------------------

// Secondary words of one production sample: splitmix64 positions c, c+1, ...
struct CtrStream {
  uint64_t st;  // seed + c * gamma  (pre-increment form)
  static constexpr bool kBounded = false;
  __device__ __forceinline__ uint64_t next() {
    st += kGamma;
    return mix13(st);
  }
  __device__ __forceinline__ bool dead() const { return false; }
  __device__ __forceinline__ uint32_t used() const { return 0; }
};

// Oracle-mode stream: logical position p reads words[(cursor + p) % nwords],
// bounded by `limit` logical positions (the buffer window being resolved).
struct BufStream {
  const uint64_t* w;
  uint64_t nwords;
  uint64_t cursor;
  uint64_t pos;
  uint64_t limit;
  uint32_t count;
  bool over;
  static constexpr bool kBounded = true;
  __device__ __forceinline__ uint64_t next() {
    if (pos >= limit) {
      over = true;
      return 0;
    }
    uint64_t idx = cursor + pos;
    if (idx >= nwords) idx %= nwords;
    ++pos;
    ++count;
    return __ldg(reinterpret_cast<const unsigned long long*>(w) + idx);
  }
  __device__ __forceinline__ bool dead() const { return over; }
};

// ---------------------------------------------------------------------------
// per-draw bookkeeping (the reference's counter slots, _kernels.py:23-27)
// ---------------------------------------------------------------------------

struct NoCount {
  __device__ __forceinline__ void add(int, uint32_t = 1) {}
  static constexpr bool kOn = false;
  uint8_t path = 0;
  uint16_t attempts = 0;
};

struct Count {
  uint32_t c[6] = {0, 0, 0, 0, 0, 0};
  uint8_t path = 0;
  uint16_t attempts = 0;
  static constexpr bool kOn = true;
  __device__ __forceinline__ void add(int slot, uint32_t v = 1) { c[slot] += v; }
};

// ---------------------------------------------------------------------------
// draw bodies
// ---------------------------------------------------------------------------

// The rejection test `y < exp(arg)` (_kernels.py:178, :492) with the decision
// of the full double-precision exp, at a fraction of its cost: an fp32
// MUFU-based estimate e = __expf(arg) has relative error below 2e-6 for
// |arg| <= 20 (10 fp32 ulp of __expf plus the rounding of arg), so whenever y
// lies outside e * (1 -+ 1e-5) the comparison with ANY exp within 1 ulp of
// the true value (CUDA's exp, glibc's in the reference) is already decided.
// Only the ~1e-5 of tests inside the band evaluate the double exp.
__device__ __forceinline__ bool less_than_exp(double y, double arg) {
  constexpr double kTol = 1e-5;
  if (fabs(arg) <= 20.0) {
    const double e = (double)__expf(__double2float_rn(arg));
    if (y < e * (1.0 - kTol)) return true;
    if (y > e * (1.0 + kTol)) return false;
  }
  return y < exp(arg);
}

template <class S>
__device__ __forceinline__ int alias_pick(const DevPack& p, S& s) {
  const int n = p.nslots;
  long long k = __double2ll_rz(__dmul_rn(u01(s.next()), (double)n));
  if (k >= n) k = n - 1;
  const double up = u01(s.next());
  return up < p.prob[k] ? (int)k : p.alias[k];
}

// Exponential draw whose first byte word `u` has already been taken from the
// stream (exp_one_counted, _kernels.py:184-223).
template <class S, class C>
__device__ double exp_draw(const DevPack& p, uint64_t u, S& s, C& c) {
  double shift = 0.0;
  for (;;) {
    c.add(0);
    const int i = (int)(u & 0xFF);
    if (i < p.lmax) {
      c.add(1);
      c.path |= ZF_PATH_FAST;
      return __dadd_rn(shift, __dmul_rn(__ull2double_rn(u), p.sx[i + 1]));
    }
    const int j = alias_pick(p, s);
    if (j == 0) {
      c.add(4);
      c.path |= ZF_PATH_TAIL;
      shift = __dadd_rn(shift, p.tailx);
      u = s.next();
      if (S::kBounded && s.dead()) return 0.0;
      continue;
    }
    for (;;) {
      c.add(5);
      if (C::kOn) c.attempts++;
      double ux = u01(s.next());
      double uy = u01(s.next());
      if (S::kBounded && s.dead()) return 0.0;
      if (ux > __dsub_rn(1.0, uy)) {  // reflect the never-accept triangle
        const double t = ux;
        ux = __dsub_rn(1.0, uy);
        uy = __dsub_rn(1.0, t);
      }
      if (uy < __dsub_rn(__dsub_rn(1.0, ux), p.eps)) {  // below chord minus band
        c.add(2);
        c.path |= ZF_PATH_BOXFAST;
        return __dadd_rn(__dadd_rn(shift, p.xlo[j]), __dmul_rn(ux, p.xw[j]));
      }
      c.add(3);
      const double x = __dadd_rn(p.xlo[j], __dmul_rn(ux, p.xw[j]));
      const double y = __dadd_rn(p.flo[j], __dmul_rn(uy, p.fh[j]));
      if (less_than_exp(y, -x)) {
        c.path |= ZF_PATH_BOXEVAL;
        return __dadd_rn(shift, x);
      }
    }
  }
}

// Normal draw from its first word `u` (normal_one_counted, _kernels.py:498-594).
// The embedded exponential draws of the tail are not counted (:516-517).
template <class S, class C>
__device__ double normal_draw(const DevPack& h, const DevPack& e, uint64_t u, S& s, C& c) {
  c.add(0);
  const int i = (int)(u & 0xFF);
  const long long sg = (long long)u;
  if (i < h.lmax) {
    c.add(1);
    c.path |= ZF_PATH_FAST;
    return __dmul_rn(__ll2double_rn(sg), h.sx[i + 1]);
  }
  double val = 0.0;
  const int j = alias_pick(h, s);
  if (j == 0) {
    c.add(4);
    c.path |= ZF_PATH_TAIL;
    NoCount quiet;
    for (;;) {
      if (C::kOn) c.attempts++;
      const double e1 = exp_draw(e, s.next(), s, quiet);
      const double e2 = exp_draw(e, s.next(), s, quiet);
      if (S::kBounded && s.dead()) return 0.0;
      const double x = __ddiv_rn(e1, h.tailx);
      if (__dadd_rn(e2, e2) > __dmul_rn(x, x)) {
        val = __dadd_rn(h.tailx, x);
        break;
      }
    }
  } else {
    for (;;) {
      c.add(5);
      c.add(3);
      if (C::kOn) c.attempts++;
      const double ux = u01(s.next());
      const double uy = u01(s.next());
      if (S::kBounded && s.dead()) return 0.0;
      const double x = __dadd_rn(h.xlo[j], __dmul_rn(ux, h.xw[j]));
      const double y = __dadd_rn(h.flo[j], __dmul_rn(uy, h.fh[j]));
      if (less_than_exp(y, __dmul_rn(__dmul_rn(-0.5, x), x))) {
        c.path |= ZF_PATH_BOXEVAL;
        val = x;
        break;
      }
    }
  }
  return sg < 0 ? -val : val;
}

template <int DIST, class S, class C>
__device__ __forceinline__ double draw(const DevPack& prim, const DevPack& ex, uint64_t u, S& s,
                                       C& c) {
  if constexpr (DIST == ZF_EXP) {
    return exp_draw(prim, u, s, c);
  } else {
    return normal_draw(prim, ex, u, s, c);
  }
}

// Fast-path value of a first word (valid only when (u & 0xFF) < lmax).
template <int DIST>
__device__ __forceinline__ double fast_value(const double* sx, uint64_t u) {
  const int i = (int)(u & 0xFF);
  if constexpr (DIST == ZF_EXP) {
    return __dmul_rn(__ull2double_rn(u), sx[i + 1]);
  } else {
    return __dmul_rn(__ll2double_rn((long long)u), sx[i + 1]);
  }
}

template <typename T>
__device__ __forceinline__ T to_out(double v);
template <>
__device__ __forceinline__ double to_out<double>(double v) { return v; }
template <>
__device__ __forceinline__ float to_out<float>(double v) { return __double2float_rn(v); }

// Stage `bytes` (multiple of 16) from global to shared with the whole block.
__device__ __forceinline__ void stage_block(void* dst, const void* src, int bytes) {
  int4* d = reinterpret_cast<int4*>(dst);
  const int4* g = reinterpret_cast<const int4*>(src);
  for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x) d[i] = __ldg(g + i);
}

}  // namespace zf
