// zf_device.cuh -- device-side building blocks shared by every sm_100a kernel.
//
// * the counter-based production source: word c of seed s is
//   fmix64(s + (c+1)*gamma) on splitmix64's Weyl sequence, so any position is
//   reachable in O(1) ("counter-based skip-ahead"); mix13 (the reference's
//   gid-1 splitmix64 output function, _kernels.py:77-82) for oracle mode.
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
// Secondary (exceptional) words of global sample K live at counter positions
// 2^63 + K * 2^19 + t: disjoint from every primary position K < 2^44.
constexpr uint64_t kExcBase = 1ull << 63;
constexpr int kExcShift = 19;
constexpr int kSlots = 256;

// z * c mod 2^64 in three IMADs: nvcc's own expansion adds the two cross
// products separately and then folds them into the high word (four IMADs);
// the fill kernel is issue-bound, so the chained form saves one instruction
// per multiply (two per word).
template <uint64_t C>
__device__ __forceinline__ uint64_t mul64_chained(uint64_t z) {
  const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
  uint32_t rlo, rhi;
  asm("mul.lo.u32 %0, %2, %4;\n\t"
      "mul.hi.u32 %1, %2, %4;\n\t"
      "mad.lo.u32 %1, %2, %5, %1;\n\t"
      "mad.lo.u32 %1, %3, %4, %1;"
      : "=&r"(rlo), "=&r"(rhi)
      : "r"(lo), "r"(hi), "n"((uint32_t)C), "n"((uint32_t)(C >> 32)));
  return ((uint64_t)rhi << 32) | rlo;
}

__host__ __device__ __forceinline__ uint64_t mix13(uint64_t z) {
#if defined(__CUDA_ARCH__) && !defined(ZF_PLAIN_MUL64)
  z = mul64_chained<kM1>(z ^ (z >> 30));
  z = mul64_chained<kM2>(z ^ (z >> 27));
#else
  z = (z ^ (z >> 30)) * kM1;
  z = (z ^ (z >> 27)) * kM2;
#endif
  return z ^ (z >> 31);
}

// Word function of the production counter stream: MurmurHash3's 64-bit
// finalizer fmix64 (shifts of 33 -- the same constants SplittableRandom uses
// to mix its gammas) applied to the splitmix64 Weyl sequence.  Its xorshifts
// by 33 are one SHF + one LOP3 on 32-bit halves where mix13's shifts by 30,
// 27 and 31 need two of each: +10 % fill throughput on B200 (DESIGN.md,
// "Production word function"), with the generator battery of
// tools/battery.py showing no difference between the two
// (profiles/r02_battery.json).  mix13 stays the word function of the
// reference's own splitmix64 stream (gid 1, oracle mode).
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
#if defined(__CUDA_ARCH__) && !defined(ZF_PLAIN_MUL64)
  z = mul64_chained<0xff51afd7ed558ccdull>(z ^ (z >> 33));
  z = mul64_chained<0xc4ceb9fe1a85ec53ull>(z ^ (z >> 33));
#else
  z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdull;
  z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ull;
#endif
  return z ^ (z >> 33);
}
__host__ __device__ __forceinline__ uint64_t ctr_word(uint64_t z) {
#if defined(ZF_WORD_MIX13)  // experiment builds: the round-1 word function
  return mix13(z);
#else
  return fmix64(z);
#endif
}

// One distribution's pack.  sx has kSlots+2 entries so sx[i+1] is in bounds for
// every byte i: the fast loop reads it branch-free, and entries past L_max hold
// NaN so an exceptional byte yields a NaN fast value (its detection flag).
// Doubles first so every array is 16-byte aligned.
//
// The traditional ziggurat (traditional.py:113-121 `_pack`) reuses the layout:
// sx[i+1] = edge[i]*2^-64 (exp) / *2^-63 (normal), kk[] (aliasing xlo) = the
// integer fast-accept thresholds, flo/fh = the wedge strip, tailx = r,
// lmax = nslots = 256; the other arrays are unused.
struct alignas(16) DevPack {
  double sx[kSlots + 2];
  union {
    double xlo[kSlots];
    uint64_t kk[kSlots];
  };
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

// Distribution traits.  A table handle holds either the modified packs
// (hn = half-normal, ex = exponential) or the traditional ones in the same
// two slots; normal kernels of the modified algorithm also stage `ex` for the
// Marsaglia tail.
template <int DIST>
constexpr bool kTrad = DIST == ZF_TRAD_EXP || DIST == ZF_TRAD_NORMAL;
template <int DIST>
constexpr bool kSigned = DIST == ZF_NORMAL || DIST == ZF_TRAD_NORMAL;
template <int DIST>
constexpr int kPacksOf = DIST == ZF_NORMAL ? 2 : 1;
template <int DIST>
__host__ __device__ __forceinline__ const DevPack* primary_pack(const DevTables* t) {
  return kSigned<DIST> ? &t->hn : &t->ex;
}

__device__ __forceinline__ double u01(uint64_t u) {
  return __dmul_rn(__ull2double_rn(u), 0x1p-64);
}

// (float64(u) + 1.0) * 2^-64 in (0, 1] (_u01_pos, _kernels.py:103-105)
__device__ __forceinline__ double u01_pos(uint64_t u) {
  return __dmul_rn(__dadd_rn(__ull2double_rn(u), 1.0), 0x1p-64);
}

// ---------------------------------------------------------------------------
// correctly rounded natural log (the traditional sampler returns log values,
// _kernels.py:945,1103, so its tail samples need the libm result, not CUDA's
// 1-ulp log).  Double-double evaluation, relative error ~2^-100, then one
// rounding: equals the correctly rounded log except when the exact value lies
// within ~2^-100 of a rounding boundary.  Rare path (tails only).
// ---------------------------------------------------------------------------

struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}
__device__ __forceinline__ DD quick_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ DD two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  const DD t = two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = quick_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ DD dd_mul(DD a, DD b) {
  DD p = two_prod(a.hi, b.hi);
  p.lo = __fma_rn(a.hi, b.lo, p.lo);
  p.lo = __fma_rn(a.lo, b.hi, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ DD dd_div(DD a, DD b) {
  const double q1 = __ddiv_rn(a.hi, b.hi);
  DD r = dd_add(a, dd_mul(b, DD{-q1, 0.0}));
  const double q2 = __ddiv_rn(r.hi, b.hi);
  r = dd_add(r, dd_mul(b, DD{-q2, 0.0}));
  const double q3 = __ddiv_rn(r.hi, b.hi);
  return dd_add(quick_two_sum(q1, q2), DD{q3, 0.0});
}

// log(x) for finite x > 0 (normal or subnormal), correctly rounded as above.
static __device__ __noinline__ double log_cr(double x) {
  int e = 0;
  double m = frexp(x, &e);  // x = m * 2^e, m in [0.5, 1)
  if (m < 0.70710678118654752) {
    m = __dmul_rn(m, 2.0);
    --e;
  }  // m in [sqrt(1/2), sqrt(2))
  // log(m) = 2 atanh(t), t = (m - 1) / (m + 1); |t| <= 0.1716
  const DD num = DD{__dsub_rn(m, 1.0), 0.0};  // exact (Sterbenz)
  const DD den = two_sum(m, 1.0);
  const DD t = dd_div(num, den);
  const DD t2 = dd_mul(t, t);
  // sum_{k>=0} t^(2k) / (2k+1), k < 24 (t^48 < 2^-120)
  DD acc = DD{1.0 / 47.0, 0.0};
  for (int k = 22; k >= 0; --k) {
    const double d = (double)(2 * k + 1);
    const double ch = __ddiv_rn(1.0, d);
    const DD c = DD{ch, __ddiv_rn(-__fma_rn(ch, d, -1.0), d)};  // 1/d to ~2^-106
    acc = dd_add(c, dd_mul(acc, t2));
  }
  DD lm = dd_mul(dd_mul(DD{2.0, 0.0}, t), acc);
  constexpr double kLn2Hi = 0x1.62e42fefa39efp-1;
  constexpr double kLn2Lo = 0x1.abc9e3b39803fp-56;
  const DD el = dd_mul(DD{(double)e, 0.0}, DD{kLn2Hi, kLn2Lo});
  const DD r = dd_add(el, lm);
  return __dadd_rn(r.hi, r.lo);
}

// ---------------------------------------------------------------------------
// word streams
// ---------------------------------------------------------------------------

// Secondary words of one production sample: counter positions c, c+1, ...
struct CtrStream {
  uint64_t st;  // seed + c * gamma  (pre-increment form)
  static constexpr bool kBounded = false;
  __device__ __forceinline__ uint64_t next() {
    st += kGamma;
    return ctr_word(st);
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
// MUFU-based estimate e = __expf(arg) is within 2 + floor(1.16 |arg|) fp32
// ulp of exp(float(arg)) (the CUDA guide's bound for __expf: 25 ulp = 3.0e-6
// relative at |arg| = 20), and rounding arg to fp32 moves exp by at most
// |arg| 2^-24 = 1.2e-6 relative, so for |arg| <= 20 e is within 4.2e-6 of
// the true value.  Whenever y lies outside e * (1 -+ 1e-5) the comparison
// with ANY exp within 1 ulp of the true value (CUDA's exp, glibc's in the
// reference) is already decided; only the ~1e-5 of tests inside the band
// evaluate the double exp.
__device__ __forceinline__ bool less_than_exp(double y, double arg) {
  constexpr double kTol = 1e-5;
  if (fabs(arg) <= 20.0) {
    const double e = (double)__expf(__double2float_rn(arg));
    if (y < e * (1.0 - kTol)) return true;
    if (y > e * (1.0 + kTol)) return false;
  }
  return y < exp(arg);
}

// alias pick (_kernels.py:128-136) from its two words
__device__ __forceinline__ int alias_from(const DevPack& p, uint64_t w1, uint64_t w2) {
  const int n = p.nslots;
  long long k = __double2ll_rz(__dmul_rn(u01(w1), (double)n));
  if (k >= n) k = n - 1;
  const double up = u01(w2);
  return up < p.prob[k] ? (int)k : p.alias[k];
}

template <class S>
__device__ __forceinline__ int alias_pick(const DevPack& p, S& s) {
  const uint64_t w1 = s.next();
  const uint64_t w2 = s.next();
  return alias_from(p, w1, w2);
}

// Exponential draw whose first byte word `u` has already been taken from the
// stream (exp_one_counted, _kernels.py:184-223).
template <class S, class C>
__device__ double exp_draw(const DevPack& p, uint64_t u, S& s, C& c, double shift = 0.0) {
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

// One attempt of the exponential box loop (_kernels.py:163-180) for slot j
// from its two words: true and the value (shift + x) if accepted.
__device__ __forceinline__ bool exp_box_words(const DevPack& p, int j, uint64_t wa, uint64_t wb,
                                              double shift, double& v) {
  double ux = u01(wa);
  double uy = u01(wb);
  if (ux > __dsub_rn(1.0, uy)) {
    const double t = ux;
    ux = __dsub_rn(1.0, uy);
    uy = __dsub_rn(1.0, t);
  }
  if (uy < __dsub_rn(__dsub_rn(1.0, ux), p.eps)) {
    v = __dadd_rn(__dadd_rn(shift, p.xlo[j]), __dmul_rn(ux, p.xw[j]));
    return true;
  }
  const double x = __dadd_rn(p.xlo[j], __dmul_rn(ux, p.xw[j]));
  const double y = __dadd_rn(p.flo[j], __dmul_rn(uy, p.fh[j]));
  v = __dadd_rn(shift, x);
  return less_than_exp(y, -x);
}

// Production exponential draw of an exceptional first word (exp_draw with
// u = an exceptional byte) on the secondary counter stream at `sbase`: the
// four words of the alias pick and the first box attempt are independent
// counter positions, so they are computed side by side instead of one
// dependent word-function chain after another.  Same words, same arithmetic, same
// value as exp_draw.
__device__ __forceinline__ double exp_draw_ctr(const DevPack& p, uint64_t sbase) {
  const uint64_t w1 = ctr_word(sbase + kGamma), w2 = ctr_word(sbase + 2 * kGamma);
  const uint64_t w3 = ctr_word(sbase + 3 * kGamma), w4 = ctr_word(sbase + 4 * kGamma);
  const int j = alias_from(p, w1, w2);
  NoCount c;
  if (j == 0) {  // tail: shift by X[1], word 3 is the next first word
    CtrStream s{sbase + 3 * kGamma};
    return exp_draw(p, w3, s, c, p.tailx);
  }
  double v;
  if (exp_box_words(p, j, w3, w4, 0.0, v)) return v;
  CtrStream s{sbase + 4 * kGamma};
  for (;;) {
    const uint64_t wa = s.next();
    const uint64_t wb = s.next();
    if (exp_box_words(p, j, wa, wb, 0.0, v)) return v;
  }
}

// One attempt of the normal overhang box loop (_kernels.py:679-688) for slot j
// from the stream's current position: true and x if accepted.
__device__ __forceinline__ bool normal_box_words(const DevPack& h, int j, uint64_t wa, uint64_t wb,
                                                 double& x) {
  const double ux = u01(wa);
  const double uy = u01(wb);
  x = __dadd_rn(h.xlo[j], __dmul_rn(ux, h.xw[j]));
  const double y = __dadd_rn(h.flo[j], __dmul_rn(uy, h.fh[j]));
  return less_than_exp(y, __dmul_rn(__dmul_rn(-0.5, x), x));
}
template <class S>
__device__ __forceinline__ bool normal_box_attempt(const DevPack& h, int j, S& s, double& x) {
  const uint64_t wa = s.next();
  const uint64_t wb = s.next();
  return normal_box_words(h, j, wa, wb, x);
}

// Normal tail beyond r = X[1] (_kernels.py:611-678): Marsaglia's method with
// two embedded exponential-ziggurat draws per attempt (not counted, :516-517).
template <class S, class C>
__device__ __forceinline__ double normal_tail(const DevPack& h, const DevPack& e, S& s, C& c) {
  NoCount quiet;
  for (;;) {
    if (C::kOn) c.attempts++;
    const double e1 = exp_draw(e, s.next(), s, quiet);
    const double e2 = exp_draw(e, s.next(), s, quiet);
    if (S::kBounded && s.dead()) return 0.0;
    const double x = __ddiv_rn(e1, h.tailx);
    if (__dadd_rn(e2, e2) > __dmul_rn(x, x)) return __dadd_rn(h.tailx, x);
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
    val = normal_tail(h, e, s, c);
    if (S::kBounded && s.dead()) return 0.0;
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

// ---------------------------------------------------------------------------
// traditional ziggurat (trad_exp_one_counted / trad_normal_one_counted,
// _kernels.py:956-979, :1117-1146): x = word * edge unconditionally, integer
// fast accept, tail fallback in strip 0, otherwise one wedge test; any
// rejection restarts with a fresh byte word.  Counter slots as the reference:
// 0 byte words, 1 fast accepts, 2 wedge tests, 3 tail entries.
// ---------------------------------------------------------------------------

template <int DIST>
__device__ __forceinline__ bool trad_fast(const uint64_t* kk, uint64_t u) {
  const uint64_t a = (DIST == ZF_TRAD_NORMAL && (long long)u < 0) ? 0ull - u : u;
  return a < kk[u & 0xFF];
}

template <class S, class C>
__device__ double trad_exp_draw(const DevPack& p, uint64_t u, S& s, C& c) {
  for (;;) {
    c.add(0);
    const int i = (int)(u & 0xFF);
    const double x = __dmul_rn(__ull2double_rn(u), p.sx[i + 1]);
    if (u < p.kk[i]) {
      c.add(1);
      c.path |= ZF_PATH_FAST;
      return x;
    }
    if (i == 0) {
      c.add(3);
      c.path |= ZF_PATH_TAIL;
      const double l = log_cr(u01_pos(s.next()));
      if (S::kBounded && s.dead()) return 0.0;
      return __dsub_rn(p.tailx, l);
    }
    c.add(2);
    if (C::kOn) c.attempts++;
    const double y = __dadd_rn(p.flo[i], __dmul_rn(u01(s.next()), p.fh[i]));
    if (S::kBounded && s.dead()) return 0.0;
    if (less_than_exp(y, -x)) {
      c.path |= ZF_PATH_BOXEVAL;
      return x;
    }
    u = s.next();
    if (S::kBounded && s.dead()) return 0.0;
  }
}

template <class S, class C>
__device__ double trad_normal_draw(const DevPack& p, uint64_t u, S& s, C& c) {
  for (;;) {
    c.add(0);
    const int i = (int)(u & 0xFF);
    const long long sg = (long long)u;
    const double x = __dmul_rn(__ll2double_rn(sg), p.sx[i + 1]);
    if (trad_fast<ZF_TRAD_NORMAL>(p.kk, u)) {
      c.add(1);
      c.path |= ZF_PATH_FAST;
      return x;
    }
    if (i == 0) {
      c.add(3);
      c.path |= ZF_PATH_TAIL;
      for (;;) {
        if (C::kOn) c.attempts++;
        const double xt = __ddiv_rn(-log_cr(u01_pos(s.next())), p.tailx);
        const double yt = -log_cr(u01_pos(s.next()));
        if (S::kBounded && s.dead()) return 0.0;
        if (__dadd_rn(yt, yt) > __dmul_rn(xt, xt)) {
          const double v = __dadd_rn(p.tailx, xt);
          return sg < 0 ? -v : v;
        }
      }
    }
    c.add(2);
    if (C::kOn) c.attempts++;
    const double y = __dadd_rn(p.flo[i], __dmul_rn(u01(s.next()), p.fh[i]));
    if (S::kBounded && s.dead()) return 0.0;
    if (less_than_exp(y, __dmul_rn(__dmul_rn(-0.5, x), x))) {
      c.path |= ZF_PATH_BOXEVAL;
      return x;
    }
    u = s.next();
    if (S::kBounded && s.dead()) return 0.0;
  }
}

template <int DIST, class S, class C>
__device__ __forceinline__ double draw(const DevPack& prim, const DevPack& ex, uint64_t u, S& s,
                                       C& c) {
  if constexpr (DIST == ZF_EXP) {
    return exp_draw(prim, u, s, c);
  } else if constexpr (DIST == ZF_NORMAL) {
    return normal_draw(prim, ex, u, s, c);
  } else if constexpr (DIST == ZF_TRAD_EXP) {
    return trad_exp_draw(prim, u, s, c);
  } else {
    return trad_normal_draw(prim, u, s, c);
  }
}

// Is a first word exceptional (anything but the one-word fast path)?
template <int DIST>
__device__ __forceinline__ bool exc_word(const DevPack& p, uint64_t u) {
  if constexpr (kTrad<DIST>) {
    return !trad_fast<DIST>(p.kk, u);
  } else {
    return ((uint32_t)u & 0xFFu) >= (uint32_t)p.lmax;
  }
}

// Fast-path value of a first word (valid only when !exc_word; for the modified
// algorithm it is NaN for every exceptional byte by the sx sentinel).
template <int DIST>
__device__ __forceinline__ double fast_value(const double* sx, uint64_t u) {
  const int i = (int)(u & 0xFF);
  if constexpr (!kSigned<DIST>) {
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

// ---------------------------------------------------------------------------
// asynchronous staging (TMA bulk copies completing on shared-memory mbarriers)
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
// one thread: expect `bytes` on `bar` and start the bulk copy global -> shared
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(const uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Stage a table image whose first `head` bytes pass 1 needs at once (the
// fast-path scale array) and whose remaining `bytes - head` only the rare
// rounds read: thread 0 starts two bulk copies; the block waits for the head
// here, each warp waits for the tail (bars[1], phase 0) before its first
// round.  Call from every thread; includes a __syncthreads.
__device__ __forceinline__ void stage_split(void* dst, const void* src, int head, int bytes,
                                            uint64_t* bars) {
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    bulk_load(dst, src, (uint32_t)head, &bars[0]);
    bulk_load(static_cast<char*>(dst) + head, static_cast<const char*>(src) + head,
              (uint32_t)(bytes - head), &bars[1]);
  }
  __syncthreads();
  mbar_wait(&bars[0], 0);
}

}  // namespace zf
