// zf_format.cu -- the step after the path: the reference's text output
// (`zigfast gen --format text`, cli.py:100-120, "".join(f"{v:.17g}\n" ...))
// produced on the device, byte-identical to CPython's '%.17g' formatting.
//
// Exact decimal conversion: a finite double x = m * 2^q (m < 2^53) is scaled
// by 10^p (p = 16 - E, E = floor(log10 |x|)) as a 192-bit integer product and
// shifted by -q with round-half-even on the exact remainder, giving the 17
// significant digits D in [10^16, 10^17) that printf's correctly rounded
// conversion produces; trailing zeros are stripped and the C99 %g style rule
// picks fixed or exponent notation.  Supported domain: 0 and
// 1e-22 <= |x| < 1e17 (p <= 38, so 10^p fits 128 bits) -- it contains every
// value the samplers can return; other values are counted as unsupported and
// the call reports them (nothing is written for them).
//
// Two passes over the input (the text length of a block must be known before
// any block can be placed): fmt_count sums per-block lengths, a single-block
// scan turns them into byte offsets, fmt_write re-derives the digits, stages
// the block's text in shared memory and streams it out with coalesced stores.
#include <cuda_runtime.h>

#include <algorithm>

#include "zf_internal.h"

namespace zf {
namespace {

constexpr int kFmtThreads = 256;
constexpr int kFmtPer = 4;  // values per thread
constexpr int kFmtBlock = kFmtThreads * kFmtPer;
constexpr int kFmtMax = 24;  // '-' + "0.000" + 17 digits + '\n' (or d.dddde-XX)
constexpr int kMaxP = 38;

struct U128 {
  uint64_t hi, lo;
};

// 10^p, p = 0..38, as 128-bit integers
__device__ const U128 kPow10[kMaxP + 1] = {
    {0x0000000000000000ull, 0x0000000000000001ull}, {0x0000000000000000ull, 0x000000000000000aull},
    {0x0000000000000000ull, 0x0000000000000064ull}, {0x0000000000000000ull, 0x00000000000003e8ull},
    {0x0000000000000000ull, 0x0000000000002710ull}, {0x0000000000000000ull, 0x00000000000186a0ull},
    {0x0000000000000000ull, 0x00000000000f4240ull}, {0x0000000000000000ull, 0x0000000000989680ull},
    {0x0000000000000000ull, 0x0000000005f5e100ull}, {0x0000000000000000ull, 0x000000003b9aca00ull},
    {0x0000000000000000ull, 0x00000002540be400ull}, {0x0000000000000000ull, 0x000000174876e800ull},
    {0x0000000000000000ull, 0x000000e8d4a51000ull}, {0x0000000000000000ull, 0x000009184e72a000ull},
    {0x0000000000000000ull, 0x00005af3107a4000ull}, {0x0000000000000000ull, 0x00038d7ea4c68000ull},
    {0x0000000000000000ull, 0x002386f26fc10000ull}, {0x0000000000000000ull, 0x016345785d8a0000ull},
    {0x0000000000000000ull, 0x0de0b6b3a7640000ull}, {0x0000000000000000ull, 0x8ac7230489e80000ull},
    {0x0000000000000005ull, 0x6bc75e2d63100000ull}, {0x0000000000000036ull, 0x35c9adc5dea00000ull},
    {0x000000000000021eull, 0x19e0c9bab2400000ull}, {0x000000000000152dull, 0x02c7e14af6800000ull},
    {0x000000000000d3c2ull, 0x1bcecceda1000000ull}, {0x0000000000084595ull, 0x161401484a000000ull},
    {0x000000000052b7d2ull, 0xdcc80cd2e4000000ull}, {0x00000000033b2e3cull, 0x9fd0803ce8000000ull},
    {0x00000000204fce5eull, 0x3e25026110000000ull}, {0x00000001431e0faeull, 0x6d7217caa0000000ull},
    {0x0000000c9f2c9cd0ull, 0x4674edea40000000ull}, {0x0000007e37be2022ull, 0xc0914b2680000000ull},
    {0x000004ee2d6d415bull, 0x85acef8100000000ull}, {0x0000314dc6448d93ull, 0x38c15b0a00000000ull},
    {0x0001ed09bead87c0ull, 0x378d8e6400000000ull}, {0x0013426172c74d82ull, 0x2b878fe800000000ull},
    {0x00c097ce7bc90715ull, 0xb34b9f1000000000ull}, {0x0785ee10d5da46d9ull, 0x00f436a000000000ull},
    {0x4b3b4ca85a86c47aull, 0x098a224000000000ull},
};

constexpr uint64_t kE16 = 10000000000000000ull;
constexpr uint64_t kE17 = 100000000000000000ull;

// bits [s, s + 64) of the 192-bit N = n2:n1:n0; *over = any bit >= s + 64 set
__device__ __forceinline__ uint64_t shr192(uint64_t n0, uint64_t n1, uint64_t n2, int s,
                                           bool* over) {
  if (s >= 128) {
    *over = false;
    return n2 >> (s - 128);
  }
  if (s >= 64) {
    const int t = s - 64;
    *over = t ? (n2 >> t) != 0 : n2 != 0;
    return t ? (n1 >> t) | (n2 << (64 - t)) : n1;
  }
  const int t = s;
  const uint64_t hi1 = t ? (n1 >> t) | (n2 << (64 - t)) : n1;
  const uint64_t hi2 = t ? (n2 >> t) : n2;
  *over = hi1 != 0 || hi2 != 0;
  return t ? (n0 >> t) | (n1 << (64 - t)) : n0;
}

__device__ __forceinline__ bool bit192(uint64_t n0, uint64_t n1, uint64_t n2, int k) {
  const uint64_t w = k < 64 ? n0 : (k < 128 ? n1 : n2);
  return (w >> (k & 63)) & 1;
}

// any of bits [0, k) set
__device__ __forceinline__ bool any_below(uint64_t n0, uint64_t n1, uint64_t n2, int k) {
  if (k <= 0) return false;
  if (k < 64) return (n0 & ((1ull << k) - 1)) != 0;
  if (n0) return true;
  if (k == 64) return false;
  if (k < 128) return (n1 & ((1ull << (k - 64)) - 1)) != 0;
  if (n1) return true;
  if (k == 128) return false;
  return (n2 & ((1ull << (k - 128)) - 1)) != 0;
}

struct Decimal {
  uint64_t d;  // 17 significant digits, trailing zeros stripped (nd digits)
  int e;       // decimal exponent of the first digit
  int nd;      // 1..17
  bool neg;
  bool zero;
};

// Correctly rounded 17-significant-digit decimal of x; false if unsupported.
__device__ bool to_decimal17(double x, const U128* pw, Decimal* out) {
  uint64_t b = (uint64_t)__double_as_longlong(x);
  out->neg = b >> 63;
  b &= ~(1ull << 63);
  out->zero = b == 0;
  if (b == 0) {
    out->d = 0;
    out->e = 0;
    out->nd = 1;
    return true;
  }
  if (b >= 0x7ff0000000000000ull) return false;  // inf / nan
  int be = (int)(b >> 52);
  uint64_t m = b & ((1ull << 52) - 1);
  if (be == 0) be = 1;
  else m |= 1ull << 52;
  const int q = be - 1075;  // |x| = m * 2^q
  int e = (int)floor(log10(__longlong_as_double((long long)b)));
  uint64_t d = 0;
  for (int attempt = 0; attempt < 4; ++attempt) {
    const int p = 16 - e;
    if (p < 0 || p > kMaxP) {
      // the log10 estimate may be one off next to a power of ten: nudge once
      if (attempt > 0) return false;
      e += p < 0 ? -1 : 1;
      continue;
    }
    // N = m * 10^p  (192 bits: n2:n1:n0)
    const U128 t = pw[p];
    const uint64_t a0 = m * t.lo, a1 = __umul64hi(m, t.lo);
    const uint64_t c0 = m * t.hi, c1 = __umul64hi(m, t.hi);
    const uint64_t n0 = a0;
    const uint64_t n1 = a1 + c0;
    const uint64_t n2 = c1 + (n1 < a1);
    bool over = false;
    bool round_up = false;
    if (q < 0) {
      const int s = -q;
      d = shr192(n0, n1, n2, s, &over);
      const bool half = bit192(n0, n1, n2, s - 1);
      round_up = half && (any_below(n0, n1, n2, s - 1) || (d & 1));
    } else {  // exact: N * 2^q
      over = n1 != 0 || n2 != 0 || (q > 0 && (n0 >> (64 - q)) != 0);
      d = n0 << q;
    }
    if (over || d >= kE17) {
      ++e;
      continue;
    }
    if (d < kE16) {
      --e;
      continue;
    }
    d += round_up;
    if (d == kE17) {
      d = kE16;
      ++e;
    }
    int nd = 17;
    while (nd > 1 && d % 10 == 0) {
      d /= 10;
      --nd;
    }
    out->d = d;
    out->e = e;
    out->nd = nd;
    return true;
  }
  return false;
}

// bytes of the '%.17g' text plus the newline
__device__ __forceinline__ int text_len(const Decimal& v) {
  if (v.zero) return (int)v.neg + 2;  // "0\n" / "-0\n"
  int len = (int)v.neg + 1;            // sign + newline
  if (v.e < -4 || v.e >= 17) {
    const int ae = v.e < 0 ? -v.e : v.e;
    len += 1 + (v.nd > 1 ? v.nd : 0) + 2 + (ae >= 100 ? 3 : 2);
  } else if (v.e >= 0) {
    len += (v.e + 1) + (v.nd > v.e + 1 ? 1 + v.nd - (v.e + 1) : 0);
  } else {
    len += 2 + (-v.e - 1) + v.nd;
  }
  return len;
}

// write the text of v at dst (shared memory), returns bytes written
__device__ int write_text(const Decimal& v, char* dst) {
  int k = 0;
  if (v.neg) dst[k++] = '-';
  if (v.zero) {
    dst[k++] = '0';
    dst[k++] = '\n';
    return k;
  }
  char dig[17];
  {
    uint64_t d = v.d;
    for (int i = v.nd - 1; i >= 0; --i) {
      dig[i] = (char)('0' + d % 10);
      d /= 10;
    }
  }
  if (v.e < -4 || v.e >= 17) {
    dst[k++] = dig[0];
    if (v.nd > 1) {
      dst[k++] = '.';
      for (int i = 1; i < v.nd; ++i) dst[k++] = dig[i];
    }
    dst[k++] = 'e';
    dst[k++] = v.e < 0 ? '-' : '+';
    int ae = v.e < 0 ? -v.e : v.e;
    if (ae >= 100) {
      dst[k++] = (char)('0' + ae / 100);
      ae %= 100;
    }
    dst[k++] = (char)('0' + ae / 10);
    dst[k++] = (char)('0' + ae % 10);
  } else if (v.e >= 0) {
    for (int i = 0; i <= v.e; ++i) dst[k++] = i < v.nd ? dig[i] : '0';
    if (v.nd > v.e + 1) {
      dst[k++] = '.';
      for (int i = v.e + 1; i < v.nd; ++i) dst[k++] = dig[i];
    }
  } else {
    dst[k++] = '0';
    dst[k++] = '.';
    for (int i = 0; i < -v.e - 1; ++i) dst[k++] = '0';
    for (int i = 0; i < v.nd; ++i) dst[k++] = dig[i];
  }
  dst[k++] = '\n';
  return k;
}

__device__ __forceinline__ void stage_pow10(U128* s) {
  for (int i = threadIdx.x; i <= kMaxP; i += blockDim.x) s[i] = kPow10[i];
}

// block-wide exclusive scan of one int per thread (256 threads)
__device__ __forceinline__ int block_excl(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  int base = 0, tot = 0;
  for (int i = 0; i < kFmtThreads / 32; ++i) {
    if (i < w) base += warp_tot[i];
    tot += warp_tot[i];
  }
  *total = tot;
  return base + incl - v;
}

__global__ void __launch_bounds__(kFmtThreads)
    fmt_count(const double* __restrict__ x, uint64_t n, uint32_t* __restrict__ blk_len,
              unsigned long long* __restrict__ bad) {
  __shared__ U128 pw[kMaxP + 1];
  __shared__ int warp_tot[kFmtThreads / 32];
  stage_pow10(pw);
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kFmtBlock;
  int len = 0, nbad = 0;
#pragma unroll
  for (int j = 0; j < kFmtPer; ++j) {
    const uint64_t i = base + (uint64_t)j * kFmtThreads + threadIdx.x;
    if (i < n) {
      Decimal v;
      if (to_decimal17(__ldg(x + i), pw, &v)) len += text_len(v);
      else ++nbad;
    }
  }
  int total;
  block_excl(len, warp_tot, &total);
  if (threadIdx.x == 0) blk_len[blockIdx.x] = (uint32_t)total;
  if (nbad) atomicAdd(bad, (unsigned long long)nbad);
}

// exclusive scan of the per-block lengths into byte offsets; total at [nb]
__global__ void __launch_bounds__(1024)
    fmt_scan(const uint32_t* __restrict__ blk_len, uint64_t nb, uint64_t* __restrict__ off) {
  __shared__ uint64_t part[1024];
  const uint64_t per = (nb + 1023) / 1024;
  const uint64_t beg = std::min<uint64_t>(nb, threadIdx.x * per);
  const uint64_t end = std::min<uint64_t>(nb, beg + per);
  uint64_t s = 0;
  for (uint64_t i = beg; i < end; ++i) s += blk_len[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t run = 0;
    for (int i = 0; i < 1024; ++i) {
      const uint64_t v = part[i];
      part[i] = run;
      run += v;
    }
    off[nb] = run;
  }
  __syncthreads();
  uint64_t run = part[threadIdx.x];
  for (uint64_t i = beg; i < end; ++i) {
    off[i] = run;
    run += blk_len[i];
  }
}

__global__ void __launch_bounds__(kFmtThreads)
    fmt_write(const double* __restrict__ x, uint64_t n, const uint64_t* __restrict__ off,
              uint64_t nb, char* __restrict__ out, uint64_t cap) {
  __shared__ U128 pw[kMaxP + 1];
  __shared__ int warp_tot[kFmtThreads / 32];
  __shared__ __align__(16) char text[kFmtBlock * kFmtMax];
  if (off[nb] > cap) return;  // caller's buffer too small: write nothing
  stage_pow10(pw);
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kFmtBlock;
  // thread t formats values base + t*kFmtPer .. +kFmtPer-1 (consecutive, so
  // the block's text is in input order after one scan)
  Decimal v[kFmtPer];
  bool ok[kFmtPer];
  int len = 0;
#pragma unroll
  for (int j = 0; j < kFmtPer; ++j) {
    const uint64_t i = base + (uint64_t)threadIdx.x * kFmtPer + j;
    ok[j] = i < n && to_decimal17(__ldg(x + i), pw, &v[j]);
    if (ok[j]) len += text_len(v[j]);
  }
  int total;
  int pos = block_excl(len, warp_tot, &total);
#pragma unroll
  for (int j = 0; j < kFmtPer; ++j)
    if (ok[j]) pos += write_text(v[j], text + pos);
  __syncthreads();
  // stream the block's bytes out: 4-byte stores once the destination is aligned
  char* dst = out + off[blockIdx.x];
  const int head = (int)((4 - (reinterpret_cast<uintptr_t>(dst) & 3)) & 3);
  const int h = head < total ? head : total;
  if ((int)threadIdx.x < h) dst[threadIdx.x] = text[threadIdx.x];
  const int words = (total - h) / 4;
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst + h);
  for (int w = threadIdx.x; w < words; w += kFmtThreads) {
    const int s = h + 4 * w;
    dw[w] = (uint32_t)(uint8_t)text[s] | ((uint32_t)(uint8_t)text[s + 1] << 8) |
            ((uint32_t)(uint8_t)text[s + 2] << 16) | ((uint32_t)(uint8_t)text[s + 3] << 24);
  }
  for (int s = h + 4 * words + threadIdx.x; s < total; s += kFmtThreads) dst[s] = text[s];
}

}  // namespace

uint64_t format_blocks(uint64_t n) { return (n + kFmtBlock - 1) / kFmtBlock; }

int launch_format_g17(const double* x, uint64_t n, char* out, uint64_t cap, uint64_t* scratch,
                      cudaStream_t s) {
  // scratch (device, u64): [0] total length, [1] unsupported count,
  // [2 .. 2 + nb] block offsets, then nb u32 block lengths
  const uint64_t nb = format_blocks(n);
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(scratch + 1);
  uint64_t* off = scratch + 2;
  uint32_t* blen = reinterpret_cast<uint32_t*>(off + nb + 1);
  ZF_TRY(cudaMemsetAsync(scratch, 0, 2 * sizeof(uint64_t), s));
  if (n == 0) return ZF_OK;
  fmt_count<<<(uint32_t)nb, kFmtThreads, 0, s>>>(x, n, blen, bad);
  fmt_scan<<<1, 1024, 0, s>>>(blen, nb, off);
  ZF_TRY(cudaMemcpyAsync(scratch, off + nb, sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  fmt_write<<<(uint32_t)nb, kFmtThreads, 0, s>>>(x, n, off, nb, out, cap);
  return cuda_status(cudaGetLastError());
}

}  // namespace zf
