// zf_jump.cpp -- GF(2) jump-ahead for the reference's default generator.
//
// xoshiro256++ (_kernels.py:59-76) advances its 256-bit state with a linear
// map T over GF(2).  With P(x) the characteristic polynomial of T, the state
// k steps ahead is T^k s = (x^k mod P)(T) s, i.e. the xor of T^i s over the
// set coefficients of the degree-<256 polynomial x^k mod P -- the same
// "jump polynomial" scheme as the generator's published jump() routine, for
// an arbitrary k.  P is recovered once by Berlekamp-Massey from a state-bit
// sequence; the device kernel (zf_replay.cu) applies x^(d*16^r*B) mod P
// polynomials to give every thread the start of its own block of the stream.
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

namespace zf {

namespace {

struct Poly {  // degree < 256
  uint64_t w[4];
};

inline void step(uint64_t s[4]) {
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
}

// characteristic polynomial P = x^256 + low(x); `low` holds the 256 low coefficients
Poly g_low;
std::once_flag g_once;

void compute_charpoly() {
  // Berlekamp-Massey over GF(2) on bit 0 of s[0]
  const int N = 1024;
  std::vector<uint8_t> seq(N);
  uint64_t s[4] = {0x0123456789ABCDEFull, 0xFEDCBA9876543210ull, 0x0F1E2D3C4B5A6978ull,
                   0x8796A5B4C3D2E1F0ull};
  for (int i = 0; i < N; ++i) {
    seq[i] = (uint8_t)(s[0] & 1);
    step(s);
  }
  std::vector<uint8_t> C(N + 1, 0), B(N + 1, 0), T;
  C[0] = B[0] = 1;
  int L = 0, m = 1;
  for (int n = 0; n < N; ++n) {
    uint8_t d = seq[n];
    for (int i = 1; i <= L; ++i) d ^= (uint8_t)(C[i] & seq[n - i]);
    if (d == 0) {
      ++m;
    } else if (2 * L <= n) {
      T = C;
      for (int i = 0; i + m <= N; ++i) C[i + m] ^= B[i];
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      for (int i = 0; i + m <= N; ++i) C[i + m] ^= B[i];
      ++m;
    }
  }
  // L == 256 for xoshiro256 (primitive characteristic polynomial).
  // P(x) = x^L C(1/x): coefficient of x^(L-i) is C[i].
  std::memset(&g_low, 0, sizeof g_low);
  for (int i = 1; i <= L; ++i)
    if (C[i]) {
      const int d = L - i;  // < 256
      g_low.w[d >> 6] |= 1ull << (d & 63);
    }
}

// (a * b) mod P
Poly mulmod(const Poly& a, const Poly& b) {
  uint64_t prod[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < 256; ++i) {
    if (!((a.w[i >> 6] >> (i & 63)) & 1)) continue;
    const int ws = i >> 6, bs = i & 63;
    for (int k = 0; k < 4; ++k) {
      prod[k + ws] ^= b.w[k] << bs;
      if (bs) prod[k + ws + 1] ^= b.w[k] >> (64 - bs);
    }
  }
  for (int d = 511; d >= 256; --d) {
    if (!((prod[d >> 6] >> (d & 63)) & 1)) continue;
    prod[d >> 6] ^= 1ull << (d & 63);  // x^d = x^(d-256) * low(x)
    const int sh = d - 256, ws = sh >> 6, bs = sh & 63;
    for (int k = 0; k < 4; ++k) {
      prod[k + ws] ^= g_low.w[k] << bs;
      if (bs) prod[k + ws + 1] ^= g_low.w[k] >> (64 - bs);
    }
  }
  Poly r;
  std::memcpy(r.w, prod, sizeof r.w);
  return r;
}

Poly mulx(const Poly& a) {
  Poly r;
  const uint64_t top = a.w[3] >> 63;
  r.w[3] = (a.w[3] << 1) | (a.w[2] >> 63);
  r.w[2] = (a.w[2] << 1) | (a.w[1] >> 63);
  r.w[1] = (a.w[1] << 1) | (a.w[0] >> 63);
  r.w[0] = a.w[0] << 1;
  if (top)
    for (int k = 0; k < 4; ++k) r.w[k] ^= g_low.w[k];
  return r;
}

Poly xpow(uint64_t k) {  // x^k mod P
  Poly r = {{1, 0, 0, 0}};
  for (int b = 63; b >= 0; --b) {
    r = mulmod(r, r);
    if ((k >> b) & 1) r = mulx(r);
  }
  return r;
}

void apply(const Poly& p, uint64_t st[4]) {
  uint64_t acc[4] = {0, 0, 0, 0};
  uint64_t s[4] = {st[0], st[1], st[2], st[3]};
  for (int b = 0; b < 256; ++b) {
    if ((p.w[b >> 6] >> (b & 63)) & 1)
      for (int k = 0; k < 4; ++k) acc[k] ^= s[k];
    step(s);
  }
  std::memcpy(st, acc, sizeof acc);
}

}  // namespace

void xoshiro_jump_host(uint64_t st[4], uint64_t k) {
  std::call_once(g_once, compute_charpoly);
  if (k < 512) {  // cheaper to step
    for (uint64_t i = 0; i < k; ++i) step(st);
    return;
  }
  apply(xpow(k), st);
}

// Radix-2^bits jump table: out[(r * (R - 1) + d - 1) * 4 .. +4) = x^(d * R^r * B)
// mod P for r < levels, d = 1..R-1 (R = 2^bits).  A thread index t then needs
// one polynomial per nonzero base-R digit instead of one per set bit.
void xoshiro_radix_polys(uint64_t block_words, int bits, int levels, uint64_t* out) {
  std::call_once(g_once, compute_charpoly);
  const int R = 1 << bits;
  Poly q = xpow(block_words);  // x^(R^r * B) for the current level r
  for (int r = 0; r < levels; ++r) {
    Poly pd = q;
    for (int d = 1; d < R; ++d) {
      std::memcpy(out + ((size_t)r * (R - 1) + d - 1) * 4, pd.w, sizeof pd.w);
      pd = mulmod(pd, q);
    }
    q = pd;  // q^R
  }
}

// x^(2^e) mod P, exposed for the published-constant check in tests
void xoshiro_pow2_poly(int e, uint64_t out[4]) {
  std::call_once(g_once, compute_charpoly);
  Poly p = {{2, 0, 0, 0}};  // x
  for (int i = 0; i < e; ++i) p = mulmod(p, p);
  std::memcpy(out, p.w, sizeof p.w);
}

}  // namespace zf
