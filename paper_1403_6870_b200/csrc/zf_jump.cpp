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

// Fast path for the per-fill host jumps (an oracle-mode fill advances the
// host state by the words it consumed): x^k mod P as a product of the
// precomputed x^(2^i) mod P over the set bits of k, each product by a 4-bit
// comb multiplication and a byte-table reduction.  ~40 us -> a few us per
// jump of ~2^20 words.
struct FastTables {
  Poly pow2[64];           // x^(2^i) mod P
  Poly red[32][256];       // (v(x) * x^(256 + 8 j)) mod P
};
FastTables* g_fast = nullptr;
std::once_flag g_fast_once;

void build_fast() {
  auto* f = new FastTables;
  Poly p = {{2, 0, 0, 0}};  // x
  for (int i = 0; i < 64; ++i) {
    f->pow2[i] = p;
    p = mulmod(p, p);
  }
  Poly basis = {{0, 0, 0, 0}};  // x^256 mod P = low(x)
  std::memcpy(basis.w, g_low.w, sizeof basis.w);
  for (int j = 0; j < 32; ++j) {
    Poly bit[8];
    for (int b = 0; b < 8; ++b) {
      bit[b] = basis;  // x^(256 + 8 j + b) mod P
      basis = mulx(basis);
    }
    for (int v = 0; v < 256; ++v) {
      Poly r = {{0, 0, 0, 0}};
      for (int b = 0; b < 8; ++b)
        if ((v >> b) & 1)
          for (int k = 0; k < 4; ++k) r.w[k] ^= bit[b].w[k];
      f->red[j][v] = r;
    }
  }
  g_fast = f;
}

Poly mulmod_fast(const Poly& a, const Poly& b) {
  // comb: tb[c] = c(x) * b(x) for the 16 polynomials c of degree < 4 (260 bits)
  uint64_t tb[16][5];
  std::memset(tb, 0, sizeof tb);
  for (int c = 1; c < 16; ++c) {
    for (int bb = 0; bb < 4; ++bb) {
      if (!((c >> bb) & 1)) continue;
      for (int k = 0; k < 4; ++k) {
        tb[c][k] ^= b.w[k] << bb;
        if (bb) tb[c][k + 1] ^= b.w[k] >> (64 - bb);
      }
    }
  }
  uint64_t prod[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 63; i >= 0; --i) {  // nibble i of a, high to low: prod = prod * x^4 + nib * b
    for (int k = 7; k > 0; --k) prod[k] = (prod[k] << 4) | (prod[k - 1] >> 60);
    prod[0] <<= 4;
    const int nib = (int)((a.w[i >> 4] >> ((i & 15) * 4)) & 15);
    for (int k = 0; k < 5; ++k) prod[k] ^= tb[nib][k];
  }
  Poly r;
  std::memcpy(r.w, prod, sizeof r.w);
  for (int j = 0; j < 32; ++j) {  // the high 256 bits, byte by byte
    const int v = (int)((prod[4 + (j >> 3)] >> ((j & 7) * 8)) & 0xFF);
    if (v)
      for (int k = 0; k < 4; ++k) r.w[k] ^= g_fast->red[j][v].w[k];
  }
  return r;
}

Poly xpow(uint64_t k) {  // x^k mod P
  std::call_once(g_fast_once, build_fast);
  Poly r = {{1, 0, 0, 0}};
  bool one = true;
  for (int i = 0; i < 64; ++i) {
    if (!((k >> i) & 1)) continue;
    r = one ? g_fast->pow2[i] : mulmod_fast(r, g_fast->pow2[i]);
    one = false;
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
  Poly q = xpow(block_words);  // x^(R^r * B) for the current level r (builds g_fast)
  for (int r = 0; r < levels; ++r) {
    Poly pd = q;
    for (int d = 1; d < R; ++d) {
      std::memcpy(out + ((size_t)r * (R - 1) + d - 1) * 4, pd.w, sizeof pd.w);
      pd = mulmod_fast(pd, q);
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
