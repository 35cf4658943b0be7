// pipes.cu -- SASS-level issue / pipe throughput on sm_100a (not product code).
//
// Each test runs 8 independent dependency chains per thread (enough ILP to hide
// the 4-cycle ALU/FMA latency) over 4 CTAs x 8 warps per SM and reports
// cycles per warp-instruction per SMSP (1.0 = one issue slot per cycle;
// 2.0 = the pipe's reciprocal throughput on B300 for ALU / FMA).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/pipes tools/pipes.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);             \
      return 1;                                                                \
    }                                                                          \
  } while (0)

constexpr int kIters = 2048;
constexpr int kChains = 8;

struct Args {
  uint32_t a, b, c, d;  // runtime operands (opaque to ptxas)
  double fa;
};

// one "op" per chain per iteration; OPS = instructions per op (for the report)
#define TEST(NAME, OPS, DECL, BODY, FOLD)                                                    \
  __global__ void __launch_bounds__(256) NAME(Args A, uint32_t* out, long long* cyc) {     \
    DECL;                                                                                  \
    __syncthreads();                                                                       \
    const long long t0 = clock64();                                                        \
    _Pragma("unroll 1") for (int it = 0; it < kIters; ++it) {                              \
      _Pragma("unroll") for (int k = 0; k < kChains; ++k) { BODY; }                        \
    }                                                                                      \
    __syncthreads();                                                                       \
    const long long t1 = clock64();                                                        \
    uint32_t f = 0;                                                                        \
    _Pragma("unroll") for (int k = 0; k < kChains; ++k) { FOLD; }                          \
    if (f == 0x12345678u) out[threadIdx.x] = f;                                            \
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                                       \
  }                                                                                        \
  constexpr int NAME##_ops = OPS;

// ALU: 3-input xor
TEST(t_lop3, 1, uint32_t x[kChains]; for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k,
     asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[k]) : "r"(A.a), "r"(A.b)),
     f ^= x[k])
// ALU: funnel shift
TEST(t_shf, 1, uint32_t x[kChains]; for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k,
     asm volatile("shf.r.wrap.b32 %0, %0, %1, 13;" : "+r"(x[k]) : "r"(A.a)), f ^= x[k])
// FMA pipe: 32-bit multiply-add
TEST(t_imad, 1, uint32_t x[kChains]; for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k,
     asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[k]) : "r"(A.a), "r"(A.b)), f ^= x[k])
// IMAD.WIDE.U32 (64-bit result): chain through the low word, keep hi alive
TEST(t_imadwide, 1, uint32_t x[kChains]; uint32_t h[kChains];
     for (int k = 0; k < kChains; ++k) { x[k] = threadIdx.x + k; h[k] = k; },
     asm volatile("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %0, %2;\n\tmov.b64 {%0, %1}, t;\n\t}"
                  : "+r"(x[k]), "=r"(h[k]) : "r"(A.a)),
     f ^= x[k] ^ h[k])
// IMAD.HI.U32
TEST(t_imadhi, 1, uint32_t x[kChains]; for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k,
     asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[k]) : "r"(A.a), "r"(A.b)), f ^= x[k])
// ALU + FMA interleaved 1:1 (co-issue -> 1.0)
TEST(t_lop3_imad, 2, uint32_t x[kChains]; uint32_t y[kChains];
     for (int k = 0; k < kChains; ++k) { x[k] = threadIdx.x + k; y[k] = 3 * threadIdx.x + k; },
     asm volatile("lop3.b32 %0, %0, %2, %3, 0x96;\n\tmad.lo.u32 %1, %1, %2, %3;"
                  : "+r"(x[k]), "+r"(y[k]) : "r"(A.a), "r"(A.b)),
     f ^= x[k] ^ y[k])
// ALU + IMAD.WIDE 1:1
TEST(t_lop3_wide, 2, uint32_t x[kChains]; uint32_t y[kChains]; uint32_t h[kChains];
     for (int k = 0; k < kChains; ++k) { x[k] = threadIdx.x + k; y[k] = 3 * threadIdx.x + k; h[k] = 0; },
     asm volatile("{\n\t.reg .u64 t;\n\tlop3.b32 %0, %0, %3, %4, 0x96;\n\tmul.wide.u32 t, %1, %3;"
                  "\n\tmov.b64 {%1, %2}, t;\n\t}"
                  : "+r"(x[k]), "+r"(y[k]), "=r"(h[k]) : "r"(A.a), "r"(A.b)),
     f ^= x[k] ^ y[k] ^ h[k])
// ALU + IMAD.HI 1:1
TEST(t_lop3_hi, 2, uint32_t x[kChains]; uint32_t y[kChains];
     for (int k = 0; k < kChains; ++k) { x[k] = threadIdx.x + k; y[k] = 3 * threadIdx.x + k; },
     asm volatile("lop3.b32 %0, %0, %2, %3, 0x96;\n\tmad.hi.u32 %1, %1, %2, %3;"
                  : "+r"(x[k]), "+r"(y[k]) : "r"(A.a), "r"(A.b)),
     f ^= x[k] ^ y[k])
// 64-bit add (IADD3 + IADD3.X)
TEST(t_add64, 2, uint64_t x[kChains]; for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k,
     asm volatile("add.u64 %0, %0, %1;" : "+l"(x[k]) : "l"((uint64_t)A.c << 32 | A.d)),
     f ^= (uint32_t)x[k] ^ (uint32_t)(x[k] >> 32))
// I2F.F64.S64
TEST(t_i2f, 1, double x[kChains]; long long s[kChains];
     for (int k = 0; k < kChains; ++k) { x[k] = 0; s[k] = threadIdx.x + k; },
     asm volatile("{\n\t.reg .f64 t;\n\tcvt.rn.f64.s64 t, %1;\n\tadd.rn.f64 %0, %0, t;\n\t}" : "+d"(x[k]) : "l"(s[k])),
     f ^= (uint32_t)__double_as_longlong(x[k]))
// DMUL
TEST(t_dmul, 1, double x[kChains]; for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k,
     asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(x[k]) : "d"(A.fa)),
     f ^= (uint32_t)__double_as_longlong(x[k]))
// DSETP.NAN + predicated add (the mask idiom)
TEST(t_nanmask, 2, uint32_t x[kChains]; double d[kChains];
     for (int k = 0; k < kChains; ++k) { x[k] = 0; d[k] = threadIdx.x + k; },
     asm volatile("{\n\t.reg .pred p;\n\tsetp.nan.f64 p, %1, %1;\n\t@p or.b32 %0, %0, %2;\n\t}"
                  : "+r"(x[k]) : "d"(d[k]), "r"(A.a)),
     f ^= x[k])
// the same with a predicated IMAD (x = x + bit via mad with an opaque 1)
TEST(t_nanmask_fma, 2, uint32_t x[kChains]; double d[kChains];
     for (int k = 0; k < kChains; ++k) { x[k] = 0; d[k] = threadIdx.x + k; },
     asm volatile("{\n\t.reg .pred p;\n\tsetp.nan.f64 p, %1, %1;\n\t@p mad.lo.u32 %0, %2, %3, %0;\n\t}"
                  : "+r"(x[k]) : "d"(d[k]), "r"(A.a), "r"(A.d)),
     f ^= x[k])

// splitmix64 mix13 as nvcc compiles it (counter + mix), per word
__device__ __forceinline__ uint64_t mix13(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
TEST(t_mix13, 1, uint64_t x[kChains]; for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k,
     x[k] = mix13(x[k] + 0x9E3779B97F4A7C15ull), f ^= (uint32_t)x[k])
// murmur3 fmix64
__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdull;
  z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ull;
  return z ^ (z >> 33);
}
TEST(t_fmix64, 1, uint64_t x[kChains]; for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k,
     x[k] = fmix64(x[k] + 0x9E3779B97F4A7C15ull), f ^= (uint32_t)x[k])

// mix13 with the xorshift high halves on the FMA pipe: z ^ (z >> s) as
// hi' = hi ^ hi>>s (from IMAD.WIDE hi * 2^(32-s)), lo' = lo ^ funnel (SHF)
__device__ __forceinline__ void xs_wide(uint32_t& lo, uint32_t& hi, uint32_t p /*2^(32-s)*/,
                                        int s) {
  uint32_t wl, wh;
  (void)wl;
  asm("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}"
      : "=r"(wl), "=r"(wh) : "r"(hi), "r"(p));
  uint32_t f;
  asm("shf.r.clamp.b32 %0, %1, %2, %3;" : "=r"(f) : "r"(lo), "r"(hi), "r"(s));
  lo ^= f;
  hi ^= wh;
}
template <uint64_t C>
__device__ __forceinline__ void mulc(uint32_t& lo, uint32_t& hi) {
  uint32_t rlo, rhi;
  asm("mul.lo.u32 %0, %2, %4;\n\tmul.hi.u32 %1, %2, %4;\n\tmad.lo.u32 %1, %2, %5, %1;\n\t"
      "mad.lo.u32 %1, %3, %4, %1;"
      : "=&r"(rlo), "=&r"(rhi) : "r"(lo), "r"(hi), "n"((uint32_t)C), "n"((uint32_t)(C >> 32)));
  lo = rlo;
  hi = rhi;
}
__device__ __forceinline__ uint64_t mix13_wide(uint64_t z, const Args& A) {
  uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
  xs_wide(lo, hi, A.a, 30);
  mulc<0xBF58476D1CE4E5B9ull>(lo, hi);
  xs_wide(lo, hi, A.b, 27);
  mulc<0x94D049BB133111EBull>(lo, hi);
  xs_wide(lo, hi, A.c, 31);
  return ((uint64_t)hi << 32) | lo;
}
TEST(t_mix13_wide, 1, uint64_t x[kChains]; for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k,
     x[k] = mix13_wide(x[k] + 0x9E3779B97F4A7C15ull, A), f ^= (uint32_t)x[k])
// the chained 3-IMAD multiply (production) with nvcc's shifts
__device__ __forceinline__ uint64_t mix13_chain(uint64_t z) {
  uint32_t lo, hi;
  z ^= z >> 30;
  lo = (uint32_t)z; hi = (uint32_t)(z >> 32);
  mulc<0xBF58476D1CE4E5B9ull>(lo, hi);
  z = ((uint64_t)hi << 32) | lo;
  z ^= z >> 27;
  lo = (uint32_t)z; hi = (uint32_t)(z >> 32);
  mulc<0x94D049BB133111EBull>(lo, hi);
  z = ((uint64_t)hi << 32) | lo;
  return z ^ (z >> 31);
}
TEST(t_mix13_chain, 1, uint64_t x[kChains]; for (int k = 0; k < kChains; ++k) x[k] = threadIdx.x + k,
     x[k] = mix13_chain(x[k] + 0x9E3779B97F4A7C15ull), f ^= (uint32_t)x[k])
// Philox4x32 round (4 words -> 2 samples), keys opaque
TEST(t_philox_round, 1, uint32_t x0[kChains]; uint32_t x1[kChains]; uint32_t x2[kChains];
     uint32_t x3[kChains];
     for (int k = 0; k < kChains; ++k) { x0[k] = threadIdx.x + k; x1[k] = k; x2[k] = 3 * k; x3[k] = 7; },
     {
       const uint64_t p0 = (uint64_t)x0[k] * 0xD2511F53u;
       const uint64_t p1 = (uint64_t)x2[k] * 0xCD9E8D57u;
       const uint32_t n0 = (uint32_t)(p1 >> 32) ^ x1[k] ^ A.a;
       const uint32_t n2 = (uint32_t)(p0 >> 32) ^ x3[k] ^ A.b;
       x1[k] = (uint32_t)p1; x3[k] = (uint32_t)p0; x0[k] = n0; x2[k] = n2;
     },
     f ^= x0[k] ^ x1[k] ^ x2[k] ^ x3[k])

template <typename K>
static int run(const char* name, K kern, int ops, const Args& a, int sms, int bpsm) {
  uint32_t* out;
  long long* cyc;
  const int grid = sms * bpsm;
  CK(cudaMalloc(&out, 1024 * 4));
  CK(cudaMalloc(&cyc, grid * 8));
  for (int rep = 0; rep < 2; ++rep) kern<<<grid, 256>>>(a, out, cyc);
  CK(cudaDeviceSynchronize());
  long long* h = new long long[grid];
  CK(cudaMemcpy(h, cyc, grid * 8, cudaMemcpyDeviceToHost));
  double mean = 0;
  for (int i = 0; i < grid; ++i) mean += (double)h[i];
  mean /= grid;
  // warps per SMSP = bpsm * 8 / 4
  const double warp_instr_per_smsp = (double)kIters * kChains * ops * (bpsm * 8 / 4);
  printf("%-16s %7.3f cycles per warp-instr per SMSP  (%.1f cycles per op-group)\n", name,
         mean / warp_instr_per_smsp, mean / ((double)kIters * kChains * (bpsm * 8 / 4)));
  delete[] h;
  cudaFree(out);
  cudaFree(cyc);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  Args a{1u << 2, 1u << 5, 1u << 1, 0x01234567u, 1.0000001};
  const int b = 4;
#define R(n) run(#n, n, n##_ops, a, sms, b)
  R(t_lop3); R(t_shf); R(t_imad); R(t_imadwide); R(t_imadhi); R(t_lop3_imad); R(t_lop3_wide);
  R(t_lop3_hi); R(t_add64); R(t_i2f); R(t_dmul); R(t_nanmask); R(t_nanmask_fma); R(t_mix13);
  R(t_mix13_chain); R(t_mix13_wide); R(t_fmix64); R(t_philox_round);
  return 0;
}
