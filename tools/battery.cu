// battery.cu -- generator-level statistical battery for the production word
// function (validation tooling, not product code; driven by tools/battery.py).
//
// Words of the counter stream: w_K = f(seed + (K + 1) * gamma), gamma =
// 0x9E3779B97F4A7C15 (the Weyl sequence of splitmix64), f = the word function
// under test: FN 0 = splitmix64's mix13 (Stafford variant 13), FN 1 =
// MurmurHash3's fmix64.  Every test accumulates cell counts in shared memory
// per block and adds them to a global table; tools/battery.py turns the
// tables into chi-square statistics and p-values.
//
//   bat_avalanche  f(z) ^ f(z ^ 2^b) for 64 input bits b, 64x64 flip counts
//   bat_stream     kind 0: monobit counts of the 64 bit positions
//                  kind 1: (top 6 bits of w_K, top 6 bits of w_{K+lag})   4096 cells
//                  kind 2: (low byte >> 2 of w_K, low byte >> 2 of w_{K+lag}) 4096 cells
//                  kind 3: (low byte >> 2, top 6 bits) of the same word    4096 cells
//                  kind 4: Hamming-weight classes of w_K, w_{K+lag}, w_{K+2 lag}  125 cells
//                  kind 5: low-nibble triples of w_K, w_{K+lag}, w_{K+2 lag}     4096 cells
//                  kind 6: top 12 bits of w_K (uniformity)                        4096 cells
//                  kind 7: gaps between words with low byte == 0xFF (the sampler's
//                          rarest layer), lengths 0..4094 and >= 4095        4096 cells
#include <cstdint>
#include <cuda_runtime.h>

namespace {
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix13(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdull;
  z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ull;
  return z ^ (z >> 33);
}
template <int FN>
__device__ __forceinline__ uint64_t word(uint64_t z) {
  return FN == 0 ? mix13(z) : fmix64(z);
}

__device__ __forceinline__ int hw_class(uint64_t w) {
  const int h = __popcll(w);
  return h <= 28 ? 0 : h <= 31 ? 1 : h == 32 ? 2 : h <= 35 ? 3 : 4;
}

template <int FN>
__global__ void avalanche_kernel(uint64_t seed, uint64_t m, unsigned long long* out) {
  __shared__ unsigned int cnt[64 * 64];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const uint64_t z = seed + (i + 1) * kGamma;
    const uint64_t f0 = word<FN>(z);
    for (int b = 0; b < 64; ++b) {
      uint64_t d = f0 ^ word<FN>(z ^ (1ull << b));
      while (d) {
        const int o = __ffsll((long long)d) - 1;
        d &= d - 1;
        atomicAdd(&cnt[b * 64 + o], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4096; i += blockDim.x)
    if (cnt[i]) atomicAdd(out + i, (unsigned long long)cnt[i]);
}

template <int FN, int KIND>
__global__ void stream_kernel(uint64_t seed, uint64_t k0, uint64_t n, uint64_t lag,
                              unsigned long long* out) {
  __shared__ unsigned int cnt[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  if (KIND == 7) {
    // each thread owns a contiguous segment and counts every gap that STARTS
    // at an event inside it, scanning past the segment end to close the last
    // one (so no gap length is truncated by the segmentation)
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t seg = (n + nt - 1) / nt;
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t a = k0 + t * seg, b = min(k0 + n, a + seg);
    int64_t last = -1;
    for (uint64_t k = a; a < b; ++k) {
      if (k >= b && (last < 0 || k - (uint64_t)last > 4095)) {
        if (last >= 0) atomicAdd(&cnt[4095], 1u);  // open gap beyond the last cell
        break;
      }
      if ((word<FN>(seed + (k + 1) * kGamma) & 0xFF) == 0xFF) {
        if (last >= 0) {
          const uint64_t g = k - (uint64_t)last - 1;
          atomicAdd(&cnt[g < 4095 ? g : 4095], 1u);
        }
        if (k >= b) break;
        last = (int64_t)k;
      }
    }
  } else {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      const uint64_t k = k0 + i;
      const uint64_t w = word<FN>(seed + (k + 1) * kGamma);
      if (KIND == 0) {
        uint64_t d = w;
        while (d) {
          const int o = __ffsll((long long)d) - 1;
          d &= d - 1;
          atomicAdd(&cnt[o], 1u);
        }
      } else if (KIND == 1) {
        const uint64_t v = word<FN>(seed + (k + lag + 1) * kGamma);
        atomicAdd(&cnt[(w >> 58) * 64 + (v >> 58)], 1u);
      } else if (KIND == 2) {
        const uint64_t v = word<FN>(seed + (k + lag + 1) * kGamma);
        atomicAdd(&cnt[((w & 0xFF) >> 2) * 64 + ((v & 0xFF) >> 2)], 1u);
      } else if (KIND == 3) {
        atomicAdd(&cnt[((w & 0xFF) >> 2) * 64 + (w >> 58)], 1u);
      } else if (KIND == 4) {
        const uint64_t v = word<FN>(seed + (k + lag + 1) * kGamma);
        const uint64_t u = word<FN>(seed + (k + 2 * lag + 1) * kGamma);
        atomicAdd(&cnt[hw_class(w) * 25 + hw_class(v) * 5 + hw_class(u)], 1u);
      } else if (KIND == 5) {
        const uint64_t v = word<FN>(seed + (k + lag + 1) * kGamma);
        const uint64_t u = word<FN>(seed + (k + 2 * lag + 1) * kGamma);
        atomicAdd(&cnt[(w & 0xF) * 256 + (v & 0xF) * 16 + (u & 0xF)], 1u);
      } else if (KIND == 6) {
        atomicAdd(&cnt[w >> 52], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4096; i += blockDim.x)
    if (cnt[i]) atomicAdd(out + i, (unsigned long long)cnt[i]);
}

template <int FN>
int launch_stream(int kind, uint64_t seed, uint64_t k0, uint64_t n, uint64_t lag,
                  unsigned long long* out, int grid) {
  switch (kind) {
#define K(X) \
  case X: stream_kernel<FN, X><<<grid, 256>>>(seed, k0, n, lag, out); break;
    K(0) K(1) K(2) K(3) K(4) K(5) K(6) K(7)
#undef K
    default: return -1;
  }
  return (int)cudaGetLastError();
}
}  // namespace

extern "C" {
// counts_dev: 4096 u64 cells, accumulated (zero them first)
int bat_avalanche(int fn, uint64_t seed, uint64_t m, unsigned long long* counts_dev, int grid) {
  if (fn == 0) avalanche_kernel<0><<<grid, 256>>>(seed, m, counts_dev);
  else avalanche_kernel<1><<<grid, 256>>>(seed, m, counts_dev);
  return (int)cudaGetLastError();
}
int bat_stream(int fn, int kind, uint64_t seed, uint64_t k0, uint64_t n, uint64_t lag,
               unsigned long long* counts_dev, int grid) {
  return fn == 0 ? launch_stream<0>(kind, seed, k0, n, lag, counts_dev, grid)
                 : launch_stream<1>(kind, seed, k0, n, lag, counts_dev, grid);
}
}
