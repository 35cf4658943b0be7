// stores.cu -- HBM write-bandwidth microbenchmark of store patterns (not product
// code): what the fill's pass 1 could reach if it were write-bound.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/stores tools/stores.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// A: the fill's pattern -- a warp owns 512-sample tiles (8 x STG.128 of 512 B),
// tiles grid-strided over warps, 256-thread CTAs
template <int HINT>
__global__ void __launch_bounds__(256) tile_store(double* __restrict__ out, uint64_t n) {
  const uint64_t warps = (uint64_t)gridDim.x * 8;
  const int lane = threadIdx.x & 31;
  for (uint64_t t = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5); t * 512 < n; t += warps) {
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      double2* p = reinterpret_cast<double2*>(out + t * 512 + it * 64 + lane * 2);
      const double2 v = make_double2((double)it, (double)lane);
      if (HINT == 0) *p = v;
      else if (HINT == 1) __stcs(p, v);
      else __stwt(p, v);
    }
  }
}

// B: thread-contiguous grid stride (torch-like elementwise), 4 x 16 B per thread
__global__ void __launch_bounds__(256) flat_store(double* __restrict__ out, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 8;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2; i < n; i += stride) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t j = i + (uint64_t)u * (stride / 4);
      if (j < n) *reinterpret_cast<double2*>(out + j) = make_double2(1.0, 2.0);
    }
  }
}

int main() {
  const uint64_t n = 1ull << 30;  // 8 GiB
  double* out;
  if (cudaMalloc(&out, n * 8) != cudaSuccess) return 1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %7.1f GB/s\n", name, n * 8.0 * 10 / (ms * 1e-3) / 1e9);
  };
  for (int ctas : {2, 3, 4, 8}) {
    for (int waves : {1, 6, 12}) {
      const int grid = sms * ctas * waves;
      char nm[64];
      snprintf(nm, sizeof nm, "tile plain  %d CTA/SM x %2d waves", ctas, waves);
      run(nm, [&] { tile_store<0><<<grid, 256>>>(out, n); });
      snprintf(nm, sizeof nm, "tile .cs    %d CTA/SM x %2d waves", ctas, waves);
      run(nm, [&] { tile_store<1><<<grid, 256>>>(out, n); });
    }
  }
  run("tile .wt    2 CTA/SM x 6 waves", [&] { tile_store<2><<<sms * 12, 256>>>(out, n); });
  for (int g : {1, 2, 4, 8, 32})
    run(g == 1 ? "flat       grid = SMs x 1" : "flat       grid = SMs x g",
        [&] { flat_store<<<sms * g * 8, 256>>>(out, n); });
  return 0;
}
