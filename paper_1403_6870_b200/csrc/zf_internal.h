// zf_internal.h -- host-side plumbing shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "zf_device.cuh"

namespace zf {
// Request-table staging for zf_fill_batch: a ring of pinned host + device
// buffer pairs reused across calls (no cudaMallocAsync and no pageable copy
// per call).  A slot is refilled only after the event recorded behind the
// launches that read it has completed.
struct BatchStage {
  unsigned char* host = nullptr;  // pinned
  unsigned char* dev = nullptr;
  size_t cap = 0;
  cudaEvent_t done = nullptr;
};
constexpr int kStageSlots = 2;
struct StageRing {
  std::mutex mu;
  BatchStage slot[kStageSlots];
  int next = 0;
};
}  // namespace zf

struct zf_tables {
  int kind;  // zf::kKindModified or zf::kKindTraditional
  int device;
  int sm_count;
  zf::DevTables* dev;  // device copy: half-normal pack then exponential pack
  zf::DevTables host;  // host mirror (used by tests of the pack layout)
  mutable zf::StageRing stage;
};

namespace zf {

// status helpers
inline int cuda_status(cudaError_t e) { return e == cudaSuccess ? ZF_OK : (int)e; }
#define ZF_TRY(expr)                                \
  do {                                              \
    cudaError_t _e = (expr);                        \
    if (_e != cudaSuccess) return (int)_e;          \
  } while (0)
#define ZF_TRY_STATUS(expr)                         \
  do {                                              \
    int _s = (expr);                                \
    if (_s != ZF_OK) return _s;                     \
  } while (0)

// Makes the handle's device current for the scope of a call and restores the
// caller's device afterwards, so a handle works whatever device is current.
class DeviceGuard {
 public:
  explicit DeviceGuard(int device) {
    if (cudaGetDevice(&prev_) == cudaSuccess && prev_ != device) {
      status_ = cudaSetDevice(device);
      switched_ = status_ == cudaSuccess;
    }
  }
  ~DeviceGuard() {
    if (switched_) cudaSetDevice(prev_);
  }
  cudaError_t status() const { return status_; }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;

 private:
  int prev_ = -1;
  bool switched_ = false;
  cudaError_t status_ = cudaSuccess;
};
#define ZF_ON_DEVICE(t)                               \
  zf::DeviceGuard zf_guard_((t)->device);             \
  if (zf_guard_.status() != cudaSuccess) return (int)zf_guard_.status()

constexpr uint64_t kMaxCtr = 1ull << 44;  // primary counter range (see zf_device.cuh)

constexpr int kKindModified = 0;
constexpr int kKindTraditional = 1;
// a dist code must match the algorithm of the handle's packs
inline int check_kind(const zf_tables* t, int dist) {
  if (dist != ZF_EXP && dist != ZF_NORMAL && dist != ZF_TRAD_EXP && dist != ZF_TRAD_NORMAL)
    return ZF_EDIST;
  const bool trad = dist == ZF_TRAD_EXP || dist == ZF_TRAD_NORMAL;
  return trad == (t->kind == kKindTraditional) ? ZF_OK : ZF_ETABLE;
}

// launchers (zf_fill.cu)
int launch_fill(const zf_tables* t, int dist, int dtype, uint64_t seed, uint64_t ctr_base,
                void* out, uint64_t n, int64_t* counters, cudaStream_t s);
int launch_fill_batch(const zf_tables* t, const zf_request* reqs, int nreq, int dtype, void* out,
                      cudaStream_t s);
int batch_create(const zf_tables* t, const zf_request* reqs, int nreq, int dtype, zf_batch** out);
int batch_fill(const zf_batch* b, void* out, cudaStream_t s);
int batch_destroy(zf_batch* b);
// launchers (zf_stats.cu)
int launch_fill_stats(const zf_tables* t, int dist, uint64_t seed, uint64_t ctr_base, uint64_t n,
                      const zf_stats_cfg* cfg, double* partials, unsigned long long* counts,
                      cudaStream_t s);
int launch_stats(int dtype, const void* x, uint64_t n, const zf_stats_cfg* cfg, double* partials,
                 unsigned long long* counts, cudaStream_t s);
uint32_t stats_blocks(uint64_t n);
// launchers (zf_replay.cu)
int run_replay(const zf_tables* t, int dist, int dtype, const uint64_t* words, uint64_t nwords,
               uint64_t cursor, int wrap, void* out, uint64_t n, zf_path_rec* recs,
               int64_t* counters, uint64_t* consumed, cudaStream_t s);
int launch_words(int gid, const uint64_t* state, uint64_t n, uint64_t* out, cudaStream_t s);
// one oracle-mode window of L words generated from state (gid 0/1) and
// classified in the same pass; ZF_ESHORT when L was too short for n samples
int run_generated(const zf_tables* t, int dist, int dtype, int gid, const uint64_t st[4],
                  uint64_t L, void* out, uint64_t n, zf_path_rec* recs, int64_t* counters,
                  uint64_t* consumed, cudaStream_t s);
// launchers (zf_format.cu)
uint64_t format_blocks(uint64_t n);
int launch_format_g17(const double* x, uint64_t n, char* out, uint64_t cap, uint64_t* scratch,
                      cudaStream_t s);
// xoshiro jump-ahead (zf_jump.cpp)
void xoshiro_jump_host(uint64_t st[4], uint64_t k);
// x^(d * R^r * B) mod P for r < levels, d = 1..R-1, R = 2^bits:
// levels x (R - 1) x 4 words
void xoshiro_radix_polys(uint64_t block_words, int bits, int levels, uint64_t* out);

}  // namespace zf
