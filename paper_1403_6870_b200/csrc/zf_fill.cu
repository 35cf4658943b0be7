// zf_fill.cu -- production-mode fill (zf_fill) and the batched variant.
//
// Replaces the hot loops fill_exp (_kernels.py:226-260) and fill_normal
// (_kernels.py:597-689) for the counter stream.  Work decomposition: 256-thread
// CTAs, every warp walks tiles of kTile consecutive samples (zf_tile.cuh):
//
//   pass 1 (fast):  lane l, iteration it, element e handles sample
//                   base + it*32*V + l*V + e   (V = 16 B / sizeof(out))
//                   -> one counter-stream word (fmix64), one LDS.64 + I2F + DMUL, then a
//                   128-bit store per iteration (the warp writes 512 contiguous
//                   bytes per store instruction).  Exceptional samples are
//                   flagged by the NaN sentinel of the smem table.
//   pass 2 (rare):  the flagged samples are queued per warp across tiles and
//                   resolved 32 at a time (one per lane) on their secondary
//                   counter streams; results patch lines still held in L2.
// The modified fp64 fills (and the fp32 exponential) run pass 1 on two
// adjacent tiles before one round of queue bookkeeping; the grid gives every
// warp ~32 tiles (round-2 log).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <new>
#include <type_traits>
#include <vector>

#include "zf_internal.h"
#include "zf_tile.cuh"

namespace zf {

// the per-warp queues (and their 16-byte round scratch) follow the staged packs
static_assert(sizeof(DevPack) % 16 == 0 && sizeof(DevTables) % 16 == 0, "queue alignment");

// Default pass-2 policy (measured): recursive rounds of 32 have
// the smallest code and register footprint and win for both distributions.
template <int DIST, bool COUNTED>
constexpr int default_pass2() {
  return 3;
}

#ifndef ZF_MIN_BLOCKS
#define ZF_MIN_BLOCKS 1  // CTAs per SM requested from the register allocator
#endif

// fill kernels whose queue bookkeeping runs per pair of tiles (measured: the
// modified fp64 fills and the fp32 exponential gain, the traditional kernels
// and the fp32 normal lose -- DESIGN.md round-2 log)
#ifndef ZF_FILL_NT
// tiles per queue bookkeeping in the paired fill kernels (4: 64-bit lane masks
// and four inlined pass-1 bodies -- 612 vs 772 G/s, measured and dropped)
#define ZF_FILL_NT 2
#endif
template <int DIST, typename OutT>
constexpr bool kFillPaired =
    ZF_PAIR && !kTrad<DIST> && (std::is_same<OutT, double>::value || DIST == ZF_EXP);

template <int DIST, typename OutT, bool COUNTED, bool VEC, int P2>
__global__ void __launch_bounds__(kFillThreads, ZF_MIN_BLOCKS)
    fill_ctr_kernel(const DevTables* __restrict__ gt, uint64_t seed, uint64_t ctr_base,
                    OutT* __restrict__ out, uint64_t n, unsigned long long* __restrict__ counters) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kPacks = kPacksOf<DIST>;
  DevPack* sp = reinterpret_cast<DevPack*>(smem_raw);
  const int lane = threadIdx.x & 31;
  uint32_t* queue = reinterpret_cast<uint32_t*>(smem_raw + kPacks * sizeof(DevPack)) +
                    (threadIdx.x >> 5) * kQueueWords;
  const uint64_t* late = nullptr;
#if ZF_ASYNC_STAGE
  __shared__ uint64_t bars[2];
  if constexpr (!kTrad<DIST>) {
    // pass 1 reads only sx; everything after it is for the rounds
    stage_split(sp, primary_pack<DIST>(gt), (int)sizeof(sp->sx), kPacks * (int)sizeof(DevPack),
                bars);
    late = &bars[1];
  } else {
    stage_block(sp, primary_pack<DIST>(gt), kPacks * (int)sizeof(DevPack));
    __syncthreads();
  }
#else
  stage_block(sp, primary_pack<DIST>(gt), kPacks * (int)sizeof(DevPack));
  __syncthreads();
#endif
  const DevPack& P = sp[0];
  const DevPack& E = sp[kPacks - 1];

  LaneCounts lc;
  StoreSink<OutT, VEC> sink{out};
#if defined(ZF_CHECKS) && ZF_CHECKS
  sink.n_check = n;
#endif
  // modified fp64 fills (and fp32 exponential) pair adjacent tiles: warp w
  // takes tiles 2w, 2w + 1, then 2w + 2W, 2w + 2W + 1, ...
  constexpr int kNT = kFillPaired<DIST, OutT> ? ZF_FILL_NT : 1;  // adjacent tiles per warp step
  const uint64_t w = (uint64_t)blockIdx.x * kFillWarps + (threadIdx.x >> 5);
  const uint64_t nw = (uint64_t)gridDim.x * kFillWarps;
  run_tiles<DIST, COUNTED, P2, StoreSink<OutT, VEC>, kNT>(P, E, seed, ctr_base, sink, n, kNT * w,
                                                         kNT * nw, queue, lane, lc, late,
                                                         kNT > 1 ? 1 : 0);
  if (COUNTED) flush_counts(lc, counters);
}

// ---------------------------------------------------------------------------
// batched requests (config 4): one launch; every request is cut into chunks
// of kBatchChunk tiles, a warp takes whole chunks (chunk -> request from a
// host-built map, one load) and runs them like a fill -- the per-warp queue
// spans the chunk's tiles, so pass-2 rounds are mostly full.  Both packs
// staged; one resident wave so every warp gets ~equal numbers of chunks.
// ---------------------------------------------------------------------------

#ifndef ZF_BATCH_CHUNK
#define ZF_BATCH_CHUNK 4
#endif
constexpr int kBatchChunk = ZF_BATCH_CHUNK;  // tiles per chunk (2048 samples at kTile 512)

struct DevRequest {
  uint64_t seed, ctr_base, n, out_offset;
  uint64_t chunk_begin;  // prefix of chunks
  int32_t dist, pad;
};

#ifndef ZF_BATCH_WAVES
#define ZF_BATCH_WAVES 1  // resident waves of the batch kernel
#endif
#ifndef ZF_BATCH_PREFETCH
#define ZF_BATCH_PREFETCH 1  // load the next chunk's request ahead
#endif
#ifndef ZF_BATCH_MIN_BLOCKS
#define ZF_BATCH_MIN_BLOCKS 1
#endif

template <typename OutT, bool VEC>
__global__ void __launch_bounds__(kThreads, ZF_BATCH_MIN_BLOCKS)
    fill_batch_kernel(const DevTables* __restrict__ gt, const DevRequest* __restrict__ reqs,
                      const uint32_t* __restrict__ chunk_req, uint64_t total_chunks,
                      OutT* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DevTables* st = reinterpret_cast<DevTables*>(smem_raw);
  stage_block(st, gt, (int)sizeof(DevTables));
  const int lane = threadIdx.x & 31;
  uint32_t* queue =
      reinterpret_cast<uint32_t*>(smem_raw + sizeof(DevTables)) + (threadIdx.x >> 5) * kQueueWords;
  __syncthreads();
  LaneCounts lc;
  const uint64_t nw = (uint64_t)gridDim.x * kWarps;
  uint64_t chunk = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
#if ZF_BATCH_PREFETCH
  // the next chunk's request is loaded while this one runs (two dependent
  // global loads per chunk would otherwise stall the warp before pass 1)
  DevRequest nr{};
  if (chunk < total_chunks) nr = reqs[__ldg(chunk_req + chunk)];
#endif
  for (; chunk < total_chunks; chunk += nw) {
#if ZF_BATCH_PREFETCH
    const DevRequest r = nr;
    if (chunk + nw < total_chunks) nr = reqs[__ldg(chunk_req + chunk + nw)];
#else
    const DevRequest r = reqs[__ldg(chunk_req + chunk)];
#endif
    const uint64_t t0 = (chunk - r.chunk_begin) * kBatchChunk;
    // tiles [t0, t0 + kBatchChunk) of the request: cap n at the chunk's end
    const uint64_t n_eff = std::min<uint64_t>(r.n, (t0 + kBatchChunk) * kTile);
    StoreSink<OutT, VEC> sink{out + r.out_offset};
    if (r.dist == ZF_EXP)
      run_tiles<ZF_EXP, false, 3>(st->ex, st->ex, r.seed, r.ctr_base, sink, n_eff, t0, 1, queue,
                                  lane, lc);
    else
      run_tiles<ZF_NORMAL, false, 3>(st->hn, st->ex, r.seed, r.ctr_base, sink, n_eff, t0, 1,
                                     queue, lane, lc);
  }
}

// ---------------------------------------------------------------------------
// launch plumbing
// ---------------------------------------------------------------------------

template <typename K>
static int grid_for(K kernel, size_t smem, int sm_count, uint64_t ntiles, int* grid,
                    int fixed_waves = 0, int threads = kThreads, bool paired = false) {
  static_assert(sizeof(K) > 0, "");
  // the shared-memory attribute and the occupancy query once per (device,
  // kernel, shared memory): ~5 us of driver calls a small fill would pay on
  // every launch
  int dev = 0;
  ZF_TRY(cudaGetDevice(&dev));
  const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(kernel), smem, threads);
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, size_t, int>, int> cache;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) per_sm = it->second;
  }
  if (!per_sm) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return (int)e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (e != cudaSuccess) return (int)e;
    per_sm = std::max(per_sm, 1);
    std::lock_guard<std::mutex> lock(mu);
    cache[key] = per_sm;
  }
  const uint64_t want = (ntiles + threads / 32 - 1) / (threads / 32);
  // ZF_GRID_WAVES=w overrides the number of resident waves per launch.  By
  // default every warp gets ~kTilesPerWarp tiles: a warp that walks hundreds
  // of grid-strided tiles drifts away from the other resident warps, and the
  // write front spreads over more DRAM pages; many short-lived CTAs pay for
  // their table staging and drain.  Measured on B200 (tools/ab_waves_sweep.sh,
  // normal / exp G samples/s, tiles per warp in brackets): 2^32 samples 12
  // waves 735 / 773 (295), 48 waves 755 / 794 (74), 192 waves 727 / 773 (18);
  // 2^30 8 waves 713 / 764 (110), 12 waves 739 / 787 (74); 2^28 3-6 waves
  // 720 / 764 (74-37), 8 waves 711 / 760; 2^26 1 wave 660 / 701, 4 waves
  // 645 / 694.
  // (with paired tiles the optimum is ~32 tiles = 16 pairs per warp: 2^32
  // samples 55 / 110 / 220 waves 749 / 770 / 745 normal, 793 / 817 / 802 exp;
  // 2^28 6 / 12 / 24 waves 709 / 723 / 689)
  const uint64_t kTilesPerWarp = paired ? 32 : 64;
  static const int env_waves = [] {
    const char* e = getenv("ZF_GRID_WAVES");
    return e ? std::max(1, atoi(e)) : 0;
  }();
  const uint64_t resident_warps = (uint64_t)per_sm * sm_count * (threads / 32);
  const int waves =
      fixed_waves ? fixed_waves
      : env_waves ? env_waves
                  : (int)std::max<uint64_t>(
                        1, (ntiles + resident_warps * kTilesPerWarp / 2) /
                               (resident_warps * kTilesPerWarp));
  *grid = (int)std::min<uint64_t>(want, (uint64_t)per_sm * sm_count * waves);
  // a queue entry holds a warp's loop iteration in 22 bits: never give a warp
  // 2^21 or more tiles (only an enormous fill with ZF_GRID_WAVES set low could)
  const uint64_t min_grid = (ntiles + (uint64_t)(threads / 32) * (1ull << 21) - 1) /
                            ((uint64_t)(threads / 32) * (1ull << 21));
  if ((uint64_t)*grid < min_grid) *grid = (int)std::min<uint64_t>(min_grid, want);
  if (*grid < 1) *grid = 1;
  return ZF_OK;
}

// ZF_PASS2=9 (debug only) runs pass 1 alone to isolate the cost of pass 2.
static int pass2_override() {
  static const int p = [] {
    const char* e = getenv("ZF_PASS2");
    return e ? atoi(e) : 0;
  }();
  return p;
}

template <int DIST, typename OutT, bool COUNTED, bool VEC>
static int launch_typed(const zf_tables* t, uint64_t seed, uint64_t ctr_base, OutT* out,
                        uint64_t n, unsigned long long* counters, cudaStream_t s) {
  constexpr int kPacks = kPacksOf<DIST>;
  auto kernel = fill_ctr_kernel<DIST, OutT, COUNTED, VEC, default_pass2<DIST, COUNTED>()>;
  if constexpr (!COUNTED && !kTrad<DIST>) {
    const int p2 = pass2_override();
    if (p2 == 3) kernel = fill_ctr_kernel<DIST, OutT, false, VEC, 3>;
    if (p2 == 9) kernel = fill_ctr_kernel<DIST, OutT, false, VEC, 9>;
  }
#ifndef ZF_SMEM_PAD
#define ZF_SMEM_PAD 0  // experiment builds: extra shared memory per CTA (limits CTAs per SM)
#endif
  const size_t smem = kPacks * sizeof(DevPack) +
                      (size_t)kFillWarps * kQueueWords * sizeof(uint32_t) + ZF_SMEM_PAD;
  int grid = 0;
  ZF_TRY_STATUS(grid_for(kernel, smem, t->sm_count, (n + kTile - 1) / kTile, &grid, 0,
                         kFillThreads, kFillPaired<DIST, OutT>));
  kernel<<<grid, kFillThreads, smem, s>>>(t->dev, seed, ctr_base, out, n, counters);
  return cuda_status(cudaGetLastError());
}

template <int DIST, typename OutT>
static int launch_dist(const zf_tables* t, uint64_t seed, uint64_t ctr_base, void* out,
                       uint64_t n, int64_t* counters, cudaStream_t s) {
  OutT* o = static_cast<OutT*>(out);
  const bool vec = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  auto* c = reinterpret_cast<unsigned long long*>(counters);
  if (counters)
    return vec ? launch_typed<DIST, OutT, true, true>(t, seed, ctr_base, o, n, c, s)
               : launch_typed<DIST, OutT, true, false>(t, seed, ctr_base, o, n, c, s);
  return vec ? launch_typed<DIST, OutT, false, true>(t, seed, ctr_base, o, n, c, s)
             : launch_typed<DIST, OutT, false, false>(t, seed, ctr_base, o, n, c, s);
}

int launch_fill(const zf_tables* t, int dist, int dtype, uint64_t seed, uint64_t ctr_base,
                void* out, uint64_t n, int64_t* counters, cudaStream_t s) {
  ZF_TRY_STATUS(check_kind(t, dist));
  if (n == 0) return ZF_OK;
  if (dist == ZF_EXP && dtype == ZF_F64)
    return launch_dist<ZF_EXP, double>(t, seed, ctr_base, out, n, counters, s);
  if (dist == ZF_EXP && dtype == ZF_F32)
    return launch_dist<ZF_EXP, float>(t, seed, ctr_base, out, n, counters, s);
  if (dist == ZF_NORMAL && dtype == ZF_F64)
    return launch_dist<ZF_NORMAL, double>(t, seed, ctr_base, out, n, counters, s);
  if (dist == ZF_NORMAL && dtype == ZF_F32)
    return launch_dist<ZF_NORMAL, float>(t, seed, ctr_base, out, n, counters, s);
  if (dist == ZF_TRAD_EXP && dtype == ZF_F64)
    return launch_dist<ZF_TRAD_EXP, double>(t, seed, ctr_base, out, n, counters, s);
  if (dist == ZF_TRAD_EXP && dtype == ZF_F32)
    return launch_dist<ZF_TRAD_EXP, float>(t, seed, ctr_base, out, n, counters, s);
  if (dist == ZF_TRAD_NORMAL && dtype == ZF_F64)
    return launch_dist<ZF_TRAD_NORMAL, double>(t, seed, ctr_base, out, n, counters, s);
  if (dist == ZF_TRAD_NORMAL && dtype == ZF_F32)
    return launch_dist<ZF_TRAD_NORMAL, float>(t, seed, ctr_base, out, n, counters, s);
  return ZF_EDIST;
}

template <typename OutT, bool VEC>
static int launch_batch_typed(const zf_tables* t, const DevRequest* dreq,
                              const uint32_t* chunk_req, uint64_t total_chunks, OutT* out,
                              cudaStream_t s) {
  auto kernel = fill_batch_kernel<OutT, VEC>;
  const size_t smem = sizeof(DevTables) + (size_t)kWarps * kQueueWords * sizeof(uint32_t);
  int grid = 0;
  // one resident wave: every warp loops over ~equal numbers of whole chunks
  ZF_TRY_STATUS(grid_for(kernel, smem, t->sm_count, total_chunks, &grid, ZF_BATCH_WAVES));
  kernel<<<grid, kThreads, smem, s>>>(t->dev, dreq, chunk_req, total_chunks, out);
  return cuda_status(cudaGetLastError());
}

// A batch's device image: the request table, then the chunk -> request map.
// Chunk ids: every exponential request's chunks first, then the normal ones --
// a warp strides through the ids, so it switches distribution at most once
// instead of at every chunk (requests usually alternate; with alternating
// chunks a third of the stalls were instruction fetches).
struct BatchShape {
  uint64_t per_dist[2] = {0, 0};
  uint64_t chunks = 0;
  bool vec = true;  // every request keeps the output's 16-byte alignment
  size_t bytes(int nreq) const {
    return sizeof(DevRequest) * (size_t)nreq + sizeof(uint32_t) * chunks;
  }
};

static uint64_t chunks_of(uint64_t n) {
  return ((n + kTile - 1) / kTile + kBatchChunk - 1) / kBatchChunk;
}

static int batch_shape(const zf_request* reqs, int nreq, int dtype, BatchShape* sh) {
  if (dtype != ZF_F64 && dtype != ZF_F32) return ZF_EDIST;
  const size_t esz = dtype == ZF_F64 ? 8 : 4;
  for (int i = 0; i < nreq; ++i) {
    const zf_request& r = reqs[i];
    if (r.dist != ZF_EXP && r.dist != ZF_NORMAL) return ZF_EDIST;
    if (r.ctr_base > kMaxCtr || r.n > kMaxCtr - r.ctr_base) return ZF_ERANGE;
    if ((r.out_offset * esz) & 15) sh->vec = false;
    sh->per_dist[r.dist] += chunks_of(r.n);
  }
  sh->chunks = sh->per_dist[0] + sh->per_dist[1];
  return sh->chunks > 0xFFFFFFFFull ? ZF_ERANGE : ZF_OK;
}

static void batch_write(const zf_request* reqs, int nreq, const BatchShape& sh,
                        unsigned char* dst) {
  DevRequest* h = reinterpret_cast<DevRequest*>(dst);
  uint32_t* cmap = reinterpret_cast<uint32_t*>(dst + sizeof(DevRequest) * (size_t)nreq);
  uint64_t next[2] = {0, sh.per_dist[0]};
  for (int i = 0; i < nreq; ++i) {
    const zf_request& r = reqs[i];
    const uint64_t nc = chunks_of(r.n);
    h[i] = DevRequest{r.seed, r.ctr_base, r.n, r.out_offset, next[r.dist], r.dist, 0};
    for (uint64_t c = 0; c < nc; ++c) cmap[next[r.dist] + c] = (uint32_t)i;
    next[r.dist] += nc;
  }
}

static int launch_batch_image(const zf_tables* t, const unsigned char* dev_image, int nreq,
                              const BatchShape& sh, int dtype, void* out, cudaStream_t s) {
  const DevRequest* dr = reinterpret_cast<const DevRequest*>(dev_image);
  const uint32_t* dm =
      reinterpret_cast<const uint32_t*>(dev_image + sizeof(DevRequest) * (size_t)nreq);
  const bool vec = sh.vec && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (dtype == ZF_F64)
    return vec ? launch_batch_typed<double, true>(t, dr, dm, sh.chunks, (double*)out, s)
               : launch_batch_typed<double, false>(t, dr, dm, sh.chunks, (double*)out, s);
  return vec ? launch_batch_typed<float, true>(t, dr, dm, sh.chunks, (float*)out, s)
             : launch_batch_typed<float, false>(t, dr, dm, sh.chunks, (float*)out, s);
}

// One-shot batch: the image goes through the handle's pinned staging ring.
int launch_fill_batch(const zf_tables* t, const zf_request* reqs, int nreq, int dtype, void* out,
                      cudaStream_t s) {
  if (nreq <= 0) return nreq == 0 ? ZF_OK : ZF_EINVAL;
  if (t->kind != kKindModified) return ZF_ETABLE;
  BatchShape sh;
  ZF_TRY_STATUS(batch_shape(reqs, nreq, dtype, &sh));
  if (sh.chunks == 0) return ZF_OK;
  const size_t bytes = sh.bytes(nreq);
  std::lock_guard<std::mutex> lock(t->stage.mu);
  BatchStage& sl = t->stage.slot[t->stage.next];
  t->stage.next = (t->stage.next + 1) % kStageSlots;
  if (sl.done) ZF_TRY(cudaEventSynchronize(sl.done));  // its previous batch has read it
  if (sl.cap < bytes || !sl.done) {  // (re)allocate; the caller made t->device current
    cudaError_t e = cudaSuccess;
    if (sl.cap < bytes) {
      const size_t cap = std::max<size_t>(bytes + bytes / 2, 1 << 16);
      if (sl.host) cudaFreeHost(sl.host);
      if (sl.dev) cudaFree(sl.dev);
      sl.host = nullptr;
      sl.dev = nullptr;
      sl.cap = 0;
      e = cudaMallocHost(&sl.host, cap);
      if (e == cudaSuccess) e = cudaMalloc(&sl.dev, cap);
      if (e == cudaSuccess) sl.cap = cap;
    }
    if (e == cudaSuccess && !sl.done) e = cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming);
    ZF_TRY(e);
  }
  batch_write(reqs, nreq, sh, sl.host);
  ZF_TRY(cudaMemcpyAsync(sl.dev, sl.host, bytes, cudaMemcpyHostToDevice, s));
  int status = launch_batch_image(t, sl.dev, nreq, sh, dtype, out, s);
  const cudaError_t er = cudaEventRecord(sl.done, s);
  if (status == ZF_OK && er != cudaSuccess) status = (int)er;
  return status;
}

}  // namespace zf

// A batch whose image stays resident on the handle's device: re-filling it is
// a single launch with no host work (zigfast_b200.h: zf_batch_create).
struct zf_batch {
  const zf_tables* t;
  int nreq;
  int dtype;
  zf::BatchShape shape;
  unsigned char* image;  // device
};

namespace zf {

int batch_create(const zf_tables* t, const zf_request* reqs, int nreq, int dtype,
                 zf_batch** out) {
  if (nreq < 0 || (nreq > 0 && !reqs)) return ZF_EINVAL;
  if (t->kind != kKindModified) return ZF_ETABLE;
  BatchShape sh;
  ZF_TRY_STATUS(batch_shape(reqs, nreq, dtype, &sh));
  std::vector<unsigned char> host(std::max<size_t>(sh.bytes(nreq), 16));
  batch_write(reqs, nreq, sh, host.data());
  unsigned char* dev = nullptr;
  ZF_TRY(cudaMalloc(&dev, host.size()));
  const cudaError_t e = cudaMemcpy(dev, host.data(), host.size(), cudaMemcpyHostToDevice);
  zf_batch* b = e == cudaSuccess ? new (std::nothrow) zf_batch{t, nreq, dtype, sh, dev} : nullptr;
  if (!b) {
    cudaFree(dev);
    return e != cudaSuccess ? (int)e : ZF_EINVAL;
  }
  *out = b;
  return ZF_OK;
}

int batch_fill(const zf_batch* b, void* out, cudaStream_t s) {
  if (b->shape.chunks == 0) return ZF_OK;
  return launch_batch_image(b->t, b->image, b->nreq, b->shape, b->dtype, out, s);
}

int batch_destroy(zf_batch* b) {
  const cudaError_t e = cudaFree(b->image);
  delete b;
  return cuda_status(e);
}

}  // namespace zf

extern "C" const zf_tables* zf_batch_tables(const zf_batch* b) { return b ? b->t : nullptr; }

#if defined(ZF_CHECKS) && ZF_CHECKS
// debug builds: the first failed ZF_CHECK of this file's kernels (0 = none); resets it
extern "C" unsigned int zf_debug_check_line_fill(void) {
  unsigned int v = 0, z = 0;
  cudaMemcpyFromSymbol(&v, zf::zf_check_line, sizeof v);
  cudaMemcpyToSymbol(zf::zf_check_line, &z, sizeof z);
  return v;
}
#endif
