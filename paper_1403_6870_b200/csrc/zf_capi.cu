// zf_capi.cu -- the extern "C" boundary (include/zigfast_b200.h).
//
// Thin: validates arguments, maps them onto the launchers, returns status
// codes.  Tables are immutable after zf_tables_create, so one handle can be
// shared by every host thread that targets its device.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <new>

#include "zf_default_tables.h"
#include "zf_internal.h"

namespace zf {
void xoshiro_pow2_poly(int e, uint64_t out[4]);
}

using namespace zf;

namespace {

int check_pack(const zf_table_pack* p) {
  if (!p || !p->sx || !p->xlo || !p->xw || !p->flo || !p->fh || !p->prob || !p->alias)
    return ZF_EINVAL;
  if (p->lmax < 1 || p->lmax > 255 || p->nslots != p->lmax + 1) return ZF_ETABLE;
  for (int64_t k = 0; k < p->nslots; ++k)
    if (p->alias[k] < 0 || p->alias[k] >= p->nslots) return ZF_ETABLE;
  return ZF_OK;
}

void fill_devpack(const zf_table_pack* p, DevPack* d) {
  std::memset(d, 0, sizeof *d);
  const int n = (int)p->nslots;
  for (int i = 0; i < n; ++i) {
    d->sx[i] = p->sx[i];
    d->xlo[i] = p->xlo[i];
    d->xw[i] = p->xw[i];
    d->flo[i] = p->flo[i];
    d->fh[i] = p->fh[i];
    d->prob[i] = p->prob[i];
    d->alias[i] = (int32_t)p->alias[i];
  }
  d->eps = p->eps;
  d->tailx = p->tailx;
  d->lmax = (int32_t)p->lmax;
  d->nslots = (int32_t)p->nslots;
  // fast-path sentinel: bytes i >= lmax read sx[i+1] = NaN, so the fast value
  // of an exceptional word is NaN (the draw bodies never read these entries)
  for (int i = n; i < (int)(sizeof d->sx / sizeof d->sx[0]); ++i) d->sx[i] = NAN;
}

int check_trad_pack(const zf_trad_pack* p) {
  if (!p || !p->se || !p->kk || !p->flo || !p->fh) return ZF_EINVAL;
  // the kernels index by the low byte of the word (_kernels.py: i = u & MASK8)
  if (p->i_max != kSlots || !(p->r > 0.0)) return ZF_ETABLE;
  return ZF_OK;
}

// traditional pack in the DevPack layout (see zf_device.cuh)
void fill_trad_devpack(const zf_trad_pack* p, DevPack* d) {
  std::memset(d, 0, sizeof *d);
  for (int i = 0; i < kSlots; ++i) {
    d->sx[i + 1] = p->se[i];
    d->kk[i] = p->kk[i];
    d->flo[i] = p->flo[i];
    d->fh[i] = p->fh[i];
  }
  d->tailx = p->r;
  d->lmax = kSlots;
  d->nslots = kSlots;
}

// device checks, pool policy and the upload shared by both table kinds
int upload_tables(zf_tables* t, int device) {
  int ndev = 0;
  ZF_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return ZF_EDEVICE;
  cudaDeviceProp prop;
  ZF_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) return ZF_EDEVICE;  // sm_100a cubin only
  t->device = device;
  t->sm_count = prop.multiProcessorCount;
  t->dev = nullptr;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) {
    // Oracle-mode scratch comes from the device's stream-ordered pool; keep
    // freed blocks cached instead of returning them to the driver at every
    // synchronisation (re-mapping ~1 GB per fill otherwise dominates).
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    e = cudaMalloc(&t->dev, sizeof(DevTables));
  }
  if (e == cudaSuccess) e = cudaMemcpy(t->dev, &t->host, sizeof(DevTables), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    if (t->dev) cudaFree(t->dev);
    t->dev = nullptr;
    return (int)e;
  }
  return ZF_OK;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int zf_abi_version(void) { return ZF_ABI_VERSION; }

const char* zf_strerror(int status) {
  switch (status) {
    case ZF_OK: return "ok";
    case ZF_EINVAL: return "invalid argument";
    case ZF_EDIST: return "unknown distribution, dtype or generator";
    case ZF_EALIGN: return "unsupported pointer alignment";
    case ZF_ERANGE: return "counter or size outside the supported range";
    case ZF_ESHORT: return "replay buffer exhausted (wrap disabled)";
    case ZF_ETABLE: return "inconsistent table pack";
    case ZF_EDEVICE: return "no usable sm_100 device";
    default:
      return status > 0 ? cudaGetErrorString(static_cast<cudaError_t>(status)) : "unknown status";
  }
}

int zf_tables_create(const zf_table_pack* exp_pack, const zf_table_pack* hn_pack, int device,
                     zf_tables** out) {
  if (!out) return ZF_EINVAL;
  *out = nullptr;
  ZF_TRY_STATUS(check_pack(exp_pack));
  ZF_TRY_STATUS(check_pack(hn_pack));
  if (exp_pack->eps < 0.0) return ZF_ETABLE;
  zf_tables* t = new (std::nothrow) zf_tables;
  if (!t) return ZF_EINVAL;
  t->kind = kKindModified;
  fill_devpack(exp_pack, &t->host.ex);
  fill_devpack(hn_pack, &t->host.hn);
  const int rc = upload_tables(t, device);
  if (rc != ZF_OK) {
    delete t;
    return rc;
  }
  *out = t;
  return ZF_OK;
}

int zf_trad_tables_create(const zf_trad_pack* exp_pack, const zf_trad_pack* hn_pack, int device,
                          zf_tables** out) {
  if (!out) return ZF_EINVAL;
  *out = nullptr;
  ZF_TRY_STATUS(check_trad_pack(exp_pack));
  ZF_TRY_STATUS(check_trad_pack(hn_pack));
  zf_tables* t = new (std::nothrow) zf_tables;
  if (!t) return ZF_EINVAL;
  t->kind = kKindTraditional;
  fill_trad_devpack(exp_pack, &t->host.ex);
  fill_trad_devpack(hn_pack, &t->host.hn);
  const int rc = upload_tables(t, device);
  if (rc != ZF_OK) {
    delete t;
    return rc;
  }
  *out = t;
  return ZF_OK;
}

// The reference's default tables, packed at build time (build/gen, see
// _build.generate_default_tables): a non-Python host (cgo, JNI, C) gets the
// drop-in samplers without any table code of its own.
int zf_tables_create_default(int device, zf_tables** out) {
  const zf_table_pack e{kDef_exp_lmax, kDef_exp_lmax + 1, kDef_exp_scale, kDef_exp_xlo,
                        kDef_exp_xw,   kDef_exp_flo,      kDef_exp_fh,    kDef_exp_eps,
                        kDef_exp_prob, kDef_exp_alias,    kDef_exp_tailx};
  const zf_table_pack h{kDef_hn_lmax, kDef_hn_lmax + 1, kDef_hn_scale, kDef_hn_xlo,
                        kDef_hn_xw,   kDef_hn_flo,      kDef_hn_fh,    kDef_hn_eps,
                        kDef_hn_prob, kDef_hn_alias,    kDef_hn_tailx};
  return zf_tables_create(&e, &h, device, out);
}

int zf_trad_tables_create_default(int device, zf_tables** out) {
  const zf_trad_pack e{256, kDef_texp_se, kDef_texp_kk, kDef_texp_flo, kDef_texp_fh,
                       kDef_texp_r};
  const zf_trad_pack h{256, kDef_thn_se, kDef_thn_kk, kDef_thn_flo, kDef_thn_fh, kDef_thn_r};
  return zf_trad_tables_create(&e, &h, device, out);
}

int zf_tables_destroy(zf_tables* t) {
  if (!t) return ZF_OK;
  ZF_ON_DEVICE(t);
  cudaError_t e = cudaFree(t->dev);
  for (auto& sl : t->stage.slot) {
    if (sl.done) cudaEventSynchronize(sl.done), cudaEventDestroy(sl.done);
    if (sl.host) cudaFreeHost(sl.host);
    if (sl.dev) cudaFree(sl.dev);
  }
  delete t;
  return cuda_status(e);
}

int zf_fill(const zf_tables* t, int dist, int dtype, uint64_t seed, uint64_t ctr_base,
            void* out_dev, uint64_t n, int64_t* counters_dev, void* stream) {
  if (!t) return ZF_EINVAL;
  if (n == 0) return ZF_OK;
  if (!out_dev) return ZF_EINVAL;
  if (ctr_base > kMaxCtr || n > kMaxCtr - ctr_base) return ZF_ERANGE;
  const size_t esz = dtype == ZF_F32 ? 4 : 8;
  if (reinterpret_cast<uintptr_t>(out_dev) % esz) return ZF_EALIGN;
  ZF_ON_DEVICE(t);
  return launch_fill(t, dist, dtype, seed, ctr_base, out_dev, n, counters_dev, as_stream(stream));
}

int zf_fill_stats(const zf_tables* t, int dist, uint64_t seed, uint64_t ctr_base, uint64_t n,
                  const zf_stats_cfg* cfg, double* partials_dev, unsigned long long* counts_dev,
                  void* stream) {
  if (!t || !partials_dev || !counts_dev) return ZF_EINVAL;
  if (ctr_base > kMaxCtr || n > kMaxCtr - ctr_base) return ZF_ERANGE;
  ZF_ON_DEVICE(t);
  return launch_fill_stats(t, dist, seed, ctr_base, n, cfg, partials_dev, counts_dev,
                           as_stream(stream));
}

int zf_stats(int dtype, const void* x_dev, uint64_t n, const zf_stats_cfg* cfg,
             double* partials_dev, unsigned long long* counts_dev, void* stream) {
  if ((!x_dev && n) || !partials_dev || !counts_dev) return ZF_EINVAL;
  return launch_stats(dtype, x_dev, n, cfg, partials_dev, counts_dev, as_stream(stream));
}

uint32_t zf_stats_blocks(uint64_t n) { return stats_blocks(n); }

int zf_fill_replay(const zf_tables* t, int dist, int dtype, const uint64_t* words_dev,
                   uint64_t nwords, uint64_t cursor, int wrap, void* out_dev, uint64_t n,
                   zf_path_rec* recs_dev, int64_t* counters_dev, uint64_t* words_consumed,
                   void* stream) {
  if (!t || !words_consumed) return ZF_EINVAL;
  ZF_ON_DEVICE(t);
  return run_replay(t, dist, dtype, words_dev, nwords, cursor, wrap, out_dev, n, recs_dev,
                    counters_dev, words_consumed, as_stream(stream));
}

int zf_words(int gid, uint64_t* state, uint64_t n, uint64_t* words_dev, void* stream) {
  if (!state || (!words_dev && n)) return ZF_EINVAL;
  ZF_TRY_STATUS(launch_words(gid, state, n, words_dev, as_stream(stream)));
  switch (gid) {
    case ZF_GEN_XOSHIRO256PP: xoshiro_jump_host(state, n); break;
    case ZF_GEN_SPLITMIX64: state[0] += n * kGamma; break;
    case ZF_GEN_CTR: state[1] += n; break;
    default: return ZF_EDIST;
  }
  return ZF_OK;
}

int zf_xoshiro_jump(uint64_t* state, uint64_t k) {
  if (!state) return ZF_EINVAL;
  xoshiro_jump_host(state, k);
  return ZF_OK;
}

// x^(2^e) mod P(x) of xoshiro256 (test hook for the published jump constants)
int zf_xoshiro_pow2_poly(int e, uint64_t* out4) {
  if (!out4 || e < 0 || e > 4096) return ZF_EINVAL;
  xoshiro_pow2_poly(e, out4);
  return ZF_OK;
}

int zf_fill_gid(const zf_tables* t, int dist, int dtype, int gid, uint64_t* state,
                const uint64_t* replay_words_dev, uint64_t nwords, void* out_dev, uint64_t n,
                zf_path_rec* recs_dev, int64_t* counters_dev, void* stream) {
  if (!t || !state) return ZF_EINVAL;
  ZF_ON_DEVICE(t);
  cudaStream_t s = as_stream(stream);
  if (gid == ZF_GEN_CTR) {
    if (recs_dev) return ZF_EINVAL;  // production mode has no stream positions
    ZF_TRY_STATUS(zf_fill(t, dist, dtype, state[0], state[1], out_dev, n, counters_dev, stream));
    state[1] += n;
    return ZF_OK;
  }
  if (n == 0) return ZF_OK;
  // One window resolves fewer than 2^31 samples (32-bit positions): a larger
  // fill goes chunk by chunk, each continuing the stream where the previous
  // one stopped, exactly like consecutive fills.  (Per-sample records count
  // their start words from the call's first word, so a recorded fill stays
  // one window.)
  constexpr uint64_t kGidChunk = 1ull << 28;
  if (n > kGidChunk && !recs_dev) {
    if (!out_dev) return ZF_EINVAL;
    const size_t esz = dtype == ZF_F32 ? 4 : 8;
    for (uint64_t off = 0; off < n; off += kGidChunk) {
      const uint64_t m = n - off < kGidChunk ? n - off : kGidChunk;
      ZF_TRY_STATUS(zf_fill_gid(t, dist, dtype, gid, state, replay_words_dev, nwords,
                                static_cast<unsigned char*>(out_dev) + off * esz, m, nullptr,
                                counters_dev, stream));
    }
    return ZF_OK;
  }
  uint64_t consumed = 0;
  if (gid == ZF_GEN_REPLAY) {
    ZF_TRY_STATUS(run_replay(t, dist, dtype, replay_words_dev, nwords, state[0], 1, out_dev, n,
                             recs_dev, counters_dev, &consumed, s));
    state[0] += consumed;
    return ZF_OK;
  }
  if (gid != ZF_GEN_XOSHIRO256PP && gid != ZF_GEN_SPLITMIX64) return ZF_EDIST;
  // sequential generators: materialise a window of the stream on the device,
  // resolve it like a replay without wrap, then advance the host state by
  // exactly the words consumed.  Grow the window if it was too short.
  uint64_t L = n + n / 8 + 4096;
  for (int attempt = 0; attempt < 8; ++attempt, L *= 2) {
    const uint64_t st[4] = {state[0], gid == ZF_GEN_XOSHIRO256PP ? state[1] : 0,
                            gid == ZF_GEN_XOSHIRO256PP ? state[2] : 0,
                            gid == ZF_GEN_XOSHIRO256PP ? state[3] : 0};
    int rc;
    if (L >= (1ull << 22)) {
      // large windows: classify while generating (saves two passes over the
      // window); small ones keep more threads busy in the separate passes
      rc = run_generated(t, dist, dtype, gid, st, L, out_dev, n, recs_dev, counters_dev,
                         &consumed, s);
    } else {
      uint64_t* words = nullptr;
      ZF_TRY(cudaMallocAsync(&words, L * sizeof(uint64_t), s));
      uint64_t st2[4] = {st[0], st[1], st[2], st[3]};
      rc = launch_words(gid, st2, L, words, s);
      if (rc == ZF_OK)
        rc = run_replay(t, dist, dtype, words, L, 0, 0, out_dev, n, recs_dev, counters_dev,
                        &consumed, s);
      cudaFreeAsync(words, s);
    }
    if (rc == ZF_ESHORT) continue;
    ZF_TRY_STATUS(rc);
    if (gid == ZF_GEN_XOSHIRO256PP) xoshiro_jump_host(state, consumed);
    else state[0] += consumed * kGamma;
    return ZF_OK;
  }
  return ZF_ERANGE;
}

uint64_t zf_format_scratch_words(uint64_t n) {
  const uint64_t nb = format_blocks(n);
  return 2 + (nb + 1) + (nb + 1) / 2;
}

int zf_format_g17(const double* x_dev, uint64_t n, char* out_dev, uint64_t cap,
                  uint64_t* scratch_dev, void* stream) {
  if (!scratch_dev || (n && (!x_dev || !out_dev))) return ZF_EINVAL;
  return launch_format_g17(x_dev, n, out_dev, cap, scratch_dev, as_stream(stream));
}

int zf_fill_batch(const zf_tables* t, const zf_request* reqs, int nreq, int dtype,
                  void* out_dev, void* stream) {
  if (!t || (nreq > 0 && (!reqs || !out_dev))) return ZF_EINVAL;
  ZF_ON_DEVICE(t);
  return launch_fill_batch(t, reqs, nreq, dtype, out_dev, as_stream(stream));
}

int zf_host_register(void* ptr, uint64_t bytes) {
  if (!ptr || !bytes) return ZF_EINVAL;
  const cudaError_t e = cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) cudaGetLastError();  // not sticky: leave no last-error behind
  return cuda_status(e);
}

int zf_host_unregister(void* ptr) {
  if (!ptr) return ZF_EINVAL;
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) cudaGetLastError();
  return cuda_status(e);
}

int zf_batch_create(const zf_tables* t, const zf_request* reqs, int nreq, int dtype,
                    zf_batch** out) {
  if (!t || !out) return ZF_EINVAL;
  *out = nullptr;
  ZF_ON_DEVICE(t);
  return batch_create(t, reqs, nreq, dtype, out);
}

int zf_batch_fill(const zf_batch* b, void* out_dev, void* stream) {
  if (!b || !out_dev) return ZF_EINVAL;
  ZF_ON_DEVICE(zf_batch_tables(b));
  return batch_fill(b, out_dev, as_stream(stream));
}

int zf_batch_destroy(zf_batch* b) {
  if (!b) return ZF_OK;
  ZF_ON_DEVICE(zf_batch_tables(b));
  return batch_destroy(b);
}

}  // extern "C"
