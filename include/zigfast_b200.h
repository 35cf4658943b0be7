/*
 * zigfast_b200.h -- C-ABI of the B200 (sm_100a) modified-ziggurat samplers.
 *
 * This is the drop-in boundary for the reference's operator interface: the
 * numba kernels of `zigfast/_kernels.py`, which the Python samplers call with
 * a generator state array, an integer generator id and a flat table pack.
 * Plain pointers and sizes only; device pointers are raw CUDA allocations (a
 * torch tensor's data_ptr() works), `stream` is a cudaStream_t (NULL = legacy
 * default stream).  Every entry point returns 0 on success, a negative
 * ZF_E* code for invalid arguments, or a positive cudaError_t.
 *
 * Devices: a table handle belongs to the device it was created on.  Calls that
 * take a handle make that device current for their duration and restore the
 * caller's current device before returning, so they work whichever device is
 * current; their buffers and stream must belong to the handle's device.
 * Calls without a handle (zf_stats, zf_words, zf_format_g17) run on the
 * caller's current device.
 *
 * Reference interfaces each entry point replaces (file:line under
 * /root/reference/pkg/src/zigfast/):
 *
 *   zf_tables_create   _packs.exp_pack / normal_pack / make_alias      _packs.py:31-64
 *   zf_trad_tables_create  traditional._pack (trad samplers)         traditional.py:113-135
 *   zf_fill            fill_exp / fill_normal (new counter generator)  _kernels.py:226-260, 597-689
 *                      dist ZF_TRAD_*: fill_trad_exp / fill_trad_normal _kernels.py:982-1004, 1149-1176
 *   zf_fill_gid        fill_exp(state, gid, *pack, out) incl. gid 0/1/2  _kernels.py:226-228, 597-600
 *   zf_fill_replay     the same, gid 2 (replay) on a device word buffer _kernels.py:83-88
 *   zf_words           next_block(state, gid, out)                     _kernels.py:91-94
 *   zf_xoshiro_jump    (new) O(log k) skip-ahead of the gid-0 state     uniform.py:93-98
 *   zf_fill_stats      bench_exp / bench_normal + quality sums          _kernels.py:306-393, quality.py:92-106
 *   zf_stats           quality._moment_sums on a device buffer         quality.py:92-106
 *   zf_fill_batch      many (sampler, fill(8192)) requests, one launch  exponential.py:45-50
 *   zf_batch_*         the same with the request table resident on the device
 *   zf_format_g17      gen --format text: f"{v:.17g}\n" per value       cli.py:100-120
 */
#ifndef ZIGFAST_B200_H
#define ZIGFAST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZF_ABI_VERSION 1

/* distributions */
#define ZF_EXP 0    /* Exponential(1)                      */
#define ZF_NORMAL 1 /* N(0,1) = half-normal magnitude + sign */
/* traditional (Marsaglia-Tsang) ziggurat baseline, traditional.py:56-207,
 * _kernels.py:933-1277; needs a handle from zf_trad_tables_create */
#define ZF_TRAD_EXP 2
#define ZF_TRAD_NORMAL 3

/* output element types */
#define ZF_F64 0
#define ZF_F32 1

/* generator ids: 0..2 are the reference's (uniform.py:22-26); 3 is new */
#define ZF_GEN_XOSHIRO256PP 0 /* state[4], sequential stream               */
#define ZF_GEN_SPLITMIX64 1   /* state[1], sequential stream               */
#define ZF_GEN_REPLAY 2       /* state[0] = cursor into a word buffer      */
#define ZF_GEN_CTR 3          /* state[0] = seed, state[1] = sample counter */

/* status codes (negative); positive values are cudaError_t */
#define ZF_OK 0
#define ZF_EINVAL (-1)    /* bad argument                                  */
#define ZF_EDIST (-2)     /* unknown distribution / dtype / generator      */
#define ZF_EALIGN (-3)    /* pointer alignment not supported              */
#define ZF_ERANGE (-4)    /* counter / size outside the supported range   */
#define ZF_ESHORT (-5)    /* replay without wrap ran out of words          */
#define ZF_ETABLE (-6)    /* table pack inconsistent (lmax, slot count)   */
#define ZF_EDEVICE (-7)   /* no sm_100 device / wrong device               */

/* path bits in zf_path_rec.path */
#define ZF_PATH_FAST 1    /* exited through the common (one-word) path     */
#define ZF_PATH_TAIL 2    /* took at least one tail (slot 0) step          */
#define ZF_PATH_BOXFAST 4 /* accepted below the chord minus the band       */
#define ZF_PATH_BOXEVAL 8 /* accepted after a density evaluation          */

/* Flat table pack of one density: the tuple `exp_pack` / `normal_pack`
 * builds (_packs.py:31-60).  Arrays have nslots = lmax + 1 entries, slot 0
 * (tail) unused in the box arrays.  `sx` is X*2^-64 (exp) / X*2^-63 (normal). */
typedef struct zf_table_pack {
  int64_t lmax;
  int64_t nslots;
  const double* sx;
  const double* xlo;
  const double* xw;
  const double* flo;
  const double* fh;
  double eps; /* exp: epsilon_max; normal: 0 (plain rejection) */
  const double* prob;
  const int64_t* alias;
  double tailx; /* X[1] */
} zf_table_pack;

/* Traditional-ziggurat pack: the tuple traditional._pack returns
 * (traditional.py:113-121).  i_max = 256 entries each: se = edge * 2^-64
 * (exp) / 2^-63 (normal), kk = integer fast-accept thresholds
 * (_int_thresholds, traditional.py:99-110), flo/fh = wedge strip [f_{i-1},
 * f_i] (slot 0 unused), r = base abscissa (tail start). */
typedef struct zf_trad_pack {
  int64_t i_max;
  const double* se;
  const uint64_t* kk;
  const double* flo;
  const double* fh;
  double r;
} zf_trad_pack;

/* Per-sample path record (oracle mode). */
typedef struct zf_path_rec {
  uint64_t start;    /* logical word offset of the draw's first word */
  uint32_t nwords;   /* words the draw consumed                      */
  uint8_t layer;     /* low byte of the first word                   */
  uint8_t path;      /* ZF_PATH_* bits                               */
  uint16_t attempts; /* box attempts (or normal tail rounds)         */
} zf_path_rec;

/* One request of a batched fill (config 4): `n` samples of `dist` from the
 * counter stream (seed, ctr_base) written at element offset `out_offset`. */
typedef struct zf_request {
  uint64_t seed;
  uint64_t ctr_base;
  uint64_t n;
  uint64_t out_offset;
  int32_t dist;
  int32_t reserved;
} zf_request;

/* Validation statistics configuration (moments, histogram, tail counts). */
typedef struct zf_stats_cfg {
  double hist_lo;
  double hist_hi;
  int32_t nbins;      /* 0 disables the histogram; counts has nbins + 2 slots (under, over) */
  int32_t nthresh;    /* <= 8 */
  int32_t abs_thresh; /* count |x| > t instead of x > t */
  int32_t moments;    /* 5: x^1..x^5; 1 with no histogram/thresholds: the sum
                         only (aggregate, _kernels.py:306-393); 0: no moments
                         (partials are zero) -- histogram / threshold counts
                         only, and thresholds at or above every fast-path
                         value of the table (e.g. |x| > 5 for N(0,1), x > X[1]
                         for Exp(1)) are then counted on the rare path alone */
  double thresh[8];
} zf_stats_cfg;

typedef struct zf_tables zf_tables; /* opaque, immutable, thread-safe */
typedef struct zf_batch zf_batch;   /* opaque: a request table resident on a device */

int zf_abi_version(void);
const char* zf_strerror(int status);

/* Upload both packs to `device` (the normal sampler needs the exponential pack
 * for its tail).  Either pointer may describe the reference default tables. */
int zf_tables_create(const zf_table_pack* exp_pack, const zf_table_pack* halfnormal_pack,
                     int device, zf_tables** out);
/* Traditional-ziggurat handle (dists ZF_TRAD_EXP / ZF_TRAD_NORMAL only):
 * replaces the per-sampler `_pack` of _TraditionalSampler (traditional.py:124-135). */
int zf_trad_tables_create(const zf_trad_pack* exp_pack, const zf_trad_pack* hn_pack, int device,
                          zf_tables** out);
/* The reference's default tables (default_tables("exponential" /
 * "halfnormal") + make_alias, tables.py:359-372, _packs.py:31-64), or the
 * solved traditional tables (solve_traditional(kind, 256), traditional.py:56-96),
 * embedded in the library: no host-side table code needed. */
int zf_tables_create_default(int device, zf_tables** out);
int zf_trad_tables_create_default(int device, zf_tables** out);
int zf_tables_destroy(zf_tables* t);

/* Production mode: sample k (0 <= k < n) of the call is global sample
 * K = ctr_base + k of the counter stream of `seed`:
 *   words  S(K), S(2^63 + K*2^19), S(2^63 + K*2^19 + 1), ...
 *   S(c) = fmix64(seed + (c+1)*0x9E3779B97F4A7C15)   (MurmurHash3's 64-bit
 *          finalizer on splitmix64's Weyl sequence; the draw body is the
 *          reference's, so any sample can be replayed through it).
 * ctr_base + n must not exceed 2^44.  Asynchronous on `stream`: one kernel
 * launch, no allocation, synchronisation or host round trip, so the call
 * (like zf_batch_fill) may be captured into a CUDA graph; a replay redoes the
 * captured (seed, ctr_base) range.
 * counters_dev (nullable): int64[6] accumulated with the reference's slots. */
int zf_fill(const zf_tables* t, int dist, int dtype, uint64_t seed, uint64_t ctr_base,
            void* out_dev, uint64_t n, int64_t* counters_dev, void* stream);

/* Generate-and-reduce without storing (aggregate / validation at scale):
 * per-block partial sums of x^1..x^5 (fp64, [grid][5], written to
 * partials_dev which must hold zf_stats_blocks(n) * 5 doubles) and integer
 * counts (histogram + thresholds, accumulated into counts_dev). */
int zf_fill_stats(const zf_tables* t, int dist, uint64_t seed, uint64_t ctr_base, uint64_t n,
                  const zf_stats_cfg* cfg, double* partials_dev, unsigned long long* counts_dev,
                  void* stream);

/* Statistics of an existing device buffer (dtype ZF_F64/ZF_F32). */
int zf_stats(int dtype, const void* x_dev, uint64_t n, const zf_stats_cfg* cfg,
             double* partials_dev, unsigned long long* counts_dev, void* stream);
uint32_t zf_stats_blocks(uint64_t n);

/* Oracle mode over a device word buffer with the reference's replay
 * semantics: logical word p is words_dev[(cursor + p) % nwords] if wrap != 0;
 * with wrap == 0 the call fails with ZF_ESHORT instead of wrapping.
 * recs_dev / counters_dev nullable.  *words_consumed receives the number of
 * words the n draws took.  Synchronises `stream`. */
int zf_fill_replay(const zf_tables* t, int dist, int dtype, const uint64_t* words_dev,
                   uint64_t nwords, uint64_t cursor, int wrap, void* out_dev, uint64_t n,
                   zf_path_rec* recs_dev, int64_t* counters_dev, uint64_t* words_consumed,
                   void* stream);

/* The reference's kernel signature: fill n draws from generator `gid`
 * with host `state` updated in place exactly as `fill_exp(state, gid, ...)`
 * would (gid 0: xoshiro256++ state[4]; gid 1: splitmix64 state[1];
 * gid 2: state[0] = cursor, replay words in replay_words_dev/nwords;
 * gid 3: {seed, counter}).  Synchronises `stream` for gid 0..2.  Any n:
 * fills above 2^28 samples are resolved window by window inside the call
 * (with recs_dev, n must stay below 2^31: ZF_ERANGE otherwise). */
int zf_fill_gid(const zf_tables* t, int dist, int dtype, int gid, uint64_t* state,
                const uint64_t* replay_words_dev, uint64_t nwords, void* out_dev, uint64_t n,
                zf_path_rec* recs_dev, int64_t* counters_dev, void* stream);

/* next_block: n words of generator gid (0, 1 or 3) into words_dev, host
 * state advanced by n words.  xoshiro256++ is generated in parallel from
 * GF(2) jump-ahead polynomials.  Asynchronous. */
int zf_words(int gid, uint64_t* state, uint64_t n, uint64_t* words_dev, void* stream);

/* Host-side skip-ahead: state <- T^k state for xoshiro256++. */
int zf_xoshiro_jump(uint64_t* state, uint64_t k);

/* Test hook: x^(2^e) mod P(x), P the characteristic polynomial of the
 * xoshiro256 state transition (e = 128 gives the published jump() constants). */
int zf_xoshiro_pow2_poly(int e, uint64_t* out4);

/* Text output of the reference's `gen --format text` (cli.py:100-120):
 * writes "".join(f"{v:.17g}\n" for v in x) -- byte-identical to CPython's
 * '%.17g' -- for n doubles at x_dev into out_dev (capacity `cap` bytes;
 * 24 * n always suffices).  scratch_dev holds zf_format_scratch_words(n)
 * uint64 words; on completion scratch_dev[0] = total bytes and
 * scratch_dev[1] = values outside the supported domain (0 and
 * 1e-22 <= |v| < 1e17, which contains every sampler output; such values are
 * skipped).  If the total exceeds cap nothing is written.  Asynchronous. */
int zf_format_g17(const double* x_dev, uint64_t n, char* out_dev, uint64_t cap,
                  uint64_t* scratch_dev, void* stream);
uint64_t zf_format_scratch_words(uint64_t n);

/* Batched production fill (many `Sampler(...).fill(n)` requests,
 * exponential.py:45-50): one launch for all requests; request r fills
 * out_dev[out_offset_r ...] with samples ctr_base_r .. ctr_base_r + n_r - 1 of
 * its seed's counter stream.  dtype applies to all requests.  The request
 * table is copied by the call into the handle's pinned staging ring (two
 * slots, reused behind CUDA events), so `reqs` may be freed on return; the
 * call blocks only when the slot it needs still feeds the batch two calls
 * back.  Thread-safe per handle.  Asynchronous otherwise. */
int zf_fill_batch(const zf_tables* t, const zf_request* reqs, int nreq, int dtype,
                  void* out_dev, void* stream);

/* The same batch with its request table uploaded once to the handle's device
 * (synchronously, by zf_batch_create): every zf_batch_fill is then a single
 * launch with no host-side work -- a caller serving the same request layout
 * repeatedly (BatchPlan.fill, batch.py) pays the table build and upload once.
 * The batch keeps a pointer to `t`, which must outlive it. */
int zf_batch_create(const zf_tables* t, const zf_request* reqs, int nreq, int dtype,
                    zf_batch** out);
int zf_batch_fill(const zf_batch* b, void* out_dev, void* stream);
int zf_batch_destroy(zf_batch* b);
const zf_tables* zf_batch_tables(const zf_batch* b);

/* Page-lock (and release) a caller-owned host buffer in place, so fills into
 * it DMA at the link rate: how the Python layer serves `fill(np.empty(n))`
 * (the reference's pageable-array usage, exponential.py:45-50) without a
 * staging copy.  A failed registration leaves no CUDA last-error behind. */
int zf_host_register(void* ptr, uint64_t bytes);
int zf_host_unregister(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* ZIGFAST_B200_H */
