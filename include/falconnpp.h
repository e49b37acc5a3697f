/*
 * falconnpp.h -- C ABI of the B200-native Falconn++ hot path (libfalconnpp_b200.so).
 *
 * Drop-in boundary for the reference's index/query API.  The reference
 * (/root/reference) ships only rotation.{hpp,cpp}, dataset.{hpp,cpp} and
 * common.hpp; the index/query layer exists only as SPEC operations and as
 * CMake entries for missing files (proj/CMakeLists.txt:27-31).
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions: plain pointers and sizes, no torch/CUDA types.  Every function
 * returns FPP_OK or one FPP_ERR_* class; fpp_last_error() gives the message of
 * the last failure on the calling thread (the reference throws
 * std::invalid_argument with the same messages, e.g. dataset.cpp:10-18).
 * Host buffers are read/written synchronously before return.  The library owns
 * all device memory behind the opaque fpp_index.  A built index is immutable;
 * concurrent fpp_query calls on one index are allowed: each call
 * leases its own scratch context (own streams), so calls from several host
 * threads run side by side on the device.
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns FPP_ERR_CUDA.
 */
#ifndef FALCONNPP_H
#define FALCONNPP_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPP_ABI_VERSION 6  /* 2: fpp_query_stats.exact, SimHash rerank; 3: fpp_timings.score_bytes;
                              4: fpp_synth_rows, fpp_merge_topk, per-call query contexts;
                              5: fpp_timings.score_launches, fpp_query_probe_sets_device,
                                 fpp_query_from_probe_sets_device;
                              6: fpp_multi_* (single-process multi-GPU index) */

/* error classes ("one exit code per error class") */
#define FPP_OK 0
#define FPP_ERR_INVALID_ARGUMENT 1 /* invalid config: SPEC.md:234-236,249; rotation.cpp:42-49 */
#define FPP_ERR_EMPTY_DATASET 2    /* SPEC.md:249; dataset.cpp:10-11 */
#define FPP_ERR_DIMENSION 3        /* dimension mismatch: SPEC.md:325; dataset.cpp:62-65 */
#define FPP_ERR_OUT_OF_RANGE 4     /* iProbes>NB, qProbes not in [L,L*NB] (:195-197), k>n (:325) */
#define FPP_ERR_NON_FINITE 5       /* dataset.cpp:15-18 */
#define FPP_ERR_ZERO_NORM 6        /* dataset.cpp:32 */
#define FPP_ERR_CUDA 7             /* no device / CUDA runtime failure */
#define FPP_ERR_OUT_OF_MEMORY 8
#define FPP_ERR_UNSUPPORTED 9      /* valid per SPEC but outside the GPU path's envelope */
#define FPP_ERR_FORMAT 10          /* index file: bad magic, truncated, checksum / dataset mismatch
                                       */
#define FPP_ERR_IO 11              /* index file cannot be opened / written */

/* IndexConfig, SPEC.md:233-236 (mode = falconnpp, centering off). */
typedef struct fpp_params {
  uint32_t L;        /* tables >= 1 */
  uint32_t K;        /* concatenated cross-polytope hashes per table: 1 or 2 (SPEC l) */
  uint32_t D;        /* projections per function, power of two, D <= d_pad (one block) */
  uint32_t iprobes;  /* indexing probes, 1 <= iprobes <= NB */
  uint32_t kappa;    /* limit-scaling floor, default 20 */
  float alpha;       /* scaling factor, 0 < alpha <= 1 */
  uint64_t seed;     /* master seed; stack (t,f) uses derive_seed(seed,t,f,0) */
  int32_t device;    /* CUDA device ordinal (-1 = current) */
  uint32_t id_offset;/* global id of local row 0 (sharded builds) */
  uint64_t scratch_bytes; /* build scratch budget per pass (0 = auto) */
  uint32_t centering; /* 1: index the centered dataset (dataset.cpp center();
                         queries are not centered, scores are x'.q -- SPEC.md:358) */
  uint32_t mode;      /* FPP_MODE_FALCONNPP or FPP_MODE_FALCONN_BASELINE */
} fpp_params;

#define FPP_MODE_FALCONNPP 0
#define FPP_MODE_FALCONN_BASELINE 1 /* alpha = 1, iProbes = 1; probes by ascending gap score */

/* SearchResult.stats */
typedef struct fpp_query_stats {
  uint64_t probes;     /* P_q: buckets probed */
  uint64_t entries;    /* E_q: kept entries walked in the probed buckets */
  uint64_t candidates; /* U_q: unique ids collected */
  uint64_t exact;      /* exact inner products computed: U_q, or min(B, U_q) with rerank */
} fpp_query_stats;

/* per-kernel device time accumulated since the last reset (CUDA events) */
typedef struct fpp_timings {
  double hash_ms;     /* build: K1 hashing + histogram */
  double sort_ms;     /* build: scans + scatter + segmented select/sort into CSR */
  double qhash_ms;    /* query: K1 hashing + ranked lists */
  double probe_ms;    /* query: probe selection + directory reads */
  double collect_ms;  /* query: bucket walk + dedup */
  double score_ms;    /* query: row gather + fp64 dot + top-k (K3+K4) */
  uint64_t launches;  /* kernels launched */
  uint64_t score_rows;/* rows gathered by the score kernel */
  uint64_t entries;   /* bucket entries walked */
  uint64_t probes;    /* probes */
  uint64_t score_bytes; /* candidate-row bytes the score kernel read (early termination
                           reads only row prefixes of candidates that cannot reach the top-k) */
  uint64_t score_launches; /* launches of the score kernel (one per query chunk) */
} fpp_timings;

typedef struct fpp_index fpp_index;

int fpp_abi_version(void);
const char* fpp_last_error(void);
void fpp_default_params(fpp_params* p);
int fpp_device_count(void);

/*
 * Index::build (north star build(X,L,K,D,iProbes,alpha)).
 * X: host, row-major n x d fp32, already normalized (dataset.cpp:24-38) --
 * the library never re-normalizes.
 */
int fpp_build(const float* X, uint64_t n, uint32_t d, const fpp_params* p, fpp_index** out);
/* same, X already in device memory of p->device (copied into the index) */
int fpp_build_device(const float* X_dev, uint64_t n, uint32_t d, const fpp_params* p,
                     fpp_index** out);
void fpp_free(fpp_index* idx);

/*
 * Index::query (north star query(Q,k,qProbes)).
 * Q host nq x d; ids [nq*k] (0xFFFFFFFF past min(k,U_q)); scores [nq*k] fp64
 * inner products (-inf past min(k,U_q)), descending, ties by lower id;
 * stats optional [nq].  ids are global (local + id_offset).
 */
int fpp_query(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t k, uint32_t qprobes,
              uint32_t* ids, double* scores, fpp_query_stats* stats);
/* device-resident variant: Q_dev, ids_dev, scores_dev, stats_dev on the index device;
   stream is a cudaStream_t (NULL = the call context's stream), asynchronous w.r.t.
   the host on the walking-screen path (narrow rows, no stats); the collect path
   (other rows, or stats requested) reads back one small word per query chunk (the
   chunk's candidate total, which sizes its candidate buffer). */
int fpp_query_device(const fpp_index* idx, const float* Q_dev, uint64_t nq, uint32_t k,
                     uint32_t qprobes, uint32_t* ids_dev, double* scores_dev,
                     fpp_query_stats* stats_dev, void* stream);

/* Multi-GPU query split.  Stage A alone: the
   probe sets of nq queries as global bucket ids t * num_buckets + b, probes_dev
   [nq][fpp_query_probes(qprobes)] u32 in probe order (the L true buckets first).
   They depend only on the queries and the hash functions (parameters + seed), so a
   rank computes them for its slice of a batch and every shard resolves them. */
int fpp_query_probe_sets_device(const fpp_index* idx, const float* Q_dev, uint64_t nq,
                                uint32_t qprobes, uint32_t* probes_dev, void* stream);
/* Stage B from such probe sets (computed by any index with the same parameters and
   seed), resolved in this index's tables: equals fpp_query_device on the same Q. */
int fpp_query_from_probe_sets_device(const fpp_index* idx, const float* Q_dev, uint64_t nq,
                                     const uint32_t* probes_dev, uint32_t k, uint32_t qprobes,
                                     uint32_t* ids_dev, double* scores_dev,
                                     fpp_query_stats* stats_dev, void* stream);

/* search with a SimHash rerank budget B (SPEC.md:311-314 QueryParams, :330-338
 * simhash_screen): the collected candidates are screened to the B with the most
 * agreeing signature bits (64-bit signatures from the (t=0, f=0) projection signs,
 * ties by lower id) before the exact top-k.  B = 0 is fpp_query; otherwise B >= k
 * (FPP_ERR_OUT_OF_RANGE).  stats.exact = min(B, U_q). */
int fpp_query_rerank(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t k,
                     uint32_t qprobes, uint32_t rerank, uint32_t* ids, double* scores,
                     fpp_query_stats* stats);
int fpp_query_rerank_device(const fpp_index* idx, const float* Q_dev, uint64_t nq, uint32_t k,
                            uint32_t qprobes, uint32_t rerank, uint32_t* ids_dev,
                            double* scores_dev, fpp_query_stats* stats_dev, void* stream);
/* the 64-bit SimHash signatures of rows X (host), as stored for the index's points */
int fpp_signatures(const fpp_index* idx, const float* X, uint64_t n, uint64_t* out);

/* ------------------------------------------------------ introspection / parity */
typedef struct fpp_index_info {
  uint64_t n;
  uint32_t d, d_pad, L, K, D, iprobes, kappa;
  float alpha;
  uint64_t seed;
  uint64_t num_buckets;   /* NB per table = (2D)^K */
  uint64_t kept_total;    /* entries kept over all tables */
  uint64_t prefilter_total; /* n*L*iprobes */
  uint64_t device_bytes;  /* resident index bytes */
  uint32_t max_bucket;    /* largest kept bucket */
  uint32_t id_offset;
  uint32_t centering;     /* indexed rows are centered (fpp_index_center) */
  uint32_t mode;          /* FPP_MODE_* */
  int32_t device;         /* CUDA device ordinal holding the index (ABI 4) */
} fpp_index_info;

int fpp_index_info_get(const fpp_index* idx, fpp_index_info* info);
uint64_t fpp_table_size(const fpp_index* idx, uint32_t t);
/* CSR of table t (SPEC.md:237-242 FalconnPPIndex): offsets [NB+1] (relative), ids, scores */
int fpp_table_csr(const fpp_index* idx, uint32_t t, uint32_t* offsets, uint32_t* ids,
                  float* scores);
/* GPU projections of host rows X[n][d] through stack (t,f): out [n][D] (rotation.cpp:70-100) */
int fpp_project(const fpp_index* idx, const float* X, uint64_t n, uint32_t t, uint32_t f,
                float* out);
/* GPU index probes (bucket, score) of host rows for table t: [n][iprobes] */
int fpp_index_probes(const fpp_index* idx, const float* X, uint64_t n, uint32_t t,
                     uint32_t* buckets, float* scores);
/* ranked per-function query lists [nq][L][K][s] (value, code), s = fpp_query_cap */
uint32_t fpp_query_cap(const fpp_index* idx, uint32_t qprobes);
uint64_t fpp_query_probes(const fpp_index* idx, uint32_t qprobes);
int fpp_query_lists(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t qprobes,
                    float* vals, uint32_t* codes);
/* one query's probe set (t*NB+bucket, ascending) and candidate set (local ids, ascending) */
int fpp_query_debug(const fpp_index* idx, const float* q, uint32_t qprobes, uint64_t* probes,
                    uint64_t* n_probes, uint32_t* cands, uint64_t* n_cands);

int fpp_timings_get(const fpp_index* idx, fpp_timings* t);
int fpp_timings_reset(const fpp_index* idx);

/* ------------------------------------- sharded build, global filter
 * Rank g of G builds ids [id_offset, id_offset + n) of the global dataset so that
 * the union of the G shard indexes equals the 1-GPU index exactly:
 *   fpp_shard_begin        hash every table, local per-(table,bucket) histogram
 *   fpp_shard_hist         copy it to a device buffer [L*NB] -> caller all-reduces (sum)
 *   fpp_shard_slots        number of exchange slots (sum over buckets of keep(B_global))
 *   fpp_shard_prefix       this rank's sorted bucket prefixes in those slots (~0 padded)
 *                          -> caller all-gathers [G][slots]
 *   fpp_shard_finish       per-bucket global cut, keep local entries <= cut -> queryable
 * Device pointers must live on the index's device. */
int fpp_shard_begin(const float* X, uint64_t n, uint32_t d, const fpp_params* p, fpp_index** out);
int fpp_shard_begin_device(const float* X_dev, uint64_t n, uint32_t d, const fpp_params* p,
                           fpp_index** out);
uint64_t fpp_shard_hist_len(const fpp_index* idx);
int fpp_shard_hist(const fpp_index* idx, uint32_t* hist_dev);
int fpp_shard_slots(fpp_index* idx, const uint32_t* global_hist_dev, uint64_t* slots);
int fpp_shard_prefix(fpp_index* idx, const uint32_t* global_hist_dev, uint64_t* prefix_dev);
int fpp_shard_finish(fpp_index* idx, const uint32_t* global_hist_dev,
                     const uint64_t* all_prefix_dev, uint32_t world);

/* ------------------------- multi-GPU index in one process (SURVEY 8(b) num_gpus, 8(e))
 * build(dataset, config) over num_gpus devices and search
 * over the sharded index.  Shard g holds the contiguous global ids
 * [g*n/G, (g+1)*n/G) on devices[g] (NULL = devices 0..num_gpus-1; an ordinal may
 * repeat, the shards then share that device) and is built by the global-filter
 * protocol above, so the union of the shards equals the 1-GPU index and every answer
 * (ids, scores, stats) is identical for every num_gpus.  A query batch
 * is sent to every device; hashing + probe selection are split across the shards and
 * the probe sets all-gathered; every shard scores its own candidates; shard g merges
 * the G top-k lists of its slice of the batch (score desc, id asc) and writes that
 * slice of ids/scores.  Exchanges are device-to-device copies (NVLink peer access is
 * enabled between the devices at build).  X, Q, ids, scores, stats are host buffers
 * as in fpp_build / fpp_query; p->device and p->id_offset are ignored / must be 0;
 * centering is FPP_ERR_UNSUPPORTED (center X first).  Calls on one fpp_multi
 * serialise. */
typedef struct fpp_multi fpp_multi;
int fpp_multi_build(const float* X, uint64_t n, uint32_t d, const fpp_params* p, uint32_t num_gpus,
                    const int32_t* devices, fpp_multi** out);
int fpp_multi_query(const fpp_multi* m, const float* Q, uint64_t nq, uint32_t k, uint32_t qprobes,
                    uint32_t* ids, double* scores, fpp_query_stats* stats);
uint32_t fpp_multi_shards(const fpp_multi* m);
/* shard g as a plain index (introspection: fpp_index_info_get, fpp_table_csr, ...);
   owned by the fpp_multi */
const fpp_index* fpp_multi_shard(const fpp_multi* m, uint32_t g);
void fpp_multi_free(fpp_multi* m);

/* -------------------------------------------------------------- host helpers */
/* ---- multi-GPU query merge: after an all-gather of the G shards'
 * per-query top-k lists, scores/ids [lists][nq][k] on `device` (each list sorted by
 * score desc, id asc; empty slots id 0xFFFFFFFF / -inf) are merged into
 * out [nq][k] by the same key order on the device (k-way merge kernel).  The shard
 * lists must hold disjoint (global) ids.  lists <= 32, any k >= 1.  Asynchronous on stream. */
int fpp_merge_topk(const double* scores_dev, const uint32_t* ids_dev, uint32_t lists, uint64_t nq,
                   uint32_t k, double* out_scores_dev, uint32_t* out_ids_dev, int device,
                   void* stream);

/* ---- exact brute force over the index's dataset: the recall ground truth
 * (SPEC.md:490-503 brute_force_topk).  Scores are inner_product (dataset.cpp:61-69)
 * bit for bit; top-k by (score desc, id asc), ids global (id_offset added).
 * Errors as fpp_query (k <= n, dimension, finite Q).  k > 32 takes one pass over X per
 * 32 ranks. */
int fpp_brute_force(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t k, uint32_t* ids,
                    double* scores);
int fpp_brute_force_device(const fpp_index* idx, const float* Q_dev, uint64_t nq, uint32_t k,
                           uint32_t* ids_dev, double* scores_dev, void* stream);

/* ---- index persistence: FLPP files (SPEC.md:270-278 save/load, 283-287 format).
 * Replaces save(index, path) / load(path).  The dataset is stored by reference
 * (fnv1a64 content hash of the n*d fp32 bytes, common.hpp:50-57): fpp_load takes
 * the same X again and fails with FPP_ERR_FORMAT if its hash differs.  A save of
 * the same (dataset, config) is byte-identical; load(save(ix)) answers every
 * query bit-identically.  Errors: FPP_ERR_IO (open/write), FPP_ERR_FORMAT (bad
 * magic, truncated file, checksum or dataset mismatch), FPP_ERR_UNSUPPORTED
 * (other FLPP version), FPP_ERR_DIMENSION (X shape differs from the index). */
#define FPP_FLPP_VERSION 1
int fpp_save(const fpp_index* idx, const char* path);
int fpp_load(const char* path, const float* X, uint64_t n, uint32_t d, int device,
             fpp_index** out);
int fpp_load_device(const char* path, const float* X_dev, uint64_t n, uint32_t d, int device,
                    fpp_index** out);
uint64_t fpp_content_hash(const float* X, uint64_t n, uint32_t d);

/* center(Dataset) in place (dataset.cpp:40-57): mean by a sequential double sum
 * over rows per coordinate, center = float(mean / n), rows -= center in fp32 (not
 * renormalized).  center_out (d floats) may be NULL. */
int fpp_center(float* X, uint64_t n, uint32_t d, float* center_out);
/* the index's center vector (d floats; all zero unless built with centering) */
int fpp_index_center(const fpp_index* idx, float* center_out);

/* normalize(Dataset) in place (dataset.cpp:24-38); FPP_ERR_ZERO_NORM names the row */
int fpp_normalize(float* X, uint64_t n, uint32_t d);
/* seeded synthetic data: clusters=0 -> i.i.d. N(0,1);
   else mixture of `clusters` isotropic Gaussians (centers N(0,I), std sigma).
   stream selects independent draws (0 = data, 1 = queries); rows NOT normalized. */
int fpp_synth(float* X, uint64_t n, uint32_t d, uint32_t clusters, float sigma, uint64_t seed,
              uint32_t stream, int threads);
/* rows [row0, row0 + n) of the same dataset (a shard's rows) */
int fpp_synth_rows(float* X, uint64_t row0, uint64_t n, uint32_t d, uint32_t clusters, float sigma,
                   uint64_t seed, uint32_t stream, int threads);

#ifdef __cplusplus
}
#endif
#endif
