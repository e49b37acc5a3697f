/*
 * fpp_oracle.h -- CPU restatement of the Falconn++ hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path in
 * paper_2206_01382_b200/ and the CPU-baseline arm of bench.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
 * load it.  The product library never links or calls anything in oracle/.
 *
 * Parity pinning: the rotation + dataset parts restate
 * /root/reference/proj/src/rotation.cpp and dataset.cpp and are pinned against
 * (a) the unmodified reference compiled into oracle/_ref/ (oracle/Makefile) and
 * (b) the fingerprints of SURVEY.md section 8(c) (tests/golden/).  The hashing,
 * index and query parts have NO reference code; they
 * restate SPEC.md with the pinned choices of SURVEY.md section 8(c) and
 * DESIGN.md section 3.  Those parts are pinned by the SPEC worked examples and
 * the SPEC acceptance criterion #4 (exhaustive probing == brute force).
 */
#ifndef FPP_ORACLE_H
#define FPP_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t L;        /* tables */
  uint32_t K;        /* concatenated hashes per table, 1 or 2 (SPEC l) */
  uint32_t D;        /* projections per function (power of two) */
  uint32_t iprobes;  /* indexing probes */
  uint32_t kappa;    /* limit-scaling floor (default 20) */
  float alpha;       /* scaling factor (0,1] */
  uint64_t seed;     /* master seed */
  uint32_t mode;     /* 0 falconnpp, 1 falconn_baseline (alpha = 1,
                        iProbes = 1 forced; probes by ascending gap score) */
} orc_params;

typedef struct {
  uint64_t probes;      /* P_q: probes visited */
  uint64_t entries;     /* E_q: kept bucket entries walked */
  uint64_t candidates;  /* U_q: unique ids collected */
  uint64_t exact;       /* exact inner products computed (U_q, or min(B, U_q) with rerank) */
} orc_stats;

typedef struct orc_index orc_index;

/* common.hpp:18-58 */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_derive_seed(uint64_t master, uint64_t a, uint64_t b, uint64_t c);
uint64_t orc_fnv1a64(const void* data, size_t len, uint64_t h);

/* rotation.cpp */
uint32_t orc_pad_dimension(uint32_t d);
void orc_fht(float* v, uint32_t n);
/* signs for one SpinnerStack: blocks*3*P floats (+1/-1), rotation.hpp:56 */
void orc_signs(uint64_t seed, uint32_t P, uint32_t blocks, float* out);
/* project one row x[d] with stack (d, D, seed): out[D] */
void orc_project(uint32_t d, uint32_t D, uint64_t seed, const float* x, float* out);

/* batch forms (OpenMP over rows) */
void orc_project_rows(uint32_t d, uint32_t D, uint64_t seed, const float* X, uint64_t n,
                      float* out, int threads);
void orc_cp_hash_rows(const float* proj, uint64_t n, uint32_t D, uint32_t* out);
/* index probes of rows X for table t of an index */
void orc_index_probes_rows(const orc_index* idx, const float* X, uint64_t n, uint32_t t,
                           uint32_t* buckets, float* scores);

/* dataset.cpp */
int64_t orc_normalize(float* X, uint64_t n, uint32_t d);   /* -1 ok, else zero row idx */
/* dataset.cpp:40-57 center(): double mean per coordinate (rows in order), float center,
   rows -= center in fp32 */
void orc_center(float* X, uint64_t n, uint32_t d, float* center_out);
double orc_inner_product(const float* a, const float* b, uint32_t d);

/* hashing */
uint32_t orc_cp_hash(const float* p, uint32_t D);
/* ranked signed list of one function: r entries (value, code) */
void orc_rank(const float* p, uint32_t D, uint32_t r, float* vals, uint32_t* codes);
/* index probes of one point in one table, given its K projections [K][D] */
void orc_index_probes(const float* proj, uint32_t K, uint32_t D, uint32_t iprobes,
                      uint32_t* buckets, float* scores);

/* SPEC.md:257 keep count of a bucket of pre-filter size B */
uint32_t orc_keep_count(uint32_t B, float alpha, uint32_t iprobes, uint32_t kappa);
/* probe set (t*NB + bucket, unsorted) from explicit ranked lists [L][K][s] */
uint64_t orc_probe_set_lists(const float* vals, const uint32_t* codes, uint32_t L, uint32_t K,
                             uint32_t D, uint32_t s, uint64_t peff, uint64_t* probes);

/* same, OpenMP over rows */
void orc_index_probes_rows_mt(const orc_index* idx, const float* X, uint64_t n, uint32_t t,
                              uint32_t* buckets, float* scores, int threads);
/* Alg. 1 lines 5-6 for one table from its pre-filter entries eb/es [n][ip] (point ids
   id0 + i): offsets [NB+1], ids/scores (capacity n*ip); returns the kept total */
uint64_t orc_csr_from_entries(const uint32_t* eb, const float* es, uint64_t n, uint32_t ip,
                              uint32_t NB, float alpha, uint32_t kappa, uint32_t id0,
                              int threads, uint32_t* offsets, uint32_t* ids, float* scores);

/* index build */
orc_index* orc_build(const float* X, uint64_t n, uint32_t d, const orc_params* prm,
                     int threads, uint32_t t_begin, uint32_t t_end);
void orc_free(orc_index* idx);
/* wrap an already-built CSR (e.g. the GPU's, verified bit-exact) for CPU query timing:
   offsets [L][NB+1], ids/scores [table_base[L]], table_base [L+1] */
orc_index* orc_index_from_csr(const float* X, uint64_t n, uint32_t d, const orc_params* prm,
                              const uint32_t* offsets, const uint32_t* ids, const float* scores,
                              const uint64_t* table_base);
uint64_t orc_num_buckets(const orc_index* idx);
/* CSR of one table (tables [t_begin,t_end) only) */
uint64_t orc_table_size(const orc_index* idx, uint32_t t);
void orc_table(const orc_index* idx, uint32_t t, uint32_t* offsets /*NB+1*/,
               uint32_t* ids, float* scores);

/* query */
uint32_t orc_query_cap(const orc_index* idx, uint32_t qprobes);     /* s */
uint64_t orc_query_probes(const orc_index* idx, uint32_t qprobes);  /* P_eff */
int orc_query(const orc_index* idx, const float* Q, uint64_t nq, uint32_t k,
              uint32_t qprobes, uint32_t* ids, double* scores, orc_stats* stats,
              int threads);
/* per-query intermediates; probes as t*NB+bucket, sorted asc; cands sorted asc.
   returns 0; sizes written to *np / *nc (buffers must hold P_eff / n). */
/* search with SimHash rerank budget B (0 = off): candidates are
   screened to the top B by signature bit agreement (ties by lower id) before the
   exact top-k.  orc_query == orc_query_rerank(..., B = 0, ...). */
int orc_query_rerank(const orc_index* idx, const float* Q, uint64_t nq, uint32_t k,
                     uint32_t qprobes, uint32_t B, uint32_t* ids, double* scores,
                     orc_stats* stats, int threads);
/* 64-bit SimHash signature (SPEC.md "SimHash signatures"): bit j < min(64, D) is
   1 iff p[j] >= 0 for the (t=0, f=0) projection (-0.0 counts as >= 0) */
void orc_simhash_rows(const orc_index* idx, const float* X, uint64_t n, uint64_t* out, int threads);
int orc_query_debug(const orc_index* idx, const float* q, uint32_t qprobes,
                    uint64_t* probes, uint64_t* np, uint32_t* cands, uint64_t* nc);
/* query projections ranked lists [L][K][s] */
void orc_query_lists(const orc_index* idx, const float* q, uint32_t s, float* vals,
                     uint32_t* codes);

/* the pinned synthetic generator, restated for the CPU arm */
void orc_synth(float* X, uint64_t n, uint32_t d, uint32_t clusters, float sigma, uint64_t seed,
               uint32_t stream, int threads);
/* rows [row0, row0 + n) of the same dataset (one shard) */
void orc_synth_rows(float* X, uint64_t row0, uint64_t n, uint32_t d, uint32_t clusters,
                    float sigma, uint64_t seed, uint32_t stream, int threads);

/* brute force top-k */
void orc_brute_force(const float* X, uint64_t n, uint32_t d, const float* Q, uint64_t nq,
                     uint32_t k, uint32_t* ids, double* scores, int threads);

#ifdef __cplusplus
}
#endif
#endif
