/*
 * fpp_oracle.c -- CPU restatement of the Falconn++ hot path (see fpp_oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY: the parity checker and the CPU baseline.  The
 * product path (paper_2206_01382_b200/) never calls into this file.
 *
 * Every function cites the reference text it restates.  "ref:" citations are
 * relative to /root/reference/.  Pinned choices that the reference leaves open
 * are the ones of SURVEY.md section 8(c), restated in DESIGN.md section 3.
 */
#include "fpp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- common */

/* ref: proj/include/lsfann/common.hpp:18-23 (splitmix64 finalizer) */
uint64_t orc_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* ref: common.hpp:27-34 */
uint64_t orc_derive_seed(uint64_t master, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t h = orc_mix64(master);
  h = orc_mix64(h ^ (a * 0xff51afd7ed558ccdULL));
  h = orc_mix64(h ^ (b * 0xc4ceb9fe1a85ec53ULL));
  h = orc_mix64(h ^ (c * 0xd6e8feb86659fd93ULL));
  return h;
}

/* ref: common.hpp:50-58 */
uint64_t orc_fnv1a64(const void* data, size_t len, uint64_t h) {
  const unsigned char* p = (const unsigned char*)data;
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* -------------------------------------------------------------- rotation */

/* ref: proj/src/rotation.cpp:34-38 */
uint32_t orc_pad_dimension(uint32_t d) {
  uint32_t p = 1;
  while (p < d) p <<= 1;
  return p;
}

/* ref: rotation.cpp:16-32 -- radix-2, len ascending, a[j]=x+y, a[j+len]=x-y */
void orc_fht(float* a, uint32_t n) {
  for (uint32_t len = 1; len < n; len <<= 1)
    for (uint32_t i = 0; i < n; i += len << 1)
      for (uint32_t j = i; j < i + len; ++j) {
        const float x = a[j], y = a[j + len];
        a[j] = x + y;
        a[j + len] = x - y;
      }
}

/* ref: rotation.cpp:55-67 -- bit b of mix64(seed + w) is sign 64w+b, 1 -> +1 */
void orc_signs(uint64_t seed, uint32_t P, uint32_t blocks, float* out) {
  uint64_t state = seed, word = 0;
  int bits_left = 0;
  const uint64_t total = (uint64_t)blocks * 3u * P;
  for (uint64_t i = 0; i < total; ++i) {
    if (bits_left == 0) {
      word = orc_mix64(state++);
      bits_left = 64;
    }
    out[i] = (word & 1u) ? 1.0f : -1.0f;
    word >>= 1;
    --bits_left;
  }
}

static uint32_t blocks_of(uint32_t P, uint32_t D) { return D >= P ? D / P : 1u; }

/* ref: rotation.cpp:70-100 (with precomputed signs) */
static void project_signs(const float* signs, uint32_t d, uint32_t P, uint32_t D,
                          const float* x, float* out, float* buf) {
  const uint32_t blocks = blocks_of(P, D);
  const float scale = 1.0f / (float)P;
  for (uint32_t b = 0; b < blocks; ++b) {
    memcpy(buf, x, d * sizeof(float));
    memset(buf + d, 0, (P - d) * sizeof(float));
    const float* bs = signs + (uint64_t)b * 3u * P;
    for (int stage = 0; stage < 3; ++stage) {
      const float* s = bs + (uint64_t)stage * P;
      for (uint32_t j = 0; j < P; ++j) buf[j] *= s[j];
      orc_fht(buf, P);
    }
    const uint32_t take = P < D ? P : D;
    float* dst = out + (uint64_t)b * P;
    for (uint32_t j = 0; j < take; ++j) dst[j] = buf[j] * scale;
  }
}

void orc_project(uint32_t d, uint32_t D, uint64_t seed, const float* x, float* out) {
  const uint32_t P = orc_pad_dimension(d);
  const uint32_t blocks = blocks_of(P, D);
  float* signs = (float*)malloc((size_t)blocks * 3u * P * sizeof(float));
  float* buf = (float*)malloc((size_t)P * sizeof(float));
  orc_signs(seed, P, blocks, signs);
  project_signs(signs, d, P, D, x, out, buf);
  free(signs);
  free(buf);
}

void orc_project_rows(uint32_t d, uint32_t D, uint64_t seed, const float* X, uint64_t n,
                      float* out, int threads) {
  const uint32_t P = orc_pad_dimension(d);
  const uint32_t blocks = blocks_of(P, D);
  float* signs = (float*)malloc((size_t)blocks * 3u * P * sizeof(float));
  orc_signs(seed, P, blocks, signs);
  if (threads <= 0) threads = 1;
#pragma omp parallel num_threads(threads)
  {
    float* buf = (float*)malloc((size_t)P * sizeof(float));
#pragma omp for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i)
      project_signs(signs, d, P, D, X + (uint64_t)i * d, out + (uint64_t)i * D, buf);
    free(buf);
  }
  free(signs);
}

/* --------------------------------------------------------------- dataset */

/* ref: proj/src/dataset.cpp:24-38 */
int64_t orc_normalize(float* X, uint64_t n, uint32_t d) {
  for (uint64_t i = 0; i < n; ++i) {
    float* row = X + i * d;
    double sq = 0.0;
    for (uint32_t j = 0; j < d; ++j) sq += (double)row[j] * (double)row[j];
    if (sq == 0.0) return (int64_t)i;
    const float inv = (float)(1.0 / sqrt(sq));
    for (uint32_t j = 0; j < d; ++j) row[j] *= inv;
  }
  return -1;
}

/* ref: dataset.cpp:61-69 -- sequential fp64 accumulation of exact products */
double orc_inner_product(const float* a, const float* b, uint32_t d) {
  double acc = 0.0;
  for (uint32_t i = 0; i < d; ++i) acc += (double)a[i] * (double)b[i];
  return acc;
}

/* --------------------------------------------------------------- hashing */

/* argmax |p|, lowest index on ties; i if p>=0 else D+i */
uint32_t orc_cp_hash(const float* p, uint32_t D) {
  uint32_t best = 0;
  float bv = fabsf(p[0]);
  for (uint32_t i = 1; i < D; ++i) {
    const float a = fabsf(p[i]);
    if (a > bv) { bv = a; best = i; }
  }
  return p[best] >= 0.0f ? best : D + best;
}

typedef struct { float a; uint32_t i; } absidx;

static int cmp_nat(const void* x, const void* y) {  /* |p| desc, i asc */
  const absidx* u = (const absidx*)x; const absidx* v = (const absidx*)y;
  if (u->a > v->a) return -1;
  if (u->a < v->a) return 1;
  return (u->i > v->i) - (u->i < v->i);
}
static int cmp_opp(const void* x, const void* y) {  /* |p| asc, i asc */
  const absidx* u = (const absidx*)x; const absidx* v = (const absidx*)y;
  if (u->a < v->a) return -1;
  if (u->a > v->a) return 1;
  return (u->i > v->i) - (u->i < v->i);
}

/*
 * Ranked signed list of one cross-polytope function (SPEC.md:184-201 with the
 * DESIGN.md section 3 pin): the D "natural" signed vectors sign(p_i) r_i in
 * (|p| desc, i asc) order with value +|p_i|, followed by the D opposite
 * vectors -sign(p_i) r_i in (|p| asc, i asc) order with value -|p_i|.  The
 * list is non-increasing in value; entry 0 is cross_polytope_hash.  Only the
 * first r <= 2D entries are produced.
 */
void orc_rank(const float* p, uint32_t D, uint32_t r, float* vals, uint32_t* codes) {
  const uint32_t rn = r < D ? r : D;
  if (rn <= 8 && r <= D) {  /* small-r fast path: insertion top-r */
    absidx top[8];
    uint32_t cnt = 0;
    for (uint32_t i = 0; i < D; ++i) {
      const float a = fabsf(p[i]);
      if (cnt == rn && !(a > top[rn - 1].a)) continue;  /* ties keep lower i */
      uint32_t pos = cnt < rn ? cnt++ : rn - 1;
      while (pos > 0 && a > top[pos - 1].a) { top[pos] = top[pos - 1]; --pos; }
      top[pos].a = a; top[pos].i = i;
    }
    for (uint32_t k = 0; k < rn; ++k) {
      const uint32_t i = top[k].i;
      vals[k] = top[k].a;
      codes[k] = p[i] >= 0.0f ? i : D + i;
    }
    return;
  }
  absidx* tmp = (absidx*)malloc((size_t)D * sizeof(absidx));
  for (uint32_t i = 0; i < D; ++i) { tmp[i].a = fabsf(p[i]); tmp[i].i = i; }
  qsort(tmp, D, sizeof(absidx), cmp_nat);
  for (uint32_t k = 0; k < rn; ++k) {
    const uint32_t i = tmp[k].i;
    vals[k] = tmp[k].a;
    codes[k] = p[i] >= 0.0f ? i : D + i;
  }
  if (r > D) {
    qsort(tmp, D, sizeof(absidx), cmp_opp);
    for (uint32_t k = 0; k < r - D; ++k) {
      const uint32_t i = tmp[k].i;
      vals[D + k] = -fabsf(p[i]);
      codes[D + k] = p[i] >= 0.0f ? D + i : i;
    }
  }
  free(tmp);
}

typedef struct { float s; uint32_t r1, r2, t; } pairkey;

/* pair total order: score desc, r1 asc, r2 asc, t asc */
static int pair_better(const pairkey* a, const pairkey* b) {
  if (a->s != b->s) return a->s > b->s;
  if (a->r1 != b->r1) return a->r1 < b->r1;
  if (a->r2 != b->r2) return a->r2 < b->r2;
  return a->t < b->t;
}

/*
 * SPEC.md:184-192 index_probe_sequence: top-iProbes pairs of the two ranked
 * lists by fl(v1+v2).  Pairs beyond rank iProbes in either list can never
 * enter the top iProbes (the key is monotone in both ranks), so r=min(ip,2D).
 */
void orc_index_probes(const float* proj, uint32_t K, uint32_t D, uint32_t iprobes,
                      uint32_t* buckets, float* scores) {
  const uint32_t r = iprobes < 2 * D ? iprobes : 2 * D;
  float v1[64], v2[64];
  uint32_t c1[64], c2[64];
  float* V1 = r <= 64 ? v1 : (float*)malloc(r * sizeof(float));
  uint32_t* C1 = r <= 64 ? c1 : (uint32_t*)malloc(r * sizeof(uint32_t));
  orc_rank(proj, D, r, V1, C1);
  if (K == 1) {
    for (uint32_t k = 0; k < iprobes; ++k) { buckets[k] = C1[k]; scores[k] = V1[k]; }
  } else {
    float* V2 = r <= 64 ? v2 : (float*)malloc(r * sizeof(float));
    uint32_t* C2 = r <= 64 ? c2 : (uint32_t*)malloc(r * sizeof(uint32_t));
    orc_rank(proj + D, D, r, V2, C2);
    /* selection of the top iprobes of r*r pairs */
    pairkey* best = (pairkey*)malloc((size_t)iprobes * sizeof(pairkey));
    uint32_t cnt = 0;
    for (uint32_t a = 0; a < r; ++a)
      for (uint32_t b = 0; b < r; ++b) {
        pairkey k = {V1[a] + V2[b], a, b, 0};
        if (cnt == iprobes && !pair_better(&k, &best[iprobes - 1])) continue;
        uint32_t pos = cnt < iprobes ? cnt++ : iprobes - 1;
        while (pos > 0 && pair_better(&k, &best[pos - 1])) { best[pos] = best[pos - 1]; --pos; }
        best[pos] = k;
      }
    for (uint32_t k = 0; k < iprobes; ++k) {
      buckets[k] = C1[best[k].r1] * (2 * D) + C2[best[k].r2];
      scores[k] = best[k].s;
    }
    free(best);
    if (V2 != v2) { free(V2); free(C2); }
  }
  if (V1 != v1) { free(V1); free(C1); }
}

void orc_cp_hash_rows(const float* proj, uint64_t n, uint32_t D, uint32_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = orc_cp_hash(proj + i * D, D);
}

/* ----------------------------------------------------------------- index */

struct orc_index {
  orc_params p;
  uint64_t n;
  uint32_t d, P, NB;
  const float* X; /* borrowed */
  uint32_t t_begin, t_end;
  float* signs; /* [L][K][blocks*3*P] */
  uint32_t** offsets;
  uint32_t** ids;
  float** scores;
};

static const float* stack_signs(const orc_index* idx, uint32_t t, uint32_t f) {
  const uint64_t per = (uint64_t)blocks_of(idx->P, idx->p.D) * 3u * idx->P;
  return idx->signs + ((uint64_t)t * idx->p.K + f) * per;
}

typedef struct { float s; uint32_t id; } entry;

static int cmp_entry(const void* x, const void* y) {  /* score desc, id asc */
  const entry* u = (const entry*)x; const entry* v = (const entry*)y;
  if (u->s > v->s) return -1;
  if (u->s < v->s) return 1;
  return (u->id > v->id) - (u->id < v->id);
}

/* SPEC.md:257 + SURVEY 8(c): min(B, max(kappa, floor(double(alpha)*B/iProbes))) */
static uint32_t keep_count(uint32_t B, float alpha, uint32_t iprobes, uint32_t kappa) {
  double f = floor((double)alpha * (double)B / (double)iprobes);
  uint64_t k = (uint64_t)f;
  if (k < kappa) k = kappa;
  if (k > B) k = B;
  return (uint32_t)k;
}

/* SPEC.md:245-262 + PAPER.md:303-317,336-339 (Algorithm 1 + limit scaling) */
orc_index* orc_build(const float* X, uint64_t n, uint32_t d, const orc_params* prm,
                     int threads, uint32_t t_begin, uint32_t t_end) {
  if (!X || n == 0 || d == 0 || !prm) return NULL;
  if (prm->K < 1 || prm->K > 2 || prm->L == 0 || prm->D == 0 || (prm->D & (prm->D - 1)))
    return NULL;
  if (!(prm->alpha > 0.0f && prm->alpha <= 1.0f) || prm->iprobes == 0) return NULL;
  orc_index* idx = (orc_index*)calloc(1, sizeof(orc_index));
  idx->p = *prm;
  idx->n = n;
  idx->d = d;
  idx->P = orc_pad_dimension(d);
  if (prm->D >= idx->P && prm->D % idx->P) { free(idx); return NULL; }
  idx->NB = prm->K == 2 ? 4u * prm->D * prm->D : 2u * prm->D;
  if (prm->iprobes > idx->NB) { free(idx); return NULL; }
  idx->X = X;
  if (t_end > prm->L || t_end == 0) t_end = prm->L;
  idx->t_begin = t_begin;
  idx->t_end = t_end;
  const uint32_t K = prm->K, D = prm->D, P = idx->P, ip = prm->iprobes, NB = idx->NB;
  const uint64_t per = (uint64_t)blocks_of(P, D) * 3u * P;
  idx->signs = (float*)malloc((size_t)prm->L * K * per * sizeof(float));
  for (uint32_t t = 0; t < prm->L; ++t)
    for (uint32_t f = 0; f < K; ++f)  /* derive_seed(seed,t,f,0) */
      orc_signs(orc_derive_seed(prm->seed, t, f, 0), P, blocks_of(P, D),
                idx->signs + ((uint64_t)t * K + f) * per);
  const uint32_t nt = t_end - t_begin;
  idx->offsets = (uint32_t**)calloc(nt, sizeof(void*));
  idx->ids = (uint32_t**)calloc(nt, sizeof(void*));
  idx->scores = (float**)calloc(nt, sizeof(void*));
  if (threads <= 0) {
#ifdef _OPENMP
    threads = omp_get_max_threads();
#else
    threads = 1;
#endif
  }
  const uint64_t ne = n * ip;
  uint32_t* eb = (uint32_t*)malloc(ne * sizeof(uint32_t));
  float* es = (float*)malloc(ne * sizeof(float));
  uint32_t* cnt = (uint32_t*)malloc(((size_t)NB + 1) * sizeof(uint32_t));
  entry* sorted = (entry*)malloc(ne * sizeof(entry));
  for (uint32_t t = t_begin; t < t_end; ++t) {
    /* Alg. 1 lines 2-4: every point into its top-iProbes buckets */
#pragma omp parallel num_threads(threads)
    {
      float* proj = (float*)malloc((size_t)K * D * sizeof(float));
      float* buf = (float*)malloc((size_t)P * sizeof(float));
#pragma omp for schedule(static)
      for (int64_t i = 0; i < (int64_t)n; ++i) {
        for (uint32_t f = 0; f < K; ++f)
          project_signs(stack_signs(idx, t, f), d, P, D, X + (uint64_t)i * d, proj + f * D, buf);
        orc_index_probes(proj, K, D, ip, eb + (uint64_t)i * ip, es + (uint64_t)i * ip);
      }
      free(proj);
      free(buf);
    }
    /* bucket the entries (stable counting sort), then sort each bucket */
    memset(cnt, 0, ((size_t)NB + 1) * sizeof(uint32_t));
    for (uint64_t e = 0; e < ne; ++e) cnt[eb[e] + 1]++;
    for (uint32_t b = 0; b < NB; ++b) cnt[b + 1] += cnt[b];
    uint32_t* cur = (uint32_t*)malloc((size_t)NB * sizeof(uint32_t));
    memcpy(cur, cnt, (size_t)NB * sizeof(uint32_t));
    for (uint64_t e = 0; e < ne; ++e) {
      entry en = {es[e], (uint32_t)(e / ip)};
      sorted[cur[eb[e]]++] = en;
    }
    free(cur);
    uint32_t* off = (uint32_t*)malloc(((size_t)NB + 1) * sizeof(uint32_t));
    off[0] = 0;
    for (uint32_t b = 0; b < NB; ++b)
      off[b + 1] = off[b] + keep_count(cnt[b + 1] - cnt[b], prm->alpha, ip, prm->kappa);
    const uint32_t total = off[NB];
    uint32_t* ids = (uint32_t*)malloc(((size_t)total + 1) * sizeof(uint32_t));
    float* sc = (float*)malloc(((size_t)total + 1) * sizeof(float));
#pragma omp parallel for schedule(dynamic, 1024) num_threads(threads)
    for (int64_t b = 0; b < (int64_t)NB; ++b) {
      const uint32_t B = cnt[b + 1] - cnt[b];
      if (!B) continue;
      entry* seg = sorted + cnt[b];
      qsort(seg, B, sizeof(entry), cmp_entry);  /* (score desc, id asc) */
      const uint32_t kk = off[b + 1] - off[b];  /* Alg. 1 line 6 + heuristic (2) */
      for (uint32_t j = 0; j < kk; ++j) { ids[off[b] + j] = seg[j].id; sc[off[b] + j] = seg[j].s; }
    }
    idx->offsets[t - t_begin] = off;
    idx->ids[t - t_begin] = ids;
    idx->scores[t - t_begin] = sc;
  }
  free(eb); free(es); free(cnt); free(sorted);
  return idx;
}

void orc_index_probes_rows(const orc_index* idx, const float* X, uint64_t n, uint32_t t,
                           uint32_t* buckets, float* scores) {
  const uint32_t K = idx->p.K, D = idx->p.D, ip = idx->p.iprobes;
  float* proj = (float*)malloc((size_t)K * D * sizeof(float));
  float* buf = (float*)malloc((size_t)idx->P * sizeof(float));
  for (uint64_t i = 0; i < n; ++i) {
    for (uint32_t f = 0; f < K; ++f)
      project_signs(stack_signs(idx, t, f), idx->d, idx->P, D, X + i * idx->d, proj + f * D, buf);
    orc_index_probes(proj, K, D, ip, buckets + i * ip, scores + i * ip);
  }
  free(proj);
  free(buf);
}

orc_index* orc_index_from_csr(const float* X, uint64_t n, uint32_t d, const orc_params* prm,
                              const uint32_t* offsets, const uint32_t* ids, const float* scores,
                              const uint64_t* table_base) {
  orc_index* idx = (orc_index*)calloc(1, sizeof(orc_index));
  idx->p = *prm;
  idx->n = n;
  idx->d = d;
  idx->P = orc_pad_dimension(d);
  idx->NB = prm->K == 2 ? 4u * prm->D * prm->D : 2u * prm->D;
  idx->X = X;
  idx->t_begin = 0;
  idx->t_end = prm->L;
  const uint32_t K = prm->K, D = prm->D, P = idx->P, NB = idx->NB;
  const uint64_t per = (uint64_t)blocks_of(P, D) * 3u * P;
  idx->signs = (float*)malloc((size_t)prm->L * K * per * sizeof(float));
  for (uint32_t t = 0; t < prm->L; ++t)
    for (uint32_t f = 0; f < K; ++f)
      orc_signs(orc_derive_seed(prm->seed, t, f, 0), P, blocks_of(P, D),
                idx->signs + ((uint64_t)t * K + f) * per);
  idx->offsets = (uint32_t**)calloc(prm->L, sizeof(void*));
  idx->ids = (uint32_t**)calloc(prm->L, sizeof(void*));
  idx->scores = (float**)calloc(prm->L, sizeof(void*));
  for (uint32_t t = 0; t < prm->L; ++t) {
    const uint64_t cnt = table_base[t + 1] - table_base[t];
    idx->offsets[t] = (uint32_t*)malloc(((size_t)NB + 1) * sizeof(uint32_t));
    memcpy(idx->offsets[t], offsets + (uint64_t)t * (NB + 1), ((size_t)NB + 1) * sizeof(uint32_t));
    idx->ids[t] = (uint32_t*)malloc((cnt + 1) * sizeof(uint32_t));
    idx->scores[t] = (float*)malloc((cnt + 1) * sizeof(float));
    memcpy(idx->ids[t], ids + table_base[t], cnt * sizeof(uint32_t));
    memcpy(idx->scores[t], scores + table_base[t], cnt * sizeof(float));
  }
  return idx;
}

void orc_free(orc_index* idx) {
  if (!idx) return;
  for (uint32_t t = 0; t < idx->t_end - idx->t_begin; ++t) {
    free(idx->offsets[t]); free(idx->ids[t]); free(idx->scores[t]);
  }
  free(idx->offsets); free(idx->ids); free(idx->scores); free(idx->signs); free(idx);
}

uint64_t orc_num_buckets(const orc_index* idx) { return idx->NB; }

uint64_t orc_table_size(const orc_index* idx, uint32_t t) {
  return idx->offsets[t - idx->t_begin][idx->NB];
}

void orc_table(const orc_index* idx, uint32_t t, uint32_t* offsets, uint32_t* ids,
               float* scores) {
  const uint32_t tt = t - idx->t_begin;
  const uint32_t total = idx->offsets[tt][idx->NB];
  if (offsets) memcpy(offsets, idx->offsets[tt], ((size_t)idx->NB + 1) * sizeof(uint32_t));
  if (ids) memcpy(ids, idx->ids[tt], (size_t)total * sizeof(uint32_t));
  if (scores) memcpy(scores, idx->scores[tt], (size_t)total * sizeof(float));
}

/* ----------------------------------------------------------------- query */

static uint32_t isqrt_ceil(uint64_t q) {
  uint64_t r = (uint64_t)sqrt((double)q);
  while (r * r > q) --r;
  while (r * r < q) ++r;
  return (uint32_t)r;
}

/* SPEC.md:211 per-function cap s = min(2D, 2*ceil(sqrt(qProbes))); K=1: min(2D, qProbes) */
uint32_t orc_query_cap(const orc_index* idx, uint32_t qprobes) {
  const uint32_t D2 = 2 * idx->p.D;
  uint64_t s = idx->p.K == 2 ? 2ull * isqrt_ceil(qprobes) : qprobes;
  return (uint32_t)(s < D2 ? s : D2);
}

uint64_t orc_query_probes(const orc_index* idx, uint32_t qprobes) {
  const uint64_t s = orc_query_cap(idx, qprobes);
  const uint64_t avail = (uint64_t)idx->p.L * (idx->p.K == 2 ? s * s : s);
  return qprobes < avail ? qprobes : avail;
}

void orc_query_lists(const orc_index* idx, const float* q, uint32_t s, float* vals,
                     uint32_t* codes) {
  const uint32_t K = idx->p.K, D = idx->p.D;
  float* proj = (float*)malloc((size_t)D * sizeof(float));
  float* buf = (float*)malloc((size_t)idx->P * sizeof(float));
  for (uint32_t t = 0; t < idx->p.L; ++t)
    for (uint32_t f = 0; f < K; ++f) {
      project_signs(stack_signs(idx, t, f), idx->d, idx->P, D, q, proj, buf);
      orc_rank(proj, D, s, vals + ((uint64_t)t * K + f) * s, codes + ((uint64_t)t * K + f) * s);
    }
  free(proj);
  free(buf);
}

/* binary max-heap on pair_better */
static void heap_push(pairkey* h, uint64_t* n, pairkey k) {
  uint64_t i = (*n)++;
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (!pair_better(&k, &h[p])) break;
    h[i] = h[p];
    i = p;
  }
  h[i] = k;
}
static pairkey heap_pop(pairkey* h, uint64_t* n) {
  pairkey top = h[0], last = h[--(*n)];
  uint64_t i = 0;
  for (;;) {
    uint64_t c = 2 * i + 1;
    if (c >= *n) break;
    if (c + 1 < *n && pair_better(&h[c + 1], &h[c])) ++c;
    if (!pair_better(&h[c], &last)) break;
    h[i] = h[c];
    i = c;
  }
  if (*n) h[i] = last;
  return top;
}

/*
 * SPEC.md:193-201 query_probe_sequence (DESIGN.md section 3 pin): the L true
 * buckets, then the best P_eff-L remaining (t,r1,r2) by (fl(v1+v2) desc, r1,
 * r2, t), enumerated best-first over the per-table sorted grids.
 * Writes probes as t*NB+bucket (unsorted), returns count.
 */
static uint64_t probe_set(const orc_index* idx, const float* vals, const uint32_t* codes,
                          uint32_t s, uint64_t peff, uint64_t* probes, pairkey* heap) {
  const uint32_t L = idx->p.L, K = idx->p.K, D = idx->p.D;
  const uint64_t NB = idx->NB;
  uint64_t np = 0, hn = 0;
#define V(t, f, r) vals[((uint64_t)(t) * K + (f)) * s + (r)]
#define C(t, f, r) codes[((uint64_t)(t) * K + (f)) * s + (r)]
  for (uint32_t t = 0; t < L; ++t) {
    probes[np++] = t * NB + (K == 2 ? (uint64_t)C(t, 0, 0) * 2 * D + C(t, 1, 0) : C(t, 0, 0));
    if (K == 2) {
      if (s > 1) {
        pairkey a = {V(t, 0, 0) + V(t, 1, 1), 0, 1, t};
        pairkey b = {V(t, 0, 1) + V(t, 1, 0), 1, 0, t};
        heap_push(heap, &hn, a);
        heap_push(heap, &hn, b);
      }
    } else if (s > 1) {
      pairkey a = {V(t, 0, 1), 1, 0, t};
      heap_push(heap, &hn, a);
    }
  }
  while (np < peff && hn) {
    pairkey k = heap_pop(heap, &hn);
    const uint32_t t = k.t;
    if (K == 2) {
      probes[np++] = t * NB + (uint64_t)C(t, 0, k.r1) * 2 * D + C(t, 1, k.r2);
      if (k.r2 + 1 < s) {
        pairkey c = {V(t, 0, k.r1) + V(t, 1, k.r2 + 1), k.r1, k.r2 + 1, t};
        heap_push(heap, &hn, c);
      }
      if (k.r2 == 0 && k.r1 + 1 < s) {
        pairkey c = {V(t, 0, k.r1 + 1) + V(t, 1, 0), k.r1 + 1, 0, t};
        heap_push(heap, &hn, c);
      }
    } else {
      probes[np++] = t * NB + C(t, 0, k.r1);
      if (k.r1 + 1 < s) {
        pairkey c = {V(t, 0, k.r1 + 1), k.r1 + 1, 0, t};
        heap_push(heap, &hn, c);
      }
    }
  }
#undef V
#undef C
  return np;
}

typedef struct { double s; uint32_t id; } scored;

static int better_scored(const scored* a, const scored* b) {  /* score desc, id asc */
  if (a->s != b->s) return a->s > b->s;
  return a->id < b->id;
}

typedef struct {
  float* vals; uint32_t* codes; uint64_t* probes; pairkey* heap;
  uint64_t* visited; uint32_t* cands; scored* top;
} qscratch;

static void qscratch_init(qscratch* w, const orc_index* idx, uint32_t s, uint64_t peff,
                          uint32_t k) {
  const uint64_t LK = (uint64_t)idx->p.L * idx->p.K;
  w->vals = (float*)malloc(LK * s * sizeof(float));
  w->codes = (uint32_t*)malloc(LK * s * sizeof(uint32_t));
  w->probes = (uint64_t*)malloc((peff + idx->p.L) * sizeof(uint64_t));
  w->heap = (pairkey*)malloc((2 * peff + 2 * idx->p.L + 4) * sizeof(pairkey));
  w->visited = (uint64_t*)calloc((idx->n + 63) / 64, sizeof(uint64_t));
  w->cands = (uint32_t*)malloc(idx->n * sizeof(uint32_t));
  w->top = (scored*)malloc((k + 1) * sizeof(scored));
}
static void qscratch_free(qscratch* w) {
  free(w->vals); free(w->codes); free(w->probes); free(w->heap);
  free(w->visited); free(w->cands); free(w->top);
}

/* collect unique candidates of one query */
static uint64_t collect(const orc_index* idx, const float* q, uint32_t qprobes, qscratch* w,
                        uint64_t* np_out, uint64_t* ne_out) {
  const uint32_t s = orc_query_cap(idx, qprobes);
  const uint64_t peff = orc_query_probes(idx, qprobes);
  orc_query_lists(idx, q, s, w->vals, w->codes);
  const uint64_t np = probe_set(idx, w->vals, w->codes, s, peff, w->probes, w->heap);
  uint64_t nc = 0, ne = 0;
  for (uint64_t p = 0; p < np; ++p) {
    const uint32_t t = (uint32_t)(w->probes[p] / idx->NB);
    const uint32_t b = (uint32_t)(w->probes[p] % idx->NB);
    const uint32_t* off = idx->offsets[t - idx->t_begin];
    const uint32_t* ids = idx->ids[t - idx->t_begin];
    for (uint32_t e = off[b]; e < off[b + 1]; ++e) {
      const uint32_t id = ids[e];
      ++ne;
      uint64_t m = 1ull << (id & 63);
      if (w->visited[id >> 6] & m) continue;
      w->visited[id >> 6] |= m;
      w->cands[nc++] = id;
    }
  }
  *np_out = np;
  *ne_out = ne;
  return nc;
}

static void clear_visited(qscratch* w, uint64_t nc) {
  for (uint64_t c = 0; c < nc; ++c) w->visited[w->cands[c] >> 6] = 0;
}

/* SPEC.md:339-347 top_k_exact over the unique candidates */
int orc_query(const orc_index* idx, const float* Q, uint64_t nq, uint32_t k,
              uint32_t qprobes, uint32_t* ids, double* scores, orc_stats* stats,
              int threads) {
  if (idx->t_begin != 0 || idx->t_end != idx->p.L) return -1;
  if (k == 0 || qprobes < idx->p.L) return -1;
  if (threads <= 0) {
#ifdef _OPENMP
    threads = omp_get_max_threads();
#else
    threads = 1;
#endif
  }
  const uint32_t s = orc_query_cap(idx, qprobes);
  const uint64_t peff = orc_query_probes(idx, qprobes);
  const uint32_t d = idx->d;
#pragma omp parallel num_threads(threads)
  {
    qscratch w;
    qscratch_init(&w, idx, s, peff, k);
#pragma omp for schedule(dynamic, 1)
    for (int64_t qi = 0; qi < (int64_t)nq; ++qi) {
      const float* q = Q + (uint64_t)qi * d;
      uint64_t np, ne;
      const uint64_t nc = collect(idx, q, qprobes, &w, &np, &ne);
      uint32_t cnt = 0;
      for (uint64_t c = 0; c < nc; ++c) {
        scored x = {orc_inner_product(idx->X + (uint64_t)w.cands[c] * d, q, d), w.cands[c]};
        if (cnt == k && !better_scored(&x, &w.top[k - 1])) continue;
        uint32_t pos = cnt < k ? cnt++ : k - 1;
        while (pos > 0 && better_scored(&x, &w.top[pos - 1])) { w.top[pos] = w.top[pos - 1]; --pos; }
        w.top[pos] = x;
      }
      for (uint32_t j = 0; j < k; ++j) {
        ids[(uint64_t)qi * k + j] = j < cnt ? w.top[j].id : 0xFFFFFFFFu;
        scores[(uint64_t)qi * k + j] = j < cnt ? w.top[j].s : -INFINITY;
      }
      if (stats) {
        stats[qi].probes = np;
        stats[qi].entries = ne;
        stats[qi].candidates = nc;
      }
      clear_visited(&w, nc);
    }
    qscratch_free(&w);
  }
  return 0;
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}
static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

int orc_query_debug(const orc_index* idx, const float* q, uint32_t qprobes,
                    uint64_t* probes, uint64_t* np, uint32_t* cands, uint64_t* nc) {
  const uint32_t s = orc_query_cap(idx, qprobes);
  const uint64_t peff = orc_query_probes(idx, qprobes);
  qscratch w;
  qscratch_init(&w, idx, s, peff, 1);
  uint64_t ne;
  *nc = collect(idx, q, qprobes, &w, np, &ne);
  memcpy(probes, w.probes, *np * sizeof(uint64_t));
  memcpy(cands, w.cands, *nc * sizeof(uint32_t));
  qsort(probes, *np, sizeof(uint64_t), cmp_u64);
  qsort(cands, *nc, sizeof(uint32_t), cmp_u32);
  qscratch_free(&w);
  return 0;
}

/* SPEC.md:490-498 brute_force_topk, ties by lower id */
void orc_brute_force(const float* X, uint64_t n, uint32_t d, const float* Q, uint64_t nq,
                     uint32_t k, uint32_t* ids, double* scores, int threads) {
  if (threads <= 0) threads = 1;
#pragma omp parallel num_threads(threads)
  {
    scored* top = (scored*)malloc((k + 1) * sizeof(scored));
#pragma omp for schedule(dynamic, 1)
    for (int64_t qi = 0; qi < (int64_t)nq; ++qi) {
      uint32_t cnt = 0;
      for (uint64_t i = 0; i < n; ++i) {
        scored x = {orc_inner_product(X + i * d, Q + (uint64_t)qi * d, d), (uint32_t)i};
        if (cnt == k && !better_scored(&x, &top[k - 1])) continue;
        uint32_t pos = cnt < k ? cnt++ : k - 1;
        while (pos > 0 && better_scored(&x, &top[pos - 1])) { top[pos] = top[pos - 1]; --pos; }
        top[pos] = x;
      }
      for (uint32_t j = 0; j < k; ++j) {
        ids[(uint64_t)qi * k + j] = j < cnt ? top[j].id : 0xFFFFFFFFu;
        scores[(uint64_t)qi * k + j] = j < cnt ? top[j].s : -INFINITY;
      }
    }
    free(top);
  }
}

/* ------------------------------------------------------------- synthetic */
/* u(s,k) = ((mix64(derive_seed(seed,s,k,0))>>11)+0.5)*2^-53,
   N(0,1) by Box-Muller in double; centers stream 1, assignment stream 2+100*stream,
   noise stream 3+100*stream. */
static double synth_u(uint64_t seed, uint64_t stream, uint64_t k) {
  return ((double)(orc_mix64(orc_derive_seed(seed, stream, k, 0)) >> 11) + 0.5) * 0x1.0p-53;
}
static double synth_normal(uint64_t seed, uint64_t stream, uint64_t k) {
  const double u1 = synth_u(seed, stream, 2 * k), u2 = synth_u(seed, stream, 2 * k + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
void orc_synth(float* X, uint64_t n, uint32_t d, uint32_t clusters, float sigma, uint64_t seed,
               uint32_t stream, int threads) {
  const uint64_t s_noise = 3 + 100ull * stream, s_assign = 2 + 100ull * stream;
  if (threads <= 0) threads = 1;
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t i = 0; i < (int64_t)n; ++i) {
    float* row = X + (uint64_t)i * d;
    if (clusters == 0) {
      for (uint32_t j = 0; j < d; ++j) row[j] = (float)synth_normal(seed, s_noise, (uint64_t)i * d + j);
    } else {
      const uint64_t c = orc_mix64(orc_derive_seed(seed, s_assign, (uint64_t)i, 0)) % clusters;
      for (uint32_t j = 0; j < d; ++j) {
        const double ctr = synth_normal(seed, 1, c * d + j);
        const double z = synth_normal(seed, s_noise, (uint64_t)i * d + j);
        row[j] = (float)(ctr + (double)sigma * z);
      }
    }
  }
}
