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
/* ref: dataset.cpp:40-57 */
void orc_center(float* X, uint64_t n, uint32_t d, float* center_out) {
  double* mean = (double*)calloc(d, sizeof(double));
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < d; ++j) mean[j] += X[i * d + j];
  for (uint32_t j = 0; j < d; ++j) center_out[j] = (float)(mean[j] / (double)n);
  for (uint64_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < d; ++j) X[i * d + j] -= center_out[j];
  free(mean);
}

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
 * DESIGN.md section 3 pin): the D "natural" signed vectors sign(p_i) r_i
 * (closest / furthest) in (|p| desc, i asc) order, value
 * |p_i|, followed -- only when r > D -- by the opposite-signed vectors
 * -sign(p_i) r_i in the same order and with the same value |p_i|.  Entry 0 is
 * cross_polytope_hash.  Ranks D.. are the opposite part.
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
  if (r > D) {  /* opposite-signed vectors: same (|p| desc, i asc) order, flipped code */
    for (uint32_t k = 0; k < r - D; ++k) {
      const uint32_t i = tmp[k].i;
      vals[D + k] = tmp[k].a;
      codes[D + k] = p[i] >= 0.0f ? D + i : i;
    }
  }
  free(tmp);
}

typedef struct { float s; uint32_t r1, r2, t, g, a, b; } pairkey;

/* pair order within a class: score desc, r1 asc, r2 asc, t asc */
static int pair_better(const pairkey* a, const pairkey* b) {
  if (a->s != b->s) return a->s > b->s;
  if (a->r1 != b->r1) return a->r1 < b->r1;
  if (a->r2 != b->r2) return a->r2 < b->r2;
  return a->t < b->t;
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

static const float k_zero_val[1] = {0.0f};
static const uint32_t k_zero_code[1] = {0u};

typedef struct {
  const float* va; const float* vb;
  const uint32_t* ca; const uint32_t* cb;
  uint32_t na, nb, oa, ob, t;
  float ma, mb;  /* natural list maxima max|q.r| of the two functions (baseline gap) */
  int mode;
} grid;

/* pair score, larger first: falconnpp fl(v1+v2); falconn_baseline
   -(fl(m1-v1) + fl(m2-v2)), i.e. ascending gap score */
static float pscore(const grid* g, uint32_t a, uint32_t b) {
  if (g->mode == 1) return -((g->ma - g->va[a]) + (g->mb - g->vb[b]));
  return g->va[a] + g->vb[b];
}

/*
 * Class-ordered enumeration of (t, r1, r2) pairs of L tables' ranked lists
 * vals/codes [L][K][s]:
 *   class 0: natural x natural, class 1: exactly one opposite-signed entry,
 *   class 2: both opposite; inside a class (fl(v1+v2) desc, r1, r2, t).
 * Each (table, part-combination) is a grid sorted in both ranks, so a
 * best-first heap over the grids' frontiers yields the exact order.  Emits up
 * to `limit` pairs (bucket t*NB + b, score); skip_forced drops every table's
 * class-0 (0,0) (the true bucket, handled by the caller).
 */
static uint64_t enum_pairs(const float* vals, const uint32_t* codes, uint32_t L, uint32_t K,
                           uint32_t D, uint32_t s, uint64_t NB, uint64_t limit, int skip_forced,
                           uint64_t* out_b, float* out_s, int mode) {
  const uint32_t n = s < D ? s : D, o = s > D ? s - D : 0;
  grid* G = (grid*)malloc((size_t)L * 2 * sizeof(grid));
  pairkey* heap = (pairkey*)malloc((size_t)(2 * limit + 4 * L + 4) * sizeof(pairkey));
  uint64_t emitted = 0;
  const int ncls = K == 2 ? 3 : 2;
  for (int cls = 0; cls < ncls && emitted < limit; ++cls) {
    uint32_t ng = 0;
    for (uint32_t t = 0; t < L; ++t) {
      const float* v1 = vals + ((uint64_t)t * K) * s;
      const uint32_t* c1 = codes + ((uint64_t)t * K) * s;
      const float* v2 = K == 2 ? v1 + s : k_zero_val;
      const uint32_t* c2 = K == 2 ? c1 + s : k_zero_code;
      const uint32_t n2 = K == 2 ? n : 1, o2 = K == 2 ? o : 0;
      /* parts: (start, len, rank offset) natural = (0, n, 0), opposite = (D, o, D) */
      uint32_t pa[2][3] = {{0, n, 0}, {D, o, D}};
      uint32_t pb[2][3] = {{0, n2, 0}, {D, o2, D}};
      int combos[2][2];
      int nc = 0;
      if (cls == 0) { combos[nc][0] = 0; combos[nc][1] = 0; ++nc; }
      if (cls == 1) {
        combos[nc][0] = 0; combos[nc][1] = 1; ++nc;
        combos[nc][0] = 1; combos[nc][1] = 0; ++nc;
      }
      if (cls == 2) { combos[nc][0] = 1; combos[nc][1] = 1; ++nc; }
      for (int ci = 0; ci < nc; ++ci) {
        const int A = combos[ci][0], B = combos[ci][1];
        if (K == 1 && B == 1) continue;
        grid g;
        g.va = v1 + pa[A][0]; g.ca = c1 + pa[A][0]; g.na = pa[A][1]; g.oa = pa[A][2];
        g.vb = v2 + (K == 2 ? pb[B][0] : 0); g.cb = c2 + (K == 2 ? pb[B][0] : 0);
        g.nb = pb[B][1]; g.ob = K == 2 ? pb[B][2] : 0; g.t = t;
        g.ma = v1[0];
        g.mb = v2[0];
        g.mode = mode;
        if (g.na == 0 || g.nb == 0) continue;
        G[ng++] = g;
      }
    }
    uint64_t hn = 0;
    for (uint32_t gi = 0; gi < ng; ++gi) {
      const grid* g = &G[gi];
      if (cls == 0 && skip_forced) {
        if (g->nb > 1) {
          pairkey k = {pscore(g, 0, 1), g->oa, g->ob + 1, g->t, gi, 0, 1};
          heap_push(heap, &hn, k);
        }
        if (g->na > 1) {
          pairkey k = {pscore(g, 1, 0), g->oa + 1, g->ob, g->t, gi, 1, 0};
          heap_push(heap, &hn, k);
        }
      } else {
        pairkey k = {pscore(g, 0, 0), g->oa, g->ob, g->t, gi, 0, 0};
        heap_push(heap, &hn, k);
      }
    }
    while (emitted < limit && hn) {
      const pairkey k = heap_pop(heap, &hn);
      const grid* g = &G[k.g];
      const uint32_t b = K == 2 ? g->ca[k.a] * (2 * D) + g->cb[k.b] : g->ca[k.a];
      out_b[emitted] = (uint64_t)g->t * NB + b;
      if (out_s) out_s[emitted] = k.s;
      ++emitted;
      if (k.b + 1 < g->nb) {
        pairkey c = {pscore(g, k.a, k.b + 1), g->oa + k.a, g->ob + k.b + 1, g->t, k.g, k.a, k.b + 1};
        heap_push(heap, &hn, c);
      }
      if (k.b == 0 && k.a + 1 < g->na) {
        pairkey c = {pscore(g, k.a + 1, 0), g->oa + k.a + 1, g->ob, g->t, k.g, k.a + 1, 0};
        heap_push(heap, &hn, c);
      }
    }
  }
  free(G);
  free(heap);
  return emitted;
}

/*
 * SPEC.md:184-192 index_probe_sequence: the top-iProbes pairs of the point's
 * ranked lists in the class-ordered total order (the first is the true bucket).
 * Top pairs of a sorted grid lie within the first iProbes ranks, so lists of
 * r = min(iProbes, 2D) entries suffice.
 */
void orc_index_probes(const float* proj, uint32_t K, uint32_t D, uint32_t iprobes,
                      uint32_t* buckets, float* scores) {
  const uint32_t r = iprobes < 2 * D ? iprobes : 2 * D;
  float* V = (float*)malloc((size_t)K * r * sizeof(float));
  uint32_t* Cc = (uint32_t*)malloc((size_t)K * r * sizeof(uint32_t));
  uint64_t* ob = (uint64_t*)malloc((size_t)iprobes * sizeof(uint64_t));
  for (uint32_t f = 0; f < K; ++f) orc_rank(proj + (uint64_t)f * D, D, r, V + f * r, Cc + f * r);
  const uint64_t NB = K == 2 ? 4ull * D * D : 2ull * D;
  enum_pairs(V, Cc, 1, K, D, r, NB, iprobes, 0, ob, scores, 0);
  for (uint32_t k = 0; k < iprobes; ++k) buckets[k] = (uint32_t)ob[k];
  free(V);
  free(Cc);
  free(ob);
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
uint32_t orc_keep_count(uint32_t B, float alpha, uint32_t iprobes, uint32_t kappa);
static uint32_t keep_count(uint32_t B, float alpha, uint32_t iprobes, uint32_t kappa) {
  return orc_keep_count(B, alpha, iprobes, kappa);
}
uint32_t orc_keep_count(uint32_t B, float alpha, uint32_t iprobes, uint32_t kappa) {
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
  if (!(prm->alpha > 0.0f && prm->alpha <= 1.0f) || prm->iprobes == 0 || prm->mode > 1) return NULL;
  orc_index* idx = (orc_index*)calloc(1, sizeof(orc_index));
  idx->p = *prm;
  if (prm->mode == 1) {  /* SPEC.md:235 falconn_baseline forces alpha = 1, iProbes = 1 */
    idx->p.alpha = 1.0f;
    idx->p.iprobes = 1;
  }
  prm = &idx->p;
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
  for (uint32_t t = t_begin; t < t_end; ++t) {
    /* Alg. 1 lines 2-4: every point into its top-iProbes buckets */
    orc_index_probes_rows_mt(idx, X, n, t, eb, es, threads);
    uint32_t* off = (uint32_t*)malloc(((size_t)NB + 1) * sizeof(uint32_t));
    uint32_t* ids = (uint32_t*)malloc((ne + 1) * sizeof(uint32_t));
    float* sc = (float*)malloc((ne + 1) * sizeof(float));
    const uint64_t total = orc_csr_from_entries(eb, es, n, ip, NB, prm->alpha, prm->kappa, 0,
                                                threads, off, ids, sc);
    idx->offsets[t - t_begin] = off;
    idx->ids[t - t_begin] = (uint32_t*)realloc(ids, (total + 1) * sizeof(uint32_t));
    idx->scores[t - t_begin] = (float*)realloc(sc, (total + 1) * sizeof(float));
  }
  free(eb); free(es);
  (void)K; (void)D;
  return idx;
}

/* Alg. 1 lines 5-6 + limit scaling for ONE table, from its pre-filter entries:
   eb/es [n][ip] = (bucket, score) of point id0+i.  Entries are
   bucketed by a stable counting sort, each bucket sorted by (score desc, id asc),
   and keep_count(B) of its prefix kept.  offsets [NB+1]; ids/scores hold up to n*ip.
   Returns the kept total.  Used by orc_build and, streamed, by bench.py's C5 check. */
uint64_t orc_csr_from_entries(const uint32_t* eb, const float* es, uint64_t n, uint32_t ip,
                              uint32_t NB, float alpha, uint32_t kappa, uint32_t id0,
                              int threads, uint32_t* off, uint32_t* ids, float* sc) {
  if (threads <= 0) threads = 1;
  const uint64_t ne = n * ip;
  uint64_t* cnt = (uint64_t*)calloc((size_t)NB + 1, sizeof(uint64_t));
  entry* sorted = (entry*)malloc((ne + 1) * sizeof(entry));
  for (uint64_t e = 0; e < ne; ++e) cnt[eb[e] + 1]++;
  for (uint32_t b = 0; b < NB; ++b) cnt[b + 1] += cnt[b];
  uint64_t* cur = (uint64_t*)malloc((size_t)NB * sizeof(uint64_t));
  memcpy(cur, cnt, (size_t)NB * sizeof(uint64_t));
  for (uint64_t e = 0; e < ne; ++e) {
    entry en = {es[e], id0 + (uint32_t)(e / ip)};
    sorted[cur[eb[e]]++] = en;
  }
  free(cur);
  off[0] = 0;
  for (uint32_t b = 0; b < NB; ++b)
    off[b + 1] = off[b] + keep_count((uint32_t)(cnt[b + 1] - cnt[b]), alpha, ip, kappa);
#pragma omp parallel for schedule(dynamic, 1024) num_threads(threads)
  for (int64_t b = 0; b < (int64_t)NB; ++b) {
    const uint32_t B = (uint32_t)(cnt[b + 1] - cnt[b]);
    if (!B) continue;
    entry* seg = sorted + cnt[b];
    qsort(seg, B, sizeof(entry), cmp_entry);  /* (score desc, id asc) */
    const uint32_t kk = off[b + 1] - off[b];  /* Alg. 1 line 6 + heuristic (2) */
    for (uint32_t j = 0; j < kk; ++j) { ids[off[b] + j] = seg[j].id; sc[off[b] + j] = seg[j].s; }
  }
  const uint64_t total = off[NB];
  free(cnt); free(sorted);
  return total;
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

/* same, OpenMP over rows (orc_build's Alg. 1 lines 2-4; bench.py's streamed C5 check) */
void orc_index_probes_rows_mt(const orc_index* idx, const float* X, uint64_t n, uint32_t t,
                              uint32_t* buckets, float* scores, int threads) {
  const uint32_t K = idx->p.K, D = idx->p.D, ip = idx->p.iprobes;
  if (threads <= 0) threads = 1;
#pragma omp parallel num_threads(threads)
  {
    float* proj = (float*)malloc((size_t)K * D * sizeof(float));
    float* buf = (float*)malloc((size_t)idx->P * sizeof(float));
#pragma omp for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
      for (uint32_t f = 0; f < K; ++f)
        project_signs(stack_signs(idx, t, f), idx->d, idx->P, D, X + (uint64_t)i * idx->d,
                      proj + f * D, buf);
      orc_index_probes(proj, K, D, ip, buckets + (uint64_t)i * ip, scores + (uint64_t)i * ip);
    }
    free(proj);
    free(buf);
  }
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

/*
 * SPEC.md:193-201 query_probe_sequence (DESIGN.md section 3 pin): the L true
 * buckets, then the best P_eff - L remaining pairs in the class-ordered total
 * order.  Writes probes as t*NB+bucket (unsorted), returns the count.
 */
static uint64_t probe_set(const orc_index* idx, const float* vals, const uint32_t* codes,
                          uint32_t s, uint64_t peff, uint64_t* probes, pairkey* heap_unused) {
  (void)heap_unused;
  const uint32_t L = idx->p.L, K = idx->p.K, D = idx->p.D;
  const uint64_t NB = idx->NB;
  for (uint32_t t = 0; t < L; ++t) {
    const uint32_t* c1 = codes + ((uint64_t)t * K) * s;
    probes[t] = t * NB + (K == 2 ? (uint64_t)c1[0] * 2 * D + c1[s] : c1[0]);
  }
  return L + enum_pairs(vals, codes, L, K, D, s, NB, peff - L, 1, probes + L, NULL,
                        (int)idx->p.mode);
}

uint64_t orc_probe_set_lists(const float* vals, const uint32_t* codes, uint32_t L, uint32_t K,
                             uint32_t D, uint32_t s, uint64_t peff, uint64_t* probes) {
  orc_index tmp;
  memset(&tmp, 0, sizeof(tmp));
  tmp.p.L = L;
  tmp.p.K = K;
  tmp.p.D = D;
  tmp.NB = K == 2 ? 4u * D * D : 2u * D;
  return probe_set(&tmp, vals, codes, s, peff, probes, NULL);
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

/* SPEC.md "SimHash signatures": signs of the first 64 coordinates of the first
   table's first-function projection */
static uint64_t simhash_one(const orc_index* idx, const float* x, float* out, float* buf) {
  project_signs(stack_signs(idx, 0, 0), idx->d, idx->P, idx->p.D, x, out, buf);
  const uint32_t m = idx->p.D < 64 ? idx->p.D : 64;
  uint64_t s = 0;
  for (uint32_t j = 0; j < m; ++j)
    if (out[j] >= 0.0f) s |= 1ull << j;
  return s;
}

void orc_simhash_rows(const orc_index* idx, const float* X, uint64_t n, uint64_t* out, int threads) {
  if (threads <= 0) threads = 1;
  const uint32_t Dw = blocks_of(idx->P, idx->p.D) * idx->P;
#pragma omp parallel num_threads(threads)
  {
    float* o = (float*)malloc((size_t)Dw * sizeof(float));
    float* buf = (float*)malloc((size_t)idx->P * sizeof(float));
#pragma omp for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) out[i] = simhash_one(idx, X + (uint64_t)i * idx->d, o, buf);
    free(o);
    free(buf);
  }
}

typedef struct { uint32_t dis; uint32_t id; } screened;  /* dis = 64 - agreement */
static int cmp_screened(const void* x, const void* y) {    /* agreement desc, id asc */
  const screened* u = (const screened*)x; const screened* v = (const screened*)y;
  if (u->dis != v->dis) return (u->dis > v->dis) - (u->dis < v->dis);
  return (u->id > v->id) - (u->id < v->id);
}

/* SPEC.md:339-347 top_k_exact over the unique candidates */
int orc_query(const orc_index* idx, const float* Q, uint64_t nq, uint32_t k,
              uint32_t qprobes, uint32_t* ids, double* scores, orc_stats* stats,
              int threads) {
  return orc_query_rerank(idx, Q, nq, k, qprobes, 0, ids, scores, stats, threads);
}

/* search, with simhash_screen when B > 0 */
int orc_query_rerank(const orc_index* idx, const float* Q, uint64_t nq, uint32_t k,
                     uint32_t qprobes, uint32_t B, uint32_t* ids, double* scores,
                     orc_stats* stats, int threads) {
  if (idx->t_begin != 0 || idx->t_end != idx->p.L) return -1;
  if (k == 0 || qprobes < idx->p.L) return -1;
  if (B != 0 && B < k) return -1;  /* QueryParams: B = 0 or B >= k */
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
  uint64_t* sigs = NULL;
  if (B) {
    sigs = (uint64_t*)malloc((size_t)idx->n * sizeof(uint64_t));
    orc_simhash_rows(idx, idx->X, idx->n, sigs, threads);
  }
#pragma omp parallel num_threads(threads)
  {
    qscratch w;
    qscratch_init(&w, idx, s, peff, k);
    screened* scr = B ? (screened*)malloc((size_t)idx->n * sizeof(screened)) : NULL;
    float* po = B ? (float*)malloc((size_t)blocks_of(idx->P, idx->p.D) * idx->P * sizeof(float)) : NULL;
    float* pbuf = B ? (float*)malloc((size_t)idx->P * sizeof(float)) : NULL;
#pragma omp for schedule(dynamic, 1)
    for (int64_t qi = 0; qi < (int64_t)nq; ++qi) {
      const float* q = Q + (uint64_t)qi * d;
      uint64_t np, ne;
      const uint64_t nc = collect(idx, q, qprobes, &w, &np, &ne);
      uint64_t nx = nc;  /* exact inner products */
      if (B && nc > B) {  /* simhash_screen: top B by bit agreement, ties by lower id */
        const uint64_t sq = simhash_one(idx, q, po, pbuf);
        for (uint64_t c = 0; c < nc; ++c) {
          scr[c].dis = (uint32_t)__builtin_popcountll(sigs[w.cands[c]] ^ sq);
          scr[c].id = w.cands[c];
        }
        qsort(scr, nc, sizeof(screened), cmp_screened);
        nx = B;
      }
      uint32_t cnt = 0;
      for (uint64_t c = 0; c < nx; ++c) {
        const uint32_t cid = nx < nc ? scr[c].id : w.cands[c];
        scored x = {orc_inner_product(idx->X + (uint64_t)cid * d, q, d), cid};
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
        stats[qi].exact = nx;
      }
      clear_visited(&w, nc);
    }
    qscratch_free(&w);
    free(scr);
    free(po);
    free(pbuf);
  }
  free(sigs);
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
  orc_synth_rows(X, 0, n, d, clusters, sigma, seed, stream, threads);
}
/* rows [row0, row0 + n) of the same dataset (a shard) */
void orc_synth_rows(float* X, uint64_t row0, uint64_t n, uint32_t d, uint32_t clusters,
                    float sigma, uint64_t seed, uint32_t stream, int threads) {
  const uint64_t s_noise = 3 + 100ull * stream, s_assign = 2 + 100ull * stream;
  if (threads <= 0) threads = 1;
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t r = 0; r < (int64_t)n; ++r) {
    const uint64_t i = row0 + (uint64_t)r;
    float* row = X + (uint64_t)r * d;
    if (clusters == 0) {
      for (uint32_t j = 0; j < d; ++j) row[j] = (float)synth_normal(seed, s_noise, i * d + j);
    } else {
      const uint64_t c = orc_mix64(orc_derive_seed(seed, s_assign, i, 0)) % clusters;
      for (uint32_t j = 0; j < d; ++j) {
        const double ctr = synth_normal(seed, 1, c * d + j);
        const double z = synth_normal(seed, s_noise, i * d + j);
        row[j] = (float)(ctr + (double)sigma * z);
      }
    }
  }
}
