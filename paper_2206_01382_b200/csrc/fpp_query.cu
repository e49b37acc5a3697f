// fpp_query.cu -- batched multi-probe query: K1 (query hashing + ranked lists),
// probe selection, K3 (bucket walk + dedup), K3/K4 (row gather, exact fp64
// inner products, per-query top-k).
//
// Reference semantics: SPEC.md:193-201 query_probe_sequence
// search, :339-347 top_k_exact, :350-361 (dedup, probe accounting);
// dataset.cpp:61-69 inner_product; PAPER.md:318-321 (rank by |q.r|).
// Pinned choices: DESIGN.md section 3.  Oracle: oracle/fpp_oracle.c orc_query().
//
// Per chunk of queries:
//   k_query_lists   CTA per (query, table): spinner projections, bitonic rank,
//                   top-s signed lists (value, code)
//   k_probe_select  CTA per query: exact top-(P-L) pair selection by a
//                   threshold search on the fp32 pair score (two-sided prefix
//                   counts over the sorted lists), tie resolution in
//                   (r1, r2, t) order, then directory reads -> (pos, len)
//   k_collect       CTA per query: walk kept entries, test-and-set a visited
//                   bitmap (shared memory, or global for large shards),
//                   compact unique ids
//   k_score         CTA per query: 32-row batches per warp, cp.async column
//                   slices into shared memory (multi-stage ring), each lane
//                   accumulates its row's exact products in fp64 in the
//                   reference's sequential order (bit-identical scores), warp
//                   register top-k, CTA merge
#include <algorithm>
#include <cstdio>

#include "fpp_device.cuh"
#include "fpp_internal.h"

namespace fpp {

// ---------------------------------------------------------------- K1 query
template <int P>
__global__ void __launch_bounds__(256)
k_query_lists(const float* __restrict__ Q, uint32_t d, uint32_t D, uint32_t K,
              const uint32_t* __restrict__ signs, uint32_t L, uint32_t s,
              float* __restrict__ vals, uint32_t* __restrict__ codes) {
  using S = FhtShape<P>;
  __shared__ float pv[2][P];
  __shared__ uint64_t keys[P];
  const uint32_t q = blockIdx.x, t = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = threadIdx.x / S::G;
  const int g = lane % S::G;
  if (warp * S::GPW < (int)K) {  // warps that host a function's FHT group
    const int f = grp < (int)K ? grp : (int)K - 1;
    float v[S::EPT];
    load_row<P>(Q + (uint64_t)q * d, d, g, v);
    spinner_project<P>(v, signs + ((uint64_t)t * K + f) * 3 * S::W, g);
    if (grp < (int)K) {
#pragma unroll
      for (int e = 0; e < S::EPT; ++e) pv[f][g * S::EPT + e] = v[e];
    }
  }
  __syncthreads();
  const uint32_t nat = s < D ? s : D;
  for (uint32_t f = 0; f < K; ++f) {
    const uint64_t ob = (((uint64_t)q * L + t) * K + f) * s;
    for (uint32_t j = threadIdx.x; j < P; j += blockDim.x)
      keys[j] = j < D ? rank_key(pv[f][j], j) : ~0ull;
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1)
      for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
        for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
          const uint32_t ixj = i ^ jj;
          if (ixj > i) {
            const uint64_t a = keys[i], b = keys[ixj];
            if ((a > b) == ((i & k) == 0)) { keys[i] = b; keys[ixj] = a; }
          }
        }
        __syncthreads();
      }
    for (uint32_t r = threadIdx.x; r < nat; r += blockDim.x) {
      vals[ob + r] = rank_val(keys[r]);
      codes[ob + r] = rank_code(keys[r], D);
    }
    __syncthreads();
    if (s > D) {  // opposite signed vectors: (|p| asc, j asc), value -|p|
      for (uint32_t j = threadIdx.x; j < P; j += blockDim.x) {
        if (j < D) {
          const float p = pv[f][j];
          keys[j] = ((uint64_t)ord_key(fabsf(p)) << 32) | ((uint64_t)j << 1) | (p < 0.0f ? 1u : 0u);
        } else {
          keys[j] = ~0ull;
        }
      }
      __syncthreads();
      for (uint32_t k = 2; k <= P; k <<= 1)
        for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
          for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
            const uint32_t ixj = i ^ jj;
            if (ixj > i) {
              const uint64_t a = keys[i], b = keys[ixj];
              if ((a > b) == ((i & k) == 0)) { keys[i] = b; keys[ixj] = a; }
            }
          }
          __syncthreads();
        }
      for (uint32_t r = threadIdx.x; r < s - D; r += blockDim.x) {
        const uint64_t kk = keys[r];
        const uint32_t j = (uint32_t)(kk & 0xffffffffu) >> 1;
        vals[ob + D + r] = -ord_inv((uint32_t)(kk >> 32));
        codes[ob + D + r] = (kk & 1u) ? j : D + j;
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------ probe select
constexpr int PS_THREADS = 512;

struct ProbeArgs {
  const float* vals;      // [nq][L][K][s]
  const uint32_t* codes;  // [nq][L][K][s]
  uint32_t L, K, s, D;
  uint64_t NB;
  uint64_t peff;          // probes per query (incl. the L forced)
  const uint32_t* offs;   // [L][NB+1]
  const uint64_t* tbase;  // [L+1]
  uint64_t* ppos;         // [nq][peff]
  uint32_t* plen;         // [nq][peff]
  uint32_t* eq;           // [nq]
  uint64_t* dbg;          // optional [nq][peff] t*NB+b
  int use_smem;
};

__device__ __forceinline__ uint32_t prefix_ge(float v1, const float* __restrict__ v2, uint32_t n2,
                                              uint32_t T) {
  uint32_t lo = 0, hi = n2;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (ord_key(v1 + v2[mid]) >= T) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v, uint64_t* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  uint64_t t = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(PS_THREADS) k_probe_select(ProbeArgs a) {
  extern __shared__ float sv[];  // [L][K][s] values when they fit
  __shared__ uint64_t red[32];
  __shared__ uint64_t scan_sh[32];
  __shared__ float zero_row[1];
  const uint32_t q = blockIdx.x;
  const uint32_t L = a.L, K = a.K, s = a.s;
  const uint32_t S2 = K == 2 ? s : 1;
  const uint64_t LKs = (uint64_t)L * K * s;
  const float* V = a.vals + (uint64_t)q * LKs;
  const uint32_t* C = a.codes + (uint64_t)q * LKs;
  if (a.use_smem) {
    for (uint64_t i = threadIdx.x; i < LKs; i += blockDim.x) sv[i] = V[i];
    V = sv;
  }
  if (threadIdx.x == 0) zero_row[0] = 0.0f;
  __syncthreads();
  const uint64_t M = a.peff - L;  // non-forced probes
  const uint32_t items = L * s;   // item = (t, r1), t-major
  // contiguous item range per thread (for the emission scan)
  const uint32_t per = (items + blockDim.x - 1) / blockDim.x;
  const uint32_t it0 = min(items, threadIdx.x * per), it1 = min(items, it0 + per);
#define V1(t, r) V[((uint64_t)(t) * K) * s + (r)]
#define V2ROW(t) (K == 2 ? V + ((uint64_t)(t) * K + 1) * s : zero_row)
  // raw prefix count for item, excluding the forced (0,0)
  auto cnt_item = [&](uint32_t it, uint32_t T) -> uint32_t {
    const uint32_t t = it / s, r1 = it - t * s;
    uint32_t c = prefix_ge(V1(t, r1), V2ROW(t), S2, T);
    if (r1 == 0 && c > 0) c -= 1;
    return c;
  };
  uint32_t Tstar = 0;
  uint64_t cgt = 0;
  if (M > 0) {
    // largest key T with c_ge(T) >= M  (M-th best non-forced pair score)
    for (int bit = 31; bit >= 0; --bit) {
      const uint32_t cand = Tstar | (1u << bit);
      uint64_t c = 0;
      for (uint32_t it = it0; it < it1; ++it) c += cnt_item(it, cand);
      c = block_sum_u64(c, red);
      if (c >= M) Tstar = cand;
    }
    if (Tstar != 0xffffffffu) {
      uint64_t c = 0;
      for (uint32_t it = it0; it < it1; ++it) c += cnt_item(it, Tstar + 1);
      cgt = block_sum_u64(c, red);
    }
  }
  // ranges: gt = [st, ga), ties = [ga, gb) in r2, st = (r1==0)
  auto ranges = [&](uint32_t it, uint32_t& st, uint32_t& ga, uint32_t& gb) {
    const uint32_t t = it / s, r1 = it - t * s;
    st = r1 == 0 ? 1 : 0;
    const float v1 = V1(t, r1);
    const float* v2 = V2ROW(t);
    const uint32_t pa = (M == 0 || Tstar == 0xffffffffu) ? 0 : prefix_ge(v1, v2, S2, Tstar + 1);
    const uint32_t pb = M == 0 ? 0 : prefix_ge(v1, v2, S2, Tstar);
    ga = max(st, pa);
    gb = max(st, pb);
  };
  const uint64_t m = M - cgt;  // ties to take at T*
  uint64_t ties_total = 0;
  if (M > 0) {
    uint64_t c = 0;
    for (uint32_t it = it0; it < it1; ++it) {
      uint32_t st, ga, gb;
      ranges(it, st, ga, gb);
      c += gb - ga;
    }
    ties_total = block_sum_u64(c, red);
  }
  // partial ties: smallest composite key Kc with count_lt(Kc) >= m,
  // composite = (r1*S2 + r2)*L + t  -> order (r1, r2, t)
  uint64_t Kstar = ~0ull;
  if (M > 0 && ties_total > m) {
    auto count_lt = [&](uint64_t Kc) -> uint64_t {
      const uint64_t kr1 = Kc / ((uint64_t)S2 * L);
      const uint64_t rem = Kc - kr1 * S2 * L;
      const uint64_t kr2 = rem / L, kt = rem - kr2 * L;
      uint64_t c = 0;
      for (uint32_t it = it0; it < it1; ++it) {
        const uint32_t t = it / s, r1 = it - t * s;
        if (r1 > kr1) continue;
        uint32_t st, ga, gb;
        ranges(it, st, ga, gb);
        if (ga == gb) continue;
        if (r1 < kr1) { c += gb - ga; continue; }
        if (kr2 > ga) c += (kr2 < gb ? kr2 : (uint64_t)gb) - ga;
        if (kr2 >= ga && kr2 < gb && t < kt) c += 1;
      }
      return block_sum_u64(c, red);
    };
    uint64_t lo = 0, hi = (uint64_t)s * S2 * L;  // count_lt(hi) = ties_total >= m
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (count_lt(mid) >= m) hi = mid;
      else lo = mid + 1;
    }
    Kstar = lo;
  }
  auto take_tie = [&](uint32_t t, uint32_t r1, uint32_t r2) -> bool {
    if (Kstar == ~0ull) return true;
    return (((uint64_t)r1 * S2 + r2) * L + t) < Kstar;
  };
  // emission counts per thread
  uint64_t mine = 0;
  for (uint32_t it = it0; it < it1; ++it) {
    if (M == 0) break;
    uint32_t st, ga, gb;
    ranges(it, st, ga, gb);
    const uint32_t t = it / s, r1 = it - t * s;
    mine += ga - st;
    if (Kstar == ~0ull) mine += gb - ga;
    else
      for (uint32_t r2 = ga; r2 < gb; ++r2) mine += take_tie(t, r1, r2);
  }
  // exclusive block scan of `mine`
  uint64_t x = mine;
  {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) scan_sh[w] = x;
    __syncthreads();
    uint64_t wb = 0;
    for (int i = 0; i < w; ++i) wb += scan_sh[i];
    x = wb + x - mine;
    __syncthreads();
  }
  uint64_t* ppos = a.ppos + (uint64_t)q * a.peff;
  uint32_t* plen = a.plen + (uint64_t)q * a.peff;
  uint64_t* dbg = a.dbg ? a.dbg + (uint64_t)q * a.peff : nullptr;
  const uint32_t twoD = 2 * a.D;
  uint64_t esum = 0;
  auto emit = [&](uint64_t slot, uint32_t t, uint32_t b) {
    const uint32_t* of = a.offs + (uint64_t)t * (a.NB + 1);
    const uint32_t o0 = of[b], o1 = of[b + 1];
    ppos[slot] = a.tbase[t] + o0;
    plen[slot] = o1 - o0;
    esum += o1 - o0;
    if (dbg) dbg[slot] = (uint64_t)t * a.NB + b;
  };
  const uint32_t* Cq = C;
  auto bucket_of = [&](uint32_t t, uint32_t r1, uint32_t r2) -> uint32_t {
    const uint32_t c1 = Cq[((uint64_t)t * K) * s + r1];
    return K == 2 ? c1 * twoD + Cq[((uint64_t)t * K + 1) * s + r2] : c1;
  };
  for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) emit(t, t, bucket_of(t, 0, 0));
  uint64_t slot = L + x;
  for (uint32_t it = it0; it < it1; ++it) {
    if (M == 0) break;
    uint32_t st, ga, gb;
    ranges(it, st, ga, gb);
    const uint32_t t = it / s, r1 = it - t * s;
    for (uint32_t r2 = st; r2 < ga; ++r2) emit(slot++, t, bucket_of(t, r1, r2));
    for (uint32_t r2 = ga; r2 < gb; ++r2)
      if (take_tie(t, r1, r2)) emit(slot++, t, bucket_of(t, r1, r2));
  }
  esum = block_sum_u64(esum, red);
  if (threadIdx.x == 0) a.eq[q] = (uint32_t)esum;
#undef V1
#undef V2ROW
}

// exclusive scan of eq[nq] -> coff[nq+1] (single CTA)
__global__ void __launch_bounds__(1024) k_scan_eq(const uint32_t* __restrict__ eq, uint32_t nq,
                                                  uint64_t* __restrict__ coff) {
  __shared__ uint64_t sh[32];
  uint64_t carry = 0;
  for (uint32_t b = 0; b < nq; b += blockDim.x) {
    const uint32_t i = b + threadIdx.x;
    const uint64_t v = i < nq ? eq[i] : 0;
    uint64_t x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    uint64_t wb = 0, tot = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      if (k < w) wb += sh[k];
      tot += sh[k];
    }
    if (i < nq) coff[i] = carry + wb + x - v;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) coff[nq] = carry;
}

// ----------------------------------------------------------------- collect
constexpr int CO_THREADS = 512;
constexpr int CO_TILE = 1024;

struct CollectArgs {
  const uint64_t* ppos;
  const uint32_t* plen;
  uint64_t peff;
  const uint32_t* ids;
  const uint64_t* coff;
  uint32_t* cands;
  uint32_t* uq;
  uint32_t nq;
  uint32_t nwords;       // bitmap words (n bits)
  uint32_t* gbitmap;     // [gridDim.x][nwords] when not in shared memory
  uint32_t* counter;     // dynamic query fetch
};

__global__ void __launch_bounds__(CO_THREADS) k_collect(CollectArgs a) {
  extern __shared__ uint32_t sbm[];
  __shared__ uint32_t pref[CO_TILE + 1];
  __shared__ uint64_t tpos[CO_TILE];
  __shared__ uint32_t sh[32];
  __shared__ uint32_t ucount;
  __shared__ uint32_t qsh;
  uint32_t* bm = a.gbitmap ? a.gbitmap + (uint64_t)blockIdx.x * a.nwords : sbm;
  if (a.gbitmap) {  // global bitmaps start zeroed and are cleared by candidate list
  }
  for (;;) {
    if (threadIdx.x == 0) qsh = atomicAdd(a.counter, 1u);
    __syncthreads();
    const uint32_t q = qsh;
    if (q >= a.nq) break;
    if (!a.gbitmap) {
      for (uint32_t w = threadIdx.x; w < a.nwords; w += blockDim.x) bm[w] = 0;
    }
    if (threadIdx.x == 0) ucount = 0;
    __syncthreads();
    uint32_t* out = a.cands + a.coff[q];
    const uint64_t* pp = a.ppos + (uint64_t)q * a.peff;
    const uint32_t* pl = a.plen + (uint64_t)q * a.peff;
    for (uint64_t p0 = 0; p0 < a.peff; p0 += CO_TILE) {
      const uint32_t np = (uint32_t)(a.peff - p0 < (uint64_t)CO_TILE ? a.peff - p0 : (uint64_t)CO_TILE);
      uint32_t v[2] = {0, 0};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const uint32_t i = threadIdx.x * 2 + k;
        if (i < np) {
          v[k] = pl[p0 + i];
          tpos[i] = pp[p0 + i];
        }
      }
      uint32_t tot;
      const uint32_t ex = block_excl_scan_u32(v[0] + v[1], sh, &tot);
      if (threadIdx.x * 2 < np) pref[threadIdx.x * 2] = ex;
      if (threadIdx.x * 2 + 1 < np) pref[threadIdx.x * 2 + 1] = ex + v[0];
      if (threadIdx.x == 0) pref[np] = tot;
      __syncthreads();
      for (uint32_t e = threadIdx.x; e < tot; e += blockDim.x) {
        // probe containing entry e: last p with pref[p] <= e
        uint32_t lo = 0, hi = np;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (pref[mid] <= e) lo = mid;
          else hi = mid;
        }
        const uint32_t id = __ldg(a.ids + tpos[lo] + (e - pref[lo]));
        const uint32_t bit = 1u << (id & 31);
        const uint32_t old = atomicOr(bm + (id >> 5), bit);
        const bool isnew = !(old & bit);
        const unsigned act = __activemask();
        const unsigned bal = __ballot_sync(act, isnew);
        if (bal) {
          const int lane = threadIdx.x & 31;
          const int leader = __ffs(act) - 1;
          uint32_t base = 0;
          if (lane == leader) base = atomicAdd(&ucount, __popc(bal));
          base = __shfl_sync(act, base, leader);
          if (isnew) out[base + __popc(bal & ((1u << lane) - 1))] = id;
        }
      }
      __syncthreads();
    }
    const uint32_t U = ucount;
    if (threadIdx.x == 0) a.uq[q] = U;
    if (a.gbitmap) {
      __syncthreads();
      for (uint32_t c = threadIdx.x; c < U; c += blockDim.x) bm[out[c] >> 5] = 0;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------- score
constexpr int SC_WARPS = 4;
constexpr int SC_SLICE = 32;              // floats per row slice
constexpr int SC_STAGES = 4;              // cp.async ring depth per warp
constexpr int SC_ROWPAD = SC_SLICE + 4;   // odd number of 16 B units: conflict-free LDS.128
constexpr int SC_STAGE_FLOATS = 32 * SC_ROWPAD;

struct ScoreArgs {
  const float* X;
  uint32_t d;
  const float* Q;
  const uint64_t* coff;
  const uint32_t* cands;
  const uint32_t* uq;
  const uint32_t* eq;
  uint64_t peff;
  uint32_t k;
  uint32_t id_offset;
  uint32_t* out_ids;
  double* out_scores;
  fpp_query_stats* stats;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// warp top-k: lane i < k holds the i-th best (score desc, id asc)
__device__ __forceinline__ bool sbetter(double s1, uint32_t i1, double s2, uint32_t i2) {
  return s1 > s2 || (s1 == s2 && i1 < i2);
}
__device__ __forceinline__ void topk_insert(double& bs, uint32_t& bi, uint32_t k, double cs_l,
                                            uint32_t ci_l, bool valid) {
  const int lane = threadIdx.x & 31;
  double ws = __shfl_sync(FULL, bs, k - 1);
  uint32_t wi = __shfl_sync(FULL, bi, k - 1);
  unsigned m = __ballot_sync(FULL, valid && sbetter(cs_l, ci_l, ws, wi));
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const double cs = __shfl_sync(FULL, cs_l, src);
    const uint32_t ci = __shfl_sync(FULL, ci_l, src);
    ws = __shfl_sync(FULL, bs, k - 1);
    wi = __shfl_sync(FULL, bi, k - 1);
    if (!sbetter(cs, ci, ws, wi)) continue;
    const unsigned ahead = __ballot_sync(FULL, (uint32_t)lane < k && sbetter(bs, bi, cs, ci));
    const int pos = __popc(ahead);
    const double us = __shfl_up_sync(FULL, bs, 1);
    const uint32_t ui = __shfl_up_sync(FULL, bi, 1);
    if (lane > pos && (uint32_t)lane < k) { bs = us; bi = ui; }
    if (lane == pos) { bs = cs; bi = ci; }
  }
}

__global__ void __launch_bounds__(SC_WARPS * 32, 2) k_score(ScoreArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const uint32_t d = a.d;
  double* qd = reinterpret_cast<double*>(smraw);
  const uint32_t qd_bytes = ((d * 8 + 127) / 128) * 128;
  float* ring = reinterpret_cast<float*>(smraw + qd_bytes);
  __shared__ double mg_s[SC_WARPS][32];
  __shared__ uint32_t mg_i[SC_WARPS][32];
  const uint32_t q = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) qd[j] = (double)a.Q[(uint64_t)q * d + j];
  __syncthreads();
  const uint32_t U = a.uq[q];
  const uint32_t* cand = a.cands + a.coff[q];
  const uint32_t k = a.k;
  double bs = -INFINITY;
  uint32_t bi = 0xffffffffu;
  float* wring = ring + (size_t)w * SC_STAGES * SC_STAGE_FLOATS;
  const uint32_t nb = (U + 31) / 32;
  const uint32_t my_nb = nb > (uint32_t)w ? (nb - w + SC_WARPS - 1) / SC_WARPS : 0;
  const uint32_t nsl = (d + SC_SLICE - 1) / SC_SLICE;
  const uint64_t S = (uint64_t)my_nb * nsl;
  const bool vec = (d & 3u) == 0;
  uint32_t iss_id = 0;
  uint32_t iss_b = 0xffffffffu;
  auto issue = [&](uint64_t step) {
    if (step < S) {
      const uint32_t bl = (uint32_t)(step / nsl), c = (uint32_t)(step - (uint64_t)bl * nsl);
      const uint32_t bidx = w + bl * SC_WARPS;
      if (bidx != iss_b) {
        iss_b = bidx;
        const uint32_t ci = bidx * 32 + lane;
        iss_id = ci < U ? __ldg(cand + ci) : 0xffffffffu;
      }
      float* buf = wring + (size_t)(step % SC_STAGES) * SC_STAGE_FLOATS;
      const uint32_t col0 = c * SC_SLICE;
      const uint32_t len = min((uint32_t)SC_SLICE, d - col0);
      if (vec) {
        const uint32_t npc = len >> 2;  // 16 B pieces per row
        for (uint32_t it = 0; it < npc; ++it) {
          const uint32_t p = lane + 32 * it;
          const uint32_t r = p / npc, kk = p - r * npc;
          const uint32_t id = __shfl_sync(FULL, iss_id, r);
          if (id != 0xffffffffu)
            cp_async16(buf + r * SC_ROWPAD + kk * 4, a.X + (uint64_t)id * d + col0 + kk * 4);
        }
      } else {
        for (uint32_t it = 0; it < len; ++it) {
          const uint32_t p = lane + 32 * it;
          const uint32_t r = p / len, kk = p - r * len;
          const uint32_t id = __shfl_sync(FULL, iss_id, r);
          if (id != 0xffffffffu) cp_async4(buf + r * SC_ROWPAD + kk, a.X + (uint64_t)id * d + col0 + kk);
        }
      }
    }
    cp_commit();
  };
#pragma unroll
  for (int st = 0; st < SC_STAGES - 1; ++st) issue(st);
  double acc = 0.0;
  for (uint64_t step = 0; step < S; ++step) {
    issue(step + SC_STAGES - 1);
    cp_wait<SC_STAGES - 1>();
    __syncwarp();
    const uint32_t bl = (uint32_t)(step / nsl), c = (uint32_t)(step - (uint64_t)bl * nsl);
    const float* row = wring + (size_t)(step % SC_STAGES) * SC_STAGE_FLOATS + lane * SC_ROWPAD;
    const uint32_t col0 = c * SC_SLICE;
    const uint32_t len = min((uint32_t)SC_SLICE, d - col0);
    const double* qq = qd + col0;
    if (vec) {
      for (uint32_t j = 0; j < len; j += 4) {
        const float4 xv = *reinterpret_cast<const float4*>(row + j);
        // dataset.cpp:67 acc += double(a[i]) * double(b[i]), sequential i
        acc = fma((double)xv.x, qq[j], acc);
        acc = fma((double)xv.y, qq[j + 1], acc);
        acc = fma((double)xv.z, qq[j + 2], acc);
        acc = fma((double)xv.w, qq[j + 3], acc);
      }
    } else {
      for (uint32_t j = 0; j < len; ++j) acc = fma((double)row[j], qq[j], acc);
    }
    __syncwarp();
    if (c == nsl - 1) {
      const uint32_t ci = (w + bl * SC_WARPS) * 32 + lane;
      const bool valid = ci < U;
      const uint32_t id = valid ? __ldg(cand + ci) : 0xffffffffu;
      topk_insert(bs, bi, k, acc, id, valid);
      acc = 0.0;
    }
  }
  cp_wait<0>();
  // CTA merge of the warp lists
  mg_s[w][lane] = bs;
  mg_i[w][lane] = bi;
  __syncthreads();
  if (w == 0) {
    for (int w2 = 1; w2 < SC_WARPS; ++w2) {
      const bool valid = (uint32_t)lane < k && mg_i[w2][lane] != 0xffffffffu;
      topk_insert(bs, bi, k, mg_s[w2][lane], mg_i[w2][lane], valid);
    }
    if ((uint32_t)lane < k) {
      const bool ok = bi != 0xffffffffu;
      a.out_ids[(uint64_t)q * k + lane] = ok ? bi + a.id_offset : 0xffffffffu;
      a.out_scores[(uint64_t)q * k + lane] = ok ? bs : -INFINITY;
    }
    if (lane == 0 && a.stats) {
      a.stats[q].probes = a.peff;
      a.stats[q].entries = a.eq[q];
      a.stats[q].candidates = U;
    }
  }
}

static size_t score_smem(uint32_t d) {
  return ((d * 8 + 127) / 128) * 128 + (size_t)SC_WARPS * SC_STAGES * SC_STAGE_FLOATS * 4;
}

// ------------------------------------------------------------ host driver
void launch_query_lists(const Index& ix, const float* Qd, uint64_t nq, uint32_t s_cap,
                        float* vals, uint32_t* codes, cudaStream_t s) {
  if (nq == 0) return;
  dim3 grid((unsigned)nq, ix.prm.L);
  const uint32_t d = ix.d, D = ix.prm.D, K = ix.prm.K, L = ix.prm.L;
#define FPP_QL_CASE(PP)                                                                      \
  case PP:                                                                                   \
    k_query_lists<PP><<<grid, 256, 0, s>>>(Qd, d, D, K, ix.signs, L, s_cap, vals, codes);    \
    break;
  switch (ix.P) {
    FPP_QL_CASE(2) FPP_QL_CASE(4) FPP_QL_CASE(8) FPP_QL_CASE(16) FPP_QL_CASE(32)
    FPP_QL_CASE(64) FPP_QL_CASE(128) FPP_QL_CASE(256) FPP_QL_CASE(512) FPP_QL_CASE(1024)
    default: fail(FPP_ERR_UNSUPPORTED, "query: padded dimension > 1024 not supported on GPU");
  }
#undef FPP_QL_CASE
  FPP_LAUNCH();
}

static int co_smem_max() {
  static int v = -1;
  if (v < 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    v = optin;
  }
  return v;
}

// run one chunk; dbg_probes optional
static void run_chunk(const Index& ix, const float* Qd, uint32_t nqc, uint32_t k, uint32_t qprobes,
                      uint32_t* ids_d, double* scores_d, fpp_query_stats* stats_d, cudaStream_t s,
                      uint64_t* dbg_probes) {
  const uint32_t L = ix.prm.L, K = ix.prm.K;
  const uint32_t scap = query_cap(ix, qprobes);
  const uint64_t peff = query_probes(ix, qprobes);
  const uint64_t LKs = (uint64_t)L * K * scap;
  ix.q_vals.ensure((size_t)nqc * LKs);
  ix.q_codes.ensure((size_t)nqc * LKs);
  ix.q_ppos.ensure((size_t)nqc * peff);
  ix.q_plen.ensure((size_t)nqc * peff);
  ix.q_eq.ensure(nqc);
  ix.q_uq.ensure(nqc);
  ix.q_coff.ensure((size_t)nqc + 1);
  ix.q_counter.ensure(4);

  cudaEvent_t e0;
  ix.timer.begin(PH_QHASH, s, &e0);
  launch_query_lists(ix, Qd, nqc, scap, ix.q_vals.p, ix.q_codes.p, s);
  ix.timer.end(PH_QHASH, e0, s);

  ix.timer.begin(PH_PROBE, s, &e0);
  ProbeArgs pa{ix.q_vals.p, ix.q_codes.p, L, K, scap, ix.prm.D, ix.NB, peff, ix.offsets,
               ix.table_base, ix.q_ppos.p, ix.q_plen.p, ix.q_eq.p, dbg_probes, 0};
  size_t ps_smem = LKs * sizeof(float);
  const int smax = co_smem_max() - 4096;
  if ((int)ps_smem <= smax) {
    pa.use_smem = 1;
    FPP_CUDA(cudaFuncSetAttribute(k_probe_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ps_smem));
  } else {
    ps_smem = 0;
  }
  k_probe_select<<<nqc, PS_THREADS, ps_smem, s>>>(pa);
  FPP_LAUNCH();
  k_scan_eq<<<1, 1024, 0, s>>>(ix.q_eq.p, nqc, ix.q_coff.p);
  FPP_LAUNCH();
  FPP_CUDA(cudaMemcpyAsync(ix.h_pinned, ix.q_coff.p + nqc, sizeof(uint64_t),
                           cudaMemcpyDeviceToHost, s));
  ix.timer.end(PH_PROBE, e0, s);
  FPP_CUDA(cudaStreamSynchronize(s));
  const uint64_t etot = ix.h_pinned[0];
  ix.q_cands.ensure(etot + 1);

  ix.timer.begin(PH_COLLECT, s, &e0);
  const uint32_t nwords = (uint32_t)((ix.n + 31) / 32);
  CollectArgs ca{ix.q_ppos.p, ix.q_plen.p, peff, ix.ids, ix.q_coff.p, ix.q_cands.p, ix.q_uq.p,
                 nqc, nwords, nullptr, ix.q_counter.p};
  const size_t static_co = (CO_TILE + 1) * 4 + CO_TILE * 8 + 32 * 4 + 16;
  size_t co_smem = (size_t)nwords * 4;
  unsigned co_grid;
  const int sms = sm_count();
  if ((int)(co_smem + static_co) <= co_smem_max()) {
    FPP_CUDA(cudaFuncSetAttribute(k_collect, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)co_smem));
    int occ = 1;
    FPP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_collect, CO_THREADS, co_smem));
    co_grid = (unsigned)std::min<uint64_t>(nqc, (uint64_t)sms * std::max(occ, 1));
  } else {
    co_smem = 0;
    co_grid = (unsigned)std::min<uint64_t>(nqc, (uint64_t)sms * 2);
    const size_t need = (size_t)co_grid * nwords;
    if (ix.q_bitmap.n < need) {
      ix.q_bitmap.alloc(need);
      FPP_CUDA(cudaMemsetAsync(ix.q_bitmap.p, 0, need * 4, s));
    }
    ca.gbitmap = ix.q_bitmap.p;
  }
  FPP_CUDA(cudaMemsetAsync(ix.q_counter.p, 0, sizeof(uint32_t), s));
  k_collect<<<co_grid, CO_THREADS, co_smem, s>>>(ca);
  FPP_LAUNCH();
  ix.timer.end(PH_COLLECT, e0, s);

  ix.timer.begin(PH_SCORE, s, &e0);
  ScoreArgs sa{ix.X, ix.d, Qd, ix.q_coff.p, ix.q_cands.p, ix.q_uq.p, ix.q_eq.p, peff, k,
               ix.prm.id_offset, ids_d, scores_d, stats_d};
  const size_t sc_smem = score_smem(ix.d);
  FPP_CUDA(cudaFuncSetAttribute(k_score, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sc_smem));
  k_score<<<nqc, SC_WARPS * 32, sc_smem, s>>>(sa);
  FPP_LAUNCH();
  ix.timer.end(PH_SCORE, e0, s);
  ix.acc.launches += 5;  // lists, probe_select, scan_eq, collect, score
  ix.acc.probes += peff * nqc;
}

static uint32_t chunk_size(const Index& ix, uint32_t qprobes, uint64_t nq) {
  const uint64_t LKs = (uint64_t)ix.prm.L * ix.prm.K * query_cap(ix, qprobes);
  const uint64_t per_q = LKs * 8 + query_probes(ix, qprobes) * 12 + 64;
  uint64_t c = (1ull << 31) / per_q;  // ~2 GB of per-chunk scratch
  c = std::max<uint64_t>(1, std::min<uint64_t>(c, 16384));
  return (uint32_t)std::min<uint64_t>(c, nq);
}

void run_query(const Index& ix, const float* Qd, uint64_t nq, uint32_t k, uint32_t qprobes,
               uint32_t* ids_d, double* scores_d, fpp_query_stats* stats_d, cudaStream_t s) {
  const uint32_t cs = chunk_size(ix, qprobes, nq);
  for (uint64_t q0 = 0; q0 < nq; q0 += cs) {
    const uint32_t nqc = (uint32_t)std::min<uint64_t>(cs, nq - q0);
    run_chunk(ix, Qd + q0 * ix.d, nqc, k, qprobes, ids_d + q0 * k, scores_d + q0 * k,
              stats_d ? stats_d + q0 : nullptr, s, nullptr);
  }
}

void query_debug(const Index& ix, const float* qd, uint32_t qprobes, std::vector<uint64_t>& probes,
                 std::vector<uint32_t>& cands) {
  cudaStream_t s = ix.stream;
  const uint64_t peff = query_probes(ix, qprobes);
  DBuf<uint64_t> dbg(peff);
  DBuf<uint32_t> ids(32);
  DBuf<double> sc(32);
  run_chunk(ix, qd, 1, 1, qprobes, ids.p, sc.p, nullptr, s, dbg.p);
  FPP_CUDA(cudaStreamSynchronize(s));
  probes.resize(peff);
  FPP_CUDA(cudaMemcpy(probes.data(), dbg.p, peff * 8, cudaMemcpyDeviceToHost));
  uint32_t U = 0;
  uint64_t off = 0;
  FPP_CUDA(cudaMemcpy(&U, ix.q_uq.p, 4, cudaMemcpyDeviceToHost));
  FPP_CUDA(cudaMemcpy(&off, ix.q_coff.p, 8, cudaMemcpyDeviceToHost));
  cands.resize(U);
  if (U) FPP_CUDA(cudaMemcpy(cands.data(), ix.q_cands.p + off, (size_t)U * 4, cudaMemcpyDeviceToHost));
  std::sort(probes.begin(), probes.end());
  std::sort(cands.begin(), cands.end());
}

}  // namespace fpp
