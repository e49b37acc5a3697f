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
// One lane group (G = P/EPT lanes) per (query, table, function): spinner
// projections in registers, register bitonic sort of the (|p| desc, j asc) rank
// keys, the first min(s,D) written out; when s > D a second sort of the
// (|p| asc, j asc) keys supplies the opposite-signed tail.
template <int P>
__global__ void __launch_bounds__(128)
k_query_lists(const float* __restrict__ Q, uint64_t nq, uint32_t d, uint32_t D, uint32_t K,
              const uint32_t* __restrict__ signs, uint32_t L, uint32_t s,
              float* __restrict__ vals, uint32_t* __restrict__ codes) {
  using S = FhtShape<P>;
  constexpr int EPT = S::EPT;
  const int lane = threadIdx.x & 31;
  const int g = lane % S::G;
  const uint64_t gg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / S::G;
  const uint64_t total = nq * L * K;
  const bool active = gg < total;
  const uint64_t gid = active ? gg : total - 1;
  const uint32_t f = (uint32_t)(gid % K);
  const uint32_t t = (uint32_t)((gid / K) % L);
  const uint64_t q = gid / ((uint64_t)K * L);
  float v[EPT];
  load_row<P>(Q + q * d, d, g, v);
  spinner_project<P>(v, signs + ((uint64_t)t * K + f) * 3 * S::W, g);
  uint64_t key[EPT];
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const uint32_t j = (uint32_t)g * EPT + e;
    key[e] = j < D ? rank_key(v[e], j) : ~0ull;
  }
  group_bitonic_sort<P, EPT>(key, g);
  const uint64_t ob = gid * s;
  const uint32_t nat = s < D ? s : D;
  if (active) {
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t r = (uint32_t)g * EPT + e;
      if (r < nat) {
        vals[ob + r] = rank_val(key[e]);
        codes[ob + r] = rank_code(key[e], D);
      }
    }
  }
  if (s > D) {  // opposite signed vectors: (|p| asc, j asc), value -|p|
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t j = (uint32_t)g * EPT + e;
      key[e] = j < D ? (((uint64_t)ord_key(fabsf(v[e])) << 32) | ((uint64_t)j << 1) |
                        (v[e] < 0.0f ? 1u : 0u))
                     : ~0ull;
    }
    group_bitonic_sort<P, EPT>(key, g);
    if (active) {
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const uint32_t r = (uint32_t)g * EPT + e;
        if (r < s - D) {
          const uint64_t kk = key[e];
          const uint32_t j = (uint32_t)(kk & 0xffffffffu) >> 1;
          vals[ob + D + r] = -ord_inv((uint32_t)(kk >> 32));
          codes[ob + D + r] = (kk & 1u) ? j : D + j;
        }
      }
    }
  }
}

// ------------------------------------------------------------ probe select
// CTA per query, one thread per table.  The probe set is {true bucket of each
// table} U the M = P_eff - L best remaining (t, r1, r2) under
// (fl(v1[r1]+v2[r2]) desc, r1, r2, t).  fp32 rounding is
// monotone, so in every table the pairs scoring >= T form a staircase that a
// two-pointer walk counts in O(active r1 + active r2).  T* (the M-th best
// score) is found by a galloping + binary search on the ordered-key space, the
// walks touching only the active prefixes of the ranked lists (L1-resident).
// Ties at T* are resolved exactly in (r1, r2, t) order.
constexpr int PS_THREADS = 128;
constexpr int PS_TIE_CAP = 1024;

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
};

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
__device__ __forceinline__ uint32_t block_max_u32(uint32_t v, uint32_t* sh) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  uint32_t t = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = max(t, sh[i]);
  __syncthreads();
  return t;
}

__device__ const float g_zero_row[1] = {0.0f};

struct TableLists {
  const float* v1;  // [s]
  const float* v2;  // [S2] (a zero row when K == 1)
  uint32_t s1, S2;
};

// number of non-forced pairs with key >= T (two-pointer staircase walk)
__device__ __forceinline__ uint32_t walk_count(const TableLists& tl, uint32_t T) {
  uint32_t p = 0;
  const float x0 = __ldg(tl.v1);
  while (p < tl.S2 && ord_key(x0 + __ldg(tl.v2 + p)) >= T) ++p;
  uint32_t c = p > 0 ? p - 1 : 0;  // exclude the forced (0,0)
  for (uint32_t r1 = 1; r1 < tl.s1 && p > 0; ++r1) {
    const float x = __ldg(tl.v1 + r1);
    while (p > 0 && ord_key(x + __ldg(tl.v2 + p - 1)) < T) --p;
    c += p;
  }
  return c;
}

// visit (r1, pa, pb): prefixes at Ta > Tb (pa <= pb), r1 ascending while pb > 0
template <class F>
__device__ __forceinline__ void walk2(const TableLists& tl, uint32_t Ta, uint32_t Tb, F&& visit) {
  uint32_t pb = 0;
  const float x0 = __ldg(tl.v1);
  while (pb < tl.S2 && ord_key(x0 + __ldg(tl.v2 + pb)) >= Tb) ++pb;
  uint32_t pa = 0;
  while (pa < pb && ord_key(x0 + __ldg(tl.v2 + pa)) >= Ta) ++pa;
  visit(0u, pa, pb);
  for (uint32_t r1 = 1; r1 < tl.s1 && pb > 0; ++r1) {
    const float x = __ldg(tl.v1 + r1);
    while (pb > 0 && ord_key(x + __ldg(tl.v2 + pb - 1)) < Tb) --pb;
    while (pa > 0 && ord_key(x + __ldg(tl.v2 + pa - 1)) < Ta) --pa;
    if (pa > pb) pa = pb;
    visit(r1, pa, pb);
  }
}

__global__ void __launch_bounds__(PS_THREADS) k_probe_select(ProbeArgs a) {
  __shared__ uint64_t red[32];
  __shared__ uint32_t redu[32];
  __shared__ uint64_t ties[PS_TIE_CAP];
  __shared__ uint32_t n_ties;
  const uint32_t q = blockIdx.x;
  const uint32_t L = a.L, K = a.K, s = a.s;
  const uint32_t S2 = K == 2 ? s : 1;
  const uint64_t LKs = (uint64_t)L * K * s;
  const float* V = a.vals + (uint64_t)q * LKs;
  const uint32_t* Cq = a.codes + (uint64_t)q * LKs;
  if (threadIdx.x == 0) n_ties = 0;
  __syncthreads();
  auto lists = [&](uint32_t t) {
    TableLists tl;
    tl.v1 = V + (uint64_t)t * K * s;
    tl.v2 = K == 2 ? tl.v1 + s : g_zero_row;
    tl.s1 = s;
    tl.S2 = S2;
    return tl;
  };
  const uint64_t M = a.peff - L;  // non-forced probes
  auto count = [&](uint32_t T) -> uint64_t {
    uint64_t c = 0;
    for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) c += walk_count(lists(t), T);
    return block_sum_u64(c, red);
  };
  uint32_t Tstar = 0;
  if (M > 0) {
    // best non-forced key over all tables: max(v1[0]+v2[1], v1[1]+v2[0])
    uint32_t hi = 0;
    for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) {
      const TableLists tl = lists(t);
      const float x0 = __ldg(tl.v1);
      if (S2 > 1) hi = max(hi, ord_key(x0 + __ldg(tl.v2 + 1)));
      if (s > 1) hi = max(hi, ord_key(__ldg(tl.v1 + 1) + __ldg(tl.v2)));
    }
    hi = block_max_u32(hi, redu);
    // gallop down from hi until count >= M, then bisect: Tstar = max T with count(T) >= M
    uint32_t bad = 0xffffffffu;  // count(bad) < M (or sentinel)
    uint32_t T = hi, step = 1;
    bool have_bad = false;
    for (;;) {
      if (count(T) >= M) break;
      bad = T;
      have_bad = true;
      T = T > step ? T - step : 0;
      step <<= 1;
      if (T == 0) break;  // count(0) counts every pair >= M
    }
    uint32_t lo = T;
    if (have_bad) {
      while (bad - lo > 1) {
        const uint32_t mid = lo + (bad - lo) / 2;
        if (count(mid) >= M) lo = mid;
        else bad = mid;
      }
    } else {
      // count(hi) >= M already: search upward is impossible (hi is the max key)
    }
    Tstar = lo;
  }
  const uint32_t Ta = Tstar == 0xffffffffu ? 0xffffffffu : Tstar + 1;  // strictly above T*
  // per-thread gt / tie counts
  uint64_t my_gt = 0, my_tie = 0;
  if (M > 0) {
    for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) {
      walk2(lists(t), Ta, Tstar, [&](uint32_t r1, uint32_t pa, uint32_t pb) {
        const uint32_t st = r1 == 0 ? 1 : 0;
        const uint32_t ga = max(st, pa), gb = max(st, pb);
        my_gt += ga - st;
        my_tie += gb - ga;
      });
    }
  }
  const uint64_t cgt = block_sum_u64(my_gt, red);
  const uint64_t ties_total = block_sum_u64(my_tie, red);
  const uint64_t m = M > cgt ? M - cgt : 0;  // ties to take
  // composite tie key (r1*S2 + r2)*L + t: order (r1, r2, t); take keys < Kstar
  uint64_t Kstar = ~0ull;
  if (M > 0 && ties_total > m) {
    if (ties_total <= PS_TIE_CAP) {
      for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) {
        walk2(lists(t), Ta, Tstar, [&](uint32_t r1, uint32_t pa, uint32_t pb) {
          const uint32_t st = r1 == 0 ? 1 : 0;
          for (uint32_t r2 = max(st, pa); r2 < max(st, pb); ++r2)
            ties[atomicAdd(&n_ties, 1u)] = ((uint64_t)r1 * S2 + r2) * L + t;
        });
      }
      __syncthreads();
      uint32_t N = 1;
      while (N < ties_total) N <<= 1;
      for (uint32_t i = ties_total + threadIdx.x; i < N; i += blockDim.x) ties[i] = ~0ull;
      __syncthreads();
      for (uint32_t kk = 2; kk <= N; kk <<= 1)
        for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
          for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
            const uint32_t ixj = i ^ jj;
            if (ixj > i) {
              const uint64_t x = ties[i], y = ties[ixj];
              if ((x > y) == ((i & kk) == 0)) { ties[i] = y; ties[ixj] = x; }
            }
          }
          __syncthreads();
        }
      Kstar = ties[m];  // keys < ties[m] are the m smallest
      __syncthreads();
    } else {
      // many ties: bisect the composite key with counting walks
      auto count_lt = [&](uint64_t Kc) -> uint64_t {
        const uint64_t kr1 = Kc / ((uint64_t)S2 * L);
        const uint64_t rem = Kc - kr1 * S2 * L;
        const uint64_t kr2 = rem / L, kt = rem - kr2 * L;
        uint64_t c = 0;
        for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) {
          walk2(lists(t), Ta, Tstar, [&](uint32_t r1, uint32_t pa, uint32_t pb) {
            const uint32_t st = r1 == 0 ? 1 : 0;
            const uint64_t ga = max(st, pa), gb = max(st, pb);
            if (ga == gb || r1 > kr1) return;
            if (r1 < kr1) { c += gb - ga; return; }
            if (kr2 > ga) c += (kr2 < gb ? kr2 : gb) - ga;
            if (kr2 >= ga && kr2 < gb && t < kt) c += 1;
          });
        }
        return block_sum_u64(c, red);
      };
      uint64_t lo = 0, hi = (uint64_t)s * S2 * L;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (count_lt(mid) >= m) hi = mid;
        else lo = mid + 1;
      }
      Kstar = lo;
    }
  }
  // emission counts, exclusive scan over threads
  uint64_t mine = 0;
  if (M > 0) {
    for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) {
      walk2(lists(t), Ta, Tstar, [&](uint32_t r1, uint32_t pa, uint32_t pb) {
        const uint32_t st = r1 == 0 ? 1 : 0;
        const uint32_t ga = max(st, pa), gb = max(st, pb);
        mine += ga - st;
        if (Kstar == ~0ull) mine += gb - ga;
        else
          for (uint32_t r2 = ga; r2 < gb; ++r2) mine += (((uint64_t)r1 * S2 + r2) * L + t) < Kstar;
      });
    }
  }
  uint64_t x = mine;
  {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) red[w] = x;
    __syncthreads();
    uint64_t wb = 0;
    for (int i = 0; i < w; ++i) wb += red[i];
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
    const uint32_t o0 = __ldg(of + b), o1 = __ldg(of + b + 1);
    ppos[slot] = __ldg(a.tbase + t) + o0;
    plen[slot] = o1 - o0;
    esum += o1 - o0;
    if (dbg) dbg[slot] = (uint64_t)t * a.NB + b;
  };
  for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) {
    const uint32_t* c1 = Cq + (uint64_t)t * K * s;
    const uint32_t* c2 = c1 + s;
    emit(t, t, K == 2 ? __ldg(c1) * twoD + __ldg(c2) : __ldg(c1));
  }
  if (M > 0) {
    uint64_t slot = L + x;
    for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) {
      const uint32_t* c1 = Cq + (uint64_t)t * K * s;
      const uint32_t* c2 = c1 + s;
      walk2(lists(t), Ta, Tstar, [&](uint32_t r1, uint32_t pa, uint32_t pb) {
        const uint32_t st = r1 == 0 ? 1 : 0;
        const uint32_t ga = max(st, pa), gb = max(st, pb);
        const uint32_t h1 = __ldg(c1 + r1);
        for (uint32_t r2 = st; r2 < gb; ++r2) {
          if (r2 >= ga && Kstar != ~0ull && (((uint64_t)r1 * S2 + r2) * L + t) >= Kstar) continue;
          emit(slot++, t, K == 2 ? h1 * twoD + __ldg(c2 + r2) : h1);
        }
      });
    }
  }
  esum = block_sum_u64(esum, red);
  if (threadIdx.x == 0) a.eq[q] = (uint32_t)esum;
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

// Per warp: 32-candidate batches; every batch streams its rows as 32-float
// column slices through a SC_STAGES-deep cp.async ring.  Lane l copies the 16 B
// chunk (l & 7) of rows (l >> 3) + 4*it, it = 0..7, with row addresses resolved
// once per batch, so a slice costs 8 cp.async per lane.  Lane r then folds row
// r's slice into its fp64 accumulator in the reference's sequential order.
template <bool VEC>
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
  const uint32_t nsl = (d + SC_SLICE - 1) / SC_SLICE;
  const float* X = a.X;
  // issue cursor
  uint32_t ib = w, ic = 0, nissued = 0;
  const float* rp[8];
  uint32_t my_id = 0xffffffffu;
  const int kk = lane & 7, rbase = lane >> 3;
  auto load_batch = [&](uint32_t bidx) {
    const uint32_t ci = bidx * 32 + lane;
    my_id = ci < U ? __ldg(cand + ci) : 0xffffffffu;
    if (VEC) {
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const uint32_t idr = __shfl_sync(FULL, my_id, rbase + 4 * it);
        rp[it] = idr != 0xffffffffu ? X + (uint64_t)idr * d : nullptr;
      }
    }
  };
  auto issue = [&]() {
    if (ib < nb) {
      float* buf = wring + (size_t)(nissued % SC_STAGES) * SC_STAGE_FLOATS;
      const uint32_t col0 = ic * SC_SLICE;
      const uint32_t len = min((uint32_t)SC_SLICE, d - col0);
      if (VEC) {
        if ((uint32_t)kk < (len >> 2)) {
#pragma unroll
          for (int it = 0; it < 8; ++it)
            if (rp[it]) cp_async16(buf + (rbase + 4 * it) * SC_ROWPAD + kk * 4, rp[it] + col0 + kk * 4);
        }
      } else {
        for (int r = 0; r < 32; ++r) {
          const uint32_t idr = __shfl_sync(FULL, my_id, r);
          if (idr != 0xffffffffu && (uint32_t)lane < len)
            cp_async4(buf + r * SC_ROWPAD + lane, X + (uint64_t)idr * d + col0 + lane);
        }
      }
      if (++ic == nsl) {
        ic = 0;
        ib += SC_WARPS;
        if (ib < nb) load_batch(ib);
      }
    }
    cp_commit();
    ++nissued;
  };
  if ((uint32_t)w < nb) load_batch(w);
#pragma unroll
  for (int st = 0; st < SC_STAGES - 1; ++st) issue();
  double acc = 0.0;
  uint32_t cb = w, cc = 0, ncomp = 0;
  while (cb < nb) {
    issue();
    cp_wait<SC_STAGES - 1>();
    __syncwarp();
    const float* row = wring + (size_t)(ncomp % SC_STAGES) * SC_STAGE_FLOATS + lane * SC_ROWPAD;
    const uint32_t col0 = cc * SC_SLICE;
    const uint32_t len = min((uint32_t)SC_SLICE, d - col0);
    const double* qq = qd + col0;
    // dataset.cpp:67 acc += double(a[i]) * double(b[i]), sequential i (exact products)
    if (VEC && len == SC_SLICE) {
#pragma unroll
      for (int j = 0; j < SC_SLICE; j += 4) {
        const float4 xv = *reinterpret_cast<const float4*>(row + j);
        acc = fma((double)xv.x, qq[j], acc);
        acc = fma((double)xv.y, qq[j + 1], acc);
        acc = fma((double)xv.z, qq[j + 2], acc);
        acc = fma((double)xv.w, qq[j + 3], acc);
      }
    } else {
      for (uint32_t j = 0; j < len; ++j) acc = fma((double)row[j], qq[j], acc);
    }
    __syncwarp();
    ++ncomp;
    if (++cc == nsl) {
      const uint32_t ci = cb * 32 + lane;
      const bool valid = ci < U;
      const uint32_t id = valid ? __ldg(cand + ci) : 0xffffffffu;
      topk_insert(bs, bi, k, acc, id, valid);
      acc = 0.0;
      cc = 0;
      cb += SC_WARPS;
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
  const uint32_t d = ix.d, D = ix.prm.D, K = ix.prm.K, L = ix.prm.L;
  const uint32_t G = ix.P < 32 ? 1 : ix.P / 32;
  const unsigned grid = (unsigned)((nq * L * K * G + 127) / 128);
#define FPP_QL_CASE(PP)                                                                      \
  case PP:                                                                                   \
    k_query_lists<PP><<<grid, 128, 0, s>>>(Qd, nq, d, D, K, ix.signs, L, s_cap, vals, codes); \
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
               ix.table_base, ix.q_ppos.p, ix.q_plen.p, ix.q_eq.p, dbg_probes};
  k_probe_select<<<nqc, PS_THREADS, 0, s>>>(pa);
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
  if ((ix.d & 3u) == 0) {
    FPP_CUDA(cudaFuncSetAttribute(k_score<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sc_smem));
    k_score<true><<<nqc, SC_WARPS * 32, sc_smem, s>>>(sa);
  } else {
    FPP_CUDA(cudaFuncSetAttribute(k_score<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sc_smem));
    k_score<false><<<nqc, SC_WARPS * 32, sc_smem, s>>>(sa);
  }
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
