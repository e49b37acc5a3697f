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
//   k_collect       CTA per query: walk kept entries, OR them into a visited
//                   bitmap in shared memory and emit unique ids in ascending
//                   order; large shards dedup by id-range groups (counting
//                   sort + per-warp range bitmaps), else an 8-CTA DSMEM
//                   cluster or global-memory bitmap
//   k_score         CTA per query: 32-row batches per warp, cp.async column
//                   slices into shared memory (multi-stage ring), each lane
//                   accumulates its row's exact products in fp64 in the
//                   reference's sequential order (bit-identical scores), warp
//                   register top-k, CTA merge
//   k_score_pruned  the same scores with exact early termination: row heads,
//                   a Cauchy-Schwarz bound on the unread tail against the
//                   running k-th best, survivors finished as dense batches
//                   (chosen per index by the measured read fraction)
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include "fpp_device.cuh"
#include "fpp_internal.h"

namespace cg = cooperative_groups;

namespace fpp {

// ---------------------------------------------------------------- K1 query
// One lane group (G = P/EPT lanes) per (query, table, function): spinner
// projections in registers, then the ranked list.  Sorting uses 32-bit keys
// (22-bit truncated rank value | 10-bit index) -- half the shuffles and a third
// of the ALU work of 64-bit keys -- followed by an exact fix-up of the rare runs
// whose truncated values collide, so the emitted order is exactly
// (|p| desc, j asc).  When s > D the opposite-signed vectors follow in the same
// order with flipped codes.
template <bool NAT>
__device__ __forceinline__ bool rank_before(float pa, uint32_t ja, float pb, uint32_t jb) {
  const float a = fabsf(pa), b = fabsf(pb);
  if (a != b) return NAT ? a > b : a < b;
  return ja < jb;
}

// Sort the group's keys; neighbouring keys with equal quantised prefixes are
// put in the exact order by odd-even transposition passes in registers (values
// gathered from pv), falling back to a shared-memory insertion fix-up when a
// run is long (degenerate inputs).
template <int P, int EPT, bool NAT>
__device__ __forceinline__ void rank_sort_exact(uint32_t (&kk)[EPT], int g, uint32_t* sk,
                                                const float* pv) {
  constexpr int G = P / EPT;
  group_sort_u32_v2<P, EPT>(kk, g);
  auto same = [](uint32_t x, uint32_t y) {
    return x != 0xffffffffu && y != 0xffffffffu && (x >> 10) == (y >> 10);
  };
  auto before = [&](uint32_t y, uint32_t x) {  // exact: y strictly before x
    return rank_before<NAT>(pv[y & 1023u], y & 1023u, pv[x & 1023u], x & 1023u);
  };
  bool done = false;
#pragma unroll 1
  for (int round = 0; round < 4; ++round) {
    bool swapped = false;
#pragma unroll
    for (int e = 0; e + 1 < EPT; e += 2) {  // even pairs (in-lane)
      if (same(kk[e], kk[e + 1]) && before(kk[e + 1], kk[e])) {
        const uint32_t tmp = kk[e];
        kk[e] = kk[e + 1];
        kk[e + 1] = tmp;
        swapped = true;
      }
    }
#pragma unroll
    for (int e = 1; e + 1 < EPT; e += 2) {  // odd pairs (in-lane)
      if (same(kk[e], kk[e + 1]) && before(kk[e + 1], kk[e])) {
        const uint32_t tmp = kk[e];
        kk[e] = kk[e + 1];
        kk[e + 1] = tmp;
        swapped = true;
      }
    }
    if (G > 1) {  // odd pair across the lane boundary: (last of g, first of g+1)
      const uint32_t nxt = __shfl_down_sync(FULL, kk[0], 1);
      const uint32_t prv = __shfl_up_sync(FULL, kk[EPT - 1], 1);
      if (g + 1 < G && same(kk[EPT - 1], nxt) && before(nxt, kk[EPT - 1])) {
        kk[EPT - 1] = nxt;
        swapped = true;
      }
      if (g > 0 && same(prv, kk[0]) && before(kk[0], prv)) {
        kk[0] = prv;
        swapped = true;
      }
    }
    if (!__any_sync(FULL, swapped)) {
      done = true;
      break;
    }
  }
  if (done) return;
#pragma unroll
  for (int e = 0; e < EPT; ++e) sk[g * EPT + e] = kk[e];
  __syncwarp();
#pragma unroll 1
  for (int e = 0; e < EPT; ++e) {
    const int i = g * EPT + e;
    const uint32_t x = sk[i];
    if (x == 0xffffffffu || i + 1 >= P) continue;
    const uint32_t pf = x >> 10;
    if ((sk[i + 1] >> 10) != pf || sk[i + 1] == 0xffffffffu) continue;
    if (i > 0 && (sk[i - 1] >> 10) == pf) continue;  // not the run start
    int end = i + 1;
    while (end < P && sk[end] != 0xffffffffu && (sk[end] >> 10) == pf) ++end;
    for (int u = i + 1; u < end; ++u) {  // insertion sort by the exact order
      const uint32_t y = sk[u];
      const uint32_t jy = y & 1023u;
      const float py = pv[jy];
      int w = u - 1;
      while (w >= i && rank_before<NAT>(py, jy, pv[sk[w] & 1023u], sk[w] & 1023u)) {
        sk[w + 1] = sk[w];
        --w;
      }
      sk[w + 1] = y;
    }
  }
  __syncwarp();
#pragma unroll
  for (int e = 0; e < EPT; ++e) kk[e] = sk[g * EPT + e];
  __syncwarp();
}

// NS > 0: exact preselection.  Only the top nat = min(s, D) entries of the
// ranked order are emitted, so a threshold Tq on the quantised value (found by
// a few bisection steps on the group count) keeps c in [nat, NS] entries; they
// are compacted and only NS keys are sorted.  Quantisation is monotone, so
// every entry ranked before a kept one is kept too and the top nat of the kept
// set are the top nat overall.  A warp whose groups do
// not find such a threshold (heavy quantisation ties) sorts all P keys.
template <int P, int NS>
__global__ void __launch_bounds__(128)
k_query_lists(const float* __restrict__ Q, uint64_t nq, uint32_t d, uint32_t D, uint32_t K,
              const uint32_t* __restrict__ signs, uint32_t L, uint32_t s, uint64_t lstride,
              float* __restrict__ vals, uint32_t* __restrict__ codes) {
  using S = FhtShape<P>;
  constexpr int EPT = S::EPT;
  constexpr int GPB = 128 / S::G;
  constexpr bool TR = P >= 64;  // transpose FHT (cross-lane stages in registers)
  constexpr int TS = TR ? TransposeShape<P>::STRIDE : 4;
  constexpr int PVS = TS > P ? TS : P;  // the transpose buffer doubles as pv after the FHT
  __shared__ uint32_t sk_all[GPB][P];
  __shared__ __align__(16) float tb_all[GPB * PVS];
  const int lane = threadIdx.x & 31;
  const int g = lane % S::G;
  const int gl = threadIdx.x / S::G;
  uint32_t* sk = sk_all[gl];
  float* tbuf = tb_all + gl * PVS;
  float* pv = tbuf;
  // launch_query_lists keeps nq * L * K * G < 2^31: 32-bit index math
  const uint32_t gg = (blockIdx.x * blockDim.x + threadIdx.x) / S::G;
  const uint32_t total = (uint32_t)nq * L * K;
  const bool active = gg < total;
  const uint32_t gid = active ? gg : total - 1;
  const uint32_t f = gid % K;
  const uint32_t tl = gid / K;
  const uint32_t t = tl % L;
  const uint64_t q = tl / L;
  float v[EPT];
  load_row<P>(Q + q * d, d, g, v);
  if constexpr (TR) spinner_project_T<P>(v, signs + ((uint64_t)t * K + f) * 3 * S::W, g, tbuf);
  else spinner_project<P>(v, signs + ((uint64_t)t * K + f) * 3 * S::W, g);
  __syncwarp();  // transpose buffer is reused as pv below
  // 22-bit key = |p| quantised against the group maximum (monotone: fp32
  // multiply and floor are monotone), | 10-bit index; descending |p| -> ascending key
  float amax = 0.0f;
#pragma unroll
  for (int e = 0; e < EPT; ++e) amax = fmaxf(amax, fabsf(v[e]));
#pragma unroll
  for (int m = 1; m < S::G; m <<= 1) amax = fmaxf(amax, __shfl_xor_sync(FULL, amax, m));
  const float qs = amax > 0.0f ? 4194303.0f / amax : 0.0f;
  uint32_t kk[EPT];
  if constexpr (TR) store_B_natural<P>(v, g, pv);
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const uint32_t j = layout_index<P>(e, g);  // layout B / A
    if constexpr (!TR) pv[j] = v[e];
    // round(|p| * qs) via the 2^23 magic-number trick (FFMA + LOP on the FMA/ALU
    // pipes instead of F2I); monotone in |p| like the floor it replaces
    const uint32_t qv = min(__float_as_uint(fmaf(fabsf(v[e]), qs, 8388608.0f)) & 0x7fffffu, 4194303u);
    kk[e] = j < D ? (((4194303u - qv) << 10) | j) : 0xffffffffu;
  }
  __syncwarp();
  const uint64_t ob = q * lstride + (uint64_t)(t * K + f) * s;
  const uint32_t nat = s < D ? s : D;
  // the group's sorted keys go to sk (blocked layout r = g*E + e), then a rolled
  // loop writes ranks r = g, g+G, ... (coalesced stores, small code)
  auto emit_all = [&]() {
    __syncwarp();
    if (!active) return;
#pragma unroll 1
    for (uint32_t r = g; r < nat; r += S::G) {
      const uint32_t j = sk[r] & 1023u;
      const float p = pv[j];
      vals[ob + r] = fabsf(p);
      codes[ob + r] = p < 0.0f ? D + j : j;
    }
    // opposite-signed vectors: same order, value |p|, flipped code
#pragma unroll 1
    for (uint32_t r = g; r + D < s; r += S::G) {
      const uint32_t j = sk[r] & 1023u;
      const float p = pv[j];
      vals[ob + D + r] = fabsf(p);
      codes[ob + D + r] = p < 0.0f ? j : D + j;
    }
  };
  bool fast = false;
  if constexpr (NS > 0) {
    constexpr int E2 = NS / S::G;
    uint32_t lo = 0, hi = 4194302u, tq = 0;
    bool ok = false, fail = false;
#pragma unroll 1
    for (int it = 0; it < 24; ++it) {
      if (__all_sync(FULL, ok || fail)) break;
      const uint32_t mid = (lo + hi) >> 1;
      const uint32_t midk = (mid << 10) | 1023u;  // (k >> 10) <= mid  <=>  k <= midk
      uint32_t c = 0;
#pragma unroll
      for (int e = 0; e < EPT; ++e) c += kk[e] <= midk;  // sentinels: 0xffffffff > midk
#pragma unroll
      for (int m = 1; m < S::G; m <<= 1) c += __shfl_xor_sync(FULL, c, m);
      if (!ok && !fail) {
        if (c >= nat) {
          if (c <= (uint32_t)NS) { ok = true; tq = mid; }
          else if (lo >= mid) fail = true;
          else hi = mid;
        } else {
          lo = mid + 1;
          if (lo > hi) fail = true;
        }
      }
    }
    fast = __all_sync(FULL, ok);
    if (fast) {
      uint32_t cl = 0;
#pragma unroll
      for (int e = 0; e < EPT; ++e) cl += (kk[e] >> 10) <= tq;
      uint32_t x = cl;  // inclusive scan over the group's lanes
#pragma unroll
      for (int o = 1; o < S::G; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, x, o);
        if (g >= o) x += y;
      }
      const uint32_t ctot = __shfl_sync(FULL, x, (lane / S::G) * S::G + S::G - 1);
      uint32_t pos = x - cl;
#pragma unroll
      for (int e = 0; e < EPT; ++e)
        if ((kk[e] >> 10) <= tq) sk[pos++] = kk[e];
      for (uint32_t i = ctot + g; i < (uint32_t)NS; i += S::G) sk[i] = 0xffffffffu;
      __syncwarp();
      uint32_t k2[E2];
#pragma unroll
      for (int e = 0; e < E2; ++e) k2[e] = sk[g * E2 + e];
      __syncwarp();
      rank_sort_exact<NS, E2, true>(k2, g, sk, pv);
#pragma unroll
      for (int e = 0; e < E2; ++e) sk[g * E2 + e] = k2[e];
      emit_all();
    }
  }
  if (!fast) {
    rank_sort_exact<P, EPT, true>(kk, g, sk, pv);
#pragma unroll
    for (int e = 0; e < EPT; ++e) sk[g * EPT + e] = kk[e];
    emit_all();
  }
}

// ------------------------------------------------------------ probe select
// One warp per query, lanes over tables.  The probe set is {true bucket of
// each table} U the M = P_eff - L best remaining (t, r1, r2) under
// (fl(v1[r1]+v2[r2]) desc, r1, r2, t).  fp32 rounding is
// monotone, so the pairs of a table scoring >= T form a staircase; a walk over
// r1 with a binary-searched r2 boundary counts it.  T* (the M-th best score)
// is bracketed in ordered-key space and found by a safeguarded interpolation
// search on the count (exact: the loop keeps count(lo) >= M > count(hi) and
// stops at hi = lo + 1).  Ties at T* are resolved exactly in (r1, r2, t) order.
constexpr int PS_THREADS = 256;
constexpr int PS_TIE_CAP = 512;

struct ProbeArgs {
  const float* vals;      // [nq][L][K][s]
  const uint32_t* codes;  // [nq][L][K][s]
  uint32_t nq;
  uint32_t L, K, s, D;
  uint64_t NB;
  uint64_t peff;          // probes per query (incl. the L forced)
  const uint32_t* offs;   // [L][NB+1]
  const uint64_t* tbase;  // [L+1]
  uint64_t* ppos;         // [nq][peff]
  uint32_t* plen;         // [nq][peff]
  uint32_t* eq;           // [nq]
  uint64_t* dbg;          // optional [nq][peff] t*NB+b
  uint32_t* gbuf;         // [nq][peff] bucket-id scratch when not in shared memory
  uint64_t lstride;       // per-query list stride (L*K*s rounded up to 4 floats)
  long long* dbg_clk;     // optional [nq][16]: phase clocks + search iterations
  uint32_t* ckey;         // [nq][ccap] candidate pair keys (scratch)
  uint32_t* cpair;        // [nq][ccap] candidate pairs (t<<22 | r1<<11 | r2)
  uint32_t ccap;
  uint32_t beta_q8;       // first T_lo attempt at arm rank beta * m (beta = beta_q8 / 256)
  uint32_t rank_order;    // 1: keep the selection's emission order (no table-major sort)
  uint32_t* pout;         // != nullptr: write the probes as global bucket ids t * NB + b
                          // ([nq][peff], no directory reads) instead of (pos, len)
};

__device__ const float g_zero_row[1] = {0.0f};


__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Pair key, larger first:
//   falconnpp          ord(fl(a + b))                       (score sum desc)
//   falconn_baseline   ord(-(fl(ma - a) + fl(mb - b)))      (gap score asc)
// with a, b the two functions' |q.r| values and ma, mb their natural-list
// maxima.  Both are non-increasing in either rank, which is all the staircase
// machinery below relies on.
template <int MODE>
struct PairKey {
  float ma, mb;
  __device__ __forceinline__ uint32_t operator()(float a, float b) const {
    if (MODE == 1) return ord_key(-((ma - a) + (mb - b)));
    return ord_key(a + b);
  }
};

// (lists may live in shared or global memory: generic loads)
// number of r2 in [0, hi) with key(x, v2[r2]) >= T (a prefix: keys non-increasing)
template <class PK>
__device__ __forceinline__ uint32_t prefix_bs(const PK& pk, float x, const float* v2, uint32_t hi,
                                              uint32_t T) {
  uint32_t lo = 0;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (pk(x, v2[mid]) >= T) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// visit (r1, pa, pb) for rows [rb, re) while pb > 0 (prefixes at Ta > Tb)
template <class PK, class F>
__device__ __forceinline__ void walk2_rows(const PK& pk, const float* v1, const float* v2,
                                           uint32_t S2, uint32_t rb, uint32_t re, uint32_t Ta,
                                           uint32_t Tb, F&& visit) {
  if (rb >= re) return;
  const float x0 = v1[rb];
  uint32_t pb = prefix_bs(pk, x0, v2, S2, Tb);
  if (pb == 0) return;
  uint32_t pa = Ta == 0xffffffffu ? 0 : prefix_bs(pk, x0, v2, pb, Ta);
  visit(rb, pa, pb);
  for (uint32_t r1 = rb + 1; r1 < re; ++r1) {
    const float x = v1[r1];
    if (pk(x, v2[pb - 1]) < Tb) pb = prefix_bs(pk, x, v2, pb - 1, Tb);
    if (pb == 0) return;
    if (pa > pb) pa = pb;
    if (pa > 0 && pk(x, v2[pa - 1]) < Ta) pa = prefix_bs(pk, x, v2, pa - 1, Ta);
    visit(r1, pa, pb);
  }
}

__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v, uint64_t* sh) {
  v = warp_sum_u64(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  uint64_t t = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
  return t;
}

// A "grid" is one (table, list-part x list-part) block of pairs, sorted in
// both ranks: class 0 = natural x natural (one per table, its (0,0) is the
// forced true bucket), class 1 = natural x opposite and opposite x natural,
// class 2 = opposite x opposite.  Classes are taken in
// order; only the last needed class goes through selection.
struct GridRef {
  const float* va;
  const float* vb;
  uint32_t na, nb;   // extents
  uint32_t oa, ob;   // rank offsets (0 natural, D opposite)
  uint32_t t;
  bool forced;
  float ma, mb;      // natural-list maxima of the table's two functions (baseline gap)
};

// CTA per query (PS_THREADS threads, ~22 KB shared memory, so several query
// CTAs share an SM and hide each other's latency).  For the selection class:
//  1. T_lo: the grid corners bound the "arm" keys (row 0 and column 0 of every
//     grid, each a sorted run); one 4096-bin histogram pass over the arms gives
//     a bin edge with >= m arm keys above it, so T_lo <= T*;
//  2. one staircase walk materialises every pair >= T_lo (key + packed
//     (t, r1, r2)) into per-query global scratch;
//  3. radix-select T* over that flat array (balanced, coalesced passes); the
//     last digit's bin also yields the tie count and the ties to take;
//  4. ties at T* (rare) are resolved in (r1, r2, t) order;
//  5. the selected pairs are compacted (warp ballots, one pass), then every
//     probe's codes -> bucket -> CSR directory entry is resolved with 8 probes
//     per thread in flight.
// If the candidate set overflows the scratch, every pass re-walks instead.
// The emission order of the selection class is not canonical: the probe set
// (and so the candidate set and the top-k) is.
constexpr int PS_RBITS = 12;  // radix digit
template <int MODE>
__global__ void __launch_bounds__(PS_THREADS, 4) k_probe_select(ProbeArgs a) {
  __shared__ uint64_t red[PS_THREADS / 32];
  __shared__ uint64_t ties[PS_TIE_CAP];
  __shared__ uint32_t hist[1 << PS_RBITS];
  __shared__ uint32_t n_ties, n_cand, n_emit, sel_bin, sel_rem, sel_cnt;
  long long ck[8];
  ck[0] = clock64();
  const uint32_t q = blockIdx.x;
  const uint32_t L = a.L, K = a.K, s = a.s, D = a.D;
  const uint32_t n = s < D ? s : D, o = s > D ? s - D : 0;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const float* V = a.vals + (uint64_t)q * a.lstride;
  const uint32_t* Cq = a.codes + (uint64_t)q * a.lstride;
  uint32_t* ckey = a.ckey + (uint64_t)q * a.ccap;
  uint32_t* cpair = a.cpair + (uint64_t)q * a.ccap;
  if (threadIdx.x == 0) {
    n_ties = 0;
    n_cand = 0;
    n_emit = 0;
  }
  auto ngrids = [&](uint32_t cls) -> uint32_t { return (K == 2 && cls == 1) ? 2 * L : L; };
  auto grid = [&](uint32_t cls, uint32_t gi) -> GridRef {
    GridRef g;
    const uint32_t t = (K == 2 && cls == 1) ? gi >> 1 : gi;
    const float* v1 = V + (uint64_t)t * K * s;
    const float* v2 = K == 2 ? v1 + s : g_zero_row;
    const uint32_t n2 = K == 2 ? n : 1;
    g.t = t;
    g.forced = cls == 0;
    bool a_opp = false, b_opp = false;
    if (cls == 1) {
      if (K == 2) { a_opp = gi & 1; b_opp = !a_opp; }
      else a_opp = true;
    }
    if (cls == 2) a_opp = b_opp = true;
    g.va = v1 + (a_opp ? D : 0);
    g.na = a_opp ? o : n;
    g.oa = a_opp ? D : 0;
    g.vb = v2 + (b_opp ? D : 0);
    g.nb = b_opp ? o : n2;
    g.ob = b_opp ? D : 0;
    g.ma = v1[0];
    g.mb = v2[0];
    return g;
  };
  const uint64_t M = a.peff - L;  // non-forced probes
  // class sizes (non-forced pairs) and the class needing selection
  const uint64_t nn2 = K == 2 ? n : 1, oo2 = K == 2 ? o : 0;
  const uint64_t Ccls[3] = {(uint64_t)L * (n * nn2 - 1),
                            K == 2 ? 2ull * L * n * o : (uint64_t)L * o,
                            (uint64_t)L * o * oo2};
  uint32_t sel = 0;
  uint64_t m_sel = M;
  while (sel < 2 && m_sel > Ccls[sel]) { m_sel -= Ccls[sel]; ++sel; }
  // work partition of the selection class: (grid, row block)
  const uint32_t NG = ngrids(sel);
  const uint32_t TPT = NG < blockDim.x ? blockDim.x / NG : 1;
  const uint32_t units = NG * TPT;
  auto unit = [&](uint32_t u, GridRef& g, uint32_t& rb, uint32_t& re) {
    const uint32_t gi = u / TPT, part = u - gi * TPT;
    g = grid(sel, gi);
    const uint32_t RB = (g.na + TPT - 1) / TPT;
    rb = min(g.na, part * RB);
    re = min(g.na, rb + RB);
  };
  // the bin of hist[0, nb) holding the rem-th largest key (1-based, counting
  // from the top bin): sets sel_bin, sel_rem (rank inside the bin), sel_cnt
  auto pick_bin = [&](int nb, uint32_t rem) {
    constexpr int PER = (1 << PS_RBITS) / PS_THREADS;
    uint32_t hv[PER], hs = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int bin = nb - 1 - (int)(threadIdx.x * PER + j);
      hv[j] = bin >= 0 ? hist[bin] : 0;
      hs += hv[j];
    }
    uint32_t tot;
    uint32_t above = block_excl_scan_u32(hs, (uint32_t*)red, &tot);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int bin = nb - 1 - (int)(threadIdx.x * PER + j);
      if (bin >= 0 && above < rem && rem <= above + hv[j]) {
        sel_bin = (uint32_t)bin;
        sel_rem = rem - above;
        sel_cnt = hv[j];
      }
      above += hv[j];
    }
    __syncthreads();
  };
  // rank-th largest key (1-based) among enumerated keys in [base, base + 2^nbits);
  // *eqc = how many keys equal it, *eqr = its rank among them
  auto radix_select = [&](uint64_t rank, uint32_t base, int nbits, auto&& enumerate,
                          uint32_t* eqc, uint32_t* eqr) -> uint32_t {
    uint32_t prefix = 0, mask = 0, rem = (uint32_t)rank;
    int hb = nbits < 1 ? 1 : nbits;
    while (hb > 0) {
      const int w = hb < PS_RBITS ? hb : PS_RBITS, sh = hb - w, nb = 1 << w;
      for (int i = threadIdx.x; i < nb; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      enumerate([&](uint32_t key) {
        const uint32_t off = key - base;
        if ((off & mask) == prefix) smem_inc(&hist[(off >> sh) & (nb - 1)]);
      });
      __syncthreads();
      pick_bin(nb, rem);
      prefix |= sel_bin << sh;
      rem = sel_rem;
      *eqc = sel_cnt;
      mask |= (uint32_t)(nb - 1) << sh;
      hb = sh;
      __syncthreads();
    }
    *eqr = rem;
    return base + prefix;
  };
  auto bitlen = [](uint32_t x) { return x ? 32 - __clz(x) : 0; };
  auto pack = [](uint32_t t, uint32_t r1, uint32_t r2) { return (t << 22) | (r1 << 11) | r2; };
  uint32_t Tstar = 0, Tlo = 0, Tlo_safe = 0, refalls = 0;
  bool flat = false;
  uint32_t C = 0;
  auto enum_stair = [&](auto&& visit) {  // pairs >= Tlo of the selection class
    for (uint32_t u = threadIdx.x; u < units; u += blockDim.x) {
      GridRef g;
      uint32_t rb, re;
      unit(u, g, rb, re);
      const PairKey<MODE> pk{g.ma, g.mb};
      walk2_rows(pk, g.va, g.vb, g.nb, rb, re, 0xffffffffu, Tlo, [&](uint32_t r1, uint32_t, uint32_t pb) {
        const float x = g.va[r1];
        for (uint32_t r2 = (r1 == 0 && g.forced) ? 1 : 0; r2 < pb; ++r2)
          visit(pk(x, g.vb[r2]), pack(g.t, g.oa + r1, g.ob + r2));
      });
    }
  };
  constexpr int EU = 4;  // flat passes: loads of EU elements issued before use
  auto enum_keys = [&](auto&& visit) {
    if (flat) {
      for (uint32_t i0 = threadIdx.x; i0 < C; i0 += EU * blockDim.x) {
        uint32_t kk[EU];
#pragma unroll
        for (int u = 0; u < EU; ++u) {
          const uint32_t i = i0 + u * blockDim.x;
          kk[u] = i < C ? __ldcg(ckey + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < EU; ++u)
          if (i0 + u * blockDim.x < C) visit(kk[u]);
      }
    } else {
      enum_stair([&](uint32_t key, uint32_t) { visit(key); });
    }
  };
  auto enum_cand = [&](auto&& visit) {
    if (flat) {
      for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) visit(__ldcg(ckey + i), __ldcg(cpair + i));
    } else {
      enum_stair(visit);
    }
  };
  __syncthreads();
  uint32_t ties_total = 0, m = 0;  // keys == T*, and how many of them to take
  if (m_sel > 0) {
    // ---- 1. T_lo from the arms (all grids of a class have the same arm length)
    const GridRef g0 = grid(sel, 0);
    const uint32_t A = (g0.nb - (g0.forced ? 1 : 0)) + (g0.na - 1);
    uint32_t amax = 0, amin = 0xffffffffu;
    for (uint32_t gi = threadIdx.x; gi < NG; gi += blockDim.x) {  // runs are sorted: corners
      const GridRef g = grid(sel, gi);
      const PairKey<MODE> pk{g.ma, g.mb};
      const uint32_t r0 = g.forced ? 1 : 0;
      if (g.nb > r0) {
        amax = max(amax, pk(g.va[0], g.vb[r0]));
        amin = min(amin, pk(g.va[0], g.vb[g.nb - 1]));
      }
      if (g.na > 1) {
        amax = max(amax, pk(g.va[1], g.vb[0]));
        amin = min(amin, pk(g.va[g.na - 1], g.vb[0]));
      }
    }
    uint64_t pk = ((uint64_t)amax << 32) | (0xffffffffu - amin);
    for (int sft = 16; sft > 0; sft >>= 1) {
      const uint64_t y = ((uint64_t)__shfl_xor_sync(FULL, (uint32_t)(pk >> 32), sft) << 32) |
                         __shfl_xor_sync(FULL, (uint32_t)pk, sft);
      pk = (max(pk >> 32, y >> 32) << 32) | max(pk & 0xffffffffu, y & 0xffffffffu);
    }
    if (lane == 0) red[wp] = pk;
    __syncthreads();
    uint64_t mx = 0, nl = 0;
    for (int i = 0; i < nw; ++i) {
      mx = max(mx, red[i] >> 32);
      nl = max(nl, red[i] & 0xffffffffu);
    }
    amax = (uint32_t)mx;
    amin = 0xffffffffu - (uint32_t)nl;
    __syncthreads();
    if ((uint64_t)NG * A >= m_sel) {
      const int nbits = bitlen(amax - amin);
      const int sh = nbits > PS_RBITS ? nbits - PS_RBITS : 0, nb = 1 << (nbits - sh);
      for (int i = threadIdx.x; i < nb; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      // warp per grid: the row arm vb[r0, nb) and the column arm va[1, na), lanes
      // strided (coalesced), 8 loads per lane in flight
      constexpr int AU = 16;  // one pass per grid for arms of up to 512 entries (C2: 399)
      for (uint32_t gi = wp; gi < NG; gi += nw) {
        const GridRef g = grid(sel, gi);
        const PairKey<MODE> pk{g.ma, g.mb};
        const uint32_t nrow = g.nb - (g.forced ? 1 : 0);
        const float x0 = g.va[0], y0 = g.vb[0];
        for (uint32_t i0 = lane; i0 < A; i0 += 32 * AU) {
          float v[AU];
#pragma unroll
          for (int u = 0; u < AU; ++u) {
            const uint32_t i = i0 + 32 * u;
            v[u] = i < A ? (i < nrow ? g.vb[g.nb - nrow + i] : g.va[i - nrow + 1]) : 0.0f;
          }
#pragma unroll
          for (int u = 0; u < AU; ++u) {
            const uint32_t i = i0 + 32 * u;
            if (i < A) {
              const uint32_t key = i < nrow ? pk(x0, v[u]) : pk(v[u], y0);
              smem_inc(&hist[(key - amin) >> sh]);
            }
          }
        }
      }
      __syncthreads();
      pick_bin(nb, (uint32_t)m_sel);
      Tlo_safe = amin + (sel_bin << sh);
      Tlo = Tlo_safe;
      // optimistic first attempt: with >= 64 selected pairs per grid the arms
      // hold only about half of the pairs above T*, so a bin edge at arm rank
      // beta*m usually still leaves >= m pairs above it (checked after the walk;
      // the safe edge is the fallback).  Thinner staircases are mostly arm.
      const uint32_t m_try = (uint32_t)(((uint64_t)m_sel * a.beta_q8) >> 8);
      if (m_try >= 1 && m_try < m_sel && m_sel >= 64ull * NG) {
        pick_bin(nb, m_try);
        Tlo = amin + (sel_bin << sh);
      }
    }
    ck[1] = clock64();
    // ---- 2. materialise every selection-class pair >= Tlo.  Warp per grid.  The
    // pairs >= Tlo of row r1 are a prefix [0, pb(r1)) and pb is non-increasing
    // in r1.  Wide rows (pb > 32): lanes across r2, each row scanning only the
    // previous row's prefix; ballots give the coalesced writes and the next
    // bound.  Thin tail (pb <= 32): lanes across 32 rows, columns ascending
    // until every lane's prefix has ended.
    auto emit = [&](bool take, uint32_t key, uint32_t pr) {
      const uint32_t tb = __ballot_sync(FULL, take);
      if (tb) {
        uint32_t base = 0;
        if (lane == 0) base = smem_fetch_add(&n_cand, __popc(tb));
        base = __shfl_sync(FULL, base, 0);
        if (take && base + __popc(tb) <= a.ccap) {
          const uint32_t at = base + __popc(tb & ((1u << lane) - 1));
          ckey[at] = key;
          cpair[at] = pr;
        }
      }
    };
    auto materialise = [&]() {
      for (uint32_t gi = wp; gi < NG; gi += nw) {
        const GridRef g = grid(sel, gi);
        const PairKey<MODE> pk{g.ma, g.mb};
        if (gi + nw < NG) {  // the next grid's list heads into L1 while this one is walked
          const GridRef gn = grid(sel, gi + nw);
          const uint32_t la = (min(gn.na, 64u) + 31) / 32, lb = (gn.nb + 31) / 32;
          if ((uint32_t)lane < la)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(gn.va + lane * 32));
          else if ((uint32_t)lane < la + lb)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(gn.vb + (lane - la) * 32));
        }
        uint32_t pb = g.nb, r1 = 0;
        for (; r1 < g.na && pb > 32; ++r1) {
          const float x = g.va[r1];
          uint32_t npb = 0;
          for (uint32_t c0 = 0; c0 < pb; c0 += 32) {
            const uint32_t r2 = c0 + lane;
            const uint32_t key = r2 < pb ? pk(x, g.vb[r2]) : 0;
            const bool ge = r2 < pb && key >= Tlo;
            const uint32_t bal = __ballot_sync(FULL, ge);
            npb += __popc(bal);
            emit(ge && !(g.forced && r1 == 0 && r2 == 0), key, pack(g.t, g.oa + r1, g.ob + r2));
            if (bal != FULL) break;  // the prefix ended inside this chunk
          }
          pb = npb;
        }
        // thin tail: lane l takes row r1 + l and finds its prefix length by a binary
        // search below the previous bound (the staircase is non-increasing), then the
        // block's pairs are emitted as one flat range, 32 per round (lane f finds its
        // row by a 5-step search over the rows' exclusive offsets): coalesced stores,
        // one counter atomic per block
        for (; r1 < g.na && pb > 0; r1 += 32) {
          const uint32_t my = r1 + lane;
          const float x = my < g.na ? g.va[my] : 0.0f;
          const uint32_t cnt = my < g.na ? prefix_bs(pk, x, g.vb, pb, Tlo) : 0u;
          uint32_t incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
          }
          const uint32_t excl = incl - cnt, tot = __shfl_sync(FULL, incl, 31);
          // the forced pair (0, 0) is counted in the staircase but never emitted
          const uint32_t skip0 = (g.forced && r1 == 0 && __shfl_sync(FULL, cnt, 0) > 0) ? 1u : 0u;
          uint32_t base = 0;
          if (lane == 0 && tot > skip0) base = smem_fetch_add(&n_cand, tot - skip0);
          base = __shfl_sync(FULL, base, 0);
          for (uint32_t f0 = 0; f0 < tot; f0 += 32) {
            const uint32_t f = f0 + lane;
            uint32_t l = 0;
#pragma unroll
            for (int sft = 16; sft; sft >>= 1) {
              const uint32_t e = __shfl_sync(FULL, excl, l + sft);
              if (e <= f) l += sft;
            }
            const uint32_t c = f - __shfl_sync(FULL, excl, l);
            const float xr = __shfl_sync(FULL, x, l);
            if (f < tot && f >= skip0) {
              const uint32_t at = base + f - skip0;
              if (at < a.ccap) {
                ckey[at] = pk(xr, g.vb[c]);
                cpair[at] = pack(g.t, g.oa + r1 + l, g.ob + c);
              }
            }
          }
          pb = __shfl_sync(FULL, cnt, 31);  // the next block's rows lie below row r1 + 31
        }
      }
    };
    materialise();
    __syncthreads();
    C = n_cand;
    if (C < m_sel && Tlo != Tlo_safe) {  // the optimistic edge was too high: re-walk
      __syncthreads();
      if (threadIdx.x == 0) n_cand = 0;
      __syncthreads();
      Tlo = Tlo_safe;
      refalls = 1;
      materialise();
      __syncthreads();
      C = n_cand;
    }
    flat = C <= a.ccap;
    ck[2] = clock64();
    // ---- 3. T* (every arm pair is >= every other pair of its row / column, so
    // amax bounds all keys)
    Tstar = radix_select(m_sel, Tlo, bitlen(amax - Tlo), enum_keys, &ties_total, &m);
  } else {
    ck[1] = ck[2] = clock64();
  }
  ck[3] = clock64();
  // ---- 4. ties at T*: take the m smallest in (r1, r2, t) order
  auto comp = [&](uint32_t pr) {  // (r1, r2, t) order on global ranks
    const uint32_t t = pr >> 22, r1 = (pr >> 11) & 2047u, r2 = pr & 2047u;
    return ((uint64_t)r1 * 2048u + r2) * L + t;
  };
  uint64_t Kstar = ~0ull;
  if (m_sel > 0 && ties_total > m) {
    if (ties_total <= PS_TIE_CAP) {
      enum_cand([&](uint32_t key, uint32_t pr) {
        if (key == Tstar) ties[atomicAdd(&n_ties, 1u)] = comp(pr);
      });
      __syncthreads();
      uint64_t found = ~0ull;
      for (uint32_t i = threadIdx.x; i < ties_total; i += blockDim.x) {
        const uint64_t xk = ties[i];
        uint32_t rank = 0;
        for (uint32_t j = 0; j < ties_total; ++j) rank += ties[j] < xk;
        if (rank == m) found = xk;
      }
      for (int sft = 16; sft > 0; sft >>= 1) {
        const uint64_t y = ((uint64_t)__shfl_xor_sync(FULL, (uint32_t)(found >> 32), sft) << 32) |
                           __shfl_xor_sync(FULL, (uint32_t)found, sft);
        found = y < found ? y : found;
      }
      __syncthreads();
      if (lane == 0) red[wp] = found;
      __syncthreads();
      for (int i = 0; i < nw; ++i) Kstar = red[i] < Kstar ? red[i] : Kstar;
      __syncthreads();
    } else {
      auto count_lt = [&](uint64_t Kc) -> uint64_t {
        uint64_t c = 0;
        enum_cand([&](uint32_t key, uint32_t pr) { c += key == Tstar && comp(pr) < Kc; });
        return block_sum_u64(c, red);
      };
      uint64_t lo = 0, hi = (uint64_t)2048 * 2048 * L;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (count_lt(mid) >= m) hi = mid;
        else lo = mid + 1;
      }
      Kstar = lo;
    }
  }
  ck[4] = clock64();
  // ---- 5. emission of packed pairs: forced buckets, whole classes, selection
  auto selected = [&](uint32_t key, uint32_t pr) {
    return key > Tstar || (key == Tstar && (Kstar == ~0ull || comp(pr) < Kstar));
  };
  uint32_t* gb_out = a.gbuf + (uint64_t)q * a.peff;
  for (uint32_t t = threadIdx.x; t < L; t += blockDim.x) gb_out[t] = pack(t, 0, 0);
  uint64_t slot0 = L;
  // whole classes before the selection class: every pair, via per-thread counts + scan
  for (uint32_t cls = 0; cls < sel; ++cls) {
    const uint32_t ng = ngrids(cls);
    uint64_t mine = 0;
    for (uint32_t gi = threadIdx.x; gi < ng; gi += blockDim.x) {
      const GridRef g = grid(cls, gi);
      mine += (uint64_t)g.na * g.nb - (g.forced ? 1 : 0);
    }
    uint64_t x = mine;
    for (int sft = 1; sft < 32; sft <<= 1) {
      const uint64_t y = ((uint64_t)__shfl_up_sync(FULL, (uint32_t)(x >> 32), sft) << 32) |
                         __shfl_up_sync(FULL, (uint32_t)x, sft);
      if (lane >= sft) x += y;
    }
    __syncthreads();
    if (lane == 31) red[wp] = x;
    __syncthreads();
    uint64_t wb = 0;
    for (int i = 0; i < wp; ++i) wb += red[i];
    uint64_t slot = slot0 + wb + x - mine;
    for (uint32_t gi = threadIdx.x; gi < ng; gi += blockDim.x) {
      const GridRef g = grid(cls, gi);
      for (uint32_t r1 = 0; r1 < g.na; ++r1)
        for (uint32_t r2 = (r1 == 0 && g.forced) ? 1 : 0; r2 < g.nb; ++r2)
          gb_out[slot++] = pack(g.t, g.oa + r1, g.ob + r2);
    }
    slot0 += Ccls[cls];
    __syncthreads();
  }
  if (m_sel > 0) {
    uint32_t* out = gb_out + slot0;
    if (flat) {
      // warp-aggregated compaction; the warp-uniform bound keeps ballots full
      const uint32_t Cr = (C + 31) & ~31u;
      for (uint32_t i0 = threadIdx.x; i0 < Cr; i0 += EU * blockDim.x) {
        uint32_t kk[EU], pp[EU];
#pragma unroll
        for (int u = 0; u < EU; ++u) {
          const uint32_t i = i0 + u * blockDim.x;
          kk[u] = i < C ? __ldcg(ckey + i) : 0;
          pp[u] = i < C ? __ldcg(cpair + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < EU; ++u) {
          const uint32_t i = i0 + u * blockDim.x;
          if (i0 + u * blockDim.x - lane < Cr) {  // warp-uniform
            const bool take = i < C && selected(kk[u], pp[u]);
            const uint32_t bal = __ballot_sync(FULL, take);
            uint32_t base = 0;
            if (lane == 0 && bal) base = smem_fetch_add(&n_emit, __popc(bal));
            base = __shfl_sync(FULL, base, 0);
            if (take) out[base + __popc(bal & ((1u << lane) - 1))] = pp[u];
          }
        }
      }
    } else {
      enum_stair([&](uint32_t key, uint32_t pr) {
        if (selected(key, pr)) out[atomicAdd(&n_emit, 1u)] = pr;
      });
    }
  }
  __syncthreads();
  ck[5] = clock64();
  // ---- 6. resolve probes: pair -> codes -> bucket -> CSR directory entry,
  // 8 probes per thread in flight
  uint64_t* ppos = a.ppos + (uint64_t)q * a.peff;
  uint32_t* plen = a.plen + (uint64_t)q * a.peff;
  uint64_t* dbg = a.dbg ? a.dbg + (uint64_t)q * a.peff : nullptr;
  uint64_t esum = 0;
  const uint32_t P = (uint32_t)a.peff;
  const uint32_t twoD = 2 * D;
  const uint32_t NB = (uint32_t)a.NB;
  // Table-major probe order (FPP_PROBE_TABLEMAJOR=1; off by default: measured no gain):
  // the non-forced probes [L, P) are counting-sorted by table (order within a table:
  // arbitrary), so the walking score kernel
  // (k_score_screen<WALK>) sweeps the tables in order and similar queries scored side
  // by side read the same buckets' rows at about the same time (L2 reuse).  The L
  // forced true buckets stay in front (the kernel's seeds).  The probe set, hence
  // every result, is unchanged.
  uint32_t* tcur = hist;  // [L] table cursors (the selection histogram is free now)
  const bool tmajor = !a.rank_order && P > L;
  if (tmajor) {
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) tcur[i] = 0;
    __syncthreads();
    for (uint32_t pp = L + threadIdx.x; pp < P; pp += blockDim.x)
      atomicAdd(&tcur[__ldcg(gb_out + pp) >> 22], 1u);
    __syncthreads();
    const uint32_t per = (L + blockDim.x - 1) / blockDim.x;
    const uint32_t i0 = min(L, threadIdx.x * per), i1 = min(L, i0 + per);
    uint32_t loc = 0;
    for (uint32_t i = i0; i < i1; ++i) loc += tcur[i];
    uint32_t tot;
    uint32_t base = L + block_excl_scan_u32(loc, (uint32_t*)red, &tot);
    for (uint32_t i = i0; i < i1; ++i) {
      const uint32_t c = tcur[i];
      tcur[i] = base;
      base += c;
    }
    __syncthreads();
  }
  constexpr int UR = 8;
  for (uint32_t p0 = threadIdx.x; p0 < P; p0 += UR * blockDim.x) {
    uint32_t pr[UR], c1[UR], c2[UR], o0[UR], o1[UR];
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const uint32_t pp = p0 + u * blockDim.x;
      pr[u] = pp < P ? __ldcg(gb_out + pp) : 0;
    }
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const uint32_t t = pr[u] >> 22;
      const uint32_t* cq = Cq + (uint64_t)t * K * s;
      c1[u] = __ldg(cq + ((pr[u] >> 11) & 2047u));
      c2[u] = K == 2 ? __ldg(cq + s + (pr[u] & 2047u)) : 0;
    }
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const uint32_t t = pr[u] >> 22;
      c1[u] = K == 2 ? c1[u] * twoD + c2[u] : c1[u];  // bucket within table t
      if (!a.pout) {
        const uint32_t* of = a.offs + (uint64_t)t * (NB + 1) + c1[u];
        o0[u] = __ldg(of);
        o1[u] = __ldg(of + 1);
      }
    }
    if (a.pout) {  // probe sets only (multi-GPU split: resolved by each shard)
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const uint32_t pp = p0 + u * blockDim.x;
        if (pp < P) {
          const uint32_t t = pr[u] >> 22;
          const uint32_t dst = (tmajor && pp >= L) ? atomicAdd(&tcur[t], 1u) : pp;
          a.pout[(uint64_t)q * a.peff + dst] = t * NB + c1[u];
        }
      }
      continue;
    }
#pragma unroll
    for (int u = 0; u < UR; ++u) {
      const uint32_t pp = p0 + u * blockDim.x;
      if (pp < P) {
        const uint32_t t = pr[u] >> 22;
        const uint32_t dst = (tmajor && pp >= L) ? atomicAdd(&tcur[t], 1u) : pp;
        ppos[dst] = __ldg(a.tbase + t) + o0[u];
        plen[dst] = o1[u] - o0[u];
        esum += o1[u] - o0[u];
        if (dbg) dbg[dst] = (uint64_t)t * a.NB + c1[u];
      }
    }
  }
  esum = block_sum_u64(esum, red);
  if (threadIdx.x == 0) {
    a.eq[q] = (uint32_t)esum;
    if (a.dbg_clk) {
      ck[6] = clock64();
      long long* d = a.dbg_clk + (uint64_t)q * 16;
      for (int i = 0; i < 7; ++i) d[i] = ck[i];
      d[8] = flat;
      d[9] = C;
      d[10] = ties_total;
      d[11] = refalls;
    }
  }
}

// Probe sets given as global bucket ids (fpp_query_from_probes: computed by any index
// with the same parameters and seed, e.g. another shard's) -> this index's CSR
// (pos, len) and the entries per query; CTA per query.
__global__ void __launch_bounds__(256) k_resolve_probes(const uint32_t* __restrict__ probes, uint64_t peff,
                                                        uint64_t NB, const uint32_t* __restrict__ offs,
                                                        const uint64_t* __restrict__ tbase,
                                                        uint64_t* __restrict__ ppos,
                                                        uint32_t* __restrict__ plen,
                                                        uint32_t* __restrict__ eq) {
  __shared__ uint64_t red[8];
  const uint32_t q = blockIdx.x;
  const uint32_t* pb = probes + (uint64_t)q * peff;
  uint64_t esum = 0;
  for (uint64_t p = threadIdx.x; p < peff; p += blockDim.x) {
    const uint32_t gb = __ldg(pb + p);
    const uint32_t t = (uint32_t)(gb / NB), b = (uint32_t)(gb - (uint64_t)t * NB);
    const uint32_t* of = offs + (uint64_t)t * (NB + 1) + b;
    const uint32_t o0 = __ldg(of), o1 = __ldg(of + 1);
    ppos[(uint64_t)q * peff + p] = __ldg(tbase + t) + o0;
    plen[(uint64_t)q * peff + p] = o1 - o0;
    esum += o1 - o0;
  }
  esum = block_sum_u64(esum, red);
  if (threadIdx.x == 0) eq[q] = (uint32_t)esum;
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
constexpr int CO_THREADS = 1024;
#ifndef FPP_CO_CL_THREADS
#define FPP_CO_CL_THREADS 1024
#endif
constexpr int CO_CL_THREADS = FPP_CO_CL_THREADS;  // k_collect_cluster CTA size

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
  uint32_t grouped;      // 1: two-level dedup by id-range groups (large shards, stage_b)
  uint32_t gshift;       // grouped: id >> gshift < CO_NG; per-warp range bitmap 2^gshift bits
  uint32_t* uniq;        // unique candidates per query (uq = list length incl. grouped holes)
  uint64_t n;            // points (grouped: groups in use = ((n - 1) >> gshift) + 1)
  uint32_t sliced;       // 1: sliced bitmap dedup (gshift = slice bits), see collect_sliced
};

// Warp-cooperative walk over one query's probes.  A warp takes 32 probes at a
// time (lane i: probe i's (pos, len), coalesced), scans the lengths in
// registers, and then covers the chunk's entries 32 at a time: lane l takes
// entry e = e0 + l and finds its probe by a 5-step shuffle binary search over
// the exclusive offsets, so consecutive lanes read consecutive ids of a bucket.
// CO_UNROLL rounds issue their id loads before any is consumed.  `tas(id)`
// tests-and-sets the visited bit and returns whether the id is new; new ids are
// appended to `out` with one counter atomic per warp round.
#ifndef FPP_CO_UNROLL
#define FPP_CO_UNROLL 8
#endif
constexpr int CO_UNROLL = FPP_CO_UNROLL;
template <class NextChunk, class TAS>
__device__ __forceinline__ void collect_walk(const uint64_t* pp, const uint32_t* pl, uint32_t P,
                                             const uint32_t* __restrict__ ids, uint32_t* out,
                                             uint32_t* ucount, NextChunk&& next_chunk, TAS&& tas) {
  const int lane = threadIdx.x & 31;
  // the next chunk's (pos, len) are loaded while the current chunk's ids are walked
  uint32_t c = next_chunk();
  uint32_t nlen = 0;
  uint64_t npos = 0;
  if (c * 32 + lane < P) {
    nlen = pl[c * 32 + lane];
    npos = pp[c * 32 + lane];
  }
  while (c * 32 < P) {
    const uint32_t len = nlen;
    const uint64_t pos = npos;
    c = next_chunk();
    nlen = 0;
    npos = 0;
    if (c * 32 + lane < P) {
      nlen = pl[c * 32 + lane];
      npos = pp[c * 32 + lane];
    }
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t T = __shfl_sync(FULL, incl, 31);
    const uint32_t excl = incl - len;
    // the chunk's non-empty probes, compacted: lane r holds the r-th one's first
    // entry (cex) and bucket position
    const uint32_t ne = __ballot_sync(FULL, len > 0);
    const bool cval = (uint32_t)lane < (uint32_t)__popc(ne);
    const uint32_t src = cval ? __fns(ne, 0, lane + 1) : 0u;
    const uint32_t cex = __shfl_sync(FULL, excl, src);
    const uint32_t cplo = __shfl_sync(FULL, (uint32_t)pos, src);
    const uint32_t cphi = __shfl_sync(FULL, (uint32_t)(pos >> 32), src);
    for (uint32_t e0 = 0; e0 < T; e0 += 32 * CO_UNROLL) {
      uint32_t idv[CO_UNROLL];
#pragma unroll
      for (int u = 0; u < CO_UNROLL; ++u) {
        // entries E0 .. E0+31: the probe holding E0 (r0) plus the probes starting inside
        // the window (a 32-bit mask, one warp reduction) place every lane's entry
        const uint32_t E0 = e0 + 32 * u, e = E0 + lane;
        const uint32_t r0 = __popc(__ballot_sync(FULL, cval && cex <= E0)) - 1u;
        const uint32_t dd = cex - E0;
        const uint32_t sm = __reduce_or_sync(FULL, (cval && cex > E0 && dd < 32u) ? (1u << dd) : 0u);
        const uint32_t r = r0 + __popc(sm & ((2u << lane) - 1u));
        const uint32_t plo = __shfl_sync(FULL, cplo, r);
        const uint32_t phi = __shfl_sync(FULL, cphi, r);
        const uint32_t ex = __shfl_sync(FULL, cex, r);
        idv[u] = e < T ? __ldg(ids + ((((uint64_t)phi << 32) | plo) + (e - ex))) : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < CO_UNROLL; ++u) {
        const bool isnew = idv[u] != 0xffffffffu && tas(idv[u]);
        const uint32_t bal = __ballot_sync(FULL, isnew);
        if (bal) {
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(ucount, __popc(bal));
          base = __shfl_sync(FULL, base, 0);
          if (isnew) out[base + __popc(bal & ((1u << lane) - 1))] = idv[u];
        }
      }
    }
  }
}

// Grouped dedup (large shards: the n-bit visited set is off-chip).  Two walks
// form a counting sort of the walked ids into CO_NG id-range groups (2^gshift
// ids each) in the query's candidate segment (groups ascending, so similar
// queries still gather the same id ranges at about the same time); then each
// warp takes groups and tests-and-sets the group's ids in a 2^gshift-bit range
// bitmap in shared memory: a repeat is overwritten in place with 0xFFFFFFFF (a
// hole the score kernels skip), and the touched words are cleared again.  Every
// id is therefore scored once at a cost proportional to the walked
// entries.  uq[q] = the list length (holes included), uniq[q] = unique ids.
constexpr uint32_t CO_NG = 1024;
__device__ __forceinline__ void collect_grouped(const CollectArgs& a, uint32_t q, uint32_t* out,
                                                uint32_t* ucount, uint32_t* nextc, uint32_t* sm,
                                                uint32_t* scan_sh, uint32_t* U_out) {
  uint32_t* cnt = sm;             // [CO_NG] group counts -> scatter cursors (= group ends)
  uint32_t* wbm = sm + CO_NG;     // [32 warps][2^gshift / 32] range bitmaps (kept clear)
  __shared__ uint32_t dups_sh;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t P = (uint32_t)a.peff, gs = a.gshift;
  const uint32_t bw = 1u << (gs - 5);  // bitmap words per warp
  const uint64_t* pp = a.ppos + (uint64_t)q * a.peff;
  const uint32_t* pl = a.plen + (uint64_t)q * a.peff;
  auto next_chunk = [&]() {
    uint32_t c = 0;
    if (lane == 0) c = smem_fetch_add(nextc, 1u);
    return __shfl_sync(FULL, c, 0);
  };
  for (uint32_t i = threadIdx.x; i < CO_NG; i += blockDim.x) cnt[i] = 0;
  if (threadIdx.x == 0) dups_sh = 0;
  __syncthreads();
  const uint32_t cnt_base = (uint32_t)__cvta_generic_to_shared(cnt);
  collect_walk(pp, pl, P, a.ids, out, ucount, next_chunk, [&](uint32_t id) {
    asm volatile("red.shared.add.u32 [%0], 1;\n" ::"r"(cnt_base + ((id >> gs) << 2)) : "memory");
    return false;
  });
  __syncthreads();
  uint32_t E;
  {  // exclusive scan of the group counts -> scatter cursors
    static_assert(CO_NG == CO_THREADS, "one group count per thread");
    const uint32_t v = cnt[threadIdx.x];
    cnt[threadIdx.x] = block_excl_scan_u32(v, scan_sh, &E);
    if (threadIdx.x == 0) *nextc = 0;
  }
  __syncthreads();
  // walk 2 (a second probe decode measured faster than re-streaming a walk-order
  // copy: 93 vs 102 ms per C4 step): scatter into the groups
  collect_walk(pp, pl, P, a.ids, out, ucount, next_chunk, [&](uint32_t id) {
    uint32_t pos;
    asm volatile("atom.shared.add.u32 %0, [%1], 1;\n" : "=r"(pos) : "r"(cnt_base + ((id >> gs) << 2)) : "memory");
    out[pos] = id;
    return false;
  });
  __syncthreads();  // cnt[g] is now the end of group g (= the start of group g + 1)
  uint32_t* bm = wbm + (size_t)w * bw;
  const uint32_t mask = (1u << gs) - 1u;
  const uint32_t gstep = blockDim.x >> 5;
  const uint32_t ng = (uint32_t)((a.n - 1) >> gs) + 1;  // groups in use
  uint32_t dups = 0;
  const uint32_t bm_base = (uint32_t)__cvta_generic_to_shared(bm);
  auto tas = [&](uint32_t id) {  // test-and-set in the range bitmap: true = a repeat
    const uint32_t b = id & mask, bit = 1u << (b & 31);
    uint32_t old;
    asm volatile("atom.shared.or.b32 %0, [%1], %2;\n"
                 : "=r"(old)
                 : "r"(bm_base + ((b >> 5) << 2)), "r"(bit)
                 : "memory");
    return (old & bit) != 0u;
  };
  // groups g = w, w + 32, ... (~100-200 ids each): the first 256 entries of a group are
  // held in registers (8 per lane: one load round trip), tested-and-set, repeats
  // overwritten with holes, and the touched bitmap words cleared from the registers
  for (uint32_t g = w; g < ng; g += gstep) {
    const uint32_t S = g ? cnt[g - 1] : 0u, Eg = cnt[g];
    if (Eg - S <= 1) continue;  // (empty groups and single ids hold no repeats)
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t i = S + u * 32 + lane;
      v[u] = i < Eg ? out[i] : 0xffffffffu;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (v[u] != 0xffffffffu && tas(v[u])) {  // a repeat: the first occurrence stays
        out[S + u * 32 + lane] = 0xffffffffu;
        v[u] = 0xffffffffu;
        ++dups;
      }
    for (uint32_t i = S + 256 + lane; i < Eg; i += 32)
      if (tas(out[i])) {
        out[i] = 0xffffffffu;
        ++dups;
      }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 8; ++u)  // clear the touched words again
      if (v[u] != 0xffffffffu) bm[(v[u] & mask) >> 5] = 0;
    for (uint32_t i = S + 256 + lane; i < Eg; i += 32) {
      const uint32_t id = out[i];
      if (id != 0xffffffffu) bm[(id & mask) >> 5] = 0;
    }
    __syncwarp();
  }
  dups = __reduce_add_sync(FULL, dups);
  if (lane == 0 && dups) atomicAdd(&dups_sh, dups);
  __syncthreads();
  *U_out = E - dups_sh;
}

// Sliced dedup (large shards: the n-bit visited set is off-chip).  A counting sort
// of the walked ids into id slices of 2^gshift ids (two walks: counts, then the
// scatter into the query's candidate segment -- few slices, so the scatter streams
// are nearly sequential), then slice by slice: the slice's ids are ORed into a
// 2^gshift-bit bitmap in shared memory, and the bitmap is scanned (each thread a
// contiguous word range, a block scan for the positions) to emit the slice's unique
// ids in ascending order, clearing the words as it goes.  The output trails the
// input (slices 0..s hold at most as many unique ids as entries, so slice s's output
// ends at or before slice s + 1's input starts): it is written in place.  Result: the query's unique candidates in ascending
// id order, like the one-slice shared-memory path.
constexpr uint32_t CO_SLICE_BITS = 19;  // 64 KB slice bitmaps (two CTAs per SM)
__device__ __forceinline__ void collect_sliced(const CollectArgs& a, uint32_t q, uint32_t* out,
                                               uint32_t* ucount, uint32_t* nextc, uint32_t* sm,
                                               uint32_t* scan_sh, uint32_t* U_out) {
  uint32_t* cnt = sm;          // [CO_NG] slice counts -> scatter cursors (= slice ends)
  uint32_t* bmp = sm + CO_NG;  // [2^gshift / 32] slice bitmap (kept clear)
  const int lane = threadIdx.x & 31;
  const uint32_t P = (uint32_t)a.peff, sb = a.gshift;
  const uint32_t ns = (uint32_t)((a.n - 1) >> sb) + 1;
  const uint32_t bw = 1u << (sb - 5);
  const uint64_t* pp = a.ppos + (uint64_t)q * a.peff;
  const uint32_t* pl = a.plen + (uint64_t)q * a.peff;
  auto next_chunk = [&]() {
    uint32_t c = 0;
    if (lane == 0) c = smem_fetch_add(nextc, 1u);
    return __shfl_sync(FULL, c, 0);
  };
  for (uint32_t i = threadIdx.x; i < CO_NG; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  const uint32_t cnt_base = (uint32_t)__cvta_generic_to_shared(cnt);
  const uint32_t bmp_base = (uint32_t)__cvta_generic_to_shared(bmp);
  collect_walk(pp, pl, P, a.ids, out, ucount, next_chunk, [&](uint32_t id) {
    asm volatile("red.shared.add.u32 [%0], 1;\n" ::"r"(cnt_base + ((id >> sb) << 2)) : "memory");
    return false;
  });
  __syncthreads();
  {
    static_assert(CO_NG == CO_THREADS, "one slice count per thread");
    uint32_t E;
    const uint32_t v = cnt[threadIdx.x];
    cnt[threadIdx.x] = block_excl_scan_u32(v, scan_sh, &E);
    if (threadIdx.x == 0) *nextc = 0;
  }
  __syncthreads();
  collect_walk(pp, pl, P, a.ids, out, ucount, next_chunk, [&](uint32_t id) {
    uint32_t pos;
    asm volatile("atom.shared.add.u32 %0, [%1], 1;\n" : "=r"(pos) : "r"(cnt_base + ((id >> sb) << 2)) : "memory");
    out[pos] = id;
    return false;
  });
  __syncthreads();  // cnt[s] is now the end of slice s
  const uint32_t mask = (1u << sb) - 1u;
  const uint32_t per = bw / blockDim.x;  // bitmap words per thread (>= 4, multiple of 4)
  uint32_t wpos = 0;
  for (uint32_t s = 0; s < ns; ++s) {
    const uint32_t S = s ? cnt[s - 1] : 0u, Es = cnt[s];
    if (Es == S) continue;
    for (uint32_t i = S + threadIdx.x; i < Es; i += blockDim.x) {
      const uint32_t b = out[i] & mask;
      asm volatile("red.shared.or.b32 [%0], %1;\n" ::"r"(bmp_base + ((b >> 5) << 2)), "r"(1u << (b & 31))
                   : "memory");
    }
    __syncthreads();
    uint4* w4 = reinterpret_cast<uint4*>(bmp + threadIdx.x * per);
    uint32_t c = 0;
    for (uint32_t j = 0; j < per / 4; ++j) {
      const uint4 x = w4[j];
      c += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
    }
    uint32_t tot;
    uint32_t pos = wpos + block_excl_scan_u32(c, scan_sh, &tot);
    const uint32_t id0 = (s << sb) + threadIdx.x * per * 32;
    for (uint32_t j = 0; j < per / 4; ++j) {
      const uint4 x = w4[j];
      const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        for (uint32_t word = wv[e]; word; word &= word - 1)
          out[pos++] = id0 + (j * 4 + e) * 32 + (__ffs(word) - 1);
      if (x.x | x.y | x.z | x.w) w4[j] = make_uint4(0, 0, 0, 0);
    }
    wpos += tot;
    __syncthreads();  // the bitmap is clear and scan_sh free for the next slice
  }
  *U_out = wpos;
}

// CTA per query (persistent CTAs fetch queries dynamically); the visited
// bitmap lives in shared memory (n bits), or the grouped dedup runs (large
// shards), or -- beyond the grouped range -- a per-CTA global-memory bitmap that
// is cleared again through the candidate list.
__global__ void __launch_bounds__(CO_THREADS, 2) k_collect(CollectArgs a) {
  extern __shared__ __align__(16) uint32_t sbm[];
  __shared__ uint32_t ucount, qsh, nextc;
  __shared__ uint32_t scan_sh[32];
  uint32_t* bm = a.gbitmap ? a.gbitmap + (uint64_t)blockIdx.x * a.nwords : sbm;
  if (a.grouped)  // the per-warp range bitmaps start clear and are kept clear
    for (uint32_t i = threadIdx.x; i < (blockDim.x >> 5) << (a.gshift - 5); i += blockDim.x)
      sbm[CO_NG + i] = 0;
  if (a.sliced)  // the slice bitmap starts clear and is kept clear
    for (uint32_t i = threadIdx.x; i < (1u << (a.gshift - 5)); i += blockDim.x) sbm[CO_NG + i] = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      qsh = atomicAdd(a.counter, 1u);
      ucount = 0;
      nextc = 0;
    }
    if (!a.gbitmap && !a.grouped && !a.sliced) {
      const uint32_t n4 = a.nwords >> 2;
      uint4* b4 = reinterpret_cast<uint4*>(sbm);
      for (uint32_t w = threadIdx.x; w < n4; w += blockDim.x) b4[w] = make_uint4(0, 0, 0, 0);
      for (uint32_t w = n4 * 4 + threadIdx.x; w < a.nwords; w += blockDim.x) sbm[w] = 0;
    }
    __syncthreads();
    const uint32_t q = qsh;
    if (q >= a.nq) break;
    uint32_t* out = a.cands + a.coff[q];
    const uint32_t P = (uint32_t)a.peff;
    auto next_chunk = [&]() {
      uint32_t c = 0;
      if ((threadIdx.x & 31) == 0) c = smem_fetch_add(&nextc, 1u);
      return __shfl_sync(FULL, c, 0);
    };
    uint32_t U;
    if (a.sliced) {
      collect_sliced(a, q, out, &ucount, &nextc, sbm, scan_sh, &U);
    } else if (a.grouped) {
      uint32_t Uu;
      collect_grouped(a, q, out, &ucount, &nextc, sbm, scan_sh, &Uu);
      if (threadIdx.x == 0) a.uniq[q] = Uu;
      U = (uint32_t)(a.coff[q + 1] - a.coff[q]);  // list length, holes included
    } else if (!a.gbitmap) {
      // shared-memory bitmap: fire-and-forget ORs during the walk, then the set
      // bits are emitted in ascending id order (a bitmap scan), so every query's
      // candidate rows are gathered in address order and similar queries scored
      // side by side touch shared rows at about the same time
      collect_walk(a.ppos + (uint64_t)q * a.peff, a.plen + (uint64_t)q * a.peff, P, a.ids, out,
                   &ucount, next_chunk, [&](uint32_t id) {
                     asm volatile("red.shared.or.b32 [%0], %1;\n" ::"r"(
                                      (uint32_t)__cvta_generic_to_shared(bm + (id >> 5))),
                                  "r"(1u << (id & 31))
                                  : "memory");
                     return false;
                   });
      __syncthreads();
      const uint32_t per = (a.nwords + blockDim.x - 1) / blockDim.x;
      const uint32_t w0 = min(a.nwords, threadIdx.x * per), w1 = min(a.nwords, w0 + per);
      uint32_t cnt = 0;
      for (uint32_t w = w0; w < w1; ++w) cnt += __popc(sbm[w]);
      uint32_t pos = block_excl_scan_u32(cnt, scan_sh, &U);
      for (uint32_t w = w0; w < w1; ++w)
        for (uint32_t word = sbm[w]; word; word &= word - 1) out[pos++] = w * 32 + (__ffs(word) - 1);
    } else {
      collect_walk(a.ppos + (uint64_t)q * a.peff, a.plen + (uint64_t)q * a.peff, P, a.ids, out,
                   &ucount, next_chunk, [&](uint32_t id) {
                     const uint32_t bit = 1u << (id & 31);
                     return !(atomicOr(bm + (id >> 5), bit) & bit);
                   });
      __syncthreads();
      U = ucount;
    }
    if (threadIdx.x == 0) {
      a.uq[q] = U;
      if (a.uniq && !a.grouped) a.uniq[q] = U;
    }
    if (a.sliced) __syncthreads();  // (the slice counters are reused by the next query)
    if (a.gbitmap)
      for (uint32_t c = threadIdx.x; c < U; c += blockDim.x) bm[out[c] >> 5] = 0;
    __syncthreads();
  }
}

// Large shards (n bits > one SM's shared memory): one thread-block cluster of
// CO_CLUSTER CTAs per query, the visited bitmap split into per-CTA slices of
// shared memory and tested-and-set through DSMEM atomics on the owning CTA
// (cluster.map_shared_rank); the per-query candidate counter lives in CTA 0,
// and the probe chunks are dealt round-robin over the cluster's CTAs.
constexpr int CO_CLUSTER = 8;

__global__ void __cluster_dims__(CO_CLUSTER, 1, 1) __launch_bounds__(CO_CL_THREADS, 1)
k_collect_cluster(CollectArgs a, uint32_t slice_words) {
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t rank = cluster.block_rank();
  const uint32_t cid = blockIdx.x / CO_CLUSTER, ncl = gridDim.x / CO_CLUSTER;
  extern __shared__ __align__(16) uint32_t sbm[];
  __shared__ uint32_t ucount, nextc, cta_cnt;
  __shared__ uint32_t scan_sh[32];
  const uint32_t slice_bits = slice_words * 32;
  const uint32_t inv_slice = (uint32_t)(0x100000000ull / slice_bits);
  const uint32_t sbm_base = (uint32_t)__cvta_generic_to_shared(sbm);
  for (uint32_t q = cid; q < a.nq; q += ncl) {
    for (uint32_t w = threadIdx.x; w < slice_words; w += blockDim.x) sbm[w] = 0;
    if (threadIdx.x == 0) {
      ucount = 0;
      nextc = 0;
    }
    cluster.sync();
    uint32_t* out = a.cands + a.coff[q];
    const uint32_t P = (uint32_t)a.peff;
    // DSMEM ORs on the owning CTA's slice (results unused: no append during the walk)
    collect_walk(a.ppos + (uint64_t)q * a.peff, a.plen + (uint64_t)q * a.peff, P, a.ids, out,
                 &ucount,
                 [&]() {
                   uint32_t c = 0;
                   if ((threadIdx.x & 31) == 0) c = smem_fetch_add(&nextc, 1u);
                   return __shfl_sync(FULL, c, 0) * CO_CLUSTER + rank;
                 },
                 [&](uint32_t id) {
                   // owner = id / slice_bits by a reciprocal multiply (+ one-step fix-up)
                   uint32_t owner = __umulhi(id, inv_slice);
                   if ((owner + 1) * slice_bits <= id) ++owner;
                   if (owner * slice_bits > id) --owner;
                   const uint32_t lb = id - owner * slice_bits;
                   uint32_t ra;  // fire-and-forget OR into the owning CTA's slice (DSMEM)
                   asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n"
                                : "=r"(ra)
                                : "r"(sbm_base + (lb >> 5) * 4), "r"(owner));
                   asm volatile("red.shared::cluster.or.b32 [%0], %1;\n" ::"r"(ra), "r"(1u << (lb & 31))
                                : "memory");
                   return false;
                 });
    cluster.sync();
    // ascending-id emission: CTA `rank` owns ids [rank*slice_bits, ...): scan the
    // slice, prefix over the cluster's CTAs (DSMEM), write at the global offset
    const uint32_t per = (slice_words + blockDim.x - 1) / blockDim.x;
    const uint32_t w0 = min(slice_words, threadIdx.x * per), w1 = min(slice_words, w0 + per);
    uint32_t cnt = 0;
    for (uint32_t w = w0; w < w1; ++w) cnt += __popc(sbm[w]);
    uint32_t tot;
    uint32_t pos = block_excl_scan_u32(cnt, scan_sh, &tot);
    if (threadIdx.x == 0) cta_cnt = tot;
    cluster.sync();
    uint32_t base = 0, all = 0;
    for (uint32_t r = 0; r < CO_CLUSTER; ++r) {
      const uint32_t c = *cluster.map_shared_rank(&cta_cnt, r);
      if (r < rank) base += c;
      all += c;
    }
    pos += base;
    const uint32_t id0 = rank * slice_bits;
    for (uint32_t w = w0; w < w1; ++w)
      for (uint32_t word = sbm[w]; word; word &= word - 1)
        out[pos++] = id0 + w * 32 + (__ffs(word) - 1);
    if (rank == 0 && threadIdx.x == 0) a.uq[q] = all;
    cluster.sync();  // slices and cta_cnt are reused by the next query
  }
}

// ------------------------------------------------------------ SimHash screen
// CTA per query (SPEC.md:330-338 simhash_screen): keep the B candidates with the
// most agreeing signature bits, ties by lower id.  dis = popc(sig ^ q_sig) (fewer
// = better) is histogrammed; the threshold bin's ties are cut by a radix select
// on the (unique) ids; the survivors are compacted into out[q][0..B).  With
// U <= B the list is copied unchanged (identity case).
constexpr int SCR_THREADS = 256;
__global__ void __launch_bounds__(SCR_THREADS)
k_screen(const uint32_t* __restrict__ cands, const uint64_t* __restrict__ coff,
         const uint32_t* __restrict__ uq, const uint64_t* __restrict__ sigs,
         const uint64_t* __restrict__ qsig, uint32_t B, uint32_t* __restrict__ out,
         uint32_t* __restrict__ uq2) {
  __shared__ uint32_t hist[256];
  __shared__ uint32_t sh_dstar, sh_rem, sh_ties, sh_sel, n_out;
  const uint32_t q = blockIdx.x;
  const uint32_t U = uq[q];
  const uint32_t* c = cands + coff[q];
  uint32_t* o = out + (uint64_t)q * B;
  if (U <= B) {
    for (uint32_t i = threadIdx.x; i < U; i += blockDim.x) o[i] = c[i];
    if (threadIdx.x == 0) uq2[q] = U;
    return;
  }
  const uint64_t sq = qsig[q];
  auto dis_of = [&](uint32_t id) { return (uint32_t)__popcll(__ldg(sigs + id) ^ sq); };
  for (int i = threadIdx.x; i < 65; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x == 0) n_out = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < U; i += blockDim.x) smem_inc(&hist[dis_of(c[i])]);
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t cum = 0, dd = 0;
    for (; dd < 65; ++dd) {
      if (cum + hist[dd] >= B) break;
      cum += hist[dd];
    }
    sh_dstar = dd;
    sh_rem = B - cum;  // ties to take at dstar (1-based rank among them)
    sh_ties = hist[dd];
  }
  __syncthreads();
  const uint32_t dstar = sh_dstar;
  uint32_t idstar = 0xffffffffu;
  if (sh_ties > sh_rem) {  // the sh_rem smallest ids among dis == dstar
    uint32_t prefix = 0, mask = 0, r = sh_rem;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < U; i += blockDim.x) {
        const uint32_t id = c[i];
        if ((id & mask) == prefix && dis_of(id) == dstar) smem_inc(&hist[(id >> shift) & 255u]);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t cum = 0, dg = 0;
        for (; dg < 256; ++dg) {
          if (cum + hist[dg] >= r) break;
          cum += hist[dg];
        }
        sh_sel = dg;
        sh_rem = r - cum;
      }
      __syncthreads();
      prefix |= sh_sel << shift;
      mask |= 255u << shift;
      r = sh_rem;
      __syncthreads();
    }
    idstar = prefix;
  }
  const int lane = threadIdx.x & 31;
  const uint32_t Ur = (U + 31) & ~31u;
  for (uint32_t i = threadIdx.x; i < Ur; i += blockDim.x) {
    const uint32_t id = i < U ? c[i] : 0;
    uint32_t dd = 0;
    if (i < U) dd = dis_of(id);
    const bool take = i < U && (dd < dstar || (dd == dstar && id <= idstar));
    const uint32_t bal = __ballot_sync(FULL, take);
    uint32_t base = 0;
    if (lane == 0 && bal) base = smem_fetch_add(&n_out, __popc(bal));
    base = __shfl_sync(FULL, base, 0);
    if (take) o[base + __popc(bal & ((1u << lane) - 1))] = id;
  }
  if (threadIdx.x == 0) uq2[q] = B;
}

// ------------------------------------------------------------------- score
#ifndef FPP_SC_WARPS
#define FPP_SC_WARPS 4
#endif
constexpr int SC_WARPS = FPP_SC_WARPS;
// Ring geometry <SL, ST>: SL floats per row slice (a multiple of 32), ST stages
// per warp (chosen per row width at launch, see stage_b).
template <int SL>
struct ScRing {
  static constexpr int ROWPAD = SL + 4;  // odd number of 16 B units: conflict-free LDS.128
  static constexpr int STAGE_FLOATS = 32 * ROWPAD;
};

struct ScoreArgs {
  const float* X;
  uint32_t d;
  uint32_t ldx;  // row stride of X (floats)
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
  const uint32_t* uq_all;  // collected candidates per query (stats); nullptr: = uq
  uint32_t cstride;        // != 0: candidates of query q start at q * cstride (screened lists)
  uint32_t* qctr;          // != nullptr: persistent grid, queries fetched from this counter
  uint32_t nq;
  const float* xtail;      // k_score_pruned: row tail norms [xt_n][n] (Index::xtail)
  uint32_t xt_n;
  uint32_t xt_head;        // head slice width (Index::xt_head)
  uint64_t n;
  unsigned long long* dbg;  // FPP_DEBUG_PRUNE: [rows, row slices read]
  unsigned long long* rbytes;  // += candidate-row bytes read (fpp_timings.score_bytes)
  // k_score_screen seeds: the query's first `nseedp` probes (the forced true buckets)
  const uint64_t* ppos;
  const uint32_t* plen;
  const uint32_t* ids;
  uint32_t nseedp;
  // k_score_screen<WALK>: the kernel walks the probes itself (no candidate lists);
  // exact-score dedup through a per-CTA visited bitmap [gridDim.x][nwords] that is
  // left clear (cleared through the per-CTA log of set ids, [gridDim.x][logcap])
  uint32_t* gbm;
  uint32_t nwords;
  uint32_t* wlog;
  uint32_t logcap;
  uint32_t seedcap;  // k_score_screen: seed entries per query (whole leading true buckets)
  const uint4* csrrec;  // WALK: stage-1 records in CSR entry order [kept_total][4] (Index::q8csr)
  // k > 32 (k_score + k_topk_more): the kernel keeps ranks [0, k) of an answer row of
  // `ostride` slots (0: = k) and dumps every candidate's exact score to allsc (same
  // offsets as the candidate lists), from which k_topk_more selects the later ranks
  uint32_t ostride;
  double* allsc;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16s(uint32_t sa, const void* gmem) {  // shared address
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// mbarrier + TMA bulk copies (k_score_pruned<..., TMA = true>)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

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
template <bool VEC, int SC_SLICE, int SC_STAGES, int MINB = 2>
__global__ void __launch_bounds__(SC_WARPS * 32, MINB) k_score(ScoreArgs a) {
  constexpr int SC_ROWPAD = ScRing<SC_SLICE>::ROWPAD;
  constexpr int SC_STAGE_FLOATS = ScRing<SC_SLICE>::STAGE_FLOATS;
  extern __shared__ __align__(16) unsigned char smraw[];
  const uint32_t d = a.d;
  double* qd = reinterpret_cast<double*>(smraw);
  const uint32_t qd_bytes = ((d * 8 + 127) / 128) * 128;
  float* ring = reinterpret_cast<float*>(smraw + qd_bytes);
  __shared__ double mg_s[SC_WARPS][32];
  __shared__ uint32_t mg_i[SC_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ uint32_t q_sh;
  uint32_t q = blockIdx.x;
  for (;;) {
  if (a.qctr) {  // persistent grid: dynamic query fetch
    if (threadIdx.x == 0) q_sh = atomicAdd(a.qctr, 1u);
    __syncthreads();
    q = q_sh;
    if (q >= a.nq) return;
  }
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) qd[j] = (double)a.Q[(uint64_t)q * d + j];
  __syncthreads();
  const uint32_t U = a.uq[q];
  const uint32_t* cand = a.cands + (a.cstride ? (uint64_t)q * a.cstride : a.coff[q]);
  const uint32_t k = a.k;
  double bs = -INFINITY;
  uint32_t bi = 0xffffffffu;
  float* wring = ring + (size_t)w * SC_STAGES * SC_STAGE_FLOATS;
  const uint32_t nb = (U + 31) / 32;
  const uint32_t nsl = (d + SC_SLICE - 1) / SC_SLICE;
  const float* X = a.X;
  // issue cursor
  uint32_t ib = w, ic = 0, nissued = 0;
  // Copy mapping (VEC): with 64-float slices an instruction covers 2 rows x 256 contiguous
  // bytes (16 lanes per row); with 32-float slices 4 rows x 128 bytes.  B200 serves random
  // 256-byte row segments requested by ONE instruction at 6.0-6.2 TB/s, the same bytes as
  // two 128-byte halves from two instructions at 4.7-4.8 (profiles/probes/gather4_probe.cu;
  // TMA tile::gather4 with a 64-float box: 6.2-6.4)
  constexpr int LPR = SC_SLICE >= 64 ? 16 : 8;  // lanes per row
  constexpr int RPI = 32 / LPR;                 // rows per instruction
  constexpr int NIT = 32 / RPI;
  const float* rp[NIT];
  uint32_t my_id = 0xffffffffu;
  const int kk = lane % LPR, rbase = lane / LPR;
  auto load_batch = [&](uint32_t bidx) {
    const uint32_t ci = bidx * 32 + lane;
    my_id = ci < U ? __ldg(cand + ci) : 0xffffffffu;
    if (VEC) {
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        const uint32_t idr = __shfl_sync(FULL, my_id, rbase + RPI * it);
        rp[it] = idr != 0xffffffffu ? X + (uint64_t)idr * a.ldx : nullptr;
      }
    }
  };
  auto issue = [&]() {
    if (ib < nb) {
      float* buf = wring + (size_t)(nissued % SC_STAGES) * SC_STAGE_FLOATS;
      const uint32_t col0 = ic * SC_SLICE;
      const uint32_t len = min((uint32_t)SC_SLICE, d - col0);
      if (VEC) {
#pragma unroll
        for (int h = 0; h < SC_SLICE / (4 * LPR); ++h) {  // 16 B chunks kk + LPR*h of each row
          const uint32_t ch = kk + LPR * h;
          if (ch < (len >> 2)) {
#pragma unroll
            for (int it = 0; it < NIT; ++it)
              if (rp[it]) cp_async16(buf + (rbase + RPI * it) * SC_ROWPAD + ch * 4, rp[it] + col0 + ch * 4);
          }
        }
      } else {
        for (int r = 0; r < 32; ++r) {
          const uint32_t idr = __shfl_sync(FULL, my_id, r);
          if (idr != 0xffffffffu)
            for (uint32_t c = lane; c < len; c += 32)
              cp_async4(buf + r * SC_ROWPAD + c, X + (uint64_t)idr * a.ldx + col0 + c);
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
      const uint32_t id = ci < U ? __ldg(cand + ci) : 0xffffffffu;
      if (a.allsc && ci < U) a.allsc[(cand - a.cands) + ci] = acc;
      topk_insert(bs, bi, k, acc, id, id != 0xffffffffu);  // (grouped lists carry holes)
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
      const uint64_t o = (uint64_t)q * (a.ostride ? a.ostride : k) + lane;
      a.out_ids[o] = ok ? bi + a.id_offset : 0xffffffffu;
      a.out_scores[o] = ok ? bs : -INFINITY;
    }
    // unique candidates scored: the list length, or (grouped lists with holes) the
    // collect's unique count; with a SimHash screen the screened list
    const uint32_t Uu = a.cstride ? U : (a.uq_all ? a.uq_all[q] : U);
    if (lane == 0 && a.stats) {
      a.stats[q].probes = a.peff;
      a.stats[q].entries = a.eq[q];
      a.stats[q].candidates = a.uq_all ? a.uq_all[q] : U;
      a.stats[q].exact = Uu;
    }
    if (lane == 0 && a.rbytes) atomicAdd(a.rbytes, (unsigned long long)Uu * d * 4ull);
  }
  if (!a.qctr) return;
  __syncthreads();  // qd, mg_* and q_sh are reused by the next query
  }
}

// Ranks [32, k) of an answer (k > 32).  k_score kept ranks [0, 32) in its warp lists
// and dumped every candidate's exact score (ScoreArgs::allsc), so every exact score is
// computed once.  Pass p streams the query's (score, id) pairs again and
// keeps the 32 best that come strictly after the previous pass's last entry (the
// cursor) in the answer order (score desc, id asc): ranks [32p, 32p + 32).  A pass
// that ends short (cursor = none) leaves the rest of the row empty.
constexpr int TM_WARPS = 8;
__global__ void __launch_bounds__(TM_WARPS * 32) k_topk_more(ScoreArgs a) {
  __shared__ double mg_s[TM_WARPS][32];
  __shared__ uint32_t mg_i[TM_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t q = blockIdx.x;
  const uint32_t U = a.uq[q];
  const uint64_t base = a.cstride ? (uint64_t)q * a.cstride : a.coff[q];
  const uint32_t* cand = a.cands + base;
  const double* sc = a.allsc + base;
  const uint32_t K = a.ostride;
  uint32_t* oid = a.out_ids + (uint64_t)q * K;
  double* osc = a.out_scores + (uint64_t)q * K;
  for (uint32_t off = 32; off < K; off += 32) {
    const uint32_t k = min(32u, K - off);
    const uint32_t cg = oid[off - 1];  // the cursor (a global id)
    const double cs = osc[off - 1];
    if (cg == 0xffffffffu) {  // the candidates ran out (uniform over the CTA)
      for (uint32_t i = off + threadIdx.x; i < K; i += blockDim.x) {
        oid[i] = 0xffffffffu;
        osc[i] = -INFINITY;
      }
      return;
    }
    const uint32_t ci = cg - a.id_offset;
    double bs = -INFINITY;
    uint32_t bi = 0xffffffffu;
    for (uint32_t c0 = (uint32_t)w * 32; c0 < U; c0 += TM_WARPS * 32) {
      const uint32_t c = c0 + lane;
      const uint32_t id = c < U ? __ldg(cand + c) : 0xffffffffu;
      const double s = c < U ? sc[c] : 0.0;
      topk_insert(bs, bi, k, s, id, id != 0xffffffffu && sbetter(cs, ci, s, id));
    }
    mg_s[w][lane] = bs;
    mg_i[w][lane] = bi;
    __syncthreads();
    if (w == 0) {
      for (int w2 = 1; w2 < TM_WARPS; ++w2)
        topk_insert(bs, bi, k, mg_s[w2][lane], mg_i[w2][lane],
                    (uint32_t)lane < k && mg_i[w2][lane] != 0xffffffffu);
      if ((uint32_t)lane < k) {
        const bool ok = bi != 0xffffffffu;
        oid[off + lane] = ok ? bi + a.id_offset : 0xffffffffu;
        osc[off + lane] = ok ? bs : -INFINITY;
      }
    }
    __syncthreads();  // the next pass reads this pass's last entry and reuses mg_*
  }
}

// Exact early termination of the row gather (results identical to k_score).
// Rows are read as 64-float slices.  Every candidate's first slice (its head) is
// read and summed; lane r then bounds row r's final score by Cauchy-Schwarz,
//   S <= s_m + ||x[m:d)|| * ||q[m:d)||   (+1e-10 relative: fp64 summation error),
// where s_m is the sequential fp64 prefix after m columns (the very value the full
// sum continues from) and ||x[m:d)|| the index's rounded-up tail norm
// (Index::xtail).  A row whose bound is below the CTA's running k-th best score
// (max over the warps' lists; each is the k-th best of distinct candidates, so a
// lower bound of the final one) ends strictly below the final k-th best: it cannot
// enter the top-k and its tail is never read.  Survivors (id, s_m) go to a per-warp
// queue in shared memory and are finished 32 at a time as dense tail batches, with
// the same check after each of the first xt_n slices.  Jobs (a head slice of 32
// candidates, a tail slice of 32 survivors, or a bubble) run through an ST-stage
// cp.async ring per warp (ST-1 jobs in flight); the next job is chosen when it is
// issued and handed to the compute side through shared memory.  Ring rows are
// rotated in 16 B chunks (chunk c of row r at (c + r) mod 16: conflict-free LDS.128
// without padding).  TMA = true moves each row slice with one or two
// cp.async.bulk copies issued by the row's lane, completing on a per-stage mbarrier
// (the rotation splits a slice at the wrap point), instead of 16 cp.async per lane.  Whether the
// bound pays is data dependent (cluster structure): the host measures the read
// fraction and falls back to k_score where it does not (stage_b).
template <int NW, int ST>
struct PrunedCfg {
  static constexpr int SL = (int)XT_SLICE;
  static constexpr int STAGE = 32 * SL;                 // floats per ring stage
  static constexpr uint32_t QCAP = 32u * (ST + 2);      // >= 31 + 32 (ST - 1) + 64
  static constexpr size_t ring_bytes = (size_t)NW * ST * STAGE * 4;
};
template <bool VEC, int NW, int ST, int MINB, bool TMA = false>
__global__ void __launch_bounds__(NW * 32, MINB) k_score_pruned(ScoreArgs a) {
  static_assert(!TMA || VEC, "bulk copies need 16 B-aligned row slices (d % 4 == 0)");
  using C = PrunedCfg<NW, ST>;
  constexpr int SL = C::SL;
  constexpr int STAGE = C::STAGE;
  constexpr uint32_t QCAP = C::QCAP;
  constexpr uint32_t NONE = 0xffffffffu, TNONE = 0xffu;
  constexpr uint32_t J_NOP = 0, J_HEAD = 1, J_TAIL = 2, J_END = 3;
  extern __shared__ __align__(16) unsigned char smraw[];
  const uint32_t d = a.d;
  float* ring = reinterpret_cast<float*>(smraw);
  double* qd = reinterpret_cast<double*>(smraw + C::ring_bytes);
  __shared__ double qt_s[XT_MAX];
  __shared__ double thr_s[NW];   // per warp: k-th best (each a lower bound of the final)
  __shared__ double thr2_s[NW];  // per warp: ceil(k/NW)-th best (the min over warps is one)
  __shared__ uint32_t q_sh;
  __shared__ double sq_acc[NW][QCAP];  // survivor queue: prefix sums
  __shared__ uint32_t sq_id[NW][QCAP];  //                 and ids
  __shared__ uint32_t jd_s[NW][ST];     // job hand-over: descriptor,
  __shared__ uint32_t jid_s[NW][ST][32];  // row id per lane,
  __shared__ float jx_s[NW][ST][32];      // prefetched tail norm per lane
  __shared__ __align__(8) uint64_t mbar[NW][ST];  // TMA: ring stage completion
  volatile double* thr_v = thr_s;
  volatile double* thr2_v = thr2_s;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int kk = lane & 7, rbase = lane >> 3;
  const uint32_t lt_mask = (1u << lane) - 1u;
  const uint32_t hw = a.xt_head;           // head slice width (32 or 64)
  const uint32_t nsl = xt_nslices(d, hw);  // head [0, hw) + 64-wide slices; >= 2 (host: d >= 64)
  const uint32_t nt = a.xt_n;          // checks after slices 0 .. nt-1 (nt < nsl)
  auto col0_of = [&](uint32_t sl) { return sl == 0 ? 0u : hw + (sl - 1) * (uint32_t)SL; };
  auto len_of = [&](uint32_t sl) {
    return sl == 0 ? min(hw, d) : min((uint32_t)SL, d - col0_of(sl));
  };
  float* wring = ring + (size_t)w * ST * STAGE;
  double* qacc = sq_acc[w];
  uint32_t* qid = sq_id[w];
  uint32_t ph = 0;  // TMA: parity of the next wait, bit per stage
  if (TMA) {
    if (lane == 0)
      for (int i = 0; i < ST; ++i) mbar_init(&mbar[w][i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
  }
  uint32_t q = blockIdx.x;
  for (;;) {
    if (a.qctr) {
      if (threadIdx.x == 0) q_sh = atomicAdd(a.qctr, 1u);
      __syncthreads();
      q = q_sh;
      if (q >= a.nq) return;
    }
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) qd[j] = (double)a.Q[(uint64_t)q * d + j];
    if (threadIdx.x < NW) thr_s[threadIdx.x] = thr2_s[threadIdx.x] = -INFINITY;
    __syncthreads();
    if ((uint32_t)w < nt) {  // query tail norms, rounded up
      for (uint32_t t = w; t < nt; t += NW) {
        double sq = 0.0;
        for (uint32_t c = hw + t * SL + lane; c < d; c += 32) sq = fma(qd[c], qd[c], sq);
        for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(FULL, sq, o);
        if (lane == 0) qt_s[t] = __dsqrt_ru(sq) * (1.0 + 1e-12);
      }
    }
    __syncthreads();
    const uint32_t U = a.uq[q];
    const uint32_t* cand = a.cands + (a.cstride ? (uint64_t)q * a.cstride : a.coff[q]);
    const uint32_t k = a.k;
    double bs = -INFINITY;
    uint32_t bi = NONE;
    const uint32_t nb = (U + 31) / 32;
    const uint32_t nbw = nb > (uint32_t)w ? (nb - w + NW - 1) / NW : 0;
    // issue side: next head batch, heads issued, batch in progress (next slice tis,
    // row id per lane), queue head
    uint32_t hb = 0, nh = 0, tis = TNONE, tbase = 0, tcnt = 0, qh = 0, islot = 0, tgen = 0;
    uint32_t bid = NONE;
    unsigned long long wbytes = 0;  // row bytes this warp read (lane 0)
    // written by the compute side, read by the issue side
    uint32_t qtl = 0, hdone = 0, tmask = FULL;
    auto issue = [&]() {
      uint32_t type, s = 0, m = FULL, jid = NONE;
      float jx = 0.f;
      if (tis != TNONE && tmask == 0) tis = TNONE;  // every row of the batch is out
      if (tis != TNONE) {
        type = J_TAIL;
        s = tis;
        m = tmask;
        tis = s + 1 < nsl ? s + 1 : TNONE;
      } else if (qtl - qh >= 32 || (hb == nbw && hdone == nh && qtl != qh)) {
        type = J_TAIL;  // a new tail batch (the last one may be partial)
        s = 1;
        tbase = qh;
        tcnt = min(qtl - qh, 32u);
        qh += tcnt;
        tmask = FULL;
        ++tgen;
        tis = nsl > 2 ? 2 : TNONE;
        jid = bid = (uint32_t)lane < tcnt ? qid[(tbase + lane) % QCAP] : NONE;
        if (jid != NONE && nt > 1) jx = __ldg(a.xtail + a.n + jid);
      } else if (hb < nbw) {
        const uint32_t ci = (w + hb * NW) * 32 + lane;
        jid = ci < U ? __ldg(cand + ci) : NONE;
        if (jid != NONE) jx = __ldg(a.xtail + jid);
        ++hb;
        type = J_HEAD;
        ++nh;
      } else {
        type = hdone < nh ? J_NOP : J_END;
      }
      if ((type == J_HEAD || type == J_TAIL) && m) {
        float* buf = wring + (size_t)islot * STAGE;
        const uint32_t col0 = col0_of(s);
        const uint32_t len = len_of(s);
        const uint32_t rows = __ballot_sync(FULL, (type == J_HEAD ? jid : bid) != NONE);
        wbytes += (unsigned long long)__popc(rows & m) * len * 4u;
        if (a.dbg) {
          if (lane == 0) {
            if (type == J_HEAD) atomicAdd(a.dbg, (unsigned long long)__popc(rows));
            atomicAdd(a.dbg + 1, (unsigned long long)__popc(rows & m) * len);  // floats read
          }
        }
        if (TMA) {  // lane r copies row r's slice (rotated by r & 15: at most two copies)
          if (lane == 0) mbar_arrive_tx(&mbar[w][islot], __popc(rows & m) * len * 4u);
          __syncwarp();
          const uint32_t idr = type == J_HEAD ? jid : bid;
          if (idr != NONE && ((m >> lane) & 1u)) {
            const float* src = a.X + (uint64_t)idr * a.ldx + col0;
            float* dst = buf + lane * SL;
            const uint32_t rot = lane & 15, nch = len >> 2, n1 = min(nch, 16u - rot);
            bulk_g2s(dst + rot * 4, src, n1 * 16, &mbar[w][islot]);
            if (nch > n1) bulk_g2s(dst, src + n1 * 4, (nch - n1) * 16, &mbar[w][islot]);
          }
        // (4 rows x 128 B per instruction; the 2 rows x 256 B mapping of k_score measured
        // slower here: C2 2.76 vs 2.64 ms per launch -- this kernel is bound by job latency)
        } else if (VEC) {
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int rr = rbase + 4 * it;
            const uint32_t idr = __shfl_sync(FULL, type == J_HEAD ? jid : bid, rr);
            if (idr != NONE && ((m >> rr) & 1u)) {
              const float* src = a.X + (uint64_t)idr * a.ldx + col0;
              float* dst = buf + rr * SL;
#pragma unroll
              for (int h = 0; h < SL / 32; ++h) {
                const uint32_t ch = kk + 8 * h;
                if (ch < (len >> 2)) cp_async16(dst + (((ch + rr) & 15) << 2), src + ch * 4);
              }
            }
          }
        } else {
          for (int r = 0; r < 32; ++r) {
            const uint32_t idr = __shfl_sync(FULL, type == J_HEAD ? jid : bid, r);
            if (idr != NONE && ((m >> r) & 1u))
              for (uint32_t c = lane; c < len; c += 32)
                cp_async4(buf + r * SL + ((((c >> 2) + r) & 15) << 2) + (c & 3),
                          a.X + (uint64_t)idr * a.ldx + col0 + c);
          }
        }
      } else if (TMA && lane == 0) {
        mbar_arrive_tx(&mbar[w][islot], 0);  // every issue completes one stage phase
      }
      if (lane == 0)
        jd_s[w][islot] = type << 30 | (tgen & 3u) << 28 | s << 20 | tcnt << 12 | (tbase % QCAP);
      jid_s[w][islot][lane] = jid;
      jx_s[w][islot][lane] = jx;
      if (!TMA) cp_commit();
      islot = islot + 1 == ST ? 0 : islot + 1;
    };
    // compute side: the tail batch in progress
    double tacc = 0.0;
    uint32_t ctid = NONE;
    bool tlive = false;
    float txn = 0.f;
#pragma unroll
    for (int i = 0; i < ST - 1; ++i) issue();
    uint32_t cslot = 0;
    for (;; cslot = cslot + 1 == ST ? 0 : cslot + 1) {
      issue();
      if (TMA) {
        mbar_wait(&mbar[w][cslot], (ph >> cslot) & 1u);
        ph ^= 1u << cslot;
      } else {
        cp_wait<ST - 1>();
      }
      __syncwarp();
      const uint32_t desc = jd_s[w][cslot];
      const uint32_t type = desc >> 30;
      if (type == J_END) break;
      if (type == J_NOP) continue;
      const uint32_t s = (desc >> 20) & 31u;
      const uint32_t jid = jid_s[w][cslot][lane];
      const float jx = jx_s[w][cslot][lane];
      const float* row = wring + (size_t)cslot * STAGE + lane * SL;
      const int sw = lane & 15;
      auto fold = [&](double acc) {
        const uint32_t col0 = col0_of(s);
        const uint32_t len = len_of(s);
        const double* qq = qd + col0;
        // dataset.cpp:67 acc += double(a[i]) * double(b[i]), sequential i (exact products)
        if (VEC && len == SL) {
#pragma unroll
          for (int j = 0; j < SL; j += 4) {
            const float4 xv = *reinterpret_cast<const float4*>(row + ((((j >> 2) + sw) & 15) << 2));
            acc = fma((double)xv.x, qq[j], acc);
            acc = fma((double)xv.y, qq[j + 1], acc);
            acc = fma((double)xv.z, qq[j + 2], acc);
            acc = fma((double)xv.w, qq[j + 3], acc);
          }
        } else if (VEC && len == 32) {  // a 32-wide head slice
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 xv = *reinterpret_cast<const float4*>(row + ((((j >> 2) + sw) & 15) << 2));
            acc = fma((double)xv.x, qq[j], acc);
            acc = fma((double)xv.y, qq[j + 1], acc);
            acc = fma((double)xv.z, qq[j + 2], acc);
            acc = fma((double)xv.w, qq[j + 3], acc);
          }
        } else if (VEC) {  // the last, partial slice (len % 4 == 0)
#pragma unroll 2
          for (uint32_t j = 0; j < len; j += 4) {
            const float4 xv = *reinterpret_cast<const float4*>(row + ((((j >> 2) + sw) & 15) << 2));
            acc = fma((double)xv.x, qq[j], acc);
            acc = fma((double)xv.y, qq[j + 1], acc);
            acc = fma((double)xv.z, qq[j + 2], acc);
            acc = fma((double)xv.w, qq[j + 3], acc);
          }
        } else {
          for (uint32_t j = 0; j < len; ++j)
            acc = fma((double)row[((((j >> 2) + sw) & 15) << 2) + (j & 3)], qq[j], acc);
        }
        return acc;
      };
      // lower bound of the final k-th best: the best warp's k-th, or the worst warp's
      // ceil(k/NW)-th (the warps' lists hold disjoint candidates: NW * ceil(k/NW) >= k
      // scores are at least that); read only where a check needs it
      auto thr_now = [&] {
        double t = thr_v[0], t2 = thr2_v[0];
#pragma unroll
        for (int i = 1; i < NW; ++i) {
          t = fmax(t, thr_v[i]);
          t2 = fmin(t2, thr2_v[i]);
        }
        return fmax(t, t2);
      };
      if (type == J_HEAD) {
        const double acc = fold(0.0);
        bool live = jid != NONE;
        const double T = (double)jx * qt_s[0];
        if (live && acc + T + 1e-10 * (fabs(acc) + T) < thr_now()) live = false;
        const uint32_t bal = __ballot_sync(FULL, live);
        if (live) {
          const uint32_t pos = (qtl + __popc(bal & lt_mask)) % QCAP;
          qid[pos] = jid;
          qacc[pos] = acc;
        }
        qtl += __popc(bal);
        ++hdone;
      } else {  // slice s of a tail batch (queue slots b0 .. b0 + c0 - 1)
        if (s == 1) {
          const uint32_t b0 = desc & 0xfffu, c0 = (desc >> 12) & 63u;
          ctid = jid;
          tacc = (uint32_t)lane >= c0 ? 0.0 : qacc[(b0 + lane) % QCAP];
          tlive = ctid != NONE;
          txn = jx;
        }
        if (tmask || s == 1) tacc = fold(tacc);
        if (s < nt) {
          if (tlive) {
            const double T = (double)txn * qt_s[s];
            if (tacc + T + 1e-10 * (fabs(tacc) + T) < thr_now()) tlive = false;
            if (tlive && s + 1 < nt) txn = __ldg(a.xtail + (uint64_t)(s + 1) * a.n + ctid);
          }
          const uint32_t nm = __ballot_sync(FULL, tlive);
          // slices of an aborted batch may finish after the next batch started:
          // only the current batch owns tmask
          if (((desc >> 28) & 3u) == (tgen & 3u)) tmask = nm;
        }
        if (s + 1 == nsl) {  // batch done: rows still live enter the warp top-k
          topk_insert(bs, bi, k, tacc, ctid, tlive);
          const uint32_t ks = (k + NW - 1) / NW;
          const uint32_t wi = __shfl_sync(FULL, bi, k - 1), wi2 = __shfl_sync(FULL, bi, ks - 1);
          const double ws = __shfl_sync(FULL, bs, k - 1), ws2 = __shfl_sync(FULL, bs, ks - 1);
          if (lane == 0) {
            if (wi != NONE) thr_v[w] = ws;
            if (wi2 != NONE) thr2_v[w] = ws2;
          }
        }
      }
      __syncwarp();
    }
    if (TMA) {  // drain the ST-1 jobs issued past END (no copies): phases stay in step
      for (int i = 0; i < ST - 1; ++i) {
        cslot = cslot + 1 == ST ? 0 : cslot + 1;
        mbar_wait(&mbar[w][cslot], (ph >> cslot) & 1u);
        ph ^= 1u << cslot;
      }
    } else {
      cp_wait<0>();
    }
    if (lane == 0 && a.rbytes && wbytes) atomicAdd(a.rbytes, wbytes);
    __syncthreads();  // the ring is reused for the CTA merge
    double* mg_s = reinterpret_cast<double*>(ring);
    uint32_t* mg_i = reinterpret_cast<uint32_t*>(ring + 2 * NW * 32);
    mg_s[w * 32 + lane] = bs;
    mg_i[w * 32 + lane] = bi;
    __syncthreads();
    if (w == 0) {
      for (int w2 = 1; w2 < NW; ++w2) {
        const bool valid = (uint32_t)lane < k && mg_i[w2 * 32 + lane] != NONE;
        topk_insert(bs, bi, k, mg_s[w2 * 32 + lane], mg_i[w2 * 32 + lane], valid);
      }
      if ((uint32_t)lane < k) {
        const bool ok = bi != NONE;
        a.out_ids[(uint64_t)q * k + lane] = ok ? bi + a.id_offset : NONE;
        a.out_scores[(uint64_t)q * k + lane] = ok ? bs : -INFINITY;
      }
      if (lane == 0 && a.stats) {
        a.stats[q].probes = a.peff;
        a.stats[q].entries = a.eq[q];
        a.stats[q].candidates = a.uq_all ? a.uq_all[q] : U;
        a.stats[q].exact = a.cstride ? U : (a.uq_all ? a.uq_all[q] : U);
      }
    }
    __syncthreads();  // mg_* (ring), qd, thr_s are reused by the next query
    if (TMA) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> TMA
    if (!a.qctr) return;
  }
}

// --------------------------------------------- narrow rows: screen + exact finish
// k_score_screen: the score gather for narrow rows (64 <= d <= 256: C1, C4), with
// exact early termination restructured around bytes and instructions (the fp64
// sequential fold of every candidate head made k_score_pruned issue-bound, and the
// fp32 head is 128 B per candidate).
//   Screen.  Every row has a 64-byte record built with the index (k_q8_records):
//   dims [0, 48) as int8 codes c with a per-row scale s_x, and {s_x, r_x = ||x_h -
//   s_x c||, m_x = ||s_x c||, t_x = ||x[48:d)||} rounded up.  The query head is
//   quantized the same way per CTA (q~ = s_q c_q, r_q = ||q_h - q~||).  A warp takes
//   32 candidates: four lanes read one record (16 B each; eight records per load
//   instruction), three of them form the integer dot product I = c.c_q with DP4A,
//   a 2-step shuffle sums it and the record's fourth lane bounds the row's final
//   computed score:
//     S <= s_x s_q I + r_x ||q_h|| + m_x r_q + t_x ||q_t|| + 1e-6 (|.| terms)
//   (x.q = x~.q~ + (x_h - x~).q_h + x~.(q_h - q~) + x_t.q_t, each by Cauchy-Schwarz;
//   every term is evaluated with upward rounding, and the 1e-6 relative margin also
//   covers the fp64 summation error of the final score).  A row whose bound is below
//   the CTA's running k-th best lower bound (the best warp's k-th, or the worst
//   warp's ceil(k/NW)-th: the warps hold disjoint candidates) ends strictly below
//   the final k-th best: it cannot enter the top-k nor tie.
//   Exact.  Survivor ids queue per warp (shared memory); every 32 are finished as
//   one dense batch: 32-float chunks of the 32 rows are loaded coalesced (4 rows
//   per instruction), staged in shared memory (row stride 36 floats: conflict-free
//   STS.128/LDS.128), and lane r folds row r in the reference's sequential fp64
//   order (dataset.cpp:67), so the score equals inner_product bit for bit; the next
//   chunk's loads are in flight meanwhile.  The batch enters the warp's register
//   top-k and raises the CTA thresholds.
// Results are identical to k_score / k_score_pruned / the oracle.  Grouped candidate
// lists may carry holes (0xFFFFFFFF): skipped.
constexpr int NS_W = 8;            // warps per CTA
constexpr uint32_t NS_QCAP = 64;   // survivor queue per warp (<= 31 + 32 queued)
#ifndef FPP_NS_RING
#define FPP_NS_RING 3  // (1 KB slots + a 2 KB exact staging buffer per warp; C4 screen 95.3 ms, depth 4: 97.5)
#endif
constexpr int NS_RING = FPP_NS_RING;  // stage-1 record ring depth per warp (cp.async)
constexpr int NS_IDR = 2 * NS_RING;   // candidate-id ring depth per warp (lists mode only)
constexpr int NS_SLOT = 64;           // uint4 per ring slot: 32 records of 32 B
constexpr int NS_STG = 128;           // uint4 of the per-warp exact staging buffer (32 rows x 16 floats)
#ifndef FPP_NS_TMA
#define FPP_NS_TMA 0  // measured: C4 511 vs 538 k q/s with the cp.async ring
#endif
constexpr int NS_TMA = FPP_NS_TMA;    // WALK: stage-1 records by TMA bulk copies per run
#ifndef FPP_NS_SH_BITS
#define FPP_NS_SH_BITS 11
#endif
constexpr uint32_t NS_SH_BITS = FPP_NS_SH_BITS, NS_SH = 1u << NS_SH_BITS;  // seed id hash (lists) /
                                                                // admission hash (WALK)
constexpr int WK_HPROBE = 32;  // admission hash: probes before the bitmap takes an id
#ifndef FPP_NS_PF
#define FPP_NS_PF 0  // (measured on C4: each bit costs ~2 ms of 100: the kernel is issue-bound) bit 0: stage-A survivors prefetch their stage-B record into L2;
#endif               // bit 1: rows admitted to the exact stage prefetch their lines
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

__device__ __forceinline__ unsigned long long dkey(double x) {  // order-preserving
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}
__device__ __forceinline__ int fkey(float x) {  // order-preserving (signed compare)
  const int b = __float_as_int(x);
  return b ^ ((b >> 31) & 0x7fffffff);
}

// Seeds: all entries of the leading true buckets (whole buckets, up to a cap) are
// scored exactly first, straight into the warps' lists, so the scan starts near the
// final k-th best.  Every id is scored exactly at most once: the
// collect's lists hold each id once, and their seeds are recognised by a
// shared-memory hash of the seed ids at the exact stage's admission.
// WALK = true (the default; FPP_SC_WALK=0 reads lists): the kernel walks the query's
// probes itself -- no collect pass, no candidate lists, no host sync.  Warps take
// 32-probe chunks from a CTA counter and cover each chunk's entries 32 at a time (the
// warp-cooperative walk of k_collect), the ids moving by cp.async into the id ring
// ahead of their records.  Entries repeat across tables, so admission is a
// test-and-set in a per-CTA visited bitmap (global memory, n bits, L2 atomics on the
// few stage-2 survivors; its set bits are logged and cleared at the end of the
// query); persistent CTAs (one bitmap each) fetch queries from a counter.  On C4 the
// walk reads ~30% more DRAM bytes than the screen over the collect's id-ordered lists
// (12.2 vs 9.3 MB per query: repeats, and rows gathered in probe order hit L2 less),
// but saves the collect pass: 231 ms per step against 97 + 148.
constexpr uint32_t WK_SEEDCAP = 64;  // seed entries per query (whole leading true buckets; C4: 64 -> 686 k, 512 -> 668 k, none -> 678 k q/s)

template <int NW, int MINB, bool WALK>
__global__ void __launch_bounds__(NW * 32, MINB) k_score_screen(ScoreArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr uint32_t NONE = 0xffffffffu;
  const uint32_t d = a.d, nch = (d + 31) / 32;  // 32-float chunks (rows padded with zeros)
  // fixed-size parts first (compile-time offsets: the compiler rematerialises these
  // addresses under the register cap), the d-dependent query copy last
  uint4* ring_all = reinterpret_cast<uint4*>(smraw);                   // [NW][RING][1 KB]
  uint4* stg_all = ring_all + (size_t)NW * NS_RING * NS_SLOT;          // [NW][2 KB] exact staging
  uint32_t* idr_all = reinterpret_cast<uint32_t*>(stg_all + (size_t)NW * NS_STG);  // lists: [NW][IDR][32]
  uint32_t* sq_all = idr_all + (WALK ? (size_t)0 : (size_t)NW * NS_IDR * 32);  // [NW][QCAP]
  uint32_t* s1_all = sq_all + (size_t)NW * NS_QCAP;                    // [NW][QCAP] stage-2 queue ids
  float2* s1v_all = reinterpret_cast<float2*>(s1_all + (size_t)NW * NS_QCAP);  // [NW][QCAP] (A1, N1)
  double* qd = reinterpret_cast<double*>(s1v_all + (size_t)NW * NS_QCAP);  // [32 * nch]
  __shared__ unsigned long long thr_key;  // lower bound of the final k-th best (ordered key)
  __shared__ int thr_fk;  // the same bound rounded down to fp32, as an ordered int key (fkey)
  __shared__ double thr2_s[NW];          // per warp: its ceil(k/NW)-th best
  __shared__ uint32_t nseed_s;
  __shared__ float qn_s[Q8_STAGES][4];   // per stage: s_q, ||q_h||, r_q, ||q after the stage||
  __shared__ __align__(16) int32_t q8_s[Q8_STAGES][Q8B_DIMS / 4];  // the query's stage codes
  __shared__ double mg_s[NW][32];
  __shared__ uint32_t mg_i[NW][32];
  __shared__ uint32_t q_s, wctr_s[2], logn_s;  // query, walker chunk counters, log length
  __shared__ uint32_t wk_rng_s[2][2];          // walker ranges: seeds, main walk
  __shared__ uint32_t cnt_s[NW][2];            // per warp: stage-2 records, exact rows
  __shared__ uint32_t seedh[NS_SH];     // lists: the seeds' ids (open addressing)
  __shared__ __align__(8) uint64_t smbar[WALK && NS_TMA ? NW : 1][NS_RING];  // TMA: per ring slot
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint4* ring = ring_all + (size_t)w * NS_RING * NS_SLOT;
  uint32_t* idr = idr_all + (size_t)w * NS_IDR * 32;  // candidate ids of batch b: slot b % IDR
  const uint32_t ring_sa = (uint32_t)__cvta_generic_to_shared(ring);
  uint32_t* sq = sq_all + (size_t)w * NS_QCAP;    // survivors of stage 2 -> exact
  uint32_t* s1q = s1_all + (size_t)w * NS_QCAP;   // survivors of stage 1 -> stage 2
  float2* s1v = s1v_all + (size_t)w * NS_QCAP;
  // WALK: the CTA's visited bitmap (exact-stage admission, every id scored once)
  // (the visited bitmap / log pointers are formed where used, from the parameters:
  // no registers held across the hot loop)
  auto bm_of = [&] { return a.gbm + (size_t)blockIdx.x * a.nwords; };
  auto wlog_of = [&] { return a.wlog + (size_t)blockIdx.x * a.logcap; };
  const uint4* rec = reinterpret_cast<const uint4*>(a.xtail);  // [stages][n][4] 16 B parts
  uint32_t mph = 0;  // TMA: parity of each ring slot's next completion (bit per slot)
  if constexpr (WALK && NS_TMA) {
    if (lane == 0)
      for (int i = 0; i < NS_RING; ++i) mbar_init(&smbar[w][i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
  }
  const float* X = a.X;
  const uint32_t ldx = a.ldx;
  const uint32_t k = a.k;
  for (uint32_t qi = 0;; ++qi) {
  if (!a.qctr && qi) break;  // (one query per CTA unless persistent)
  if (threadIdx.x == 0) {  // persistent CTAs fetch queries from a counter
    q_s = a.qctr ? atomicAdd(a.qctr, 1u) : blockIdx.x;
    wctr_s[0] = wctr_s[1] = 0;
    wk_rng_s[0][0] = wk_rng_s[0][1] = wk_rng_s[1][0] = 0;
    wk_rng_s[1][1] = (uint32_t)a.peff;
    logn_s = 0;
  }
  for (uint32_t i = threadIdx.x; i < NS_SH; i += blockDim.x) seedh[i] = NONE;
  __syncthreads();
  const uint32_t q = q_s;
  if (q >= a.nq) break;
  const float* Qr = a.Q + (uint64_t)q * d;
  for (uint32_t j = threadIdx.x; j < nch * 32; j += blockDim.x) qd[j] = j < d ? (double)Qr[j] : 0.0;
  if (threadIdx.x == 0) {
    thr_key = dkey(-INFINITY);
    thr_fk = fkey(-INFINITY);
  }
  if (threadIdx.x < NW) {
    thr2_s[threadIdx.x] = -INFINITY;
    cnt_s[threadIdx.x][0] = cnt_s[threadIdx.x][1] = 0;
  }
  if ((uint32_t)w < Q8_STAGES) {  // quantize the query like the records (k_q8_records)
    const uint32_t W = w ? Q8B_DIMS : Q8A_DIMS;
    const uint32_t lo = w ? Q8A_DIMS : 0u, hi = min(d, lo + W);
    float x[3];
    float mx = 0.f;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint32_t kk = lane + 32 * j;
      x[j] = (kk < W && lo + kk < hi) ? Qr[lo + kk] : 0.f;
      mx = fmaxf(mx, fabsf(x[j]));
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
    const float sc = mx / 127.0f;
    double er = 0.0, hh = 0.0, tt = 0.0;
    int c[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      c[j] = sc > 0.f ? max(-127, min(127, __float2int_rn(x[j] / sc))) : 0;
      const double e = (double)x[j] - (double)sc * c[j];
      er = fma(e, e, er);
      hh = fma((double)x[j], (double)x[j], hh);
    }
    for (uint32_t j = lo + W + lane; j < d; j += 32) tt = fma((double)Qr[j], (double)Qr[j], tt);
    for (int o = 16; o; o >>= 1) {
      er += __shfl_xor_sync(FULL, er, o);
      hh += __shfl_xor_sync(FULL, hh, o);
      tt += __shfl_xor_sync(FULL, tt, o);
    }
    unsigned char* qb = reinterpret_cast<unsigned char*>(q8_s[w]);
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (lane + 32 * j < (int)Q8B_DIMS) qb[lane + 32 * j] = (unsigned char)(signed char)c[j];
    if (lane == 0) {
      qn_s[w][0] = sc;
      qn_s[w][1] = __double2float_ru(__dsqrt_ru(hh) * (1.0 + 1e-12));
      qn_s[w][2] = __double2float_ru(__dsqrt_ru(er) * (1.0 + 1e-12));
      qn_s[w][3] = __double2float_ru(__dsqrt_ru(tt) * (1.0 + 1e-12));
    }
  }
  __syncthreads();
  const uint32_t Len = WALK ? 0u : a.uq[q];
  const uint32_t* cand = WALK ? nullptr : a.cands + a.coff[q];
  double bs = -INFINITY;
  uint32_t bi = NONE;
  uint32_t qhead = 0, qtail = 0, h1 = 0, t1 = 0;  // exact queue, stage-2 queue
  uint32_t nrows = 0;  // rows screened (stage-2 records and exact rows: cnt_s)

  auto thr_now = [&] { return dkey_inv(*(volatile unsigned long long*)&thr_key); };
  // ---------------------------------------------------------------- exact rows
  // lane r folds row `id` of lane r (NONE: nothing) in the reference's order; `stg` is
  // a free 2 KB slot of the warp's record ring
  auto exact_fold = [&](uint32_t id, float* stg) {
    // 16-float half chunks of the 32 rows: 4 lanes per row (16 B each), 8 rows per
    // load instruction, staged in shared memory (row r's 16 B chunk c at r * 16 +
    // 4 * (c ^ ((r >> 1) & 3)) floats: conflict-free STS.128 / LDS.128 without
    // padding); the next half chunk is in flight while lane r folds row r's 16 floats
    float4 v[4];
    const int p4 = lane & 3, r8 = lane >> 2;
    const uint32_t nh = nch * 2;
    auto load_h = [&](uint32_t hc) {
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const uint32_t idr = __shfl_sync(FULL, id, it * 8 + r8);
        v[it] = idr != NONE ? __ldcg(reinterpret_cast<const float4*>(X + (uint64_t)idr * ldx + hc * 16) + p4)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    load_h(0);
    double acc = 0.0;
    for (uint32_t hc = 0; hc < nh; ++hc) {
      __syncwarp();  // the previous half chunk's readers are done with the staging rows
#pragma unroll
      for (int it = 0; it < 4; ++it)
        *reinterpret_cast<float4*>(stg + (it * 8 + r8) * 16 + 4 * (p4 ^ (((it * 8 + r8) >> 1) & 3))) = v[it];
      if (hc + 1 < nh) load_h(hc + 1);
      __syncwarp();
      const float* row = stg + lane * 16;
      const int sw = (lane >> 1) & 3;
      const double* qq = qd + hc * 16;
      // dataset.cpp:67 acc += double(a[i]) * double(b[i]), sequential i (exact products)
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 xv = *reinterpret_cast<const float4*>(row + 4 * ((j >> 2) ^ sw));
        acc = fma((double)xv.x, qq[j], acc);
        acc = fma((double)xv.y, qq[j + 1], acc);
        acc = fma((double)xv.z, qq[j + 2], acc);
        acc = fma((double)xv.w, qq[j + 3], acc);
      }
    }
    return acc;
  };
  // lower bounds of the final k-th best from a family of NW disjoint per-warp lists
  // (lb[] = that family's per-warp ceil(k/NW)-th bests): this warp's k-th score, and
  // the worst warp's ceil(k/NW)-th (NW * ceil(k/NW) >= k distinct scores are at least
  // that); folded into one word by atomicMax (a max of lower bounds is one), so
  // readers load a single value per batch
  auto publish = [&](double lbs, uint32_t lbi, volatile double* lb) {
    const uint32_t ks = (k + NW - 1) / NW;
    const uint32_t kid = __shfl_sync(FULL, lbi, k - 1), kid2 = __shfl_sync(FULL, lbi, ks - 1);
    const double kth = __shfl_sync(FULL, lbs, k - 1), kth2 = __shfl_sync(FULL, lbs, ks - 1);
    if (lane == 0) {
      if (kid2 != NONE) lb[w] = kth2;
      double t2 = INFINITY;
#pragma unroll
      for (int i = 0; i < NW; ++i) t2 = fmin(t2, lb[i]);
      const double t = kid != NONE ? fmax(kth, t2) : t2;
      if (t > -INFINITY) {
        atomicMax(&thr_key, dkey(t));
        // fp32 copy for the record screens: rounded down (a lower bound still), zeros as
        // -0 (the smallest key of the two zeros, so ub = +-0 >= thr compares as floats do)
        float tf = __double2float_rd(t);
        if (tf == 0.f) tf = -0.f;
        atomicMax(&thr_fk, fkey(tf));
      }
    }
  };
  auto exact_batch = [&](uint32_t cnt, float* stg) {
    const uint32_t id = (uint32_t)lane < cnt ? sq[(qhead + lane) % NS_QCAP] : NONE;
    qhead += cnt;
    const double acc = exact_fold(id, stg);
    // rows below the CTA's lower bound of the final k-th best cannot enter the top-k
    // nor tie: kept out of the warp list (its entries stay distinct real candidates,
    // so the bounds published from it stay valid), fewer insertions
    topk_insert(bs, bi, k, acc, id, id != NONE && acc >= thr_now());
    if (lane == 0) cnt_s[w][1] += cnt;
    publish(bs, bi, thr2_s);
  };
  // admission to the exact stage (lanes with `want`): true for an id not scored exactly
  // before in this query.  WALK: a shared-memory hash of the admitted ids, backed by a
  // test-and-set in the CTA's visited bitmap for the ids the hash cannot hold.
  // Lists (deduplicated by the collect) meet only the seeds again: an id found in the
  // seed hash is not admitted (the seeds are scored from the hash itself).
  auto hslot = [](uint32_t id) { return (id * 2654435761u) >> (32 - NS_SH_BITS); };
  auto seed_insert = [&](uint32_t id) {
    for (uint32_t h = hslot(id);; h = (h + 1) & (NS_SH - 1)) {
      const uint32_t old = atomicCAS(&seedh[h], NONE, id);
      if (old == NONE) return true;
      if (old == id) return false;
    }
  };
  auto seed_has = [&](uint32_t id) {
    for (uint32_t h = hslot(id);; h = (h + 1) & (NS_SH - 1)) {
      const uint32_t v = seedh[h];
      if (v == id) return true;
      if (v == NONE) return false;
    }
  };
  auto admit = [&](uint32_t id, bool want) {
    bool fresh = false;
    if (a.gbm) {  // WALK: lists repeat ids
      // first the shared-memory hash (a CAS on the first empty slot of the id's probe
      // sequence; slots only fill, so an id whose sequence is full of other ids can
      // never enter later either): 1 = inserted, 0 = present; ids with a full
      // sequence (-1) take the visited bitmap, whose set bits are logged
      int res = -1;
      if (want) {
        uint32_t h = hslot(id);
        for (int t = 0; t < WK_HPROBE; ++t, h = (h + 1) & (NS_SH - 1)) {
          const uint32_t old = atomicCAS(&seedh[h], NONE, id);
          if (old == NONE || old == id) {
            res = old == NONE;
            break;
          }
        }
      }
      bool viab = false;
      if (want && res < 0) {
        const uint32_t bit = 1u << (id & 31);
        viab = !(atomicOr(bm_of() + (id >> 5), bit) & bit);
      }
      fresh = res == 1 || viab;
      const uint32_t bal = __ballot_sync(FULL, viab);
      if (bal) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&logn_s, (uint32_t)__popc(bal));
        base = __shfl_sync(FULL, base, 0) + __popc(bal & lt_mask);
        if (viab && base < a.logcap) wlog_of()[base] = id;
      }
    } else {
      fresh = want && !seed_has(id);
    }
    return fresh;
  };
  // sq push of the lanes with `live` (ids), ballot-compacted
  auto push_exact = [&](uint32_t id, bool live) {
    const uint32_t live_m = __ballot_sync(FULL, live);
    if (live) sq[(qtail + __popc(live_m & lt_mask)) % NS_QCAP] = id;
    qtail += __popc(live_m);
  };

  // ----------------------------------------------------------- probe walker (WALK)
  // Warp-cooperative walk over probes [wk_p0, wk_p1): 32-probe chunks from a CTA
  // counter (the next chunk's (pos, len) loads in flight while the current one is
  // walked); wk_next() returns lane l's id of the next 32-entry window (NONE past a
  // chunk's end) and sets wk_done, with NONE, once the range is exhausted.
  // (the walk's range and chunk counter live in shared memory, wk_rng_s[phase]: read
  // once per 32-probe chunk, they need no registers in the hot loop)
  const uint32_t* pl = a.plen + (uint64_t)q * a.peff;
  uint32_t wk_T = 0, wk_e0 = 0, wk_nc = 0, wk_cex = 0, wk_plo = 0, wk_phi = 0;
  uint32_t wk_nlen = 0, nprod = 0, wk_tot = 0, wk_ph = 0;  // wk_tot: entries walked
  uint64_t wk_npos = 0;
  bool wk_nhas = false, wk_done = true;
  auto wk_fetch = [&] {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(&wctr_s[wk_ph], 1u);
    c = __shfl_sync(FULL, c, 0);
    const uint32_t p0 = wk_rng_s[wk_ph][0], p1 = wk_rng_s[wk_ph][1];
    const uint32_t p = p0 + c * 32 + lane;
    wk_nhas = p0 + c * 32 < p1;
    wk_nlen = 0;
    wk_npos = 0;
    if (p < p1) {
      const uint64_t o = (uint64_t)q_s * a.peff + p;
      wk_nlen = __ldg(a.plen + o);
      wk_npos = __ldg(a.ppos + o);
    }
  };
  auto wk_begin = [&](uint32_t ph) {
    wk_ph = ph;
    wk_T = wk_e0 = 0;
    wk_done = false;
    nprod = 0;
    wk_fetch();
  };
  // wk_step: the next 32-entry window; lane l's CSR position in gp, false for lanes
  // past a chunk's end and, with wk_done set, once the range is exhausted
  auto wk_step = [&](uint64_t& gp) -> bool {
    while (wk_e0 >= wk_T) {
      if (!wk_nhas) {
        wk_done = true;
        return false;
      }
      const uint32_t len = wk_nlen;
      const uint64_t pos = wk_npos;
      wk_fetch();
      uint32_t incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      wk_T = __shfl_sync(FULL, incl, 31);
      wk_tot += wk_T;
      const uint32_t ne = __ballot_sync(FULL, len > 0);
      wk_nc = __popc(ne);
      const uint32_t src = (uint32_t)lane < wk_nc ? __fns(ne, 0, lane + 1) : 0u;
      wk_cex = __shfl_sync(FULL, incl - len, src);
      wk_plo = __shfl_sync(FULL, (uint32_t)pos, src);
      wk_phi = __shfl_sync(FULL, (uint32_t)(pos >> 32), src);
      wk_e0 = 0;
    }
    const uint32_t E0 = wk_e0, e = E0 + lane;
    const bool cval = (uint32_t)lane < wk_nc;
    const uint32_t r0 = __popc(__ballot_sync(FULL, cval && wk_cex <= E0)) - 1u;
    const uint32_t dd = wk_cex - E0;
    const uint32_t sm = __reduce_or_sync(FULL, (cval && wk_cex > E0 && dd < 32u) ? (1u << dd) : 0u);
    const uint32_t r = r0 + __popc(sm & ((2u << lane) - 1u));
    const uint32_t plo = __shfl_sync(FULL, wk_plo, r);
    const uint32_t phi = __shfl_sync(FULL, wk_phi, r);
    const uint32_t ex = __shfl_sync(FULL, wk_cex, r);
    wk_e0 += 32;
    ++nprod;
    gp = (((uint64_t)phi << 32) | plo) + (e - ex);
    return e < wk_T;
  };
  auto wk_next = [&]() -> uint32_t {  // lane l's id of the next window (NONE: none)
    uint64_t gp;
    return wk_step(gp) ? __ldg(a.ids + gp) : NONE;
  };

  // ---------------------------------------------------------------- seeds
  // The candidates in the query's true buckets (its first nseedp probes, one per
  // table) are mostly its near neighbours: scored exactly first, so the scan below
  // starts near the final k-th best instead of at -inf.  Every entry of the leading
  // true buckets (whole buckets, up to WK_SEEDCAP entries) is admitted through the
  // visited bitmap and scored into the warps' main lists; WALK then starts the walk
  // after those probes, and lists meet the seeds again in the scan, where the
  // bitmap drops them before the exact stage.
  uint32_t pstart = 0;
  float* const stg0 = reinterpret_cast<float*>(stg_all + (size_t)w * NS_STG);  // exact staging rows
  if (a.nseedp) {
    // leading true buckets whose cumulative length stays <= the seed cap (lists: half
    // the seed hash, so its load stays <= 1/2)
    const uint32_t seedcap = a.gbm ? a.seedcap : min(a.seedcap, NS_SH / 2);
    if (w == 0) {
      uint32_t acc = 0, cnt = 0;
      for (uint32_t p0 = 0; p0 < a.nseedp; p0 += 32) {
        const uint32_t p = p0 + lane;
        const uint32_t len = p < a.nseedp ? pl[p] : 0u;
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += y;
        }
        const uint32_t ok = __ballot_sync(FULL, p < a.nseedp && acc + incl <= seedcap);
        cnt += __popc(ok);
        if (ok != FULL) break;
        acc += __shfl_sync(FULL, incl, 31);
      }
      if (lane == 0) {
        nseed_s = cnt;
        wk_rng_s[0][1] = wk_rng_s[1][0] = cnt;
      }
    }
    __syncthreads();
    pstart = nseed_s;
    wk_begin(0);
    if (a.gbm) {  // WALK: admitted through the bitmap and scored as they come
      for (;;) {
        const uint32_t id = wk_next();
        if (wk_done) break;
        push_exact(id, admit(id, id != NONE));
        if (qtail - qhead >= 32) {
          __syncwarp();
          exact_batch(32, stg0);
        }
      }
    } else {
      // lists: insert every seed id into the hash (a short, balanced walk), then each
      // warp scores the ids of its slice of the hash.  The barrier between the two
      // makes the hash complete before any admission of the scan reads it.
      for (;;) {
        const uint32_t id = wk_next();
        if (wk_done) break;
        if (id != NONE) seed_insert(id);
      }
      __syncthreads();
      for (uint32_t h0 = w * (NS_SH / NW); h0 < (w + 1) * (NS_SH / NW); h0 += 32) {
        const uint32_t id = seedh[h0 + lane];
        push_exact(id, id != NONE);
        if (qtail - qhead >= 32) {
          __syncwarp();
          exact_batch(32, stg0);
        }
      }
    }
    if (qtail != qhead) {
      __syncwarp();
      exact_batch(qtail - qhead, stg0);
    }
  }

  // -------------------------------------------------------- record stage bounds
  // Stage A (32 B records, two 16 B parts: codes 0-15 | codes 16-19, the id slot and
  // the half2 terms): 32 candidates, lane c <-> candidate c (id NONE = none), each lane
  // reading its own record.  Returns A = s_x s_q I + r_x ||q_h|| + m_x r_q (rounded
  // up) and, in `tx`, the norm of the row after the stage.
  struct Recs {
    uint4 r[1];  // part 0
    uint4 m;     // part 1
  };
  const int p2 = lane & 1, g16 = lane >> 1;
  // lane c bounds its own candidate: the record's 20 codes are part 0 (16 B) and the
  // first word of part 1 (R.m), five DP4A against the query's codes (qa, qa4)
  auto terms_bound = [&](int dot, float sx, float rx, float mxn, uint32_t stage) {
    const float qs = qn_s[stage][0], qh = qn_s[stage][1], qr = qn_s[stage][2];
    const float If = (float)dot;  // |I| <= 96 * 127^2 < 2^24: exact in fp32
    // s_x s_q I rounded up: round the scale product toward the side that raises it
    const float sp = dot >= 0 ? __fmul_ru(sx, qs) : __fmul_rd(sx, qs);
    return __fadd_ru(__fmul_ru(sp, If), __fmaf_ru(rx, qh, __fmul_ru(mxn, qr)));
  };
  auto stageA_bound = [&](const Recs& R, float& tx, float& nx, const int4 qa, const int qa4) {
    int d0 = __dp4a((int)R.r[0].x, qa.x, 0);  // (two chains: shorter dependency)
    int d1 = __dp4a((int)R.r[0].z, qa.z, 0);
    d0 = __dp4a((int)R.r[0].y, qa.y, d0);
    d1 = __dp4a((int)R.r[0].w, qa.w, d1);
    d0 = __dp4a((int)R.m.x, qa4, d0);
    const int dot = d0 + d1;
    const __half2 sr = *reinterpret_cast<const __half2*>(&R.m.z);
    const __half2 mt = *reinterpret_cast<const __half2*>(&R.m.w);
    const float sx = __low2float(sr), rx = __high2float(sr), mxn = __low2float(mt);
    tx = __high2float(mt);
    nx = __fadd_ru(mxn, rx);  // >= ||x_h||
    return terms_bound(dot, sx, rx, mxn, 0);
  };
  // Stage B (128 B records by id): eight lanes per record (parts 0-5 codes, 6 the fp32
  // terms, 7 padding), four records per round, eight rounds; each round's integer
  // dot is reduced over its 8-lane group and handed to the candidate's lane.
  auto stageB_bound = [&](uint32_t id, float& tx) {
    const int p8 = lane & 7, g8 = lane >> 3;
    const uint4* rs = rec + (uint64_t)a.n * 2;  // [n][8] uint4
    const uint4 m = id != NONE ? __ldcg(rs + (uint64_t)id * 8 + 6) : make_uint4(0, 0, 0, 0);
    const int4 qw = p8 < 6 ? *reinterpret_cast<const int4*>(&q8_s[1][4 * p8]) : make_int4(0, 0, 0, 0);
    int dot = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // two halves of four rounds (register budget)
      uint4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t idr = __shfl_sync(FULL, id, (h * 4 + j) * 4 + g8);
        v[j] = (idr != NONE && p8 < 6) ? __ldcg(rs + (uint64_t)idr * 8 + p8) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int it = h * 4 + j;
        int t = __dp4a((int)v[j].x, qw.x, 0);
        t = __dp4a((int)v[j].y, qw.y, t);
        t = __dp4a((int)v[j].z, qw.z, t);
        t = __dp4a((int)v[j].w, qw.w, t);
        t += __shfl_xor_sync(FULL, t, 4);
        t += __shfl_xor_sync(FULL, t, 2);
        t += __shfl_xor_sync(FULL, t, 1);
        const int got = __shfl_sync(FULL, t, (lane & 3) * 8);  // candidate it * 4 + (lane & 3)
        if ((lane >> 2) == it) dot = got;
      }
    }
    tx = __uint_as_float(m.w);
    return terms_bound(dot, __uint_as_float(m.x), __uint_as_float(m.y), __uint_as_float(m.z), 1);
  };
  const float qt1 = qn_s[0][3], qt2 = qn_s[1][3];
  const float qnorm = __fadd_ru(qn_s[0][1], qt1);  // >= ||q||
  // the threshold as an fp32 ordered key (one LDS + integer compare per lane)
  auto thr_fnow = [&] { return *(volatile int*)&thr_fk; };

  // stage 2 of 32 stage-1 survivors: bound A1 + A2 + t2 ||q after stage 2||
  auto stage2_batch = [&](uint32_t cnt) {
    const uint32_t slot = (h1 + lane) % NS_QCAP;
    const uint32_t id = (uint32_t)lane < cnt ? s1q[slot] : NONE;
    const float2 an = (uint32_t)lane < cnt ? s1v[slot] : make_float2(0.f, 0.f);
    h1 += cnt;
    float tx;
    const float A2 = stageB_bound(id, tx);
    bool live = false;
    if (id != NONE) {
      const float A = __fadd_ru(an.x, A2);
      const float mag = __fadd_ru(__fadd_ru(fabsf(an.x), fabsf(A2)), an.y);
      const float ub = __fadd_ru(__fmaf_ru(tx, qt2, A), __fmul_ru(mag, 1e-6f));
      live = fkey(ub) >= thr_fnow();
    }
    live = admit(id, live);  // every id scored exactly at most once
    if constexpr ((FPP_NS_PF & 2) != 0) {  // the row's lines on their way to L2 before exact_fold
      if (live)
        for (uint32_t c = 0; c < nch; ++c) prefetch_l2(X + (uint64_t)id * ldx + c * 32);
    }
    push_exact(id, live);
    if (lane == 0) cnt_s[w][0] += cnt;
  };

  // ---------------------------------------------------------------- stage 1
  // A per-warp ring of NS_RING batches: the 32 stage-1 records of batch i + RING - 1
  // move by cp.async (16 B per lane, four per lane) while batch i is bounded, so
  // RING - 1 batches (6 KB) per warp are in flight without holding registers.  The
  // candidate ids move the same way, RING batches ahead of their records, into an id
  // ring of IDR = 2 RING slots (one 4 B cp.async per lane -- from the lists, or from
  // the CSR at the walker's entries -- in the same commit group as the records of
  // iteration i).  Commit group i holds records(i + RING - 1) and
  // ids(i + 2 RING - 1); the wait for group i - RING at the end of iteration i - 1
  // covers both the records of batch i and the ids of batch i + RING - 1.
  const uint32_t nb = (Len + 31) / 32;
  const uint32_t nbw = nb > (uint32_t)w ? (nb - w + NW - 1) / NW : 0;  // this warp's batches
  // Slots are kept as wrapping counters (NS_RING = 3 is not a power of two: a modulo
  // per use was a multiply-shift sequence).  islot: an id-ring slot, rslot: a ring slot.
  auto ids_async = [&](uint32_t b, uint32_t islot) {  // lists: ids of batch b -> id ring
    if constexpr (!WALK) {
      const uint32_t ci = (w + b * NW) * 32 + lane;
      uint32_t* dst = idr + islot * 32 + lane;
      if (b < nbw && ci < Len) cp_async4(dst, cand + ci);
      else *dst = NONE;
    }
  };
  auto more = [&](uint32_t i) { return WALK ? !(wk_done && i >= nprod) : i < nbw; };
  auto issue = [&](uint32_t rslot, uint32_t islot) {  // records of a batch (ids in the id ring)
    const uint32_t slot = rslot;
    const uint32_t id = idr[islot * 32 + lane];
#pragma unroll
    for (int it = 0; it < 2; ++it) {  // record r = it * 16 + g16, 16 B part p2 per lane
      const uint32_t r = it * 16 + g16;
      const uint32_t idv = __shfl_sync(FULL, id, r);
      if (idv != NONE)
        cp_async16s(ring_sa + (slot * NS_SLOT + r * 2 + p2) * 16, rec + (uint64_t)idv * 2 + p2);
    }
  };
  // WALK: the walker's next window -> batch b's slot: its ids (4 B cp.async per lane
  // from the CSR ids) and its stage-1 records, inline in CSR order (a.csrrec: the
  // window's entries are runs of consecutive records, so the copies are coalesced and
  // whole 128 B lines are used), one commit group
  // this lane's record address in ring slot 0 (shared window); kept opaque per iteration
  // so it stays in a register instead of being rebuilt from tid / the window base
  uint32_t my_sa = ring_sa + lane * 32;
  auto produce = [&](uint32_t slot) {
    uint64_t gp = 0;
    const bool v = wk_step(gp);
    // a lane without an entry marks its own record slot empty (id NONE; the lane reads
    // it back itself, so no ordering beyond program order is needed)
    const uint32_t sa = my_sa + slot * (NS_SLOT * 16);  // this lane's record in the slot
    if (!v) asm volatile("st.shared.v4.u32 [%0+16], {%1, %2, %1, %1};" ::"r"(sa), "r"(0u), "r"(NONE) : "memory");
    const uint4* cr = reinterpret_cast<const uint4*>(a.csrrec);
    if constexpr (NS_TMA) {
      // the window's valid lanes are a prefix, split into runs of consecutive CSR
      // entries (one bucket each): one bulk copy per run (TMA), completing on the
      // slot's mbarrier; the slot's previous generic-proxy use (exact staging) is
      // fenced first
      const uint64_t gprev = __shfl_up_sync(FULL, gp, 1);
      const uint32_t starts = __ballot_sync(FULL, v && (lane == 0 || gp != gprev + 1));
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      const uint32_t vm = __ballot_sync(FULL, v);
      if (lane == 0) mbar_arrive_tx(&smbar[w][slot], (uint32_t)__popc(vm) * 32u);
      __syncwarp();
      if ((starts >> lane) & 1u) {
        const uint32_t after = starts & ~((2u << lane) - 1u);  // later run starts
        const uint32_t end = after ? (uint32_t)(__ffs(after) - 1) : (uint32_t)__popc(vm);
        bulk_g2s(ring + slot * NS_SLOT + lane * 2, cr + gp * 2, (end - lane) * 32u, &smbar[w][slot]);
      }
      return;
    }
    if (v) {  // each lane copies its own record (2 x 16 B: no address shuffles)
      cp_async16s(sa, cr + gp * 2);
      cp_async16s(sa + 16, cr + gp * 2 + 1);
    }
  };
  if constexpr (WALK) {
    wk_begin(1);
    nrows = wk_tot;  // (the seeds' entries; subtracted below)
#pragma unroll
    for (uint32_t j = 0; j + 1 < NS_RING; ++j) {
      produce(j);
      cp_commit();
    }
  } else {
    for (uint32_t b = 0; b < NS_RING; ++b) ids_async(b, b);
    cp_commit();
    cp_wait<0>();
    __syncwarp();
#pragma unroll
    for (uint32_t j = 0; j + 1 < NS_RING; ++j) {
      issue(j, j);
      ids_async(j + NS_RING, j + NS_RING);
      cp_commit();
    }
  }
  // batch i: ring slot cs = i % RING, id-ring slot ci = i % IDR; the refill of this
  // iteration goes to ring slot (i + RING - 1) % RING (the slot consumed last), its ids
  // from id-ring slot (i + RING - 1) % IDR, and the ids of batch i + 2 RING - 1 to
  // id-ring slot (i - 1) % IDR
  uint32_t cs = 0, ci = 0;
  for (uint32_t i = 0; more(i); ++i) {
    asm volatile("" : "+r"(my_sa));
    const uint32_t ps = cs == 0 ? NS_RING - 1 : cs - 1;
    // full queues are drained first (their own loads; the ring stays in flight)
    float* const stg = stg0;
    if (qtail - qhead >= 32) {
      __syncwarp();
      exact_batch(32, stg);
    }
    if (t1 - h1 >= 32) stage2_batch(32);
    __syncwarp();  // (the staging slot's readers are done before its refill)
    if constexpr (WALK) {
      produce(ps);
    } else {
      const uint32_t pi = ci + NS_RING - 1 < NS_IDR ? ci + NS_RING - 1 : ci + NS_RING - 1 - NS_IDR;
      issue(ps, pi);   // (an empty commit past the end keeps the count)
      ids_async(i + 2 * NS_RING - 1, ci == 0 ? NS_IDR - 1 : ci - 1);
    }
    if constexpr (WALK && NS_TMA) {
      mbar_wait(&smbar[w][cs], (mph >> cs) & 1u);
      mph ^= 1u << cs;
    } else {
      cp_commit();
      cp_wait<NS_RING - 1>();
      __syncwarp();
    }
    const uint32_t slot = cs;
    Recs cur;
    if constexpr (WALK) {
      const uint32_t ca = my_sa + slot * (NS_SLOT * 16);
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(cur.r[0].x), "=r"(cur.r[0].y), "=r"(cur.r[0].z), "=r"(cur.r[0].w) : "r"(ca));
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+16];"
                   : "=r"(cur.m.x), "=r"(cur.m.y), "=r"(cur.m.z), "=r"(cur.m.w) : "r"(ca));
    } else {
      cur.r[0] = ring[slot * NS_SLOT + lane * 2];
      cur.m = ring[slot * NS_SLOT + lane * 2 + 1];
    }
    const uint32_t cid = WALK ? cur.m.y : idr[ci * 32 + lane];  // (WALK: the record's id)
    cs = cs + 1 == NS_RING ? 0 : cs + 1;
    ci = ci + 1 == NS_IDR ? 0 : ci + 1;
    float tx, nx;
    // the query codes re-read from shared memory per batch (a broadcast LDS.128 + LDS:
    // hoisted into registers they were spilled under the 80-register cap)
    int4 qa;
    int qa4;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%5];\n\tld.shared.s32 %4, [%5+16];"
                 : "=r"(qa.x), "=r"(qa.y), "=r"(qa.z), "=r"(qa.w), "=r"(qa4)
                 : "r"((uint32_t)__cvta_generic_to_shared(&q8_s[0][0])));
    const float A1 = stageA_bound(cur, tx, nx, qa, qa4);
    // (branch-free: lanes without an entry compute on the empty record and drop out
    // at the compare; ||q|| terms re-read from shared memory: kept in registers they
    // were spilled)
    const float qh1 = *(volatile float*)&qn_s[0][1], qt1v = *(volatile float*)&qn_s[0][3];
    const float N1 = __fmul_ru(__fadd_ru(nx, tx), __fadd_ru(qh1, qt1v));  // >= ||x|| ||q||
    const float mag = __fadd_ru(fabsf(A1), N1);
    const float ub = __fadd_ru(__fmaf_ru(tx, qt1v, A1), __fmul_ru(mag, 1e-6f));
    const bool live = cid != NONE && fkey(ub) >= thr_fnow();
    const uint32_t live_m = __ballot_sync(FULL, live);
    if (live) {
      const uint32_t pos = (t1 + __popc(live_m & lt_mask)) % NS_QCAP;
      s1q[pos] = cid;
      s1v[pos] = make_float2(A1, N1);
      // its stage-B record (one 128 B line) on its way to L2 before stage2_batch reads it
      if constexpr ((FPP_NS_PF & 1) != 0) prefetch_l2(rec + ((uint64_t)a.n * 2 + (uint64_t)cid * 8));
    }
    t1 += __popc(live_m);
    if constexpr (!WALK) nrows += __popc(__ballot_sync(FULL, cid != NONE));  // (WALK: chunk totals)
    __syncwarp();  // slot i % RING is refilled by the next iteration's issue
  }
  if constexpr (WALK && NS_TMA) {  // the RING - 1 windows produced past the end (empty)
#pragma unroll
    for (int j = 0; j + 1 < NS_RING; ++j) {
      mbar_wait(&smbar[w][cs], (mph >> cs) & 1u);
      mph ^= 1u << cs;
      cs = cs + 1 == NS_RING ? 0 : cs + 1;
    }
  }
  cp_wait<0>();
  __syncwarp();
  if constexpr (WALK) nrows = wk_tot - nrows;
  while (t1 != h1 || qtail != qhead) {
    if (t1 != h1 && qtail - qhead < 32) {
      stage2_batch(min(32u, t1 - h1));
    } else {
      __syncwarp();
      exact_batch(min(32u, qtail - qhead), stg0);
    }
  }
  if (lane == 0) {
    // bytes read: 32 B stage-A record per candidate, 128 B stage-B record per stage-A
    // survivor, and the exact rows
    const uint32_t nst2 = cnt_s[w][0], nex = cnt_s[w][1];
    const unsigned long long nfl = (unsigned long long)nex * nch * 32;  // exact row floats
    if (a.rbytes) atomicAdd(a.rbytes, nrows * 32ull + nst2 * 128ull + nfl * 4ull);
    if (a.dbg) {  // read fraction in row floats: records count as 8 and 32 floats
      atomicAdd(a.dbg, (unsigned long long)nrows);
      atomicAdd(a.dbg + 1, nrows * 8ull + nst2 * 32ull + nfl);
      atomicAdd(a.dbg + 2, (unsigned long long)nst2);
      atomicAdd(a.dbg + 3, (unsigned long long)nex);
    }
  }
  // CTA merge of the warp lists
  mg_s[w][lane] = bs;
  mg_i[w][lane] = bi;
  __syncthreads();
  if (w == 0) {
    for (int w2 = 1; w2 < NW; ++w2) {
      const bool valid = (uint32_t)lane < k && mg_i[w2][lane] != NONE;
      topk_insert(bs, bi, k, mg_s[w2][lane], mg_i[w2][lane], valid);
    }
    if ((uint32_t)lane < k) {
      const bool ok = bi != NONE;
      a.out_ids[(uint64_t)q * k + lane] = ok ? bi + a.id_offset : NONE;
      a.out_scores[(uint64_t)q * k + lane] = ok ? bs : -INFINITY;
    }
    if (lane == 0 && a.stats) {
      a.stats[q].probes = a.peff;
      a.stats[q].entries = a.eq[q];
      a.stats[q].candidates = a.uq_all ? a.uq_all[q] : Len;
      a.stats[q].exact = a.uq_all ? a.uq_all[q] : Len;
    }
  }
  if (a.gbm) {  // leave the visited bitmap clear for the next query
    uint32_t* const bm = bm_of();
    const uint32_t* const wlog = wlog_of();
    __syncthreads();
    const uint32_t nl = logn_s;
    if (nl > a.logcap) {  // log overflow (pathological survivor counts): clear it all
      for (uint32_t i = threadIdx.x; i < a.nwords; i += blockDim.x) bm[i] = 0;
    } else {
      for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) bm[wlog[i] >> 5] = 0;
    }
    __syncthreads();
  }
  }  // queries
}

static size_t screen_smem(uint32_t d, bool walk) {
  const uint32_t nch = (d + 31) / 32;
  return (size_t)nch * 32 * 8 + (size_t)NS_W * (NS_RING * NS_SLOT + NS_STG) * 16 +
         (walk ? (size_t)0 : (size_t)NS_W * NS_IDR * 32 * 4) + (size_t)NS_W * NS_QCAP * (4 + 4 + 8);
}

static size_t score_smem(uint32_t d, int sl, int st) {
  return ((d * 8 + 127) / 128) * 128 + (size_t)SC_WARPS * st * 32 * (sl + 4) * 4;
}

// ------------------------------------------------------------ host driver
void launch_query_lists(const Index& ix, const float* Qd, uint64_t nq, uint32_t s_cap,
                        float* vals, uint32_t* codes, cudaStream_t s, uint64_t lstride) {
  if (!lstride) lstride = (uint64_t)ix.prm.L * ix.prm.K * s_cap;
  if (nq == 0) return;
  const uint32_t d = ix.d, D = ix.prm.D, K = ix.prm.K, L = ix.prm.L;
  const uint32_t G = ix.P < 32 ? 1 : ix.P / 32;
  // sub-batches keep nq * L * K * G < 2^31 (32-bit index math in the kernel)
  const uint64_t qmax = std::max<uint64_t>(1, ((1ull << 31) - 1) / ((uint64_t)L * K * G));
  if (nq > qmax) {
    for (uint64_t q0 = 0; q0 < nq; q0 += qmax)
      launch_query_lists(ix, Qd + q0 * d, std::min(qmax, nq - q0), s_cap, vals + q0 * lstride,
                         codes + q0 * lstride, s, lstride);
    return;
  }
  const unsigned grid = (unsigned)((nq * L * K * G + 127) / 128);
  // preselection width: the smallest of P/4, P/2 leaving a margin of P/16 above
  // nat = min(s, D) (0 = sort all P keys)
  const uint32_t nat = std::min(s_cap, D), P = ix.P;
  // (margin P/32 for P = 1024: C3's nat = 200 then sorts 256 of 1024 keys, not 512)
  const uint32_t marg = P >= 1024 ? P / 32 : P / 16;
  const int ns = P < 256 ? 0 : (nat + marg <= P / 4 ? 4 : (nat + marg <= P / 2 ? 2 : 0));
#define FPP_QL_LAUNCH(PP, NSV) \
  k_query_lists<PP, NSV><<<grid, 128, 0, s>>>(Qd, nq, d, D, K, ix.signs, L, s_cap, lstride, vals, codes)
#define FPP_QL_CASE(PP)         \
  case PP:                      \
    FPP_QL_LAUNCH(PP, 0);       \
    break;
#define FPP_QL_CASE_NS(PP)                         \
  case PP:                                         \
    if (ns == 4) FPP_QL_LAUNCH(PP, PP / 4);        \
    else if (ns == 2) FPP_QL_LAUNCH(PP, PP / 2);   \
    else FPP_QL_LAUNCH(PP, 0);                     \
    break;
  switch (ix.P) {
    FPP_QL_CASE(2) FPP_QL_CASE(4) FPP_QL_CASE(8) FPP_QL_CASE(16) FPP_QL_CASE(32)
    FPP_QL_CASE(64) FPP_QL_CASE(128) FPP_QL_CASE_NS(256) FPP_QL_CASE_NS(512) FPP_QL_CASE_NS(1024)
    default: fail(FPP_ERR_UNSUPPORTED, "query: padded dimension > 1024 not supported on GPU");
  }
#undef FPP_QL_CASE_NS
#undef FPP_QL_LAUNCH
#undef FPP_QL_CASE
  FPP_LAUNCH();
}

static int co_smem_max() { return smem_optin_max(); }

// Stage A of one chunk on stream `st`: query hashing, probe selection,
// candidate offsets; the total candidate count is copied to the slot's pinned
// word and ev_probe recorded.
static uint32_t cand_cap(const Index& ix, uint32_t qprobes) {
  const uint64_t peff = query_probes(ix, qprobes);
  const uint64_t scap = query_cap(ix, qprobes);
  return (uint32_t)std::min<uint64_t>(std::max<uint64_t>(4 * peff + 4096, 16384),
                                      (uint64_t)ix.prm.L * ix.prm.K * scap * scap);
}

using QSlot = QueryCtx::QSlot;

// size a slot's chunk buffers for up to nqc queries (before any launch uses it)
static void prepare_slot(const Index& ix, QSlot& sl, uint32_t nqc, uint32_t qprobes) {
  const uint64_t LKs = (uint64_t)ix.prm.L * ix.prm.K * query_cap(ix, qprobes);
  const uint64_t lstride = (LKs + 3) & ~3ull;
  const uint64_t peff = query_probes(ix, qprobes);
  const uint32_t ccap = cand_cap(ix, qprobes);
  sl.vals.ensure((size_t)nqc * lstride);
  sl.codes.ensure((size_t)nqc * lstride);
  sl.ppos.ensure((size_t)nqc * peff);
  sl.plen.ensure((size_t)nqc * peff);
  sl.gbuf.ensure((size_t)nqc * peff);
  sl.ckey.ensure((size_t)nqc * ccap);
  sl.cpair.ensure((size_t)nqc * ccap);
  sl.eq.ensure(nqc);
  sl.uq.ensure(nqc);
  sl.coff.ensure((size_t)nqc + 1);
  sl.counter.ensure(4);
}

static void stage_a(const Index& ix, QueryCtx& cx, QSlot& sl, const float* Qd, uint32_t nqc,
                    uint32_t qprobes, cudaStream_t st, uint64_t* dbg_probes,
                    uint32_t* probes_out = nullptr) {
  const uint32_t L = ix.prm.L, K = ix.prm.K;
  const uint32_t scap = query_cap(ix, qprobes);
  const uint64_t peff = query_probes(ix, qprobes);
  const uint64_t LKs = (uint64_t)L * K * scap;
  const uint64_t lstride = (LKs + 3) & ~3ull;  // 16-byte aligned per-query blocks
  prepare_slot(ix, sl, nqc, qprobes);

  cudaEvent_t e0;
  cx.timer.begin(PH_QHASH, st, &e0);
  launch_query_lists(ix, Qd, nqc, scap, sl.vals.p, sl.codes.p, st, lstride);
  cx.timer.end(PH_QHASH, e0, st);

  cx.timer.begin(PH_PROBE, st, &e0);
  const uint32_t ccap = cand_cap(ix, qprobes);
  ProbeArgs pa{sl.vals.p, sl.codes.p, nqc, L, K, scap, ix.prm.D, ix.NB, peff, ix.offsets,
               ix.table_base, sl.ppos.p, sl.plen.p, sl.eq.p, dbg_probes, sl.gbuf.p, lstride,
               nullptr, sl.ckey.p, sl.cpair.p, ccap, 0};
  // first T_lo attempt at arm rank 0.7 m (no re-walks on C2; FPP_PS_BETA overrides,
  // e.g. tests force the exact re-walk fallback with a low beta)
  const char* beta_env = getenv("FPP_PS_BETA");
  pa.beta_q8 = beta_env ? (uint32_t)(atof(beta_env) * 256) : 179u;
  // table-major probe order only on request: the walk measured the same either way and
  // the sort's 50-counter atomics cost ~1 ms of probe selection per C4 step
  static const bool table_major = getenv("FPP_PROBE_TABLEMAJOR") != nullptr;
  pa.rank_order = table_major ? 0u : 1u;
  pa.pout = probes_out;
  static const bool dbg_probe = getenv("FPP_DEBUG_PROBE") != nullptr;
  if (dbg_probe) {
    sl.dbgclk.ensure((size_t)nqc * 16);
    pa.dbg_clk = reinterpret_cast<long long*>(sl.dbgclk.p);
  }
  if (ix.prm.mode == FPP_MODE_FALCONN_BASELINE) k_probe_select<1><<<nqc, PS_THREADS, 0, st>>>(pa);
  else k_probe_select<0><<<nqc, PS_THREADS, 0, st>>>(pa);
  FPP_LAUNCH();
  if (dbg_probe) {
    std::vector<long long> h((size_t)nqc * 16);
    FPP_CUDA(cudaMemcpyAsync(h.data(), pa.dbg_clk, h.size() * 8, cudaMemcpyDeviceToHost, st));
    FPP_CUDA(cudaStreamSynchronize(st));
    double acc[6] = {0}, fl = 0, cn = 0, ti = 0, rf = 0;
    for (uint32_t i = 0; i < nqc; ++i) {
      for (int j = 0; j < 6; ++j) acc[j] += (double)(h[i * 16 + j + 1] - h[i * 16 + j]);
      fl += (double)h[i * 16 + 8];
      cn += (double)h[i * 16 + 9];
      ti += (double)h[i * 16 + 10];
      rf += (double)h[i * 16 + 11];
    }
    fprintf(stderr, "[probe dbg] per query cycles: arms %.0f materialise %.0f radix %.0f ties %.0f "
            "emit %.0f resolve %.0f | flat %.2f candidates %.1f ties %.2f re-walks %.4f\n",
            acc[0] / nqc, acc[1] / nqc, acc[2] / nqc, acc[3] / nqc, acc[4] / nqc, acc[5] / nqc,
            fl / nqc, cn / nqc, ti / nqc, rf / nqc);
  }
  k_scan_eq<<<1, 1024, 0, st>>>(sl.eq.p, nqc, sl.coff.p);
  FPP_LAUNCH();
  FPP_CUDA(cudaMemcpyAsync(sl.pinned, sl.coff.p + nqc, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  cx.timer.end(PH_PROBE, e0, st);
  cx.acc.launches += 3;  // lists, probe_select, scan_eq
  FPP_CUDA(cudaEventRecord(sl.ev_probe, st));
}

// grouped-dedup geometry for an index of n points: id >> gshift < CO_NG; 0 when the
// per-warp range bitmaps (32 x 2^gshift bits) would not fit shared memory
static uint32_t grouped_shift(uint64_t n) {
  uint32_t gs = 10;  // >= 1024-id groups: 128-word per-warp bitmaps at least
  while (gs < 32 && ((n - 1) >> gs) >= CO_NG) ++gs;
  const size_t sm = (size_t)CO_NG * 4 + (size_t)32 * ((1ull << gs) / 8);
  return sm + 64 <= (size_t)co_smem_max() ? gs : 0u;
}

// Index::q8csr: entry e's stage-A record = q8rec[ids[e]] (two threads per entry, 16 B
// each) with the entry's id in the id slot, so the walking screen reads the id with
// the record and no separate ids stream
__global__ void k_q8_inline(const uint4* __restrict__ rec, const uint32_t* __restrict__ ids,
                            uint64_t kept, uint4* __restrict__ out) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < kept * 2;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = __ldg(ids + (t >> 1));
    uint4 v = __ldg(rec + (uint64_t)id * 2 + (t & 1));
    if (t & 1) v.y = id;
    out[t] = v;
  }
}

static void ensure_q8csr(const Index& ix) {
  std::lock_guard<std::mutex> lk(ix.mu);
  if (ix.q8csr || !ix.q8rec) return;
  uint4* p = static_cast<uint4*>(dmalloc((size_t)(ix.kept_total + 1) * 32));
  if (ix.kept_total) {
    k_q8_inline<<<sm_count() * 8, 256, 0, ix.stream>>>(ix.q8rec, ix.ids, ix.kept_total, p);
    FPP_LAUNCH();
  }
  FPP_CUDA(cudaStreamSynchronize(ix.stream));  // (one-time; later calls read it on any stream)
  ix.q8csr = p;
}

// zero-initialised on (re)allocation; every kernel using it leaves it clear
static uint32_t* slot_bitmap(QSlot& sl, size_t words, cudaStream_t st) {
  if (sl.bitmap.n < words) {
    sl.bitmap.alloc(words);
    FPP_CUDA(cudaMemsetAsync(sl.bitmap.p, 0, words * 4, st));
  }
  return sl.bitmap.p;
}

constexpr uint32_t WK_LOGCAP = 16384;  // per-CTA log of ids admitted to the exact stage

// Stage B on stream `st`: bucket walk + dedup, then row gather + fp64 dot + top-k.
// The collect pass needs the slot's candidate total on the host (it sizes the
// lists): it waits for stage A's readback.  The walking screen kernel (narrow rows
// with screening records) needs no lists and no host sync; it still runs the
// collect when per-query stats (unique candidate counts) or the lists themselves
// (`lists`: fpp_query_debug) are requested.
static void stage_b(const Index& ix, QueryCtx& cx, QSlot& sl, const float* Qd, uint32_t nqc,
                    uint32_t k, uint32_t qprobes, uint32_t* ids_d, double* scores_d,
                    fpp_query_stats* stats_d, cudaStream_t st, uint32_t rerank = 0,
                    bool lists = false) {
  const uint64_t peff = query_probes(ix, qprobes);
  const uint32_t nwords = (uint32_t)((ix.n + 31) / 32);
  // score policy first: exact early termination (k_score_pruned / k_score_screen)
  // when the index has tail norms (d > 64) and the bound pays on this data: the read
  // fraction (row slices read / all) is probed on the first chunk and every 16th after
  // (async readback); above 0.65 the job overhead outweighs the saved bytes (C1 iid:
  // 1.0, 1.36x slower; C3: 0.77, 1.2x slower; C2: 0.33, 2.1x faster) and k_score runs.
  // FPP_NO_PRUNE=1 / FPP_PRUNE=1 force either; FPP_DEBUG_PRUNE=1 prints every chunk's
  // fraction.
  const bool no_prune = getenv("FPP_NO_PRUNE") != nullptr;
  const bool force_prune = getenv("FPP_PRUNE") != nullptr;
  const bool dbg = getenv("FPP_DEBUG_PRUNE") != nullptr;
  bool use_pruned = false, probe = false;
  // k > 32: the warp lists hold 32 ranks, so k_score keeps ranks [0, 32), dumps every
  // exact score, and k_topk_more selects the later ranks from the dump
  const bool bigk = k > 32;
  if (ix.xt_n && !no_prune && !bigk) {
    std::lock_guard<std::mutex> lk(ix.mu);  // the index-wide policy (concurrent calls)
    if (cx.prune_pending && cudaEventQuery(cx.prune_ev) == cudaSuccess) {
      if (cx.prune_h[0]) ix.prune_frac = (double)cx.prune_h[1] / ((double)cx.prune_h[0] * ix.d);
      cx.prune_pending = false;
    }
    probe = dbg || (!cx.prune_pending && (ix.prune_frac < 0 || ix.prune_chunks % 16 == 0));
    use_pruned = force_prune || probe || ix.prune_frac < 0 || ix.prune_frac <= 0.65;
    ++ix.prune_chunks;
  }
  // narrow rows: the record screen (k_score_screen) unless FPP_SC_NARROW=0.  It walks
  // the probes itself (no collect pass and no host sync; C4: 231 ms per step against
  // 97 + 148 ms for collect + the screen over the collect's id-ordered lists, which
  // FPP_SC_WALK=0 selects).  With stats requested the collect still runs, for the
  // unique candidate counts.
  static const bool narrow_off = getenv("FPP_SC_NARROW") && atoi(getenv("FPP_SC_NARROW")) == 0;
  static const bool walk_on = !(getenv("FPP_SC_WALK") && atoi(getenv("FPP_SC_WALK")) == 0);
  const bool screen = use_pruned && ix.q8rec && !narrow_off && !rerank;
  const bool walk = screen && walk_on && !lists;
  const bool collect = !walk || stats_d != nullptr;
  cudaEvent_t e0;
  sl.uniq.ensure(nqc);
  CollectArgs ca{sl.ppos.p, sl.plen.p, peff, ix.ids, sl.coff.p, sl.cands.p, sl.uq.p,
                 nqc, nwords, nullptr, sl.counter.p, 0, 0, sl.uniq.p, ix.n};
  uint64_t etot = 0;
  if (collect) {
  FPP_CUDA(cudaEventSynchronize(sl.ev_probe));  // the candidate total (stage A readback)
  etot = sl.pinned[0];
  sl.cands.ensure(etot + 1);
  ca.cands = sl.cands.p;
  cx.timer.begin(PH_COLLECT, st, &e0);
  // Visited set (every id scored once): an n-bit bitmap in shared memory
  // where it fits one SM (n <= ~1.8 M); beyond that the grouped dedup (id-range
  // counting sort + per-warp range bitmaps; C4's 10 M points); beyond its range an
  // 8-CTA DSMEM cluster bitmap or per-CTA global bitmaps.  All emit ascending ids.
  // FPP_FORCE_COLLECT=grouped|cluster|global selects a large-shard path at any n (tests).
  const char* force = getenv("FPP_FORCE_COLLECT");
  const bool f_grouped = force && !strcmp(force, "grouped");
  const bool f_sliced = force && !strcmp(force, "sliced");
  const bool f_cluster = force && !strcmp(force, "cluster"), f_global = force && !strcmp(force, "global");
  const size_t static_co = 64;
  const int sms = sm_count();
  const uint32_t slice_words = (nwords + CO_CLUSTER - 1) / CO_CLUSTER;
  const uint32_t gshift = grouped_shift(ix.n);
  unsigned co_grid;
  if (!force && (size_t)nwords * 4 + static_co <= (size_t)co_smem_max()) {
    const size_t co_smem = (size_t)nwords * 4;
    allow_dynamic_smem(k_collect);
    int occ = 1;
    FPP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_collect, CO_THREADS, co_smem));
    co_grid = (unsigned)std::min<uint64_t>(nqc, (uint64_t)sms * std::max(occ, 1));
    FPP_CUDA(cudaMemsetAsync(sl.counter.p, 0, sizeof(uint32_t), st));
    k_collect<<<co_grid, CO_THREADS, co_smem, st>>>(ca);
  } else if ((!force || f_grouped) && gshift && !rerank) {
    // (the SimHash screen needs hole-free lists: rerank takes the bitmap paths below)
    ca.grouped = 1;
    ca.gshift = gshift;
    const size_t co_smem = (size_t)CO_NG * 4 + (size_t)32 * ((1ull << gshift) / 8);
    allow_dynamic_smem(k_collect);
    int occ = 1;
    FPP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_collect, CO_THREADS, co_smem));
    co_grid = (unsigned)std::min<uint64_t>(nqc, (uint64_t)sms * std::max(occ, 1));
    FPP_CUDA(cudaMemsetAsync(sl.counter.p, 0, sizeof(uint32_t), st));
    k_collect<<<co_grid, CO_THREADS, co_smem, st>>>(ca);
  } else if ((!force || f_sliced) && ((ix.n - 1) >> CO_SLICE_BITS) < CO_NG &&
             (size_t)CO_NG * 4 + (4ull << (CO_SLICE_BITS - 5)) + 64 <= (size_t)co_smem_max()) {
    // sliced bitmap dedup: unique ids in ascending order (beyond the grouped range;
    // on C4 it measured slower than grouped: 118 vs 97 ms per step)
    ca.sliced = 1;
    ca.gshift = CO_SLICE_BITS;
    const size_t co_smem = (size_t)CO_NG * 4 + (4ull << (CO_SLICE_BITS - 5));
    allow_dynamic_smem(k_collect);
    int occ = 1;
    FPP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_collect, CO_THREADS, co_smem));
    co_grid = (unsigned)std::min<uint64_t>(nqc, (uint64_t)sms * std::max(occ, 1));
    FPP_CUDA(cudaMemsetAsync(sl.counter.p, 0, sizeof(uint32_t), st));
    k_collect<<<co_grid, CO_THREADS, co_smem, st>>>(ca);
  } else if (!f_global && (size_t)slice_words * 4 + static_co <= (size_t)co_smem_max()) {
    // bitmap split over a CO_CLUSTER-CTA cluster (DSMEM)
    const size_t sm = (size_t)slice_words * 4;
    allow_dynamic_smem(k_collect_cluster);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CO_CLUSTER);
    cfg.blockDim = dim3(CO_CL_THREADS);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    int ncl = 0;
    FPP_CUDA(cudaOccupancyMaxActiveClusters(&ncl, k_collect_cluster, &cfg));
    ncl = std::max(1, std::min<int>(ncl, (int)nqc));
    k_collect_cluster<<<ncl * CO_CLUSTER, CO_CL_THREADS, sm, st>>>(ca, slice_words);
  } else {
    co_grid = (unsigned)std::min<uint64_t>(nqc, (uint64_t)sms * 2);
    ca.gbitmap = slot_bitmap(sl, (size_t)co_grid * nwords, st);
    FPP_CUDA(cudaMemsetAsync(sl.counter.p, 0, sizeof(uint32_t), st));
    k_collect<<<co_grid, CO_THREADS, 0, st>>>(ca);
  }
  FPP_LAUNCH();
  cx.timer.end(PH_COLLECT, e0, st);
  cx.acc.launches += 1;
  }  // collect

  cx.timer.begin(PH_SCORE, st, &e0);
  ScoreArgs sa{ix.X, ix.d, ix.ldx, Qd, sl.coff.p, sl.cands.p, sl.uq.p, sl.eq.p, peff, k,
               ix.prm.id_offset, ids_d, scores_d, stats_d, nullptr, 0};
  sa.rbytes = ix.score_bytes_d.p;
  if (ca.grouped) sa.uq_all = sl.uniq.p;  // lists carry holes: unique counts for the stats
  else if (walk && collect) sa.uq_all = sl.uq.p;  // (the walking kernel reads no lists)
  if (rerank) {  // SimHash screen: at most B candidates per query reach the exact scores
    sa.uq_all = nullptr;
    sl.qsig.ensure(nqc);
    sl.cands2.ensure((size_t)nqc * rerank);
    sl.uq2.ensure(nqc);
    launch_signatures(ix, Qd, nqc, ix.d, sl.qsig.p, st);
    k_screen<<<nqc, SCR_THREADS, 0, st>>>(sl.cands.p, sl.coff.p, sl.uq.p, ix.sigs, sl.qsig.p, rerank,
                                          sl.cands2.p, sl.uq2.p);
    FPP_LAUNCH();
    cx.acc.launches += 2;
    sa.cands = sl.cands2.p;
    sa.uq = sl.uq2.p;
    sa.uq_all = sl.uq.p;
    sa.cstride = rerank;
  }
  // FPP_SC_CTAS=c: persistent grid of c CTAs per SM fetching queries from a counter,
  // so the remaining SM resources stay free for the next chunk's stage A
  static const int sc_ctas = getenv("FPP_SC_CTAS") ? atoi(getenv("FPP_SC_CTAS")) : 0;
  sa.nq = nqc;
  if (bigk) {
    sl.allsc.ensure(rerank ? (size_t)nqc * rerank : (size_t)etot + 1);
    sa.allsc = sl.allsc.p;
    sa.ostride = k;
    sa.k = 32;
  }
  auto launch_score = [&](auto kern, int slice, int stg) {
    const size_t sm = score_smem(ix.d, slice, stg);
    allow_dynamic_smem(kern);
    unsigned grid = nqc;
    if (sc_ctas > 0 && (uint64_t)sm_count() * sc_ctas < nqc) {
      grid = (unsigned)(sm_count() * sc_ctas);
      sa.qctr = sl.counter.p + 1;
      FPP_CUDA(cudaMemsetAsync(sa.qctr, 0, sizeof(uint32_t), st));
    }
    kern<<<grid, SC_WARPS * 32, sm, st>>>(sa);
  };
  // ring geometry: 64-float slices x 2 stages, 3 CTAs per SM for d >= 64 (with the
  // ascending-id candidate lists more queries in flight share more rows in L2:
  // C2 96x2 @ 2/SM 344k -> 64x2 @ 3/SM 352k q/s; C4 +5%); 32 x 4 below
  const bool wide = ix.d >= 64;
  if (screen) {
    sa.xtail = reinterpret_cast<const float*>(ix.q8rec);
    sa.n = ix.n;
    if (probe) {
      if (!cx.prune_h) {
        FPP_CUDA(cudaMallocHost(&cx.prune_h, 32));
        FPP_CUDA(cudaEventCreateWithFlags(&cx.prune_ev, cudaEventDisableTiming));
        cx.prune_d.alloc(4);
      }
      FPP_CUDA(cudaMemsetAsync(cx.prune_d.p, 0, 32, st));
      sa.dbg = cx.prune_d.p;
    }
    // seeds: the true buckets (the first L probes); FPP_SC_SEEDS=0 disables
    static const bool no_seeds = getenv("FPP_SC_SEEDS") && atoi(getenv("FPP_SC_SEEDS")) == 0;
    sa.ppos = sl.ppos.p;
    sa.plen = sl.plen.p;
    sa.ids = ix.ids;
    sa.nseedp = no_seeds ? 0u : ix.prm.L;
    static const uint32_t seedcap =
        getenv("FPP_SC_SEEDCAP") ? (uint32_t)atoi(getenv("FPP_SC_SEEDCAP")) : WK_SEEDCAP;
    sa.seedcap = seedcap;
    const size_t sm = screen_smem(ix.d, walk);
    // 3 CTAs/SM (24 warps: 80 registers, a 3-batch ring and a 2048-slot admission hash
    // so three CTAs' shared memory fits): C4 533 vs 522 k q/s for 2 CTAs/SM with a
    // 4-batch ring; FPP_SC_SCR_MINB=2 selects the 2-CTA register budget
    static const int scr_minb = getenv("FPP_SC_SCR_MINB") ? atoi(getenv("FPP_SC_SCR_MINB")) : 3;
    auto launch_scr = [&](auto kern) {
      allow_dynamic_smem(kern);
      unsigned grid = nqc;
      if (walk) {  // persistent CTAs, one visited bitmap + admission log each
        ensure_q8csr(ix);
        sa.csrrec = ix.q8csr;
        int occ = 1;
        FPP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NS_W * 32, sm));
        grid = (unsigned)std::min<uint64_t>(nqc, (uint64_t)sm_count() * std::max(occ, 1));
        sa.gbm = slot_bitmap(sl, (size_t)grid * nwords, st);
        sa.nwords = nwords;
        sl.wlog.ensure((size_t)grid * WK_LOGCAP);
        sa.wlog = sl.wlog.p;
        sa.logcap = WK_LOGCAP;
        sa.qctr = sl.counter.p + 1;
        FPP_CUDA(cudaMemsetAsync(sa.qctr, 0, sizeof(uint32_t), st));
      }
      kern<<<grid, NS_W * 32, sm, st>>>(sa);
    };
    if (walk) {
      if (scr_minb == 2) launch_scr(k_score_screen<NS_W, 2, true>);
      else launch_scr(k_score_screen<NS_W, 3, true>);
    } else {
      if (scr_minb == 2) launch_scr(k_score_screen<NS_W, 2, false>);
      else launch_scr(k_score_screen<NS_W, 3, false>);
    }
    if (probe) {
      FPP_CUDA(cudaMemcpyAsync(cx.prune_h, cx.prune_d.p, 32, cudaMemcpyDeviceToHost, st));
      FPP_CUDA(cudaEventRecord(cx.prune_ev, st));
      cx.prune_pending = true;
      if (dbg) {
        FPP_CUDA(cudaEventSynchronize(cx.prune_ev));
        const unsigned long long* h = cx.prune_h;
        fprintf(stderr, "[prune dbg] screen: rows %llu, floats read per row %.1f of %u (%.1f%% of row bytes); "
                "stage-2 records %llu (%.2f%%), exact rows %llu (%.2f%%)\n",
                h[0], h[0] ? (double)h[1] / h[0] : 0.0, ix.d, h[0] ? 100.0 * h[1] / h[0] / ix.d : 0.0,
                h[2], h[0] ? 100.0 * h[2] / h[0] : 0.0, h[3], h[0] ? 100.0 * h[3] / h[0] : 0.0);
      }
    }
  } else if (use_pruned) {
    sa.xtail = ix.xtail;
    sa.xt_n = ix.xt_n;
    sa.xt_head = ix.xt_head;
    sa.n = ix.n;
    if (probe) {
      if (!cx.prune_h) {
        FPP_CUDA(cudaMallocHost(&cx.prune_h, 32));
        FPP_CUDA(cudaEventCreateWithFlags(&cx.prune_ev, cudaEventDisableTiming));
        cx.prune_d.alloc(4);
      }
      FPP_CUDA(cudaMemsetAsync(cx.prune_d.p, 0, 32, st));
      sa.dbg = cx.prune_d.p;
    }
    // ring geometry (FPP_SC_PR = NW,ST,MINB digits; default 4 warps x 2 stages, 3 CTAs/SM:
    // C2 score 8.0 ms vs 11.2 (4x3 @ 2/SM, kept for the tests), 12.9 (2x4 @ 3/SM) and
    // 20.7 (4x4 @ 1/SM))
    auto launch_pruned = [&](auto kern, int nw, int stg) {
      const size_t sm = (size_t)nw * stg * 32 * XT_SLICE * 4 + ((ix.d * 8 + 127) / 128) * 128;
      allow_dynamic_smem(kern);
      unsigned grid = nqc;
      if (sc_ctas > 0 && (uint64_t)sm_count() * sc_ctas < nqc) {
        grid = (unsigned)(sm_count() * sc_ctas);
        sa.qctr = sl.counter.p + 1;
        FPP_CUDA(cudaMemsetAsync(sa.qctr, 0, sizeof(uint32_t), st));
      }
      kern<<<grid, nw * 32, sm, st>>>(sa);
    };
    const char* prc = getenv("FPP_SC_PR");
    // narrow rows (32-float heads, d <= 192): 3-warp CTAs, 4 per SM (C4 score 411 -> 395
    // ms); wider rows: 4-warp CTAs, 3 per SM (C2 7.5 ms vs 8.8 with 3 warps)
    const int pr = prc ? atoi(prc) : (ix.xt_head == 32 ? 324 : 423);
    const bool vec = (ix.d & 3u) == 0;
    // FPP_SC_TMA=1: TMA bulk row copies instead of the cp.async ring.  Measured slower
    // (C2 score 12.4 vs 7.6 ms: 256 B bulk copies are TMA-issue bound), kept as an option
    const bool tma = getenv("FPP_SC_TMA") && atoi(getenv("FPP_SC_TMA")) != 0;
#define FPP_PR_CASE(NW_, ST_, MB_)                                                       \
  case NW_ * 100 + ST_ * 10 + MB_:                                                       \
    if (vec && tma) launch_pruned(k_score_pruned<true, NW_, ST_, MB_, true>, NW_, ST_);  \
    else if (vec) launch_pruned(k_score_pruned<true, NW_, ST_, MB_>, NW_, ST_);          \
    else launch_pruned(k_score_pruned<false, NW_, ST_, MB_>, NW_, ST_);                  \
    break;
    switch (pr) {
      FPP_PR_CASE(4, 3, 2)
      FPP_PR_CASE(3, 2, 4)
      default:
      FPP_PR_CASE(4, 2, 3)
    }
#undef FPP_PR_CASE
    if (probe) {
      FPP_CUDA(cudaMemcpyAsync(cx.prune_h, cx.prune_d.p, 32, cudaMemcpyDeviceToHost, st));
      FPP_CUDA(cudaEventRecord(cx.prune_ev, st));
      cx.prune_pending = true;
      if (dbg) {
        FPP_CUDA(cudaEventSynchronize(cx.prune_ev));
        const unsigned long long* h = cx.prune_h;
        fprintf(stderr, "[prune dbg] rows %llu, floats read per row %.1f of %u (%.1f%% of row bytes)\n",
                h[0], h[0] ? (double)h[1] / h[0] : 0.0, ix.d, h[0] ? 100.0 * h[1] / h[0] / ix.d : 0.0);
      }
    }
  } else if ((ix.d & 3u) == 0) {
    if (wide) launch_score(k_score<true, 64, 2, 3>, 64, 2);
    else launch_score(k_score<true, 32, 4>, 32, 4);
  } else {
    if (wide) launch_score(k_score<false, 64, 2, 3>, 64, 2);
    else launch_score(k_score<false, 32, 4>, 32, 4);
  }
  FPP_LAUNCH();
  if (bigk) {
    k_topk_more<<<nqc, TM_WARPS * 32, 0, st>>>(sa);
    FPP_LAUNCH();
    cx.acc.launches += 1;
  }
  cx.timer.end(PH_SCORE, e0, st);
  cx.acc.launches += 1;  // score (stage A: lists, probe_select, scan_eq)
  cx.acc.score_launches += 1;
  cx.acc.probes += peff * nqc;
}

static uint32_t chunk_size(const Index& ix, uint32_t qprobes, uint64_t nq) {
  const uint64_t LKs = (uint64_t)ix.prm.L * ix.prm.K * query_cap(ix, qprobes);
  const uint64_t pe = query_probes(ix, qprobes);
  const uint64_t per_q = LKs * 8 + pe * 16 + (4 * pe + 16384) * 8 + 64;
  // ~4 GB of per-chunk scratch per slot, at most 8192 queries (FPP_CHUNK_GB / FPP_CHUNK_MAX)
  static const uint64_t cgb = getenv("FPP_CHUNK_GB") ? std::max(1, atoi(getenv("FPP_CHUNK_GB"))) : 4;
  static const uint64_t cmax = getenv("FPP_CHUNK_MAX") ? std::max(1, atoi(getenv("FPP_CHUNK_MAX"))) : 8192;
  uint64_t c = (cgb << 30) / per_q;
  c = std::max<uint64_t>(1, std::min<uint64_t>(c, cmax));
  // at least 3 chunks when the batch allows, so the two-stream pipeline overlaps
  // (C2 sweep: 2 chunks 288k, 3 -> 300k, 4 -> 295k, 6 -> 290k, 8 -> 275k q/s);
  // FPP_CHUNKS overrides
  static const int nch_min = getenv("FPP_CHUNKS") ? std::max(1, atoi(getenv("FPP_CHUNKS"))) : 3;
  const uint64_t quarter = (nq + nch_min - 1) / nch_min;
  if (quarter >= 512) c = std::min(c, quarter);
  return (uint32_t)std::min<uint64_t>(c, nq);
}

// Two-stream software pipeline over query chunks: stage A (ALU/latency bound:
// hashing + probe selection) runs on a low-priority stream, stage B (HBM bound:
// collect + gather/score) on a high-priority one, so the scheduler hands freed
// SM slots to the bandwidth-bound kernel first and fills the rest with stage A
// of the next chunk.  Slots alternate; events order slot reuse.
static void run_query_core(const Index& ix, QueryCtx& cx, const float* Qd, uint64_t nq, uint32_t k,
                           uint32_t qprobes, uint32_t* ids_d, double* scores_d,
                           fpp_query_stats* stats_d, cudaStream_t s, uint32_t rerank) {
  const uint32_t cs = chunk_size(ix, qprobes, nq);
  const uint64_t nch = (nq + cs - 1) / cs;
  // Stage order: the two-stream pipeline pays where stage A is a large share (C2:
  // 19.6 vs 20.2 ms per step); the narrow-row screen kernel (rows with screening
  // records, C4) is L2-latency bound and loses to the overlapped stage A (327 vs 323
  // ms), so those indexes run the stages in stream order.  FPP_PIPELINE=0/1 forces
  // either (FPP_SERIAL=1 = serial).
  static const char* pe = getenv("FPP_PIPELINE");
  const bool serial = getenv("FPP_SERIAL") != nullptr ||
                      (pe ? atoi(pe) == 0 : ix.q8rec != nullptr);
  if (serial) {  // single-stream order (per-kernel timing without overlap)
    for (uint64_t c = 0; c < nch; ++c) {
      const uint64_t q0 = c * cs;
      const uint32_t n = (uint32_t)std::min<uint64_t>(cs, nq - q0);
      stage_a(ix, cx, cx.slot[0], Qd + q0 * ix.d, n, qprobes, s, nullptr);
      stage_b(ix, cx, cx.slot[0], Qd + q0 * ix.d, n, k, qprobes, ids_d + q0 * k, scores_d + q0 * k,
              stats_d ? stats_d + q0 : nullptr, s, rerank);
    }
    return;
  }
  prepare_slot(ix, cx.slot[0], cs, qprobes);
  prepare_slot(ix, cx.slot[1], cs, qprobes);
  FPP_CUDA(cudaEventRecord(cx.ev_fork, s));
  FPP_CUDA(cudaStreamWaitEvent(cx.sA, cx.ev_fork, 0));
  FPP_CUDA(cudaStreamWaitEvent(cx.sB, cx.ev_fork, 0));
  auto issue_a = [&](uint64_t c) {
    QSlot& sl = cx.slot[c & 1];
    if (c >= 2) FPP_CUDA(cudaStreamWaitEvent(cx.sA, sl.ev_bdone, 0));  // slot free again
    const uint64_t q0 = c * cs;
    const uint32_t n = (uint32_t)std::min<uint64_t>(cs, nq - q0);
    stage_a(ix, cx, sl, Qd + q0 * ix.d, n, qprobes, cx.sA, nullptr);
  };
  issue_a(0);
  if (nch > 1) issue_a(1);
  for (uint64_t c = 0; c < nch; ++c) {
    QSlot& sl = cx.slot[c & 1];
    FPP_CUDA(cudaStreamWaitEvent(cx.sB, sl.ev_probe, 0));
    const uint64_t q0 = c * cs;
    const uint32_t n = (uint32_t)std::min<uint64_t>(cs, nq - q0);
    stage_b(ix, cx, sl, Qd + q0 * ix.d, n, k, qprobes, ids_d + q0 * k, scores_d + q0 * k,
            stats_d ? stats_d + q0 : nullptr, cx.sB, rerank);
    FPP_CUDA(cudaEventRecord(sl.ev_bdone, cx.sB));
    if (c + 2 < nch) issue_a(c + 2);
  }
  FPP_CUDA(cudaEventRecord(cx.ev_join, cx.sA));
  FPP_CUDA(cudaEventRecord(cx.ev_join2, cx.sB));
  FPP_CUDA(cudaStreamWaitEvent(s, cx.ev_join, 0));
  FPP_CUDA(cudaStreamWaitEvent(s, cx.ev_join2, 0));
}

__global__ void k_gather_rows(const float* __restrict__ Q, const uint32_t* __restrict__ perm,
                              uint64_t nq, uint32_t d, float* __restrict__ out) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nq * d;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = e / d;
    out[e] = Q[(uint64_t)perm[i] * d + (e - i * d)];
  }
}
__global__ void k_scatter_results(const uint32_t* __restrict__ perm, uint64_t nq, uint32_t k,
                                  const uint32_t* __restrict__ ids_p,
                                  const double* __restrict__ sc_p,
                                  const fpp_query_stats* __restrict__ st_p, uint32_t* ids,
                                  double* sc, fpp_query_stats* st) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nq * k;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = e / k, j = e - i * k;
    const uint64_t o = (uint64_t)perm[i] * k + j;
    ids[o] = ids_p[e];
    sc[o] = sc_p[e];
    if (st && j == 0) st[perm[i]] = st_p[i];
  }
}

// Batch order: a stable counting sort of the queries by their order key (the
// cross-polytope code of stack (0, K-1): fewer than 2D <= 2048 values) in one
// CTA: histogram, scan, then the tiles of 1024 queries in order, warps in order
// (match_any ranks within a warp, one __syncthreads per warp for the cursors).
constexpr uint32_t ORD_BINS = 2048;
__global__ void __launch_bounds__(1024) k_order_sort(const uint64_t* __restrict__ keys, uint32_t nq,
                                                     uint32_t* __restrict__ perm) {
  __shared__ uint32_t cur[ORD_BINS];
  __shared__ uint32_t scan_sh[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < ORD_BINS; i += blockDim.x) cur[i] = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nq; i += blockDim.x)
    smem_inc(&cur[(uint32_t)keys[i] & (ORD_BINS - 1)]);
  __syncthreads();
  {
    const uint32_t v0 = cur[2 * threadIdx.x], v1 = cur[2 * threadIdx.x + 1];
    uint32_t tot;
    const uint32_t b = block_excl_scan_u32(v0 + v1, scan_sh, &tot);
    cur[2 * threadIdx.x] = b;
    cur[2 * threadIdx.x + 1] = b + v0;
  }
  __syncthreads();
  for (uint32_t base = 0; base < nq; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const bool valid = i < nq;
    const uint32_t key = valid ? ((uint32_t)keys[i] & (ORD_BINS - 1)) : ORD_BINS;
    const uint32_t peers = __match_any_sync(FULL, key);
    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    const bool leader = rank == 0;
    uint32_t pos = 0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) {
      if (w == w2 && valid && leader) {
        pos = cur[key];
        cur[key] = pos + __popc(peers);
      }
      __syncthreads();
    }
    const uint32_t lead = __ffs(peers) - 1;
    pos = __shfl_sync(FULL, pos, lead);
    if (valid) perm[pos + rank] = i;
  }
}

// Batched query.  Large batches are processed ordered by the cross-polytope code
// of stack (0, K-1) (similar queries adjacent; the sort is stable): with the
// ascending-id candidate lists, concurrently scored queries then gather shared
// rows through L2 (C2: +8% over input order; the full table-0 bucket or the
// SimHash signature as key group less well).  Results are scattered back to
// the caller's order; FPP_NO_REORDER=1 keeps the input order.  Results are
// identical either way (every query is independent).  The context's previous
// call (possibly on another stream) completes before its scratch is reused.
static void ensure_score_bytes(const Index& ix) {
  if (!ix.score_bytes_d.p) {
    std::lock_guard<std::mutex> lk(ix.mu);
    if (!ix.score_bytes_d.p) {
      ix.score_bytes_d.alloc(1);
      FPP_CUDA(cudaMemset(ix.score_bytes_d.p, 0, 8));
    }
  }
}

// Multi-GPU query split: stage A alone for a
// slice of the batch -- the probe sets as global bucket ids, [nq][P_eff] in probe
// order (the L true buckets first).  They depend on the queries and the hash
// functions only, so any shard's index (same parameters and seed) can resolve them.
void run_query_probes(const Index& ix, QueryCtx& cx, const float* Qd, uint64_t nq, uint32_t qprobes,
                  uint32_t* probes_d, cudaStream_t s) {
  if (cx.done_recorded) FPP_CUDA(cudaStreamWaitEvent(s, cx.ev_done, 0));
  const uint32_t cs = chunk_size(ix, qprobes, nq);
  const uint64_t peff = query_probes(ix, qprobes);
  for (uint64_t q0 = 0; q0 < nq; q0 += cs) {
    const uint32_t n = (uint32_t)std::min<uint64_t>(cs, nq - q0);
    stage_a(ix, cx, cx.slot[0], Qd + q0 * ix.d, n, qprobes, s, nullptr, probes_d + q0 * peff);
  }
  FPP_CUDA(cudaEventRecord(cx.ev_done, s));
  cx.done_recorded = true;
}

// ... and stage B from such probe sets: resolved in this index's tables
// (k_resolve_probes), then the same collect / score path as run_query.
void run_query_from_probes(const Index& ix, QueryCtx& cx, const float* Qd, uint64_t nq,
                       const uint32_t* probes_d, uint32_t k, uint32_t qprobes, uint32_t* ids_d,
                       double* scores_d, fpp_query_stats* stats_d, cudaStream_t s) {
  if (cx.done_recorded) FPP_CUDA(cudaStreamWaitEvent(s, cx.ev_done, 0));
  ensure_score_bytes(ix);
  const uint32_t cs = chunk_size(ix, qprobes, nq);
  const uint64_t peff = query_probes(ix, qprobes);
  QSlot& sl = cx.slot[0];
  for (uint64_t q0 = 0; q0 < nq; q0 += cs) {
    const uint32_t n = (uint32_t)std::min<uint64_t>(cs, nq - q0);
    prepare_slot(ix, sl, n, qprobes);
    cudaEvent_t e0;
    cx.timer.begin(PH_PROBE, s, &e0);
    k_resolve_probes<<<n, 256, 0, s>>>(probes_d + q0 * peff, peff, ix.NB, ix.offsets, ix.table_base,
                                       sl.ppos.p, sl.plen.p, sl.eq.p);
    FPP_LAUNCH();
    k_scan_eq<<<1, 1024, 0, s>>>(sl.eq.p, n, sl.coff.p);
    FPP_LAUNCH();
    FPP_CUDA(cudaMemcpyAsync(sl.pinned, sl.coff.p + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    cx.timer.end(PH_PROBE, e0, s);
    cx.acc.launches += 2;
    FPP_CUDA(cudaEventRecord(sl.ev_probe, s));
    stage_b(ix, cx, sl, Qd + q0 * ix.d, n, k, qprobes, ids_d + q0 * k, scores_d + q0 * k,
            stats_d ? stats_d + q0 : nullptr, s);
  }
  FPP_CUDA(cudaEventRecord(cx.ev_done, s));
  cx.done_recorded = true;
}

void run_query(const Index& ix, QueryCtx& cx, const float* Qd, uint64_t nq, uint32_t k,
               uint32_t qprobes, uint32_t* ids_d, double* scores_d, fpp_query_stats* stats_d,
               cudaStream_t s, uint32_t rerank) {
  if (cx.done_recorded) FPP_CUDA(cudaStreamWaitEvent(s, cx.ev_done, 0));
  ensure_score_bytes(ix);
  static const bool no_reorder = getenv("FPP_NO_REORDER") != nullptr;
  // the reorder costs a fixed ~35 us plus a gather of Q; its gain scales with the
  // score gather (C1, 1000 x 128 i.i.d.: -5%; C3, 1000 x 960 clustered: +4%)
  if (no_reorder || nq < 256 || nq * ix.d < (512ull << 10) || nq >= (1ull << 31)) {
    run_query_core(ix, cx, Qd, nq, k, qprobes, ids_d, scores_d, stats_d, s, rerank);
  } else {
    const uint32_t d = ix.d;
    cx.ord_key.ensure(2 * nq);  // u64 order keys viewed as 2 x u32 words
    cx.ord_perm.ensure(nq);
    cx.ord_q.ensure(nq * d);
    cx.ord_ids.ensure(nq * k);
    cx.ord_sc.ensure(nq * k);
    if (stats_d) cx.ord_st.ensure(nq);
    const int sms = sm_count();
    uint64_t* okeys = reinterpret_cast<uint64_t*>(cx.ord_key.p);
    launch_order_keys(ix, Qd, nq, okeys, s);
    k_order_sort<<<1, 1024, 0, s>>>(okeys, (uint32_t)nq, cx.ord_perm.p);
    FPP_LAUNCH();
    k_gather_rows<<<sms * 8, 256, 0, s>>>(Qd, cx.ord_perm.p, nq, d, cx.ord_q.p);
    FPP_LAUNCH();
    run_query_core(ix, cx, cx.ord_q.p, nq, k, qprobes, cx.ord_ids.p, cx.ord_sc.p,
                   stats_d ? cx.ord_st.p : nullptr, s, rerank);
    k_scatter_results<<<sms * 4, 256, 0, s>>>(cx.ord_perm.p, nq, k, cx.ord_ids.p, cx.ord_sc.p,
                                              stats_d ? cx.ord_st.p : nullptr, ids_d, scores_d,
                                              stats_d);
    FPP_LAUNCH();
    cx.acc.launches += 4;  // order keys, sort, gather, scatter
  }
  FPP_CUDA(cudaEventRecord(cx.ev_done, s));
  cx.done_recorded = true;
}

void query_debug(const Index& ix, QueryCtx& cx, const float* qd, uint32_t qprobes,
                 std::vector<uint64_t>& probes, std::vector<uint32_t>& cands) {
  cudaStream_t s = cx.own;
  if (cx.done_recorded) FPP_CUDA(cudaStreamWaitEvent(s, cx.ev_done, 0));
  const uint64_t peff = query_probes(ix, qprobes);
  DBuf<uint64_t> dbg(peff);
  DBuf<uint32_t> ids(32);
  DBuf<double> sc(32);
  QSlot& sl = cx.slot[0];
  stage_a(ix, cx, sl, qd, 1, qprobes, s, dbg.p);
  FPP_CUDA(cudaEventSynchronize(sl.ev_probe));
  stage_b(ix, cx, sl, qd, 1, 1, qprobes, ids.p, sc.p, nullptr, s, 0, true);
  FPP_CUDA(cudaStreamSynchronize(s));
  probes.resize(peff);
  FPP_CUDA(cudaMemcpy(probes.data(), dbg.p, peff * 8, cudaMemcpyDeviceToHost));
  uint32_t U = 0;
  uint64_t off = 0;
  FPP_CUDA(cudaMemcpy(&U, sl.uq.p, 4, cudaMemcpyDeviceToHost));
  FPP_CUDA(cudaMemcpy(&off, sl.coff.p, 8, cudaMemcpyDeviceToHost));
  cands.resize(U);
  if (U) FPP_CUDA(cudaMemcpy(cands.data(), sl.cands.p + off, (size_t)U * 4, cudaMemcpyDeviceToHost));
  cands.erase(std::remove(cands.begin(), cands.end(), 0xffffffffu), cands.end());  // grouped holes
  std::sort(probes.begin(), probes.end());
  std::sort(cands.begin(), cands.end());
}

// k-way merge of per-shard top-k lists (multi-GPU query): warp per
// query; lane l < lists holds the head of list l; k rounds of a warp arg-best by
// (score desc, id asc), empty slots (id 0xFFFFFFFF, -inf) last.  The lists hold
// disjoint global ids, so the merged order is the 1-GPU top-k's.
__global__ void k_merge_topk(const double* __restrict__ sc, const uint32_t* __restrict__ ids,
                             uint32_t lists, uint64_t nq, uint32_t k, double* __restrict__ osc,
                             uint32_t* __restrict__ oid) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t q = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < nq; q += nw) {
    uint32_t pos = 0;
    const bool mine = (uint32_t)lane < lists;
    const uint64_t base = ((uint64_t)lane * nq + q) * k;
    double hs = -INFINITY;
    uint32_t hi = 0xffffffffu;
    if (mine) { hs = sc[base]; hi = ids[base]; }
    for (uint32_t r = 0; r < k; ++r) {
      double bs = hs;
      uint32_t bi = hi;
      int bl = lane;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double os = __shfl_xor_sync(FULL, bs, o);
        const uint32_t oi = __shfl_xor_sync(FULL, bi, o);
        const int ol = __shfl_xor_sync(FULL, bl, o);
        // valid entries first, then score desc, id asc (lane asc: a total order)
        const bool ov = oi != 0xffffffffu, mv = bi != 0xffffffffu;
        const bool take = (ov && !mv) ||
                          (ov == mv && (os > bs || (os == bs && (oi < bi || (oi == bi && ol < bl)))));
        if (take) { bs = os; bi = oi; bl = ol; }
      }
      if (lane == 0) {
        oid[q * k + r] = bi;
        osc[q * k + r] = bi != 0xffffffffu ? bs : -INFINITY;
      }
      if (lane == bl && bi != 0xffffffffu) {
        ++pos;
        if (pos < k) { hs = sc[base + pos]; hi = ids[base + pos]; }
        else { hs = -INFINITY; hi = 0xffffffffu; }
      }
    }
  }
}

void launch_merge_topk(const double* sc, const uint32_t* ids, uint32_t lists, uint64_t nq,
                       uint32_t k, double* out_sc, uint32_t* out_ids, cudaStream_t s) {
  if (!nq) return;
  const unsigned grid = (unsigned)std::min<uint64_t>((nq + 7) / 8, (uint64_t)sm_count() * 16);
  k_merge_topk<<<grid, 256, 0, s>>>(sc, ids, lists, nq, k, out_sc, out_ids);
  FPP_LAUNCH();
}

}  // namespace fpp
