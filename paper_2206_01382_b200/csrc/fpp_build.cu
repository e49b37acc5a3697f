// fpp_build.cu -- index build: K1 (cross-polytope hashing + index probes) and
// K2 (bucketing, alpha/kappa limit-scaling filter, CSR).
//
// Reference semantics: SPEC.md:245-262 build / filter_bucket
// (Algorithm 1), PAPER.md:336-339 (limit scaling), rotation.cpp:70-100
// (projection).  Pinned choices: DESIGN.md section 3.  Oracle: oracle/fpp_oracle.c
// orc_build().
//
// Pipeline per chunk of T tables:
//   k_hash_build   one lane-group per point: x stays in registers, for every
//                  table/function run the spinner stack (3 x signs+FHT), rank
//                  top-R coordinates, pick top-iProbes pairs, emit
//                  (bucket, score) and bump the bucket histogram
//   k_scan_*       per-table exclusive scans: histogram -> pre-filter starts,
//                  keep(B) -> kept CSR offsets
//   k_scatter      (score desc, id asc) 64-bit keys into bucket segments
//   k_classify     B=1 written directly; B<=32 -> warp list; B>32 with keep<=32 ->
//                  warp top-k list; other B>32 -> CTA list
//   k_sort_small   warp bitonic sort, keep prefix -> CSR
//   k_sort_topk    warp streams the bucket, keeps the sorted top-keep in registers
//   k_sort_large   CTA smem bitonic (B<=4096) or radix-select + chunked sort
#include <algorithm>
#include <cstdio>

#include "fpp_device.cuh"
#include "fpp_internal.h"

namespace fpp {

// ------------------------------------------------------------------ K1 build
constexpr int HB_SEL = 32;  // keys sorted after the threshold preselection
// k_hash_build CTA size and CTAs per SM (FPP_HB_THREADS x FPP_HB_MINB warps resident)
#ifndef FPP_HB_THREADS
#define FPP_HB_THREADS 256
#endif
#ifndef FPP_HB_MINB
#define FPP_HB_MINB 3
#endif
constexpr int HB_THREADS = FPP_HB_THREADS;

// Rank pairs (a, b) with (a + 1)(b + 1) <= R: the only candidates for the top ip <= R
// pairs (every pair with a' <= a, b' <= b strictly precedes (a, b)); D(R) = sum_a
// floor(R / (a + 1)) of them (8, 20, 50 for R = 4, 8, 16) instead of R^2 slots.
template <int R>
struct PairList {
  static constexpr int N = [] {
    int n = 0;
    for (int a = 0; a < R; ++a) n += R / (a + 1);
    return n;
  }();
  uint16_t ab[N];  // a << 8 | b
};
template <int R>
constexpr PairList<R> make_pairs() {
  PairList<R> p{};
  int i = 0;
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < R / (a + 1); ++b) p.ab[i++] = (uint16_t)(a << 8 | b);
  return p;
}
__constant__ PairList<4> c_pairs4 = make_pairs<4>();
__constant__ PairList<8> c_pairs8 = make_pairs<8>();
__constant__ PairList<16> c_pairs16 = make_pairs<16>();
template <int R>
__device__ __forceinline__ uint32_t pair_ab(int i) {
  if constexpr (R == 4) return c_pairs4.ab[i];
  else if constexpr (R == 8) return c_pairs8.ab[i];
  else return c_pairs16.ab[i];
}

// k_hash_build shared memory: NGRP transpose buffers (TS >= P floats, reused
// for the v dump of the preselection) + per group HB_SEL scratch keys and the
// two sorted top-R lists
template <int P>
__host__ __device__ constexpr int hb_tbuf_bytes() {
  return (HB_THREADS / (P < 32 ? 1 : P / 32)) * (P >= 64 ? TransposeShape<P>::STRIDE : 4) * 4;
}
template <int P, int R>
constexpr int hb_smem_bytes() {
  return hb_tbuf_bytes<P>() + (HB_THREADS / (P < 32 ? 1 : P / 32)) * (HB_SEL + 2 * R) * 8;
}

// Top-r selection of one projection (r = min(iProbes, D) <= R), exact order
// (|p| desc, j asc) as 64-bit rank keys, written sorted to sel[0..R).
//  * P >= 64 (fast path): bisect a threshold T in [0, amax] until the group
//    count of |p| >= T lies in [r, HB_SEL]; every entry ranked before a kept one
//    is kept too (|p| is compared exactly), so the top r of the kept set are the
//    top r overall.  The <= HB_SEL kept keys are compacted and bitonic-sorted.
//  * otherwise, or when some group of the warp finds no such T (ties at the
//    threshold): lane-local top-R insertion + butterfly merge of the group.
template <int P, int R>
__device__ __forceinline__ void hb_select(const float (&v)[FhtShape<P>::EPT], int g, uint32_t D,
                                          uint32_t r, float* vbuf, uint64_t* scratch, uint64_t* sel) {
  using S = FhtShape<P>;
  constexpr bool TR = P >= 64;
  const bool full = D >= (uint32_t)P;  // no truncation: skip the j < D test
  auto jof = [&](int e) -> uint32_t {
    if constexpr (TR) return jB<P>(e, g);
    else return (uint32_t)g * S::EPT + e;
  };
  bool fast = false;
  if constexpr (TR) {
    float amax = 0.0f;
#pragma unroll
    for (int e = 0; e < S::EPT; ++e)
      if (full || jof(e) < D) amax = fmaxf(amax, fabsf(v[e]));
#pragma unroll
    for (int m = 1; m < S::G; m <<= 1) amax = fmaxf(amax, __shfl_xor_sync(FULL, amax, m));
    float lo = 0.0f, hi = 1.0f;
    uint32_t macc = 0;  // this lane's kept elements at the accepted threshold
    bool ok = false, fail = !(amax > 0.0f);
#pragma unroll 1
    for (int it = 0; it < 24; ++it) {
      if (__all_sync(FULL, ok || fail)) break;
      const float mid = it == 0 ? 0.625f : 0.5f * (lo + hi);  // typical band for r ~ 5
      const float T = amax * mid;
      uint32_t m = 0;
#pragma unroll
      for (int e = 0; e < S::EPT; ++e)
        m |= (((full || jof(e) < D) && fabsf(v[e]) >= T) ? 1u : 0u) << e;
      uint32_t c = __popc(m);
#pragma unroll
      for (int k = 1; k < S::G; k <<= 1) c += __shfl_xor_sync(FULL, c, k);
      if (!ok && !fail) {
        if (c > (uint32_t)HB_SEL) lo = mid;
        else if (c < r) hi = mid;
        else { ok = true; macc = m; }
        if (!(hi - lo > 1e-7f)) fail = !ok;
      }
    }
    fast = __all_sync(FULL, ok);
    if (fast) {
      // v -> shared memory in natural order (the lane reads back only its own
      // entries), then each lane appends its kept keys at its exclusive offset
      store_B_natural<P>(v, g, vbuf);
      const uint32_t cl = __popc(macc);
      uint32_t x = cl;
#pragma unroll
      for (int o = 1; o < S::G; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, x, o);
        if (g >= o) x += y;
      }
      const int lane = threadIdx.x & 31;
      const uint32_t ctot = __shfl_sync(FULL, x, (lane / S::G) * S::G + S::G - 1);
      uint32_t pos = x - cl;
      for (uint32_t mm = macc; mm; mm &= mm - 1) {
        const uint32_t j = jof(__ffs(mm) - 1);
        scratch[pos++] = rank_key(vbuf[j], j);
      }
      for (uint32_t i = ctot + g; i < (uint32_t)HB_SEL; i += S::G) scratch[i] = ~0ull;
      __syncwarp();
      // the r smallest of the <= HB_SEL kept keys, in order: r rounds of a group
      // minimum (keys are unique: they carry the index), the owner retiring its key
      // (cheaper than sorting all HB_SEL 64-bit keys when r << HB_SEL)
      constexpr int E = HB_SEL / S::G;
      uint64_t k[E];
#pragma unroll
      for (int e = 0; e < E; ++e) k[e] = scratch[g * E + e];
      for (uint32_t qq = 0; qq < r; ++qq) {
        uint64_t m = k[0];
#pragma unroll
        for (int e = 1; e < E; ++e) m = k[e] < m ? k[e] : m;
#pragma unroll
        for (int o = 1; o < S::G; o <<= 1) {
          const uint64_t y = shfl_xor_u64(m, o);
          m = y < m ? y : m;
        }
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (k[e] == m) k[e] = ~0ull;
        if (g == 0) sel[qq] = m;
      }
      __syncwarp();
    }
  }
  if (!fast) {
    float tp[R];
    uint32_t tj[R];
#pragma unroll
    for (int q = 0; q < R; ++q) { tp[q] = 0.0f; tj[q] = 0xffffffffu; }
    float thr = -1.0f;
#pragma unroll
    for (int e = 0; e < S::EPT; ++e) {
      const uint32_t j = jof(e);  // j increases with e in both layouts
      const float a = fabsf(v[e]);
      if ((full || j < D) && a > thr) {
        float cp = v[e];
        uint32_t cj = j;
        bool shift = false;
#pragma unroll
        for (int q = 0; q < R; ++q) {  // insert, shifting the tail down
          // once the new entry is placed every later slot shifts unconditionally: a
          // displaced entry must stay AHEAD of the entries it was ahead of, also of those
          // with an equal |p| (j ascending among ties) -- a strict compare here would
          // let a displaced entry slip behind its tied successor
          const bool ins = shift || tj[q] == 0xffffffffu || fabsf(cp) > fabsf(tp[q]);
          const float op = tp[q];
          const uint32_t oj = tj[q];
          if (ins) { tp[q] = cp; tj[q] = cj; cp = op; cj = oj; shift = true; }
        }
        thr = tj[R - 1] == 0xffffffffu ? -1.0f : fabsf(tp[R - 1]);
      }
    }
    uint64_t tk[R];
#pragma unroll
    for (int q = 0; q < R; ++q) tk[q] = tj[q] == 0xffffffffu ? ~0ull : rank_key(tp[q], tj[q]);
    topr_group_merge<R, S::G>(tk);
    if (g == 0) {
#pragma unroll
      for (int q = 0; q < R; ++q) sel[q] = tk[q];
    }
    __syncwarp();
  }
}

template <int P, int R>
__global__ void __launch_bounds__(HB_THREADS, FPP_HB_MINB)
k_hash_build(const float* __restrict__ X, uint64_t n, uint32_t d, uint32_t ldx, uint32_t D,
             uint32_t K,
             const uint32_t* __restrict__ signs, uint32_t t0, uint32_t T, uint32_t ip,
             uint2* __restrict__ ent, uint32_t* __restrict__ counts, uint64_t NB) {
  using S = FhtShape<P>;
  constexpr bool TR = P >= 64;  // transpose FHT (cross-lane stages in registers)
  constexpr int TS = TR ? TransposeShape<P>::STRIDE : 4;
  // dynamic shared memory (hb_smem_bytes): per group a transpose buffer of TS
  // floats (reused as the 32-key sort scratch once the FHT is done), then per
  // group the sorted top-R lists of the K functions
  extern __shared__ __align__(16) unsigned char hb_smem[];
  constexpr int NGRP = HB_THREADS / S::G;
  const int lane = threadIdx.x & 31;
  const int g = lane % S::G;
  const int grp = threadIdx.x / S::G;
  float* buf = reinterpret_cast<float*>(hb_smem) + grp * TS;  // also the v dump (P <= TS)
  uint64_t* scratch = reinterpret_cast<uint64_t*>(hb_smem + hb_tbuf_bytes<P>()) + grp * (HB_SEL + 2 * R);
  uint64_t* sel0 = scratch + HB_SEL;
  uint64_t* sel1 = sel0 + R;
  const uint64_t gid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / S::G;
  const bool active = gid < n;
  const uint64_t i = active ? gid : n - 1;  // inactive groups shadow a real row
  float x[S::EPT];
  load_row<P>(X + i * ldx, d, g, x);
  const uint32_t r = ip < D ? ip : D;  // ranks needed per function (host ensures <= R)
  const uint32_t twoD = 2 * D;
  // candidate pairs: (a+1)(b+1) <= ip (every pair with a' <= a, b' <= b strictly
  // precedes (a, b), so no other pair can be among the top ip): PairList<R>
  constexpr int NPL = (PairList<R>::N + S::G - 1) / S::G;
  for (uint32_t tt = 0; tt < T; ++tt) {
    const uint32_t t = t0 + tt;
#pragma unroll 1
    for (int f = 0; f < (int)K; ++f) {
      float v[S::EPT];
#pragma unroll
      for (int e = 0; e < S::EPT; ++e) v[e] = x[e];
      const uint32_t* sw = signs + ((uint64_t)t * K + f) * 3 * S::W;
      if constexpr (TR) spinner_project_T<P>(v, sw, g, buf);  // layout B: j = jB<P>(e, g)
      else spinner_project<P>(v, sw, g);                      // layout A: j = g*EPT + e
      hb_select<P, R>(v, g, D, r, buf, scratch, f == 0 ? sel0 : sel1);
      __syncwarp();  // the v dump aliases the next projection's transpose buffer
    }
    uint32_t* cnt = counts ? counts + (uint64_t)tt * NB : nullptr;
    uint2* out = ent + ((uint64_t)tt * n + i) * ip;
    if (K == 1) {
      // SPEC.md:184-192 with l=1: the top-iProbes signed vectors themselves
      if (g == 0 && active) {
        for (uint32_t q = 0; q < ip; ++q) {
          const uint32_t b = rank_code(sel0[q], D);
          out[q] = make_uint2(b, __float_as_uint(rank_val(sel0[q])));
          if (cnt) atomicAdd(cnt + b, 1u);
        }
      }
      __syncwarp();
      continue;
    }
    // top-iProbes pairs by (fl(v1+v2) desc, r1 asc, r2 asc), group-parallel:
    // composite max-key (ord(score), 0xFFFF-r1, 0xFFFF-r2); each round takes the
    // group maximum strictly below the previous selection.
    uint64_t pk[NPL];
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      const uint32_t pi = (uint32_t)g + (uint32_t)k * S::G;
      const uint32_t ab = pi < (uint32_t)PairList<R>::N ? pair_ab<R>((int)pi) : 0xffffu;
      const uint32_t a = ab >> 8, b = ab & 0xffu;
      pk[k] = 0;
      if (pi < (uint32_t)PairList<R>::N && a < r && b < r && (a + 1) * (b + 1) <= ip) {
        const float sc = rank_val(sel0[a]) + rank_val(sel1[b]);
        pk[k] = ((uint64_t)ord_key(sc) << 32) | ((uint64_t)(0xffffu - a) << 16) | (0xffffu - b);
      }
    }
    uint64_t prev = ~0ull;
    for (uint32_t sl = 0; sl < ip; ++sl) {
      uint64_t best = 0;
#pragma unroll
      for (int k = 0; k < NPL; ++k) best = (pk[k] < prev && pk[k] > best) ? pk[k] : best;
#pragma unroll
      for (int m = 1; m < S::G; m <<= 1) {
        const uint64_t o = shfl_xor_u64(best, m);
        best = o > best ? o : best;
      }
      prev = best;
      if (g == 0 && active) {
        const uint32_t a = 0xffffu - (uint32_t)((best >> 16) & 0xffffu);
        const uint32_t b = 0xffffu - (uint32_t)(best & 0xffffu);
        const uint32_t bucket = rank_code(sel0[a], D) * twoD + rank_code(sel1[b], D);
        out[sl] = make_uint2(bucket, __float_as_uint(ord_inv((uint32_t)(best >> 32))));
        if (cnt) atomicAdd(cnt + bucket, 1u);
      }
    }
    __syncwarp();
  }
}

template <int P>
__global__ void __launch_bounds__(256)
k_project(const float* __restrict__ X, uint64_t n, uint32_t d, uint32_t D,
          const uint32_t* __restrict__ sw, float* __restrict__ out) {
  using S = FhtShape<P>;
  constexpr bool TR = P >= 64;
  constexpr int TS = TR ? TransposeShape<P>::STRIDE : 4;
  __shared__ __align__(16) float tbuf[(256 / S::G) * TS];
  const int lane = threadIdx.x & 31;
  const int g = lane % S::G;
  float* buf = tbuf + (threadIdx.x / S::G) * TS;
  const uint64_t gid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / S::G;
  const bool active = gid < n;
  const uint64_t i = active ? gid : n - 1;
  float v[S::EPT];
  load_row<P>(X + i * d, d, g, v);
  if constexpr (TR) spinner_project_T<P>(v, sw, g, buf);
  else spinner_project<P>(v, sw, g);
  if (!active) return;
#pragma unroll
  for (int e = 0; e < S::EPT; ++e) {
    const uint32_t j = layout_index<P>(e, g);
    if (j < D) out[i * D + j] = v[e];
  }
}

// SimHash signatures (SPEC.md "SimHash signatures"; :330-338): bit j < min(64, D)
// is 1 iff p[j] >= 0 for the (t=0, f=0) projection (-0.0 counts as >= 0, as in
// cross_polytope_hash).  One lane group per row; partial masks OR-reduced.
template <int P>
__global__ void __launch_bounds__(256)
k_signatures(const float* __restrict__ X, uint64_t n, uint32_t d, uint32_t ld, uint32_t D,
             const uint32_t* __restrict__ sw, uint64_t* __restrict__ out) {
  using S = FhtShape<P>;
  constexpr bool TR = P >= 64;
  constexpr int TS = TR ? TransposeShape<P>::STRIDE : 4;
  __shared__ __align__(16) float tbuf[(256 / S::G) * TS];
  const int lane = threadIdx.x & 31;
  const int g = lane % S::G;
  float* buf = tbuf + (threadIdx.x / S::G) * TS;
  const uint64_t gid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / S::G;
  const bool active = gid < n;
  const uint64_t i = active ? gid : n - 1;
  float v[S::EPT];
  load_row<P>(X + i * ld, d, g, v);
  if constexpr (TR) spinner_project_T<P>(v, sw, g, buf);
  else spinner_project<P>(v, sw, g);
  const uint32_t m = D < 64 ? D : 64;
  uint64_t sig = 0;
#pragma unroll
  for (int e = 0; e < S::EPT; ++e) {
    const uint32_t j = layout_index<P>(e, g);
    if (j < m && v[e] >= 0.0f) sig |= 1ull << j;
  }
#pragma unroll
  for (int k = 1; k < S::G; k <<= 1) sig |= shfl_xor_u64(sig, k);
  if (active && g == 0) out[i] = sig;
}

void launch_signatures(const Index& ix, const float* Xd, uint64_t n, uint32_t ld, uint64_t* out,
                       cudaStream_t s) {
  if (n == 0) return;
  const uint32_t P = ix.P;
  const uint32_t G = P < 32 ? 1 : P / 32;
  const unsigned blocks = (unsigned)((n * G + 255) / 256);
  const uint32_t* sw = ix.signs;  // stack (t=0, f=0)
#define FPP_SIG_CASE(PP)                                                            \
  case PP:                                                                          \
    k_signatures<PP><<<blocks, 256, 0, s>>>(Xd, n, ix.d, ld, ix.prm.D, sw, out);    \
    break;
  switch (P) {
    FPP_SIG_CASE(2) FPP_SIG_CASE(4) FPP_SIG_CASE(8) FPP_SIG_CASE(16) FPP_SIG_CASE(32)
    FPP_SIG_CASE(64) FPP_SIG_CASE(128) FPP_SIG_CASE(256) FPP_SIG_CASE(512) FPP_SIG_CASE(1024)
    default: fail(FPP_ERR_UNSUPPORTED, "signatures: padded dimension > 1024 not supported on GPU");
  }
#undef FPP_SIG_CASE
  FPP_LAUNCH();
}

// Query-batch ordering keys (fpp_query.cu run_query): the cross-polytope code of
// stack (0, 0) of each row (the first half of its table-0 bucket).  Queries with
// equal keys are processed next to each other, so concurrently scored queries
// share more candidate rows in L2.  Scheduling only: results are per query.
template <int P>
__global__ void __launch_bounds__(256)
k_order_keys(const float* __restrict__ X, uint64_t n, uint32_t d, uint32_t D, uint32_t K,
             const uint32_t* __restrict__ signs, uint64_t* __restrict__ out) {
  using S = FhtShape<P>;
  constexpr bool TR = P >= 64;
  constexpr int TS = TR ? TransposeShape<P>::STRIDE : 4;
  __shared__ __align__(16) float tbuf[(256 / S::G) * TS];
  const int lane = threadIdx.x & 31;
  const int g = lane % S::G;
  float* buf = tbuf + (threadIdx.x / S::G) * TS;
  const uint64_t gid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / S::G;
  const bool active = gid < n;
  const uint64_t i = active ? gid : n - 1;
  uint64_t key = 0;
  for (uint32_t f = 0; f < K; ++f) {
    float v[S::EPT];
    load_row<P>(X + i * d, d, g, v);
    const uint32_t* sw = signs + (uint64_t)f * 3 * S::W;  // stack (t = 0, f)
    if constexpr (TR) spinner_project_T<P>(v, sw, g, buf);
    else spinner_project<P>(v, sw, g);
    // argmax |p| (lowest index on ties), sign in bit 0
    uint64_t best = 0;
#pragma unroll
    for (int e = 0; e < S::EPT; ++e) {
      const uint32_t j = layout_index<P>(e, g);
      if (j < D) {
        const uint64_t c = ((uint64_t)ord_key(fabsf(v[e])) << 32) |
                           ((uint64_t)(0x7fffffffu - j) << 1) | (v[e] < 0.0f ? 1u : 0u);
        best = c > best ? c : best;
      }
    }
#pragma unroll
    for (int m = 1; m < S::G; m <<= 1) {
      const uint64_t o = shfl_xor_u64(best, m);
      best = o > best ? o : best;
    }
    const uint32_t j = 0x7fffffffu - ((uint32_t)best >> 1);
    key = (key << 32) | ((best & 1u) ? D + j : j);
  }
  if (active && g == 0) out[i] = key;
}

void launch_order_keys(const Index& ix, const float* Qd, uint64_t n, uint64_t* out, cudaStream_t s) {
  if (n == 0) return;
  const uint32_t P = ix.P;
  const uint32_t G = P < 32 ? 1 : P / 32;
  const unsigned blocks = (unsigned)((n * G + 255) / 256);
#define FPP_ORD_CASE(PP)                                                                      \
  case PP:                                                                                    \
    k_order_keys<PP><<<blocks, 256, 0, s>>>(Qd, n, ix.d, ix.prm.D, 1u, ix.signs, out);        \
    break;
  switch (P) {
    FPP_ORD_CASE(2) FPP_ORD_CASE(4) FPP_ORD_CASE(8) FPP_ORD_CASE(16) FPP_ORD_CASE(32)
    FPP_ORD_CASE(64) FPP_ORD_CASE(128) FPP_ORD_CASE(256) FPP_ORD_CASE(512) FPP_ORD_CASE(1024)
    default: fail(FPP_ERR_UNSUPPORTED, "order keys: padded dimension > 1024 not supported on GPU");
  }
#undef FPP_ORD_CASE
  FPP_LAUNCH();
}

// ------------------------------------------------------------- per-table scan
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_PER_THREAD = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_PER_THREAD;

struct KeepXform {
  int mode;  // 0 identity, 1 keep(B)
  float alpha;
  uint32_t ip, kappa;
  __device__ __forceinline__ uint32_t operator()(uint32_t B) const {
    return mode ? keep_count(B, alpha, ip, kappa) : B;
  }
};

__global__ void __launch_bounds__(SCAN_THREADS)
k_scan_reduce(const uint32_t* __restrict__ in, uint64_t NB, uint32_t ntiles, KeepXform xf,
              uint32_t* __restrict__ tile_sums) {
  __shared__ uint32_t sh[32];
  const uint32_t tile = blockIdx.x, t = blockIdx.y;
  const uint32_t* src = in + (uint64_t)t * NB;
  uint32_t s = 0;
  const uint64_t base = (uint64_t)tile * SCAN_TILE + threadIdx.x * SCAN_PER_THREAD;
#pragma unroll
  for (int k = 0; k < SCAN_PER_THREAD; ++k)
    if (base + k < NB) s += xf(src[base + k]);
  uint32_t tot;
  block_excl_scan_u32(s, sh, &tot);
  if (threadIdx.x == 0) tile_sums[(uint64_t)t * ntiles + tile] = tot;
}

__global__ void __launch_bounds__(SCAN_THREADS)
k_scan_tiles(uint32_t* __restrict__ tile_sums, uint32_t ntiles, uint32_t* __restrict__ totals) {
  __shared__ uint32_t sh[32];
  uint32_t* ts = tile_sums + (uint64_t)blockIdx.x * ntiles;
  uint32_t carry = 0;
  for (uint32_t b = 0; b < ntiles; b += blockDim.x) {
    const uint32_t i = b + threadIdx.x;
    const uint32_t v = i < ntiles ? ts[i] : 0;
    uint32_t tot;
    const uint32_t ex = block_excl_scan_u32(v, sh, &tot);
    if (i < ntiles) ts[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(SCAN_THREADS)
k_scan_apply(const uint32_t* __restrict__ in, uint64_t NB, uint32_t ntiles, KeepXform xf,
             const uint32_t* __restrict__ tile_sums, const uint32_t* __restrict__ totals,
             uint32_t* __restrict__ out /* [T][NB+1] */) {
  __shared__ uint32_t sh[32];
  const uint32_t tile = blockIdx.x, t = blockIdx.y;
  const uint32_t* src = in + (uint64_t)t * NB;
  uint32_t* dst = out + (uint64_t)t * (NB + 1);
  const uint64_t base = (uint64_t)tile * SCAN_TILE + threadIdx.x * SCAN_PER_THREAD;
  uint32_t v[SCAN_PER_THREAD];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_PER_THREAD; ++k) {
    v[k] = base + k < NB ? xf(src[base + k]) : 0;
    s += v[k];
  }
  uint32_t run = tile_sums[(uint64_t)t * ntiles + tile] + block_excl_scan_u32(s, sh, nullptr);
#pragma unroll
  for (int k = 0; k < SCAN_PER_THREAD; ++k) {
    if (base + k < NB) dst[base + k] = run;
    run += v[k];
  }
  if (tile == 0 && threadIdx.x == 0) dst[NB] = totals[t];
}

// in [T][NB] -> out [T][NB+1] exclusive, totals [T]
static void scan_tables(const uint32_t* in, uint64_t NB, uint32_t T, KeepXform xf, uint32_t* out,
                        uint32_t* totals, DBuf<uint32_t>& tile_buf, cudaStream_t s) {
  const uint32_t ntiles = (uint32_t)((NB + SCAN_TILE - 1) / SCAN_TILE);
  tile_buf.ensure((size_t)ntiles * T);
  dim3 grid(ntiles, T);
  k_scan_reduce<<<grid, SCAN_THREADS, 0, s>>>(in, NB, ntiles, xf, tile_buf.p);
  FPP_LAUNCH();
  k_scan_tiles<<<T, SCAN_THREADS, 0, s>>>(tile_buf.p, ntiles, totals);
  FPP_LAUNCH();
  k_scan_apply<<<grid, SCAN_THREADS, 0, s>>>(in, NB, ntiles, xf, tile_buf.p, totals, out);
  FPP_LAUNCH();
}

// ------------------------------------------------------------------ scatter
// Thread per (point, table): the point's iProbes entries are read together
// (coalesced across the warp) and their bucket-cursor atomics issued before
// any result is used.  Order inside a bucket is irrelevant (sorted afterwards).
constexpr int SCATTER_UNROLL = 4;
__global__ void __launch_bounds__(256)
k_scatter(const uint2* __restrict__ ent, uint32_t n, uint32_t ip, uint64_t NB,
          const uint32_t* __restrict__ starts, uint32_t* __restrict__ cursor,
          uint64_t* __restrict__ keys, uint32_t id_add = 0) {
  const uint32_t tt = blockIdx.y;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t nip = (uint64_t)n * ip;
  const uint2* e = ent + (uint64_t)tt * nip + (uint64_t)i * ip;
  const uint32_t* st = starts + (uint64_t)tt * (NB + 1);
  uint32_t* cur = cursor + (uint64_t)tt * NB;
  uint64_t* kout = keys + (uint64_t)tt * nip;
  for (uint32_t q0 = 0; q0 < ip; q0 += SCATTER_UNROLL) {
    uint2 en[SCATTER_UNROLL];
    uint32_t pos[SCATTER_UNROLL];
#pragma unroll
    for (int u = 0; u < SCATTER_UNROLL; ++u)
      if (q0 + u < ip) en[u] = e[q0 + u];
#pragma unroll
    for (int u = 0; u < SCATTER_UNROLL; ++u)
      if (q0 + u < ip) pos[u] = atomicAdd(cur + en[u].x, 1u);
#pragma unroll
    for (int u = 0; u < SCATTER_UNROLL; ++u)
      if (q0 + u < ip)
        kout[st[en[u].x] + pos[u]] = desc_score_key(__uint_as_float(en[u].y), i + id_add);
  }
}

struct CsrOut {
  const uint32_t* offs;     // [T][NB+1] kept offsets of this chunk's tables
  const uint64_t* base;     // [T] table bases (global positions)
  uint32_t* ids;
  float* scores;
  uint64_t* keys_out;       // sharded build: sorted keys instead of (ids, scores)
};

__device__ __forceinline__ void csr_put(const CsrOut& o, uint32_t tt, uint64_t NB, uint32_t b,
                                        uint32_t j, uint64_t key) {
  const uint64_t pos = o.base[tt] + o.offs[(uint64_t)tt * (NB + 1) + b] + j;
  if (o.keys_out) {
    o.keys_out[pos] = key;
    return;
  }
  o.ids[pos] = (uint32_t)(key & 0xffffffffu);
  o.scores[pos] = desc_score_val(key);
}

constexpr uint32_t SMALL_MAX = 32;
constexpr uint32_t LARGE_CAP = 4096;
constexpr uint32_t TOPK_MAX = 32;  // B > 32 with keep <= 32 -> k_sort_topk

__global__ void __launch_bounds__(256)
k_classify(const uint32_t* __restrict__ starts, const uint64_t* __restrict__ keys, uint64_t nip,
           uint32_t T, uint64_t NB, CsrOut o, uint32_t* __restrict__ small_list,
           uint32_t* __restrict__ large_list, uint32_t* __restrict__ ctr, uint64_t large_cap) {
  const uint64_t total = NB * T;
  uint32_t local_max = 0;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t tt = (uint32_t)(x / NB);
    const uint32_t b = (uint32_t)(x - (uint64_t)tt * NB);
    const uint32_t* st = starts + (uint64_t)tt * (NB + 1);
    const uint32_t B = st[b + 1] - st[b];
    if (B == 0) continue;
    const uint32_t* of = o.offs + (uint64_t)tt * (NB + 1);
    const uint32_t k = of[b + 1] - of[b];
    local_max = max(local_max, k);
    if (k == 0) continue;
    if (B == 1) {
      csr_put(o, tt, NB, b, 0, keys[(uint64_t)tt * nip + st[b]]);
    } else if (B <= SMALL_MAX) {
      small_list[atomicAdd(ctr + 0, 1u)] = (uint32_t)x;
    } else if (k <= TOPK_MAX && !o.keys_out) {  // keep << B: warp streaming top-k
      large_list[large_cap - 1 - atomicAdd(ctr + 3, 1u)] = (uint32_t)x;
    } else {
      large_list[atomicAdd(ctr + 1, 1u)] = (uint32_t)x;
    }
  }
  // block max, one atomic per block
  for (int o2 = 16; o2 > 0; o2 >>= 1) local_max = max(local_max, __shfl_xor_sync(FULL, local_max, o2));
  if ((threadIdx.x & 31) == 0 && local_max) atomicMax(ctr + 2, local_max);
}

__global__ void __launch_bounds__(256)
k_sort_small(const uint32_t* __restrict__ starts, const uint64_t* __restrict__ keys, uint64_t nip,
             uint64_t NB, CsrOut o, const uint32_t* __restrict__ list,
             const uint32_t* __restrict__ ctr) {
  const int lane = threadIdx.x & 31;
  const uint32_t count = ctr[0];
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t it = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < count; it += nwarps) {
    const uint32_t x = list[it];
    const uint32_t tt = (uint32_t)(x / NB), b = (uint32_t)(x - (uint64_t)tt * NB);
    const uint32_t* st = starts + (uint64_t)tt * (NB + 1);
    const uint32_t B = st[b + 1] - st[b];
    const uint32_t* of = o.offs + (uint64_t)tt * (NB + 1);
    const uint32_t k = of[b + 1] - of[b];
    uint64_t key = lane < (int)B ? keys[(uint64_t)tt * nip + st[b] + lane] : ~0ull;
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        const uint64_t other = __shfl_xor_sync(FULL, key, j);
        const bool up = (lane & kk) == 0;
        const bool lower = (lane & j) == 0;
        const uint64_t mn = key < other ? key : other, mx = key < other ? other : key;
        key = (lower == up) ? mn : mx;
      }
    }
    if ((uint32_t)lane < k) csr_put(o, tt, NB, b, lane, key);
  }
}

// Warp per bucket with B > 32 and keep <= 32: the first 32 keys are bitonic
// sorted across the lanes (lane i = i-th smallest), then every later key below
// the current keep-th smallest is inserted (ballot rank + shift up).  Keys are
// unique (id in the low bits), so the result equals the sorted prefix.
__global__ void __launch_bounds__(256)
k_sort_topk(const uint32_t* __restrict__ starts, const uint64_t* __restrict__ keys, uint64_t nip,
            uint64_t NB, CsrOut o, const uint32_t* __restrict__ list,
            const uint32_t* __restrict__ ctr, uint64_t large_cap) {
  const int lane = threadIdx.x & 31;
  const uint32_t count = ctr[3];
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t it = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < count; it += nwarps) {
    const uint32_t x = list[large_cap - 1 - it];
    const uint32_t tt = (uint32_t)(x / NB), b = (uint32_t)(x - (uint64_t)tt * NB);
    const uint32_t* st = starts + (uint64_t)tt * (NB + 1);
    const uint32_t B = st[b + 1] - st[b];
    const uint32_t* of = o.offs + (uint64_t)tt * (NB + 1);
    const uint32_t k = of[b + 1] - of[b];
    const uint64_t* seg = keys + (uint64_t)tt * nip + st[b];
    uint64_t top = seg[lane];  // B > 32
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        const uint64_t other = __shfl_xor_sync(FULL, top, j);
        const bool up = (lane & kk) == 0;
        const bool lower = (lane & j) == 0;
        const uint64_t mn = top < other ? top : other, mx = top < other ? other : top;
        top = (lower == up) ? mn : mx;
      }
    }
    uint64_t thr = __shfl_sync(FULL, top, k - 1);
    for (uint32_t c0 = 32; c0 < B; c0 += 32) {
      const uint64_t key = c0 + lane < B ? seg[c0 + lane] : ~0ull;
      uint32_t m = __ballot_sync(FULL, key < thr);
      while (m) {
        const int src = __ffs(m) - 1;
        m &= m - 1;
        const uint64_t v = __shfl_sync(FULL, key, src);
        if (v >= thr) continue;  // thr only decreases (warp-uniform)
        const int pos = __popc(__ballot_sync(FULL, top < v));
        const uint64_t upv = __shfl_up_sync(FULL, top, 1);
        if (lane > pos) top = upv;
        if (lane == pos) top = v;
        thr = __shfl_sync(FULL, top, k - 1);
      }
    }
    if ((uint32_t)lane < k) csr_put(o, tt, NB, b, lane, top);
  }
}

__device__ void block_bitonic(uint64_t* s, uint32_t N) {
  for (uint32_t k = 2; k <= N; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = s[i], b = s[ixj];
          const bool asc = (i & k) == 0;
          if ((a > b) == asc) {
            s[i] = b;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// key of 0-based rank `rank` (ascending) among seg[0..B), keys unique
__device__ uint64_t block_radix_select(const uint64_t* __restrict__ seg, uint32_t B, uint32_t rank,
                                       uint32_t* hist, uint64_t* sh_prefix, uint32_t* sh_rank) {
  uint64_t prefix = 0, mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) {
      const uint64_t k = seg[i];
      if ((k & mask) == prefix) smem_inc(hist + ((k >> shift) & 255u));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t cum = 0, dg = 0;
      for (; dg < 256; ++dg) {
        if (cum + hist[dg] > rank) break;
        cum += hist[dg];
      }
      rank -= cum;
      *sh_prefix = prefix | ((uint64_t)dg << shift);
      *sh_rank = rank;
    }
    __syncthreads();
    prefix = *sh_prefix;
    rank = *sh_rank;
    mask |= 255ull << shift;
    __syncthreads();
  }
  return prefix;
}

__global__ void __launch_bounds__(256)
k_sort_large(const uint32_t* __restrict__ starts, const uint64_t* __restrict__ keys, uint64_t nip,
             uint64_t NB, CsrOut o, const uint32_t* __restrict__ list,
             const uint32_t* __restrict__ ctr) {
  __shared__ uint64_t s[LARGE_CAP];
  __shared__ uint32_t hist[256];
  __shared__ uint64_t sh_prefix;
  __shared__ uint32_t sh_rank, sh_cnt;
  const uint32_t count = ctr[1];
  for (uint32_t it = blockIdx.x; it < count; it += gridDim.x) {
    const uint32_t x = list[it];
    const uint32_t tt = (uint32_t)(x / NB), b = (uint32_t)(x - (uint64_t)tt * NB);
    const uint32_t* st = starts + (uint64_t)tt * (NB + 1);
    const uint32_t B = st[b + 1] - st[b];
    const uint32_t* of = o.offs + (uint64_t)tt * (NB + 1);
    const uint32_t k = of[b + 1] - of[b];
    const uint64_t* seg = keys + (uint64_t)tt * nip + st[b];
    if (B <= LARGE_CAP) {
      uint32_t N = 1;
      while (N < B) N <<= 1;
      for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) s[i] = i < B ? seg[i] : ~0ull;
      __syncthreads();
      block_bitonic(s, N);
      for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) csr_put(o, tt, NB, b, j, s[j]);
      __syncthreads();
      continue;
    }
    // radix-select the cut of each CAP-sized chunk of the kept prefix, sort the chunk
    uint64_t lo = 0;
    bool have_lo = false;
    for (uint32_t c0 = 0; c0 < k; c0 += LARGE_CAP) {
      const uint32_t cnt = min(LARGE_CAP, k - c0);
      const uint64_t hi = block_radix_select(seg, B, c0 + cnt - 1, hist, &sh_prefix, &sh_rank);
      if (threadIdx.x == 0) sh_cnt = 0;
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) {
        const uint64_t kk = seg[i];
        if (kk <= hi && (!have_lo || kk > lo)) s[atomicAdd(&sh_cnt, 1u)] = kk;
      }
      __syncthreads();
      uint32_t N = 1;
      while (N < cnt) N <<= 1;
      for (uint32_t i = cnt + threadIdx.x; i < N; i += blockDim.x) s[i] = ~0ull;
      __syncthreads();
      block_bitonic(s, N);
      for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) csr_put(o, tt, NB, b, c0 + j, s[j]);
      __syncthreads();
      lo = hi;
      have_lo = true;
    }
  }
}

// ------------------------------------------------------------ host dispatch
template <int R>
static void launch_hash_R(const Index& ix, const float* X, uint32_t ld, uint64_t n, uint32_t t0,
                          uint32_t T,
                          uint2* ent, uint32_t* counts, cudaStream_t s) {
  const uint32_t P = ix.P;
  uint32_t G = P < 32 ? 1 : P / 32;
  const uint64_t threads = n * G;
  const unsigned blocks = (unsigned)((threads + HB_THREADS - 1) / HB_THREADS);
  const uint32_t K = ix.prm.K, D = ix.prm.D, ip = ix.prm.iprobes;
#define FPP_HASH_CASE(PP)                                                                      \
  case PP: {                                                                                   \
    constexpr int sm = hb_smem_bytes<PP, R>();                                                 \
    if (sm > 48 * 1024) allow_dynamic_smem(k_hash_build<PP, R>);                               \
    k_hash_build<PP, R><<<blocks, HB_THREADS, sm, s>>>(X, n, ix.d, ld, D, K, ix.signs, t0, T, ip, ent, \
                                                counts, ix.NB);                                \
    break;                                                                                     \
  }
  switch (P) {
    FPP_HASH_CASE(2) FPP_HASH_CASE(4) FPP_HASH_CASE(8) FPP_HASH_CASE(16) FPP_HASH_CASE(32)
    FPP_HASH_CASE(64) FPP_HASH_CASE(128) FPP_HASH_CASE(256) FPP_HASH_CASE(512)
    FPP_HASH_CASE(1024)
    default: fail(FPP_ERR_UNSUPPORTED, "build: padded dimension > 1024 not supported on GPU");
  }
#undef FPP_HASH_CASE
  FPP_LAUNCH();
}

static void launch_hash(const Index& ix, const float* X, uint32_t ld, uint64_t n, uint32_t t0,
                        uint32_t T,
                        uint2* ent, uint32_t* counts, cudaStream_t s) {
  const uint32_t r = std::min(ix.prm.iprobes, ix.prm.D);
  if (r <= 4) launch_hash_R<4>(ix, X, ld, n, t0, T, ent, counts, s);
  else if (r <= 8) launch_hash_R<8>(ix, X, ld, n, t0, T, ent, counts, s);
  else launch_hash_R<16>(ix, X, ld, n, t0, T, ent, counts, s);
}

void launch_index_probes(const Index& ix, const float* Xd, uint64_t n, uint32_t t, uint2* out,
                         cudaStream_t s) {
  launch_hash(ix, Xd, ix.d, n, t, 1, out, nullptr, s);
}

void launch_project(const Index& ix, const float* Xd, uint64_t n, uint32_t t, uint32_t f,
                    float* out, cudaStream_t s) {
  const uint32_t P = ix.P;
  uint32_t G = P < 32 ? 1 : P / 32;
  const unsigned blocks = (unsigned)((n * G + 255) / 256);
  const uint32_t* sw = ix.signs + ((uint64_t)t * ix.prm.K + f) * 3 * ix.W;
#define FPP_PROJ_CASE(PP)                                                                       \
  case PP:                                                                                      \
    k_project<PP><<<blocks, 256, 0, s>>>(Xd, n, ix.d, ix.prm.D, sw, out);                      \
    break;
  switch (P) {
    FPP_PROJ_CASE(2) FPP_PROJ_CASE(4) FPP_PROJ_CASE(8) FPP_PROJ_CASE(16) FPP_PROJ_CASE(32)
    FPP_PROJ_CASE(64) FPP_PROJ_CASE(128) FPP_PROJ_CASE(256) FPP_PROJ_CASE(512)
    FPP_PROJ_CASE(1024)
    default: fail(FPP_ERR_UNSUPPORTED, "project: padded dimension > 1024 not supported on GPU");
  }
#undef FPP_PROJ_CASE
  FPP_LAUNCH();
}

void build_tables(Index& ix) {
  const uint32_t L = ix.prm.L, ip = ix.prm.iprobes;
  const uint64_t n = ix.n, NB = ix.NB, nip = n * ip;
  cudaStream_t s = ix.stream;
  if (nip >= (1ull << 32)) fail(FPP_ERR_UNSUPPORTED, "build: n*iProbes must be < 2^32 per shard");
  // scratch per table in one pass
  const uint64_t per_table = nip * (8 + 8) + NB * 4 * 2 + (NB + 1) * 4 + (nip / 2 + 1) * 4 +
                             (nip / (SMALL_MAX + 1) + 1) * 4;
  uint64_t budget = ix.prm.scratch_bytes;
  if (!budget) {
    size_t fr = 0, tot = 0;
    FPP_CUDA(cudaMemGetInfo(&fr, &tot));
    budget = std::min<uint64_t>((uint64_t)(fr * 0.6), 48ull << 30);
  }
  uint32_t T = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(L, budget / per_table));
  while ((uint64_t)T * NB >= (1ull << 32) && T > 1) --T;
  if ((uint64_t)T * NB >= (1ull << 32)) fail(FPP_ERR_UNSUPPORTED, "build: NB too large");

  DBuf<uint2> ent((size_t)T * nip);
  DBuf<uint64_t> keys((size_t)T * nip);
  DBuf<uint32_t> counts((size_t)T * NB);
  DBuf<uint32_t> starts((size_t)T * (NB + 1));
  DBuf<uint32_t> small_list((size_t)T * (nip / 2 + 1));
  DBuf<uint32_t> large_list((size_t)T * (nip / (SMALL_MAX + 1) + 1));
  DBuf<uint32_t> tiles, totals(T), ctr(4);
  DBuf<uint64_t> base_d(T);

  ix.offsets = static_cast<uint32_t*>(dmalloc((size_t)L * (NB + 1) * sizeof(uint32_t)));
  ix.table_base = static_cast<uint64_t*>(dmalloc((size_t)(L + 1) * sizeof(uint64_t)));
  ix.table_base_h.assign(L + 1, 0);
  uint64_t cap = 0;
  std::vector<uint32_t> tot_h(T);
  const int sms = sm_count();
  KeepXform ident{0, 0.f, 1, 0};
  KeepXform keepx{1, ix.prm.alpha, ip, ix.prm.kappa};
  uint32_t max_keep = 0;

  for (uint32_t t0 = 0; t0 < L; t0 += T) {
    const uint32_t Tc = std::min(T, L - t0);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ix.timer.begin(PH_HASH, s, &e0);
    FPP_CUDA(cudaMemsetAsync(counts.p, 0, (size_t)Tc * NB * sizeof(uint32_t), s));
    launch_hash(ix, ix.X, ix.ldx, n, t0, Tc, ent.p, counts.p, s);
    ix.timer.end(PH_HASH, e0, s);
    ix.timer.begin(PH_SORT, s, &e1);
    uint32_t* offs = ix.offsets + (uint64_t)t0 * (NB + 1);
    scan_tables(counts.p, NB, Tc, ident, starts.p, totals.p, tiles, s);
    scan_tables(counts.p, NB, Tc, keepx, offs, totals.p, tiles, s);
    FPP_CUDA(cudaMemcpyAsync(tot_h.data(), totals.p, Tc * sizeof(uint32_t),
                             cudaMemcpyDeviceToHost, s));
    FPP_CUDA(cudaStreamSynchronize(s));
    for (uint32_t tt = 0; tt < Tc; ++tt)
      ix.table_base_h[t0 + tt + 1] = ix.table_base_h[t0 + tt] + tot_h[tt];
    const uint64_t need = ix.table_base_h[t0 + Tc];
    if (need > cap) {  // grow the contiguous CSR arrays, keep built tables
      uint64_t ncap = std::max<uint64_t>(need + need / 2,
                                         need + (uint64_t)(L - t0 - Tc) * tot_h[0]);
      if (t0 + Tc == L) ncap = need;
      uint32_t* nids = static_cast<uint32_t*>(dmalloc((ncap + 1) * sizeof(uint32_t)));
      float* nsc = static_cast<float*>(dmalloc((ncap + 1) * sizeof(float)));
      const uint64_t have = ix.table_base_h[t0];
      if (have) {
        FPP_CUDA(cudaMemcpyAsync(nids, ix.ids, have * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        FPP_CUDA(cudaMemcpyAsync(nsc, ix.scores, have * sizeof(float), cudaMemcpyDeviceToDevice, s));
        FPP_CUDA(cudaStreamSynchronize(s));
      }
      if (ix.ids) dfree(ix.ids);
      if (ix.scores) dfree(ix.scores);
      ix.ids = nids;
      ix.scores = nsc;
      cap = ncap;
    }
    FPP_CUDA(cudaMemcpyAsync(base_d.p, ix.table_base_h.data() + t0, Tc * sizeof(uint64_t),
                             cudaMemcpyHostToDevice, s));
    FPP_CUDA(cudaMemsetAsync(counts.p, 0, (size_t)Tc * NB * sizeof(uint32_t), s));
    FPP_CUDA(cudaMemsetAsync(ctr.p, 0, 4 * sizeof(uint32_t), s));
    {
      const dim3 grid((unsigned)((n + 255) / 256), Tc);
      k_scatter<<<grid, 256, 0, s>>>(ent.p, (uint32_t)n, ip, NB, starts.p, counts.p, keys.p);
      FPP_LAUNCH();
    }
    CsrOut o{offs, base_d.p, ix.ids, ix.scores, nullptr};
    {
      const uint64_t tot = NB * Tc;
      const unsigned blocks = (unsigned)std::min<uint64_t>((tot + 255) / 256, (uint64_t)sms * 32);
      k_classify<<<blocks, 256, 0, s>>>(starts.p, keys.p, nip, Tc, NB, o, small_list.p,
                                        large_list.p, ctr.p, large_list.n);
      FPP_LAUNCH();
    }
    k_sort_small<<<sms * 8, 256, 0, s>>>(starts.p, keys.p, nip, NB, o, small_list.p, ctr.p);
    FPP_LAUNCH();
    k_sort_topk<<<sms * 8, 256, 0, s>>>(starts.p, keys.p, nip, NB, o, large_list.p, ctr.p,
                                        large_list.n);
    FPP_LAUNCH();
    k_sort_large<<<sms * 4, 256, 0, s>>>(starts.p, keys.p, nip, NB, o, large_list.p, ctr.p);
    FPP_LAUNCH();
    uint32_t mk = 0;
    FPP_CUDA(cudaMemcpyAsync(&mk, ctr.p + 2, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    ix.timer.end(PH_SORT, e1, s);
    FPP_CUDA(cudaStreamSynchronize(s));
    max_keep = std::max(max_keep, mk);
  }
  ix.kept_total = ix.table_base_h[L];
  ix.max_bucket = max_keep;
  if (!ix.ids) {
    ix.ids = static_cast<uint32_t*>(dmalloc(sizeof(uint32_t)));
    ix.scores = static_cast<float*>(dmalloc(sizeof(float)));
  }
  FPP_CUDA(cudaMemcpyAsync(ix.table_base, ix.table_base_h.data(), (L + 1) * sizeof(uint64_t),
                           cudaMemcpyHostToDevice, s));
  FPP_CUDA(cudaStreamSynchronize(s));
}


// ------------------------------------------------------ sharded build (8(e) B)
// Global-filter sharding: every shard keeps exactly its part of the 1-GPU
// index.  begin: hash every table, local histogram, every bucket fully sorted
// by (score desc, GLOBAL id asc).  prefix: given the all-reduced histogram,
// export min(keep_g, B_local) sorted keys per bucket into globally agreed
// slots (Sum keep_g, padded with ~0).  finish: from all ranks' slots, the
// bucket's cut = keep_g-th smallest key; keep the local keys <= cut as CSR.
struct ShardState {
  DBuf<uint64_t> sorted;     // [L][nip] bucket segments, sorted
  DBuf<uint32_t> starts;     // [L][NB+1]
  DBuf<uint32_t> hist;       // [L][NB] local
  DBuf<uint32_t> slot_off;   // [L][NB+1] keep_g offsets within a table's slots
  DBuf<uint64_t> slot_base;  // [L]
  std::vector<uint64_t> slot_base_h;
  uint64_t slots = 0;
};

void shard_begin(Index& ix) {
  const uint32_t L = ix.prm.L, ip = ix.prm.iprobes;
  const uint64_t n = ix.n, NB = ix.NB, nip = n * ip;
  cudaStream_t s = ix.stream;
  if (nip >= (1ull << 32)) fail(FPP_ERR_UNSUPPORTED, "build: n*iProbes must be < 2^32 per shard");
  if ((uint64_t)L * NB >= (1ull << 32)) fail(FPP_ERR_UNSUPPORTED, "build: L*NB too large");
  auto* st = new ShardState();
  ix.shard = st;
  DBuf<uint2> ent((size_t)L * nip);
  DBuf<uint64_t> keys((size_t)L * nip);
  st->sorted.alloc((size_t)L * nip);
  st->hist.alloc((size_t)L * NB);
  st->starts.alloc((size_t)L * (NB + 1));
  DBuf<uint32_t> tiles, totals(L), ctr(4), cursor((size_t)L * NB);
  DBuf<uint32_t> small_list((size_t)L * (nip / 2 + 1)), large_list((size_t)L * (nip / (SMALL_MAX + 1) + 1));
  cudaEvent_t e0;
  ix.timer.begin(PH_HASH, s, &e0);
  FPP_CUDA(cudaMemsetAsync(st->hist.p, 0, (size_t)L * NB * 4, s));
  launch_hash(ix, ix.X, ix.ldx, n, 0, L, ent.p, st->hist.p, s);
  ix.timer.end(PH_HASH, e0, s);
  ix.timer.begin(PH_SORT, s, &e0);
  KeepXform ident{0, 0.f, 1, 0};
  scan_tables(st->hist.p, NB, L, ident, st->starts.p, totals.p, tiles, s);
  FPP_CUDA(cudaMemsetAsync(cursor.p, 0, (size_t)L * NB * 4, s));
  FPP_CUDA(cudaMemsetAsync(ctr.p, 0, 16, s));
  const int sms = sm_count();
  {
    const dim3 grid((unsigned)((n + 255) / 256), L);
    k_scatter<<<grid, 256, 0, s>>>(ent.p, (uint32_t)n, ip, NB, st->starts.p, cursor.p, keys.p,
                                   ix.prm.id_offset);
    FPP_LAUNCH();
  }
  std::vector<uint64_t> tb(L);
  for (uint32_t t = 0; t < L; ++t) tb[t] = (uint64_t)t * nip;
  DBuf<uint64_t> tbd(L);
  FPP_CUDA(cudaMemcpyAsync(tbd.p, tb.data(), L * 8, cudaMemcpyHostToDevice, s));
  CsrOut o{st->starts.p, tbd.p, nullptr, nullptr, st->sorted.p};  // keep = B: full sort
  {
    const uint64_t tot = NB * L;
    const unsigned blocks = (unsigned)std::min<uint64_t>((tot + 255) / 256, (uint64_t)sms * 32);
    k_classify<<<blocks, 256, 0, s>>>(st->starts.p, keys.p, nip, L, NB, o, small_list.p,
                                      large_list.p, ctr.p, large_list.n);
    FPP_LAUNCH();
  }
  k_sort_small<<<sms * 8, 256, 0, s>>>(st->starts.p, keys.p, nip, NB, o, small_list.p, ctr.p);
  FPP_LAUNCH();
  k_sort_large<<<sms * 4, 256, 0, s>>>(st->starts.p, keys.p, nip, NB, o, large_list.p, ctr.p);
  FPP_LAUNCH();
  ix.timer.end(PH_SORT, e0, s);
  FPP_CUDA(cudaStreamSynchronize(s));
}

__global__ void k_shard_prefix(const uint32_t* __restrict__ ghist, const uint32_t* __restrict__ lhist,
                               const uint32_t* __restrict__ starts, const uint64_t* __restrict__ sorted,
                               const uint32_t* __restrict__ slot_off,
                               const uint64_t* __restrict__ slot_base, uint32_t L, uint64_t NB,
                               uint64_t nip, KeepXform kx, uint64_t* __restrict__ prefix) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < NB * L;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(x / NB), b = (uint32_t)(x - (uint64_t)t * NB);
    const uint32_t kg = kx(ghist[x]);
    if (!kg) continue;
    const uint32_t bl = lhist[x];
    const uint64_t dst = slot_base[t] + slot_off[(uint64_t)t * (NB + 1) + b];
    const uint64_t src = (uint64_t)t * nip + starts[(uint64_t)t * (NB + 1) + b];
    for (uint32_t j = 0; j < kg; ++j) prefix[dst + j] = j < bl ? sorted[src + j] : ~0ull;
  }
}

// cut = kg-th smallest over `world` sorted runs of kg keys; local kept = #keys <= cut
__global__ void k_shard_cut(const uint32_t* __restrict__ ghist, const uint32_t* __restrict__ lhist,
                            const uint32_t* __restrict__ starts, const uint64_t* __restrict__ sorted,
                            const uint32_t* __restrict__ slot_off,
                            const uint64_t* __restrict__ slot_base, uint64_t slots,
                            const uint64_t* __restrict__ all_prefix, uint32_t world, uint32_t L,
                            uint64_t NB, uint64_t nip, KeepXform kx, uint32_t* __restrict__ kept,
                            uint64_t* __restrict__ cuts) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < NB * L;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(x / NB), b = (uint32_t)(x - (uint64_t)t * NB);
    const uint32_t Bg = ghist[x], kg = kx(Bg), bl = lhist[x];
    uint64_t cut;
    if (kg == 0) cut = 0;
    else if (kg >= Bg) cut = ~0ull;
    else {
      const uint64_t off = slot_base[t] + slot_off[(uint64_t)t * (NB + 1) + b];
      uint32_t ptr[16];
      for (uint32_t r = 0; r < world; ++r) ptr[r] = 0;
      cut = ~0ull;
      for (uint32_t k = 0; k < kg; ++k) {  // k-way merge up to the kg-th key
        uint32_t br = 0;
        uint64_t bk = ~0ull;
        for (uint32_t r = 0; r < world; ++r) {
          const uint64_t v = ptr[r] < kg ? all_prefix[(uint64_t)r * slots + off + ptr[r]] : ~0ull;
          if (v < bk) { bk = v; br = r; }
        }
        ++ptr[br];
        cut = bk;
      }
    }
    cuts[x] = cut;
    // local keys <= cut form a prefix of the sorted local segment
    const uint64_t src = (uint64_t)t * nip + starts[(uint64_t)t * (NB + 1) + b];
    uint32_t lo = 0, hi = bl;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (sorted[src + mid] <= cut) lo = mid + 1;
      else hi = mid;
    }
    kept[x] = kg == 0 ? 0 : lo;
  }
}

__global__ void k_shard_write(const uint32_t* __restrict__ starts, const uint64_t* __restrict__ sorted,
                              const uint32_t* __restrict__ offs, const uint64_t* __restrict__ tbase,
                              uint32_t L, uint64_t NB, uint64_t nip, uint32_t id_sub,
                              uint32_t* __restrict__ ids, float* __restrict__ scores,
                              uint32_t* __restrict__ maxk) {
  uint32_t lm = 0;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < NB * L;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(x / NB), b = (uint32_t)(x - (uint64_t)t * NB);
    const uint32_t* of = offs + (uint64_t)t * (NB + 1);
    const uint32_t k = of[b + 1] - of[b];
    lm = max(lm, k);
    const uint64_t src = (uint64_t)t * nip + starts[(uint64_t)t * (NB + 1) + b];
    const uint64_t dst = tbase[t] + of[b];
    for (uint32_t j = 0; j < k; ++j) {
      const uint64_t key = sorted[src + j];
      ids[dst + j] = (uint32_t)(key & 0xffffffffu) - id_sub;
      scores[dst + j] = desc_score_val(key);
    }
  }
  for (int o2 = 16; o2 > 0; o2 >>= 1) lm = max(lm, __shfl_xor_sync(FULL, lm, o2));
  if ((threadIdx.x & 31) == 0 && lm) atomicMax(maxk, lm);
}

uint64_t shard_slots(Index& ix, const uint32_t* ghist) {
  ShardState* st = ix.shard;
  if (!st) fail(FPP_ERR_INVALID_ARGUMENT, "shard: fpp_shard_begin was not called");
  const uint32_t L = ix.prm.L;
  const uint64_t NB = ix.NB;
  cudaStream_t s = ix.stream;
  KeepXform kx{1, ix.prm.alpha, ix.prm.iprobes, ix.prm.kappa};
  st->slot_off.ensure((size_t)L * (NB + 1));
  DBuf<uint32_t> tiles, totals(L);
  scan_tables(ghist, NB, L, kx, st->slot_off.p, totals.p, tiles, s);
  std::vector<uint32_t> th(L);
  FPP_CUDA(cudaMemcpyAsync(th.data(), totals.p, L * 4, cudaMemcpyDeviceToHost, s));
  FPP_CUDA(cudaStreamSynchronize(s));
  st->slot_base_h.assign(L + 1, 0);
  for (uint32_t t = 0; t < L; ++t) st->slot_base_h[t + 1] = st->slot_base_h[t] + th[t];
  st->slot_base.ensure(L + 1);
  FPP_CUDA(cudaMemcpyAsync(st->slot_base.p, st->slot_base_h.data(), (L + 1) * 8,
                           cudaMemcpyHostToDevice, s));
  st->slots = st->slot_base_h[L];
  return st->slots;
}

void shard_prefix(Index& ix, const uint32_t* ghist, uint64_t* prefix) {
  ShardState* st = ix.shard;
  if (!st || !st->slot_off.p) fail(FPP_ERR_INVALID_ARGUMENT, "shard: call fpp_shard_slots first");
  const uint32_t L = ix.prm.L;
  KeepXform kx{1, ix.prm.alpha, ix.prm.iprobes, ix.prm.kappa};
  const unsigned blocks = (unsigned)std::min<uint64_t>((ix.NB * L + 255) / 256, (uint64_t)sm_count() * 32);
  k_shard_prefix<<<blocks, 256, 0, ix.stream>>>(ghist, st->hist.p, st->starts.p, st->sorted.p,
                                                st->slot_off.p, st->slot_base.p, L, ix.NB,
                                                ix.n * ix.prm.iprobes, kx, prefix);
  FPP_LAUNCH();
  FPP_CUDA(cudaStreamSynchronize(ix.stream));
}

void shard_finish(Index& ix, const uint32_t* ghist, const uint64_t* all_prefix, uint32_t world) {
  ShardState* st = ix.shard;
  if (!st || !st->slot_off.p) fail(FPP_ERR_INVALID_ARGUMENT, "shard: call fpp_shard_slots first");
  if (world == 0 || world > 16) fail(FPP_ERR_UNSUPPORTED, "shard: world size must be 1..16");
  const uint32_t L = ix.prm.L;
  const uint64_t NB = ix.NB, nip = ix.n * ix.prm.iprobes;
  cudaStream_t s = ix.stream;
  KeepXform kx{1, ix.prm.alpha, ix.prm.iprobes, ix.prm.kappa};
  KeepXform ident{0, 0.f, 1, 0};
  DBuf<uint32_t> kept((size_t)L * NB), tiles, totals(L), mk(1);
  DBuf<uint64_t> cuts((size_t)L * NB);
  const unsigned blocks = (unsigned)std::min<uint64_t>((NB * L + 255) / 256, (uint64_t)sm_count() * 32);
  k_shard_cut<<<blocks, 256, 0, s>>>(ghist, st->hist.p, st->starts.p, st->sorted.p, st->slot_off.p,
                                     st->slot_base.p, st->slots, all_prefix, world, L, NB, nip, kx,
                                     kept.p, cuts.p);
  FPP_LAUNCH();
  ix.offsets = static_cast<uint32_t*>(dmalloc((size_t)L * (NB + 1) * sizeof(uint32_t)));
  scan_tables(kept.p, NB, L, ident, ix.offsets, totals.p, tiles, s);
  std::vector<uint32_t> th(L);
  FPP_CUDA(cudaMemcpyAsync(th.data(), totals.p, L * 4, cudaMemcpyDeviceToHost, s));
  FPP_CUDA(cudaStreamSynchronize(s));
  ix.table_base_h.assign(L + 1, 0);
  for (uint32_t t = 0; t < L; ++t) ix.table_base_h[t + 1] = ix.table_base_h[t] + th[t];
  ix.kept_total = ix.table_base_h[L];
  ix.table_base = static_cast<uint64_t*>(dmalloc((size_t)(L + 1) * sizeof(uint64_t)));
  FPP_CUDA(cudaMemcpyAsync(ix.table_base, ix.table_base_h.data(), (L + 1) * 8,
                           cudaMemcpyHostToDevice, s));
  ix.ids = static_cast<uint32_t*>(dmalloc((ix.kept_total + 1) * sizeof(uint32_t)));
  ix.scores = static_cast<float*>(dmalloc((ix.kept_total + 1) * sizeof(float)));
  FPP_CUDA(cudaMemsetAsync(mk.p, 0, 4, s));
  k_shard_write<<<blocks, 256, 0, s>>>(st->starts.p, st->sorted.p, ix.offsets, ix.table_base, L, NB,
                                       nip, ix.prm.id_offset, ix.ids, ix.scores, mk.p);
  FPP_LAUNCH();
  uint32_t mx = 0;
  FPP_CUDA(cudaMemcpyAsync(&mx, mk.p, 4, cudaMemcpyDeviceToHost, s));
  FPP_CUDA(cudaStreamSynchronize(s));
  ix.max_bucket = mx;
  delete st;
  ix.shard = nullptr;
}

const uint32_t* shard_hist_ptr(const Index& ix) { return ix.shard->hist.p; }

void shard_release(Index& ix) {
  delete ix.shard;
  ix.shard = nullptr;
}

}  // namespace fpp
