// fpp_brute.cu -- exact brute-force top-k over the index's resident dataset:
// the recall ground truth (SPEC.md:490-503 brute_force_topk).
//
// Scores are `inner_product` (dataset.cpp:61-69) bit for bit: each (row, query)
// pair accumulates double(x_j) * double(q_j) with fp64 FMAs in j order (the
// products are exact, so fma(x, q, acc) == acc + x*q rounded once).  Top-k
// order is (score desc, id asc), ties to the lower id as SPEC requires.
//
//   k_brute  grid (row split, 16-query tile).  A warp streams 32 rows at a time
//            through a cp.async ring of 32-float column slices (as k_score); lane
//            r folds row r into 16 fp64 accumulators, one per query of the tile,
//            whose operands are shared-memory broadcasts.  Per query a warp
//            register top-k; the CTA merges its warps and writes the split's
//            partial list.
//   k_brute_merge  warp per query: merges the splits' partial lists.
#include <cstdio>

#include "fpp_device.cuh"
#include "fpp_internal.h"

namespace fpp {

constexpr int BF_WARPS = 4;
constexpr int BF_QT = 16;       // queries per tile
constexpr int BF_SLICE = 32;    // floats per row slice
constexpr int BF_STAGES = 2;
constexpr int BF_ROWPAD = BF_SLICE + 4;
constexpr int BF_STAGE_FLOATS = 32 * BF_ROWPAD;

__device__ __forceinline__ bool bf_better(double s1, uint32_t i1, double s2, uint32_t i2) {
  return s1 > s2 || (s1 == s2 && i1 < i2);
}
// warp top-k list (lane i < k holds the i-th best): insert the lanes' candidates
__device__ __forceinline__ void bf_insert(double& bs, uint32_t& bi, uint32_t k, double cs,
                                          uint32_t ci, bool valid) {
  const int lane = threadIdx.x & 31;
  double ws = __shfl_sync(FULL, bs, k - 1);
  uint32_t wi = __shfl_sync(FULL, bi, k - 1);
  unsigned m = __ballot_sync(FULL, valid && bf_better(cs, ci, ws, wi));
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const double s = __shfl_sync(FULL, cs, src);
    const uint32_t i = __shfl_sync(FULL, ci, src);
    ws = __shfl_sync(FULL, bs, k - 1);
    wi = __shfl_sync(FULL, bi, k - 1);
    if (!bf_better(s, i, ws, wi)) continue;
    const int pos = __popc(__ballot_sync(FULL, (uint32_t)lane < k && bf_better(bs, bi, s, i)));
    const double us = __shfl_up_sync(FULL, bs, 1);
    const uint32_t ui = __shfl_up_sync(FULL, bi, 1);
    if (lane > pos && (uint32_t)lane < k) { bs = us; bi = ui; }
    if (lane == pos) { bs = s; bi = i; }
  }
}

__device__ __forceinline__ void bf_cp16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void bf_cp4(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}

struct BruteArgs {
  const float* X;
  uint64_t n;
  uint32_t d;
  uint32_t ldx;  // row stride of X (floats)
  const float* Q;
  uint32_t nq, k;
  uint64_t rows_per_split;
  uint32_t* part_ids;     // [split][nq][k]
  double* part_scores;
  // k > 32: pass p keeps ranks [32p, 32p + k) -- the k best rows that come strictly
  // after the previous pass's last answer entry (the cursor) in (score desc, id asc)
  const uint32_t* cur_ids;  // answer rows [nq][ostride] (global ids); nullptr on pass 0
  const double* cur_scores;
  uint32_t ostride, ooff, id_offset;
};

template <bool VEC>
__global__ void __launch_bounds__(BF_WARPS * 32) k_brute(BruteArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const uint32_t d = a.d;
  double* qd = reinterpret_cast<double*>(smraw);  // [d][BF_QT] (query-minor: one LDS.128 per 2)
  float* ring = reinterpret_cast<float*>(smraw + (size_t)d * BF_QT * 8);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t split = blockIdx.x, q0 = blockIdx.y * BF_QT;
  const uint32_t nqt = min((uint32_t)BF_QT, a.nq - q0);
  for (uint32_t i = threadIdx.x; i < d * BF_QT; i += blockDim.x) {
    const uint32_t j = i / BF_QT, qi = i - j * BF_QT;
    qd[i] = qi < nqt ? (double)a.Q[(uint64_t)(q0 + qi) * d + j] : 0.0;
  }
  // per-query cursor: (+inf, 0) admits every row (pass 0), (-inf, 0) none (the rows ran out)
  __shared__ double cur_s[BF_QT];
  __shared__ uint32_t cur_i[BF_QT];
  if (threadIdx.x < BF_QT) {
    double cs = INFINITY;
    uint32_t ci = 0;
    if (a.cur_ids && threadIdx.x < nqt) {
      const uint64_t o = (uint64_t)(q0 + threadIdx.x) * a.ostride + a.ooff - 1;
      const uint32_t g = a.cur_ids[o];
      cs = g == 0xffffffffu ? -INFINITY : a.cur_scores[o];
      ci = g == 0xffffffffu ? 0u : g - a.id_offset;
    }
    cur_s[threadIdx.x] = cs;
    cur_i[threadIdx.x] = ci;
  }
  __syncthreads();
  const uint64_t r_begin = (uint64_t)split * a.rows_per_split;
  const uint64_t r_end = min(a.n, r_begin + a.rows_per_split);
  const uint32_t k = a.k;
  double bs[BF_QT];
  uint32_t bi[BF_QT];
#pragma unroll
  for (int qi = 0; qi < BF_QT; ++qi) { bs[qi] = -INFINITY; bi[qi] = 0xffffffffu; }
  float* wring = ring + (size_t)w * BF_STAGES * BF_STAGE_FLOATS;
  const uint32_t nsl = (d + BF_SLICE - 1) / BF_SLICE;
  const uint64_t nb = (r_end > r_begin) ? (r_end - r_begin + 31) / 32 : 0;
  const int kk = lane & 7, rbase = lane >> 3;
  // issue cursor over (batch, slice)
  uint64_t ib = w;
  uint32_t ic = 0, nissued = 0;
  auto issue = [&]() {
    if (ib < nb) {
      float* buf = wring + (size_t)(nissued % BF_STAGES) * BF_STAGE_FLOATS;
      const uint32_t col0 = ic * BF_SLICE;
      const uint32_t len = min((uint32_t)BF_SLICE, d - col0);
      const uint64_t row0 = r_begin + ib * 32;
      if (VEC) {
        if ((uint32_t)kk < (len >> 2)) {
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const uint64_t row = row0 + rbase + 4 * it;
            if (row < r_end)
              bf_cp16(buf + (rbase + 4 * it) * BF_ROWPAD + kk * 4, a.X + row * a.ldx + col0 + kk * 4);
          }
        }
      } else {
        for (int r = 0; r < 32; ++r) {
          const uint64_t row = row0 + r;
          if (row < r_end)
            for (uint32_t c = lane; c < len; c += 32)
              bf_cp4(buf + r * BF_ROWPAD + c, a.X + row * a.ldx + col0 + c);
        }
      }
      if (++ic == nsl) {
        ic = 0;
        ib += BF_WARPS;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    ++nissued;
  };
#pragma unroll
  for (int st = 0; st < BF_STAGES - 1; ++st) issue();
  double acc[BF_QT];
#pragma unroll
  for (int qi = 0; qi < BF_QT; ++qi) acc[qi] = 0.0;
  uint64_t cb = w;
  uint32_t cc = 0, ncomp = 0;
  while (cb < nb) {
    issue();
    asm volatile("cp.async.wait_group %0;\n" ::"n"(BF_STAGES - 1) : "memory");
    __syncwarp();
    const float* row = wring + (size_t)(ncomp % BF_STAGES) * BF_STAGE_FLOATS + lane * BF_ROWPAD;
    const uint32_t col0 = cc * BF_SLICE;
    const uint32_t len = min((uint32_t)BF_SLICE, d - col0);
    // dataset.cpp:67 acc += double(a[i]) * double(b[i]), sequential i, per query
    for (uint32_t j = 0; j < len; ++j) {
      const double x = (double)row[j];
      const double* qj = qd + (size_t)(col0 + j) * BF_QT;
#pragma unroll
      for (int qi = 0; qi < BF_QT; qi += 2) {
        const double2 qq = *reinterpret_cast<const double2*>(qj + qi);
        acc[qi] = fma(x, qq.x, acc[qi]);
        acc[qi + 1] = fma(x, qq.y, acc[qi + 1]);
      }
    }
    __syncwarp();
    ++ncomp;
    if (++cc == nsl) {
      const uint64_t rid = r_begin + cb * 32 + lane;
      const bool valid = rid < r_end;
#pragma unroll
      for (int qi = 0; qi < BF_QT; ++qi) {
        const double cs = cur_s[qi];
        const bool after = cs > acc[qi] || (cs == acc[qi] && cur_i[qi] < (uint32_t)rid);
        bf_insert(bs[qi], bi[qi], k, acc[qi], (uint32_t)rid, valid && (uint32_t)qi < nqt && after);
        acc[qi] = 0.0;
      }
      cc = 0;
      cb += BF_WARPS;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();  // the ring is free: it holds the warps' lists for the merge
  double* mg_s = reinterpret_cast<double*>(ring);                        // [w][qi][32]
  uint32_t* mg_i = reinterpret_cast<uint32_t*>(mg_s + BF_WARPS * BF_QT * 32);
#pragma unroll
  for (int qi = 0; qi < BF_QT; ++qi) {
    mg_s[(w * BF_QT + qi) * 32 + lane] = bs[qi];
    mg_i[(w * BF_QT + qi) * 32 + lane] = bi[qi];
  }
  __syncthreads();
  // warp w merges queries w, w + BF_WARPS, ... of the tile
  for (uint32_t qi = w; qi < nqt; qi += BF_WARPS) {
    double s = mg_s[qi * 32 + lane];
    uint32_t i = mg_i[qi * 32 + lane];
    for (int w2 = 1; w2 < BF_WARPS; ++w2) {
      const uint32_t o = (w2 * BF_QT + qi) * 32 + lane;
      bf_insert(s, i, k, mg_s[o], mg_i[o], (uint32_t)lane < k && mg_i[o] != 0xffffffffu);
    }
    if ((uint32_t)lane < k) {
      const uint64_t o = ((uint64_t)split * a.nq + q0 + qi) * k + lane;
      a.part_ids[o] = i;
      a.part_scores[o] = s;
    }
  }
}

__global__ void __launch_bounds__(256) k_brute_merge(const uint32_t* __restrict__ part_ids,
                                                     const double* __restrict__ part_scores,
                                                     uint32_t splits, uint32_t nq, uint32_t k,
                                                     uint32_t id_offset, uint32_t* out_ids,
                                                     double* out_scores, uint32_t ostride,
                                                     uint32_t ooff) {
  const int lane = threadIdx.x & 31;
  const uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  double bs = -INFINITY;
  uint32_t bi = 0xffffffffu;
  for (uint32_t sp = 0; sp < splits; ++sp) {
    const bool in = (uint32_t)lane < k;
    const uint64_t o = ((uint64_t)sp * nq + q) * k + (in ? lane : 0);
    const double s = in ? part_scores[o] : -INFINITY;
    const uint32_t i = in ? part_ids[o] : 0xffffffffu;
    bf_insert(bs, bi, k, s, i, in && i != 0xffffffffu);
  }
  if ((uint32_t)lane < k) {
    const bool ok = bi != 0xffffffffu;
    out_ids[(uint64_t)q * ostride + ooff + lane] = ok ? bi + id_offset : 0xffffffffu;
    out_scores[(uint64_t)q * ostride + ooff + lane] = ok ? bs : -INFINITY;
  }
}

void run_brute_force(const Index& ix, const float* Qd, uint64_t nq, uint32_t k, uint32_t* ids_d,
                     double* scores_d, cudaStream_t s) {
  if (nq == 0) return;
  const uint32_t d = ix.d;
  const uint32_t tiles = (uint32_t)((nq + BF_QT - 1) / BF_QT);
  // enough (split, tile) CTAs to fill the GPU a few times over
  const uint64_t want = (uint64_t)sm_count() * 8;
  uint64_t splits = std::max<uint64_t>(1, (want + tiles - 1) / tiles);
  splits = std::min<uint64_t>(splits, (ix.n + 1023) / 1024);
  splits = std::max<uint64_t>(splits, 1);
  const uint64_t rows_per_split = (ix.n + splits - 1) / splits;
  const uint32_t kp_max = std::min<uint32_t>(k, 32);
  DBuf<uint32_t> pids((size_t)splits * nq * kp_max);
  DBuf<double> psc((size_t)splits * nq * kp_max);
  static_assert(BF_WARPS * BF_QT * 32 * 12 <= BF_WARPS * BF_STAGES * BF_STAGE_FLOATS * 4,
                "merge lists must fit in the ring");
  const size_t smem = (size_t)d * BF_QT * 8 + (size_t)BF_WARPS * BF_STAGES * BF_STAGE_FLOATS * 4;
  const dim3 grid((unsigned)splits, tiles);
  // k > 32: one pass over X per 32 ranks (the warp lists hold 32 entries)
  for (uint32_t off = 0; off < k; off += 32) {
    const uint32_t kp = std::min<uint32_t>(32, k - off);
    BruteArgs a{ix.X, ix.n, d, ix.ldx, Qd, (uint32_t)nq, kp, rows_per_split, pids.p, psc.p,
                off ? ids_d : nullptr, scores_d, k, off, ix.prm.id_offset};
    if ((d & 3u) == 0) {
      allow_dynamic_smem(k_brute<true>);
      k_brute<true><<<grid, BF_WARPS * 32, smem, s>>>(a);
    } else {
      allow_dynamic_smem(k_brute<false>);
      k_brute<false><<<grid, BF_WARPS * 32, smem, s>>>(a);
    }
    FPP_LAUNCH();
    k_brute_merge<<<(unsigned)((nq + 7) / 8), 256, 0, s>>>(pids.p, psc.p, (uint32_t)splits,
                                                            (uint32_t)nq, kp, ix.prm.id_offset, ids_d,
                                                            scores_d, k, off);
    FPP_LAUNCH();
  }
  FPP_CUDA(cudaStreamSynchronize(s));  // scratch is freed on return
}

}  // namespace fpp
