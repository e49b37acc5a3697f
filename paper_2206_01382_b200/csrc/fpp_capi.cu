// fpp_capi.cu -- the C ABI (include/falconnpp.h): validation with the
// reference's error classes, device ownership, host<->device staging, and the
// host helpers (normalize, synthetic data).  No CPU compute fallback: every
// compute entry point runs the CUDA kernels or fails with FPP_ERR_CUDA.
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <new>
#include <string>
#include <vector>

#include <cuda_fp16.h>

#include "fpp_device.cuh"
#include "fpp_internal.h"

namespace fpp {

static thread_local std::string g_err;

void fail(int code, const std::string& msg) { throw Error(code, msg); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  const int code = e == cudaErrorMemoryAllocation ? FPP_ERR_OUT_OF_MEMORY : FPP_ERR_CUDA;
  fail(code, std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + what + " (" + file +
                 ":" + std::to_string(line) + ")");
}

void* dmalloc(size_t bytes) {
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, bytes ? bytes : 1);
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? FPP_ERR_OUT_OF_MEMORY : FPP_ERR_CUDA,
         "cudaMalloc(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  }
  return p;
}
void dfree(void* p) {
  if (p) cudaFree(p);
}

cudaEvent_t PhaseTimer::get() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  FPP_CUDA(cudaEventCreate(&e));
  return e;
}
void PhaseTimer::begin(int, cudaStream_t s, cudaEvent_t* out) {
  *out = get();
  FPP_CUDA(cudaEventRecord(*out, s));
}
void PhaseTimer::end(int ph, cudaEvent_t start, cudaStream_t s) {
  cudaEvent_t e = get();
  FPP_CUDA(cudaEventRecord(e, s));
  open.push_back({ph, {start, e}});
}
void PhaseTimer::collect(double* ms) {
  for (auto& o : open) {
    cudaEventSynchronize(o.second.second);
    float t = 0.f;
    if (cudaEventElapsedTime(&t, o.second.first, o.second.second) == cudaSuccess) ms[o.first] += t;
    pool.push_back(o.second.first);
    pool.push_back(o.second.second);
  }
  open.clear();
}
PhaseTimer::~PhaseTimer() {
  for (auto& o : open) {
    cudaEventDestroy(o.second.first);
    cudaEventDestroy(o.second.second);
  }
  for (auto e : pool) cudaEventDestroy(e);
}

Index::~Index() {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  for (QueryCtx* c : ctx_all) delete c;
  ctx_all.clear();
  ctx_free.clear();
  dfree(X);
  dfree(signs);
  dfree(sigs);
  dfree(xtail);
  dfree(q8rec);
  dfree(q8csr);
  dfree(offsets);
  dfree(table_base);
  dfree(ids);
  dfree(scores);
  if (shard) shard_release(*this);
  if (h_pinned) cudaFreeHost(h_pinned);
  score_bytes_d.release();
  if (stream) cudaStreamDestroy(stream);
  cudaSetDevice(cur);
}

void QueryCtx::QSlot::release() {
  vals.release(); codes.release(); ppos.release(); plen.release(); gbuf.release();
  ckey.release(); cpair.release(); dbgclk.release(); eq.release(); coff.release();
  uq.release(); uniq.release(); cands.release(); bitmap.release(); counter.release();
  qsig.release(); cands2.release(); uq2.release(); wlog.release(); allsc.release();
  if (pinned) cudaFreeHost(pinned);
  if (ev_probe) cudaEventDestroy(ev_probe);
  if (ev_bdone) cudaEventDestroy(ev_bdone);
  ev_bdone = nullptr;
  pinned = nullptr;
  ev_probe = nullptr;
}

QueryCtx::~QueryCtx() {
  if (done_recorded) cudaEventSynchronize(ev_done);
  if (sA) cudaStreamSynchronize(sA);
  if (sB) cudaStreamSynchronize(sB);
  if (own) cudaStreamSynchronize(own);
  for (auto& sl : slot) sl.release();
  for (cudaEvent_t e : {ev_fork, ev_join, ev_join2, ev_done, prune_ev})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t t : {sA, sB, own})
    if (t) cudaStreamDestroy(t);
  if (prune_h) cudaFreeHost(prune_h);
}

CtxLease::CtxLease(const Index& ix_) : ix(ix_), c(nullptr) {
  {
    std::lock_guard<std::mutex> lk(ix.mu);
    if (!ix.ctx_free.empty()) {
      c = ix.ctx_free.back();
      ix.ctx_free.pop_back();
    }
  }
  if (c) return;
  auto* n = new QueryCtx();
  try {
    n->device = ix.device;
    int lo = 0, hi = 0;
    FPP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    FPP_CUDA(cudaStreamCreateWithPriority(&n->sA, cudaStreamNonBlocking, lo));
    FPP_CUDA(cudaStreamCreateWithPriority(&n->sB, cudaStreamNonBlocking, hi));
    FPP_CUDA(cudaStreamCreateWithFlags(&n->own, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&n->ev_fork, &n->ev_join, &n->ev_join2, &n->ev_done})
      FPP_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    for (auto& sl : n->slot) {
      FPP_CUDA(cudaEventCreateWithFlags(&sl.ev_probe, cudaEventDisableTiming));
      FPP_CUDA(cudaEventCreateWithFlags(&sl.ev_bdone, cudaEventDisableTiming));
      FPP_CUDA(cudaMallocHost(&sl.pinned, 64));
    }
  } catch (...) {
    delete n;
    throw;
  }
  std::lock_guard<std::mutex> lk(ix.mu);
  ix.ctx_all.push_back(n);
  c = n;
}

CtxLease::~CtxLease() {
  {
    std::lock_guard<std::mutex> lk(ix.mu);
    ix.ctx_free.push_back(c);
  }
  ix.ctx_cv.notify_all();
}

void collect_query_timings(const Index& ix) {
  std::unique_lock<std::mutex> lk(ix.mu);
  ix.ctx_cv.wait(lk, [&] { return ix.ctx_free.size() == ix.ctx_all.size(); });
  for (QueryCtx* c : ix.ctx_all) {
    double ms[PH_COUNT] = {0};
    c->timer.collect(ms);
    ix.acc.qhash_ms += ms[PH_QHASH];
    ix.acc.probe_ms += ms[PH_PROBE];
    ix.acc.collect_ms += ms[PH_COLLECT];
    ix.acc.score_ms += ms[PH_SCORE];
    ix.acc.launches += c->acc.launches;
    ix.acc.probes += c->acc.probes;
    ix.acc.score_launches += c->acc.score_launches;
    c->acc = fpp_timings{};
  }
}

uint64_t host_mix64(uint64_t z) {  // common.hpp:18-23
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
uint64_t host_derive_seed(uint64_t m, uint64_t a, uint64_t b, uint64_t c) {  // common.hpp:27-34
  uint64_t h = host_mix64(m);
  h = host_mix64(h ^ (a * 0xff51afd7ed558ccdULL));
  h = host_mix64(h ^ (b * 0xc4ceb9fe1a85ec53ULL));
  h = host_mix64(h ^ (c * 0xd6e8feb86659fd93ULL));
  return h;
}

// Sign bitmasks [L][K][3][W]: bit e of word g of round s is the sign of index
// sign_index<P>(s, e, g) of that round's P signs of the stack's stream (rotation.cpp:55-67;
// bit = 1 -> +1): layout A (index 32g + e), except rounds 1 and 2 of the shuffle FHT plan,
// whose words are in layout B (fpp_device.cuh).
template <int P>
static void pack_words(const std::vector<uint8_t>& bits, uint32_t* out) {
  constexpr uint32_t W = P < 32 ? 1 : P / 32;
  constexpr int EPT = P < 32 ? P : 32;
  for (int s = 0; s < 3; ++s)
    for (int g = 0; g < (int)W; ++g)
      for (int e = 0; e < EPT; ++e)
        if (bits[(size_t)s * P + sign_index<P>(s, e, g)]) out[s * W + g] |= 1u << e;
}

void pack_signs(const fpp_params& p, uint32_t P, std::vector<uint32_t>& words) {
  const uint32_t W = P < 32 ? 1 : P / 32;
  words.assign((size_t)p.L * p.K * 3 * W, 0u);
  std::vector<uint8_t> bits(3 * (size_t)P);
  for (uint32_t t = 0; t < p.L; ++t)
    for (uint32_t f = 0; f < p.K; ++f) {
      uint64_t state = host_derive_seed(p.seed, t, f, 0), word = 0;
      int left = 0;
      for (size_t i = 0; i < bits.size(); ++i) {
        if (left == 0) { word = host_mix64(state++); left = 64; }
        bits[i] = (uint8_t)(word & 1u);
        word >>= 1;
        --left;
      }
      uint32_t* out = words.data() + ((size_t)t * p.K + f) * 3 * W;
      switch (P) {
        case 1: pack_words<1>(bits, out); break;
        case 2: pack_words<2>(bits, out); break;
        case 4: pack_words<4>(bits, out); break;
        case 8: pack_words<8>(bits, out); break;
        case 16: pack_words<16>(bits, out); break;
        case 32: pack_words<32>(bits, out); break;
        case 64: pack_words<64>(bits, out); break;
        case 128: pack_words<128>(bits, out); break;
        case 256: pack_words<256>(bits, out); break;
        case 512: pack_words<512>(bits, out); break;
        case 1024: pack_words<1024>(bits, out); break;
        default: fail(FPP_ERR_UNSUPPORTED, "pack_signs: padded dimension > 1024 not supported on GPU");
      }
    }
}

static uint32_t isqrt_ceil(uint64_t q) {
  uint64_t r = (uint64_t)std::sqrt((double)q);
  while (r * r > q) --r;
  while (r * r < q) ++r;
  return (uint32_t)r;
}

// SPEC.md:211 per-function cap; K=1 uses min(2D, qProbes)
uint32_t query_cap(const Index& ix, uint32_t qprobes) {
  const uint64_t D2 = 2ull * ix.prm.D;
  const uint64_t s = ix.prm.K == 2 ? 2ull * isqrt_ceil(qprobes) : qprobes;
  return (uint32_t)std::min(s, D2);
}
uint64_t query_probes(const Index& ix, uint32_t qprobes) {
  const uint64_t s = query_cap(ix, qprobes);
  const uint64_t avail = (uint64_t)ix.prm.L * (ix.prm.K == 2 ? s * s : s);
  return std::min<uint64_t>(qprobes, avail);
}

int smem_optin_max() {
  static int v = -1;
  if (v < 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    v = optin;
  }
  return v;
}

int sm_count() {
  static int v = -1;
  if (v < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

// center(Dataset) (dataset.cpp:40-57) on the device: thread per coordinate, the
// rows summed in order in double (so the mean is the reference's bit for bit),
// center = float(mean / n); then rows -= center in fp32.
__global__ void k_center_mean(const float* __restrict__ X, uint64_t n, uint32_t d, uint32_t ldx,
                              float* __restrict__ center) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  double m = 0.0;
  for (uint64_t i = 0; i < n; ++i) m += (double)X[i * ldx + j];
  center[j] = (float)(m / (double)n);
}
__global__ void k_center_sub(float* __restrict__ X, uint64_t n, uint32_t d, uint32_t ldx,
                             const float* __restrict__ center) {
  const uint64_t cnt = n * d;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = e / d;
    const uint32_t j = (uint32_t)(e - i * d);
    X[i * ldx + j] -= center[j];
  }
}

// Row tail norms (score-gather early termination, fpp_query.cu k_score_pruned):
// warp per row; fp64 sums of exact squares per segment, suffix-combined; sqrt
// rounded up to fp32 (with a 1e-12 relative margin for the summation error).
__global__ void k_tail_norms(const float* __restrict__ X, uint64_t n, uint32_t d, uint32_t ldx,
                             uint32_t nt, uint32_t head, float* __restrict__ xt) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
    const float* r = X + i * ldx;
    double seg[XT_MAX] = {0.0, 0.0, 0.0, 0.0};
    for (uint32_t c = head + lane; c < d; c += 32) {
      const uint32_t j = min((c - head) / XT_SLICE, nt - 1);
      const double v = (double)r[c];
#pragma unroll
      for (uint32_t t = 0; t < XT_MAX; ++t)
        if (t == j) seg[t] = fma(v, v, seg[t]);
    }
    double suf = 0.0;
#pragma unroll
    for (int t = XT_MAX - 1; t >= 0; --t) {
      double v = seg[t];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      suf += v;
      if (lane == 0 && t < (int)nt) xt[(uint64_t)t * n + i] = __double2float_ru(__dsqrt_ru(suf) * (1.0 + 1e-12));
    }
  }
}

// Screening records for k_score_screen (warp per row; layout: fpp_internal.h Q8A/Q8B).
// Stage A covers dims [0, 20), stage B dims [20, 116): int8 codes with the stage's
// scale s = max|x_i| / 127 (stage A: rounded up to an fp16-exact value, the records
// keep it in fp16), codes rint(x_i / s); then, in fp64 and rounded up (x 1+1e-12):
// r = ||x_h - s code|| (quantization error), m = ||s code|| and t = ||x[hi : d)||
// (everything after the stage).  The score kernel bounds the stage's part of x.q by
// s_q s I + r ||q_h|| + m ||q_h - q~_h|| (I = the integer dot product of the codes)
// and the rest by t ||q_t|| (Cauchy-Schwarz).
__global__ void k_q8_records(const float* __restrict__ X, uint64_t n, uint32_t d, uint32_t ldx,
                             uint4* __restrict__ rec) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
    const float* r = X + i * ldx;
#pragma unroll
    for (uint32_t stage = 0; stage < 2; ++stage) {
      const uint32_t W = stage ? Q8B_DIMS : Q8A_DIMS;  // code bytes
      const uint32_t lo = stage ? Q8A_DIMS : 0u, hi = min(d, lo + W);
      float x[3];
      float mx = 0.f;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const uint32_t k = lane + 32 * j;
        x[j] = (k < W && lo + k < hi) ? r[lo + k] : 0.f;
        mx = fmaxf(mx, fabsf(x[j]));
      }
      for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float sc = stage == 0 ? __half2float(__float2half_ru(mx / 127.0f)) : mx / 127.0f;
      double er = 0.0, mm = 0.0, tt = 0.0;
      int c[3];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        c[j] = sc > 0.f ? max(-127, min(127, __float2int_rn(x[j] / sc))) : 0;
        const double e = (double)x[j] - (double)sc * c[j], m = (double)sc * c[j];
        er = fma(e, e, er);
        mm = fma(m, m, mm);
      }
      for (uint32_t j = lo + W + lane; j < d; j += 32) tt = fma((double)r[j], (double)r[j], tt);
      for (int o = 16; o; o >>= 1) {
        er += __shfl_xor_sync(0xffffffffu, er, o);
        mm += __shfl_xor_sync(0xffffffffu, mm, o);
        tt += __shfl_xor_sync(0xffffffffu, tt, o);
      }
      unsigned char* rb = reinterpret_cast<unsigned char*>(stage ? rec + (uint64_t)n * 2 + i * 8 : rec + i * 2);
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (lane + 32 * j < (int)W) rb[lane + 32 * j] = (unsigned char)(signed char)c[j];
      if (lane == 0) {
        const float rr = __double2float_ru(__dsqrt_ru(er) * (1.0 + 1e-12));
        const float m2 = __double2float_ru(__dsqrt_ru(mm) * (1.0 + 1e-12));
        const float t2 = __double2float_ru(__dsqrt_ru(tt) * (1.0 + 1e-12));
        if (stage == 0) {  // bytes 20..31: id slot, {s, r}, {m, t} half2
          const __half2 sr = __halves2half2(__float2half_ru(sc), __float2half_ru(rr));
          const __half2 mt = __halves2half2(__float2half_ru(m2), __float2half_ru(t2));
          uint32_t* w32 = reinterpret_cast<uint32_t*>(rb + Q8A_DIMS);
          w32[0] = 0u;
          w32[1] = *reinterpret_cast<const uint32_t*>(&sr);
          w32[2] = *reinterpret_cast<const uint32_t*>(&mt);
        } else {
          *reinterpret_cast<float4*>(rb + Q8B_DIMS) = make_float4(sc, rr, m2, t2);
          *reinterpret_cast<float4*>(rb + Q8B_DIMS + 16) = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
}

void launch_tail_norms(Index& ix) {
  // FPP_L2_FETCH=32|64|128: cudaLimitMaxL2FetchGranularity hint (experiments)
  if (getenv("FPP_L2_FETCH")) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(getenv("FPP_L2_FETCH")));
  // FPP_SC_DMAX: widest rows that get screening records (default 256; experiments)
  static const uint32_t sc_dmax = getenv("FPP_SC_DMAX") ? (uint32_t)atoi(getenv("FPP_SC_DMAX")) : 256u;
  if (ix.d >= 64 && ix.d <= sc_dmax && ix.d % 4 == 0) {  // k_score_screen's records
    ix.q8rec = static_cast<uint4*>(dmalloc((size_t)ix.n * (32 + 128)));
    k_q8_records<<<sm_count() * 8, 256, 0, ix.stream>>>(ix.X, ix.n, ix.d, ix.ldx, ix.q8rec);
    FPP_LAUNCH();
  }
  // head width: 32 floats for rows of <= 192 floats (C4's d = 128: the score gather is
  // HBM-bound there and a far candidate then costs 128 B instead of 256 B: 157k -> 200k
  // q/s), else 64 (C2's d = 300 is latency-bound: a narrower head only adds a tail job
  // per survivor, 10.2 vs 7.7 ms)
  ix.xt_head = ix.d <= 192 ? 32u : 64u;
  if (getenv("FPP_XT_HEAD")) {  // experiments: a multiple of 4 in [32, 64]
    const int h = atoi(getenv("FPP_XT_HEAD"));
    if (h >= 32 && h <= 64 && h % 4 == 0) ix.xt_head = (uint32_t)h;
  }
  const uint32_t nsl = xt_nslices(ix.d, ix.xt_head);
  // one checkpoint (after the head) by default: the later in-tail checks prune few rows
  // (read fraction 0.3202 vs 0.3219 on C2) and cost more than they save (C2 score 7.81
  // vs 7.50 ms, C4 414 vs 409 ms); FPP_XT_N=2..4 restores them
  const uint32_t want = getenv("FPP_XT_N") ? (uint32_t)std::max(1, atoi(getenv("FPP_XT_N"))) : 1u;
  ix.xt_n = ix.d >= XT_SLICE ? std::min<uint32_t>({nsl - 1, XT_MAX, want}) : 0;
  if (!ix.xt_n) return;
  ix.xtail = static_cast<float*>(dmalloc((size_t)ix.xt_n * ix.n * sizeof(float)));
  k_tail_norms<<<sm_count() * 8, 256, 0, ix.stream>>>(ix.X, ix.n, ix.d, ix.ldx, ix.xt_n, ix.xt_head, ix.xtail);
  FPP_LAUNCH();
}

__global__ void k_check_finite(const float* __restrict__ X, uint64_t cnt, unsigned long long* bad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (!isfinite(X[i])) atomicMin(bad, (unsigned long long)i);
}

static void set_device(int dev) {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(FPP_ERR_CUDA, "no CUDA device available (the GPU path has no CPU fallback)");
  }
  if (dev >= count) fail(FPP_ERR_INVALID_ARGUMENT, "device ordinal out of range");
  if (dev >= 0) FPP_CUDA(cudaSetDevice(dev));
}

static void validate_params(const fpp_params& p, uint64_t n, uint32_t d) {
  if (p.mode > FPP_MODE_FALCONN_BASELINE) fail(FPP_ERR_INVALID_ARGUMENT, "config: unknown mode");
  if (p.centering > 1) fail(FPP_ERR_INVALID_ARGUMENT, "config: centering must be 0 or 1");
  if (n == 0) fail(FPP_ERR_EMPTY_DATASET, "dataset: need at least one point");
  if (d == 0) fail(FPP_ERR_INVALID_ARGUMENT, "dataset: dim must be >= 1");
  if (p.L == 0) fail(FPP_ERR_INVALID_ARGUMENT, "build: L must be >= 1");
  if (p.K != 1 && p.K != 2) fail(FPP_ERR_INVALID_ARGUMENT, "build: K (concatenation l) must be 1 or 2");
  if (p.D == 0 || (p.D & (p.D - 1)))
    fail(FPP_ERR_INVALID_ARGUMENT, "SpinnerStack: D must be a power of two, got " + std::to_string(p.D));
  if (!(p.alpha > 0.0f && p.alpha <= 1.0f)) fail(FPP_ERR_INVALID_ARGUMENT, "build: alpha must be in (0,1]");
  if (p.iprobes == 0) fail(FPP_ERR_INVALID_ARGUMENT, "build: iProbes must be >= 1");
  uint32_t P = 1;
  while (P < d) P <<= 1;
  if (p.D > P && p.D % P) fail(FPP_ERR_INVALID_ARGUMENT, "SpinnerStack: D must be a multiple of padded dim");
  const uint64_t NB = p.K == 2 ? 4ull * p.D * p.D : 2ull * p.D;
  if (p.iprobes > NB) fail(FPP_ERR_OUT_OF_RANGE, "index_probe_sequence: iProbes > number of buckets");
  if (p.D > P) fail(FPP_ERR_UNSUPPORTED, "GPU path: D > d_pad (multi-block stacks) not supported");
  if (p.L > 1024) fail(FPP_ERR_UNSUPPORTED, "GPU path: L must be <= 1024");
  if ((uint64_t)p.L * NB >= (1ull << 32))
    fail(FPP_ERR_UNSUPPORTED, "GPU path: L*NB must be < 2^32 (32-bit global bucket ids)");
  if (P > 1024) fail(FPP_ERR_UNSUPPORTED, "GPU path: d_pad > 1024 not supported");
  if (p.iprobes > std::min<uint32_t>(p.D, 16))
    fail(FPP_ERR_UNSUPPORTED, "GPU path: iProbes must be <= min(D,16)");
  if (n >= (1ull << 32) || n * p.iprobes >= (1ull << 32))
    fail(FPP_ERR_UNSUPPORTED, "GPU path: n*iProbes must be < 2^32 per shard");
}

// Validated index shell: X resident on the device, sign bitmasks uploaded, no
// tables yet (build_tables, shard_begin or load_tables fill them).
Index* prepare_index(const float* X, bool on_device, uint64_t n, uint32_t d, const fpp_params* pp) {
  if (!pp) fail(FPP_ERR_INVALID_ARGUMENT, "build: params is NULL");
  if (!X && n) fail(FPP_ERR_INVALID_ARGUMENT, "build: X is NULL");
  fpp_params p = *pp;
  if (p.mode == FPP_MODE_FALCONN_BASELINE) {  // baseline forces alpha=1, iProbes=1
    p.alpha = 1.0f;
    p.iprobes = 1;
  }
  validate_params(p, n, d);
  set_device(p.device);
  if (!on_device) {  // dataset.cpp:15-18 finite check
    int64_t bad = -1;
#pragma omp parallel for schedule(static) reduction(max : bad)
    for (int64_t i = 0; i < (int64_t)(n * d); ++i)
      if (!std::isfinite(X[i]) && bad < 0) bad = i;
    if (bad >= 0)
      fail(FPP_ERR_NON_FINITE, "dataset: non-finite coordinate in row " + std::to_string(bad / d));
  }
  auto* ix = new Index();
  try {
    ix->prm = p;
    ix->n = n;
    ix->d = d;
    uint32_t P = 1;
    while (P < d) P <<= 1;
    ix->P = P;
    ix->W = P < 32 ? 1 : P / 32;
    ix->NB = p.K == 2 ? 4ull * p.D * p.D : 2ull * p.D;
    FPP_CUDA(cudaGetDevice(&ix->device));
    FPP_CUDA(cudaStreamCreateWithFlags(&ix->stream, cudaStreamNonBlocking));
    FPP_CUDA(cudaMallocHost(&ix->h_pinned, 64));
    // rows padded to a 128 B multiple (d >= 32): the score gather's row slices then
    // start on line boundaries (+5% DRAM efficiency on C2's 1200 B rows)
    ix->ldx = d < 32 ? d : (d + 31) / 32 * 32;
    ix->X = static_cast<float*>(dmalloc((size_t)n * ix->ldx * sizeof(float)));
    if (ix->ldx != d) FPP_CUDA(cudaMemsetAsync(ix->X, 0, (size_t)n * ix->ldx * 4, ix->stream));
    FPP_CUDA(cudaMemcpy2DAsync(ix->X, (size_t)ix->ldx * 4, X, (size_t)d * 4, (size_t)d * 4, n,
                               on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                               ix->stream));
    if (on_device) {
      DBuf<unsigned long long> bad(1);
      const unsigned long long init = ~0ull;
      FPP_CUDA(cudaMemcpyAsync(bad.p, &init, 8, cudaMemcpyHostToDevice, ix->stream));
      k_check_finite<<<sm_count() * 4, 256, 0, ix->stream>>>(ix->X, n * ix->ldx, bad.p);
      FPP_LAUNCH();
      unsigned long long b = 0;
      FPP_CUDA(cudaMemcpyAsync(&b, bad.p, 8, cudaMemcpyDeviceToHost, ix->stream));
      FPP_CUDA(cudaStreamSynchronize(ix->stream));
      if (b != ~0ull)
        fail(FPP_ERR_NON_FINITE, "dataset: non-finite coordinate in row " + std::to_string(b / ix->ldx));
    }
    std::vector<uint32_t> words;
    pack_signs(p, P, words);
    ix->signs = static_cast<uint32_t*>(dmalloc(words.size() * 4));
    FPP_CUDA(cudaMemcpyAsync(ix->signs, words.data(), words.size() * 4, cudaMemcpyHostToDevice,
                             ix->stream));
    ix->sign_words = words.size();
    if (p.centering) {  // index the centered rows
      DBuf<float> cd(d);
      k_center_mean<<<(d + 127) / 128, 128, 0, ix->stream>>>(ix->X, n, d, ix->ldx, cd.p);
      FPP_LAUNCH();
      k_center_sub<<<sm_count() * 4, 256, 0, ix->stream>>>(ix->X, n, d, ix->ldx, cd.p);
      FPP_LAUNCH();
      ix->center.resize(d);
      FPP_CUDA(cudaMemcpyAsync(ix->center.data(), cd.p, d * 4, cudaMemcpyDeviceToHost, ix->stream));
      FPP_CUDA(cudaStreamSynchronize(ix->stream));
    }
    // SimHash signatures of every point (rerank screening; n x 8 B)
    ix->sigs = static_cast<uint64_t*>(dmalloc(n * sizeof(uint64_t) + 8));
    launch_signatures(*ix, ix->X, n, ix->ldx, ix->sigs, ix->stream);
    launch_tail_norms(*ix);
    FPP_CUDA(cudaStreamSynchronize(ix->stream));
  } catch (...) {
    delete ix;
    throw;
  }
  return ix;
}

static fpp_index* build_common(const float* X, bool on_device, uint64_t n, uint32_t d,
                               const fpp_params* pp, bool sharded = false) {
  if (sharded && pp && pp->centering)
    fail(FPP_ERR_UNSUPPORTED, "sharded build: centering needs the global mean (center X first)");
  Index* ix = prepare_index(X, on_device, n, d, pp);
  try {
    if (sharded) shard_begin(*ix);
    else build_tables(*ix);
    ix->device_bytes = n * ix->ldx * 4 + ix->sign_words * 4 + (uint64_t)ix->prm.L * (ix->NB + 1) * 4 +
                       (ix->prm.L + 1) * 8 + ix->kept_total * 8;
    double ms[PH_COUNT] = {0};
    ix->timer.collect(ms);
    ix->acc.hash_ms += ms[PH_HASH];
    ix->acc.sort_ms += ms[PH_SORT];
  } catch (...) {
    delete ix;
    throw;
  }
  return reinterpret_cast<fpp_index*>(ix);
}

static const Index& IX(const fpp_index* p) {
  if (!p) fail(FPP_ERR_INVALID_ARGUMENT, "index is NULL");
  return *reinterpret_cast<const Index*>(p);
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    FPP_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

static void validate_query(const Index& ix, uint64_t nq, uint32_t k, uint32_t qprobes,
                           const void* Q, const void* ids, const void* scores) {
  if (!ix.offsets) fail(FPP_ERR_INVALID_ARGUMENT, "search: sharded build not finished (fpp_shard_finish)");
  if (k == 0) fail(FPP_ERR_INVALID_ARGUMENT, "search: k must be >= 1");
  if (k > ix.n) fail(FPP_ERR_OUT_OF_RANGE, "search: k > n");
  if (qprobes < ix.prm.L || (uint64_t)qprobes > (uint64_t)ix.prm.L * ix.NB)
    fail(FPP_ERR_OUT_OF_RANGE, "query_probe_sequence: qProbes must be in [L, L*NB]");
  if (nq && (!Q || !ids || !scores)) fail(FPP_ERR_INVALID_ARGUMENT, "search: NULL buffer");
}

static void collect_timings(const Index& ix) {
  double ms[PH_COUNT] = {0};
  ix.timer.collect(ms);
  ix.acc.hash_ms += ms[PH_HASH];
  ix.acc.sort_ms += ms[PH_SORT];
  collect_query_timings(ix);  // waits for every query context's phases
  if (ix.score_bytes_d.p) {  // the phases above have completed: the counter is final
    unsigned long long b = 0;  // monotone counter: no reset racing later launches
    FPP_CUDA(cudaMemcpy(&b, ix.score_bytes_d.p, 8, cudaMemcpyDeviceToHost));
    ix.acc.score_bytes += b - ix.score_bytes_seen;
    ix.score_bytes_seen = b;
  }
}
}  // namespace fpp

using namespace fpp;

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return FPP_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory";
    return FPP_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FPP_ERR_CUDA;
  }
}

namespace fpp {
int guarded_call(const std::function<void()>& f) { return guarded(f); }
}  // namespace fpp

extern "C" {

int fpp_abi_version(void) { return FPP_ABI_VERSION; }
const char* fpp_last_error(void) { return g_err.c_str(); }

void fpp_default_params(fpp_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->L = 50;
  p->K = 2;
  p->D = 128;
  p->iprobes = 3;
  p->kappa = 20;
  p->alpha = 0.1f;
  p->seed = 1;
  p->device = -1;
}

int fpp_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

int fpp_build(const float* X, uint64_t n, uint32_t d, const fpp_params* p, fpp_index** out) {
  return guarded([&] {
    if (!out) fail(FPP_ERR_INVALID_ARGUMENT, "build: out is NULL");
    *out = build_common(X, false, n, d, p);
  });
}

int fpp_build_device(const float* X, uint64_t n, uint32_t d, const fpp_params* p, fpp_index** out) {
  return guarded([&] {
    if (!out) fail(FPP_ERR_INVALID_ARGUMENT, "build: out is NULL");
    *out = build_common(X, true, n, d, p);
  });
}

void fpp_free(fpp_index* idx) { delete reinterpret_cast<Index*>(idx); }

static void query_host(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t k,
                       uint32_t qprobes, uint32_t rerank, uint32_t* ids, double* scores,
                       fpp_query_stats* stats) {
  const Index& ix = IX(idx);
  validate_query(ix, nq, k, qprobes, Q, ids, scores);
  if (rerank && rerank < k) fail(FPP_ERR_OUT_OF_RANGE, "search: rerank budget B must be 0 or >= k");
  if (!nq) return;
  DeviceGuard dg(ix.device);
  CtxLease cx(ix);  // this call's scratch: concurrent calls run side by side
  cudaStream_t s = cx->own;
  cx->q_in.ensure(nq * ix.d);
  cx->q_ids.ensure(nq * k);
  cx->q_scores.ensure(nq * k);
  if (stats) cx->q_stats.ensure(nq);
  FPP_CUDA(cudaMemcpyAsync(cx->q_in.p, Q, nq * ix.d * 4, cudaMemcpyHostToDevice, s));
  run_query(ix, *cx, cx->q_in.p, nq, k, qprobes, cx->q_ids.p, cx->q_scores.p,
            stats ? cx->q_stats.p : nullptr, s, rerank);
  FPP_CUDA(cudaMemcpyAsync(ids, cx->q_ids.p, nq * k * 4, cudaMemcpyDeviceToHost, s));
  FPP_CUDA(cudaMemcpyAsync(scores, cx->q_scores.p, nq * k * 8, cudaMemcpyDeviceToHost, s));
  if (stats)
    FPP_CUDA(cudaMemcpyAsync(stats, cx->q_stats.p, nq * sizeof(fpp_query_stats),
                             cudaMemcpyDeviceToHost, s));
  FPP_CUDA(cudaStreamSynchronize(s));
}

static void query_dev(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t k,
                      uint32_t qprobes, uint32_t rerank, uint32_t* ids, double* scores,
                      fpp_query_stats* stats, void* stream) {
  const Index& ix = IX(idx);
  validate_query(ix, nq, k, qprobes, Q, ids, scores);
  if (rerank && rerank < k) fail(FPP_ERR_OUT_OF_RANGE, "search: rerank budget B must be 0 or >= k");
  if (!nq) return;
  DeviceGuard dg(ix.device);
  CtxLease cx(ix);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cx->own;
  run_query(ix, *cx, Q, nq, k, qprobes, ids, scores, stats, s, rerank);
}

int fpp_query(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t k, uint32_t qprobes,
              uint32_t* ids, double* scores, fpp_query_stats* stats) {
  return guarded([&] { query_host(idx, Q, nq, k, qprobes, 0, ids, scores, stats); });
}

int fpp_query_device(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t k, uint32_t qprobes,
                     uint32_t* ids, double* scores, fpp_query_stats* stats, void* stream) {
  return guarded([&] { query_dev(idx, Q, nq, k, qprobes, 0, ids, scores, stats, stream); });
}

int fpp_query_probe_sets_device(const fpp_index* idx, const float* Q, uint64_t nq,
                                uint32_t qprobes, uint32_t* probes, void* stream) {
  return guarded([&] {
    const Index& ix = IX(idx);
    if (nq && (!Q || !probes)) fail(FPP_ERR_INVALID_ARGUMENT, "query_probe_sets: NULL buffer");
    validate_query(ix, nq, 1, qprobes, Q, probes, probes);
    if (!nq) return;
    DeviceGuard dg(ix.device);
    CtxLease cx(ix);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cx->own;
    run_query_probes(ix, *cx, Q, nq, qprobes, probes, s);
  });
}

int fpp_query_from_probe_sets_device(const fpp_index* idx, const float* Q, uint64_t nq,
                                     const uint32_t* probes, uint32_t k, uint32_t qprobes,
                                     uint32_t* ids, double* scores, fpp_query_stats* stats,
                                     void* stream) {
  return guarded([&] {
    const Index& ix = IX(idx);
    validate_query(ix, nq, k, qprobes, Q, ids, scores);
    if (nq && !probes) fail(FPP_ERR_INVALID_ARGUMENT, "query_from_probe_sets: NULL probes");
    if (!nq) return;
    DeviceGuard dg(ix.device);
    CtxLease cx(ix);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cx->own;
    run_query_from_probes(ix, *cx, Q, nq, probes, k, qprobes, ids, scores, stats, s);
  });
}

int fpp_query_rerank(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t k,
                     uint32_t qprobes, uint32_t rerank, uint32_t* ids, double* scores,
                     fpp_query_stats* stats) {
  return guarded([&] { query_host(idx, Q, nq, k, qprobes, rerank, ids, scores, stats); });
}

int fpp_query_rerank_device(const fpp_index* idx, const float* Q_dev, uint64_t nq, uint32_t k,
                            uint32_t qprobes, uint32_t rerank, uint32_t* ids_dev,
                            double* scores_dev, fpp_query_stats* stats_dev, void* stream) {
  return guarded([&] {
    query_dev(idx, Q_dev, nq, k, qprobes, rerank, ids_dev, scores_dev, stats_dev, stream);
  });
}

int fpp_signatures(const fpp_index* idx, const float* X, uint64_t n, uint64_t* out) {
  return guarded([&] {
    const Index& ix = IX(idx);
    if (n && (!X || !out)) fail(FPP_ERR_INVALID_ARGUMENT, "signatures: NULL buffer");
    if (!n) return;
    DeviceGuard dg(ix.device);
    std::lock_guard<std::mutex> lk(ix.aux_mu);
    DBuf<float> xd(n * ix.d);
    DBuf<uint64_t> od(n);
    FPP_CUDA(cudaMemcpyAsync(xd.p, X, n * ix.d * 4, cudaMemcpyHostToDevice, ix.stream));
    launch_signatures(ix, xd.p, n, ix.d, od.p, ix.stream);
    FPP_CUDA(cudaMemcpyAsync(out, od.p, n * 8, cudaMemcpyDeviceToHost, ix.stream));
    FPP_CUDA(cudaStreamSynchronize(ix.stream));
  });
}

int fpp_shard_begin(const float* X, uint64_t n, uint32_t d, const fpp_params* p, fpp_index** out) {
  return guarded([&] {
    if (!out) fail(FPP_ERR_INVALID_ARGUMENT, "build: out is NULL");
    *out = build_common(X, false, n, d, p, true);
  });
}

int fpp_shard_begin_device(const float* X, uint64_t n, uint32_t d, const fpp_params* p,
                           fpp_index** out) {
  return guarded([&] {
    if (!out) fail(FPP_ERR_INVALID_ARGUMENT, "build: out is NULL");
    *out = build_common(X, true, n, d, p, true);
  });
}

uint64_t fpp_shard_hist_len(const fpp_index* idx) {
  if (!idx) return 0;
  const Index& ix = *reinterpret_cast<const Index*>(idx);
  return (uint64_t)ix.prm.L * ix.NB;
}

int fpp_shard_hist(const fpp_index* idx, uint32_t* hist_dev) {
  return guarded([&] {
    const Index& ix = IX(idx);
    if (!ix.shard) fail(FPP_ERR_INVALID_ARGUMENT, "shard: not a sharded build in progress");
    DeviceGuard dg(ix.device);
    // on the index stream, then synchronised: the caller may use hist_dev on any stream
    FPP_CUDA(cudaMemcpyAsync(hist_dev, shard_hist_ptr(ix), (uint64_t)ix.prm.L * ix.NB * 4,
                             cudaMemcpyDeviceToDevice, ix.stream));
    FPP_CUDA(cudaStreamSynchronize(ix.stream));
  });
}

int fpp_shard_slots(fpp_index* idx, const uint32_t* global_hist_dev, uint64_t* slots) {
  return guarded([&] {
    Index& ix = *reinterpret_cast<Index*>(const_cast<fpp_index*>(idx));
    DeviceGuard dg(ix.device);
    *slots = shard_slots(ix, global_hist_dev);
  });
}

int fpp_shard_prefix(fpp_index* idx, const uint32_t* global_hist_dev, uint64_t* prefix_dev) {
  return guarded([&] {
    Index& ix = *reinterpret_cast<Index*>(idx);
    DeviceGuard dg(ix.device);
    shard_prefix(ix, global_hist_dev, prefix_dev);
  });
}

int fpp_shard_finish(fpp_index* idx, const uint32_t* global_hist_dev, const uint64_t* all_prefix_dev,
                     uint32_t world) {
  return guarded([&] {
    Index& ix = *reinterpret_cast<Index*>(idx);
    DeviceGuard dg(ix.device);
    shard_finish(ix, global_hist_dev, all_prefix_dev, world);
    ix.device_bytes = ix.n * ix.ldx * 4 + (uint64_t)ix.prm.L * (ix.NB + 1) * 4 + ix.kept_total * 8;
    double ms[PH_COUNT] = {0};
    ix.timer.collect(ms);
    ix.acc.hash_ms += ms[PH_HASH];
    ix.acc.sort_ms += ms[PH_SORT];
  });
}

int fpp_index_info_get(const fpp_index* idx, fpp_index_info* info) {
  return guarded([&] {
    const Index& ix = IX(idx);
    if (!info) fail(FPP_ERR_INVALID_ARGUMENT, "info is NULL");
    info->n = ix.n;
    info->d = ix.d;
    info->d_pad = ix.P;
    info->L = ix.prm.L;
    info->K = ix.prm.K;
    info->D = ix.prm.D;
    info->iprobes = ix.prm.iprobes;
    info->kappa = ix.prm.kappa;
    info->alpha = ix.prm.alpha;
    info->seed = ix.prm.seed;
    info->num_buckets = ix.NB;
    info->kept_total = ix.kept_total;
    info->prefilter_total = ix.n * ix.prm.L * ix.prm.iprobes;
    info->device_bytes = ix.device_bytes;
    info->max_bucket = ix.max_bucket;
    info->id_offset = ix.prm.id_offset;
    info->centering = ix.prm.centering;
    info->mode = ix.prm.mode;
    info->device = ix.device;
  });
}

uint64_t fpp_table_size(const fpp_index* idx, uint32_t t) {
  if (!idx) return 0;
  const Index& ix = *reinterpret_cast<const Index*>(idx);
  if (t >= ix.prm.L) return 0;
  return ix.table_base_h[t + 1] - ix.table_base_h[t];
}

int fpp_table_csr(const fpp_index* idx, uint32_t t, uint32_t* offsets, uint32_t* ids, float* scores) {
  return guarded([&] {
    const Index& ix = IX(idx);
    if (t >= ix.prm.L) fail(FPP_ERR_OUT_OF_RANGE, "table index out of range");
    DeviceGuard dg(ix.device);
    const uint64_t b0 = ix.table_base_h[t], cnt = ix.table_base_h[t + 1] - b0;
    if (offsets)
      FPP_CUDA(cudaMemcpy(offsets, ix.offsets + (uint64_t)t * (ix.NB + 1), (ix.NB + 1) * 4,
                          cudaMemcpyDeviceToHost));
    if (ids && cnt) FPP_CUDA(cudaMemcpy(ids, ix.ids + b0, cnt * 4, cudaMemcpyDeviceToHost));
    if (scores && cnt) FPP_CUDA(cudaMemcpy(scores, ix.scores + b0, cnt * 4, cudaMemcpyDeviceToHost));
  });
}

int fpp_project(const fpp_index* idx, const float* X, uint64_t n, uint32_t t, uint32_t f, float* out) {
  return guarded([&] {
    const Index& ix = IX(idx);
    if (t >= ix.prm.L || f >= ix.prm.K) fail(FPP_ERR_OUT_OF_RANGE, "project: (t,f) out of range");
    if (!n) return;
    DeviceGuard dg(ix.device);
    std::lock_guard<std::mutex> lk(ix.aux_mu);
    DBuf<float> xd(n * ix.d), od(n * ix.prm.D);
    FPP_CUDA(cudaMemcpyAsync(xd.p, X, n * ix.d * 4, cudaMemcpyHostToDevice, ix.stream));
    launch_project(ix, xd.p, n, t, f, od.p, ix.stream);
    FPP_CUDA(cudaStreamSynchronize(ix.stream));
    FPP_CUDA(cudaMemcpy(out, od.p, n * ix.prm.D * 4, cudaMemcpyDeviceToHost));
  });
}

int fpp_index_probes(const fpp_index* idx, const float* X, uint64_t n, uint32_t t, uint32_t* buckets,
                     float* scores) {
  return guarded([&] {
    const Index& ix = IX(idx);
    if (t >= ix.prm.L) fail(FPP_ERR_OUT_OF_RANGE, "index_probes: table out of range");
    if (!n) return;
    DeviceGuard dg(ix.device);
    std::lock_guard<std::mutex> lk(ix.aux_mu);
    const uint32_t ip = ix.prm.iprobes;
    DBuf<float> xd(n * ix.d);
    DBuf<uint2> od(n * ip);
    FPP_CUDA(cudaMemcpyAsync(xd.p, X, n * ix.d * 4, cudaMemcpyHostToDevice, ix.stream));
    launch_index_probes(ix, xd.p, n, t, od.p, ix.stream);
    FPP_CUDA(cudaStreamSynchronize(ix.stream));
    std::vector<uint2> h(n * ip);
    FPP_CUDA(cudaMemcpy(h.data(), od.p, n * ip * 8, cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < n * ip; ++i) {
      buckets[i] = h[i].x;
      std::memcpy(scores + i, &h[i].y, 4);
    }
  });
}

uint32_t fpp_query_cap(const fpp_index* idx, uint32_t qprobes) {
  return idx ? query_cap(*reinterpret_cast<const Index*>(idx), qprobes) : 0;
}
uint64_t fpp_query_probes(const fpp_index* idx, uint32_t qprobes) {
  return idx ? query_probes(*reinterpret_cast<const Index*>(idx), qprobes) : 0;
}

int fpp_query_lists(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t qprobes, float* vals,
                    uint32_t* codes) {
  return guarded([&] {
    const Index& ix = IX(idx);
    if (!nq) return;
    DeviceGuard dg(ix.device);
    std::lock_guard<std::mutex> lk(ix.aux_mu);
    const uint32_t s = query_cap(ix, qprobes);
    const uint64_t tot = nq * ix.prm.L * ix.prm.K * s;
    DBuf<float> qd(nq * ix.d), vd(tot);
    DBuf<uint32_t> cd(tot);
    FPP_CUDA(cudaMemcpyAsync(qd.p, Q, nq * ix.d * 4, cudaMemcpyHostToDevice, ix.stream));
    launch_query_lists(ix, qd.p, nq, s, vd.p, cd.p, ix.stream);
    FPP_CUDA(cudaStreamSynchronize(ix.stream));
    FPP_CUDA(cudaMemcpy(vals, vd.p, tot * 4, cudaMemcpyDeviceToHost));
    FPP_CUDA(cudaMemcpy(codes, cd.p, tot * 4, cudaMemcpyDeviceToHost));
  });
}

int fpp_query_debug(const fpp_index* idx, const float* q, uint32_t qprobes, uint64_t* probes,
                    uint64_t* n_probes, uint32_t* cands, uint64_t* n_cands) {
  return guarded([&] {
    const Index& ix = IX(idx);
    validate_query(ix, 1, 1, qprobes, q, probes, cands);
    DeviceGuard dg(ix.device);
    CtxLease cx(ix);
    DBuf<float> qd(ix.d);
    FPP_CUDA(cudaMemcpyAsync(qd.p, q, ix.d * 4, cudaMemcpyHostToDevice, cx->own));
    std::vector<uint64_t> pv;
    std::vector<uint32_t> cv;
    query_debug(ix, *cx, qd.p, qprobes, pv, cv);
    std::memcpy(probes, pv.data(), pv.size() * 8);
    std::memcpy(cands, cv.data(), cv.size() * 4);
    *n_probes = pv.size();
    *n_cands = cv.size();
  });
}

int fpp_timings_get(const fpp_index* idx, fpp_timings* t) {
  return guarded([&] {
    const Index& ix = IX(idx);
    collect_timings(ix);
    if (t) *t = ix.acc;
  });
}

int fpp_timings_reset(const fpp_index* idx) {
  return guarded([&] {
    const Index& ix = IX(idx);
    collect_timings(ix);
    ix.acc = fpp_timings{};
  });
}

// dataset.cpp:24-38, parallel over rows (per-row arithmetic is the reference's)
static void validate_brute(const Index& ix, uint64_t nq, uint32_t k, const void* Q,
                           const void* ids, const void* scores) {
  if (k == 0) fail(FPP_ERR_INVALID_ARGUMENT, "brute_force_topk: k must be >= 1");
  if (k > ix.n) fail(FPP_ERR_OUT_OF_RANGE, "brute_force_topk: k > n");
  if (nq && (!Q || !ids || !scores)) fail(FPP_ERR_INVALID_ARGUMENT, "brute_force_topk: NULL buffer");
}

int fpp_brute_force(const fpp_index* idx, const float* Q, uint64_t nq, uint32_t k, uint32_t* ids,
                    double* scores) {
  return guarded([&] {
    const Index& ix = IX(idx);
    validate_brute(ix, nq, k, Q, ids, scores);
    if (!nq) return;
    DeviceGuard dg(ix.device);
    std::lock_guard<std::mutex> lk(ix.aux_mu);
    cudaStream_t s = ix.stream;
    DBuf<float> qd(nq * ix.d);
    DBuf<uint32_t> id(nq * k);
    DBuf<double> sc(nq * k);
    FPP_CUDA(cudaMemcpyAsync(qd.p, Q, nq * ix.d * 4, cudaMemcpyHostToDevice, s));
    run_brute_force(ix, qd.p, nq, k, id.p, sc.p, s);
    FPP_CUDA(cudaMemcpyAsync(ids, id.p, nq * k * 4, cudaMemcpyDeviceToHost, s));
    FPP_CUDA(cudaMemcpyAsync(scores, sc.p, nq * k * 8, cudaMemcpyDeviceToHost, s));
    FPP_CUDA(cudaStreamSynchronize(s));
  });
}

int fpp_brute_force_device(const fpp_index* idx, const float* Q_dev, uint64_t nq, uint32_t k,
                           uint32_t* ids_dev, double* scores_dev, void* stream) {
  return guarded([&] {
    const Index& ix = IX(idx);
    validate_brute(ix, nq, k, Q_dev, ids_dev, scores_dev);
    if (!nq) return;
    DeviceGuard dg(ix.device);
    std::lock_guard<std::mutex> lk(ix.aux_mu);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ix.stream;
    run_brute_force(ix, Q_dev, nq, k, ids_dev, scores_dev, s);
  });
}

int fpp_save(const fpp_index* idx, const char* path) {
  return guarded([&] {
    const Index& ix = IX(idx);
    DeviceGuard dg(ix.device);
    std::lock_guard<std::mutex> lk(ix.aux_mu);
    save_index(ix, path, nullptr);
  });
}

int fpp_load(const char* path, const float* X, uint64_t n, uint32_t d, int device,
             fpp_index** out) {
  return guarded([&] {
    if (!out) fail(FPP_ERR_INVALID_ARGUMENT, "load: out is NULL");
    *out = reinterpret_cast<fpp_index*>(load_index(path, X, false, n, d, device));
  });
}

int fpp_load_device(const char* path, const float* X_dev, uint64_t n, uint32_t d, int device,
                    fpp_index** out) {
  return guarded([&] {
    if (!out) fail(FPP_ERR_INVALID_ARGUMENT, "load: out is NULL");
    *out = reinterpret_cast<fpp_index*>(load_index(path, X_dev, true, n, d, device));
  });
}

uint64_t fpp_content_hash(const float* X, uint64_t n, uint32_t d) {
  return X ? content_hash(X, n, d) : 0;
}

int fpp_center(float* X, uint64_t n, uint32_t d, float* center_out) {
  return guarded([&] {
    if (!X || !n || !d) fail(FPP_ERR_EMPTY_DATASET, "dataset: need at least one point");
    std::vector<float> c(d);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < (int64_t)d; ++j) {  // dataset.cpp:45-48: rows in order, per coordinate
      double m = 0.0;
      for (uint64_t i = 0; i < n; ++i) m += X[i * d + j];
      c[j] = float(m / double(n));
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i)
      for (uint32_t j = 0; j < d; ++j) X[(uint64_t)i * d + j] -= c[j];
    if (center_out) std::memcpy(center_out, c.data(), d * 4);
  });
}

int fpp_index_center(const fpp_index* idx, float* center_out) {
  return guarded([&] {
    const Index& ix = IX(idx);
    if (!center_out) fail(FPP_ERR_INVALID_ARGUMENT, "index_center: NULL buffer");
    for (uint32_t j = 0; j < ix.d; ++j) center_out[j] = ix.center.empty() ? 0.0f : ix.center[j];
  });
}

int fpp_normalize(float* X, uint64_t n, uint32_t d) {
  return guarded([&] {
    if (!X || !n || !d) fail(FPP_ERR_EMPTY_DATASET, "dataset: need at least one point");
    int64_t bad = -1;
#pragma omp parallel for schedule(static) reduction(max : bad)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
      float* row = X + (uint64_t)i * d;
      double sq = 0.0;
      for (uint32_t j = 0; j < d; ++j) sq += double(row[j]) * double(row[j]);
      if (sq == 0.0) {
        if (bad < 0) bad = i;
        continue;
      }
      const float inv = float(1.0 / std::sqrt(sq));
      for (uint32_t j = 0; j < d; ++j) row[j] *= inv;
    }
    if (bad >= 0) fail(FPP_ERR_ZERO_NORM, "normalize: zero-norm row " + std::to_string(bad));
  });
}

// pinned synthetic generator
static inline double synth_u(uint64_t seed, uint64_t stream, uint64_t k) {
  return ((double)(host_mix64(host_derive_seed(seed, stream, k, 0)) >> 11) + 0.5) * 0x1.0p-53;
}
static inline double synth_normal(uint64_t seed, uint64_t stream, uint64_t k) {
  const double u1 = synth_u(seed, stream, 2 * k), u2 = synth_u(seed, stream, 2 * k + 1);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}

int fpp_synth(float* X, uint64_t n, uint32_t d, uint32_t clusters, float sigma, uint64_t seed,
              uint32_t stream, int threads) {
  return fpp_synth_rows(X, 0, n, d, clusters, sigma, seed, stream, threads);
}

int fpp_synth_rows(float* X, uint64_t row0, uint64_t n, uint32_t d, uint32_t clusters, float sigma,
                   uint64_t seed, uint32_t stream, int threads) {
  return guarded([&] {
    if (!X || !n || !d) fail(FPP_ERR_EMPTY_DATASET, "synth: empty");
    if (threads <= 0) threads = omp_get_max_threads();
    const uint64_t s_noise = 3 + 100ull * stream, s_assign = 2 + 100ull * stream;
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t r = 0; r < (int64_t)n; ++r) {
      const uint64_t i = row0 + (uint64_t)r;
      float* row = X + (uint64_t)r * d;
      if (clusters == 0) {
        for (uint32_t j = 0; j < d; ++j) row[j] = (float)synth_normal(seed, s_noise, i * d + j);
      } else {
        const uint64_t c = host_mix64(host_derive_seed(seed, s_assign, i, 0)) % clusters;
        for (uint32_t j = 0; j < d; ++j) {
          const double ctr = synth_normal(seed, 1, c * d + j);
          const double z = synth_normal(seed, s_noise, i * d + j);
          row[j] = (float)(ctr + (double)sigma * z);
        }
      }
    }
  });
}

int fpp_merge_topk(const double* scores_dev, const uint32_t* ids_dev, uint32_t lists, uint64_t nq,
                   uint32_t k, double* out_scores_dev, uint32_t* out_ids_dev, int device,
                   void* stream) {
  return guarded([&] {
    if (lists == 0 || lists > 32) fail(FPP_ERR_INVALID_ARGUMENT, "merge_topk: lists must be in [1, 32]");
    if (k == 0) fail(FPP_ERR_INVALID_ARGUMENT, "merge_topk: k must be >= 1");
    if (nq && (!scores_dev || !ids_dev || !out_scores_dev || !out_ids_dev))
      fail(FPP_ERR_INVALID_ARGUMENT, "merge_topk: NULL buffer");
    if (!nq) return;
    set_device(device);
    launch_merge_topk(scores_dev, ids_dev, lists, nq, k, out_scores_dev, out_ids_dev,
                      static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
