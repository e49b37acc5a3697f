// fpp_internal.h -- host-side index object and kernel entry points shared by
// fpp_capi.cu, fpp_build.cu and fpp_query.cu.  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <condition_variable>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/falconnpp.h"

namespace fpp {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define FPP_CUDA(x) ::fpp::cuda_check((x), #x, __FILE__, __LINE__)
#define FPP_LAUNCH() ::fpp::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// device allocation with OOM -> FPP_ERR_OUT_OF_MEMORY
void* dmalloc(size_t bytes);
void dfree(void* p);

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count) p = static_cast<T*>(dmalloc(count * sizeof(T)));
    n = count;
  }
  // grow without preserving contents
  void ensure(size_t count) {
    if (count > n) alloc(count + count / 4);
  }
  void release() {
    if (p) dfree(p);
    p = nullptr;
    n = 0;
  }
};

// Phase timer: CUDA events recorded on the launching stream around each phase.
enum Phase { PH_HASH = 0, PH_SORT, PH_QHASH, PH_PROBE, PH_COLLECT, PH_SCORE, PH_COUNT };
struct PhaseTimer {
  bool enabled = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> open;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get();
  void begin(int ph, cudaStream_t s, cudaEvent_t* out_start);
  void end(int ph, cudaEvent_t start, cudaStream_t s);
  void collect(double* ms_by_phase);  // after stream sync
  ~PhaseTimer();
};

struct ShardState;
struct QueryCtx;

struct Index {
  fpp_params prm{};
  uint64_t n = 0;
  uint32_t d = 0, P = 0;  // P = d_pad = FHT length
  uint32_t ldx = 0;       // row stride of X in floats: d rounded up to 32 (128 B rows)
  uint64_t NB = 0;        // buckets per table
  int device = 0;
  cudaStream_t stream = nullptr;

  float* X = nullptr;         // [n][d] device, owned
  uint32_t* signs = nullptr;  // [L][K][3][W] device
  uint32_t W = 1;
  uint32_t* offsets = nullptr;  // [L][NB+1] kept offsets, relative to table base
  uint64_t* table_base = nullptr;  // [L+1] device
  std::vector<uint64_t> table_base_h;
  uint32_t* ids = nullptr;   // [kept_total] local ids
  float* scores = nullptr;   // [kept_total]
  uint64_t kept_total = 0;
  uint32_t max_bucket = 0;
  uint64_t sign_words = 0;
  uint64_t* sigs = nullptr;  // [n] SimHash signatures (rerank screening)
  // Row tail norms for exact early termination in the score gather: xtail[j][i] =
  // ||X[i][(j+1)*XT_SLICE:d)||, rounded up to fp32, checkpoints j < xt_n
  float* xtail = nullptr;
  uint32_t xt_n = 0;
  // narrow rows (64 <= d <= 256, d % 4 == 0; k_score_screen): a 32 B and a 128 B
  // screening record per row -- int8 codes with a per-row scale, plus the error /
  // norm terms of the bound (k_q8_records)
  uint4* q8rec = nullptr;
  // the stage-1 records again, in CSR entry order ([kept_total][4] uint4: entry e's
  // record is q8rec[ids[e]]), so the walking screen streams them with its bucket walk
  // instead of one random 128 B DRAM line per 64 B record; built by the first query
  // that walks (ensure_q8csr)
  mutable uint4* q8csr = nullptr;
  uint32_t xt_head = 64;  // head (screening) slice width, see launch_tail_norms
  std::vector<float> center;  // [d] when prm.centering (dataset.cpp center())
  uint64_t device_bytes = 0;
  ShardState* shard = nullptr;  // global-filter sharded build in progress

  // Query scratch lives in per-call contexts (QueryCtx, fpp_query.cu): a call
  // leases a free context for its enqueue, so concurrent queries on one index
  // neither share scratch nor serialise; a context's next user
  // stream-waits on its previous call's completion event before touching it.
  mutable std::mutex mu;                     // guards the context pool and the policy below
  mutable std::mutex aux_mu;                 // serialises the aux entry points on `stream`
  mutable std::vector<QueryCtx*> ctx_all, ctx_free;
  mutable std::condition_variable ctx_cv;
  // score-gather early termination (k_score_pruned): measured fraction of row slices
  // read, probed on the first chunks and every PRUNE_REPROBE-th chunk after
  mutable double prune_frac = -1.0;
  mutable uint64_t prune_chunks = 0;
  mutable DBuf<unsigned long long> score_bytes_d;  // [1] row bytes read by the score kernels
  mutable unsigned long long score_bytes_seen = 0;
  uint64_t* h_pinned = nullptr;  // small pinned readback

  mutable PhaseTimer timer;
  mutable fpp_timings acc{};

  ~Index();
};

// Scratch of one query call (run_query).  Two slots double-buffer query chunks
// across two streams; the reorder and host-staging buffers,
// the per-call phase timer and counters live here too.
struct QueryCtx {
  struct QSlot {
    DBuf<float> vals;
    DBuf<uint32_t> codes;
    DBuf<uint64_t> ppos;
    DBuf<uint32_t> plen;
    DBuf<uint32_t> gbuf;
    DBuf<uint32_t> ckey;
    DBuf<uint32_t> cpair;
    DBuf<uint64_t> dbgclk;
    DBuf<uint32_t> eq;
    DBuf<uint64_t> coff;
    DBuf<uint32_t> uq;
    DBuf<uint32_t> uniq;    // unique candidates per query (grouped lists carry holes)
    DBuf<uint32_t> cands;
    DBuf<uint32_t> bitmap;
    DBuf<uint32_t> counter;
    DBuf<uint64_t> qsig;    // rerank: query signatures
    DBuf<uint32_t> cands2;  // rerank: screened candidates [nqc][B]
    DBuf<uint32_t> uq2;
    DBuf<uint32_t> wlog;    // walking screen: per-CTA log of admitted ids
    DBuf<double> allsc;     // k > 32: every candidate's exact score (k_topk_more)
    uint64_t* pinned = nullptr;     // etot readback
    cudaEvent_t ev_probe = nullptr; // stage A (hash + probe select) done
    cudaEvent_t ev_bdone = nullptr; // stage B (collect + score) done
    void release();
  };
  int device = 0;
  QSlot slot[2];
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr;
  cudaEvent_t ev_done = nullptr;   // recorded on the caller's stream at the end of a call
  bool done_recorded = false;
  cudaStream_t sA = nullptr, sB = nullptr;  // pipeline streams (low / high priority)
  cudaStream_t own = nullptr;               // host-buffer calls run here
  DBuf<float> q_in;
  DBuf<uint32_t> q_ids;
  DBuf<double> q_scores;
  DBuf<fpp_query_stats> q_stats;
  // batch reordering scratch (run_query)
  DBuf<uint32_t> ord_key, ord_perm, ord_ids;
  DBuf<float> ord_q;
  DBuf<double> ord_sc;
  DBuf<fpp_query_stats> ord_st;
  // k_score_pruned read-fraction probe (async readback into the index policy)
  unsigned long long* prune_h = nullptr;  // pinned [4]: rows, row floats read, stage-2, exact rows
  DBuf<unsigned long long> prune_d;
  cudaEvent_t prune_ev = nullptr;
  bool prune_pending = false;
  PhaseTimer timer;
  fpp_timings acc{};
  ~QueryCtx();
};

// lease a free query context of `ix` for one call (created on demand)
struct CtxLease {
  const Index& ix;
  QueryCtx* c;
  explicit CtxLease(const Index& ix);
  ~CtxLease();
  QueryCtx* operator->() const { return c; }
  QueryCtx& operator*() const { return *c; }
};
// wait for every context, fold their timers/counters into ix.acc (fpp_timings_get)
void collect_query_timings(const Index& ix);

// host helpers (fpp_capi.cu)
uint64_t host_mix64(uint64_t z);
uint64_t host_derive_seed(uint64_t m, uint64_t a, uint64_t b, uint64_t c);
void pack_signs(const fpp_params& p, uint32_t P, std::vector<uint32_t>& words);
uint32_t query_cap(const Index& ix, uint32_t qprobes);
uint64_t query_probes(const Index& ix, uint32_t qprobes);
int sm_count();
int smem_optin_max();  // cudaDevAttrMaxSharedMemoryPerBlockOptin of the current device
// Let `kern` be launched with any dynamic shared-memory size the device allows.  The
// limit is a per-function, per-device attribute shared by every host thread: setting it to
// each launch's own size raced between threads driving indexes of different sizes on one
// device (thread A: set 324 B, thread B: set 320 B, thread A: launch with 324 B ->
// "invalid argument"), so every caller sets the same, largest value.
template <class Kern>
inline void allow_dynamic_smem(Kern kern) {
  cudaFuncAttributes fa;
  FPP_CUDA(cudaFuncGetAttributes(&fa, kern));
  FPP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem_optin_max() - (int)fa.sharedSizeBytes));
}

// build (fpp_build.cu)
void build_tables(Index& ix);
Index* prepare_index(const float* X, bool on_device, uint64_t n, uint32_t d, const fpp_params* pp);
uint64_t content_hash(const float* X, uint64_t n, uint32_t d);
void save_index(const Index& ix, const char* path, const float* X_host);
void launch_signatures(const Index& ix, const float* Xd, uint64_t n, uint32_t ld, uint64_t* out,
                       cudaStream_t s);
// k_score_screen records (k_q8_records), two per row:
//   stage A, 32 B: int8 codes of dims [0, Q8A_DIMS) (20 B), a 4 B id slot (the inline
//     CSR-order copy stores the entry's id there), {scale, ||x_h - x~_h||, ||x~_h||,
//     ||x[Q8A_DIMS:d)||} as half2 pairs (8 B: the scale fp16-exact, the norms rounded
//     up);
//   stage B, 128 B (a random access costs a 128 B DRAM line anyway): codes of dims
//     [Q8A_DIMS, Q8A_DIMS + Q8B_DIMS) (96 B) + the same four terms in fp32 (16 B) +
//     16 B padding.
// Tables: [n][32 B] (A), then [n][128 B] (B).
constexpr uint32_t Q8A_DIMS = 20;
constexpr uint32_t Q8B_DIMS = 96;
constexpr uint32_t Q8_STAGES = 2;
constexpr uint32_t XT_SLICE = 64;  // = the score ring's row-slice width for d >= 64
constexpr uint32_t XT_MAX = 4;     // tail-norm checkpoints per row
// score-gather slices of a d-wide row: a head [0, h) (h = Index::xt_head, 32 or 64),
// then XT_SLICE-wide slices; checkpoint j (after slice j) is column h + j * XT_SLICE
__host__ __device__ inline uint32_t xt_nslices(uint32_t d, uint32_t h) {
  return d <= h ? 1u : 1u + (d - h + XT_SLICE - 1) / XT_SLICE;
}
void launch_tail_norms(Index& ix);
void launch_order_keys(const Index& ix, const float* Qd, uint64_t n, uint64_t* out, cudaStream_t s);
void run_brute_force(const Index& ix, const float* Qd, uint64_t nq, uint32_t k, uint32_t* ids_d,
                     double* scores_d, cudaStream_t s);
Index* load_index(const char* path, const float* X, bool on_device, uint64_t n, uint32_t d,
                  int device);
void launch_project(const Index& ix, const float* Xd, uint64_t n, uint32_t t, uint32_t f,
                    float* out, cudaStream_t s);
void launch_index_probes(const Index& ix, const float* Xd, uint64_t n, uint32_t t,
                         uint2* out, cudaStream_t s);

// global-filter sharded build (fpp_build.cu)
void shard_begin(Index& ix);
uint64_t shard_slots(Index& ix, const uint32_t* global_hist);
void shard_prefix(Index& ix, const uint32_t* global_hist, uint64_t* prefix);
void shard_finish(Index& ix, const uint32_t* global_hist, const uint64_t* all_prefix,
                  uint32_t world);
void shard_release(Index& ix);
const uint32_t* shard_hist_ptr(const Index& ix);

// query (fpp_query.cu)
void run_query(const Index& ix, QueryCtx& cx, const float* Qd, uint64_t nq, uint32_t k,
               uint32_t qprobes, uint32_t* ids_d, double* scores_d, fpp_query_stats* stats_d,
               cudaStream_t s, uint32_t rerank = 0);
void launch_query_lists(const Index& ix, const float* Qd, uint64_t nq, uint32_t s_cap,
                        float* vals, uint32_t* codes, cudaStream_t s, uint64_t lstride = 0);
// probes (t*NB+b) and candidates of query 0 of Qd (debug/parity)
void run_query_probes(const Index& ix, QueryCtx& cx, const float* Qd, uint64_t nq, uint32_t qprobes,
                  uint32_t* probes_d, cudaStream_t s);
void run_query_from_probes(const Index& ix, QueryCtx& cx, const float* Qd, uint64_t nq,
                       const uint32_t* probes_d, uint32_t k, uint32_t qprobes, uint32_t* ids_d,
                       double* scores_d, fpp_query_stats* stats_d, cudaStream_t s);
void query_debug(const Index& ix, QueryCtx& cx, const float* qd, uint32_t qprobes,
                 std::vector<uint64_t>& probes, std::vector<uint32_t>& cands);
// k-way merge of `lists` per-shard top-k lists [lists][nq][k] (each sorted by score
// desc, id asc; empty slots id 0xFFFFFFFF / -inf) into [nq][k] (fpp_merge_topk)
void launch_merge_topk(const double* sc, const uint32_t* ids, uint32_t lists, uint64_t nq,
                       uint32_t k, double* out_sc, uint32_t* out_ids, cudaStream_t s);

}  // namespace fpp
