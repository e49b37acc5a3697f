// fpp_multi.cu -- single-process multi-GPU index behind the C ABI (fpp_multi_*):
// build(X, config) over num_gpus devices and search over the sharded index
// (SURVEY.md 8(b) num_gpus, 8(e)).
//
// Shard g owns the contiguous global ids [g*n/G, (g+1)*n/G) on devices[g] and is an
// ordinary fpp_index built by the global-filter protocol (fpp_shard_*), so the union
// of the shards is the 1-GPU index exactly and answers do not depend on G
// (SPEC.md:605).  One host thread per shard drives its device; the exchange steps are
// pull copies between the shards' device buffers (cudaMemcpyPeerAsync: NVLink P2P when
// peer access can be enabled, which build does for every device pair) followed by a
// local kernel:
//   build   histogram all-reduce   = gather [G][L*NB] + k_sum_u32
//           prefix all-gather      = gather [G][slots] -> fpp_shard_finish
//   query   stage A split          : shard g hashes + probe-selects its query slice,
//           probe-set all-gather   = gather [G][per][P_eff] u32
//           stage B                : every shard resolves + scores the whole chunk
//           top-k merge, scattered : shard g gathers the G lists of ITS slice
//                                    [G][per][k] and merges them (k_merge_topk), then
//                                    copies its slice of the answer to the host
// A device may appear several times in `devices` (shards then share it): that is how
// the layer is tested on a one-GPU box.  The one-process-per-GPU form of the same
// protocol (torch.distributed / NCCL collectives) is paper_2206_01382_b200/dist.py.
#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>
#include <thread>

#include "fpp_internal.h"

namespace fpp {

int guarded_call(const std::function<void()>& f);  // fpp_capi.cu: exception -> code + message

namespace {

struct DevGuard {
  int prev = 0;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    FPP_CUDA(cudaSetDevice(dev));
  }
  ~DevGuard() { cudaSetDevice(prev); }
};

// C-ABI call on a worker thread: failure -> Error with the callee's message
void ok(int rc) {
  if (rc != FPP_OK) throw Error(rc, fpp_last_error());
}

// run fn(g) for every shard, one host thread each (the library calls synchronise
// internally); the first failure is rethrown on the caller
void par(uint32_t G, const std::function<void(uint32_t)>& fn) {
  if (G == 1) {
    fn(0);
    return;
  }
  std::vector<int> code(G, FPP_OK);
  std::vector<std::string> msg(G);
  std::vector<std::thread> th;
  th.reserve(G);
  for (uint32_t g = 0; g < G; ++g)
    th.emplace_back([&, g] {
      try {
        fn(g);
      } catch (const Error& e) {
        code[g] = e.code;
        msg[g] = e.what();
      } catch (const std::bad_alloc&) {
        code[g] = FPP_ERR_OUT_OF_MEMORY;
        msg[g] = "host out of memory";
      } catch (const std::exception& e) {
        code[g] = FPP_ERR_CUDA;
        msg[g] = e.what();
      }
    });
  for (auto& t : th) t.join();
  for (uint32_t g = 0; g < G; ++g)
    if (code[g] != FPP_OK) throw Error(code[g], "shard " + std::to_string(g) + ": " + msg[g]);
}

__global__ void k_sum_u32(const uint32_t* __restrict__ in, uint32_t lists, uint64_t len,
                          uint32_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) {
    uint32_t s = 0;
    for (uint32_t l = 0; l < lists; ++l) s += in[(uint64_t)l * len + i];
    out[i] = s;
  }
}

// dst (on ddev) <- src (on sdev), ordered on ddev's stream s
void pull(void* dst, int ddev, const void* src, int sdev, size_t bytes, cudaStream_t s) {
  if (!bytes) return;
  if (ddev == sdev) FPP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
  else FPP_CUDA(cudaMemcpyPeerAsync(dst, ddev, src, sdev, bytes, s));
}

struct Shard {
  fpp_index* ix = nullptr;
  int device = 0;
  uint64_t lo = 0, hi = 0;  // global id range
  cudaStream_t s = nullptr;
  // query scratch of this shard's device (guarded by Multi::qmu)
  DBuf<float> Q;             // [nqc][d]
  DBuf<uint32_t> probes;     // [G*per][P_eff]
  DBuf<uint32_t> ids;        // [G*per][k] this shard's lists of the whole chunk
  DBuf<double> sc;
  DBuf<fpp_query_stats> st;  // [nqc]
  DBuf<uint32_t> l_ids;      // [G][per][k] every shard's lists of this shard's slice
  DBuf<double> l_sc;
  DBuf<uint32_t> m_ids;      // [per][k] merged
  DBuf<double> m_sc;
};

}  // namespace

struct Multi {
  uint32_t G = 0;
  uint64_t n = 0;
  uint32_t d = 0;
  fpp_params prm{};
  std::unique_ptr<Shard[]> sh;
  mutable std::mutex qmu;  // one fpp_multi_query at a time (the shards' scratch is per index)
  ~Multi() {
    for (uint32_t g = 0; sh && g < G; ++g) {
      Shard& x = sh[g];
      cudaSetDevice(x.device);
      x.Q.release(); x.probes.release(); x.ids.release(); x.sc.release(); x.st.release();
      x.l_ids.release(); x.l_sc.release(); x.m_ids.release(); x.m_sc.release();
      if (x.s) cudaStreamDestroy(x.s);
      if (x.ix) fpp_free(x.ix);
    }
  }
};

namespace {

void enable_peers(const std::vector<int>& devs) {
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      int can = 0;
      FPP_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can) continue;  // cudaMemcpyPeerAsync then stages through the host
      DevGuard dg(a);
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else FPP_CUDA(e);
    }
}

Multi* multi_build(const float* X, uint64_t n, uint32_t d, const fpp_params* pp, uint32_t G,
                   const int32_t* devices) {
  if (!pp) fail(FPP_ERR_INVALID_ARGUMENT, "build: params is NULL");
  if (G == 0 || G > 32) fail(FPP_ERR_INVALID_ARGUMENT, "build: num_gpus must be in [1, 32]");
  if (!X || n == 0) fail(FPP_ERR_EMPTY_DATASET, "build: empty dataset");
  if (n < G) fail(FPP_ERR_INVALID_ARGUMENT, "build: fewer points than shards");
  if (pp->id_offset) fail(FPP_ERR_INVALID_ARGUMENT, "multi build: id_offset must be 0");
  int ndev = fpp_device_count();
  if (ndev < 1) {  // the single-index build reports the config error, else "no CPU fallback"
    fpp_index* none = nullptr;
    ok(fpp_build(X, n, d, pp, &none));
    fpp_free(none);
    fail(FPP_ERR_CUDA, "no CUDA device (there is no CPU fallback)");
  }
  std::unique_ptr<Multi> m(new Multi);
  m->G = G; m->n = n; m->d = d; m->prm = *pp;
  m->sh.reset(new Shard[G]);
  std::vector<int> uniq;
  for (uint32_t g = 0; g < G; ++g) {
    int dev = devices ? devices[g] : (int)g;
    if (dev < 0 || dev >= ndev)
      fail(FPP_ERR_INVALID_ARGUMENT, "build: device ordinal " + std::to_string(dev) + " of shard " +
                                         std::to_string(g) + " does not exist");
    m->sh[g].device = dev;
    if (std::find(uniq.begin(), uniq.end(), dev) == uniq.end()) uniq.push_back(dev);
    const uint64_t base = n / G, rem = n % G;  // dist.py::shard_range
    m->sh[g].lo = g * base + std::min<uint64_t>(g, rem);
    m->sh[g].hi = m->sh[g].lo + base + (g < rem ? 1 : 0);
  }
  enable_peers(uniq);
  for (uint32_t g = 0; g < G; ++g) {
    Shard& x = m->sh[g];
    DevGuard dg(x.device);
    FPP_CUDA(cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking));
  }
  if (G == 1) {  // the plain 1-GPU build
    fpp_params p = *pp;
    p.device = m->sh[0].device;
    ok(fpp_build(X, n, d, &p, &m->sh[0].ix));
    return m.release();
  }
  // 1. every shard hashes its rows and histograms (table, bucket)
  par(G, [&](uint32_t g) {
    Shard& x = m->sh[g];
    fpp_params p = *pp;
    p.device = x.device;
    p.id_offset = (uint32_t)x.lo;
    ok(fpp_shard_begin(X + x.lo * d, x.hi - x.lo, d, &p, &x.ix));
  });
  const uint64_t hl = fpp_shard_hist_len(m->sh[0].ix);
  std::vector<DBuf<uint32_t>> hist(G), ghist(G), hall(G);
  std::vector<uint64_t> slots(G, 0);
  std::vector<DBuf<uint64_t>> pre(G), pall(G);
  par(G, [&](uint32_t g) {
    Shard& x = m->sh[g];
    DevGuard dg(x.device);
    hist[g].alloc(hl);
    ok(fpp_shard_hist(x.ix, hist[g].p));  // synchronised on return
  });
  // 2. all-reduce(sum): gather the G histograms, add them locally
  par(G, [&](uint32_t g) {
    Shard& x = m->sh[g];
    DevGuard dg(x.device);
    hall[g].alloc((uint64_t)G * hl);
    ghist[g].alloc(hl);
    for (uint32_t h = 0; h < G; ++h)
      pull(hall[g].p + (uint64_t)h * hl, x.device, hist[h].p, m->sh[h].device, hl * 4, x.s);
    k_sum_u32<<<(unsigned)std::min<uint64_t>((hl + 255) / 256, (uint64_t)sm_count() * 8), 256, 0,
                x.s>>>(hall[g].p, G, hl, ghist[g].p);
    FPP_LAUNCH();
    FPP_CUDA(cudaStreamSynchronize(x.s));
    hall[g].release();
    // 3. this shard's sorted bucket prefixes in the globally agreed slots
    ok(fpp_shard_slots(x.ix, ghist[g].p, &slots[g]));
    pre[g].alloc(std::max<uint64_t>(slots[g], 1));
    ok(fpp_shard_prefix(x.ix, ghist[g].p, pre[g].p));
    FPP_CUDA(cudaDeviceSynchronize());
  });
  for (uint32_t g = 1; g < G; ++g)
    if (slots[g] != slots[0]) fail(FPP_ERR_CUDA, "multi build: shards disagree on the slot count");
  // 4. all-gather the prefixes, cut every bucket at its global keep-th key
  par(G, [&](uint32_t g) {
    Shard& x = m->sh[g];
    DevGuard dg(x.device);
    const uint64_t sl = slots[0];
    pall[g].alloc(std::max<uint64_t>((uint64_t)G * sl, 1));
    for (uint32_t h = 0; h < G; ++h)
      pull(pall[g].p + (uint64_t)h * sl, x.device, pre[h].p, m->sh[h].device, sl * 8, x.s);
    FPP_CUDA(cudaStreamSynchronize(x.s));
  });
  par(G, [&](uint32_t g) {  // (after every gather: finish may free what peers still read)
    Shard& x = m->sh[g];
    DevGuard dg(x.device);
    ok(fpp_shard_finish(x.ix, ghist[g].p, pall[g].p, G));
    FPP_CUDA(cudaDeviceSynchronize());
    pall[g].release(); pre[g].release(); ghist[g].release(); hist[g].release();
  });
  return m.release();
}

void multi_query(const Multi& m, const float* Q, uint64_t nq, uint32_t k, uint32_t qprobes,
                 uint32_t* ids, double* scores, fpp_query_stats* stats) {
  const uint32_t G = m.G;
  if (G == 1) {
    ok(fpp_query(m.sh[0].ix, Q, nq, k, qprobes, ids, scores, stats));
    return;
  }
  if (k == 0) fail(FPP_ERR_INVALID_ARGUMENT, "search: k must be >= 1");
  if (k > m.n) fail(FPP_ERR_OUT_OF_RANGE, "search: k > n");
  if (nq && (!Q || !ids || !scores)) fail(FPP_ERR_INVALID_ARGUMENT, "search: NULL buffer");
  const uint64_t pe = fpp_query_probes(m.sh[0].ix, qprobes);
  if (qprobes < m.prm.L || pe == 0)
    fail(FPP_ERR_OUT_OF_RANGE, "query_probe_sequence: qProbes must be in [L, L*NB]");
  if (!nq) return;
  std::lock_guard<std::mutex> lk(m.qmu);
  Shard* sh = m.sh.get();
  // chunk the batch so a chunk's probe sets stay within ~2 GiB per device
  uint64_t qch = std::max<uint64_t>((2ull << 30) / (pe * 4), 64ull * G);
  if (const char* e = getenv("FPP_MULTI_CHUNK")) qch = std::max<uint64_t>(1, strtoull(e, nullptr, 10));
  std::vector<fpp_query_stats> hst;
  for (uint64_t q0 = 0; q0 < nq; q0 += qch) {
    const uint64_t nqc = std::min(qch, nq - q0);
    const uint64_t per = (nqc + G - 1) / G;  // dist.py::query_slice
    auto slice = [&](uint32_t g, uint64_t& lo, uint64_t& hi) {
      lo = std::min(nqc, g * per);
      hi = std::min(nqc, (g + 1) * per);
    };
    // stage A on the shard's slice (probe sets depend only on the query and the hash
    // functions, which every shard shares)
    par(G, [&](uint32_t g) {
      Shard& x = sh[g];
      DevGuard dg(x.device);
      x.Q.ensure(nqc * m.d);
      x.probes.ensure(G * per * pe);
      x.ids.ensure(G * per * k);
      x.sc.ensure(G * per * k);
      if (stats) x.st.ensure(nqc);
      x.l_ids.ensure(G * per * k);
      x.l_sc.ensure(G * per * k);
      x.m_ids.ensure(per * k);
      x.m_sc.ensure(per * k);
      FPP_CUDA(cudaMemcpyAsync(x.Q.p, Q + q0 * m.d, nqc * m.d * 4, cudaMemcpyHostToDevice, x.s));
      uint64_t lo, hi;
      slice(g, lo, hi);
      if (hi > lo)
        ok(fpp_query_probe_sets_device(x.ix, x.Q.p + lo * m.d, hi - lo, qprobes,
                                       x.probes.p + lo * pe, x.s));
      FPP_CUDA(cudaStreamSynchronize(x.s));
    });
    // all-gather the probe sets; stage B over the whole chunk in this shard's tables
    par(G, [&](uint32_t g) {
      Shard& x = sh[g];
      DevGuard dg(x.device);
      for (uint32_t h = 0; h < G; ++h) {
        if (h == g) continue;
        uint64_t lo, hi;
        slice(h, lo, hi);
        pull(x.probes.p + lo * pe, x.device, sh[h].probes.p + lo * pe, sh[h].device,
             (hi - lo) * pe * 4, x.s);
      }
      ok(fpp_query_from_probe_sets_device(x.ix, x.Q.p, nqc, x.probes.p, k, qprobes, x.ids.p,
                                          x.sc.p, stats ? x.st.p : nullptr, x.s));
      FPP_CUDA(cudaStreamSynchronize(x.s));
    });
    // the G lists of this shard's query slice -> k-way merge -> host
    if (stats) hst.resize((uint64_t)G * nqc);
    par(G, [&](uint32_t g) {
      Shard& x = sh[g];
      DevGuard dg(x.device);
      uint64_t lo, hi;
      slice(g, lo, hi);
      const uint64_t c = hi - lo;
      if (c) {
        for (uint32_t h = 0; h < G; ++h) {
          pull(x.l_ids.p + (uint64_t)h * c * k, x.device, sh[h].ids.p + lo * k, sh[h].device,
               c * k * 4, x.s);
          pull(x.l_sc.p + (uint64_t)h * c * k, x.device, sh[h].sc.p + lo * k, sh[h].device,
               c * k * 8, x.s);
        }
        launch_merge_topk(x.l_sc.p, x.l_ids.p, G, c, k, x.m_sc.p, x.m_ids.p, x.s);
        FPP_CUDA(cudaMemcpyAsync(ids + (q0 + lo) * k, x.m_ids.p, c * k * 4, cudaMemcpyDeviceToHost,
                                 x.s));
        FPP_CUDA(cudaMemcpyAsync(scores + (q0 + lo) * k, x.m_sc.p, c * k * 8,
                                 cudaMemcpyDeviceToHost, x.s));
      }
      if (stats)
        FPP_CUDA(cudaMemcpyAsync(hst.data() + (uint64_t)g * nqc, x.st.p,
                                 nqc * sizeof(fpp_query_stats), cudaMemcpyDeviceToHost, x.s));
      FPP_CUDA(cudaStreamSynchronize(x.s));
    });
    if (stats)  // probes are the same on every shard; the shards' candidates are disjoint
      for (uint64_t q = 0; q < nqc; ++q) {
        fpp_query_stats t = hst[q];
        for (uint32_t g = 1; g < G; ++g) {
          const fpp_query_stats& o = hst[(uint64_t)g * nqc + q];
          t.entries += o.entries;
          t.candidates += o.candidates;
          t.exact += o.exact;
        }
        stats[q0 + q] = t;
      }
  }
}

}  // namespace
}  // namespace fpp

using namespace fpp;

extern "C" {

int fpp_multi_build(const float* X, uint64_t n, uint32_t d, const fpp_params* p, uint32_t num_gpus,
                    const int32_t* devices, fpp_multi** out) {
  return guarded_call([&] {
    if (!out) fail(FPP_ERR_INVALID_ARGUMENT, "build: out is NULL");
    *out = reinterpret_cast<fpp_multi*>(multi_build(X, n, d, p, num_gpus, devices));
  });
}

int fpp_multi_query(const fpp_multi* mi, const float* Q, uint64_t nq, uint32_t k, uint32_t qprobes,
                    uint32_t* ids, double* scores, fpp_query_stats* stats) {
  return guarded_call([&] {
    if (!mi) fail(FPP_ERR_INVALID_ARGUMENT, "index is NULL");
    multi_query(*reinterpret_cast<const Multi*>(mi), Q, nq, k, qprobes, ids, scores, stats);
  });
}

uint32_t fpp_multi_shards(const fpp_multi* mi) {
  return mi ? reinterpret_cast<const Multi*>(mi)->G : 0;
}

const fpp_index* fpp_multi_shard(const fpp_multi* mi, uint32_t g) {
  if (!mi) return nullptr;
  const Multi& m = *reinterpret_cast<const Multi*>(mi);
  return g < m.G ? m.sh[g].ix : nullptr;
}

void fpp_multi_free(fpp_multi* mi) { delete reinterpret_cast<Multi*>(mi); }

}  // extern "C"
