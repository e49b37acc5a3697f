// lsfann/falconnpp_gpu.hpp -- header-only C++ host API over the C ABI
// (include/falconnpp.h), mirroring the reference's namespace (common.hpp:12)
// and its SPEC operations: Index::build, Index::query
// (with SimHash rerank :330-338), brute_force (:490-503) and
// save / load (:270-287).  Errors are rethrown as the reference does:
// std::invalid_argument for configuration / range / data errors
// (dataset.cpp:10-18, rotation.cpp:18-20,42-49), std::runtime_error for CUDA.
#pragma once
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "falconnpp.h"

namespace lsfann::gpu {

inline void check(int rc) {
  if (rc == FPP_OK) return;
  const std::string msg = fpp_last_error();
  switch (rc) {
    case FPP_ERR_INVALID_ARGUMENT:
    case FPP_ERR_EMPTY_DATASET:
    case FPP_ERR_DIMENSION:
    case FPP_ERR_OUT_OF_RANGE:
    case FPP_ERR_NON_FINITE:
    case FPP_ERR_ZERO_NORM:
    case FPP_ERR_FORMAT:  // magic / truncation / checksum errors
      throw std::invalid_argument(msg);
    case FPP_ERR_OUT_OF_MEMORY:
      throw std::bad_alloc();
    default:
      throw std::runtime_error(msg);
  }
}

struct QueryResult {
  std::vector<uint32_t> ids;   // [nq][k], 0xFFFFFFFF past min(k, candidates)
  std::vector<double> scores;  // [nq][k], -inf past min(k, candidates)
  std::vector<fpp_query_stats> stats;
};

class Index {
 public:
  // build(X, L, K, D, iProbes, alpha) -- X row-major n x d, already normalized
  static Index build(std::span<const float> X, std::size_t n, std::size_t d, uint32_t L,
                     uint32_t K, uint32_t D, uint32_t iProbes, float alpha, uint32_t kappa = 20,
                     uint64_t seed = 1, int device = -1, uint32_t id_offset = 0,
                     bool centering = false, uint32_t mode = FPP_MODE_FALCONNPP) {
    if (X.size() != n * d) throw std::invalid_argument("build: X.size() != n*d");
    fpp_params p;
    fpp_default_params(&p);
    p.L = L; p.K = K; p.D = D; p.iprobes = iProbes; p.alpha = alpha; p.kappa = kappa;
    p.seed = seed; p.device = device; p.id_offset = id_offset;
    p.centering = centering ? 1u : 0u; p.mode = mode;
    fpp_index* h = nullptr;
    check(fpp_build(X.data(), n, static_cast<uint32_t>(d), &p, &h));
    return Index(h);
  }

  // query(Q, k, qProbes) -- batch over the rows of Q
  QueryResult query(std::span<const float> Q, std::size_t nq, uint32_t k, uint32_t qProbes,
                    bool with_stats = false) const {
    QueryResult r;
    r.ids.resize(nq * k);
    r.scores.resize(nq * k);
    if (with_stats) r.stats.resize(nq);
    check(fpp_query(h_, Q.data(), nq, k, qProbes, r.ids.data(), r.scores.data(),
                    with_stats ? r.stats.data() : nullptr));
    return r;
  }

  // search with a SimHash rerank budget B; 0 = off
  QueryResult query_rerank(std::span<const float> Q, std::size_t nq, uint32_t k,
                           uint32_t qProbes, uint32_t B, bool with_stats = false) const {
    QueryResult r;
    r.ids.resize(nq * k);
    r.scores.resize(nq * k);
    if (with_stats) r.stats.resize(nq);
    check(fpp_query_rerank(h_, Q.data(), nq, k, qProbes, B, r.ids.data(), r.scores.data(),
                           with_stats ? r.stats.data() : nullptr));
    return r;
  }

  // brute_force_topk over the index's dataset: recall ground truth
  QueryResult brute_force(std::span<const float> Q, std::size_t nq, uint32_t k) const {
    QueryResult r;
    r.ids.resize(nq * k);
    r.scores.resize(nq * k);
    check(fpp_brute_force(h_, Q.data(), nq, k, r.ids.data(), r.scores.data()));
    return r;
  }

  // save(index, path) / load(path) -- FLPP; load takes X again
  void save(const std::string& path) const { check(fpp_save(h_, path.c_str())); }
  static Index load(const std::string& path, std::span<const float> X, std::size_t n,
                    std::size_t d, int device = 0) {
    if (X.size() != n * d) throw std::invalid_argument("load: X.size() != n*d");
    fpp_index* h = nullptr;
    check(fpp_load(path.c_str(), X.data(), n, static_cast<uint32_t>(d), device, &h));
    return Index(h);
  }

  fpp_index_info info() const {
    fpp_index_info i;
    check(fpp_index_info_get(h_, &i));
    return i;
  }

  Index(Index&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  Index& operator=(Index&& o) noexcept {
    if (this != &o) { fpp_free(h_); h_ = std::exchange(o.h_, nullptr); }
    return *this;
  }
  Index(const Index&) = delete;
  Index& operator=(const Index&) = delete;
  ~Index() { fpp_free(h_); }
  const fpp_index* handle() const { return h_; }

 private:
  explicit Index(fpp_index* h) : h_(h) {}
  fpp_index* h_ = nullptr;
};

// build(X, L, K, D, iProbes, alpha, ..., num_gpus) / query over num_gpus devices of one
// process (fpp_multi_*): contiguous id shards with the global alpha/kappa filter, so
// the answers equal Index's for every num_gpus.  devices: one CUDA
// ordinal per shard (empty = 0..num_gpus-1; ordinals may repeat).
class MultiIndex {
 public:
  static MultiIndex build(std::span<const float> X, std::size_t n, std::size_t d, uint32_t L,
                          uint32_t K, uint32_t D, uint32_t iProbes, float alpha,
                          uint32_t num_gpus, std::span<const int32_t> devices = {},
                          uint32_t kappa = 20, uint64_t seed = 1,
                          uint32_t mode = FPP_MODE_FALCONNPP) {
    if (X.size() != n * d) throw std::invalid_argument("build: X.size() != n*d");
    if (!devices.empty() && devices.size() != num_gpus)
      throw std::invalid_argument("build: devices.size() != num_gpus");
    fpp_params p;
    fpp_default_params(&p);
    p.L = L; p.K = K; p.D = D; p.iprobes = iProbes; p.alpha = alpha; p.kappa = kappa;
    p.seed = seed; p.mode = mode;
    fpp_multi* h = nullptr;
    check(fpp_multi_build(X.data(), n, static_cast<uint32_t>(d), &p, num_gpus,
                          devices.empty() ? nullptr : devices.data(), &h));
    return MultiIndex(h);
  }

  QueryResult query(std::span<const float> Q, std::size_t nq, uint32_t k, uint32_t qProbes,
                    bool with_stats = false) const {
    QueryResult r;
    r.ids.resize(nq * k);
    r.scores.resize(nq * k);
    if (with_stats) r.stats.resize(nq);
    check(fpp_multi_query(h_, Q.data(), nq, k, qProbes, r.ids.data(), r.scores.data(),
                          with_stats ? r.stats.data() : nullptr));
    return r;
  }

  uint32_t num_shards() const { return fpp_multi_shards(h_); }
  fpp_index_info shard_info(uint32_t g) const {
    fpp_index_info i;
    check(fpp_index_info_get(fpp_multi_shard(h_, g), &i));
    return i;
  }

  MultiIndex(MultiIndex&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  MultiIndex& operator=(MultiIndex&& o) noexcept {
    if (this != &o) { fpp_multi_free(h_); h_ = std::exchange(o.h_, nullptr); }
    return *this;
  }
  MultiIndex(const MultiIndex&) = delete;
  MultiIndex& operator=(const MultiIndex&) = delete;
  ~MultiIndex() { fpp_multi_free(h_); }

 private:
  explicit MultiIndex(fpp_multi* h) : h_(h) {}
  fpp_multi* h_ = nullptr;
};

}  // namespace lsfann::gpu
