// fpp_persist.cu -- FLPP index persistence (SPEC.md:270-278 save/load, External
// Interfaces :283-287, determinism :283).
//
// Little-endian file, version 1:
//   header  "FLPP" | u32 version | IndexConfig: u32 L, u32 K, u32 D, f32 alpha,
//           u32 iProbes, u32 kappa, u32 centering, u32 mode, u32 id_offset |
//           u64 seed | u64 n | u32 d | f32 center[d] (centering only) |
//           dataset reference: u32 path_len, path bytes, u64 content hash
//           (fnv1a64 of the indexed n*d fp32 rows -- after centering --
//           common.hpp:50-57)
//   body    per table t: u32 non-empty buckets, then per bucket (ascending id):
//           u32 bucket, u32 count, count x (u32 point_id, f32 score) in the
//           bucket's (score desc, id asc) order
//   footer  u64 fnv1a64 of the body bytes
// The dataset is stored by reference: load() takes X again and checks its hash.
// A save of the same (dataset, config) is byte-identical (the CSR is
// deterministic), and load(save(ix)) answers every query bit-identically.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "fpp_internal.h"

namespace fpp {

static constexpr uint64_t FNV_BASIS = 0xcbf29ce484222325ull, FNV_PRIME = 0x100000001b3ull;
static uint64_t fnv1a64(const void* data, size_t len, uint64_t h = FNV_BASIS) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= FNV_PRIME;
  }
  return h;
}

uint64_t content_hash(const float* X, uint64_t n, uint32_t d) {
  return fnv1a64(X, (size_t)n * d * sizeof(float));
}

namespace {

struct Writer {
  FILE* f;
  uint64_t body_hash = FNV_BASIS;
  bool in_body = false;
  void put(const void* p, size_t len) {
    if (len && fwrite(p, 1, len, f) != len) fail(FPP_ERR_IO, "save: write failed");
    if (in_body) body_hash = fnv1a64(p, len, body_hash);
  }
  template <class T>
  void put(T v) { put(&v, sizeof(T)); }
};

struct Reader {
  FILE* f;
  uint64_t body_hash = FNV_BASIS;
  bool in_body = false;
  void get(void* p, size_t len, const char* field) {
    if (len && fread(p, 1, len, f) != len)
      fail(FPP_ERR_FORMAT, std::string("load: truncated file (reading ") + field + ")");
    if (in_body) body_hash = fnv1a64(p, len, body_hash);
  }
  template <class T>
  T get(const char* field) {
    T v;
    get(&v, sizeof(T), field);
    return v;
  }
};

struct FileCloser {
  void operator()(FILE* f) const { if (f) fclose(f); }
};

}  // namespace

void save_index(const Index& ix, const char* path, const float* X_host) {
  if (!path) fail(FPP_ERR_INVALID_ARGUMENT, "save: path is NULL");
  if (ix.shard) fail(FPP_ERR_INVALID_ARGUMENT, "save: sharded build not finished");
  const uint32_t L = ix.prm.L;
  const uint64_t NB = ix.NB;
  // content hash of the indexed rows (after centering, if any): from the caller's
  // host copy, else from the device copy
  uint64_t chash;
  if (X_host) {
    chash = content_hash(X_host, ix.n, ix.d);
  } else {
    std::vector<float> xh((size_t)ix.n * ix.d);
    FPP_CUDA(cudaMemcpy2DAsync(xh.data(), (size_t)ix.d * 4, ix.X, (size_t)ix.ldx * 4,
                               (size_t)ix.d * 4, ix.n, cudaMemcpyDeviceToHost, ix.stream));
    FPP_CUDA(cudaStreamSynchronize(ix.stream));
    chash = content_hash(xh.data(), ix.n, ix.d);
  }
  std::unique_ptr<FILE, FileCloser> fh(fopen(path, "wb"));
  if (!fh) fail(FPP_ERR_IO, std::string("save: cannot open ") + path);
  Writer w{fh.get()};
  w.put("FLPP", 4);
  w.put<uint32_t>(FPP_FLPP_VERSION);
  w.put<uint32_t>(ix.prm.L);
  w.put<uint32_t>(ix.prm.K);
  w.put<uint32_t>(ix.prm.D);
  w.put<float>(ix.prm.alpha);
  w.put<uint32_t>(ix.prm.iprobes);
  w.put<uint32_t>(ix.prm.kappa);
  w.put<uint32_t>(ix.prm.centering);
  w.put<uint32_t>(ix.prm.mode);
  w.put<uint32_t>(ix.prm.id_offset);
  w.put<uint64_t>(ix.prm.seed);
  w.put<uint64_t>(ix.n);
  w.put<uint32_t>(ix.d);
  if (ix.prm.centering) w.put(ix.center.data(), (size_t)ix.d * 4);
  w.put<uint32_t>(0);  // dataset path: not recorded (the caller passes X to load)
  w.put<uint64_t>(chash);
  w.in_body = true;
  std::vector<uint32_t> offs(NB + 1), ids;
  std::vector<float> sc;
  std::vector<uint32_t> rec;
  for (uint32_t t = 0; t < L; ++t) {
    FPP_CUDA(cudaMemcpyAsync(offs.data(), ix.offsets + (uint64_t)t * (NB + 1), (NB + 1) * 4,
                             cudaMemcpyDeviceToHost, ix.stream));
    const uint64_t b0 = ix.table_base_h[t], cnt = ix.table_base_h[t + 1] - b0;
    ids.resize(cnt);
    sc.resize(cnt);
    if (cnt) {
      FPP_CUDA(cudaMemcpyAsync(ids.data(), ix.ids + b0, cnt * 4, cudaMemcpyDeviceToHost, ix.stream));
      FPP_CUDA(cudaMemcpyAsync(sc.data(), ix.scores + b0, cnt * 4, cudaMemcpyDeviceToHost, ix.stream));
    }
    FPP_CUDA(cudaStreamSynchronize(ix.stream));
    uint32_t nonempty = 0;
    for (uint64_t b = 0; b < NB; ++b) nonempty += offs[b + 1] != offs[b];
    w.put<uint32_t>(nonempty);
    rec.clear();
    for (uint64_t b = 0; b < NB; ++b) {
      const uint32_t o0 = offs[b], o1 = offs[b + 1];
      if (o0 == o1) continue;
      rec.push_back((uint32_t)b);
      rec.push_back(o1 - o0);
      for (uint32_t j = o0; j < o1; ++j) {
        rec.push_back(ids[j]);
        uint32_t bits;
        std::memcpy(&bits, &sc[j], 4);
        rec.push_back(bits);
      }
    }
    w.put(rec.data(), rec.size() * 4);
  }
  w.in_body = false;
  w.put<uint64_t>(w.body_hash);
  if (fflush(fh.get()) != 0) fail(FPP_ERR_IO, "save: flush failed");
}

Index* load_index(const char* path, const float* X, bool on_device, uint64_t n, uint32_t d,
                  int device) {
  if (!path) fail(FPP_ERR_INVALID_ARGUMENT, "load: path is NULL");
  std::unique_ptr<FILE, FileCloser> fh(fopen(path, "rb"));
  if (!fh) fail(FPP_ERR_IO, std::string("load: cannot open ") + path);
  Reader r{fh.get()};
  char magic[4];
  r.get(magic, 4, "magic");
  if (std::memcmp(magic, "FLPP", 4) != 0) fail(FPP_ERR_FORMAT, "load: bad magic (expected \"FLPP\")");
  const uint32_t version = r.get<uint32_t>("version");
  if (version != FPP_FLPP_VERSION)
    fail(FPP_ERR_UNSUPPORTED, "load: unsupported FLPP version " + std::to_string(version));
  fpp_params p{};
  p.L = r.get<uint32_t>("config.L");
  p.K = r.get<uint32_t>("config.K");
  p.D = r.get<uint32_t>("config.D");
  p.alpha = r.get<float>("config.alpha");
  p.iprobes = r.get<uint32_t>("config.iProbes");
  p.kappa = r.get<uint32_t>("config.kappa");
  const uint32_t centering = r.get<uint32_t>("config.centering");
  const uint32_t mode = r.get<uint32_t>("config.mode");
  p.id_offset = r.get<uint32_t>("config.id_offset");
  p.seed = r.get<uint64_t>("seed");
  const uint64_t fn = r.get<uint64_t>("n");
  const uint32_t fd = r.get<uint32_t>("d");
  if (centering > 1 || mode > FPP_MODE_FALCONN_BASELINE)
    fail(FPP_ERR_FORMAT, "load: config.centering / config.mode out of range");
  if (fd == 0 || fd > (1u << 20)) fail(FPP_ERR_FORMAT, "load: d out of range");
  std::vector<float> center;
  if (centering) {
    center.resize(fd);
    r.get(center.data(), (size_t)fd * 4, "center");
  }
  const uint32_t plen = r.get<uint32_t>("dataset.path_len");
  if (plen > 4096) fail(FPP_ERR_FORMAT, "load: dataset.path_len out of range");
  std::string dpath(plen, '\0');
  r.get(&dpath[0], plen, "dataset.path");
  const uint64_t chash = r.get<uint64_t>("dataset.content_hash");
  if (fn != n || fd != d)
    fail(FPP_ERR_DIMENSION, "load: dataset shape " + std::to_string(n) + "x" + std::to_string(d) +
                                " does not match the index (" + std::to_string(fn) + "x" +
                                std::to_string(fd) + ")");
  // dataset reference check before anything is allocated.  The hash covers the
  // indexed rows: for a centered index the caller passes the raw rows and the
  // stored center is subtracted in fp32 first (dataset.cpp:52-55: bit for bit).
  if (!X && n) fail(FPP_ERR_INVALID_ARGUMENT, "load: X is NULL");
  std::vector<float> xh;
  const float* xsrc = X;
  bool src_dev = on_device;
  if (on_device || centering) {
    xh.resize((size_t)n * d);
    if (on_device) FPP_CUDA(cudaMemcpy(xh.data(), X, xh.size() * 4, cudaMemcpyDeviceToHost));
    else std::memcpy(xh.data(), X, xh.size() * 4);
    if (centering)
      for (uint64_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < d; ++j) xh[i * d + j] -= center[j];
    xsrc = xh.data();
    src_dev = false;
  }
  if (content_hash(xsrc, n, d) != chash)
    fail(FPP_ERR_FORMAT, "load: dataset content hash does not match the index");
  p.device = device;
  p.scratch_bytes = 0;
  p.mode = mode;
  p.centering = 0;  // xsrc is already centered
  Index* ix = prepare_index(xsrc, src_dev, n, d, &p);
  ix->prm.centering = centering;
  ix->center = center;
  try {
    const uint32_t L = p.L;
    const uint64_t NB = ix->NB;
    r.in_body = true;
    std::vector<uint32_t> offs((size_t)L * (NB + 1), 0);
    std::vector<uint32_t> ids;
    std::vector<float> sc;
    ix->table_base_h.assign(L + 1, 0);
    uint32_t mx = 0;
    for (uint32_t t = 0; t < L; ++t) {
      const uint32_t nonempty = r.get<uint32_t>("table.buckets");
      if (nonempty > NB) fail(FPP_ERR_FORMAT, "load: table.buckets out of range");
      uint32_t* of = offs.data() + (uint64_t)t * (NB + 1);
      uint64_t prev = 0, pos = 0;
      bool first = true;
      for (uint32_t k = 0; k < nonempty; ++k) {
        const uint32_t b = r.get<uint32_t>("bucket.id");
        const uint32_t cnt = r.get<uint32_t>("bucket.count");
        if (b >= NB || (!first && b <= prev) || cnt == 0 || cnt > n)
          fail(FPP_ERR_FORMAT, "load: bucket.id/count out of range or out of order");
        for (uint64_t bb = first ? 0 : prev + 1; bb <= b; ++bb) of[bb] = (uint32_t)pos;
        const size_t old = ids.size();
        ids.resize(old + cnt);
        sc.resize(old + cnt);
        std::vector<uint32_t> rec(2 * (size_t)cnt);
        r.get(rec.data(), rec.size() * 4, "bucket.entries");
        for (uint32_t j = 0; j < cnt; ++j) {
          if (rec[2 * j] >= n) fail(FPP_ERR_FORMAT, "load: point_id out of range");
          ids[old + j] = rec[2 * j];
          std::memcpy(&sc[old + j], &rec[2 * j + 1], 4);
        }
        pos += cnt;
        mx = std::max(mx, cnt);
        prev = b;
        first = false;
      }
      for (uint64_t bb = first ? 0 : prev + 1; bb <= NB; ++bb) of[bb] = (uint32_t)pos;
      ix->table_base_h[t + 1] = ix->table_base_h[t] + pos;
    }
    r.in_body = false;
    const uint64_t footer = r.get<uint64_t>("footer.checksum");
    if (footer != r.body_hash) fail(FPP_ERR_FORMAT, "load: body checksum mismatch");
    char extra;
    if (fread(&extra, 1, 1, fh.get()) == 1) fail(FPP_ERR_FORMAT, "load: trailing bytes after footer");
    ix->kept_total = ix->table_base_h[L];
    ix->max_bucket = mx;
    ix->offsets = static_cast<uint32_t*>(dmalloc(offs.size() * 4));
    ix->table_base = static_cast<uint64_t*>(dmalloc((size_t)(L + 1) * 8));
    ix->ids = static_cast<uint32_t*>(dmalloc((ix->kept_total + 1) * 4));
    ix->scores = static_cast<float*>(dmalloc((ix->kept_total + 1) * 4));
    FPP_CUDA(cudaMemcpyAsync(ix->offsets, offs.data(), offs.size() * 4, cudaMemcpyHostToDevice,
                             ix->stream));
    FPP_CUDA(cudaMemcpyAsync(ix->table_base, ix->table_base_h.data(), (L + 1) * 8,
                             cudaMemcpyHostToDevice, ix->stream));
    if (ix->kept_total) {
      FPP_CUDA(cudaMemcpyAsync(ix->ids, ids.data(), ix->kept_total * 4, cudaMemcpyHostToDevice,
                               ix->stream));
      FPP_CUDA(cudaMemcpyAsync(ix->scores, sc.data(), ix->kept_total * 4, cudaMemcpyHostToDevice,
                               ix->stream));
    }
    FPP_CUDA(cudaStreamSynchronize(ix->stream));
    ix->device_bytes = n * ix->ldx * 4 + ix->sign_words * 4 + offs.size() * 4 + (L + 1) * 8 +
                       ix->kept_total * 8;
  } catch (...) {
    delete ix;
    throw;
  }
  return ix;
}

}  // namespace fpp
