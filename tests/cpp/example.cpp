// Smoke program for the C++ host API (include/lsfann/falconnpp_gpu.hpp).
// Built by tests/test_capi.py; run by the GPU test.  Exit 0 on success,
// 2 if no GPU is present (the build step still validates the API).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "lsfann/falconnpp_gpu.hpp"

int main() {
  const std::size_t n = 2000, d = 32, nq = 8;
  std::vector<float> X(n * d), Q(nq * d);
  if (fpp_synth(X.data(), n, d, 4, 0.3f, 1, 0, 0) || fpp_normalize(X.data(), n, d)) return 1;
  if (fpp_synth(Q.data(), nq, d, 4, 0.3f, 1, 1, 0) || fpp_normalize(Q.data(), nq, d)) return 1;
  try {  // configuration errors surface as std::invalid_argument, like the reference
    lsfann::gpu::Index::build(X, n, d, 4, 3, 32, 3, 0.1f);
    return 1;
  } catch (const std::invalid_argument&) {
  }
  if (fpp_device_count() == 0) return 2;
  auto ix = lsfann::gpu::Index::build(X, n, d, 4, 2, 32, 3, 0.1f);
  auto r = ix.query(Q, nq, 10, 64, true);
  for (std::size_t i = 0; i < nq; ++i)
    for (int j = 0; j + 1 < 10; ++j)
      if (r.ids[i * 10 + j + 1] != 0xFFFFFFFFu && r.scores[i * 10 + j] < r.scores[i * 10 + j + 1])
        return 1;
  // rerank, ground truth and FLPP round trip through the C++ surface
  auto rr = ix.query_rerank(Q, nq, 10, 64, 40, true);
  for (std::size_t i = 0; i < nq; ++i)
    if (rr.stats[i].exact > 40) return 1;
  auto gt = ix.brute_force(Q, nq, 10);
  const char* path = "/tmp/fpp_cpp_example.flpp";
  ix.save(path);
  auto iy = lsfann::gpu::Index::load(path, X, n, d);
  auto r2 = iy.query(Q, nq, 10, 64, true);
  if (r2.ids != r.ids || r2.scores != r.scores) return 1;
  std::remove(path);
  // the same index over three shards of one process (all on device 0 here)
  const int32_t devs[3] = {0, 0, 0};
  auto mx = lsfann::gpu::MultiIndex::build(X, n, d, 4, 2, 32, 3, 0.1f, 3, devs);
  auto r3 = mx.query(Q, nq, 10, 64, true);
  if (mx.num_shards() != 3 || r3.ids != r.ids || r3.scores != r.scores) return 1;
  for (std::size_t i = 0; i < nq; ++i)
    if (r3.stats[i].probes != r.stats[i].probes || r3.stats[i].entries != r.stats[i].entries ||
        r3.stats[i].candidates != r.stats[i].candidates)
      return 1;
  std::printf("cpp ok: kept %llu, top1 %u (gt %u)\n", (unsigned long long)ix.info().kept_total,
              r.ids[0], gt.ids[0]);
  return 0;
}
