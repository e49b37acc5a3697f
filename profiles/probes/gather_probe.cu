// DRAM fetch granularity probe: random gathers of R-byte records from a large table.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
template <int R>  // bytes per record (16..128), 16 B per lane
__global__ void gather(const uint4* __restrict__ tab, uint64_t nrec, uint64_t nreq, uint4* out) {
  constexpr int LPR = R / 16;  // lanes per record
  const int lane = threadIdx.x & 31;
  uint4 acc = make_uint4(0, 0, 0, 0);
  const uint64_t nw = (uint64_t)gridDim.x * blockDim.x / 32;
  const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  for (uint64_t i = wid; i < nreq; i += nw) {  // one instruction: 32/LPR records
    const uint32_t rec = hsh((uint32_t)(i * (32 / LPR) + lane / LPR)) % nrec;
    const uint4 v = __ldcg(tab + (uint64_t)rec * LPR + lane % LPR);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678) out[0] = acc;
}
int main(int argc, char** argv) {
  if (argc > 1) {  // L2 fetch granularity hint (cudaLimitMaxL2FetchGranularity)
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, atoi(argv[1]));
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("set L2 fetch granularity %s -> %s, now %zu\n", argv[1], cudaGetErrorString(e), v);
  } else {
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("default L2 fetch granularity %zu\n", v);
  }
  const size_t bytes = 640ull << 20;
  uint4* tab; uint4* out;
  cudaMalloc(&tab, bytes); cudaMalloc(&out, 64);
  cudaMemset(tab, 1, bytes);
  const uint64_t nreq = 1ull << 22;  // warp-instructions
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
#define RUN(R) { const uint64_t nrec = bytes / R; gather<R><<<148 * 8, 256>>>(tab, nrec, nreq, out); \
  cudaEventRecord(a); gather<R><<<148 * 8, 256>>>(tab, nrec, nreq, out); cudaEventRecord(b); cudaEventSynchronize(b); \
  float ms; cudaEventElapsedTime(&ms, a, b); double req = (double)nreq * 512; \
  printf("R=%3d requested %.2f GB in %.3f ms = %.0f GB/s\n", R, req / 1e9, ms, req / ms / 1e6); }
  RUN(16) RUN(32) RUN(64) RUN(128)
  return 0;
}
