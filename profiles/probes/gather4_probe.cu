// Row-gather probe: random rows of X[n][d] (fp32) streamed into shared memory as
// 32-row x 64-float slices per warp, the way k_score / k_score_pruned stage candidate
// rows, by (A) the per-lane 16-byte cp.async ring the product kernels use (LDGSTS) and
// (B) TMA tile::gather4 (UTMALDG.2D.GATHER4: one instruction = 4 arbitrary rows x 64
// floats, completion on an mbarrier).  Same ring depth, same light consumer (one
// float4 per row slice).  Reports requested GB/s; build and run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o gather4_probe gather4_probe.cu
//   ./gather4_probe [box_rows]      (box_rows: boxDim[1] of the tensor map, 4 or 1)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int WARPS = 4, STAGES = 2, SL = 64;        // floats per row slice
constexpr int STAGE_FLOATS_A = 32 * (SL + 4);        // padded rows (conflict-free LDS.128)
constexpr int STAGE_FLOATS_B = 32 * SL;              // TMA box rows are dense

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void fill(float* X, uint64_t n, uint32_t d) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * d; i += (uint64_t)gridDim.x * blockDim.x)
    X[i] = (float)((i / d) % 4096) + (float)(i % d) / 1024.f;
}
__device__ __forceinline__ float expect(uint32_t row, uint32_t col) { return (float)(row % 4096) + (float)col / 1024.f; }

// ---------------------------------------------------------------- A: LDGSTS ring
// WIDE: an instruction covers 2 rows x 256 contiguous bytes (16 lanes per row) instead of
// 4 rows x 128 bytes (8 lanes per row, the product kernels' mapping)
template <bool WIDE>
__global__ void __launch_bounds__(WARPS * 32) gather_ldgsts(const float* __restrict__ X, uint32_t n, uint32_t d,
                                                            uint32_t batches, float* out, unsigned* bad) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* ring = reinterpret_cast<float*>(sm) + (size_t)w * STAGES * STAGE_FLOATS_A;
  const uint32_t nsl = d / SL;
  const uint32_t wid = blockIdx.x * WARPS + w, nw = gridDim.x * WARPS;
  const int kk = lane & 7, rbase = lane >> 3;
  float acc = 0.f;
  uint32_t ib = wid, ic = 0, nissued = 0;
  const float* rp[WIDE ? 16 : 8];
  auto load_batch = [&](uint32_t b) {
    const uint32_t id = hsh(b * 32 + lane) % n;
    if (WIDE) {
#pragma unroll
      for (int it = 0; it < 16; ++it) rp[it] = X + (uint64_t)__shfl_sync(0xffffffffu, id, (lane >> 4) + 2 * it) * d;
    } else {
#pragma unroll
      for (int it = 0; it < 8; ++it) rp[it] = X + (uint64_t)__shfl_sync(0xffffffffu, id, rbase + 4 * it) * d;
    }
  };
  auto issue = [&]() {
    if (ib < batches) {
      float* buf = ring + (size_t)(nissued % STAGES) * STAGE_FLOATS_A;
      if (WIDE) {
#pragma unroll
        for (int it = 0; it < 16; ++it) {
          const uint32_t sa = smem_u32(buf + ((lane >> 4) + 2 * it) * (SL + 4) + (lane & 15) * 4);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(rp[it] + ic * SL + (lane & 15) * 4) : "memory");
        }
      } else {
#pragma unroll
      for (int h = 0; h < SL / 32; ++h)
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const uint32_t sa = smem_u32(buf + (rbase + 4 * it) * (SL + 4) + (kk + 8 * h) * 4);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(rp[it] + ic * SL + (kk + 8 * h) * 4) : "memory");
        }
      }
      if (++ic == nsl) { ic = 0; ib += nw; if (ib < batches) load_batch(ib); }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    ++nissued;
  };
  if (ib < batches) load_batch(ib);
  for (int s = 0; s < STAGES - 1; ++s) issue();
  uint32_t cb = wid, cc = 0, ncomp = 0;
  while (cb < batches) {
    issue();
    asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 1) : "memory");
    __syncwarp();
    const float* row = ring + (size_t)(ncomp % STAGES) * STAGE_FLOATS_A + lane * (SL + 4);
    const float4 v = *reinterpret_cast<const float4*>(row + 4 * (lane & 15));
    acc += v.x + v.y + v.z + v.w;
    if (v.y != expect(hsh(cb * 32 + lane) % n, cc * SL + 4 * (lane & 15) + 1)) atomicAdd(bad, 1u);
    __syncwarp();
    ++ncomp;
    if (++cc == nsl) { cc = 0; cb += nw; }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (acc == 12345.678f) out[0] = acc;
}

// ---------------------------------------------------------------- B: TMA gather4 ring
// SWZ: box = 32 floats (128 B) with CU_TENSOR_MAP_SWIZZLE_128B; a stage is [2 halves][32 rows][128 B],
// 1024-byte aligned, so row r's 16-byte chunk c sits at chunk c ^ (r & 7) and lane r reading its own
// row sequentially (the product kernels' access) is bank-conflict free; 16 instructions per slice
template <bool SWZ>
__global__ void __launch_bounds__(WARPS * 32) gather_tma4(const __grid_constant__ CUtensorMap tm, uint32_t n, uint32_t d,
                                                          uint32_t batches, float* out, unsigned* fail) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[WARPS][STAGES];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // the swizzle pattern is a function of the shared-memory address: 1024-byte aligned stages
  float* ring = reinterpret_cast<float*>(sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u)) +
                (size_t)w * STAGES * STAGE_FLOATS_B;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[w][s])) : "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncwarp();
  const uint32_t nsl = d / SL;
  const uint32_t wid = blockIdx.x * WARPS + w, nw = gridDim.x * WARPS;
  float acc = 0.f;
  uint32_t ib = wid, ic = 0, nissued = 0;
  int r0 = 0, r1 = 0, r2 = 0, r3 = 0;  // lanes 0..7: the four rows of their gather4
  auto load_batch = [&](uint32_t b) {
    const uint32_t id = hsh(b * 32 + lane) % n;
    const int s4 = 4 * (lane & 7);
    r0 = (int)__shfl_sync(0xffffffffu, id, s4);
    r1 = (int)__shfl_sync(0xffffffffu, id, s4 + 1);
    r2 = (int)__shfl_sync(0xffffffffu, id, s4 + 2);
    r3 = (int)__shfl_sync(0xffffffffu, id, s4 + 3);
  };
  auto issue = [&]() {
    if (ib < batches) {
      const int st = nissued % STAGES;
      float* buf = ring + (size_t)st * STAGE_FLOATS_B;
      const uint32_t mb = smem_u32(&bar[w][st]);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(32 * SL * 4) : "memory");
      __syncwarp();
      if (lane < (SWZ ? 16 : 8)) {
        const uint32_t dst = SWZ ? smem_u32(buf + (lane >> 3) * 32 * 32 + (lane & 7) * 4 * 32)
                                 : smem_u32(buf + lane * 4 * SL);
        const int col = (int)(ic * SL) + (SWZ ? (lane >> 3) * 32 : 0);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];\n" ::"r"(dst),
            "l"(&tm), "r"(mb), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
            : "memory");
      }
      if (++ic == nsl) { ic = 0; ib += nw; if (ib < batches) load_batch(ib); }
    }
    ++nissued;
  };
  if (ib < batches) load_batch(ib);
  for (int s = 0; s < STAGES - 1; ++s) issue();
  uint32_t cb = wid, cc = 0, ncomp = 0;
  while (cb < batches) {
    issue();
    const int st = ncomp % STAGES;
    const uint32_t mb = smem_u32(&bar[w][st]), par = (ncomp / STAGES) & 1;
    uint32_t done = 0, spins = 0;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(mb), "r"(par) : "memory");
    } while (!done && ++spins < (1u << 22));
    if (!done) { if (lane == 0) atomicAdd(fail, 1u); return; }  // bounded: never hang the box
    const int c4 = SWZ ? (int)(ncomp & 15) : ((lane + (lane >> 3)) & 15);  // SWZ: every lane the same column
    const float* row = SWZ ? ring + (size_t)st * STAGE_FLOATS_B + (c4 >> 3) * 32 * 32 + lane * 32 +
                                 4 * ((c4 & 7) ^ (lane & 7)) - 4 * c4
                           : ring + (size_t)st * STAGE_FLOATS_B + lane * SL;
    const float4 v = *reinterpret_cast<const float4*>(row + 4 * c4);
    acc += v.x + v.y + v.z + v.w;
    if (v.y != expect(hsh(cb * 32 + lane) % n, cc * SL + 4 * c4 + 1)) atomicAdd(fail + 1, 1u);
    __syncwarp();
    ++ncomp;
    if (++cc == nsl) { cc = 0; cb += nw; }
  }
  if (acc == 12345.678f) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int box_rows = argc > 1 ? atoi(argv[1]) : 1;  // gather4 wants boxDim[1] = 1 (4: illegal instruction)
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
  if (!fn) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  float* out; unsigned* fail;
  CK(cudaMalloc(&out, 64)); CK(cudaMalloc(&fail, 16));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  const uint32_t ds[] = {128, 320, 960};
  for (uint32_t d : ds) {
    const uint64_t bytes = 3ull << 30;
    const uint32_t n = (uint32_t)(bytes / (d * 4ull));
    float* X; CK(cudaMalloc(&X, (size_t)n * d * 4)); fill<<<148 * 8, 256>>>(X, n, d); CK(cudaDeviceSynchronize());
    const uint32_t batches = (uint32_t)((2ull << 30) / (32ull * d * 4));  // 2 GB of rows per run
    const int grid = 148 * 3;
    const size_t smA = (size_t)WARPS * STAGES * STAGE_FLOATS_A * 4, smB = (size_t)WARPS * STAGES * STAGE_FLOATS_B * 4;
    CK(cudaFuncSetAttribute(gather_ldgsts<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA));
    CK(cudaFuncSetAttribute(gather_ldgsts<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA));
    CK(cudaFuncSetAttribute(gather_tma4<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB + 1024));
    CK(cudaFuncSetAttribute(gather_tma4<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB + 1024));
    float ms;
    unsigned hb[4] = {0, 0, 0, 0};
    const double gb = (double)batches * 32 * d * 4 / 1e9;
    for (int wide = 0; wide < 2; ++wide) {
      CK(cudaMemset(fail, 0, 16));
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(a));
        if (wide) gather_ldgsts<true><<<grid, WARPS * 32, smA>>>(X, n, d, batches, out, fail + 2);
        else gather_ldgsts<false><<<grid, WARPS * 32, smA>>>(X, n, d, batches, out, fail + 2);
        CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b)); CK(cudaEventElapsedTime(&ms, a, b));
      }
      CK(cudaMemcpy(hb, fail, 16, cudaMemcpyDeviceToHost));
      printf("d=%4u LDGSTS ring %s: %.2f GB in %7.3f ms = %6.0f GB/s  (mismatches %u)\n", d,
             wide ? "2 rows x 256 B / instruction " : "4 rows x 128 B / instruction ", gb, ms, gb / ms * 1e3, hb[2]);
    }
    for (int swz = 0; swz < 2; ++swz) {
      CUtensorMap tm;
      const cuuint64_t gdim[2] = {d, n};
      const cuuint64_t gstr[1] = {(cuuint64_t)d * 4};
      const cuuint32_t box[2] = {swz ? 32u : (cuuint32_t)SL, (cuuint32_t)box_rows};
      const cuuint32_t estr[2] = {1, 1};
      CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, gdim, gstr, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("d=%u cuTensorMapEncodeTiled(box rows %d) failed: %d\n", d, box_rows, (int)r); continue; }
      CK(cudaMemset(fail, 0, 16));
      const size_t smT = smB + 1024;
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(a));
        if (swz) gather_tma4<true><<<grid, WARPS * 32, smT>>>(tm, n, d, batches, out, fail);
        else gather_tma4<false><<<grid, WARPS * 32, smT>>>(tm, n, d, batches, out, fail);
        CK(cudaEventRecord(b));
        cudaError_t e = cudaEventSynchronize(b);
        if (e != cudaSuccess) { printf("d=%u gather4 kernel: %s\n", d, cudaGetErrorString(e)); return 2; }
        CK(cudaEventElapsedTime(&ms, a, b));
      }
      CK(cudaMemcpy(hb, fail, 16, cudaMemcpyDeviceToHost));
      printf("d=%4u TMA gather4 %s: %.2f GB in %7.3f ms = %6.0f GB/s  (timed-out waits %u, mismatches %u)\n", d,
             swz ? "32-float box, 128B swizzle" : "64-float box, no swizzle  ", gb, ms, gb / ms * 1e3, hb[0], hb[1]);
    }
    CK(cudaFree(X));
  }
  return 0;
}
