// fpp_device.cuh -- device primitives shared by the build and query kernels.
//
// * order-preserving float keys (total orders of DESIGN.md section 3)
// * the warp-group Fast Hadamard Transform with the reference butterfly graph
//   (rotation.cpp:16-32: len ascending, a[j]=x+y, a[j+len]=x-y), which is what
//   makes GPU projections bit-identical to SpinnerStack::project
// * group-wide top-R selection of (|p| desc, index asc) keys
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fpp {

constexpr unsigned FULL = 0xffffffffu;

// Monotone map float -> uint32 (ascending).  -0.0 is canonicalised to +0.0 so
// that key equality coincides with float equality (ties compare equal).
__device__ __forceinline__ uint32_t ord_key(float f) {
  uint32_t u = __float_as_uint(f + 0.0f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// ---------------------------------------------------------------- FHT group
// A group of G = P/EPT consecutive lanes holds one length-P vector, lane g
// owning elements j = g*EPT + e (e in [0,EPT)).  Stages with len < EPT are
// in-register; len >= EPT exchange with lane g ^ (len/EPT) through shfl.xor.
// The stage ORDER is the reference's (len ascending), and each output element
// is computed with the same operand order (x+y for the lower, x-y for the upper
// element), so every intermediate is bit-identical to rotation.cpp:22-31.
template <int P>
struct FhtShape {
  static constexpr int EPT = P < 32 ? P : 32;
  static constexpr int G = P / EPT;    // lanes per vector
  static constexpr int GPW = 32 / G;   // vectors per warp
  static constexpr int W = P < 32 ? 1 : P / 32;  // 32-bit sign words per stage
};

template <int P, int EPT>
__device__ __forceinline__ void fht_group(float (&v)[EPT], int g) {
#pragma unroll
  for (int len = 1; len < EPT; len <<= 1) {
#pragma unroll
    for (int i = 0; i < EPT; i += 2 * len) {
#pragma unroll
      for (int j = i; j < i + len; ++j) {
        const float x = v[j], y = v[j + len];
        v[j] = x + y;
        v[j + len] = x - y;
      }
    }
  }
  // cross-lane stages: the upper lane needs x - y = o - v, computed as (-v) + o
  // (IEEE a - b is a + (-b): bit-identical), so every lane does one XOR + FADD.
#pragma unroll 1
  for (int m = 1; m < P / EPT; m <<= 1) {
    const uint32_t neg = (g & m) ? 0x80000000u : 0u;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const float o = __shfl_xor_sync(FULL, v[e], m);
      v[e] = __uint_as_float(__float_as_uint(v[e]) ^ neg) + o;
    }
  }
}

// Multiply by the +/-1 diagonal of one stage: bit e of `w` set -> +1, clear -> -1
// (rotation.cpp:55-67,93).  Done as a sign-bit XOR, bit-identical to x * (+/-1.0f).
template <int EPT>
__device__ __forceinline__ void apply_signs(float (&v)[EPT], uint32_t w) {
#pragma unroll
  for (int e = 0; e < EPT; ++e)
    v[e] = __uint_as_float(__float_as_uint(v[e]) ^ (((~w >> e) & 1u) << 31));
}

// Full SpinnerStack::project of one block (rotation.cpp:81-98): 3 x (signs, FHT),
// then the exact power-of-two scale 1/P.  `sw` points at this stack's
// [3][W] sign words.
template <int P>
__device__ __forceinline__ void spinner_project(float (&v)[FhtShape<P>::EPT], const uint32_t* sw,
                                                int g) {
  using S = FhtShape<P>;
  // the three rounds' sign words are loaded up front (one latency, not three)
  const uint32_t gi = S::G > 1 ? g : 0;
  const uint32_t w0 = __ldg(sw + gi), w1 = __ldg(sw + S::W + gi), w2 = __ldg(sw + 2 * S::W + gi);
#pragma unroll 1
  for (int stage = 0; stage < 3; ++stage) {
    const uint32_t w = stage == 0 ? w0 : (stage == 1 ? w1 : w2);
    apply_signs<S::EPT>(v, w);
    fht_group<P, S::EPT>(v, g);
  }
  const float scale = 1.0f / (float)P;
#pragma unroll
  for (int e = 0; e < S::EPT; ++e) v[e] = v[e] * scale;
}

// ------------------------------------------------- packed FP32 butterflies
// Two butterflies in one FADD2 pair (add/sub.rn.f32x2, sm_100a): (a0, a1) <- (a0 + b0,
// a1 + b1) and (b0, b1) <- (a0 - b0, a1 - b1).  Each lane of the packed op is the IEEE
// round-to-nearest add / subtract of the scalar code (same operands, same order), so
// results are bit-identical; the FP32 instruction count of the FHT halves.
__device__ __forceinline__ void bfly2(float& a0, float& a1, float& b0, float& b1) {
  asm("{.reg .b64 ra, rb, rs, rd;\n\t"
      "mov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %3};\n\t"
      "add.rn.f32x2 rs, ra, rb;\n\tsub.rn.f32x2 rd, ra, rb;\n\t"
      "mov.b64 {%0, %1}, rs;\n\tmov.b64 {%2, %3}, rd;\n\t}"
      : "+f"(a0), "+f"(a1), "+f"(b0), "+f"(b1));
}

// one in-register butterfly stage of stride `len` over 32 registers (reference
// operand order x + y low, x - y high); strides >= 2 pair neighbouring butterflies
// (j, j + 1) into one FADD2
template <int len>
__device__ __forceinline__ void fht_stage32(float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 32; i += 2 * len) {
    if constexpr (len >= 2) {
#pragma unroll
      for (int j = i; j < i + len; j += 2) bfly2(v[j], v[j + 1], v[j + len], v[j + len + 1]);
    } else {
      const float x = v[i], y = v[i + 1];
      v[i] = x + y;
      v[i + 1] = x - y;
    }
  }
}

// x * s for 32 registers, two per FMUL2 (mul.rn.f32x2: per-lane IEEE products)
__device__ __forceinline__ void scale32(float (&v)[32], float s) {
#pragma unroll
  for (int e = 0; e < 32; e += 2)
    asm("{.reg .b64 ra, rs, rd;\n\t"
        "mov.b64 ra, {%0, %1};\n\tmov.b64 rs, {%2, %2};\n\t"
        "mul.rn.f32x2 rd, ra, rs;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "+f"(v[e]), "+f"(v[e + 1])
        : "f"(s));
}

// ------------------------------------------------ transpose FHT (P >= 64)
// Same butterfly graph as fht_group, but the cross-lane stages run in
// registers after one shared-memory transpose per round instead of log2(G)
// shuffle stages:
//   layout A: lane g holds j = g*32 + e              (index bits 0..4 in registers)
//   layout B: lane g holds j = (e / RUN)*32 + g*RUN + (e % RUN), RUN = 32/G
//             (index bits 0..lgRUN-1 and 5..5+lgG-1 in registers: runs of RUN
//             contiguous elements, so both sides of the transpose move 16-byte
//             vectors for P <= 256, 8-byte for P = 512; P = 1024: RUN = 1)
// Register stride RUN*2^m is index bit 5 + m in layout B, so the cross-lane stages are
// the in-register strides RUN .. 16 (fht_regs_B).
// Per-group scratch: TransposeShape<P>::STRIDE floats (16-byte aligned), padded
// (4 floats per 32) so the vectorised A rows (36 floats apart) and the B runs are
// free of bank conflicts, and group regions are offset to different banks.
template <int P>
struct TransposeShape {
  static constexpr int G = P / 32;
  static constexpr int STRIDE = P / 32 * 36 + (G < 4 ? 4 : (G % 32));
};
__device__ __forceinline__ int tpad(int j) { return j + ((j >> 5) << 2); }

// layout B: the index held by register e of lane g
template <int P>
__host__ __device__ constexpr uint32_t jB(int e, int g) {
  constexpr int RUN = 32 / (P / 32);
  return (uint32_t)((e / RUN) * 32 + g * RUN + (e % RUN));
}

// in-register butterflies of layout B: run the stages of index bits 5 .. 5+lgG-1
// (register strides 32/G .. 16)
template <int P>
__device__ __forceinline__ void fht_regs_B(float (&v)[32]) {
  constexpr int G = P / 32;
  if constexpr (32 / G <= 1) fht_stage32<1>(v);
  if constexpr (32 / G <= 2) fht_stage32<2>(v);
  if constexpr (32 / G <= 4) fht_stage32<4>(v);
  if constexpr (32 / G <= 8) fht_stage32<8>(v);
  fht_stage32<16>(v);
}

// Layout-B registers <-> the padded buffer: register e = c*RUN + r lives at float
// offset 36*c + g*RUN + r (tpad of jB: the run stays inside one 32-block).  Every
// access is base register + immediate.
template <int P, bool LOAD>
__device__ __forceinline__ void move_B(float (&v)[32], float* rb) {
  constexpr int G = P / 32, RUN = 32 / G;
#pragma unroll
  for (int c = 0; c < G; ++c) {
    if constexpr (RUN >= 4) {
#pragma unroll
      for (int i = 0; i < RUN; i += 4) {
        float4* p4 = reinterpret_cast<float4*>(rb + 36 * c + i);
        const int e = c * RUN + i;
        if constexpr (LOAD) {
          const float4 q = *p4;
          v[e] = q.x; v[e + 1] = q.y; v[e + 2] = q.z; v[e + 3] = q.w;
        } else {
          *p4 = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
        }
      }
    } else if constexpr (RUN == 2) {
      float2* p2 = reinterpret_cast<float2*>(rb + 36 * c);
      if constexpr (LOAD) {
        const float2 q = *p2;
        v[2 * c] = q.x; v[2 * c + 1] = q.y;
      } else {
        *p2 = make_float2(v[2 * c], v[2 * c + 1]);
      }
    } else {
      if constexpr (LOAD) v[c] = rb[36 * c];
      else rb[36 * c] = v[c];
    }
  }
}

template <int P>
__device__ __forceinline__ void transpose_A_to_B(float (&v)[32], int g, float* buf) {
  constexpr int RUN = 32 / (P / 32);
  float* ra = buf + 36 * g;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    *reinterpret_cast<float4*>(ra + 4 * k) =
        make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  __syncwarp();
  move_B<P, true>(v, buf + g * RUN);
  __syncwarp();
}

template <int P>
__device__ __forceinline__ void transpose_B_to_A(float (&v)[32], int g, float* buf) {
  constexpr int RUN = 32 / (P / 32);
  float* ra = buf + 36 * g;
  move_B<P, false>(v, buf + g * RUN);
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float4 q = *reinterpret_cast<const float4*>(ra + 4 * k);
    v[4 * k] = q.x; v[4 * k + 1] = q.y; v[4 * k + 2] = q.z; v[4 * k + 3] = q.w;
  }
  __syncwarp();
}

// The index held by register e of lane g after a projection: layout B after the
// transpose FHT (P >= 64), layout A (j = g*EPT + e) after the shuffle FHT.
template <int P>
__host__ __device__ constexpr uint32_t layout_index(int e, int g) {
  if constexpr (P >= 64) return jB<P>(e, g);
  else return (uint32_t)(g * (P < 32 ? P : 32) + e);
}

// Layout-B registers to an UNPADDED natural-order buffer (nat[j] = value of index j),
// vectorised by runs (16-byte aligned buffer).
template <int P>
__device__ __forceinline__ void store_B_natural(const float (&v)[32], int g, float* nat) {
  constexpr int G = P / 32, RUN = 32 / G;
  float* rb = nat + g * RUN;
#pragma unroll
  for (int c = 0; c < G; ++c) {
    if constexpr (RUN >= 4) {
#pragma unroll
      for (int i = 0; i < RUN; i += 4) {
        const int e = c * RUN + i;
        *reinterpret_cast<float4*>(rb + 32 * c + i) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
      }
    } else if constexpr (RUN == 2) {
      *reinterpret_cast<float2*>(rb + 32 * c) = make_float2(v[2 * c], v[2 * c + 1]);
    } else {
      rb[32 * c] = v[c];
    }
  }
}

// Rounds 2 and 3 of the transpose FHT without leaving layout B (P <= 128, FPP_FHT_SHFL):
// k_hash_build is bound by shared-memory wavefronts, and the B->A->B transposes of a
// round cost 2 x 2 x P x 4 bytes of them.  Layout B already holds index bits
// 0..lgRUN-1 and 5.. in registers; the lgG bits in between live in the lane id, so
// their stages are a shuffle plus one FMA per element,
//   lower lane:  x + y = fma(v, +1, o)      upper lane:  x - y = o - v = fma(v, -1, o)
// (the product is exact, so the FMA is the IEEE add / subtract of the reference
// butterfly, operands in its order).  The stage order stays len ascending.
// Measured (B200): shuffles load the same crossbar as shared memory, so the plan pays
// while lgG shuffle stages (32 SHFL each) cost less than the two transposes (128
// wavefronts): P = 128 query hashing 8.2 -> 7.4 ms (C4), P = 256 build hashing 3.70 ->
// 3.86 s (C5, three stages: kept on the transposes).
#ifndef FPP_FHT_SHFL
#define FPP_FHT_SHFL 1
#endif
template <int P>
struct FhtPlan {
  static constexpr int G = P / 32;
  static constexpr bool SHFL = FPP_FHT_SHFL && P >= 64 && P <= 128;
};

// index of the sign bit that bit e of lane g's word of round `round` holds (host packing
// and device use must agree): layout A, except rounds 1 and 2 of the shuffle plan (B)
template <int P>
__host__ __device__ constexpr uint32_t sign_index(int round, int e, int g) {
  if constexpr (P >= 64) {
    if (FhtPlan<P>::SHFL && round > 0) return jB<P>(e, g);
  }
  return (uint32_t)(g * (P < 32 ? P : 32) + e);
}

__device__ __forceinline__ void fma2_lane(float& a0, float& a1, float s, float o0, float o1) {
  asm("{.reg .b64 ra, rs, ro, rd;\n\t"
      "mov.b64 ra, {%0, %1};\n\tmov.b64 rs, {%2, %2};\n\tmov.b64 ro, {%3, %4};\n\t"
      "fma.rn.f32x2 rd, ra, rs, ro;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(s), "f"(o0), "f"(o1));
}

// one cross-lane butterfly stage (lane bit m): every register of the lane pairs with
// the same register of lane g ^ m
__device__ __forceinline__ void fht_stage_lane(float (&v)[32], int g, int m) {
  const float sg = (g & m) ? -1.0f : 1.0f;
#pragma unroll
  for (int e = 0; e < 32; e += 2) {
    const float o0 = __shfl_xor_sync(FULL, v[e], m);
    const float o1 = __shfl_xor_sync(FULL, v[e + 1], m);
    fma2_lane(v[e], v[e + 1], sg, o0, o1);
  }
}

// SpinnerStack::project with transpose FHTs: input in layout A, output in
// layout B (element e of lane g is index jB<P>(e, g)), scaled by 1/P.
template <int P>
__device__ __forceinline__ void spinner_project_T(float (&v)[32], const uint32_t* sw, int g,
                                                  float* buf) {
  constexpr int G = P / 32;
  // the three rounds' sign words are loaded up front (one latency, not three)
  const uint32_t w0 = __ldg(sw + g), w1 = __ldg(sw + G + g), w2 = __ldg(sw + 2 * G + g);
  if constexpr (FhtPlan<P>::SHFL) {
    constexpr int RUN = 32 / G;
    apply_signs<32>(v, w0);
    fht_stage32<1>(v);
    fht_stage32<2>(v);
    fht_stage32<4>(v);
    fht_stage32<8>(v);
    fht_stage32<16>(v);
    transpose_A_to_B<P>(v, g, buf);
    fht_regs_B<P>(v);
#pragma unroll 1
    for (int stage = 1; stage < 3; ++stage) {
      apply_signs<32>(v, stage == 1 ? w1 : w2);  // words packed in layout B (sign_index)
      // index bits 0 .. lgRUN-1: register strides 1 .. RUN/2
      fht_stage32<1>(v);
      if constexpr (RUN > 2) fht_stage32<2>(v);
      if constexpr (RUN > 4) fht_stage32<4>(v);
      if constexpr (RUN > 8) fht_stage32<8>(v);
      // index bits lgRUN .. 4: lane bits 0 .. lgG-1
#pragma unroll
      for (int m = 1; m < G; m <<= 1) fht_stage_lane(v, g, m);
      // index bits 5 ..: register strides RUN .. 16
      fht_regs_B<P>(v);
    }
  } else {
#pragma unroll 1
    for (int stage = 0; stage < 3; ++stage) {
      if (stage) transpose_B_to_A<P>(v, g, buf);
      apply_signs<32>(v, stage == 0 ? w0 : (stage == 1 ? w1 : w2));
      fht_stage32<1>(v);
      fht_stage32<2>(v);
      fht_stage32<4>(v);
      fht_stage32<8>(v);
      fht_stage32<16>(v);
      transpose_A_to_B<P>(v, g, buf);
      fht_regs_B<P>(v);
    }
  }
  scale32(v, 1.0f / (float)P);
}

// Load row x[0..d) into the group layout, zero-padded to P (rotation.cpp:88-89).
template <int P>
__device__ __forceinline__ void load_row(const float* __restrict__ x, uint32_t d, int g,
                                         float (&v)[FhtShape<P>::EPT]) {
  constexpr int EPT = FhtShape<P>::EPT;
  const uint32_t base = (uint32_t)g * EPT;
  if ((d & 3u) == 0 && (EPT % 4) == 0) {
#pragma unroll
    for (int e = 0; e < EPT; e += 4) {
      if (base + e < d) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(x + base + e));
        v[e] = q.x; v[e + 1] = q.y; v[e + 2] = q.z; v[e + 3] = q.w;
      } else {
        v[e] = v[e + 1] = v[e + 2] = v[e + 3] = 0.0f;
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < EPT; ++e) v[e] = (base + e < d) ? __ldg(x + base + e) : 0.0f;
  }
}

// -------------------------------------------------------- top-R rank keys
// key = (~ord(|p|)) << 32 | (j << 1) | (p < 0): ascending key order is
// (|p| desc, j asc) -- the natural ranked list of DESIGN.md section 3; the low
// bit carries the sign so the code (j or D+j) can be recovered.
__device__ __forceinline__ uint64_t rank_key(float p, uint32_t j) {
  const uint32_t hi = ~ord_key(fabsf(p));
  return ((uint64_t)hi << 32) | ((uint64_t)j << 1) | (p < 0.0f ? 1u : 0u);
}
__device__ __forceinline__ float rank_val(uint64_t k) { return ord_inv(~(uint32_t)(k >> 32)); }
__device__ __forceinline__ uint32_t rank_code(uint64_t k, uint32_t D) {
  const uint32_t j = (uint32_t)(k & 0xffffffffu) >> 1;
  return (k & 1u) ? D + j : j;
}


// merge sorted lists across the G lanes of a group (butterfly; every lane ends
// with the group's R smallest keys, ascending).  Bitonic merge per step.
template <int R, int G>
__device__ __forceinline__ void topr_group_merge(uint64_t (&t)[R]) {
#pragma unroll
  for (int m = 1; m < G; m <<= 1) {
    uint64_t o[R];
#pragma unroll
    for (int i = 0; i < R; ++i) o[i] = __shfl_xor_sync(FULL, t[i], m);
    // t ascending, o ascending: min(t[i], o[R-1-i]) is bitonic and holds the R smallest
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint64_t b = o[R - 1 - i];
      t[i] = t[i] < b ? t[i] : b;
    }
#pragma unroll
    for (int k = R / 2; k > 0; k >>= 1) {
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int p = i ^ k;
        if (p > i) {
          const uint64_t a = t[i], b = t[p];
          t[i] = a < b ? a : b;
          t[p] = a < b ? b : a;
        }
      }
    }
  }
}

// Bitonic sort (ascending) of the P = G*EPT keys held by a lane group, element
// index i = g*EPT + e.  In-register compare-exchanges for strides < EPT,
// shfl.xor for strides >= EPT.  Fully unrolled (P, EPT compile-time).
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  const uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)v, m);
  const uint32_t hi = __shfl_xor_sync(FULL, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}

template <int P, int EPT>
__device__ __forceinline__ void group_bitonic_sort(uint64_t (&k)[EPT], int g) {
#pragma unroll
  for (int size = 2; size <= P; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= EPT) {
        const int m = stride / EPT;
        const bool lower = (g & m) == 0;
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          const uint64_t o = shfl_xor_u64(k[e], m);
          const bool asc = (((g * EPT + e) & size) == 0);
          const uint64_t mn = k[e] < o ? k[e] : o, mx = k[e] < o ? o : k[e];
          k[e] = (lower == asc) ? mn : mx;
        }
      } else {
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          if (e & stride) continue;
          const int e2 = e | stride;
          const bool asc = (((g * EPT + e) & size) == 0);
          const uint64_t a = k[e], b = k[e2];
          const uint64_t mn = a < b ? a : b, mx = a < b ? b : a;
          k[e] = asc ? mn : mx;
          k[e2] = asc ? mx : mn;
        }
      }
    }
  }
}

// Bitonic sort v2 (ascending, 32-bit keys, index i = g*EPT + e).  Sizes below
// EPT have compile-time directions; for sizes >= EPT every lane's elements share
// one direction, so descending blocks are complemented (~k) and all stages run
// as plain ascending min/max (the complement reverses the order exactly).
template <int S, int EPT>
__device__ __forceinline__ void ce_up_u32(uint32_t (&k)[EPT]) {
  if (S >= EPT) return;
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    if (e & S) continue;
    const uint32_t a = k[e], b = k[e | S];
    k[e] = min(a, b);
    k[e | S] = max(a, b);
  }
}

template <int P, int EPT>
__device__ __forceinline__ void group_sort_u32_v2(uint32_t (&k)[EPT], int g) {
#pragma unroll
  for (int size = 2; size < EPT; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        if (e & stride) continue;
        const uint32_t a = k[e], b = k[e | stride];
        const bool asc = (e & size) == 0;  // compile-time per element
        k[e] = asc ? min(a, b) : max(a, b);
        k[e | stride] = asc ? max(a, b) : min(a, b);
      }
    }
  }
#pragma unroll 1
  for (int size = EPT; size <= P; size <<= 1) {
    const uint32_t flip = ((g * EPT) & size) ? 0xffffffffu : 0u;
#pragma unroll
    for (int e = 0; e < EPT; ++e) k[e] ^= flip;
#pragma unroll 1
    for (int stride = size >> 1; stride >= EPT; stride >>= 1) {
      const int m = stride / EPT;
      const bool lower = (g & m) == 0;
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const uint32_t o = __shfl_xor_sync(FULL, k[e], m);
        k[e] = lower ? min(k[e], o) : max(k[e], o);
      }
    }
    ce_up_u32<16, EPT>(k);
    ce_up_u32<8, EPT>(k);
    ce_up_u32<4, EPT>(k);
    ce_up_u32<2, EPT>(k);
    ce_up_u32<1, EPT>(k);
#pragma unroll
    for (int e = 0; e < EPT; ++e) k[e] ^= flip;
  }
}

// Shared-memory increment without a result (red.shared): plain atomicAdd on a
// data-dependent address gets a compiler-generated warp-aggregation sequence
// (vote / find-leader / popc loop) that costs ~10 instructions per call.
__device__ __forceinline__ void smem_inc(uint32_t* p) {
  asm volatile("red.shared.add.u32 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
}

// Shared-memory fetch-add issued by one lane (same reason as smem_inc).
__device__ __forceinline__ uint32_t smem_fetch_add(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;\n"
               : "=r"(old)
               : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v)
               : "memory");
  return old;
}

// exclusive block-wide scan (all threads must call); sh >= 32 words
__device__ __forceinline__ uint32_t block_excl_scan_u32(uint32_t v, uint32_t* sh, uint32_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t s = lane < nw ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) sh[lane] = s;
  }
  __syncthreads();
  const uint32_t wbase = w ? sh[w - 1] : 0;
  if (total) *total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return wbase + x - v;
}


// ------------------------------------------------------------ misc helpers
__device__ __forceinline__ uint64_t desc_score_key(float s, uint32_t id) {
  return ((uint64_t)(~ord_key(s)) << 32) | id;  // ascending = (score desc, id asc)
}
__device__ __forceinline__ float desc_score_val(uint64_t k) {
  return ord_inv(~(uint32_t)(k >> 32));
}

// exact keep count, SPEC.md:257 / SURVEY 8(c): min(B, max(kappa, floor(double(alpha)*B/iP)))
__device__ __host__ __forceinline__ uint32_t keep_count(uint32_t B, float alpha, uint32_t ip,
                                                        uint32_t kappa) {
  const double f = floor((double)alpha * (double)B / (double)ip);
  uint64_t k = (uint64_t)f;
  if (k < kappa) k = kappa;
  if (k > B) k = B;
  return (uint32_t)k;
}

}  // namespace fpp
