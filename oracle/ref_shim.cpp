// ref_shim.cpp -- extern "C" wrapper over the UNMODIFIED reference sources
// (/root/reference/proj/src/rotation.cpp, dataset.cpp, include/lsfann/common.hpp),
// compiled together by oracle/Makefile into oracle/_ref/libfpp_ref.so.
// TEST INFRASTRUCTURE ONLY: pins the oracle restatement (tests/test_oracle_pins.py).
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <vector>

#include "lsfann/common.hpp"
#include "lsfann/dataset.hpp"
#include "lsfann/rotation.hpp"

extern "C" {

uint64_t ref_mix64(uint64_t z) { return lsfann::mix64(z); }
uint64_t ref_derive_seed(uint64_t m, uint64_t a, uint64_t b, uint64_t c) {
  return lsfann::derive_seed(m, a, b, c);
}
uint64_t ref_fnv1a64(const void* p, uint64_t len, uint64_t h) { return lsfann::fnv1a64(p, len, h); }

int ref_fht(float* v, uint64_t n) {
  try {
    lsfann::fht(std::span<float>(v, n));
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

// rows x[n][d] projected with SpinnerStack(d, D, seed) -> out[n][D]
int ref_project(uint32_t d, uint32_t D, uint64_t seed, const float* x, uint64_t n, float* out) {
  try {
    lsfann::SpinnerStack st(d, D, seed);
    std::vector<float> scratch(st.padded_dim());
    for (uint64_t i = 0; i < n; ++i)
      st.project(std::span<const float>(x + i * d, d), std::span<float>(out + i * D, D), scratch);
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

// normalize(Dataset) in place; returns -1 ok, else -2 on error
int64_t ref_normalize(float* X, uint64_t n, uint32_t d) {
  try {
    lsfann::Dataset ds(std::vector<float>(X, X + n * d), d);
    lsfann::Dataset out = lsfann::normalize(ds);
    std::memcpy(X, out.raw().data(), n * d * sizeof(float));
    return -1;
  } catch (const std::invalid_argument&) {
    return -2;
  }
}

// center(Dataset) in place, center vector out; returns -1 ok, -2 on error
int64_t ref_center(float* X, uint64_t n, uint32_t d, float* center_out) {
  try {
    lsfann::Dataset ds(std::vector<float>(X, X + n * d), d);
    lsfann::Dataset out = lsfann::center(ds);
    std::memcpy(X, out.raw().data(), n * d * sizeof(float));
    std::memcpy(center_out, out.center().data(), d * sizeof(float));
    return -1;
  } catch (const std::invalid_argument&) {
    return -2;
  }
}

double ref_inner_product(const float* a, const float* b, uint32_t d) {
  return lsfann::inner_product(std::span<const float>(a, d), std::span<const float>(b, d));
}
}
