// common.cuh — shared device-side types and helpers for libmltune_b200.
//
// Layouts (all device-resident, built once per call or per plan):
//   DSpace   : radices + value LUT + rules of a parameter space (mlt_space)
//   DEns     : fp64 ensemble weights packed [W1 | b1 | w2 | b2 | mean | std]
// Reference semantics cited per helper (paths under /root/reference/pkg/src/mltune).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "mltune_b200.h"

namespace mlt {

constexpr int kMaxP = MLT_MAX_PARAMS;
constexpr int kMaxRules = 64;
constexpr int kMaxOps = 256;
constexpr int kH = 30;          // padded hidden units per member in the fp32 sweep

// Parameter space, passed BY VALUE as a kernel argument (~2.9 KB).
struct DSpace {
  int P;
  int R;
  int radix[kMaxP];
  int voff[kMaxP];              // offset of parameter p's value list in `values`
  const int64_t* values;        // device
  // rules (kind, operand range) — operands in rpos/rcoeff (device)
  int rkind[kMaxRules];
  int roff[kMaxRules + 1];
  int64_t rbound[kMaxRules];
  const int* rpos;              // device
  const int64_t* rcoeff;        // device
};

// fp64 ensemble weights in device memory.
struct DEns {
  int k, d, h;
  int counts[kMaxP];
  const double* w1;             // [k][h][d]
  const double* b1;             // [k][h]
  const double* w2;             // [k][h]
  const double* b2;             // [k]
  const double* mean;           // [k]
  const double* std_;           // [k]
};

// Mixed-radix digits, last parameter fastest (paramspace.py:149-158).
__device__ __forceinline__ void decode_digits(const DSpace& s, uint64_t idx, int* dig) {
  if (idx <= 0xffffffffull) {
    uint32_t r = (uint32_t)idx;
    for (int p = s.P - 1; p >= 0; --p) {
      uint32_t q = r / (uint32_t)s.radix[p];
      dig[p] = (int)(r - q * (uint32_t)s.radix[p]);
      r = q;
    }
  } else {
    for (int p = s.P - 1; p >= 0; --p) {
      uint64_t q = idx / (uint64_t)s.radix[p];
      dig[p] = (int)(idx - q * (uint64_t)s.radix[p]);
      idx = q;
    }
  }
}

__device__ __forceinline__ int64_t value_of(const DSpace& s, int p, int digit) {
  return s.values[s.voff[p] + digit];
}

// Every static rule satisfied? numpy int64 semantics: products and sums wrap
// modulo 2^64, comparisons are signed (paramspace.py:92-107, :205-213).
__device__ __forceinline__ bool rules_ok(const DSpace& s, const int* dig) {
  for (int r = 0; r < s.R; ++r) {
    const int a = s.roff[r], b = s.roff[r + 1];
    const int kind = s.rkind[r];
    if (kind == MLT_RULE_FORBIDDEN) {
      bool hit = true;
      for (int o = a; o < b; ++o) {
        const int p = s.rpos[o];
        hit = hit && (value_of(s, p, dig[p]) == s.rcoeff[o]);
      }
      if (hit) return false;
    } else {
      uint64_t acc = (kind == MLT_RULE_MAX_PRODUCT) ? 1ull : 0ull;
      for (int o = a; o < b; ++o) {
        const int p = s.rpos[o];
        const uint64_t term = (uint64_t)s.rcoeff[o] * (uint64_t)value_of(s, p, dig[p]);
        acc = (kind == MLT_RULE_MAX_PRODUCT) ? acc * term : acc + term;
      }
      if (!((int64_t)acc <= s.rbound[r])) return false;
    }
  }
  return true;
}

// Order-preserving float <-> uint32 key (for atomicMin thresholds, radix select).
__device__ __forceinline__ uint32_t fkey(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(b);
}

}  // namespace mlt
