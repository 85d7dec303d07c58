// host_rng.cu — the per-epoch permutations of model._fit (reference
// model.py:218, `rng.permutation(n)` once per epoch) produced natively, many
// generators at a time on host threads.
//
// Bit-identical to numpy by construction: the random bits come from numpy's
// OWN bit generator through its C interface (`Generator.bit_generator.ctypes
// .bit_generator`, numpy/random/bitgen.h), and the shuffle is numpy's
// Generator.shuffle on arange(n) — Fisher-Yates from the last element down to
// index 1 with j = random_interval(i) (mask rejection on 32-bit draws for
// bounds < 2^32). tests/test_host.py checks every output against numpy.
#include <cstdint>
#include <thread>
#include <vector>

#include "mltune_b200.h"

namespace {

// numpy/random/bitgen.h
struct bitgen_t {
  void* state;
  uint64_t (*next_uint64)(void* st);
  uint32_t (*next_uint32)(void* st);
  double (*next_double)(void* st);
  uint64_t (*next_raw)(void* st);
};

inline uint64_t random_interval(bitgen_t* g, uint64_t max) {
  if (max == 0) return 0;
  uint64_t mask = max;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  uint64_t v;
  if (max <= 0xffffffffull) {
    while ((v = (g->next_uint32(g->state) & mask)) > max) {
    }
  } else {
    while ((v = (g->next_uint64(g->state) & mask)) > max) {
    }
  }
  return v;
}

void permutations_one(bitgen_t* g, int32_t n, int32_t count, int32_t* out) {
  for (int32_t c = 0; c < count; ++c) {
    int32_t* a = out + (size_t)c * n;
    for (int32_t i = 0; i < n; ++i) a[i] = i;
    for (int64_t i = (int64_t)n - 1; i >= 1; --i) {
      const int64_t j = (int64_t)random_interval(g, (uint64_t)i);
      const int32_t t = a[i];
      a[i] = a[j];
      a[j] = t;
    }
  }
}

}  // namespace

extern "C" {

MLT_API int mlt_host_permutations(void* const* bitgens, int32_t n_gen, const int32_t* n, int32_t count,
                                  int32_t* out, int32_t threads) {
  if (n_gen < 0 || count < 0 || (n_gen > 0 && (!bitgens || !n || !out))) return MLT_EINVAL;
  std::vector<size_t> off(n_gen + 1, 0);
  for (int32_t g = 0; g < n_gen; ++g) {
    if (n[g] < 0 || !bitgens[g]) return MLT_EINVAL;
    off[g + 1] = off[g] + (size_t)count * n[g];
  }
  int nt = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (nt > n_gen) nt = n_gen;
  auto work = [&](int t) {
    for (int32_t g = t; g < n_gen; g += nt)
      permutations_one(static_cast<bitgen_t*>(bitgens[g]), n[g], count, out + off[g]);
  };
  if (nt <= 1) {
    if (n_gen > 0) work(0);
    return MLT_OK;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(work, t);
  for (auto& th : pool) th.join();
  return MLT_OK;
}

}  // extern "C"
