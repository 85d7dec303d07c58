// select.cuh — block-wide selection helpers shared by the sweep and the
// final top-m stage.
#pragma once

#include "common.cuh"

namespace mlt {

// ---------------------------------------------------------------------------
// block-wide radix select: the exact m-th smallest ordered key (1-based)
// among keys visited by `visit` (each thread visits its own keys).
// ---------------------------------------------------------------------------
template <typename V>
__device__ __forceinline__ uint32_t block_select(V visit, int m, uint32_t* s_hist, uint32_t* s_sel) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t prefix = 0;
  uint32_t want = (uint32_t)m;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int b = tid; b < 256; b += blockDim.x) s_hist[b] = 0u;
    __syncthreads();
    visit([&](uint32_t key) {
      if (pass == 0 || (key >> (shift + 8)) == prefix) {
        const uint32_t bin = (key >> shift) & 255u;
        const uint32_t peers = __match_any_sync(__activemask(), bin);
        if (lane == __ffs(peers) - 1) atomicAdd(&s_hist[bin], (uint32_t)__popc(peers));
      }
    });
    __syncthreads();
    if (warp == 0) {
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        c[b] = s_hist[lane * 8 + b];
        tot += c[b];
      }
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const uint32_t excl = incl - tot;
      if (excl < want && want <= incl) {
        uint32_t run = excl;
        int bin = lane * 8 + 7;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          if (run + c[b] >= want) {
            bin = lane * 8 + b;
            break;
          }
          run += c[b];
        }
        s_sel[0] = (prefix << 8) | (uint32_t)bin;
        s_sel[1] = want - run;
      }
    }
    __syncthreads();
    prefix = s_sel[0];
    want = s_sel[1];
  }
  return prefix;
}

}  // namespace mlt
