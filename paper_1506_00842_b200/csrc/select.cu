// select.cu — the final stage of the guard-band top-m (reference: the
// global lexsort of tuner.py:128-131).
//
//   k_band_filter  one CTA: the exact m-th smallest fp32 mean log tau_m over all
//                  candidates (radix select), then keep f32 <= tau_m + 2*delta.
//                  Every configuration of the true top-m passes.
//   k_rescore      (predict.cu) fp64 prediction of the survivors, one CTA each.
//   k_sort_small   one CTA: bitonic sort of <= kSmallSort (prediction, index)
//                  pairs in shared memory and the first m written out; larger
//                  survivor sets are sorted by the caller with CUB.
#include "kernels.cuh"

namespace mlt {

__global__ void __launch_bounds__(1024) k_band_filter(const int64_t* __restrict__ cidx, const float* __restrict__ cval,
                                                      const uint32_t* __restrict__ count_ptr, uint32_t cap, int m,
                                                      float band, int64_t* __restrict__ out_idx,
                                                      float* __restrict__ out_val, uint32_t* __restrict__ out_n) {
  __shared__ uint32_t s_hist[256], s_sel[2], s_n;
  const int tid = threadIdx.x;
  const uint32_t count = *count_ptr;   // written by the sweep (stream order)
  if (count > cap) {                   // the buffer overflowed: the caller takes the exact path
    if (tid == 0) *out_n = 0;
    return;
  }
  float theta = __int_as_float(0x7f800000);   // +inf: keep everything when count < m
  if (count >= (uint32_t)m) {
    const uint32_t key = block_select(
        [&](auto&& f) {
          for (uint32_t e = tid; e < count; e += blockDim.x) f(fkey(cval[e]));
        },
        m, s_hist, s_sel);
    theta = __fadd_ru(fkey_inv(key), band);
  }
  if (tid == 0) s_n = 0;
  __syncthreads();
  for (uint32_t e = tid; e < count; e += blockDim.x) {
    const float v = cval[e];
    if (!(v > theta)) {
      const uint32_t slot = atomicAdd(&s_n, 1u);
      out_idx[slot] = cidx[e];
      out_val[slot] = v;
    }
  }
  __syncthreads();
  if (tid == 0) *out_n = s_n;
}

__global__ void __launch_bounds__(1024) k_sort_small(const double* __restrict__ pred, const int64_t* __restrict__ idx,
                                                     const uint32_t* __restrict__ n_ptr, int m,
                                                     double* __restrict__ out_pred, int64_t* __restrict__ out_idx,
                                                     uint32_t* __restrict__ status) {
  extern __shared__ unsigned long long sk[];     // [N] prediction bits, then [N] indices
  const uint32_t n = *n_ptr;
  const int tid = threadIdx.x;
  if (n > (uint32_t)kSmallSort) {
    if (tid == 0) status[0] = 1;                 // caller sorts with CUB
    for (int e = tid; e < m; e += blockDim.x) {  // defined padding (the host copies the
      out_pred[e] = __longlong_as_double(0x7ff0000000000000ll);   // lists unconditionally)
      out_idx[e] = INT64_MAX;
    }
    return;
  }
  unsigned long long* key = sk;
  long long* ix = reinterpret_cast<long long*>(sk + kSmallSort);
  if (n <= (uint32_t)kRankSort) {
    // Rank sort: (prediction, index) pairs are distinct (indices are), so the
    // rank of an entry -- how many entries precede it -- is its position. One
    // pass of broadcast shared-memory reads, two barriers (a bitonic network
    // over n = 256 takes 36 barrier-separated passes).
    for (uint32_t e = tid; e < n; e += blockDim.x) {
      key[e] = (unsigned long long)__double_as_longlong(pred[e]);
      ix[e] = idx[e];
    }
    __syncthreads();
    const uint32_t take = min((uint32_t)m, n);
    for (uint32_t e0 = 0; e0 < n; e0 += blockDim.x) {
      const uint32_t e = e0 + tid;
      if (e0 + (tid & ~31u) >= n) break;   // whole warp past the end: skip the O(n) scan
      const unsigned long long ke = e < n ? key[e] : 0ull;
      const long long ie = e < n ? ix[e] : 0ll;
      uint32_t rank = 0;
#pragma unroll 8
      for (uint32_t u = 0; u < n; ++u) {
        const unsigned long long ku = key[u];
        rank += (ku < ke || (ku == ke && ix[u] < ie)) ? 1u : 0u;
      }
      if (e < n && rank < take) {
        out_pred[rank] = __longlong_as_double((long long)ke);
        out_idx[rank] = ie;
      }
    }
    for (uint32_t e = take + tid; e < (uint32_t)m; e += blockDim.x) {   // padded past `take`
      out_pred[e] = __longlong_as_double(0x7ff0000000000000ll);
      out_idx[e] = INT64_MAX;
    }
    if (tid == 0) {
      status[0] = 0;
      status[1] = take;
    }
    return;
  }
  uint32_t N = 1;
  while (N < n) N <<= 1;
  for (uint32_t e = tid; e < N; e += blockDim.x) {
    key[e] = e < n ? (unsigned long long)__double_as_longlong(pred[e]) : 0x7ff0000000000000ull;
    ix[e] = e < n ? idx[e] : INT64_MAX;
  }
  __syncthreads();
  // predictions are positive doubles: their bit patterns order like the values
  for (uint32_t k = 2; k <= N; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t e = tid; e < N; e += blockDim.x) {
        const uint32_t p = e ^ j;
        if (p > e) {
          const bool up = (e & k) == 0;
          const bool gt = key[e] > key[p] || (key[e] == key[p] && ix[e] > ix[p]);
          if (gt == up) {
            const unsigned long long tk = key[e];
            key[e] = key[p];
            key[p] = tk;
            const long long ti = ix[e];
            ix[e] = ix[p];
            ix[p] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
  const uint32_t take = min((uint32_t)m, n);
  for (uint32_t e = tid; e < (uint32_t)m; e += blockDim.x) {   // padded past `take`
    out_pred[e] = e < take ? __longlong_as_double((long long)key[e]) : __longlong_as_double(0x7ff0000000000000ll);
    out_idx[e] = e < take ? ix[e] : INT64_MAX;
  }
  if (tid == 0) {
    status[0] = 0;
    status[1] = take;
  }
}

}  // namespace mlt
