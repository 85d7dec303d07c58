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
                                                     uint32_t* __restrict__ status, int cap,
                                                     uint32_t* __restrict__ host_out, const uint32_t* __restrict__ gs,
                                                     int64_t* __restrict__ rec, uint32_t cand_cap) {
  // cap: entries the launch's dynamic shared memory holds (a power of two <=
  // kSmallSort, chosen by the host from m): a small launch keeps the SM's
  // shared-memory carveout of the kernels around it (a 128 KB request forces
  // a reconfiguration: 15 -> 3 us for m = 200)
  // host_out (optional): pinned host memory the kernel writes the step's
  // result into directly -- a 16-word header (gs[0..1] sweep threshold and
  // candidate count, n, status, take, gs[8..9] pruning work) then m
  // predictions and m indices -- so the host needs no copy after its one wait.
  extern __shared__ unsigned long long sk[];     // [cap] prediction bits, then [cap] indices
  const uint32_t n = *n_ptr;
  const int tid = threadIdx.x;
  // rec (optional): the sharded step's device record (mlt_plan_top_m_record):
  // m indices (-1 pads), m prediction bit patterns (+inf pads), status word
  // (1 = the sweep's candidate buffer overflowed, 2 = too many survivors for
  // this kernel; the caller's protocol redoes such a shard)
  auto mirror = [&](uint32_t big, uint32_t take) {
    if (rec) {
      __syncthreads();
      const uint32_t count = gs[1];
      const long long st = count > cand_cap ? 1 : (big ? 2 : 0);
      const int tk = st ? 0 : (int)min(take, (uint32_t)m);
      for (int t = tid; t < m; t += blockDim.x) {
        const bool ok = t < tk && out_idx[t] != INT64_MAX && out_idx[t] >= 0;
        rec[t] = ok ? out_idx[t] : -1;
        rec[m + t] = ok ? __double_as_longlong(out_pred[t]) : 0x7ff0000000000000ll;
      }
      if (tid == 0) rec[2 * m] = st;
    }
    if (!host_out) return;
    __syncthreads();   // out_pred / out_idx complete
    double* hp = reinterpret_cast<double*>(host_out + 16);
    long long* hi = reinterpret_cast<long long*>(hp + m);
    for (int e = tid; e < m; e += blockDim.x) {
      hp[e] = out_pred[e];
      hi[e] = out_idx[e];
    }
    if (tid == 0) {
      host_out[0] = gs[0];
      host_out[1] = gs[1];
      host_out[2] = n;
      host_out[3] = big;
      host_out[4] = take;
      host_out[8] = gs[8];
      host_out[9] = gs[9];
    }
  };
  if (n > (uint32_t)cap) {
    if (tid == 0) status[0] = 1;                 // caller sorts with CUB
    for (int e = tid; e < m; e += blockDim.x) {  // defined padding (the host copies the
      out_pred[e] = __longlong_as_double(0x7ff0000000000000ll);   // lists unconditionally)
      out_idx[e] = INT64_MAX;
    }
    mirror(1u, 0u);
    return;
  }
  unsigned long long* key = sk;
  long long* ix = reinterpret_cast<long long*>(sk + cap);
  if (n <= (uint32_t)kRankSort) {
    // Rank sort: (prediction, index) pairs are distinct (indices are), so the
    // rank of an entry -- how many entries precede it -- is its position.
    // Entries are stored as {key, index} so one broadcast LDS.128 reads one;
    // four threads per entry each count a quarter of the entries, branch-free,
    // and add into the entry's rank (a bitonic network over n = 256 takes 36
    // barrier-separated passes; the first, one-thread-per-entry version with a
    // short-circuit compare was latency-bound at ~30 us for n = 200).
    static_assert(1024 % kRankSort == 0, "segments per entry");
    constexpr uint32_t S = 1024 / kRankSort;
    __shared__ uint32_t s_rank[kRankSort];
    ulonglong2* kv = reinterpret_cast<ulonglong2*>(sk);
    for (uint32_t e = tid; e < n; e += blockDim.x) {
      kv[e] = make_ulonglong2((unsigned long long)__double_as_longlong(pred[e]), (unsigned long long)idx[e]);
      s_rank[e] = 0;
    }
    __syncthreads();
    const uint32_t take = min((uint32_t)m, n);
    {
      const uint32_t e = tid % kRankSort, sg = tid / kRankSort;
      if (e < n) {
        const ulonglong2 me = kv[e];
        const uint32_t u0 = sg * n / S, u1 = (sg + 1) * n / S;
        uint32_t r = 0;
#pragma unroll 4
        for (uint32_t u = u0; u < u1; ++u) {
          const ulonglong2 o = kv[u];
          r += (uint32_t)(o.x < me.x) | ((uint32_t)(o.x == me.x) & (uint32_t)((long long)o.y < (long long)me.y));
        }
        atomicAdd(&s_rank[e], r);
      }
    }
    __syncthreads();
    for (uint32_t e = tid; e < n; e += blockDim.x) {
      const uint32_t rank = s_rank[e];
      if (rank < take) {
        const ulonglong2 me = kv[e];
        out_pred[rank] = __longlong_as_double((long long)me.x);
        out_idx[rank] = (long long)me.y;
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
    mirror(0u, take);
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
  mirror(0u, take);
}

}  // namespace mlt
