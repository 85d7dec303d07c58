// predict.cu — exact (fp64) device kernels:
//   k_decode / k_valid / k_encode      A1-A3  (paramspace.py:184-213, model.py:88-97)
//   k_predict64                        A4-A6  (model.py:146-170, :290-301)
// k_predict64 is also the guard-band rescorer of the fp32 sweep and the
// materialising path of top_m; it evaluates each configuration in the
// reference's operation order (dot + b1, 1/(1+exp(-z)), h.w2 + b2,
// out*std + mean with two roundings, member sum in member order, /k, exp).
#include "kernels.cuh"

namespace mlt {

__global__ void k_decode(DSpace s, const int64_t* __restrict__ idx, int64_t n, int64_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int dig[kMaxP];
    decode_digits(s, (uint64_t)idx[t], dig);
    for (int p = 0; p < s.P; ++p) out[t * s.P + p] = value_of(s, p, dig[p]);
  }
}

__global__ void k_valid(DSpace s, const int64_t* __restrict__ idx, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int dig[kMaxP];
    decode_digits(s, (uint64_t)idx[t], dig);
    out[t] = rules_ok(s, dig) ? 1 : 0;
  }
}

// feature = digit / max(count - 1, 1); IEEE division matches numpy bit-for-bit.
__global__ void k_encode(DEns e, const int64_t* __restrict__ idx, int64_t n, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t r = (uint64_t)idx[t];
    for (int p = e.d - 1; p >= 0; --p) {
      const uint64_t c = (uint64_t)e.counts[p];
      const uint64_t q = r / c;
      const int dig = (int)(r - q * c);
      r = q;
      out[t * e.d + p] = (double)dig / (double)(e.counts[p] > 1 ? e.counts[p] - 1 : 1);
    }
  }
}

// Stage the fp64 weights in shared memory: [W1 | b1 | w2 | b2 | mean | std].
__device__ __forceinline__ void stage_weights(const DEns& e, double* sm) {
  const int nw = e.k * e.h * e.d, nh = e.k * e.h;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) sm[i] = e.w1[i];
  for (int i = threadIdx.x; i < nh; i += blockDim.x) {
    sm[nw + i] = e.b1[i];
    sm[nw + nh + i] = e.w2[i];
  }
  for (int i = threadIdx.x; i < e.k; i += blockDim.x) {
    sm[nw + 2 * nh + i] = e.b2[i];
    sm[nw + 2 * nh + e.k + i] = e.mean[i];
    sm[nw + 2 * nh + 2 * e.k + i] = e.std_[i];
  }
}

// Mean over members of the de-standardized log time for one feature vector.
__device__ __forceinline__ double mean_log64(const DEns& e, const double* sm, const double (&x)[kMaxP]) {
  const int nw = e.k * e.h * e.d, nh = e.k * e.h;
  const double* W1 = sm;
  const double* B1 = sm + nw;
  const double* W2 = sm + nw + nh;
  const double* B2 = sm + nw + 2 * nh;
  const double* MU = B2 + e.k;
  const double* SD = MU + e.k;
  double acc = 0.0;
  for (int m = 0; m < e.k; ++m) {
    double out = 0.0;
    for (int j = 0; j < e.h; ++j) {
      const double* w = W1 + (m * e.h + j) * e.d;
      double z = 0.0;
#pragma unroll
      for (int p = 0; p < kMaxP; ++p)
        if (p < e.d) z = fma(x[p], w[p], z);
      z = __dadd_rn(z, B1[m * e.h + j]);
      const double hj = 1.0 / (1.0 + exp(-z));      // overflow saturates to 0 (model.py:167-170)
      out = fma(hj, W2[m * e.h + j], out);
    }
    out = __dadd_rn(out, B2[m]);
    const double lg = __dadd_rn(__dmul_rn(out, SD[m]), MU[m]);
    acc = (m == 0) ? lg : __dadd_rn(acc, lg);
  }
  return __ddiv_rn(acc, (double)e.k);
}

// Source of configurations: a contiguous range, an index list, or a feature matrix.
// Output: pred[t] = exp(mean log) (or +inf for statically invalid entries when
// `s_check` is set), and optionally the key bits of pred for sorting.
__global__ void k_predict64(DEns e, DSpace s, int check_rules, int64_t begin, const int64_t* __restrict__ idx,
                            const double* __restrict__ feat, int64_t n, double* __restrict__ pred,
                            int64_t* __restrict__ idx_out, const float* __restrict__ band_v, float band_theta) {
  extern __shared__ double sm[];
  stage_weights(e, sm);
  __syncthreads();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double x[kMaxP];
    bool ok = true;
    int64_t id = -1;
    if (feat) {
#pragma unroll
      for (int p = 0; p < kMaxP; ++p) x[p] = (p < e.d) ? feat[t * e.d + p] : 0.0;
    } else {
      id = idx ? idx[t] : begin + t;
      if (band_v && !(band_v[t] <= band_theta)) ok = false;   // outside the final guard band
      uint64_t r = (uint64_t)id;
      int dig[kMaxP];
#pragma unroll
      for (int p = kMaxP - 1; p >= 0; --p) {
        if (p < e.d) {
          const uint64_t c = (uint64_t)e.counts[p];
          const uint64_t q = r / c;
          dig[p] = (int)(r - q * c);
          r = q;
          x[p] = (double)dig[p] / (double)(e.counts[p] > 1 ? e.counts[p] - 1 : 1);
        } else {
          dig[p] = 0;
          x[p] = 0.0;
        }
      }
      if (ok && check_rules && s.R > 0) ok = rules_ok(s, dig);
    }
    double v = __longlong_as_double(0x7ff0000000000000ll);   // +inf: sorts last
    if (ok) v = exp(mean_log64(e, sm, x));
    pred[t] = v;
    if (idx_out) idx_out[t] = ok ? id : INT64_MAX;
  }
}

// Raw output of every member (Network.forward_batch): out[m][t].
__global__ void k_member_out64(DEns e, const double* __restrict__ feat, int64_t n, double* __restrict__ out) {
  extern __shared__ double sm[];
  stage_weights(e, sm);
  __syncthreads();
  const int nw = e.k * e.h * e.d, nh = e.k * e.h;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double x[kMaxP];
#pragma unroll
    for (int p = 0; p < kMaxP; ++p) x[p] = (p < e.d) ? feat[t * e.d + p] : 0.0;
    for (int m = 0; m < e.k; ++m) {
      double o = 0.0;
      for (int j = 0; j < e.h; ++j) {
        const double* w = sm + (m * e.h + j) * e.d;
        double z = 0.0;
#pragma unroll
        for (int p = 0; p < kMaxP; ++p)
          if (p < e.d) z = fma(x[p], w[p], z);
        z = __dadd_rn(z, sm[nw + m * e.h + j]);
        o = fma(1.0 / (1.0 + exp(-z)), sm[nw + nh + m * e.h + j], o);
      }
      out[(int64_t)m * n + t] = __dadd_rn(o, sm[nw + 2 * nh + m]);
    }
  }
}

size_t predict64_smem(const DEns& e) {
  return sizeof(double) * ((size_t)e.k * e.h * e.d + 2 * (size_t)e.k * e.h + 3 * (size_t)e.k);
}

}  // namespace mlt

namespace mlt {

// Guard-band rescoring: one warp per candidate; lane j evaluates hidden unit j
// of every member, each member output is a warp reduction. The per-unit and
// per-member rounding sequence is k_predict64's (out*std + mean, member
// order, /k, exp). The members' chains are independent: they run kRU at a
// time (the exp / divide latencies overlap), weights straight from L2 (a
// survivor reads its 53 KB once; no per-CTA staging of the whole ensemble).
__global__ void __launch_bounds__(256) k_rescore_warp(DEns e, const int64_t* __restrict__ idx,
                                                      const uint32_t* __restrict__ n_ptr, double* __restrict__ pred) {
  constexpr int kRU = 4;
  const uint32_t n = *n_ptr;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (uint32_t t = blockIdx.x * wpb + (threadIdx.x >> 5); t < n; t += gridDim.x * wpb) {
    uint64_t r = (uint64_t)idx[t];
    double x[kMaxP];
#pragma unroll
    for (int p = kMaxP - 1; p >= 0; --p) {
      if (p < e.d) {
        const uint32_t c = (uint32_t)e.counts[p];
        uint64_t q;
        if (r <= 0xffffffffull) {   // 32-bit division (the 64-bit one is a ~60-instruction call)
          q = (uint32_t)r / c;
        } else {
          q = r / c;
        }
        x[p] = (double)(r - q * c) / (double)(c > 1 ? c - 1 : 1);
        r = q;
      } else {
        x[p] = 0.0;
      }
    }
    double acc = 0.0;
    for (int m0 = 0; m0 < e.k; m0 += kRU) {
      double part[kRU];
#pragma unroll
      for (int u = 0; u < kRU; ++u) {
        part[u] = 0.0;
        const int m = m0 + u;
        if (m < e.k) {
          for (int j = lane; j < e.h; j += 32) {
            const double* w = e.w1 + ((size_t)m * e.h + j) * e.d;
            double z = 0.0;
#pragma unroll
            for (int p = 0; p < kMaxP; ++p)
              if (p < e.d) z = fma(x[p], __ldg(w + p), z);
            z = __dadd_rn(z, __ldg(e.b1 + m * e.h + j));
            part[u] = fma(1.0 / (1.0 + exp(-z)), __ldg(e.w2 + m * e.h + j), part[u]);
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < kRU; ++u) part[u] += __shfl_xor_sync(0xffffffffu, part[u], o);
#pragma unroll
      for (int u = 0; u < kRU; ++u) {
        const int m = m0 + u;
        if (m < e.k) {
          const double out = __dadd_rn(part[u], __ldg(e.b2 + m));
          const double lg = __dadd_rn(__dmul_rn(out, __ldg(e.std_ + m)), __ldg(e.mean + m));
          acc = (m == 0) ? lg : __dadd_rn(acc, lg);
        }
      }
    }
    if (lane == 0) pred[t] = exp(__ddiv_rn(acc, (double)e.k));
  }
}

}  // namespace mlt
