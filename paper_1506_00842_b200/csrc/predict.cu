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

// Static validity of the contiguous range [lo, lo + n) (for the order-preserving
// selection of the first valid indices).
__global__ void k_valid_range(DSpace s, int64_t lo, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int dig[kMaxP];
    decode_digits(s, (uint64_t)(lo + t), dig);
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
                            int64_t* __restrict__ idx_out, const float* __restrict__ band_v, float band_theta,
                            int staged) {
  // staged: the weights fit the launch's shared memory; otherwise (very wide
  // ensembles) they are read from the packed global block through L1
  extern __shared__ double sm_dyn[];
  if (staged) {
    stage_weights(e, sm_dyn);
    __syncthreads();
  }
  const double* sm = staged ? sm_dyn : e.w1;   // [W1 | b1 | w2 | b2 | mean | std], the same layout
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
__global__ void k_member_out64(DEns e, const double* __restrict__ feat, int64_t n, double* __restrict__ out,
                               int staged) {
  extern __shared__ double sm_dyn[];
  if (staged) {
    stage_weights(e, sm_dyn);
    __syncthreads();
  }
  const double* sm = staged ? sm_dyn : e.w1;
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

// Guard-band rescoring (fp64, the reference's per-member arithmetic): one CTA
// per survivor. The CTA decodes the configuration once (a thread per
// parameter), evaluates all k*h hidden units in parallel (a unit per thread:
// z = x.W1 + b1, w2 * sigmoid(z)), sums each member's units, de-standardises
// (out*std + mean) and adds the members in member order, /k, exp -- the
// k_predict64 sequence; only the order of the h-term sums differs (as it
// does between any two BLAS dgemv builds). Survivors are few (~m), so the
// latency of one survivor is what counts: its dependent chain here is one
// unit plus two short reductions, not k units in a row.
__global__ void __launch_bounds__(256) k_rescore(DEns e, const int64_t* __restrict__ idx,
                                                 const uint32_t* __restrict__ n_ptr, double* __restrict__ pred) {
  extern __shared__ double s_dyn[];   // [k*h] unit terms, [k] member logs
  __shared__ double s_x[kMaxP];
  double* s_term = s_dyn;
  double* s_lg = s_dyn + (size_t)e.k * e.h;
  const uint32_t n = *n_ptr;
  const int tid = threadIdx.x;
  const int nh = e.k * e.h;
  for (uint32_t t = blockIdx.x; t < n; t += gridDim.x) {
    if (tid < e.d) {   // digit of parameter tid: (idx / stride) % count, last parameter fastest
      uint64_t stride = 1;
      for (int q = e.d - 1; q > tid; --q) stride *= (uint64_t)e.counts[q];
      const uint64_t id = (uint64_t)idx[t];
      const uint64_t c = (uint64_t)e.counts[tid];
      const uint64_t dig = ((id | stride) <= 0xffffffffull ? (uint64_t)((uint32_t)id / (uint32_t)stride) : id / stride) % c;
      s_x[tid] = (double)dig / (double)(c > 1 ? c - 1 : 1);
    }
    __syncthreads();
    for (int u = tid; u < nh; u += blockDim.x) {
      const double* w = e.w1 + (size_t)u * e.d;
      double z = 0.0;
#pragma unroll
      for (int p = 0; p < kMaxP; ++p)
        if (p < e.d) z = fma(s_x[p], __ldg(w + p), z);
      z = __dadd_rn(z, __ldg(e.b1 + u));
      s_term[u] = fma(1.0 / (1.0 + exp(-z)), __ldg(e.w2 + u), 0.0);
    }
    __syncthreads();
    for (int mm = tid; mm < e.k; mm += blockDim.x) {
      double out = 0.0;
      for (int j = 0; j < e.h; ++j) out = __dadd_rn(out, s_term[mm * e.h + j]);
      out = __dadd_rn(out, __ldg(e.b2 + mm));
      s_lg[mm] = __dadd_rn(__dmul_rn(out, __ldg(e.std_ + mm)), __ldg(e.mean + mm));
    }
    __syncthreads();
    if (tid == 0) {
      double acc = s_lg[0];
      for (int m = 1; m < e.k; ++m) acc = __dadd_rn(acc, s_lg[m]);
      pred[t] = exp(__ddiv_rn(acc, (double)e.k));
    }
    __syncthreads();   // s_x / s_term are rewritten for the next survivor
  }
}

}  // namespace mlt
