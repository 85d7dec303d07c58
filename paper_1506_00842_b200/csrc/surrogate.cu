// surrogate.cu — the analytic surrogate device on the B200 (SURVEY §8(a) A12,
// §8(f) next #2): SurrogateRunner.true_times / measured_times
// (measurement.py:212-238) with the splitmix64 noise of unit_normals
// (measurement.py:125-142), plus the fused exhaustive search over an index
// range (tuner.py:191-224) that the reference can only do chunk by chunk.
//
// Per configuration: t = base_time, then for each term in spec order
// t *= factor when every named parameter takes the matched value (the
// product order of the reference, so noise-free times are bit-identical);
// launch rules -> NaN / not ok. With noise, z = min over repetitions of
// ndtri(u(h)) with u = ((h >> 11) + 0.5) * 2^-53 and t *= exp(sigma * z).
// The hash and u are integer/IEEE-exact; ndtri is CUDA's normcdfinv and exp
// CUDA's exp (a few ulp from scipy's cephes ndtri and glibc's exp), so noisy
// times agree to ~1e-15 relative.
#include "kernels.cuh"

namespace mlt {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

// measurement.py:135-142
__device__ __forceinline__ double unit_normal(uint64_t seed, uint64_t idx, int rep) {
  const uint64_t G = 0x9E3779B97F4A7C15ull;
  uint64_t h = mix64(seed + G * (idx + 1));
  h = mix64(h + G * (uint64_t)(((uint64_t)rep + 1) & 0xffffffffull));
  const double u = __dmul_rn(__dadd_rn((double)(h >> 11), 0.5), 0x1p-53);
  return normcdfinv(u);
}

// Stage the term table in shared memory (all threads read it uniformly).
__device__ __forceinline__ void stage_terms(const DSurr& su, int* s_pos, int* s_dig, double* s_fac) {
  for (int t = threadIdx.x; t < su.T; t += blockDim.x) {
    s_pos[2 * t] = su.tpos[2 * t];
    s_pos[2 * t + 1] = su.tpos[2 * t + 1];
    s_dig[2 * t] = su.tdig[2 * t];
    s_dig[2 * t + 1] = su.tdig[2 * t + 1];
    s_fac[t] = su.tfac[t];
  }
  __syncthreads();
}

__device__ __forceinline__ double surr_time(const DSurr& su, const int* s_pos, const int* s_dig, const double* s_fac,
                                            uint64_t idx, const int* dig) {
  double t = su.base;
  for (int q = 0; q < su.T; ++q) {
    const int p1 = s_pos[2 * q + 1];
    const bool hit = dig[s_pos[2 * q]] == s_dig[2 * q] && (p1 < 0 || dig[p1] == s_dig[2 * q + 1]);
    if (hit) t = __dmul_rn(t, s_fac[q]);
  }
  if (su.reps > 0 && su.sigma > 0.0) {
    double z = unit_normal(su.seed, idx, 0);
    for (int r = 1; r < su.reps; ++r) z = fmin(z, unit_normal(su.seed, idx, r));
    t = __dmul_rn(t, exp(__dmul_rn(su.sigma, z)));
  }
  return t;
}

__global__ void k_surr_times(DSpace lr, DSurr su, const int64_t* __restrict__ idx, int64_t n, double* __restrict__ times,
                             uint8_t* __restrict__ ok) {
  extern __shared__ double s_fac[];
  int* s_pos = reinterpret_cast<int*>(s_fac + su.T);
  int* s_dig = s_pos + 2 * su.T;
  stage_terms(su, s_pos, s_dig, s_fac);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int dig[kMaxP];
    const uint64_t x = (uint64_t)idx[i];
    decode_digits(lr, x, dig);
    const bool good = rules_ok(lr, dig);
    ok[i] = good;
    times[i] = good ? surr_time(su, s_pos, s_dig, s_fac, x, dig) : __longlong_as_double(0x7ff8000000000000ll);
  }
}

// (time, index) lexicographic minimum
__device__ __forceinline__ bool key_less(double t, int64_t i, double bt, int64_t bi) {
  return t < bt || (t == bt && i < bi);
}

// Exhaustive search over [begin, end): statically valid (space rules) and
// launchable (spec rules) configurations; per-CTA best (time, index), the
// number of valid configurations and of those strictly faster than `thr`.
__global__ void k_surr_best(DSpace sp, DSpace lr, DSurr su, int64_t begin, int64_t end, double thr,
                            SurrPart* __restrict__ part) {
  extern __shared__ double s_fac[];
  int* s_pos = reinterpret_cast<int*>(s_fac + su.T);
  int* s_dig = s_pos + 2 * su.T;
  stage_terms(su, s_pos, s_dig, s_fac);
  double bt = __longlong_as_double(0x7ff0000000000000ll);   // +inf
  int64_t bi = INT64_MAX;
  unsigned long long nv = 0, nb = 0;
  // contiguous per-thread runs keep the decode warp-coherent
  for (int64_t i = begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < end;
       i += (int64_t)gridDim.x * blockDim.x) {
    int dig[kMaxP];
    decode_digits(sp, (uint64_t)i, dig);
    if (!rules_ok(sp, dig) || !rules_ok(lr, dig)) continue;
    const double t = surr_time(su, s_pos, s_dig, s_fac, (uint64_t)i, dig);
    ++nv;
    nb += (t < thr);
    if (key_less(t, i, bt, bi)) {
      bt = t;
      bi = i;
    }
  }
  // warp then CTA reduction
  for (int o = 16; o > 0; o >>= 1) {
    const double ot = __shfl_down_sync(0xffffffffu, bt, o);
    const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
    nv += __shfl_down_sync(0xffffffffu, nv, o);
    nb += __shfl_down_sync(0xffffffffu, nb, o);
    if (key_less(ot, oi, bt, bi)) {
      bt = ot;
      bi = oi;
    }
  }
  __shared__ SurrPart w[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) w[wid] = SurrPart{bt, bi, (int64_t)nv, (int64_t)nb};
  __syncthreads();
  if (threadIdx.x == 0) {
    SurrPart r = w[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) {
      if (key_less(w[q].t, w[q].i, r.t, r.i)) {
        r.t = w[q].t;
        r.i = w[q].i;
      }
      r.n_valid += w[q].n_valid;
      r.n_below += w[q].n_below;
    }
    part[blockIdx.x] = r;
  }
}

// Exhaustive search (the ground truth of the tuner's slowdown), <= 64 terms:
// each thread walks a run of consecutive indices with an odometer over the
// digits held in registers, and tracks which terms hit as two 64-bit masks
// (bit q of A: term q's first (parameter, digit) matches; of B: its second,
// or always for one-parameter terms), updated by XOR when a digit changes.
// The time is base times the hit factors in ascending term order -- the same
// multiplications, in the same order, as surr_time, so it is bit-identical.
constexpr int PMAX = 16;   // parameters handled by k_surr_best_runs (digits in registers)
__global__ void __launch_bounds__(256) k_surr_best_runs(DSpace sp, DSpace lr, DSurr su, const uint64_t* __restrict__ gmask,
                                                        int nm, uint64_t b_ones, int64_t begin, int64_t end, int run,
                                                        double thr, SurrPart* __restrict__ part) {
  extern __shared__ double s_fac[];                 // [T] factors, then A masks [nm], B masks [nm]
  uint64_t* sA = reinterpret_cast<uint64_t*>(s_fac + su.T);
  uint64_t* sB = sA + nm;
  for (int t = threadIdx.x; t < su.T; t += blockDim.x) s_fac[t] = su.tfac[t];
  for (int q = threadIdx.x; q < 2 * nm; q += blockDim.x) sA[q] = gmask[q];
  __syncthreads();
  const int P = sp.P;
  const bool rules = sp.R > 0 || lr.R > 0;
  double bt = __longlong_as_double(0x7ff0000000000000ll);   // +inf
  int64_t bi = INT64_MAX;
  unsigned long long nv = 0, nb = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * run;
  for (int64_t r0 = begin + (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * run; r0 < end; r0 += stride) {
    const int64_t r1 = r0 + run < end ? r0 + run : end;
    int dig[PMAX];    // registers (static indices only)
    int dl[kMaxP];    // the same digits for the rule checks (dynamic indices: local memory)
    uint64_t x = (uint64_t)r0;
#pragma unroll
    for (int p = PMAX - 1; p >= 0; --p) {
      dig[p] = 0;
      if (p < P) {
        const uint64_t q = x / (uint64_t)sp.radix[p];
        dig[p] = (int)(x - q * (uint64_t)sp.radix[p]);
        x = q;
      }
      if (rules) dl[p] = dig[p];
    }
    uint64_t A = 0, B = b_ones;
#pragma unroll
    for (int p = 0; p < PMAX; ++p)
      if (p < P) {
        A |= sA[sp.voff[p] + dig[p]];
        B |= sB[sp.voff[p] + dig[p]];
      }
    for (int64_t i = r0; i < r1; ++i) {
      if (!rules || (rules_ok(sp, dl) && rules_ok(lr, dl))) {
        uint64_t h = A & B;
        double t = su.base;
        while (h) {
          t = __dmul_rn(t, s_fac[__ffsll((long long)h) - 1]);
          h &= h - 1;
        }
        if (su.reps > 0 && su.sigma > 0.0) {   // measured times: exactly surr_time's noise
          double z = unit_normal(su.seed, (uint64_t)i, 0);
          for (int r = 1; r < su.reps; ++r) z = fmin(z, unit_normal(su.seed, (uint64_t)i, r));
          t = __dmul_rn(t, exp(__dmul_rn(su.sigma, z)));
        }
        ++nv;
        nb += (t < thr);
        if (key_less(t, i, bt, bi)) {
          bt = t;
          bi = i;
        }
      }
#pragma unroll
      for (int p = PMAX - 1; p >= 0; --p) {   // odometer: next index, last parameter fastest
        if (p < P) {
          const int o = dig[p];
          int nw = o + 1;
          const bool wrap = nw == sp.radix[p];
          if (wrap) nw = 0;
          A ^= sA[sp.voff[p] + o] ^ sA[sp.voff[p] + nw];
          B ^= sB[sp.voff[p] + o] ^ sB[sp.voff[p] + nw];
          dig[p] = nw;
          if (rules) dl[p] = nw;
          if (!wrap) break;
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ot = __shfl_down_sync(0xffffffffu, bt, o);
    const int64_t oi = __shfl_down_sync(0xffffffffu, bi, o);
    nv += __shfl_down_sync(0xffffffffu, nv, o);
    nb += __shfl_down_sync(0xffffffffu, nb, o);
    if (key_less(ot, oi, bt, bi)) {
      bt = ot;
      bi = oi;
    }
  }
  __shared__ SurrPart w[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) w[wid] = SurrPart{bt, bi, (int64_t)nv, (int64_t)nb};
  __syncthreads();
  if (threadIdx.x == 0) {
    SurrPart r = w[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) {
      if (key_less(w[q].t, w[q].i, r.t, r.i)) {
        r.t = w[q].t;
        r.i = w[q].i;
      }
      r.n_valid += w[q].n_valid;
      r.n_below += w[q].n_below;
    }
    part[blockIdx.x] = r;
  }
}


// k_surr_times with the term-hit masks of k_surr_best_runs (<= 64 terms,
// <= 16 parameters): digits decoded into registers, the same products in the
// same term order, the same noise.
__global__ void __launch_bounds__(256) k_surr_times_masks(DSpace lr, DSurr su, const uint64_t* __restrict__ gmask,
                                                          int nm, uint64_t b_ones, const int64_t* __restrict__ idx,
                                                          int64_t n, double* __restrict__ times,
                                                          uint8_t* __restrict__ ok) {
  extern __shared__ double s_fac[];
  uint64_t* sA = reinterpret_cast<uint64_t*>(s_fac + su.T);
  uint64_t* sB = sA + nm;
  for (int t = threadIdx.x; t < su.T; t += blockDim.x) s_fac[t] = su.tfac[t];
  for (int q = threadIdx.x; q < 2 * nm; q += blockDim.x) sA[q] = gmask[q];
  __syncthreads();
  const int P = lr.P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x0 = (uint64_t)idx[i];
    int dl[kMaxP];
    uint64_t x = x0, A = 0, B = b_ones;
#pragma unroll
    for (int p = PMAX - 1; p >= 0; --p) {
      if (p < P) {
        const uint64_t q = x / (uint64_t)lr.radix[p];
        const int d = (int)(x - q * (uint64_t)lr.radix[p]);
        x = q;
        A |= sA[lr.voff[p] + d];
        B |= sB[lr.voff[p] + d];
        dl[p] = d;
      }
    }
    const bool good = lr.R == 0 || rules_ok(lr, dl);
    ok[i] = good;
    double t = __longlong_as_double(0x7ff8000000000000ll);
    if (good) {
      uint64_t h = A & B;
      t = su.base;
      while (h) {
        t = __dmul_rn(t, s_fac[__ffsll((long long)h) - 1]);
        h &= h - 1;
      }
      if (su.reps > 0 && su.sigma > 0.0) {
        double z = unit_normal(su.seed, x0, 0);
        for (int r = 1; r < su.reps; ++r) z = fmin(z, unit_normal(su.seed, x0, r));
        t = __dmul_rn(t, exp(__dmul_rn(su.sigma, z)));
      }
    }
    times[i] = t;
  }
}

__global__ void k_surr_best_final(const SurrPart* __restrict__ part, int n, SurrPart* __restrict__ out) {
  __shared__ SurrPart w[1024];
  SurrPart r{__longlong_as_double(0x7ff0000000000000ll), INT64_MAX, 0, 0};
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    const SurrPart p = part[q];
    if (key_less(p.t, p.i, r.t, r.i)) {
      r.t = p.t;
      r.i = p.i;
    }
    r.n_valid += p.n_valid;
    r.n_below += p.n_below;
  }
  w[threadIdx.x] = r;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      SurrPart& a = w[threadIdx.x];
      const SurrPart b = w[threadIdx.x + s];
      if (key_less(b.t, b.i, a.t, a.i)) {
        a.t = b.t;
        a.i = b.i;
      }
      a.n_valid += b.n_valid;
      a.n_below += b.n_below;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = w[0];
}

}  // namespace mlt
