// train.cu — on-device fp64 ensemble training (north-star subsystem 3;
// reference model.py:194-249 `_fit`, :308-341 `train_ensemble`).
//
// One CTA per ensemble member, persistent over all epochs. Lane j of every
// warp owns hidden unit j (h <= 32); the 32 rows of a mini-batch chunk are
// split over the CTA's 16 warps (2 rows each: the per-step dependency chain is
// latency-bound, so more warps per scheduler beat more rows per warp — 4 warps
// 0.17 s, 8 warps 0.21 s, 16 warps 0.13 s for k = 16 x 500 epochs), each warp
// accumulates its rows' gradients in registers, and one reduction through
// shared memory per step feeds the momentum update. Exact-width instances for
// d <= 16 remove the per-element bounds checks of the input loops (0.10 s).
// The caller supplies every random draw (initial weights, per-epoch
// permutations) from the reference's own PCG64 stream, so the device follows
// the reference step sequence exactly; arithmetic mirrors the reference's
// rounding sequence (separate multiplies/subtractions where numpy does them),
// leaving only BLAS summation-order differences (~1e-16 relative per step).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kernels.cuh"

namespace mlt {

#ifndef MLT_TW
#define MLT_TW 16
#endif
constexpr int kTW = MLT_TW;      // warps per member CTA
constexpr int kTMaxD = 32;
constexpr int kRowsPerWarp = 32 / kTW;  // rows of a 32-row chunk per warp

struct TrainArgs {
  int k, d, h, epochs, B;
  double lr, mu;
  const double* x;               // [n_rows][d]
  const double* t;               // member-major standardized targets
  const int* rows;               // member-major row ids into x
  const int* n_m;                // [k]
  const int64_t* off;            // [k] offset of member m in t/rows
  const int64_t* poff;           // [k] offset of member m in perms
  const int* perms;              // per member: epochs x n_m
  const double* iw1;             // [k][h][d]
  const double* iw2;             // [k][h]
  // compact features: x[r][p] == ftab[foff[p] + codes[r*d + p]] (every column has <= 256 values)
  const uint8_t* codes;          // [n_rows][d] or null
  const double* ftab;
  int foff[kTMaxD + 1];
  int smem_rows;                 // rows staged per member (0: read x / t from global memory)
  double *ow1, *ob1, *ow2, *ob2, *lfirst, *llast;
  int* div_epoch;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// dynamic shared memory: part [kTW][kTMaxD + 2][32] doubles, then (SMEM) the
// member's targets [n] doubles, the feature table, and its codes [n][d] bytes
size_t train_smem(const TrainArgs& a, int n_max, int ftab_n) {
  size_t b = sizeof(double) * kTW * (a.d + 2) * 32;
  if (a.smem_rows) b += sizeof(double) * ((size_t)n_max + ftab_n) + (size_t)n_max * a.d;
  return (b + 15) & ~(size_t)15;
}

// SMEM: the member's rows live in shared memory as 1-byte feature codes (+ a
// small fp64 table) and its targets as fp64, so a step's only global access
// is the permutation chunk, prefetched one step ahead. Rows of a warp are
// processed with instruction-level parallelism (8 independent forward
// chains, interleaved butterflies); per-row arithmetic and every
// accumulation order are unchanged.
template <bool SMEM, int DC>
__global__ void __launch_bounds__(kTW * 32) k_train(TrainArgs a, int ftab_n) {
  constexpr int DU = DC ? DC : kTMaxD;     // unrolled width of the input loops
  const int m = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = DC ? DC : a.d, h = a.h;
  const int n = a.n_m[m];
  const double* T = a.t + a.off[m];
  const int* R = a.rows + a.off[m];
  const int* PERM = a.perms + a.poff[m];

  __shared__ double W1[kTMaxD][32], V1[kTMaxD][32];
  __shared__ double B1[32], VB1[32], W2[32], VW2[32];
  extern __shared__ double dyn[];
  double* part = dyn;                                // [kTW][d + 2][32] per-warp gradient partials
  auto P = [&](int w, int p, int j) -> double& { return part[((size_t)w * (d + 2) + p) * 32 + j]; };
  double* s_t = dyn + kTW * (d + 2) * 32;            // SMEM: [n] targets
  double* s_f = s_t + (SMEM ? n : 0);                // SMEM: feature table
  uint8_t* s_c = reinterpret_cast<uint8_t*>(s_f + (SMEM ? ftab_n : 0));   // SMEM: [n][d] codes
  __shared__ double pscal[kTW][2];            // per-warp (sum dout, sum r^2)
  __shared__ double xs[kTW][kRowsPerWarp][kTMaxD];
  __shared__ double ts[kTW][kRowsPerWarp];
  __shared__ double s_b2, s_vb2, s_sse;

  for (int q = tid; q < kTMaxD * 32; q += blockDim.x) {
    const int p = q / 32, j = q % 32;
    W1[p][j] = (p < d && j < h) ? a.iw1[((size_t)m * h + j) * d + p] : 0.0;
    V1[p][j] = 0.0;
  }
  if (tid < 32) {
    B1[tid] = 0.0;
    VB1[tid] = 0.0;
    W2[tid] = tid < h ? a.iw2[(size_t)m * h + tid] : 0.0;
    VW2[tid] = 0.0;
  }
  if (tid == 0) {
    s_b2 = 0.0;
    s_vb2 = 0.0;
  }
  if (SMEM) {
    for (int q = tid; q < n; q += blockDim.x) s_t[q] = T[q];
    for (int q = tid; q < ftab_n; q += blockDim.x) s_f[q] = a.ftab[q];
    for (int q = tid; q < n * d; q += blockDim.x) {
      const int ex = q / d, p = q - ex * d;
      s_c[q] = a.codes[(size_t)R[ex] * d + p];
    }
  }
  __syncthreads();
  const bool active = lane < h;
  // register-owned parameters (see the momentum update): needs exact-width
  // inputs with one warp per parameter row and two spare lanes in warp 0
  constexpr bool kOwn = DC != 0 && DC + 2 <= kTW;
  const bool own = kOwn && h <= 30;
  double own_w = 0.0, own_v = 0.0;
  if (own && lane < h && warp < d + 2) own_w = warp < d ? W1[warp][lane] : (warp == d ? B1[lane] : W2[lane]);
  if (own && warp == 0 && lane == 30) own_w = s_b2;
  double first = nan(""), last = nan("");
  int diverged = 0;

  for (int e = 1; e <= a.epochs; ++e) {
    const int* perm = PERM + (size_t)(e - 1) * n;
    if (tid == 0) s_sse = 0.0;
    int pf = 0;   // SMEM: prefetched permutation entry of this lane's row in the next chunk
    if (SMEM && lane < max(0, min(kRowsPerWarp, min(a.B, n) - warp * kRowsPerWarp))) pf = perm[warp * kRowsPerWarp + lane];
    for (int s = 0; s < n; s += a.B) {
      const int mb = min(a.B, n - s);
      const double c2m = 2.0 / (double)mb;
      double gW[DU];
#pragma unroll
      for (int p = 0; p < DU; ++p) gW[p] = 0.0;
      double gb1 = 0.0, gw2 = 0.0, gb2 = 0.0, sse = 0.0;
      const double w2j = W2[lane], b1j = B1[lane], b2 = s_b2;
      for (int c0 = 0; c0 < mb; c0 += 32) {
        const int rbase = c0 + warp * kRowsPerWarp;
        const int nr = max(0, min(kRowsPerWarp, mb - rbase));
        // stage this warp's rows (features + targets)
        if (SMEM) {
          // this chunk's permutation entries were prefetched one chunk ahead
          // (the permutations stream from DRAM: a dependent load per step
          // would put its latency on the critical path)
          const int ex_l = pf;
          {
            int ns = s, nc = c0 + 32;
            if (nc >= mb) {
              ns = s + a.B;
              nc = 0;
            }
            const int nrb = nc + warp * kRowsPerWarp;
            const int nmb = min(a.B, n - ns);
            pf = (ns < n && lane < max(0, min(kRowsPerWarp, nmb - nrb))) ? __ldcs(perm + ns + nrb + lane) : 0;
          }
          for (int base = 0; base < nr * d; base += 32) {   // uniform trip count: every lane shuffles
            const int q = base + lane;
            const int rr = q < nr * d ? q / d : 0, p = q - rr * d;
            const int ex = __shfl_sync(0xffffffffu, ex_l, rr);
            if (q < nr * d) xs[warp][rr][p] = s_f[a.foff[p] + s_c[ex * d + p]];
          }
          if (lane < nr) ts[warp][lane] = s_t[ex_l];
        } else {
          for (int q = lane; q < nr * d; q += 32) {
            const int rr = q / d, p = q - rr * d;
            const int ex = perm[s + rbase + rr];
            xs[warp][rr][p] = a.x[(size_t)R[ex] * d + p];
          }
          if (lane < nr) ts[warp][lane] = T[perm[s + rbase + lane]];
        }
        __syncwarp();
        if (nr == kRowsPerWarp) {
          // forward of 8 rows, interleaved
          double z[kRowsPerWarp];
#pragma unroll
          for (int rr = 0; rr < kRowsPerWarp; ++rr) z[rr] = 0.0;
#pragma unroll
          for (int p = 0; p < DU; ++p)
            if (DC || p < d) {
              const double w = W1[p][lane];
#pragma unroll
              for (int rr = 0; rr < kRowsPerWarp; ++rr) z[rr] = fma(xs[warp][rr][p], w, z[rr]);
            }
          double hj[kRowsPerWarp], o[kRowsPerWarp];
#pragma unroll
          for (int rr = 0; rr < kRowsPerWarp; ++rr) {
            hj[rr] = 1.0 / (1.0 + exp(-__dadd_rn(z[rr], b1j)));
            o[rr] = active ? hj[rr] * w2j : 0.0;
          }
#pragma unroll
          for (int sh = 16; sh > 0; sh >>= 1)
#pragma unroll
            for (int rr = 0; rr < kRowsPerWarp; ++rr) o[rr] += __shfl_xor_sync(0xffffffffu, o[rr], sh);
#pragma unroll
          for (int rr = 0; rr < kRowsPerWarp; ++rr) {
            const double r = __dsub_rn(__dadd_rn(o[rr], b2), ts[warp][rr]);
            const double dout = __dmul_rn(c2m, r);
            sse = fma(r, r, sse);
            gb2 = __dadd_rn(gb2, dout);
            if (active) {
              gw2 = fma(hj[rr], dout, gw2);
              const double dz = __dmul_rn(__dmul_rn(__dmul_rn(dout, w2j), hj[rr]), __dsub_rn(1.0, hj[rr]));
              gb1 = __dadd_rn(gb1, dz);
              z[rr] = dz;
            }
          }
          if (active) {
#pragma unroll
            for (int p = 0; p < DU; ++p)
              if (DC || p < d) {
#pragma unroll
                for (int rr = 0; rr < kRowsPerWarp; ++rr) gW[p] = fma(z[rr], xs[warp][rr][p], gW[p]);
              }
          }
        } else {
          for (int rr = 0; rr < nr; ++rr) {
            double zz = 0.0;
#pragma unroll
            for (int p = 0; p < DU; ++p)
              if (DC || p < d) zz = fma(xs[warp][rr][p], W1[p][lane], zz);
            zz = __dadd_rn(zz, b1j);
            const double hh = 1.0 / (1.0 + exp(-zz));
            const double out = __dadd_rn(warp_sum(active ? hh * w2j : 0.0), b2);
            const double r = __dsub_rn(out, ts[warp][rr]);
            const double dout = __dmul_rn(c2m, r);
            sse = fma(r, r, sse);
            gb2 = __dadd_rn(gb2, dout);
            if (active) {
              gw2 = fma(hh, dout, gw2);
              const double dz = __dmul_rn(__dmul_rn(__dmul_rn(dout, w2j), hh), __dsub_rn(1.0, hh));
              gb1 = __dadd_rn(gb1, dz);
#pragma unroll
              for (int p = 0; p < DU; ++p)
                if (DC || p < d) gW[p] = fma(dz, xs[warp][rr][p], gW[p]);
            }
          }
        }
        __syncwarp();
      }
      // per-warp partials -> shared memory
#pragma unroll
      for (int p = 0; p < DU; ++p)
        if (DC || p < d) P(warp, p, lane) = gW[p];
      P(warp, d, lane) = gb1;
      P(warp, d + 1, lane) = gw2;
      if (lane == 0) {
        pscal[warp][0] = gb2;
        pscal[warp][1] = sse;
      }
      __syncthreads();
      // momentum update: v = mu*v - lr*g ; w += v   (model.py:233-240)
      if (own) {
        // warp p updates parameter row p, lane j unit j, from registers (the
        // weight and its velocity live in the updating thread; the shared
        // copy is what the next step's forward reads); the two idle lanes of
        // warp 0 (h <= 30) reduce the output bias and the loss
        if (warp < d + 2 && lane < h) {
          double g = P(0, warp, lane);
#pragma unroll
          for (int w = 1; w < kTW; ++w) g = __dadd_rn(g, P(w, warp, lane));
          own_v = __dsub_rn(__dmul_rn(a.mu, own_v), __dmul_rn(a.lr, g));
          own_w = __dadd_rn(own_w, own_v);
          if (warp < d) W1[warp][lane] = own_w;
          else if (warp == d) B1[lane] = own_w;
          else W2[lane] = own_w;
        } else if (warp == 0 && lane == 30) {
          double g = pscal[0][0];
#pragma unroll
          for (int w = 1; w < kTW; ++w) g = __dadd_rn(g, pscal[w][0]);
          own_v = __dsub_rn(__dmul_rn(a.mu, own_v), __dmul_rn(a.lr, g));
          own_w = __dadd_rn(own_w, own_v);
          s_b2 = own_w;
        } else if (warp == 0 && lane == 31) {
          double ss = pscal[0][1];
#pragma unroll
          for (int w = 1; w < kTW; ++w) ss = __dadd_rn(ss, pscal[w][1]);
          s_sse = __dadd_rn(s_sse, ss);
        }
        __syncthreads();
        continue;
      }
      for (int q = tid; q < (d + 2) * 32; q += blockDim.x) {
        const int p = q / 32, j = q % 32;
        if (j >= h) continue;
        double g = P(0, p, j);
#pragma unroll
        for (int w = 1; w < kTW; ++w) g = __dadd_rn(g, P(w, p, j));
        if (p < d) {
          const double v = __dsub_rn(__dmul_rn(a.mu, V1[p][j]), __dmul_rn(a.lr, g));
          V1[p][j] = v;
          W1[p][j] = __dadd_rn(W1[p][j], v);
        } else if (p == d) {
          const double v = __dsub_rn(__dmul_rn(a.mu, VB1[j]), __dmul_rn(a.lr, g));
          VB1[j] = v;
          B1[j] = __dadd_rn(B1[j], v);
        } else {
          const double v = __dsub_rn(__dmul_rn(a.mu, VW2[j]), __dmul_rn(a.lr, g));
          VW2[j] = v;
          W2[j] = __dadd_rn(W2[j], v);
        }
      }
      if (tid == 0) {
        double g = pscal[0][0], ss = pscal[0][1];
        for (int w = 1; w < kTW; ++w) {
          g = __dadd_rn(g, pscal[w][0]);
          ss = __dadd_rn(ss, pscal[w][1]);
        }
        const double v = __dsub_rn(__dmul_rn(a.mu, s_vb2), __dmul_rn(a.lr, g));
        s_vb2 = v;
        s_b2 = __dadd_rn(s_b2, v);
        s_sse = __dadd_rn(s_sse, ss);
      }
      __syncthreads();
    }
    const double loss = s_sse / (double)n;
    __syncthreads();   // everyone has read s_sse before thread 0 resets it
    if (!isfinite(loss)) {
      diverged = e;
      break;
    }
    if (e == 1) first = loss;
    last = loss;
  }
  // outputs
  for (int q = tid; q < h * d; q += blockDim.x) {
    const int j = q / d, p = q % d;
    a.ow1[((size_t)m * h + j) * d + p] = W1[p][j];
  }
  for (int j = tid; j < h; j += blockDim.x) {
    a.ob1[(size_t)m * h + j] = B1[j];
    a.ow2[(size_t)m * h + j] = W2[j];
  }
  if (tid == 0) {
    a.ob2[m] = s_b2;
    a.lfirst[m] = first;
    a.llast[m] = last;
    a.div_epoch[m] = diverged;
  }
}

typedef void (*TrainKernel)(TrainArgs, int);

// exact-width instances for the inputs of real spaces (unrolled loops with no
// per-element bounds checks); any other width up to 32 uses the generic one
template <bool SMEM>
TrainKernel pick_train_w(int d) {
  switch (d) {
#define MLT_TRAIN_D(n) \
  case n: return k_train<SMEM, n>;
    MLT_TRAIN_D(1) MLT_TRAIN_D(2) MLT_TRAIN_D(3) MLT_TRAIN_D(4) MLT_TRAIN_D(5) MLT_TRAIN_D(6)
    MLT_TRAIN_D(7) MLT_TRAIN_D(8) MLT_TRAIN_D(9) MLT_TRAIN_D(10) MLT_TRAIN_D(11) MLT_TRAIN_D(12)
    MLT_TRAIN_D(13) MLT_TRAIN_D(14) MLT_TRAIN_D(15) MLT_TRAIN_D(16)
#undef MLT_TRAIN_D
  }
  return k_train<SMEM, 0>;
}
TrainKernel pick_train(bool smem, int d) { return smem ? pick_train_w<true>(d) : pick_train_w<false>(d); }

}  // namespace mlt

// ---------------------------------------------------------------------------
// host entry point
// ---------------------------------------------------------------------------
namespace {
thread_local char g_terr[256];
}

extern "C" int mlt_train_members_impl(int dev, cudaStream_t stream, int64_t* launches, const mlt_train_desc* dd,
                                      double* w1, double* b1, double* w2, double* b2, double* lf, double* ll,
                                      int32_t* div, const char** err) {
  using namespace mlt;
  *err = g_terr;
  g_terr[0] = 0;
  const mlt_train_desc& D = *dd;
  auto bad = [&](int code, const char* msg) {
    snprintf(g_terr, sizeof g_terr, "%s", msg);
    return code;
  };
  if (D.k < 1) return bad(MLT_EINVAL, "k must be >= 1");
  if (D.d < 1 || D.d > kTMaxD) return bad(MLT_EINVAL, "training supports 1..32 inputs");
  if (D.h < 1 || D.h > 32) return bad(MLT_EINVAL, "training supports 1..32 hidden units");
  if (D.epochs < 1 || D.batch_size < 1) return bad(MLT_EINVAL, "epochs and batch_size must be positive");
  std::vector<int64_t> off(D.k), poff(D.k);
  int64_t tot = 0, ptot = 0;
  for (int m = 0; m < D.k; ++m) {
    if (D.n_m[m] < 1) return bad(MLT_EDATA, "a member has no training examples");
    off[m] = tot;
    poff[m] = ptot;
    tot += D.n_m[m];
    ptot += (int64_t)D.epochs * D.n_m[m];
  }
  cudaError_t e = cudaSetDevice(dev);
  auto cuda_fail = [&](cudaError_t ce) {
    snprintf(g_terr, sizeof g_terr, "CUDA error in training: %s", cudaGetErrorString(ce));
    return MLT_ECUDA;
  };
  if (e != cudaSuccess) return cuda_fail(e);
  const size_t kh = (size_t)D.k * D.h;
  const size_t bytes_x = (size_t)D.n_rows * D.d * 8, bytes_t = tot * 8, bytes_r = tot * 4, bytes_n = D.k * 4,
               bytes_o = D.k * 8 * 2, bytes_p = ptot * 4, bytes_w1 = kh * D.d * 8, bytes_w2 = kh * 8;
  const size_t outb = bytes_w1 + 2 * kh * 8 + (size_t)D.k * 8 * 3 + (size_t)D.k * 4;
  char* buf = nullptr;
  const size_t total = bytes_x + bytes_t + bytes_r + bytes_n + bytes_o + bytes_p + bytes_w1 + bytes_w2 + outb + 1024;
  if ((e = cudaMallocAsync(&buf, total, stream)) != cudaSuccess) return cuda_fail(e);
  size_t at = 0;
  auto take = [&](size_t nb) {
    char* p = buf + at;
    at += (nb + 15) & ~(size_t)15;
    return p;
  };
  double* dx = (double*)take(bytes_x);
  double* dt = (double*)take(bytes_t);
  int* dr = (int*)take(bytes_r);
  int* dn = (int*)take(bytes_n);
  int64_t* doff = (int64_t*)take(bytes_o);
  int64_t* dpoff = doff + D.k;
  int* dp = (int*)take(bytes_p);
  double* diw1 = (double*)take(bytes_w1);
  double* diw2 = (double*)take(bytes_w2);
  double* ow1 = (double*)take(bytes_w1);
  double* ob1 = (double*)take(kh * 8);
  double* ow2 = (double*)take(kh * 8);
  double* ob2 = (double*)take(D.k * 8);
  double* olf = (double*)take(D.k * 8);
  double* oll = (double*)take(D.k * 8);
  int* odiv = (int*)take(D.k * 4);
  cudaMemcpyAsync(dx, D.x, bytes_x, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dt, D.t, bytes_t, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dr, D.rows, bytes_r, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dn, D.n_m, bytes_n, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(doff, off.data(), D.k * 8, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dpoff, poff.data(), D.k * 8, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dp, D.perms, bytes_p, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(diw1, D.init_w1, bytes_w1, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(diw2, D.init_w2, bytes_w2, cudaMemcpyHostToDevice, stream);
  TrainArgs a;
  std::memset(&a, 0, sizeof a);
  // compact feature codes: every column of x takes few distinct values (digit / (count - 1))
  std::vector<double> ftab;
  std::vector<uint8_t> codes;
  bool compact = D.d <= kTMaxD;
  {
    std::vector<std::vector<double>> cols(D.d);
    for (int p = 0; compact && p < D.d; ++p) {
      std::vector<double>& v = cols[p];
      for (int64_t r = 0; r < D.n_rows; ++r) v.push_back(D.x[(size_t)r * D.d + p]);
      std::sort(v.begin(), v.end(), [](double u, double w) { return u < w || (u == w && std::signbit(u) && !std::signbit(w)); });
      v.erase(std::unique(v.begin(), v.end(), [](double u, double w) {
                return std::memcmp(&u, &w, 8) == 0;
              }), v.end());
      if (v.size() > 256) compact = false;
    }
    if (compact) {
      codes.resize((size_t)D.n_rows * D.d);
      for (int p = 0; p < D.d; ++p) {
        a.foff[p] = (int)ftab.size();
        ftab.insert(ftab.end(), cols[p].begin(), cols[p].end());
        for (int64_t r = 0; r < D.n_rows; ++r) {
          const double xv = D.x[(size_t)r * D.d + p];
          int c = -1;
          for (size_t u = 0; u < cols[p].size(); ++u)
            if (std::memcmp(&cols[p][u], &xv, 8) == 0) {
              c = (int)u;
              break;
            }
          if (c < 0) compact = false;
          codes[(size_t)r * D.d + p] = (uint8_t)(c < 0 ? 0 : c);
        }
      }
      a.foff[D.d] = (int)ftab.size();
    }
  }
  int n_max = 0;
  for (int m = 0; m < D.k; ++m) n_max = std::max(n_max, (int)D.n_m[m]);
  a.k = D.k;
  a.d = D.d;
  a.h = D.h;
  a.epochs = D.epochs;
  a.B = D.batch_size;
  a.lr = D.learning_rate;
  a.mu = D.momentum;
  a.x = dx;
  a.t = dt;
  a.rows = dr;
  a.n_m = dn;
  a.off = doff;
  a.poff = dpoff;
  a.perms = dp;
  a.iw1 = diw1;
  a.iw2 = diw2;
  a.ow1 = ow1;
  a.ob1 = ob1;
  a.ow2 = ow2;
  a.ob2 = ob2;
  a.lfirst = olf;
  a.llast = oll;
  a.div_epoch = odiv;
  a.smem_rows = compact ? 1 : 0;
  size_t smem = train_smem(a, n_max, (int)ftab.size());
  if (smem > 200 * 1024) {          // the member's rows do not fit: read them from global memory
    a.smem_rows = 0;
    smem = train_smem(a, n_max, 0);
  }
  uint8_t* dcodes = nullptr;
  double* dftab = nullptr;
  if (a.smem_rows) {
    if ((e = cudaMallocAsync(&dcodes, codes.size() + ftab.size() * 8 + 16, stream)) != cudaSuccess) {
      cudaFreeAsync(buf, stream);
      return cuda_fail(e);
    }
    dftab = reinterpret_cast<double*>(dcodes + ((codes.size() + 15) & ~(size_t)15));
    cudaMemcpyAsync(dcodes, codes.data(), codes.size(), cudaMemcpyHostToDevice, stream);
    cudaMemcpyAsync(dftab, ftab.data(), ftab.size() * 8, cudaMemcpyHostToDevice, stream);
    a.codes = dcodes;
    a.ftab = dftab;
  }
  void (*kern)(TrainArgs, int) = pick_train(a.smem_rows != 0, D.d);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const bool trace = std::getenv("MLT_STEP_TRACE") != nullptr;   // diagnostics: upload / kernel split
  cudaEvent_t tev[3];
  if (trace) {
    for (auto& ev : tev) cudaEventCreate(&ev);
    cudaEventRecord(tev[0], stream);   // (uploads were enqueued before: time from the call start on host)
  }
  kern<<<D.k, kTW * 32, smem, stream>>>(a, (int)ftab.size());
  if (trace) cudaEventRecord(tev[1], stream);
  (*launches)++;
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    cudaMemcpyAsync(w1, ow1, bytes_w1, cudaMemcpyDeviceToHost, stream);
    cudaMemcpyAsync(b1, ob1, kh * 8, cudaMemcpyDeviceToHost, stream);
    cudaMemcpyAsync(w2, ow2, kh * 8, cudaMemcpyDeviceToHost, stream);
    cudaMemcpyAsync(b2, ob2, D.k * 8, cudaMemcpyDeviceToHost, stream);
    cudaMemcpyAsync(lf, olf, D.k * 8, cudaMemcpyDeviceToHost, stream);
    cudaMemcpyAsync(ll, oll, D.k * 8, cudaMemcpyDeviceToHost, stream);
    cudaMemcpyAsync(div, odiv, D.k * 4, cudaMemcpyDeviceToHost, stream);
    e = cudaStreamSynchronize(stream);
  }
  if (trace) {
    float kms = 0;
    cudaEventElapsedTime(&kms, tev[0], tev[1]);
    std::fprintf(stderr, "{\"train_kernel_ms\": %.3f, \"steps_per_member\": %lld}\n", kms,
                 (long long)D.epochs * ((D.n_m[0] + D.batch_size - 1) / D.batch_size));
    for (auto& ev : tev) cudaEventDestroy(ev);
  }
  cudaFreeAsync(buf, stream);
  if (dcodes) cudaFreeAsync(dcodes, stream);
  if (e != cudaSuccess) return cuda_fail(e);
  for (int m = 0; m < D.k; ++m)
    if (div[m] != 0) {
      snprintf(g_terr, sizeof g_terr, "training loss became non-finite at epoch %d (member %d)", div[m], m);
      return MLT_EDIVERGED;
    }
  return MLT_OK;
}
