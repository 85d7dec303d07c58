// sweep.cu — the fp32 factored full-space sweep with a streaming guard-band
// top-m (north-star subsystems 1 + 2; reference tuner.py:95-131 over
// paramspace.py:184-213 and model.py:88-97, :146-170, :290-301).
//
// Algebra (exact, no approximation beyond fp32 rounding):
//   z_mj(idx) = A_mj(outer digits) + B_mj(inner digits)     (first layer is linear)
//   E = exp(-z) = Ea(outer) * Eb(inner),  Ea = exp(-(A - c)), Eb = exp(-(B + c))
//   w'_mj = w2_mj * std_m / k,   w' * sigmoid(z) = 1 / d',   d' = Ea * (Eb/w') + 1/w'
// so one hidden unit of one member costs ONE fp32 FMA for d' (no exp, no
// dot product). G units share one reciprocal:
//   G=3: 1/d0 + 1/d1 + 1/d2 = (d2*(d0+d1) + d0*d1) / (d0*d1*d2)
// which balances the FMA pipe (8/3 lane-ops per unit) against the MUFU pipe
// (1/3 reciprocal per unit). Two outer configurations ride in one f32x2
// register (FFMA2/FMUL2/FADD2), halving issue slots.
//
// Mean log time = sum over all units of 1/d' + cst.  Every value within
// `band` (= 2*delta, an a-priori fp32 error bound) of the running m-th best is
// kept as a candidate; candidates are rescored exactly in fp64 (k_predict64)
// and sorted by (prediction, index), which reproduces the reference's
// lexsort((indices, preds)) selection exactly.
#include "kernels.cuh"

#include <cub/block/block_radix_sort.cuh>

namespace mlt {

// ---------------------------------------------------------------------------
// Tables (fp64 products, rounded once to fp32; see TableArgs in kernels.cuh)
// ---------------------------------------------------------------------------

__global__ void k_table_factors(TableArgs t) {
  const int KH = t.k * kH;
  const int fs = t.foff[t.d];
  const int64_t total = (int64_t)KH * fs;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int pos = (int)(q / fs), r = (int)(q % fs);
    const int mj = t.unit_of[pos];
    const int m = mj / kH, j = mj % kH;
    int p = 0;
    while (t.foff[p + 1] <= r) ++p;
    const int dig = r - t.foff[p];
    double f = 1.0;
    if (j < t.h) {
      const double x = (double)dig / (double)(t.radix[p] > 1 ? t.radix[p] - 1 : 1);
      f = exp(-(t.w1[((size_t)m * t.h + j) * t.d + p] * x));
    }
    t.F[q] = f;
  }
}

// Partial products of the factor rows over a parameter range:
//   P[mj][q] = prod_{p in [p_lo, p_hi)} F[mj][foff[p] + digit_p(base + q)]
// where digits are those of the sub-index over [p_lo, p_hi) (last fastest),
// multiplied from the last parameter down (fp64; the tables are fp32).
// Every table entry is then ca|cb * P_hi * P_lo: two fp64 multiplies.

// x / d for non-negative operands, in 32 bits when both fit (a 64-bit
// division is a ~60-instruction sequence; these index splits run per thread)
__device__ __forceinline__ int64_t udiv(int64_t x, int64_t d) {
  return ((uint64_t)x | (uint64_t)d) <= 0xffffffffull ? (int64_t)((uint32_t)x / (uint32_t)d) : x / d;
}

// The four partial-product tables of one build (outer hi / lo, inner hi / lo)
// in ONE launch: each is a few tens of thousands of entries, so four launches
// cost ~10 us each in launch latency and tails. Both arguments are
// __grid_constant__: the job fields and the per-parameter radix / offset /
// divisor arrays are indexed at run time straight from the parameter bank,
// so each entry walks only its own job's parameters (a loop unrolled over all
// kMaxP parameters with predicates cost ~1,460 instructions per entry).
__global__ void k_table_partial4(const __grid_constant__ TableArgs t, const __grid_constant__ PartialJobs j) {
  const int KH = t.k * kH;
  const int64_t e0 = KH * j.count[0], e1 = e0 + KH * j.count[1], e2 = e1 + KH * j.count[2],
                tot = e2 + KH * j.count[3];
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < tot; q += (int64_t)gridDim.x * blockDim.x) {
    const int r = q < e0 ? 0 : (q < e1 ? 1 : (q < e2 ? 2 : 3));
    const int64_t off = q - (r == 0 ? 0 : (r == 1 ? e0 : (r == 2 ? e1 : e2)));
    const int64_t mj64 = fdiv(off, j.f_count[r]);
    const int mj = (int)mj64;
    uint64_t id = (uint64_t)(j.base[r] + (off - mj64 * j.count[r]));
    const double* Fj = t.F + (size_t)mj * t.foff[t.d];
    // digits of the sub-index over [p_lo, p_hi), last parameter fastest
    double e = 1.0;
    for (int p = j.p_hi[r] - 1; p >= j.p_lo[r]; --p) {
      const uint64_t qt = (uint64_t)fdiv((int64_t)id, t.f_radix[p]);
      e *= __ldg(Fj + t.foff[p] + (int)(id - qt * (uint64_t)t.radix[p]));
      id = qt;
    }
    j.out[r][off] = e;
  }
}


// Outer table Ea[ob][mj][r], one thread per element in output order
// (consecutive threads: consecutive outers of one position, so the PoH / PoL
// reads of a warp share rows; one thread per (block, position) writing float4s
// was slower, 22 -> 40 us on the 10^8 space, its loads stride over positions).
// Row o = o_lo + ob*kOB + r = (o / nlo) * nlo + o % nlo over the outer split.
template <typename I>   // index type: uint32_t when every index of the build fits (TableArgs::idx32)
__device__ __forceinline__ void table_outer(const TableArgs& t, int bid, int nblk) {
  const int KH = t.k * kH;
  const I total = (I)t.n_ob * KH * kOB, stride = (I)nblk * blockDim.x;
  for (I q = (I)bid * blockDim.x + threadIdx.x; q < total; q += stride) {
    const int r = (int)(q % kOB);
    const I q8 = q / kOB, ob = (I)fdiv((int64_t)q8, t.f_kh);
    const int mj = (int)(q8 - ob * KH);
    const I o = (I)t.o_lo + ob * kOB + r;
    float out = 1.0f;
    if ((int64_t)o < t.o_card && t.wprime[mj] != 0.0) {
      const I oh = (I)fdiv((int64_t)o, t.f_onlo);
      const I a = oh - (I)t.o_hi_base, b = o - oh * (I)t.o_nlo;
      out = (float)(t.ca[mj] * __ldg(t.PoH + (size_t)mj * t.o_nhi + a) * __ldg(t.PoL + (size_t)mj * t.o_nlo + b));
    }
    t.ea[q] = out;
  }
}

// Extremes of the inner part per (table position, inner block): over the
// block's inners, exp(-(B + c)) = exp(-c) * P_hi * P_lo in fp64 — its maximum
// for w' > 0 (sigmoid smallest), its minimum for w' < 0 — widened by 1e-12
// relative so fp64 rounding cannot make the bound optimistic.
__global__ void k_table_ebext(TableArgs t, double* ext) {
  // one warp per (position, inner block): lanes stride over the block's
  // inners; max / min are exact, so the reduction order does not matter
  const int KH = t.k * kH;
  const int64_t total = (int64_t)KH * t.n_ib;
  const int lane = threadIdx.x & 31;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < total; q += wstride) {
    const int pos = (int)(q / t.n_ib), ib = (int)(q % t.n_ib);
    const double wp = t.wprime[pos];
    double e = 0.0;
    if (wp != 0.0) {
      const double base = t.cb[pos] * wp;      // exp(-c)
      double mx = 0.0, mn = INFINITY;
      const int64_t i0 = (int64_t)ib * kInnerBlock;
      const int64_t i1 = i0 + kInnerBlock < t.c_in ? i0 + kInnerBlock : t.c_in;
#pragma unroll 4
      for (int64_t i = i0 + lane; i < i1; i += 32) {
        const int64_t ih = fdiv(i, t.f_inlo);
        const double v = base * __ldg(t.PiH + (size_t)pos * t.i_nhi + ih) *
                         __ldg(t.PiL + (size_t)pos * t.i_nlo + (i - ih * t.i_nlo));
        mx = fmax(mx, v);
        mn = fmin(mn, v);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      }
      e = wp > 0 ? mx * (1.0 + 1e-12) : mn * (1.0 - 1e-12);
    }
    if (lane == 0) ext[q] = e;
  }
}

// Sort key of each work item for the best-first order of the pruned sweep:
// the smallest checkpoint-0 bound over its outer rows (exactly what the
// kernel's checkpoint-0 test compares, so the early stop there is sound).
__global__ void k_item_keys(const float* remlo, int n_ck, int n_ib, int items, float* keys, int* vals) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < items; w += gridDim.x * blockDim.x) {
    const int ob = w / n_ib, ib = w - ob * n_ib;
    float mn = __int_as_float(0x7f800000);
#pragma unroll
    for (int r = 0; r < kOB; ++r) mn = fminf(mn, __ldg(remlo + (((size_t)ob * kOB + r) * n_ib + ib) * n_ck));
    keys[w] = mn;
    vals[w] = w;
  }
}

// Best-first order of up to kItemSortMax work items in two launches (the
// device-wide radix sort takes six, plus four allocations): k_item_runs sorts
// runs of kItemRun items, one CTA each (keys as k_item_keys; a stable
// cub::BlockRadixSort), and k_item_merge (a CTA per 1024 items, each with all
// the keys in shared memory) places every item at its rank in the
// whole: its position in its run plus, per other run, a binary search for the
// items ahead of it -- keys compared as cub's order-preserving bits, ties by
// item index (runs are index-contiguous: an earlier run's equal keys come
// first). The order is exactly the stable device-wide sort's. (A single CTA
// sorting all 6144 items of the 10^8 space: 58 us; a one-CTA bitonic: 121 us.)
__device__ __forceinline__ unsigned item_key_bits(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u ^ 0x80000000u);
}
__global__ void __launch_bounds__(kItemRunThreads) k_item_runs(const float* remlo, int n_ck, int n_ib, int items,
                                                               unsigned* run_key, int* run_val) {
  using Sort = cub::BlockRadixSort<float, kItemRunThreads, kItemRun / kItemRunThreads, int>;
  constexpr int kPer = kItemRun / kItemRunThreads;
  __shared__ typename Sort::TempStorage tmp;
  const int r0 = blockIdx.x * kItemRun;
  float key[kPer];
  int val[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int w = r0 + threadIdx.x * kPer + j;   // blocked arrangement: input rank = item index
    key[j] = __int_as_float(0x7f800000);
    val[j] = 0x7fffffff;                        // padding: after every item, +inf ones included
    if (w < items) {
      const int ob = w / n_ib, ib = w - ob * n_ib;
      float mn = __int_as_float(0x7f800000);
#pragma unroll
      for (int r = 0; r < kOB; ++r) mn = fminf(mn, __ldg(remlo + (((size_t)ob * kOB + r) * n_ib + ib) * n_ck));
      key[j] = mn;
      val[j] = w;
    }
  }
  Sort(tmp).Sort(key, val);
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int w = r0 + threadIdx.x * kPer + j;
    if (w < items) {
      run_key[w] = item_key_bits(key[j]);
      run_val[w] = val[j];
    }
  }
}
__global__ void __launch_bounds__(kItemSortThreads) k_item_merge(const unsigned* run_key, const int* run_val,
                                                                 int items, int* order) {
  extern __shared__ unsigned s_rk[];   // [kItemSortMax] keys: every CTA stages all of them
  for (int e = threadIdx.x; e < items; e += blockDim.x) s_rk[e] = run_key[e];
  __syncthreads();
  const int n_runs = (items + kItemRun - 1) / kItemRun;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < items; e += gridDim.x * blockDim.x) {
    const int r = e / kItemRun;
    const unsigned k = s_rk[e];
    int rank = e - r * kItemRun;
    for (int r2 = 0; r2 < n_runs; ++r2) {
      if (r2 == r) continue;
      const int b0 = r2 * kItemRun;
      int lo = 0, hi = min(kItemRun, items - b0);
      if (r2 < r) {   // earlier items: equal keys come first
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (s_rk[b0 + mid] <= k) lo = mid + 1; else hi = mid;
        }
      } else {
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (s_rk[b0 + mid] < k) lo = mid + 1; else hi = mid;
        }
      }
      rank += lo;
    }
    order[rank] = run_val[e];
  }
}

// Lower bounds of the units still to come, per (outer row, inner block) and checkpoint:
//   remlo[o][ib][c] = sum_{pos >= ck.unit[c]} min over the block's inners of w'*sigmoid(z)
// = w' / (1 + Ea64(o) * ext(pos, ib)) in fp64 (dummy units contribute exactly 1),
// rounded down with a safety margin so it stays a bound.
// CTAs stride over the outer rows: exp(-A') of each position is formed once
// per row (not once per inner block), and the row's terms go through shared
// memory in chunks of 256 positions x 8 inner blocks, last chunk first. Warp w
// owns inner block w: lane l sums positions [8l, 8l + 8) of the chunk from the
// last one down, a reverse warp scan adds the later runs and a carry the later
// chunks, and the lane holding a checkpoint's first unit u writes its bound --
// the suffix sum over [u, KH) -- straight from registers. Each bound is rounded
// down by 1e-9 (1 + |sum|) + 1e-12 sum_{pos >= u} |w'| (CkList::mag; every
// term is at most |w'| in magnitude, a dummy unit's exactly 1), which covers the fp64 error of summing
// <= 4096 terms in any order plus the 2-ulp reciprocal below, whatever the
// cancellation. (Round 2's thread per (row, interval, block) with a serial
// loop of dependent loads and divisions: ~250 us on the 10^8 space,
// profiles/r02_launches_bench_summary.txt.)
namespace {
constexpr int kRemIB = 8;        // inner blocks per pass = warps per CTA
constexpr int kRemChunk = 256;   // positions per pass = threads per CTA
// 1/d for 1 <= d <= 2^100: the MUFU fp64 reciprocal estimate (MUFU.RCP64H,
// ~2^-20) and two Newton steps (-> 2^-40 -> rounding): within 2 ulp of the
// correctly rounded quotient, with no fp32 round trip through the converter
__device__ __forceinline__ double rcp_newton(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}
}  // namespace

__global__ void __launch_bounds__(kRemChunk) k_table_rem(TableArgs t, CkList ck, const double* ext,
                                                           float* remlo) {
  // s_term[ib][p + p / 8]: one pad slot per 8 positions, so the lanes of a
  // warp reading position 8l + j of their own run hit distinct bank pairs
  constexpr int kLd = kRemChunk + kRemChunk / 8;
  __shared__ double s_term[kRemIB][kLd];
  __shared__ signed char s_ckat[kMaxUnitsParam];       // checkpoint whose first unit is pos, or -1
  __shared__ __align__(4) unsigned char s_runck[kMaxUnitsParam / 8];  // bit j: a checkpoint starts at pos 8 run + j
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int KH = t.k * kH, n_ck = ck.n, n_ib = t.n_ib;
  const int64_t rows = (int64_t)t.n_ob * kOB;
  for (int q = tid; q < KH; q += blockDim.x) s_ckat[q] = -1;
  for (int q = tid; q < (KH + 31) / 32; q += blockDim.x) reinterpret_cast<unsigned int*>(s_runck)[q] = 0u;
  __syncthreads();
  if (tid < n_ck) {
    s_ckat[ck.unit[tid]] = (signed char)tid;
    atomicOr(reinterpret_cast<unsigned int*>(s_runck) + ck.unit[tid] / 32, 1u << (ck.unit[tid] % 32));
  }
  __syncthreads();
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t o = t.o_lo + row;
    float* out = remlo + row * n_ib * n_ck;
    if (o >= t.o_card) {   // no configuration: prune freely (uniform over the CTA)
      for (int q = tid; q < n_ib * n_ck; q += blockDim.x) out[q] = __int_as_float(0x7f800000);
      continue;
    }
    const int64_t oh = udiv(o, t.o_nlo);
    const int64_t a = oh - t.o_hi_base, b = o - oh * t.o_nlo;
    for (int ib0 = 0; ib0 < n_ib; ib0 += kRemIB) {
      const int nb = min(kRemIB, n_ib - ib0);
      double carry = 0.0;   // warp `warp`: the sum over the chunks done (all later positions)
      for (int base = (KH - 1) / kRemChunk * kRemChunk; base >= 0; base -= kRemChunk) {
        const int pos = base + tid;
        double* st = &s_term[0][tid + tid / 8];
        if (pos >= KH) {   // past the last position: zero terms, so the sums need no guard
#pragma unroll
          for (int x = 0; x < kRemIB; ++x)
            if (x < nb) st[x * kLd] = 0.0;
        } else {
          // every load up front, then kRemIB independent chains; d >= 2^100
          // leaves a term below 2^-100 |w'| -- 0 for w' > 0, w' * 2^-100 for
          // w' < 0, both still lower bounds, and no branch
          const double wp = t.wprime[pos];
          const double* ex = ext + (size_t)pos * n_ib + ib0;
          const double ea = t.ca[pos] * __ldg(t.PoH + (size_t)pos * t.o_nhi + a) *
                            __ldg(t.PoL + (size_t)pos * t.o_nlo + b);
          auto term = [&](double e) {
            const double d = 1.0 + ea * e;
            return (wp > 0.0 && !(d < 0x1p100)) ? 0.0 : wp * rcp_newton(fmin(d, 0x1p100));
          };
          if (wp == 0.0) {   // dummy unit: exactly 1
#pragma unroll
            for (int x = 0; x < kRemIB; ++x)
              if (x < nb) st[x * kLd] = 1.0;
          } else if (nb == kRemIB) {   // (uniform) all eight blocks: no predicates
            double e8[kRemIB];
#pragma unroll
            for (int x = 0; x < kRemIB; ++x) e8[x] = __ldg(ex + x);
#pragma unroll
            for (int x = 0; x < kRemIB; ++x) st[x * kLd] = term(e8[x]);
          } else {
#pragma unroll
            for (int x = 0; x < kRemIB; ++x)
              if (x < nb) st[x * kLd] = term(__ldg(ex + x));
          }
        }
        __syncthreads();
        if (warp < nb) {
          // lane run [p0, p0 + 8) of the chunk (positions >= KH hold 0)
          const int p0 = 8 * lane;
          const double* sw = &s_term[warp][p0 + lane];   // (p0 + j) + (p0 + j) / 8 = p0 + lane + j
          double suf[8], run = 0.0;
#pragma unroll
          for (int j = 7; j >= 0; --j) {
            run += sw[j];
            suf[j] = run;
          }
          double inc = run;   // inclusive reverse scan over the lanes
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const double y = __shfl_down_sync(0xffffffffu, inc, off);
            if (lane + off < 32) inc += y;
          }
          const double after = inc - run + carry;
          carry += __shfl_sync(0xffffffffu, inc, 0);   // the whole chunk
          // the checkpoints whose first unit lies in this run (usually none or
          // one: a loop over the set bits, suf[j] picked by a select chain)
          const int pb = base + p0;
          unsigned mask = pb < KH ? s_runck[pb / 8] : 0u;
          while (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            double sj = suf[0];
#pragma unroll
            for (int q = 1; q < 8; ++q) sj = j == q ? suf[q] : sj;
            const int c = s_ckat[pb + j];
            const double sum = sj + after;
            out[(ib0 + warp) * n_ck + c] = __double2float_rd(sum - 1e-9 * (1.0 + fabs(sum)) - 1e-12 * ck.mag[c]);
          }
        }
        __syncthreads();
      }
    }
  }
}

// Inner table in the sweep's thread-contiguous layout ebp[ib][group][thread][4*ebw]
// (slot x*kInner + s = unit x of the group for inner ib*kInnerBlock + s*kThreads
// + thread; pad slots are zero): one thread per (inner block, group, thread)
// computes its 4*ebw slots and writes them as float4s -- consecutive threads
// write consecutive 16-byte chunks and read consecutive PiL entries.
template <int G, typename I>
__device__ __forceinline__ void table_inner(const TableArgs& t, int bid, int nblk) {
  constexpr int W = ebw_of(G), WF = 4 * W;
  const int ngroups = t.k * kH / G;
  const I total = (I)(t.c_in_pad / kInnerBlock) * ngroups * kThreads, stride = (I)nblk * blockDim.x;
  for (I q = (I)bid * blockDim.x + threadIdx.x; q < total; q += stride) {
    const int th = (int)(q % kThreads);
    const I rest = q / kThreads;
    const I ib = (I)fdiv((int64_t)rest, t.f_ngroups);
    const int gi = (int)(rest - ib * ngroups);
    I a[kInner], b[kInner];
    bool in[kInner];
#pragma unroll
    for (int s = 0; s < kInner; ++s) {
      const I i = ib * kInnerBlock + (I)s * kThreads + th;
      in[s] = (int64_t)i < t.c_in;
      a[s] = (I)fdiv((int64_t)i, t.f_inlo);
      b[s] = i - a[s] * (I)t.i_nlo;
    }
    float out[WF];
#pragma unroll
    for (int slot = 0; slot < WF; ++slot) {
      const int x = slot / kInner, s = slot % kInner;
      out[slot] = 0.0f;
      if (x < G && in[s]) {
        const int mj = gi * G + x;     // cb = 0 for dummy units
        out[slot] = (float)(t.cb[mj] * __ldg(t.PiH + (size_t)mj * t.i_nhi + a[s]) *
                            __ldg(t.PiL + (size_t)mj * t.i_nlo + b[s]));
      }
    }
    float4* dst = reinterpret_cast<float4*>(t.ebp + (size_t)q * WF);
#pragma unroll
    for (int w = 0; w < W; ++w) dst[w] = make_float4(out[4 * w], out[4 * w + 1], out[4 * w + 2], out[4 * w + 3]);
  }
}
// Both sweep tables in ONE launch: blocks [0, nb_outer) build the outer
// table, the rest the inner one -- the two are independent and each is
// latency-bound, so they overlap instead of running back to back.
template <int G>
__global__ void k_table_tiles(TableArgs t, int nb_outer) {
  const int b = blockIdx.x;
  if (b < nb_outer) {
    if (t.idx32)
      table_outer<uint32_t>(t, b, nb_outer);
    else
      table_outer<int64_t>(t, b, nb_outer);
  } else {
    if (t.idx32)
      table_inner<G, uint32_t>(t, b - nb_outer, (int)gridDim.x - nb_outer);
    else
      table_inner<G, int64_t>(t, b - nb_outer, (int)gridDim.x - nb_outer);
  }
}

// ---------------------------------------------------------------------------
// packed fp32 helpers (sm_100: FFMA2 / FMUL2 / FADD2)
// ---------------------------------------------------------------------------
typedef unsigned long long f2;

__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk(f2 v, float& lo, float& hi) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2 fmul2(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float rcpa(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// G hidden units -> (num, den) with sum_g 1/d_g = num/den.
template <int G>
__device__ __forceinline__ void combine(const f2 (&d)[G], f2& num, f2& den);
template <>
__device__ __forceinline__ void combine<1>(const f2 (&d)[1], f2& num, f2& den) {
  num = pk(1.0f, 1.0f);
  den = d[0];
}
template <>
__device__ __forceinline__ void combine<2>(const f2 (&d)[2], f2& num, f2& den) {
  num = fadd2(d[0], d[1]);
  den = fmul2(d[0], d[1]);
}
template <>
__device__ __forceinline__ void combine<3>(const f2 (&d)[3], f2& num, f2& den) {
  const f2 s = fadd2(d[0], d[1]);
  const f2 p = fmul2(d[0], d[1]);
  // den then num with d2 in the same (first) operand slot: the second
  // instruction takes d2 from the operand reuse cache (register-bank reads,
  // see group_step)
  den = fmul2(d[2], p);
  num = ffma2(d[2], s, p);
}

template <>
__device__ __forceinline__ void combine<4>(const f2 (&d)[4], f2& num, f2& den) {
  // 1/d0 + 1/d1 + 1/d2 + 1/d3 = (s01*p23 + s23*p01) / (p01*p23)
  const f2 s01 = fadd2(d[0], d[1]);
  const f2 p01 = fmul2(d[0], d[1]);
  const f2 s23 = fadd2(d[2], d[3]);
  const f2 p23 = fmul2(d[2], d[3]);
  num = ffma2(s23, p01, fmul2(s01, p23));
  den = fmul2(p01, p23);
}

// Per-thread factors of one group of G units: exp(-B')/w' of the thread's
// two inners for each unit, stored thread-contiguously (k_table_tiles layout,
// slot x*kInner + s) so that unit x's pair (inner 0, inner 1) is one aligned
// 64-bit register pair (1/w' comes from the parameter block, see group_step).
static_assert(kInner == 2, "the sweep packs the thread's two inners into one f32x2 register");
template <int G>
__device__ __forceinline__ void load_group(const float4* pe, f2 (&eb)[G]) {
  constexpr int W = ebw_of(G);
  f2 f[2 * W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(pe) + w);
    f[2 * w] = v.x;
    f[2 * w + 1] = v.y;
  }
#pragma unroll
  for (int x = 0; x < G; ++x) eb[x] = f[x];
}

// One group of G units for all kInner x OBU configurations of the thread.
// Packing: one f32x2 register holds the thread's TWO INNERS of one outer, so
//   d' = exp(-B')/w' (pair, per thread) * exp(-A') (scalar, broadcast LDS) + 1/w' (uniform)
// is ONE FFMA2 that reads three vector registers (the pair and the scalar):
// 1/w' comes from the kernel's parameter block through a uniform register.
// That matters because the FMA pipe's issue cost is max(2 cycles, distinct
// even / odd source registers read) per FFMA2 (B300_MICROARCH.md, "RF
// banking"): round 1's packing (two OUTERS per register, 1/w' and exp(-B')/w'
// as vector scalars) read 3 even or 3 odd registers in most of these FFMA2s
// and lost ~17 % of the FMA pipe (tools/sass_rf.py).
// Then the G-term rational combination, two reciprocals, one accumulate.
// (Tried: ONE reciprocal per register pair, r = 1/(den_0*den_1), acc +=
// (num_0*den_1, num_1*den_0)*r -- half the MUFU work for 3 + 1/(2G) instead
// of 3 - 1/G FMA-pipe lane-ops per unit: 5.46 vs 4.90 ms on the 10^8 space,
// the FMA pipe then saturates at ~80 % on its own (profiles/r02_sweep_pair_ab.jsonl).)
//
// OBU: the outers of the item this thread evaluates (kOB, or a part of the
// item in the tail launch); E points at the first of them in each unit row.
template <int G, int OBU>
__device__ __forceinline__ void group_step(f2 (&acc)[OBU], const float* E, const f2 (&eb)[G],
                                           const SweepArgs& a, int ug) {
  static_assert(OBU == 2 || OBU % 4 == 0, "outers per part: 2 or a multiple of 4");
  constexpr int NO = OBU >= 4 ? 4 : OBU;   // outers per exp(-A') load
#pragma unroll
  for (int q = 0; q < (OBU + 3) / 4; ++q) {
    float ea[G][4];
#pragma unroll
    for (int x = 0; x < G; ++x) {
      if (OBU >= 4) {
        const float4 t = *reinterpret_cast<const float4*>(E + x * kOB + 4 * q);
        ea[x][0] = t.x, ea[x][1] = t.y, ea[x][2] = t.z, ea[x][3] = t.w;
      } else {
        const float2 t = *reinterpret_cast<const float2*>(E + x * kOB);
        ea[x][0] = t.x, ea[x][1] = t.y, ea[x][2] = 0.f, ea[x][3] = 0.f;
      }
    }
    {
      // the outers of one exp(-A') load, unit-major: the FFMA2s of a unit share
      // eb / 1/w' (2 at a time: 4.90 ms; 4 at a time: 4.79 ms on the 10^8 case)
      f2 d[NO][G];
#pragma unroll
      for (int x = 0; x < G; ++x)
#pragma unroll
        for (int j = 0; j < NO; ++j) d[j][x] = ffma2(eb[x], pk(ea[x][j], ea[x][j]), pk(a.uc[ug + x], a.uc[ug + x]));
#pragma unroll
      for (int j = 0; j < NO; ++j) {
        f2 num, den;
        combine<G>(d[j], num, den);
        float d0, d1;
        upk(den, d0, d1);
        f2& ac = acc[4 * q + j];
        const f2 r = pk(rcpa(d0), rcpa(d1));
        ac = (G == 1) ? fadd2(ac, r) : ffma2(num, r, ac);
      }
    }
  }
}

__device__ __forceinline__ void gappend(const SweepArgs& a, int64_t idx, float v) {
  const uint32_t slot = atomicAdd(a.g_count, 1u);
  if (slot < a.cap) {
    a.g_cidx[slot] = idx;
    a.g_cval[slot] = v;
  }
}

__device__ __forceinline__ void lower_threshold(const SweepArgs& a, uint32_t* s_th, uint32_t nth_key) {
  // new threshold = (m-th best) + band, rounded up so it stays an upper bound
  const uint32_t nk = fkey(__fadd_ru(fkey_inv(nth_key), a.band));
  if (threadIdx.x == 0) {
    // only thread 0 touches s_th here (volatile: the compiler may not widen
    // or hoist this load into the other threads, where it would race with
    // the store below -- compute-sanitizer racecheck)
    if (nk < *reinterpret_cast<volatile uint32_t*>(s_th)) {
      *s_th = nk;
      atomicMin(a.g_theta, nk);
    }
  }
}

// byte offset of the second exp(-A') tile buffer (the next item's tile lands
// there by cp.async while the current item computes)
__host__ __device__ inline size_t ea2_offset(int k, int sb) {
  const size_t KH = (size_t)k * kH;
  const size_t b = KH * kOB * 4 + (size_t)sb * (8 + 4) + 256 * 4;
  return (b + 15) & ~(size_t)15;
}

size_t sweep_smem(int k, int sb) {
  const size_t KH = (size_t)k * kH;
  return ea2_offset(k, sb) + KH * kOB * 4;   // ... + the second exp(-A') buffer
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// ---------------------------------------------------------------------------
// the sweep
//
// One persistent CTA of kThreads = 1024 threads per SM (64 registers, 32
// warps); a work item is kOB = 8 outer x kInnerBlock = 2048 inner
// configurations. Thread t owns inners {t, t + 1024} of the block and all 8
// outers, so every broadcast LDS.128 of exp(-A') feeds 2 x 4 configurations
// and every per-thread exp(-B')/w' register pair feeds 8. acc[o] holds the
// f32x2 pair (inner 0, inner 1) of outer o. (Tile constants: kernels.cuh,
// overridable for A/B builds with tools/build_variants.sh.)
// ---------------------------------------------------------------------------
// NT: threads per CTA. NT = kThreads: one CTA per SM, a CTA owns whole work
// items. NT = kThreads / 2: two CTAs per SM, each owning one HALF of an item
// (layout threads [h*NT, h*NT + NT) of the inner block; same per-thread work
// and table layout): used for short slices, where the last wave of whole
// items would leave SMs idle -- a straggler CTA then has its SM to itself.
//
// OBU: outers per work unit. kOB = whole items; smaller in the TAIL launch,
// which splits the last, partial wave's items into kOB / OBU parts so that
// wave ends with a short round instead of a full item-time on a few SMs.
template <int G, bool PRUNE, int SB, int NT, int OBU>
__global__ void __launch_bounds__(NT, MLT_MINB * (kThreads / NT)) k_sweep(SweepArgs a) {
  // SB: per-CTA candidate slots (kSB; kSBBig for m > kMaxTopMSmall)
  constexpr int kSB = SB;
  constexpr int kSBLimit = SB * 3 / 4;
  constexpr int HALVES = kThreads / NT;   // CTA work units per item (inner halves)
  constexpr int PARTS = kOB / OBU;        // ... (outer parts)
  constexpr int SUB = HALVES * PARTS;
  static_assert(!PRUNE || OBU == kOB, "the pruned sweep works on whole items");
  extern __shared__ __align__(16) unsigned char smraw[];
  const int KH = a.k * kH;
  float* s_ea = reinterpret_cast<float*>(smraw);                 // [KH][kOB]
  int64_t* s_bidx = reinterpret_cast<int64_t*>(s_ea + (size_t)KH * kOB);
  float* s_bval = reinterpret_cast<float*>(s_bidx + kSB);
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(s_bval + kSB);
  float* s_ea2 = reinterpret_cast<float*>(smraw + ea2_offset(a.k, SB));   // [KH][kOB], the other tile buffer
  __shared__ int s_n, s_tot;
  __shared__ unsigned int s_work;   // pruning: groups evaluated by the warps of this item
  __shared__ uint32_t s_th, s_sel[2], s_wsum[NT / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
    s_n = 0;
    s_th = *reinterpret_cast<volatile uint32_t*>(a.g_theta);
  }
  const int ngroups = KH / G;
  const int n_items = (a.item_hi - a.item_lo) * SUB;   // CTA work units of this launch
  constexpr int kV = kInner * OBU;   // configurations per thread per work unit (16)

  __shared__ __align__(16) float s_cr[kOB * kMaxCk];   // pruning: cst + remaining-unit lower bound per outer, checkpoint
  // pruning makes work items uneven: they are handed out dynamically then
  __shared__ int s_next;
  if (PRUNE && tid == 0) s_next = atomicAdd(a.g_next, 1);
  int pf_ob = -1, pf_buf = 0, cur = 0;   // prefetched outer block, its buffer; the buffer in use
  for (int w = PRUNE ? -1 : (int)blockIdx.x; ; w = PRUNE ? w : w + (int)gridDim.x) {
    if (PRUNE) {
      __syncthreads();
      w = s_next;
      __syncthreads();
      if (tid == 0 && w < n_items) s_next = atomicAdd(a.g_next, 1);
    }
    if (w >= n_items) break;
    // pruning visits work items best-first (ascending lower bound of their
    // mean log time), so the threshold reaches its final value within the first wave
    const int half = HALVES == 1 ? 0 : w % HALVES;
    const int part = PARTS == 1 ? 0 : (w / HALVES) % PARTS;
    const int wi = PRUNE ? __ldg(a.item_order + w / SUB) : a.item_lo + w / SUB;
    const int ob = wi / a.n_ib, ib = wi - ob * a.n_ib;
    const int tl = half * NT + tid;   // this thread's column of the item's (layout) thread block
    __syncthreads();
    if (PRUNE) {
      for (int q = tid; q < kOB * a.n_ck; q += NT) {   // s_cr[checkpoint][outer]
        const int c = q / kOB, r = q - c * kOB;
        s_cr[q] = a.cst + __ldg(a.remlo + (((size_t)ob * kOB + r) * a.n_ib + ib) * a.n_ck + c);
      }
      __syncthreads();
      // checkpoint 0 (no unit evaluated): the item's lower bound alone decides
      const float thf = fkey_inv(*reinterpret_cast<volatile uint32_t*>(&s_th)) + a.prune_eps;
      bool above = true;
#pragma unroll
      for (int r = 0; r < kOB; ++r) above = above && s_cr[r] > thf;
      if (__syncthreads_and(above)) {
        // Items come in ascending order of exactly this bound (min over the rows
        // of cst + remlo[checkpoint 0], rounded monotonically) and θ only falls:
        // every later item fails the same test, so stop handing items out.
        if (tid == 0) atomicMax(a.g_next, n_items);
        break;
      }
    }
    if (pf_ob == ob) {
      // this outer block's exp(-A') tile was prefetched during the previous item
      cur = pf_buf;
      cp_async_wait<0>();   // (visible to every thread after the barrier below)
    } else {  // stage it now: [KH][kOB] floats, contiguous in global
      cp_async_wait<0>();   // no prefetch may still be landing in the buffer
      cur = 0;
      const float4* src = reinterpret_cast<const float4*>(a.ea + (size_t)ob * KH * kOB);
      float4* dst = reinterpret_cast<float4*>(s_ea);
      for (int q = tid; q < KH * kOB / 4; q += NT) dst[q] = __ldg(src + q);
    }
    if (tid == 0) {
      s_tot = 0;
      s_work = 0;
      const uint32_t g = *reinterpret_cast<volatile uint32_t*>(a.g_theta);
      if (g < s_th) s_th = g;
    }
    __syncthreads();

    const float* s_cur = cur ? s_ea2 : s_ea;
    // Prefetch the next item's tile into the other buffer (cp.async, no wait):
    // full sweep 5.00 -> 4.92 ms on the 10^8 case. Not in the pruned sweep,
    // where the next item is often rejected at checkpoint 0 (2.483 -> 2.496 ms).
    if (!PRUNE) {
      const int wn = w + (int)gridDim.x;
      pf_ob = -1;
      if (wn < n_items) {
        const int obn = (a.item_lo + wn / SUB) / a.n_ib;
        if (obn == ob) {
          pf_ob = ob;
          pf_buf = cur;
        } else {
          const float4* src = reinterpret_cast<const float4*>(a.ea + (size_t)obn * KH * kOB);
          float* dst = cur ? s_ea : s_ea2;
          for (int q = tid; q < KH * kOB / 4; q += NT) cp_async16(dst + 4 * q, src + q);
          cp_async_commit();
          pf_ob = obn;
          pf_buf = cur ^ 1;
        }
      }
    }

    const int64_t ibase = (int64_t)ib * kInnerBlock + tl;      // inner s is ibase + s*kThreads
    bool pruned = false;   // this WARP's configurations are all provably above the threshold
    int done = ngroups;    // groups this warp evaluated
    f2 acc[OBU];   // acc[o] = (inner 0, inner 1) of outer o
#pragma unroll
    for (int o = 0; o < OBU; ++o) acc[o] = 0ull;

    constexpr int W = ebw_of(G);
    const size_t gstride = (size_t)kThreads * W;   // float4s per group
    const float4* pe = reinterpret_cast<const float4*>(a.ebp) + ((size_t)ib * ngroups * kThreads + tl) * W;
    int ug = 0;                              // first unit of the current group (1/w': a.uc[ug + x])
    const float* E = s_cur + part * OBU;     // exp(-A') rows of the current group (this part's outers)
    {
      // Three register sets (A, B, C) rotate so the next two groups' per-thread
      // factors are in flight from L2 while the current group computes. (With
      // two sets ptxas hoists the reload of a set above its last use and
      // renames through ~10 IMAD.MOVs per loop trip on the FMA pipe: 4.79 ->
      // 4.62 ms.) Pruning checkpoints sit on multiples of kSweepStep groups.
      // (Loading the next trip's 1/w' one trip ahead: ptxas sinks the LDCUs to
      // the loop end anyway, 4.75 ms.)
      static_assert(kSweepStep == 3, "the loop below steps three groups");
      f2 ebA[G], ebB[G], ebC[G];
      load_group<G>(pe, ebA);
      int ck = PRUNE ? 1 : 0;     // checkpoint 0 was decided before staging
      uint32_t gth = PRUNE ? *reinterpret_cast<volatile uint32_t*>(a.g_theta) : 0u;
#pragma unroll 1
      for (int gi = 0; gi < ngroups; gi += kSweepStep) {
        if (PRUNE && ck < a.n_ck && gi == a.ck_group[ck]) {
          // Every configuration of this warp provably above the threshold? The
          // decision is per warp (no block barrier): a warp whose 32 x kV
          // configurations are excluded stops and leaves its issue slots to
          // the others. The global threshold is read live: other CTAs lower it.
          // (the global value was loaded at the previous checkpoint: its L2
          // latency hides behind the groups in between)
          const uint32_t tk = min(*reinterpret_cast<volatile uint32_t*>(&s_th), gth);
          gth = *reinterpret_cast<volatile uint32_t*>(a.g_theta);
          const float thf = fkey_inv(tk) + a.prune_eps;
          static_assert(kOB % 4 == 0, "checkpoint bounds are read as float4");
          float cr[kOB];   // this checkpoint's bounds of the outers: broadcast LDS.128s
#pragma unroll
          for (int r = 0; r < kOB; r += 4)
            *reinterpret_cast<float4*>(cr + r) = *reinterpret_cast<const float4*>(s_cr + ck * kOB + r);
          bool above = true;
#pragma unroll
          for (int o = 0; o < OBU; ++o) {
            float lo, hi;
            upk(acc[o], lo, hi);
            above = above && (lo + cr[o] > thf) && (hi + cr[o] > thf);
          }
          ++ck;
          if (__all_sync(0xffffffffu, above)) {
            pruned = true;
            done = gi;
            break;
          }
        }
        // No bounds selects: the tables carry padding groups past the end
        // (ebp allocation), so the prefetches of groups gi + 1 / gi + 2 / gi + 3
        // near the end read valid memory they never use; group counts that are
        // not multiples of 3 end below.
        if (gi + 1 >= ngroups) {
          group_step<G, OBU>(acc, E, ebA, a, ug);
          break;
        }
        load_group<G>(pe + gstride, ebB);
        if (gi + 2 >= ngroups) {
          group_step<G, OBU>(acc, E, ebA, a, ug);
          group_step<G, OBU>(acc, E + G * kOB, ebB, a, ug + G);
          break;
        }
        load_group<G>(pe + 2 * gstride, ebC);
        group_step<G, OBU>(acc, E, ebA, a, ug);
        load_group<G>(pe + 3 * gstride, ebA);
        group_step<G, OBU>(acc, E + G * kOB, ebB, a, ug + G);
        group_step<G, OBU>(acc, E + 2 * G * kOB, ebC, a, ug + 2 * G);
        pe += 3 * gstride;
        ug += 3 * G;
        E += 3 * G * kOB;
      }
    }

    if (PRUNE) {
      if (lane == 0) atomicAdd(&s_work, (unsigned int)done);
      const bool all_pruned = __syncthreads_and(pruned);
      if (tid == 0) atomicAdd(a.g_work, (unsigned long long)s_work);
      if (all_pruned) continue;   // no configuration of this item can be kept
    }

    // ---- candidates: bit (s*kOB + r) <-> inner s, outer r -----------------------
    float v[kV];
#pragma unroll
    for (int o = 0; o < OBU; ++o) {
      upk(acc[o], v[o], v[OBU + o]);
      v[o] += a.cst;
      v[OBU + o] += a.cst;
    }
    const int64_t obase = a.o_lo + (int64_t)ob * kOB + part * OBU;
    auto cfg_index = [&](int b) -> int64_t {
      return (obase + (b % OBU)) * a.c_in + ibase + (b / OBU) * kThreads;
    };
    uint32_t mask = 0;
    {
      const float thf = fkey_inv(s_th);
#pragma unroll
      for (int b = 0; b < kV; ++b) {
        const int64_t i = ibase + (b / OBU) * kThreads;
        const int64_t idx = cfg_index(b);
        const bool in = i < a.c_in && idx >= a.begin && idx < a.end;
        if (in && !(PRUNE && pruned) && !(v[b] > thf)) mask |= 1u << b;   // NaN passes (never silently dropped)
      }
    }
    if (a.check_rules && mask) {
#pragma unroll 1
      for (int b = 0; b < kV; ++b) {
        if (mask & (1u << b)) {
          int dig[kMaxP];
          decode_digits(a.sp, (uint64_t)cfg_index(b), dig);
          if (!rules_ok(a.sp, dig)) mask &= ~(1u << b);
        }
      }
    }
    // s_n is read BEFORE the barrier: after it, a fast warp may already be
    // appending (atomicAdd on s_n) while a slow one evaluates the refine
    // condition -- with a live read the two could disagree and diverge at the
    // block_select barriers (compute-sanitizer synccheck)
    const int n_held = s_n;
    {
      int c = __popc(mask);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0 && c) atomicAdd(&s_tot, c);
    }
    __syncthreads();
    if (n_held + s_tot > kSBLimit && s_tot >= a.m) {
      // too many pass: the m-th best of this work item bounds the global m-th best
      const uint32_t key = block_select(
          [&](auto&& f) {
#pragma unroll
            for (int b = 0; b < kV; ++b)
              if (mask & (1u << b)) f(fkey(v[b]));
          },
          a.m, s_hist, s_sel);
      lower_threshold(a, &s_th, key);
      __syncthreads();
      const float thf = fkey_inv(s_th);
#pragma unroll
      for (int b = 0; b < kV; ++b)
        if (v[b] > thf) mask &= ~(1u << b);
    }
    {  // append: warp-aggregated slot reservation
      const int c = __popc(mask);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int base = 0;
      if (lane == 31 && incl) base = atomicAdd(&s_n, incl);
      base = __shfl_sync(0xffffffffu, base, 31) + incl - c;
#pragma unroll
      for (int b = 0; b < kV; ++b) {
        if (mask & (1u << b)) {
          const int64_t idx = cfg_index(b);
          if (base < kSB) {
            s_bidx[base] = idx;
            s_bval[base] = v[b];
          } else {
            gappend(a, idx, v[b]);
          }
          ++base;
        }
      }
    }
    __syncthreads();
    if (s_n > kSBLimit) {
      // compact the CTA buffer around its own m-th best
      const int n = min(s_n, kSB);
      if (n >= a.m) {
        const uint32_t key = block_select(
            [&](auto&& f) {
              for (int e = tid; e < n; e += NT) f(fkey(s_bval[e]));
            },
            a.m, s_hist, s_sel);
        lower_threshold(a, &s_th, key);
        __syncthreads();
      }
      const float thf = fkey_inv(s_th);
      constexpr int kPer = (kSB + NT - 1) / NT;   // any block size (768: 3 slots per thread)
      int64_t ki[kPer];
      float kv[kPer];
      uint32_t keep = 0;
#pragma unroll
      for (int e = 0; e < kPer; ++e) {
        const int slot = tid * kPer + e;
        if (slot < n) {
          ki[e] = s_bidx[slot];
          kv[e] = s_bval[slot];
          if (!(kv[e] > thf)) keep |= 1u << e;
        }
      }
      const int c = __popc(keep);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_wsum[warp] = incl;
      __syncthreads();
      int off = incl - c, total = 0;
      for (int q = 0; q < NT / 32; ++q) {
        if (q < warp) off += s_wsum[q];
        total += s_wsum[q];
      }
#pragma unroll
      for (int e = 0; e < kPer; ++e) {
        if (keep & (1u << e)) {
          s_bidx[off] = ki[e];
          s_bval[off] = kv[e];
          ++off;
        }
      }
      __syncthreads();
      if (total > kSBLimit) {  // a crowded band: spill everything to the global buffer
        for (int e = tid; e < total; e += NT) gappend(a, s_bidx[e], s_bval[e]);
        total = 0;
      }
      if (tid == 0) s_n = total;
    }
  }
  __syncthreads();
  cp_async_wait<0>();   // a prefetch for an item this CTA never ran
  {  // final flush of this CTA's candidates, against the freshest global threshold
    const uint32_t g = *reinterpret_cast<volatile uint32_t*>(a.g_theta);
    const float thf = fkey_inv(min(s_th, g));
    const int n = min(s_n, kSB);
    for (int e = tid; e < n; e += NT)
      if (!(s_bval[e] > thf)) gappend(a, s_bidx[e], s_bval[e]);
  }
}

template __global__ void k_table_tiles<1>(TableArgs t, int nb_outer);
template __global__ void k_table_tiles<2>(TableArgs t, int nb_outer);
template __global__ void k_table_tiles<3>(TableArgs t, int nb_outer);
template __global__ void k_table_tiles<4>(TableArgs t, int nb_outer);
// every G of the host's dispatch table (abi.cu) for each instance shape
// (MLT_SWEEP_INSPECT: only the default full-sweep instance, for SASS inspection)
#ifdef MLT_SWEEP_INSPECT
template __global__ void k_sweep<3, false, kSB, kThreads, kOB>(SweepArgs);
#else
#define MLT_SWEEP_ROW(PR, SBV, NTV, OB)                            \
  template __global__ void k_sweep<1, PR, SBV, NTV, OB>(SweepArgs); \
  template __global__ void k_sweep<2, PR, SBV, NTV, OB>(SweepArgs); \
  template __global__ void k_sweep<3, PR, SBV, NTV, OB>(SweepArgs); \
  template __global__ void k_sweep<4, PR, SBV, NTV, OB>(SweepArgs);
MLT_SWEEP_ROW(false, kSB, kThreads, kOB)
MLT_SWEEP_ROW(true, kSB, kThreads, kOB)
MLT_SWEEP_ROW(false, kSBBig, kThreads, kOB)
MLT_SWEEP_ROW(true, kSBBig, kThreads, kOB)
MLT_SWEEP_ROW(false, kSB, kThreads / 2, kOB)
MLT_SWEEP_ROW(true, kSB, kThreads / 2, kOB)
MLT_SWEEP_ROW(false, kSBBig, kThreads / 2, kOB)
MLT_SWEEP_ROW(true, kSBBig, kThreads / 2, kOB)
MLT_SWEEP_ROW(false, kSB, kThreads, 2)
MLT_SWEEP_ROW(false, kSBBig, kThreads, 2)
MLT_SWEEP_ROW(false, kSB, kThreads, 4)
MLT_SWEEP_ROW(false, kSBBig, kThreads, 4)
#undef MLT_SWEEP_ROW
#endif

}  // namespace mlt
