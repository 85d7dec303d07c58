// kernels.cuh — declarations shared by the kernel translation units and the
// host-side C-ABI implementation (abi.cu).
#pragma once

#include "common.cuh"
#include "select.cuh"

namespace mlt {

// ---- exact fp64 kernels (predict.cu) --------------------------------------
__global__ void k_decode(DSpace s, const int64_t* idx, int64_t n, int64_t* out);
__global__ void k_valid(DSpace s, const int64_t* idx, int64_t n, uint8_t* out);
__global__ void k_valid_range(DSpace s, int64_t lo, int64_t n, uint8_t* out);
__global__ void k_encode(DEns e, const int64_t* idx, int64_t n, double* out);
__global__ void k_predict64(DEns e, DSpace s, int check_rules, int64_t begin, const int64_t* idx,
                            const double* feat, int64_t n, double* pred, int64_t* idx_out,
                            const float* band_v, float band_theta, int staged);
__global__ void k_member_out64(DEns e, const double* feat, int64_t n, double* out, int staged);
size_t predict64_smem(const DEns& e);
__global__ void k_rescore(DEns e, const int64_t* idx, const uint32_t* n_ptr, double* pred);

// ---- analytic surrogate device (surrogate.cu) -------------------------------
struct DSurr {
  double base;                  // base_time
  double sigma;                 // log-time noise std (0 = noise-free)
  uint64_t seed;
  int T;                        // terms
  int reps;                     // 0 = true times; >= 1 = measured (min over reps of the noise)
  const int* tpos;              // [T][2] parameter positions (second -1 for one-parameter terms)
  const int* tdig;              // [T][2] matched DIGITS (-1: the value is not in the list, never hits)
  const double* tfac;           // [T]
};
struct SurrPart {
  double t;
  int64_t i;
  int64_t n_valid, n_below;
};
__global__ void k_surr_times(DSpace lr, DSurr su, const int64_t* idx, int64_t n, double* times, uint8_t* ok);
__global__ void k_surr_best(DSpace sp, DSpace lr, DSurr su, int64_t begin, int64_t end, double thr, SurrPart* part);
__global__ void k_surr_best_runs(DSpace sp, DSpace lr, DSurr su, const uint64_t* gmask, int nm, uint64_t b_ones, int64_t begin,
                                 int64_t end, int run, double thr, SurrPart* part);
__global__ void k_surr_times_masks(DSpace lr, DSurr su, const uint64_t* gmask, int nm, uint64_t b_ones,
                                   const int64_t* idx, int64_t n, double* times, uint8_t* ok);
__global__ void k_surr_best_final(const SurrPart* part, int n, SurrPart* out);

// ---- final guard-band stage (select.cu) ------------------------------------
constexpr int kSmallSort = 8192;  // survivors sorted in one CTA's shared memory (128 KB)
constexpr int kRankSort = 256;    // ... by rank counting up to this many, bitonic above
__global__ void k_band_filter(const int64_t* cidx, const float* cval, const uint32_t* count_ptr, uint32_t cap, int m,
                              float band, int64_t* out_idx, float* out_val, uint32_t* out_n);
__global__ void k_sort_small(const double* pred, const int64_t* idx, const uint32_t* n_ptr, int m, double* out_pred,
                             int64_t* out_idx, uint32_t* status, int cap, uint32_t* host_out = nullptr,
                             const uint32_t* gs = nullptr, int64_t* rec = nullptr, uint32_t cand_cap = 0);
// entries of k_sort_small's shared buffer for at most n survivors (power of two, >= 256)
inline int sort_small_cap(int64_t n) {
  int c = 256;
  while (c < n && c < kSmallSort) c <<= 1;
  return c;
}

// ---- fp32 factored sweep (sweep.cu) ---------------------------------------
#ifndef MLT_THREADS
#define MLT_THREADS 1024
#endif
#ifndef MLT_INNER
#define MLT_INNER 2
#endif
#ifndef MLT_OB
#define MLT_OB 8
#endif
#ifndef MLT_MINB
#define MLT_MINB 1
#endif
constexpr int kThreads = MLT_THREADS;   // threads per sweep CTA
constexpr int kInner = MLT_INNER;   // inner configurations per thread (share every exp(-A') load)
constexpr int kInnerBlock = kThreads * kInner;   // inner configurations per work item
constexpr int kOB = MLT_OB;         // outer configurations per work item (per thread)

// float4s per thread per group in the thread-contiguous exp(-B')/w' layout
__host__ __device__ constexpr int ebw_of(int G) { return (kInner * G + 3) / 4; }
#ifndef MLT_DEFAULT_GROUP
#define MLT_DEFAULT_GROUP 3
#endif
constexpr int kDefaultGroup = MLT_DEFAULT_GROUP;   // units per shared reciprocal unless MLT_OPT_GROUP says otherwise
constexpr int kSB = kThreads >= 512 ? 2 * kThreads : 1024;   // per-CTA guard-band candidate slots
constexpr int kSBBig = 8192;   // ... in the instance for large m (kMaxTopMSmall < m <= kMaxTopM)
constexpr int kMaxTopMSmall = 1024;  // largest m of the default sweep instance
constexpr int kMaxTopM = 4096;       // largest m served by the guard-band path (kSBBig instance)
constexpr int kMaxCk = 32;      // pruning checkpoints per work item
constexpr int kSweepStep = 3;   // groups per trip of the sweep's inner loop (checkpoints sit on multiples)
constexpr int kMaxUnitsParam = 4096;   // k*kH (+ 2 groups of padding) the sweep's parameter block holds

struct SweepArgs {
  int k;                        // members
  const float* ea;              // [n_ob][k*kH][kOB]  exp(-A') of outer configurations
  const float* ebp;             // [n_ib][group][thread][4*ebw] exp(-B') / w' of inner configurations
  int64_t c_in, c_in_pad;       // inner cardinality (and padded to kThreads)
  int64_t o_lo;                 // outer index of ea block 0, row 0
  int n_ob, n_ib;               // outer blocks x inner blocks = work items
  int item_lo, item_hi;         // the work items [item_lo, item_hi) of this launch (row-major over (ob, ib))
  int64_t begin, end;           // configuration range of this call
  float cst;                    // sum_m (b2*std + mean)/k - (#dummy units)
  float band;                   // 2*delta (rounded up)
  int m;
  uint32_t* g_theta;            // ordered-key threshold (atomicMin)
  uint32_t* g_count;            // candidates appended (may exceed cap -> overflow)
  int64_t* g_cidx;
  float* g_cval;
  uint32_t cap;
  int check_rules;
  // optional exact pruning (MLT_OPT_PRUNE): at group ck_group[c] a work item is
  // abandoned when every configuration's partial sum + cst + a lower bound of
  // the remaining units (remlo, per outer) exceeds the threshold by prune_eps
  int prune, n_ck;
  int ck_group[kMaxCk];
  const float* remlo;           // [outer - o_lo][inner block][n_ck] lower bound of the units still to come
  float prune_eps;
  const int* item_order;        // pruning: work items best-first (ascending lower bound)
  unsigned long long* g_work;   // pruning: groups evaluated, summed over work items
  int* g_next;                  // pruning: next work item (dynamic distribution)
  DSpace sp;
  // 1/w' of every table position (+ padding), read through the constant bank:
  // the sweep's FFMA2s take it as a uniform-register operand, which costs no
  // vector register-file bank read (kernel parameter space, per launch).
  float uc[kMaxUnitsParam];
};

// Tables of the factored first layer (sweep.cu).
// Tables of the factored first layer. exp(-z) factorises over parameters:
//   F[mj][p][digit] = exp(-W1[mj][p] * x_p(digit))           (k_table_factors, once per plan)
//   Ea(outer) = ca[mj] * prod_{p <  split} F[mj][p][digit_p]  ca = exp(-(b1 - c))
//   Eb'(inner) = cb[mj] * prod_{p >= split} F[mj][p][digit_p] cb = exp(-c) / w'
// so every table entry is a handful of fp64 multiplies (no exp), rounded once to fp32.
// Division by a per-launch constant: q = umulhi64(x, ceil(2^64 / d)) is exact
// for x < 2^32 and 2 <= d < 2^32 (the error term stays below 1 / d); other
// operands take the plain division. ~4 instructions instead of a ~20-60
// instruction division sequence in the table kernels' index math.
struct FDiv {
  uint64_t m;   // ceil(2^64 / d), 0 when d < 2
  int64_t d;
};
inline FDiv make_fdiv(int64_t d) {
  FDiv f;
  f.d = d;
  f.m = (d >= 2 && d < (int64_t(1) << 32)) ? (~0ull / (uint64_t)d) + 1 : 0;
  return f;
}
__device__ __forceinline__ int64_t fdiv(int64_t x, const FDiv& f) {
  // floor(x * m / 2^64) for x < 2^32 in two 32-bit multiplies: x * m_hi
  // (m < 2^63, so no overflow) plus the high word of x * m_lo, shifted
  if (f.m && (uint64_t)x <= 0xffffffffull) {
    const uint32_t x32 = (uint32_t)x;
    return (int64_t)(((uint64_t)x32 * (uint32_t)(f.m >> 32) + __umulhi(x32, (uint32_t)f.m)) >> 32);
  }
  return x / f.d;
}

struct TableArgs {
  int k, d, h, split;           // params [0, split) are outer, [split, d) inner
  int G;                        // units per reciprocal group of the sweep (inner-table layout)
  int radix[kMaxP];
  int foff[kMaxP + 1];          // offset of parameter p's digits in a row of F
  const double* w1;             // [k][h][d]
  const int* unit_of;           // [k*kH] original unit (m*kH + j) of each table position
  double* F;                    // [k*kH][foff[d]]  (position order)
  const double* ca;             // [k*kH]
  const double* cb;             // [k*kH]  (0 for dummy units)
  const double* wprime;         // [k*kH]  w2*std/k (0 for dummy units)
  int n_ib;                     // inner blocks of kInnerBlock inners
  int idx32;                    // every outer / inner table index of this build < 2^31 (32-bit index math)
  int64_t o_lo, o_card, c_in, c_in_pad;   // o_card = number of outer configurations
  // two-level split of each table: entry = const * P_hi[index / nlo] * P_lo[index % nlo]
  const double *PoH, *PoL, *PiH, *PiL;    // [k*kH][n_hi] / [k*kH][n_lo]
  int64_t o_nlo, o_nhi, o_hi_base, i_nlo, i_nhi;
  int n_ob;
  FDiv f_radix[kMaxP], f_kh, f_onlo, f_inlo, f_ngroups;   // fast divisions (make_fdiv of the above)
  float* ea;
  float* ebp;
};

__global__ void k_table_factors(TableArgs t);
struct PartialJobs {             // k_table_partial4: four (parameter range, sub-index range) tables
  int p_lo[4], p_hi[4];
  int64_t base[4], count[4];
  FDiv f_count[4];
  double* out[4];
};
__global__ void k_table_partial4(const __grid_constant__ TableArgs t, const __grid_constant__ PartialJobs j);
struct CkList {
  int n;
  int unit[kMaxCk];             // first table position still to come at checkpoint c
  double mag[kMaxCk];           // sum over positions >= unit[c] of |w'| (1 for dummy units)
};
__global__ void k_table_ebext(TableArgs t, double* ext);
__global__ void k_item_keys(const float* remlo, int n_ck, int n_ib, int items, float* keys, int* vals);
// best-first item order for <= kItemSortMax items: sorted runs, then a rank merge
constexpr int kItemSortThreads = 1024, kItemSortMax = 8192, kItemRun = 1024, kItemRunThreads = 256;
__global__ void k_item_runs(const float* remlo, int n_ck, int n_ib, int items, unsigned* run_key, int* run_val);
__global__ void k_item_merge(const unsigned* run_key, const int* run_val, int items, int* order);
__global__ void k_table_rem(TableArgs t, CkList ck, const double* ext, float* remlo);
template <int G>
__global__ void k_table_tiles(TableArgs t, int nb_outer);   // outer + inner tables, one launch

template <int G, bool PRUNE, int SB, int NT, int OBU>
__global__ void k_sweep(SweepArgs a);
size_t sweep_smem(int k, int sb);

}  // namespace mlt
