// abi.cu — host side of libmltune_b200.so: the extern "C" entry points of
// include/mltune_b200.h, device-memory management, the fp32-sweep setup
// (split choice, centring, range checks, a-priori error bound) and the
// selection (CUB radix sort by (prediction, index)).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "kernels.cuh"

using namespace mlt;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(expr)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(MLT_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),    \
                  __FILE__, __LINE__);                                                  \
  } while (0)

#define CTX_GUARD(c) std::lock_guard<std::recursive_mutex> ctx_guard_((c)->mu)

#define TRY(expr)            \
  do {                       \
    int rc_ = (expr);        \
    if (rc_ != MLT_OK) return rc_; \
  } while (0)

}  // namespace

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct mlt_ctx {
  int dev = 0;
  int sms = 148;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  bool prof = false;
  int64_t launches = 0;
  int opt_path = -1, opt_group = -1, opt_prune = 0;
  int opt_table_cache = 1;            // MLT_OPT_TABLE_CACHE
  int opt_half_items = 0;             // MLT_OPT_HALF_ITEMS
  int opt_tail_split = 1;             // MLT_OPT_TAIL_SPLIT
  int64_t chunk = int64_t(1) << 27;   // configurations per sweep chunk (MLT_OPT_CHUNK)
  int64_t cand_cap = 1 << 20;
  std::vector<void*> slots = std::vector<void*>(32, nullptr);
  std::vector<size_t> sizes = std::vector<size_t>(32, 0);
  void* pinned = nullptr;       // small pinned staging for scalars
  void* res_pin = nullptr;      // pinned landing zone of a step's top-m (prediction, index) lists
  void* merge_pin = nullptr;    // ... and of a record merge (mlt_merge_records)
  size_t merge_cap = 0;
  size_t res_cap = 0;
  void* stage = nullptr;        // pinned staging ring for plan uploads (weights, value tables)
  size_t stage_cap = 0;
  size_t stage_off = 0;         // next free byte of the ring
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_switch = nullptr;   // orders work across mlt_ctx_set_stream
  // Serialises every entry point on this context (workspace slots, pinned
  // staging and the stream are per-context state): concurrent callers of one
  // context queue instead of racing. Recursive: mlt_top_m -> mlt_plan_create.
  std::recursive_mutex mu;
  // kernel -> (dynamic shared memory last granted, resident CTAs per SM at it):
  // the attribute call and the occupancy query cost host microseconds on every
  // step otherwise, while the GPU waits for the step's first kernel
  std::map<const void*, std::pair<size_t, int>> kattr;
};

namespace {

enum Slot {
  S_SPACE_VALUES, S_SPACE_RPOS, S_SPACE_RCOEFF, S_ENS, S_IDX, S_OUT_A, S_OUT_B, S_OUT_C, S_OUT_D,
  S_EA, S_EBP, S_U, S_TAB, S_GSCAL, S_CIDX, S_CVAL, S_SORT_TMP, S_FEAT, S_TOPI, S_TOPP, S_POH, S_POL, S_PIH, S_PIL,
  S_L_VALUES, S_L_RPOS, S_L_RCOEFF, S_SURR, S_PART
};

int ws(mlt_ctx* c, int slot, size_t bytes, void** out) {
  if (bytes == 0) bytes = 16;
  if (c->sizes[slot] < bytes) {
    if (c->slots[slot]) CU(cudaFree(c->slots[slot]));
    c->slots[slot] = nullptr;
    c->sizes[slot] = 0;
    size_t want = bytes + bytes / 4;
    CU(cudaMalloc(&c->slots[slot], want));
    c->sizes[slot] = want;
  }
  *out = c->slots[slot];
  return MLT_OK;
}

template <typename T>
int ws_t(mlt_ctx* c, int slot, size_t count, T** out) {
  void* p;
  TRY(ws(c, slot, count * sizeof(T), &p));
  *out = static_cast<T*>(p);
  return MLT_OK;
}

// Plan-owned buffers come from the device's stream-ordered memory pool
// (cudaMallocAsync / cudaFreeAsync on the context stream; the pool keeps its
// memory, see mlt_ctx_create), so a per-call plan costs no cudaMalloc/cudaFree
// round trips or device-wide synchronisation.
void pool_free(mlt_ctx* c, void* ptr) {
  if (ptr) cudaFreeAsync(ptr, c->stream);
}

// Host -> device upload through the context's pinned staging ring (the
// caller's arrays are pageable), so every upload of a plan comes from pinned
// memory and is truly asynchronous.
int upload_pinned(mlt_ctx* c, void* dst, const void* src, size_t bytes) {
  // Successive uploads take successive slots of the ring, so a plan's several
  // uploads queue without host waits; the stream is synchronised only when
  // the ring wraps (every earlier copy out of it has then landed) or grows.
  if (bytes == 0) return MLT_OK;
  const size_t need = (bytes + 255) & ~(size_t)255;
  if (c->stage_cap < need) {
    CU(cudaStreamSynchronize(c->stream));
    if (c->stage) CU(cudaFreeHost(c->stage));
    c->stage = nullptr;
    c->stage_cap = 0;
    const size_t cap = std::max<size_t>(need * 2, (size_t)4 << 20);
    CU(cudaMallocHost(&c->stage, cap));
    c->stage_cap = cap;
    c->stage_off = 0;
  } else if (c->stage_off + need > c->stage_cap) {
    CU(cudaStreamSynchronize(c->stream));
    c->stage_off = 0;
  }
  char* slot = static_cast<char*>(c->stage) + c->stage_off;
  c->stage_off += need;
  std::memcpy(slot, src, bytes);
  CU(cudaMemcpyAsync(dst, slot, bytes, cudaMemcpyHostToDevice, c->stream));
  return MLT_OK;
}

int check_launch(mlt_ctx* c) {
  c->launches++;
  CU(cudaGetLastError());
  return MLT_OK;
}

// Grant `kern` `smem` bytes of dynamic shared memory (once per size) and
// return its resident CTAs per SM at `threads` threads.
template <typename K>
int kernel_smem(mlt_ctx* c, K* kern, int threads, size_t smem, int* nb_out = nullptr) {
  const void* key = reinterpret_cast<const void*>(kern);
  auto it = c->kattr.find(key);
  if (it == c->kattr.end() || it->second.first != smem) {
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int nb = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem));
    c->kattr[key] = {smem, nb};
    it = c->kattr.find(key);
  }
  if (nb_out) *nb_out = it->second.second;
  return MLT_OK;
}

int grid_for(mlt_ctx* c, int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)c->sms * 16));
}

// ---- host copies of the descriptors ---------------------------------------
struct HostSpace {
  int P = 0;
  std::vector<int> radix;
  std::vector<int64_t> values;
  std::vector<int> rkind, roff, rpos;
  std::vector<int64_t> rcoeff, rbound;
  double card = 0;              // as double for range checks
  int64_t card_i = 0;           // exact when it fits
  bool card_fits = true;
};

int read_space(const mlt_space* s, HostSpace* h) {
  if (!s) return fail(MLT_EINVAL, "space is NULL");
  if (s->n_params < 1 || s->n_params > kMaxP)
    return fail(MLT_EINVAL, "space must have 1..%d parameters, got %d", kMaxP, s->n_params);
  if (s->n_rules < 0 || s->n_rules > kMaxRules)
    return fail(MLT_EINVAL, "space must have 0..%d rules, got %d", kMaxRules, s->n_rules);
  h->P = s->n_params;
  h->radix.assign(s->radix, s->radix + h->P);
  int64_t nv = 0;
  h->card = 1;
  h->card_i = 1;
  h->card_fits = true;
  for (int p = 0; p < h->P; ++p) {
    if (h->radix[p] < 1) return fail(MLT_EINVAL, "parameter %d has an empty value list", p);
    nv += h->radix[p];
    h->card *= h->radix[p];
    if (h->card_fits && h->card_i > INT64_MAX / h->radix[p]) h->card_fits = false;
    if (h->card_fits) h->card_i *= h->radix[p];
  }
  if (!h->card_fits) return fail(MLT_EINVAL, "space cardinality exceeds 2^63");
  h->values.assign(s->values, s->values + nv);
  h->rkind.assign(s->rule_kind, s->rule_kind + s->n_rules);
  h->roff.assign(1, 0);
  int nops = 0;
  for (int r = 0; r < s->n_rules; ++r) {
    if (h->rkind[r] < 0 || h->rkind[r] > 2) return fail(MLT_EINVAL, "unknown rule kind %d", h->rkind[r]);
    nops += s->rule_nops[r];
    h->roff.push_back(nops);
  }
  if (nops > kMaxOps) return fail(MLT_EINVAL, "too many rule operands (%d > %d)", nops, kMaxOps);
  h->rpos.assign(s->rule_pos, s->rule_pos + nops);
  for (int o = 0; o < nops; ++o)
    if (h->rpos[o] < 0 || h->rpos[o] >= h->P) return fail(MLT_EINVAL, "rule operand position %d out of range", h->rpos[o]);
  h->rcoeff.assign(s->rule_coeff, s->rule_coeff + nops);
  h->rbound.assign(s->rule_bound, s->rule_bound + s->n_rules);
  return MLT_OK;
}

int upload_space(mlt_ctx* c, const HostSpace& h, DSpace* d, int base_slot_values = S_SPACE_VALUES,
                 int slot_rpos = S_SPACE_RPOS, int slot_rcoeff = S_SPACE_RCOEFF) {
  std::memset(d, 0, sizeof *d);
  d->P = h.P;
  d->R = (int)h.rkind.size();
  int off = 0;
  for (int p = 0; p < h.P; ++p) {
    d->radix[p] = h.radix[p];
    d->voff[p] = off;
    off += h.radix[p];
  }
  int64_t* vals;
  TRY(ws_t(c, base_slot_values, h.values.size(), &vals));
  CU(cudaMemcpyAsync(vals, h.values.data(), h.values.size() * 8, cudaMemcpyHostToDevice, c->stream));
  d->values = vals;
  for (int r = 0; r < d->R; ++r) {
    d->rkind[r] = h.rkind[r];
    d->rbound[r] = h.rbound[r];
  }
  for (int r = 0; r <= d->R; ++r) d->roff[r] = h.roff[r];
  int* rp;
  int64_t* rc;
  TRY(ws_t(c, slot_rpos, std::max<size_t>(1, h.rpos.size()), &rp));
  TRY(ws_t(c, slot_rcoeff, std::max<size_t>(1, h.rcoeff.size()), &rc));
  if (!h.rpos.empty()) {
    CU(cudaMemcpyAsync(rp, h.rpos.data(), h.rpos.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(rc, h.rcoeff.data(), h.rcoeff.size() * 8, cudaMemcpyHostToDevice, c->stream));
  }
  d->rpos = rp;
  d->rcoeff = rc;
  return MLT_OK;
}

struct HostEns {
  int k = 0, d = 0, h = 0;
  std::vector<int> counts;
  std::vector<double> packed;   // [w1 | b1 | w2 | b2 | mean | std]
  const double* w1() const { return packed.data(); }
  const double* b1() const { return w1() + (size_t)k * h * d; }
  const double* w2() const { return b1() + (size_t)k * h; }
  const double* b2() const { return w2() + (size_t)k * h; }
  const double* mean() const { return b2() + k; }
  const double* sd() const { return mean() + k; }
};

int read_ens(const mlt_ensemble* e, HostEns* h) {
  if (!e) return fail(MLT_EINVAL, "ensemble is NULL");
  if (e->k < 1) return fail(MLT_EINVAL, "an ensemble needs at least one member");
  if (e->d < 1 || e->d > kMaxP) return fail(MLT_EINVAL, "input dimension must be 1..%d, got %d", kMaxP, e->d);
  if (e->h < 1 || e->h > 4096) return fail(MLT_EINVAL, "bad hidden size %d", e->h);
  h->k = e->k;
  h->d = e->d;
  h->h = e->h;
  h->counts.assign(e->counts, e->counts + e->d);
  for (int p = 0; p < e->d; ++p)
    if (h->counts[p] < 1) return fail(MLT_EINVAL, "encoder parameter %d has no values", p);
  const size_t nw = (size_t)e->k * e->h * e->d, nh = (size_t)e->k * e->h;
  h->packed.resize(nw + 2 * nh + 3 * (size_t)e->k);
  double* o = h->packed.data();
  std::memcpy(o, e->w1, nw * 8);
  std::memcpy(o + nw, e->b1, nh * 8);
  std::memcpy(o + nw + nh, e->w2, nh * 8);
  std::memcpy(o + nw + 2 * nh, e->b2, (size_t)e->k * 8);
  std::memcpy(o + nw + 2 * nh + e->k, e->mean, (size_t)e->k * 8);
  std::memcpy(o + nw + 2 * nh + 2 * e->k, e->std, (size_t)e->k * 8);
  for (double x : h->packed)
    if (!std::isfinite(x)) return fail(MLT_EINVAL, "network weights must be finite");
  return MLT_OK;
}

int upload_ens(mlt_ctx* c, const HostEns& h, DEns* d, int slot = S_ENS) {
  std::memset(d, 0, sizeof *d);
  d->k = h.k;
  d->d = h.d;
  d->h = h.h;
  for (int p = 0; p < h.d; ++p) d->counts[p] = h.counts[p];
  double* buf;
  TRY(ws_t(c, slot, h.packed.size(), &buf));
  CU(cudaMemcpyAsync(buf, h.packed.data(), h.packed.size() * 8, cudaMemcpyHostToDevice, c->stream));
  const size_t nw = (size_t)h.k * h.h * h.d, nh = (size_t)h.k * h.h;
  d->w1 = buf;
  d->b1 = buf + nw;
  d->w2 = buf + nw + nh;
  d->b2 = buf + nw + 2 * nh;
  d->mean = d->b2 + h.k;
  d->std_ = d->mean + h.k;
  return MLT_OK;
}

int launch_predict64(mlt_ctx* c, const DEns& e, const DSpace& s, int check_rules, int64_t begin,
                     const int64_t* idx, const double* feat, int64_t n, double* pred, int64_t* idx_out,
                     const float* band_v = nullptr, float band_theta = 0.f) {
  if (n <= 0) return MLT_OK;
  // the weights are staged in shared memory when they fit; the packed block
  // in global memory serves wider ensembles (the packed layouts are the same)
  const int staged = predict64_smem(e) <= 200 * 1024 ? 1 : 0;
  const size_t smem = staged ? predict64_smem(e) : 0;
  CU(cudaFuncSetAttribute(k_predict64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int nb = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_predict64, 128, smem));
  nb = std::max(nb, 1);
  const int64_t want = (n + 127) / 128;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nb * c->sms));
  k_predict64<<<grid, 128, smem, c->stream>>>(e, s, check_rules, begin, idx, feat, n, pred, idx_out, band_v,
                                              band_theta, staged);
  return check_launch(c);
}

// Sort (pred, idx) pairs ascending by pred, ties by idx. If `by_idx_first`,
// the input is not already in index order and an index sort runs first
// (radix sort is stable). Result lands in (*pred, *idx) (pointers may swap).
int sort_pairs(mlt_ctx* c, double** pred, int64_t** idx, double* pred_alt, int64_t* idx_alt, int64_t n,
               bool by_idx_first) {
  if (n <= 1) return MLT_OK;
  if (n > INT32_MAX) return fail(MLT_EINVAL, "too many entries to sort (%lld)", (long long)n);
  cub::DoubleBuffer<double> kp(*pred, pred_alt);
  cub::DoubleBuffer<int64_t> ki(*idx, idx_alt);
  size_t tmp_bytes = 0, t2 = 0;
  CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kp, ki, (int)n, 0, 64, c->stream));
  CU(cub::DeviceRadixSort::SortPairs(nullptr, t2, ki, kp, (int)n, 0, 64, c->stream));
  tmp_bytes = std::max(tmp_bytes, t2);
  void* tmp;
  TRY(ws(c, S_SORT_TMP, tmp_bytes, &tmp));
  if (by_idx_first) {
    CU(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ki, kp, (int)n, 0, 64, c->stream));
    c->launches += 4;
  }
  CU(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kp, ki, (int)n, 0, 64, c->stream));
  c->launches += 4;
  CU(cudaGetLastError());
  *pred = kp.Current();
  *idx = ki.Current();
  return MLT_OK;
}

// Copy the first min(m, n) sorted entries to the host; valid ones have idx != INT64_MAX.
int emit_top(mlt_ctx* c, const double* pred, const int64_t* idx, int64_t n, int64_t m, int64_t* out_idx,
             double* out_pred, int64_t* out_n) {
  const int64_t take = std::min(m, n);
  std::vector<int64_t> hi(take);
  std::vector<double> hp(take);
  if (take > 0) {
    CU(cudaMemcpyAsync(hi.data(), idx, take * 8, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaMemcpyAsync(hp.data(), pred, take * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  CU(cudaStreamSynchronize(c->stream));
  int64_t cnt = 0;
  for (int64_t t = 0; t < take; ++t) {
    if (hi[t] == INT64_MAX || hi[t] < 0) break;
    out_idx[cnt] = hi[t];
    out_pred[cnt] = hp[t];
    ++cnt;
  }
  *out_n = cnt;
  return MLT_OK;
}

__global__ void k_merge_prep(const int64_t* idx, const double* pred, int64_t n, int64_t* io, double* po) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx[t];
    const bool ok = i >= 0 && i != INT64_MAX;
    io[t] = ok ? i : INT64_MAX;
    po[t] = ok ? pred[t] : __longlong_as_double(0x7ff0000000000000ll);
  }
}

// One CTA merges n_rec sorted records (each: m indices -- -1 pads at the end
// -- then m prediction bit patterns, then a status word) by RANK: entry i of
// record r lands at position
//   i + sum_{r' < r} #{e in r' : e <= x} + sum_{r' > r} #{e in r' : e < x}
// in (prediction, index) order (equal entries ordered by record, so ranks are
// distinct), found by binary searches over the records staged in shared
// memory -- the records are already sorted, so no sort is needed. The first m
// land in host-mapped memory ([0] count, [1] OR of the status words, then m
// predictions and m indices), so the caller's single wait returns the answer.
constexpr int kMergeMaxEntries = 8192;   // n_rec * m staged in shared memory (128 KB)
constexpr int kMergeMaxRec = 256;
__global__ void __launch_bounds__(1024) k_merge_records(const int64_t* __restrict__ recs, int n_rec, int m,
                                                        int64_t* __restrict__ host_out) {
  extern __shared__ unsigned long long sm_rec[];   // [n] prediction bits, then [n] indices
  __shared__ int s_valid[kMergeMaxRec];
  __shared__ unsigned long long s_status;
  __shared__ int s_total;
  const int n = n_rec * m, tid = threadIdx.x;
  const int64_t stride = 2 * (int64_t)m + 1;
  unsigned long long* kp = sm_rec;
  long long* ki = reinterpret_cast<long long*>(sm_rec + n);
  for (int r = tid; r < n_rec; r += blockDim.x) s_valid[r] = m;
  if (tid == 0) {
    s_status = 0;
    s_total = 0;
  }
  __syncthreads();
  for (int e = tid; e < n; e += blockDim.x) {
    const int r = e / m, i = e - r * m;
    const long long x = recs[r * stride + i];
    kp[e] = (unsigned long long)recs[r * stride + m + i];
    ki[e] = x;
    if (x < 0) atomicMin(&s_valid[r], i);
  }
  for (int r = tid; r < n_rec; r += blockDim.x)
    if (recs[r * stride + 2 * m] != 0) atomicOr(&s_status, (unsigned long long)recs[r * stride + 2 * m]);
  __syncthreads();
  for (int r = tid; r < n_rec; r += blockDim.x) atomicAdd(&s_total, s_valid[r]);
  unsigned long long* hp = reinterpret_cast<unsigned long long*>(host_out + 2);
  long long* hx = reinterpret_cast<long long*>(host_out + 2 + m);
  for (int e = tid; e < n; e += blockDim.x) {
    const int r = e / m, i = e - r * m;
    if (i >= s_valid[r]) continue;
    const unsigned long long p = kp[e];   // positive doubles: bit patterns order like the values
    const long long x = ki[e];
    int rank = i;
    for (int r2 = 0; r2 < n_rec; ++r2) {
      if (r2 == r) continue;
      const bool le = r2 < r;           // earlier records win ties
      int lo = 0, hi = s_valid[r2];
      const int base = r2 * m;
      while (lo < hi) {                 // first entry of r2 that comes after (p, x)
        const int mid = (lo + hi) >> 1;
        const unsigned long long q = kp[base + mid];
        const long long y = ki[base + mid];
        const bool before = q < p || (q == p && (le ? y <= x : y < x));
        if (before) lo = mid + 1;
        else hi = mid;
      }
      rank += lo;
    }
    if (rank < m) {
      hp[rank] = p;
      hx[rank] = x;
    }
  }
  __syncthreads();
  if (tid == 0) {
    host_out[0] = min(m, s_total);
    host_out[1] = (long long)s_status;
  }
}

// Gathered records -> (index, prediction) pairs for the merge sort; padding
// becomes (INT64_MAX, +inf); the status words are OR-ed into *status.
__global__ void k_merge_rec_prep(const int64_t* recs, int64_t n_rec, int m, int64_t* io, double* po,
                                 unsigned long long* status) {
  const int64_t n = n_rec * m, stride = 2 * (int64_t)m + 1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / m, j = t - r * m;
    const int64_t* rec = recs + r * stride;
    const int64_t i = rec[j];
    const bool ok = i >= 0 && i != INT64_MAX;
    io[t] = ok ? i : INT64_MAX;
    po[t] = ok ? __longlong_as_double(rec[m + j]) : __longlong_as_double(0x7ff0000000000000ll);
    if (j == 0 && rec[2 * m] != 0) atomicOr(status, (unsigned long long)rec[2 * m]);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// plan: resident descriptors + the fp32-sweep setups
// ---------------------------------------------------------------------------
namespace {
// Everything the factored sweep needs for one split point (outer params
// [0, split), inner params [split, P)); computed once per split and cached.
struct BandSetup {
  bool ok = false;
  std::string why;
  int split = 0, G = 3, dummies = 0;
  int64_t c_in = 1, c_in_pad = kInnerBlock;
  double delta = 0, cst = 0;
  double mag = 0;               // sum |w'| + dummies + |cst|: scale of every partial sum
  double* d_tab = nullptr;      // [ca | cb | wprime] (k*kH each)
  std::vector<float> u;         // [k*kH] 1/w' (the sweep's parameter block, SweepArgs::uc)
  std::vector<double> wabs;     // [k*kH] |w'| per table position, 1 for dummy units
};
}  // namespace

struct mlt_plan {
  mlt_ctx* ctx = nullptr;
  HostSpace hs;
  HostEns he;
  // device copies (plan-owned, not workspace slots)
  int64_t* d_values = nullptr;
  int* d_rpos = nullptr;
  int64_t* d_rcoeff = nullptr;
  double* d_ens = nullptr;
  double* d_F = nullptr;        // per-parameter exp factors [k*kH][sum radix]
  int foff[kMaxP + 1] = {0};
  DSpace ds{};
  DEns de{};
  bool factors_ok = false;
  std::vector<int> unit_of;     // table position -> original unit m*kH + j
  int* d_unit_of = nullptr;
  bool units_sorted = false;    // unit_of in plan_sort_units' order (pruning), else the identity
  std::map<int, BandSetup> setups;
  // Every configuration gets the SAME prediction, bit for bit, in the
  // reference's arithmetic: each hidden unit with a nonzero output weight has
  // zero first-layer weights on every parameter with more than one value (and
  // finite ones on the single-valued parameters, whose feature is 0), so
  // z = b1 for every configuration (plan_create). The top-m is then the first
  // m statically valid indices -- lexsort's tie order (run_constant).
  bool constant = false;
  // Factored tables of the last band sweep: a derived, resident layout of the
  // weights for one (split, group, outer range); repeated sweeps of the same
  // slice with this plan reuse them instead of rebuilding.
  float* t_ea = nullptr;
  float* t_ebp = nullptr;
  float* t_remlo = nullptr;     // pruning bounds [outer][checkpoint]
  int* t_order = nullptr;       // pruning: outer blocks in ascending order of their lower bound
  size_t t_order_cap = 0;
  size_t t_ea_cap = 0, t_ebp_cap = 0, t_remlo_cap = 0;
  int64_t t_key[5] = {-1, -1, -1, -1, -1};
};

namespace {

// Inner/outer split for a sweep over n configurations: the inner factor must
// fit a 512-thread-pair work item well (padding waste) and stay small enough
// for the L2-resident table; table entries cost ~10 configuration-units each.
int choose_split(const mlt_plan* p, int64_t n) {
  const HostSpace& s = p->hs;
  int best = s.P;
  double best_cost = 1e300;
  int64_t cin = 1;
  for (int sp = s.P - 1; sp >= 0; --sp) {
    cin *= s.radix[sp];
    if (cin > 16384 || s.P - sp > 16) break;    // k_table_tiles handles <= 16 inner params
    const int64_t pad = (cin + kInnerBlock - 1) / kInnerBlock * kInnerBlock;
    const double rows = std::ceil((double)n / cin) + 1.0;
    const double waste = (double)n * ((double)pad / cin - 1.0);
    const double cost = waste + 10.0 * ((double)pad + std::ceil(rows / kOB) * kOB);
    if (cost < best_cost) {
      best_cost = cost;
      best = sp;
    }
  }
  return best == s.P ? s.P - 1 : best;
}

int band_setup(mlt_plan* p, int split, BandSetup& b) {
  const HostEns& e = p->he;
  const HostSpace& s = p->hs;
  b = BandSetup();
  b.split = split;
  if (e.h > kH || !p->factors_ok) {
    b.why = e.h > kH ? "hidden size > 30" : "first-layer weights too large for the factored tables";
    return MLT_OK;
  }
  int64_t cin = 1;
  for (int q = split; q < s.P; ++q) cin *= s.radix[q];
  b.c_in = cin;
  b.c_in_pad = (cin + kInnerBlock - 1) / kInnerBlock * kInnerBlock;

  const int KH = e.k * kH;
  if (KH > kMaxUnitsParam) {
    b.why = "more hidden units than the sweep's parameter block holds";
    return MLT_OK;
  }
  std::vector<double> tab(3 * (size_t)KH, 0.0);
  double* ca = tab.data();
  double* cb = ca + KH;
  double* wpv = cb + KH;
  std::vector<float> u(KH, 1.0f);
  double S = 0, log2dmax = -1e300, log2dmin = 1e300;
  // log2 of the largest d' = (1 + exp(-zmin)) / |w'| needs log1p(exp(.)) per
  // unit; first an upper bound with log1p(e^x) <= max(x, 0) + ln 2 (no
  // transcendental), the exact value only when the bound decides nothing
  double log2dmax_ub = -1e300;
  std::vector<std::pair<double, double>> zl;   // (-zmin, log|w'|) per real unit
  zl.reserve(KH);
  int dummies = 0;
  // the multi-valued parameters, outer ones (q < split) first: single-valued
  // parameters never move z
  int act[kMaxP], n_act = 0, n_out = 0;
  for (int q = 0; q < s.P; ++q)
    if (s.radix[q] >= 2) {
      act[n_act++] = q;
      if (q < split) n_out = n_act;
    }
  // table position `mj` holds original unit unit_of[mj] (plan_factors' order)
  for (int pos = 0; pos < KH; ++pos) {
    {
      const int mj = pos;
      const int m = p->unit_of[pos] / kH, j = p->unit_of[pos] % kH;
      const double wp = (j < e.h) ? e.w2()[(size_t)m * e.h + j] * e.sd()[m] / e.k : 0.0;
      if (wp == 0.0) {
        ++dummies;                // contributes exactly 1/d' = 1/(Ea*0 + 1) = 1
        ca[mj] = 1.0;
        continue;
      }
      const double b1 = e.b1()[(size_t)m * e.h + j];
      double amin = b1, amax = b1, bmin = 0, bmax = 0;
      const double* w = e.w1() + ((size_t)m * e.h + j) * e.d;
      for (int t = 0; t < n_out; ++t) {
        amin += std::min(0.0, w[act[t]]);
        amax += std::max(0.0, w[act[t]]);
      }
      for (int t = n_out; t < n_act; ++t) {
        bmin += std::min(0.0, w[act[t]]);
        bmax += std::max(0.0, w[act[t]]);
      }
      const double c = 0.5 * (amin - bmin);   // centring: both tables span zmin/2 at their low end
      const double zmin = amin + bmin;
      const double lw = std::log(std::fabs(wp));
      const double lim = 80.0;
      // exp(-A'), exp(-B')/w' and 1/w' must be normal fp32 numbers
      if (!(amax - c <= lim && -(amin - c) <= lim && (bmax + c) + lw <= lim && -(bmin + c) - lw <= lim &&
            std::fabs(lw) <= lim)) {
        b.why = "first-layer range too wide for fp32 tables";
        return MLT_OK;
      }
      ca[mj] = std::exp(-(b1 - c));
      cb[mj] = std::exp(-c) / wp;
      wpv[mj] = wp;
      u[mj] = (float)(1.0 / wp);
      S += std::fabs(wp);
      log2dmax_ub = std::max(log2dmax_ub, (std::max(-zmin, 0.0) + std::log(2.0) - lw) / std::log(2.0));
      zl.emplace_back(-zmin, lw);
      log2dmin = std::min(log2dmin, -lw / std::log(2.0));
    }
  }
  // Units per shared reciprocal: the largest G <= the requested maximum
  // (MLT_OPT_GROUP, default kDefaultGroup) whose G-fold products of d' stay
  // inside the normal fp32 range and that divides the unit count.
  const int gmax = (p->ctx->opt_group >= 1 && p->ctx->opt_group <= 4) ? p->ctx->opt_group : kDefaultGroup;
  if (gmax * std::max(log2dmax_ub, 0.0) < 124.0) {
    log2dmax = log2dmax_ub;   // the bound already admits the largest grouping
  } else {
    for (const auto& v : zl)
      log2dmax = std::max(log2dmax, (std::log1p(std::exp(std::min(v.first, 700.0))) - v.second) / std::log(2.0));
  }
  int G = 0;
  for (int g = gmax; g >= 1; --g) {
    if (KH % g == 0 && g * std::max(log2dmax, 0.0) < 124.0 && g * std::min(log2dmin, 0.0) > -124.0) {
      G = g;
      break;
    }
  }
  if (G == 0) {
    b.why = "reciprocal products would overflow fp32";
    return MLT_OK;
  }
  b.G = G;
  b.dummies = dummies;
  S += dummies;
  double cst = 0;
  for (int m = 0; m < e.k; ++m) cst += (e.b2()[m] * e.sd()[m] + e.mean()[m]) / e.k;
  cst -= dummies;
  b.cst = cst;
  b.mag = S + std::fabs(cst);
  const double uu = std::ldexp(1.0, -24);
  // A-priori |fp32 - exact| bound on the mean log:
  //  * each unit term 1/d' = w' sigma carries <= 4u relative error from the
  //    rounded tables and the FMA; the G-unit rational combination and the
  //    approximate reciprocal add <= cg*u relative to the group's sum of |terms|;
  //  * the running accumulator is rounded once per group, each time by at most
  //    u * |partial sum| <= u * (prefix sum of |w'| up to that group);
  //  * + cst (rounded) and the final add.
  const double cg = G == 4 ? 40.0 : (G == 3 ? 30.0 : (G == 2 ? 16.0 : 8.0));
  double prefix = 0.0, acc_bound = 0.0;
  for (int q = 0; q < KH; q += G) {
    for (int x = 0; x < G; ++x) prefix += wpv[q + x] != 0.0 ? std::fabs(wpv[q + x]) : 1.0;
    acc_bound += prefix;
  }
  b.delta = 1.5 * uu * (cg * S + acc_bound + S + 3.0 * std::fabs(cst)) + 1e-12 * (1.0 + std::fabs(cst));

  mlt_ctx* c = p->ctx;
  CU(cudaMallocAsync(&b.d_tab, tab.size() * 8, c->stream));
  TRY(upload_pinned(c, b.d_tab, tab.data(), tab.size() * 8));
  b.u = std::move(u);
  b.wabs.resize(KH);
  for (int q = 0; q < KH; ++q) b.wabs[q] = wpv[q] != 0.0 ? std::fabs(wpv[q]) : 1.0;
  b.ok = true;
  return MLT_OK;
}

int get_setup(mlt_plan* p, int split, BandSetup** out) {
  // keyed by the split and the requested reciprocal grouping (MLT_OPT_GROUP
  // may change between calls on a resident plan)
  const int key = split | (std::max(p->ctx->opt_group, 0) << 8);
  auto it = p->setups.find(key);
  if (it == p->setups.end()) {
    BandSetup b;
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = band_setup(p, split, b);
    if (std::getenv("MLT_STEP_TRACE"))
      std::fprintf(stderr, "{\"band_setup_us\": %.1f}\n",
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    if (rc != MLT_OK) {
      pool_free(p->ctx, b.d_tab);
      return rc;
    }
    it = p->setups.emplace(key, b).first;
  }
  *out = &it->second;
  return MLT_OK;
}

// F[position][digit] = exp factors of the unit at each table position
int launch_factors(mlt_plan* p) {
  const HostEns& e = p->he;
  const HostSpace& s = p->hs;
  mlt_ctx* c = p->ctx;
  const int KH = e.k * kH;
  TableArgs ta;
  std::memset(&ta, 0, sizeof ta);
  ta.k = e.k;
  ta.d = e.d;
  ta.h = e.h;
  for (int q = 0; q < s.P; ++q) ta.radix[q] = s.radix[q];
  for (int q = 0; q <= s.P; ++q) ta.foff[q] = p->foff[q];
  ta.w1 = p->de.w1;
  ta.unit_of = p->d_unit_of;
  ta.F = p->d_F;
  k_table_factors<<<grid_for(c, (int64_t)KH * p->foff[s.P], 256), 256, 0, c->stream>>>(ta);
  TRY(check_launch(c));
  return MLT_OK;
}

// Unit order for the pruned sweep: decreasing range of the unit's
// contribution over the whole space, |w'| * (sigmoid(zmax) - sigmoid(zmin)),
// so that the sweep's partial sums settle early (the pruning bounds of the
// remaining units are then tight); padding / zero-weight units last. Done on
// the first pruned call of a plan: F is rebuilt in the new order and every
// setup and table derived from the old one is dropped.
int plan_sort_units(mlt_plan* p) {
  const HostEns& e = p->he;
  const HostSpace& s = p->hs;
  mlt_ctx* c = p->ctx;
  const int KH = e.k * kH;
  // (-range, unit) ascending == a stable sort by decreasing range; the
  // single-valued parameters never move z, so they are skipped up front
  int act[kMaxP], n_act = 0;
  for (int q = 0; q < s.P; ++q)
    if (s.radix[q] >= 2) act[n_act++] = q;
  std::vector<std::pair<double, int>> key(KH);
  for (int mj = 0; mj < KH; ++mj) {
    key[mj] = {1.0, mj};   // padding / zero-weight units: after every real unit
    const int m = mj / kH, j = mj % kH;
    if (j >= e.h) continue;
    const double wp = e.w2()[(size_t)m * e.h + j] * e.sd()[m] / e.k;
    if (wp == 0.0) continue;
    double zmin = e.b1()[(size_t)m * e.h + j], zmax = zmin;
    const double* w = e.w1() + ((size_t)m * e.h + j) * e.d;
    for (int t = 0; t < n_act; ++t) {
      zmin += std::min(0.0, w[act[t]]);
      zmax += std::max(0.0, w[act[t]]);
    }
    auto sg = [](double z) { return 1.0 / (1.0 + std::exp(-z)); };
    key[mj].first = -(std::fabs(wp) * (sg(zmax) - sg(zmin)));
  }
  std::sort(key.begin(), key.end());
  for (int mj = 0; mj < KH; ++mj) p->unit_of[mj] = key[mj].second;
  TRY(upload_pinned(c, p->d_unit_of, p->unit_of.data(), (size_t)KH * 4));
  TRY(launch_factors(p));
  for (auto& kv : p->setups) pool_free(c, kv.second.d_tab);
  p->setups.clear();
  std::fill(p->t_key, p->t_key + 5, -1);
  p->units_sorted = true;
  return MLT_OK;
}

// exp factors of every (unit, parameter, digit): computed once per plan.
int plan_factors(mlt_plan* p) {
  const HostEns& e = p->he;
  const HostSpace& s = p->hs;
  p->factors_ok = false;
  double wmax = 0;
  for (size_t q = 0; q < (size_t)e.k * e.h * e.d; ++q) wmax = std::max(wmax, std::fabs(e.w1()[q]));
  if (wmax > 600.0) return MLT_OK;          // a single factor could overflow fp64
  p->foff[0] = 0;
  for (int q = 0; q < s.P; ++q) p->foff[q + 1] = p->foff[q] + s.radix[q];
  const int KH = e.k * kH;
  mlt_ctx* c = p->ctx;
  // Table position = unit (m*kH + j) until a pruned sweep asks for the
  // range order (plan_sort_units): the full sweep's exactness does not depend
  // on the order, so a fresh plan skips the ordering's host math
  p->unit_of.resize(KH);
  for (int mj = 0; mj < KH; ++mj) p->unit_of[mj] = mj;
  p->units_sorted = false;
  CU(cudaMallocAsync(&p->d_unit_of, (size_t)KH * 4, c->stream));
  TRY(upload_pinned(c, p->d_unit_of, p->unit_of.data(), (size_t)KH * 4));
  CU(cudaMallocAsync(&p->d_F, (size_t)KH * p->foff[s.P] * 8, c->stream));
  TRY(launch_factors(p));
  p->factors_ok = true;
  return MLT_OK;
}

int plan_upload(mlt_plan* p) {
  mlt_ctx* c = p->ctx;
  const HostSpace& h = p->hs;
  DSpace& d = p->ds;
  std::memset(&d, 0, sizeof d);
  d.P = h.P;
  d.R = (int)h.rkind.size();
  int off = 0;
  for (int q = 0; q < h.P; ++q) {
    d.radix[q] = h.radix[q];
    d.voff[q] = off;
    off += h.radix[q];
  }
  CU(cudaMallocAsync(&p->d_values, h.values.size() * 8, c->stream));
  TRY(upload_pinned(c, p->d_values, h.values.data(), h.values.size() * 8));
  d.values = p->d_values;
  for (int r = 0; r < d.R; ++r) {
    d.rkind[r] = h.rkind[r];
    d.rbound[r] = h.rbound[r];
  }
  for (int r = 0; r <= d.R; ++r) d.roff[r] = h.roff[r];
  CU(cudaMallocAsync(&p->d_rpos, std::max<size_t>(1, h.rpos.size()) * 4, c->stream));
  CU(cudaMallocAsync(&p->d_rcoeff, std::max<size_t>(1, h.rcoeff.size()) * 8, c->stream));
  if (!h.rpos.empty()) {
    TRY(upload_pinned(c, p->d_rpos, h.rpos.data(), h.rpos.size() * 4));
    TRY(upload_pinned(c, p->d_rcoeff, h.rcoeff.data(), h.rcoeff.size() * 8));
  }
  d.rpos = p->d_rpos;
  d.rcoeff = p->d_rcoeff;

  const HostEns& e = p->he;
  DEns& de = p->de;
  std::memset(&de, 0, sizeof de);
  de.k = e.k;
  de.d = e.d;
  de.h = e.h;
  for (int q = 0; q < e.d; ++q) de.counts[q] = e.counts[q];
  CU(cudaMallocAsync(&p->d_ens, e.packed.size() * 8, c->stream));
  TRY(upload_pinned(c, p->d_ens, e.packed.data(), e.packed.size() * 8));
  const size_t nw = (size_t)e.k * e.h * e.d, nh = (size_t)e.k * e.h;
  de.w1 = p->d_ens;
  de.b1 = p->d_ens + nw;
  de.w2 = p->d_ens + nw + nh;
  de.b2 = p->d_ens + nw + 2 * nh;
  de.mean = de.b2 + e.k;
  de.std_ = de.mean + e.k;
  return MLT_OK;
}

void plan_free(mlt_plan* p) {
  mlt_ctx* c = p->ctx;
  pool_free(c, p->d_values);
  pool_free(c, p->d_rpos);
  pool_free(c, p->d_rcoeff);
  pool_free(c, p->d_ens);
  pool_free(c, p->d_F);
  pool_free(c, p->d_unit_of);
  for (auto& kv : p->setups) {
    pool_free(c, kv.second.d_tab);
  }
  p->setups.clear();
  pool_free(c, p->t_ea);
  pool_free(c, p->t_ebp);
  pool_free(c, p->t_remlo);
  pool_free(c, p->t_order);
  p->t_ea = p->t_ebp = p->t_remlo = nullptr;
  p->t_order = nullptr;
}

// fp64 materialise over a range or list, then sort: exact and general.
int run_full(mlt_plan* p, int64_t m, int64_t begin, int64_t end, const int64_t* d_list, int64_t n_list,
             int64_t* out_idx, double* out_pred, int64_t* out_n) {
  mlt_ctx* c = p->ctx;
  const int64_t n = d_list ? n_list : end - begin;
  double *pa, *pb;
  int64_t *ia, *ib;
  TRY(ws_t(c, S_OUT_A, n, &pa));
  TRY(ws_t(c, S_OUT_B, n, &pb));
  TRY(ws_t(c, S_OUT_C, n, &ia));
  TRY(ws_t(c, S_OUT_D, n, &ib));
  TRY(launch_predict64(c, p->de, p->ds, 1, begin, d_list, nullptr, n, pa, ia));
  TRY(sort_pairs(c, &pa, &ia, pb, ib, n, d_list != nullptr));
  return emit_top(c, pa, ia, n, m, out_idx, out_pred, out_n);
}

// Constant ensemble (mlt_plan::constant): every configuration ties, so the
// reference's lexsort((indices, preds)) returns the first m statically valid
// indices of the slice. Validity is evaluated chunk by chunk from `begin` and
// the valid indices selected in order (CUB DeviceSelect over a counting
// iterator) until m are found; the one prediction value is computed once by
// the fp64 kernel. Replaces a guard band that holds every configuration (an
// fp32 sweep + overflow + the fp64 materialising path: 350 ms on the 10^8
// space) by a validity scan of the first ~m configurations.
int run_constant(mlt_plan* p, int64_t m, int64_t begin, int64_t end, int64_t* out_idx, double* out_pred,
                 int64_t* out_n) {
  mlt_ctx* c = p->ctx;
  std::vector<int64_t> found;
  found.reserve(m);
  const int64_t chunk = std::max<int64_t>(4 * m, int64_t(1) << 20);
  void* fv;
  int64_t *sel, *nsel;
  TRY(ws(c, S_OUT_C, (size_t)chunk, &fv));
  uint8_t* flags = static_cast<uint8_t*>(fv);
  TRY(ws_t(c, S_OUT_D, (size_t)chunk + 1, &sel));
  nsel = sel + chunk;
  size_t tmp_bytes = 0;
  CU(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, cub::CountingInputIterator<int64_t>(0), flags, sel, nsel,
                                chunk, c->stream));
  void* tmp;
  TRY(ws(c, S_SORT_TMP, tmp_bytes, &tmp));
  std::vector<int64_t> hsel;
  for (int64_t lo = begin; lo < end && (int64_t)found.size() < m; lo += chunk) {
    const int64_t n = std::min(chunk, end - lo);
    int64_t ns = n;
    if (p->ds.R > 0) {
      k_valid_range<<<grid_for(c, n, 256), 256, 0, c->stream>>>(p->ds, lo, n, flags);
      TRY(check_launch(c));
      CU(cub::DeviceSelect::Flagged(tmp, tmp_bytes, cub::CountingInputIterator<int64_t>(lo), flags, sel, nsel, n,
                                    c->stream));
      CU(cudaMemcpyAsync(&ns, nsel, 8, cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      const int64_t take = std::min<int64_t>(ns, m - (int64_t)found.size());
      hsel.resize(take);
      if (take > 0) {
        CU(cudaMemcpyAsync(hsel.data(), sel, take * 8, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
      }
      found.insert(found.end(), hsel.begin(), hsel.end());
    } else {
      for (int64_t t = 0; t < n && (int64_t)found.size() < m; ++t) found.push_back(lo + t);
    }
  }
  if (found.empty()) {
    *out_n = 0;
    return MLT_OK;
  }
  double* pv;
  int64_t* iv;
  TRY(ws_t(c, S_OUT_A, 1, &pv));
  TRY(ws_t(c, S_OUT_B, 1, &iv));
  TRY(launch_predict64(c, p->de, p->ds, 0, found[0], nullptr, nullptr, 1, pv, iv));
  double v = 0;
  CU(cudaMemcpyAsync(&v, pv, 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (size_t t = 0; t < found.size(); ++t) {
    out_idx[t] = found[t];
    out_pred[t] = v;
  }
  *out_n = (int64_t)found.size();
  return MLT_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// extern "C" API
// ---------------------------------------------------------------------------
extern "C" {

int mlt_abi_version(void) { return MLT_ABI_VERSION; }
const char* mlt_last_error(void) { return g_err.c_str(); }

int mlt_ctx_create(int device, mlt_ctx** out) {
  if (!out) return fail(MLT_EINVAL, "out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(MLT_ECUDA, "no CUDA device available (%s); libmltune_b200 has no CPU fallback",
                e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
  if (device < 0 || device >= n) return fail(MLT_EINVAL, "device %d out of range (%d devices)", device, n);
  CU(cudaSetDevice(device));
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(MLT_ECUDA, "device %d is sm_%d%d; libmltune_b200 is built for sm_100a only", device, prop.major,
                prop.minor);
  mlt_ctx* c = new mlt_ctx();
  c->dev = device;
  c->sms = prop.multiProcessorCount;
  CU(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
  c->stream = c->own;
  {
    cudaMemPool_t pool;
    CU(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;   // never trim: per-call plans reuse the same blocks
    CU(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  CU(cudaMallocHost(&c->pinned, 4096));
  for (auto& ev : c->ev) CU(cudaEventCreate(&ev));
  CU(cudaEventCreateWithFlags(&c->ev_switch, cudaEventDisableTiming));
  *out = c;
  return MLT_OK;
}

int mlt_ctx_destroy(mlt_ctx* c) {
  if (!c) return MLT_OK;
  cudaSetDevice(c->dev);
  cudaStreamSynchronize(c->stream);
  for (void* p : c->slots)
    if (p) cudaFree(p);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->stage) cudaFreeHost(c->stage);
  if (c->res_pin) cudaFreeHost(c->res_pin);
  if (c->merge_pin) cudaFreeHost(c->merge_pin);
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  if (c->ev_switch) cudaEventDestroy(c->ev_switch);
  if (c->own) cudaStreamDestroy(c->own);
  // stream-ordered frees (plans, tables, trainer buffers) return memory to the
  // device's default pool; hand the pool's idle memory back to the driver
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, c->dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  delete c;
  return MLT_OK;
}

int mlt_ctx_set_stream(mlt_ctx* c, void* stream) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  cudaStream_t next = stream ? static_cast<cudaStream_t>(stream) : c->own;
  if (next != c->stream) {
    // work already queued on the old stream (workspace slots, pinned staging,
    // device results) must precede everything queued on the new one
    CU(cudaEventRecord(c->ev_switch, c->stream));
    CU(cudaStreamWaitEvent(next, c->ev_switch, 0));
    c->stream = next;
  }
  return MLT_OK;
}

int mlt_ctx_set_profiling(mlt_ctx* c, int on) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  c->prof = on != 0;
  return MLT_OK;
}

int64_t mlt_ctx_launches(mlt_ctx* c) { return c ? c->launches : -1; }

int mlt_ctx_set_option(mlt_ctx* c, int key, int64_t value) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  switch (key) {
    case MLT_OPT_PATH: c->opt_path = (int)value; return MLT_OK;
    case MLT_OPT_GROUP: c->opt_group = (int)value; return MLT_OK;
    case MLT_OPT_CAND_CAP: c->cand_cap = value < 0 ? (1 << 20) : std::max<int64_t>(value, 1); return MLT_OK;
    case MLT_OPT_PRUNE: c->opt_prune = value == 1 ? 1 : 0; return MLT_OK;
    case MLT_OPT_CHUNK: c->chunk = value < 0 ? (int64_t(1) << 27) : std::max<int64_t>(value, 4096); return MLT_OK;
    case MLT_OPT_TABLE_CACHE: c->opt_table_cache = value == 0 ? 0 : 1; return MLT_OK;
    case MLT_OPT_HALF_ITEMS: c->opt_half_items = value == 1 ? 1 : 0; return MLT_OK;
    case MLT_OPT_TAIL_SPLIT: c->opt_tail_split = value == 0 ? 0 : 1; return MLT_OK;
    default: return fail(MLT_EINVAL, "unknown option %d", key);
  }
}

int mlt_decode(mlt_ctx* c, const mlt_space* space, const int64_t* idx, int64_t n, int64_t* values_out) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  if (n < 0) return fail(MLT_EINVAL, "negative count");
  if (n == 0) return MLT_OK;
  CU(cudaSetDevice(c->dev));
  HostSpace hs;
  TRY(read_space(space, &hs));
  for (int64_t t = 0; t < n; ++t)
    if (idx[t] < 0 || idx[t] >= hs.card_i)
      return fail(MLT_EINVAL, "index %lld out of range for %lld configurations", (long long)idx[t],
                  (long long)hs.card_i);
  DSpace ds;
  TRY(upload_space(c, hs, &ds));
  int64_t *di, *dv;
  TRY(ws_t(c, S_IDX, n, &di));
  TRY(ws_t(c, S_OUT_C, (size_t)n * hs.P, &dv));
  CU(cudaMemcpyAsync(di, idx, n * 8, cudaMemcpyHostToDevice, c->stream));
  k_decode<<<grid_for(c, n, 256), 256, 0, c->stream>>>(ds, di, n, dv);
  TRY(check_launch(c));
  CU(cudaMemcpyAsync(values_out, dv, (size_t)n * hs.P * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MLT_OK;
}

int mlt_valid_mask(mlt_ctx* c, const mlt_space* space, const int64_t* idx, int64_t n, uint8_t* mask_out) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  if (n < 0) return fail(MLT_EINVAL, "negative count");
  if (n == 0) return MLT_OK;
  CU(cudaSetDevice(c->dev));
  HostSpace hs;
  TRY(read_space(space, &hs));
  for (int64_t t = 0; t < n; ++t)
    if (idx[t] < 0 || idx[t] >= hs.card_i)
      return fail(MLT_EINVAL, "index %lld out of range for %lld configurations", (long long)idx[t],
                  (long long)hs.card_i);
  DSpace ds;
  TRY(upload_space(c, hs, &ds));
  int64_t* di;
  uint8_t* dm;
  TRY(ws_t(c, S_IDX, n, &di));
  TRY(ws_t(c, S_OUT_C, n, &dm));
  CU(cudaMemcpyAsync(di, idx, n * 8, cudaMemcpyHostToDevice, c->stream));
  k_valid<<<grid_for(c, n, 256), 256, 0, c->stream>>>(ds, di, n, dm);
  TRY(check_launch(c));
  CU(cudaMemcpyAsync(mask_out, dm, n, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MLT_OK;
}

int mlt_encode(mlt_ctx* c, const int32_t* counts, int32_t d, const int64_t* idx, int64_t n, double* feat_out) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  if (d < 1 || d > kMaxP) return fail(MLT_EINVAL, "input dimension must be 1..%d", kMaxP);
  if (n < 0) return fail(MLT_EINVAL, "negative count");
  if (n == 0) return MLT_OK;
  CU(cudaSetDevice(c->dev));
  DEns e;
  std::memset(&e, 0, sizeof e);
  e.d = d;
  for (int p = 0; p < d; ++p) {
    if (counts[p] < 1) return fail(MLT_EINVAL, "encoder parameter %d has no values", p);
    e.counts[p] = counts[p];
  }
  int64_t* di;
  double* df;
  TRY(ws_t(c, S_IDX, n, &di));
  TRY(ws_t(c, S_FEAT, (size_t)n * d, &df));
  CU(cudaMemcpyAsync(di, idx, n * 8, cudaMemcpyHostToDevice, c->stream));
  k_encode<<<grid_for(c, n, 256), 256, 0, c->stream>>>(e, di, n, df);
  TRY(check_launch(c));
  CU(cudaMemcpyAsync(feat_out, df, (size_t)n * d * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MLT_OK;
}

int mlt_predict_indices(mlt_ctx* c, const mlt_ensemble* ens, const int64_t* idx, int64_t n, double* pred_out) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  if (n < 0) return fail(MLT_EINVAL, "negative count");
  CU(cudaSetDevice(c->dev));
  HostEns he;
  TRY(read_ens(ens, &he));
  if (n == 0) return MLT_OK;
  for (int64_t t = 0; t < n; ++t)
    if (idx[t] < 0) return fail(MLT_EINVAL, "negative configuration index %lld", (long long)idx[t]);
  DEns de;
  TRY(upload_ens(c, he, &de));
  DSpace ds;
  std::memset(&ds, 0, sizeof ds);
  int64_t* di;
  double* dp;
  TRY(ws_t(c, S_IDX, n, &di));
  TRY(ws_t(c, S_OUT_A, n, &dp));
  CU(cudaMemcpyAsync(di, idx, n * 8, cudaMemcpyHostToDevice, c->stream));
  TRY(launch_predict64(c, de, ds, 0, 0, di, nullptr, n, dp, nullptr));
  CU(cudaMemcpyAsync(pred_out, dp, n * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MLT_OK;
}

int mlt_predict_features(mlt_ctx* c, const mlt_ensemble* ens, const double* x, int64_t n, double* pred_out) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  if (n < 0) return fail(MLT_EINVAL, "negative count");
  CU(cudaSetDevice(c->dev));
  HostEns he;
  TRY(read_ens(ens, &he));
  if (n == 0) return MLT_OK;
  DEns de;
  TRY(upload_ens(c, he, &de));
  DSpace ds;
  std::memset(&ds, 0, sizeof ds);
  double *dx, *dp;
  TRY(ws_t(c, S_FEAT, (size_t)n * he.d, &dx));
  TRY(ws_t(c, S_OUT_A, n, &dp));
  CU(cudaMemcpyAsync(dx, x, (size_t)n * he.d * 8, cudaMemcpyHostToDevice, c->stream));
  TRY(launch_predict64(c, de, ds, 0, 0, nullptr, dx, n, dp, nullptr));
  CU(cudaMemcpyAsync(pred_out, dp, n * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MLT_OK;
}

int mlt_member_outputs(mlt_ctx* c, const mlt_ensemble* ens, const double* x, int64_t n, double* out) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  if (n < 0) return fail(MLT_EINVAL, "negative count");
  CU(cudaSetDevice(c->dev));
  HostEns he;
  TRY(read_ens(ens, &he));
  if (n == 0) return MLT_OK;
  DEns de;
  TRY(upload_ens(c, he, &de));
  double *dx, *dp;
  TRY(ws_t(c, S_FEAT, (size_t)n * he.d, &dx));
  TRY(ws_t(c, S_OUT_A, (size_t)n * he.k, &dp));
  CU(cudaMemcpyAsync(dx, x, (size_t)n * he.d * 8, cudaMemcpyHostToDevice, c->stream));
  const int staged = predict64_smem(de) <= 200 * 1024 ? 1 : 0;
  const size_t smem = staged ? predict64_smem(de) : 0;
  CU(cudaFuncSetAttribute(k_member_out64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_member_out64<<<grid_for(c, n, 128), 128, smem, c->stream>>>(de, dx, n, dp, staged);
  TRY(check_launch(c));
  CU(cudaMemcpyAsync(out, dp, (size_t)n * he.k * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MLT_OK;
}

int mlt_plan_create(mlt_ctx* c, const mlt_space* space, const mlt_ensemble* ens, mlt_plan** out) {
  if (!c || !out) return fail(MLT_EINVAL, "ctx/out is NULL");
  CTX_GUARD(c);
  *out = nullptr;
  CU(cudaSetDevice(c->dev));
  const bool trace = std::getenv("MLT_STEP_TRACE") != nullptr;   // diagnostics: host time of the phases
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto us = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double, std::micro>(b - a).count();
  };
  const auto t0 = now();
  mlt_plan* p = new mlt_plan();
  p->ctx = c;
  int rc = read_space(space, &p->hs);
  if (rc == MLT_OK) rc = read_ens(ens, &p->he);
  const auto t1 = now();
  if (rc == MLT_OK && p->he.d != p->hs.P)
    rc = fail(MLT_EMISMATCH, "ensemble has %d inputs but the space has %d parameters", p->he.d, p->hs.P);
  for (int q = 0; rc == MLT_OK && q < p->hs.P; ++q)
    if (p->he.counts[q] != p->hs.radix[q])
      rc = fail(MLT_EMISMATCH, "encoder parameter %d has %d values, space has %d", q, p->he.counts[q],
                p->hs.radix[q]);
  if (rc == MLT_OK) rc = plan_upload(p);
  const auto t2 = now();
  if (rc == MLT_OK) rc = plan_factors(p);
  const auto t3 = now();
  if (trace)
    std::fprintf(stderr, "{\"plan_read_us\": %.1f, \"plan_upload_us\": %.1f, \"plan_factors_us\": %.1f}\n",
                 us(t0, t1), us(t1, t2), us(t2, t3));
  if (rc == MLT_OK) {
    const HostEns& e = p->he;
    bool constant = true;
    for (int u = 0; constant && u < e.k * e.h; ++u) {
      if (e.w2()[u] == 0.0) continue;
      for (int q = 0; q < e.d; ++q) {
        const double w = e.w1()[(size_t)u * e.d + q];
        if (p->hs.radix[q] >= 2 ? w != 0.0 : !std::isfinite(w)) {
          constant = false;
          break;
        }
      }
    }
    p->constant = constant;
  }
  if (rc != MLT_OK) {
    plan_free(p);
    delete p;
    return rc;
  }
  *out = p;   // no host wait: uploads come from the pinned ring, and all use is stream-ordered
  return MLT_OK;
}

int mlt_plan_destroy(mlt_plan* p) {
  if (!p) return MLT_OK;
  CTX_GUARD(p->ctx);
  cudaSetDevice(p->ctx->dev);
  plan_free(p);   // stream-ordered frees: no host wait
  delete p;
  return MLT_OK;
}

// d_rec != nullptr: the device-record variant (mlt_plan_top_m_record): the
// band path is only enqueued (its result packed into d_rec, no host wait) and
// the function returns with *out_n = -1; callers fall back to the host-output
// path when the band path does not apply.
static int plan_top_m_impl(mlt_plan* p, int64_t m, int64_t begin, int64_t end, const int64_t* idx_list,
                           int64_t n_list, int64_t* out_idx, double* out_pred, int64_t* out_n,
                           mlt_sweep_stats* st, int64_t* d_rec = nullptr) {
  mlt_ctx* c = p->ctx;
  if (m < 1) return fail(MLT_EINVAL, "m must be >= 1");
  if (!out_idx || !out_pred || !out_n) return fail(MLT_EINVAL, "output pointers are NULL");
  CU(cudaSetDevice(c->dev));
  *out_n = 0;
  mlt_sweep_stats local;
  std::memset(&local, 0, sizeof local);
  local.evaluated_frac = 1.0;
  const int64_t l0 = c->launches;
  const int64_t card = p->hs.card_i;
  int64_t n;
  if (idx_list) {
    if (n_list < 0) return fail(MLT_EINVAL, "negative list length");
    for (int64_t t = 0; t < n_list; ++t)
      if (idx_list[t] < 0 || idx_list[t] >= card)
        return fail(MLT_EINVAL, "index %lld out of range for %lld configurations", (long long)idx_list[t],
                    (long long)card);
    n = n_list;
  } else {
    if (begin < 0 || end > card || begin > end)
      return fail(MLT_EINVAL, "slice [%lld, %lld) outside [0, %lld)", (long long)begin, (long long)end,
                  (long long)card);
    n = end - begin;
  }
  local.configs = n;
  if (n == 0) {
    if (st) *st = local;
    return MLT_OK;
  }
  if (p->constant && !idx_list && c->opt_path != 1) {
    // every configuration ties (mlt_plan::constant): the first m valid indices
    local.path = 2;
    TRY(run_constant(p, m, begin, end, out_idx, out_pred, out_n));
    local.candidates = *out_n;
    local.launches = (int32_t)(c->launches - l0);
    if (st) *st = local;
    return MLT_OK;
  }
  if (c->prof) CU(cudaEventRecord(c->ev[0], c->stream));

  BandSetup* bs = nullptr;
  if (!idx_list && m <= kMaxTopM && c->opt_path != 1) {
    if (c->opt_prune == 1 && p->factors_ok && !p->units_sorted) TRY(plan_sort_units(p));
    TRY(get_setup(p, choose_split(p, n), &bs));
  }
  bool band = bs && bs->ok && (n >= 4096 || c->opt_path == 0);
  // the sweep stages two exp(-A') tiles of k*30*8 floats plus its candidate
  // slots in shared memory: very large ensembles take the exact path instead
  if (band && sweep_smem(p->he.k, m > kMaxTopMSmall ? kSBBig : kSB) > 227 * 1024) band = false;

  if (band) {
    const BandSetup& B = *bs;
    local.split = p->hs.P - B.split;
    const int KH = p->he.k * kH;
    const int64_t o_lo = begin / B.c_in;
    const int64_t o_hi = (end - 1) / B.c_in + 1;
    const int n_ob = (int)((o_hi - o_lo + kOB - 1) / kOB);
    const int n_ib = (int)(B.c_in_pad / kInnerBlock);
    float *ea, *ebp, *cval;
    int64_t* cidx;
    uint32_t* gs;
    const int ebw = ebw_of(B.G);
    const size_t n_ea = (size_t)n_ob * KH * kOB, n_ebp = ((size_t)n_ib * (KH / B.G) + 2) * kThreads * ebw * 4;   // + 2 groups
                                                                             // of padding (the sweep's prefetch)
    const bool prune = c->opt_prune == 1;
    const int ngroups = KH / B.G;
    CkList ck;
    std::memset(&ck, 0, sizeof ck);
    int ck_group[kMaxCk] = {0};
    if (prune) {
      ck_group[0] = 0;            // before any unit: the item's lower bound alone
      ck.unit[0] = 0;
      ck.n = 1;
      // every 2.5 % of the units from 20 % to 95 % (A/B on the 10^8 case: 5 % steps
      // from 25 % 2.676 ms, 2.5 % from 10 % 2.661, this schedule 2.649)
      for (int f = 8; f <= 38 && ck.n < kMaxCk; ++f) {
        const int g = (int)((int64_t)f * ngroups / 40) / kSweepStep * kSweepStep;
        if (g > 0 && g < ngroups && (ck.n == 0 || g > ck_group[ck.n - 1])) {
          ck_group[ck.n] = g;
          ck.unit[ck.n] = g * B.G;
          ++ck.n;
        }
      }
      for (int q = 0; q < ck.n; ++q) {
        double m = 0.0;
        for (int pos = KH - 1; pos >= ck.unit[q]; --pos) m += B.wabs[pos];
        ck.mag[q] = m;
      }
    }
    const size_t n_remlo = prune ? (size_t)n_ob * kOB * n_ib * ck.n : 0;
    const int64_t key[5] = {B.split, B.G, o_lo, n_ob, prune ? 1 : 0};
    const bool tables_cached = c->opt_table_cache && std::equal(key, key + 5, p->t_key);
    if (!tables_cached) {
      if (p->t_remlo_cap < n_remlo) {
        pool_free(c, p->t_remlo);
        p->t_remlo = nullptr;
        p->t_remlo_cap = 0;
        CU(cudaMallocAsync(&p->t_remlo, n_remlo * 4, c->stream));
        p->t_remlo_cap = n_remlo;
      }
      if (p->t_ea_cap < n_ea) {
        pool_free(c, p->t_ea);
        p->t_ea = nullptr;
        p->t_ea_cap = 0;
        CU(cudaMallocAsync(&p->t_ea, n_ea * 4, c->stream));
        p->t_ea_cap = n_ea;
      }
      if (p->t_ebp_cap < n_ebp) {
        pool_free(c, p->t_ebp);
        p->t_ebp = nullptr;
        p->t_ebp_cap = 0;
        CU(cudaMallocAsync(&p->t_ebp, n_ebp * 4, c->stream));
        p->t_ebp_cap = n_ebp;
        // the padding past the last group is read (never used) by the sweep's
        // prefetch: give it defined contents once
        const size_t pad = (size_t)2 * kThreads * ebw * 4;
        CU(cudaMemsetAsync(p->t_ebp + (n_ebp - pad), 0, pad * 4, c->stream));
      }
      std::fill(p->t_key, p->t_key + 5, -1);   // valid again only once the tables below are built
    }
    ea = p->t_ea;
    ebp = p->t_ebp;
    TRY(ws_t(c, S_GSCAL, 16, &gs));
    TRY(ws_t(c, S_CIDX, (size_t)c->cand_cap, &cidx));
    TRY(ws_t(c, S_CVAL, (size_t)c->cand_cap, &cval));
    TableArgs ta;
    std::memset(&ta, 0, sizeof ta);
    ta.k = p->he.k;
    ta.d = p->he.d;
    ta.h = p->he.h;
    ta.split = B.split;
    ta.G = B.G;
    for (int q = 0; q < p->hs.P; ++q) {
      ta.radix[q] = p->hs.radix[q];
      ta.f_radix[q] = make_fdiv(p->hs.radix[q]);
    }
    ta.f_kh = make_fdiv(KH);
    ta.f_ngroups = make_fdiv(KH / B.G);
    for (int q = 0; q <= p->hs.P; ++q) ta.foff[q] = p->foff[q];
    ta.w1 = p->de.w1;
    ta.F = p->d_F;
    ta.ca = B.d_tab;
    ta.cb = B.d_tab + KH;
    ta.wprime = B.d_tab + 2 * KH;
    ta.o_lo = o_lo;
    ta.o_card = card / B.c_in;
    ta.c_in = B.c_in;
    ta.c_in_pad = B.c_in_pad;
    ta.n_ob = n_ob;
    ta.ea = ea;
    ta.ebp = ebp;
    {
      const int64_t lim = int64_t(1) << 31;
      ta.idx32 = (int64_t)n_ob * KH * kOB < lim && o_lo + (int64_t)n_ob * kOB < lim &&
                 (int64_t)n_ib * (KH / B.G) * kThreads < lim && B.c_in_pad < lim;
    }
    // gs[0] theta key, [1] candidate count, [2..4] band-stage counters (n,
    // status, take), [8..9] pruning work (64-bit), [10] pruning: next work item
    {
      uint32_t init[16] = {0xFF800000u};   // [0] = fkey(+inf), the rest 0
      TRY(upload_pinned(c, gs, init, sizeof init));   // the ring: safe with no host wait behind it
    }
    if (!tables_cached) {
      // two-level split of each side: lo = trailing parameters with <= 64 combinations
      auto lo_split = [&](int p_lo, int p_hi, int* sa, int64_t* nlo) {
        int64_t n = 1;
        int q = p_hi;
        while (q > p_lo && n * p->hs.radix[q - 1] <= 64) n *= p->hs.radix[--q];
        *sa = q;
        *nlo = n;
      };
      int sa_o, sa_i;
      int64_t nlo_o, nlo_i;
      lo_split(0, B.split, &sa_o, &nlo_o);
      lo_split(B.split, p->hs.P, &sa_i, &nlo_i);
      const int64_t o_end = std::min<int64_t>(o_lo + (int64_t)n_ob * kOB, card / B.c_in);
      const int64_t hb = o_lo / nlo_o, he = (std::max<int64_t>(o_end, o_lo + 1) - 1) / nlo_o + 1;
      const int64_t nhi_i = B.c_in / nlo_i;
      double *PoH, *PoL, *PiH, *PiL;
      TRY(ws_t(c, S_POH, (size_t)KH * (he - hb), &PoH));
      TRY(ws_t(c, S_POL, (size_t)KH * nlo_o, &PoL));
      TRY(ws_t(c, S_PIH, (size_t)KH * nhi_i, &PiH));
      TRY(ws_t(c, S_PIL, (size_t)KH * nlo_i, &PiL));
      {
        const PartialJobs jobs = {{0, sa_o, B.split, sa_i},
                                  {sa_o, B.split, sa_i, p->hs.P},
                                  {hb, 0, 0, 0},
                                  {he - hb, nlo_o, nhi_i, nlo_i},
                                  {make_fdiv(he - hb), make_fdiv(nlo_o), make_fdiv(nhi_i), make_fdiv(nlo_i)},
                                  {PoH, PoL, PiH, PiL}};
        const int64_t tot = (int64_t)KH * (he - hb + nlo_o + nhi_i + nlo_i);
        k_table_partial4<<<grid_for(c, tot, 256), 256, 0, c->stream>>>(ta, jobs);
        TRY(check_launch(c));
      }
      ta.PoH = PoH;
      ta.PoL = PoL;
      ta.PiH = PiH;
      ta.PiL = PiL;
      ta.o_nlo = nlo_o;
      ta.o_nhi = he - hb;
      ta.o_hi_base = hb;
      ta.i_nlo = nlo_i;
      ta.i_nhi = nhi_i;
      ta.f_onlo = make_fdiv(nlo_o);
      ta.f_inlo = make_fdiv(nlo_i);
      {
        const int nb_outer = grid_for(c, (int64_t)n_ob * KH * kOB, 256);
        const int nb_inner = grid_for(c, (int64_t)n_ib * (KH / B.G) * kThreads, 256);
        void (*tiles)(TableArgs, int) = B.G == 4 ? k_table_tiles<4>
                                        : B.G == 3 ? k_table_tiles<3> : (B.G == 2 ? k_table_tiles<2> : k_table_tiles<1>);
        tiles<<<nb_outer + nb_inner, 256, 0, c->stream>>>(ta, nb_outer);
        TRY(check_launch(c));
      }
      if (prune) {
        double* ext;
        TRY(ws_t(c, S_SORT_TMP, (size_t)KH * n_ib, &ext));
        ta.n_ib = n_ib;
        k_table_ebext<<<grid_for(c, (int64_t)KH * n_ib * 32, 256), 256, 0, c->stream>>>(ta, ext);
        TRY(check_launch(c));
        // CTAs stride over the outer rows (k_table_rem: 256 threads, 22 KB of
        // shared memory, 6 resident per SM: one wave)
        const int64_t rows = (int64_t)n_ob * kOB;
        k_table_rem<<<(int)std::min<int64_t>(rows, (int64_t)c->sms * 6), 256, 0, c->stream>>>(ta, ck, ext,
                                                                                            p->t_remlo);
        TRY(check_launch(c));
        // best-first order of the work items: by the smallest whole-item lower
        // bound, sorted on the device (a stable radix sort: ties keep index order)
        const int items = n_ob * n_ib;
        if (p->t_order_cap < (size_t)items) {
          pool_free(c, p->t_order);
          p->t_order = nullptr;
          p->t_order_cap = 0;
          CU(cudaMallocAsync(&p->t_order, (size_t)items * 4, c->stream));
          p->t_order_cap = items;
        }
        if (items <= kItemSortMax) {   // sorted runs + rank merge (the 10^8 space: 6144 items)
          unsigned* run_key;
          CU(cudaMallocAsync(&run_key, (size_t)items * 8, c->stream));
          int* run_val = reinterpret_cast<int*>(run_key + items);
          k_item_runs<<<(items + kItemRun - 1) / kItemRun, kItemRunThreads, 0, c->stream>>>(p->t_remlo, ck.n, n_ib,
                                                                                           items, run_key, run_val);
          TRY(check_launch(c));
          const size_t smem = (size_t)kItemSortMax * 4;
          TRY(kernel_smem(c, k_item_merge, kItemSortThreads, smem));
          k_item_merge<<<(items + kItemSortThreads - 1) / kItemSortThreads, kItemSortThreads, smem, c->stream>>>(
              run_key, run_val, items, p->t_order);
          TRY(check_launch(c));
          CU(cudaFreeAsync(run_key, c->stream));
        } else {
          float *kin, *kout;
          int* vin;
          void* tmp = nullptr;
          size_t tmp_bytes = 0;
          CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, (const float*)nullptr, (float*)nullptr,
                                             (const int*)nullptr, (int*)nullptr, items, 0, 32, c->stream));
          CU(cudaMallocAsync(&kin, (size_t)items * 4, c->stream));
          CU(cudaMallocAsync(&kout, (size_t)items * 4, c->stream));
          CU(cudaMallocAsync(&vin, (size_t)items * 4, c->stream));
          CU(cudaMallocAsync(&tmp, std::max<size_t>(tmp_bytes, 16), c->stream));
          k_item_keys<<<grid_for(c, items, 256), 256, 0, c->stream>>>(p->t_remlo, ck.n, n_ib, items, kin, vin);
          TRY(check_launch(c));
          CU(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kin, kout, vin, p->t_order, items, 0, 32, c->stream));
          for (void* q : {(void*)kin, (void*)kout, (void*)vin, tmp}) CU(cudaFreeAsync(q, c->stream));
        }
      }
      std::copy(key, key + 5, p->t_key);
    }

    SweepArgs sa;
    std::memset(&sa, 0, sizeof sa);
    sa.k = p->he.k;
    sa.ea = ea;
    sa.ebp = ebp;
    std::copy(B.u.begin(), B.u.end(), sa.uc);
    sa.c_in = B.c_in;
    sa.c_in_pad = B.c_in_pad;
    sa.o_lo = o_lo;
    sa.n_ob = n_ob;
    sa.n_ib = n_ib;
    sa.begin = begin;
    sa.end = end;
    sa.cst = (float)B.cst;
    sa.band = (float)(2.0 * B.delta * (1.0 + 1e-6));
    sa.m = (int)m;
    sa.g_theta = gs;
    sa.g_count = gs + 1;
    sa.g_cidx = cidx;
    sa.g_cval = cval;
    sa.cap = (uint32_t)std::min<int64_t>(c->cand_cap, UINT32_MAX);
    sa.check_rules = p->ds.R > 0;
    sa.prune = prune ? 1 : 0;
    sa.n_ck = ck.n;
    for (int q = 0; q < ck.n; ++q) sa.ck_group[q] = ck_group[q];
    sa.remlo = p->t_remlo;
    // fp32 rounding of T = acc + (cst + remlo): a few ulps of the largest partial sum
    sa.prune_eps = (float)(16.0 * std::ldexp(1.0, -23) * (B.mag + 1.0));
    sa.item_order = p->t_order;
    sa.g_work = reinterpret_cast<unsigned long long*>(gs + 8);
    sa.g_next = reinterpret_cast<int*>(gs + 10);
    sa.sp = p->ds;
    const bool big = m > kMaxTopMSmall;   // the instance with kSBBig candidate slots per CTA
    const size_t smem = sweep_smem(p->he.k, big ? kSBBig : kSB);
    if (smem > 227 * 1024) return fail(MLT_EINTERNAL, "sweep needs %zu B of shared memory", smem);
    using KF = void (*)(SweepArgs);
#define MLT_KROW(SBV, PR, NTV, OB) \
  { k_sweep<1, PR, SBV, NTV, OB>, k_sweep<2, PR, SBV, NTV, OB>, k_sweep<3, PR, SBV, NTV, OB>, \
    k_sweep<4, PR, SBV, NTV, OB> }
    static const KF kerns[2][2][2][4] = {
        {{MLT_KROW(kSB, false, kThreads, kOB), MLT_KROW(kSB, true, kThreads, kOB)},
         {MLT_KROW(kSBBig, false, kThreads, kOB), MLT_KROW(kSBBig, true, kThreads, kOB)}},
        {{MLT_KROW(kSB, false, kThreads / 2, kOB), MLT_KROW(kSB, true, kThreads / 2, kOB)},
         {MLT_KROW(kSBBig, false, kThreads / 2, kOB), MLT_KROW(kSBBig, true, kThreads / 2, kOB)}}};
    static const KF tails[2][2][4] = {{MLT_KROW(kSB, false, kThreads, 2), MLT_KROW(kSBBig, false, kThreads, 2)},
                                      {MLT_KROW(kSB, false, kThreads, 4), MLT_KROW(kSBBig, false, kThreads, 4)}};
#undef MLT_KROW
    // Wave quantisation: whole items (8 outers x 2048 inners, one 1024-thread
    // CTA per SM) run in full waves; when the items of the last, partial wave
    // fit ONE round of quarter (else half) items, they go to a second TAIL
    // launch split that way, so the step ends with a short round on many SMs
    // instead of a whole item-time on a few (1/8 of the 10^8 space: 768 items
    // = 5.2 waves, 28 left over: 0.734 -> 0.692 ms). A split needing several
    // rounds of parts loses to the plain last wave (parts are less efficient
    // than whole items), so it is not taken then. MLT_OPT_TAIL_SPLIT = 0 turns
    // it off; MLT_OPT_HALF_ITEMS = 1 instead runs two 512-thread CTAs per SM
    // on half items (the earlier alternative, kept for A/B).
    const int whole_items = n_ob * n_ib;
    const bool halves = c->opt_half_items == 1;
    const int nt = halves ? kThreads / 2 : kThreads;
    KF kern = kerns[halves ? 1 : 0][big ? 1 : 0][prune ? 1 : 0][B.G - 1];
    int nb = 0;
    TRY(kernel_smem(c, kern, nt, smem, &nb));
    nb = std::max(nb, 1);
    const int slots = nb * c->sms;   // CTAs resident at once
    int main_hi = whole_items, tail_obu = 0;
    if (!prune && !halves && c->opt_tail_split != 0 && whole_items > slots && whole_items % slots != 0) {
      const int rem = whole_items % slots;
      tail_obu = rem * (kOB / 2) <= slots ? 2 : (rem * (kOB / 4) <= slots ? 4 : 0);
      if (tail_obu) main_hi = whole_items - rem;
    }
    sa.item_lo = 0;
    sa.item_hi = main_hi;
    const int64_t units = (int64_t)main_hi * (kThreads / nt);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(units, slots));
    if (c->prof) CU(cudaEventRecord(c->ev[1], c->stream));
    kern<<<grid, nt, smem, c->stream>>>(sa);
    TRY(check_launch(c));
    if (main_hi < whole_items) {
      KF tk = tails[tail_obu == 2 ? 0 : 1][big ? 1 : 0][B.G - 1];
      TRY(kernel_smem(c, tk, kThreads, smem));
      SweepArgs ta2 = sa;
      ta2.item_lo = main_hi;
      ta2.item_hi = whole_items;
      const int64_t tunits = (int64_t)(whole_items - main_hi) * (kOB / tail_obu);
      tk<<<(int)std::min<int64_t>(tunits, slots), kThreads, smem, c->stream>>>(ta2);
      TRY(check_launch(c));
    }
    if (c->prof) CU(cudaEventRecord(c->ev[2], c->stream));
    // Snapshot the sweep's counters (the band stage reuses gs[2..4]) and launch
    // the band stage right behind the sweep, without a host round trip: its
    // buffers are sized for the candidate capacity and its kernels read the
    // candidate count on the device. One host wait at the end of the step.
    const uint32_t cap = (uint32_t)std::min<int64_t>(c->cand_cap, UINT32_MAX);
    const size_t cap1 = std::max<size_t>(cap, 1);
    double *pa, *pb, *tp;
    int64_t *ia, *ib, *ti;
    float* fv;
    TRY(ws_t(c, S_OUT_A, cap1, &pa));
    TRY(ws_t(c, S_OUT_B, cap1, &pb));
    TRY(ws_t(c, S_OUT_C, cap1, &ia));
    TRY(ws_t(c, S_OUT_D, cap1, &ib));
    TRY(ws_t(c, S_FEAT, cap1, &fv));
    TRY(ws_t(c, S_TOPI, (size_t)m, &ti));
    TRY(ws_t(c, S_TOPP, (size_t)m, &tp));
    // 1) exact global tau_m over the candidates, keep f32 <= tau_m + 2*delta
    //    (a count beyond the capacity: no survivors, the host falls back below)
    k_band_filter<<<1, 1024, 0, c->stream>>>(cidx, cval, gs + 1, cap, (int)m, sa.band, ia, fv, gs + 2);
    TRY(check_launch(c));
    // 2) fp64 rescoring of the survivors, one warp each (grid-stride over the
    //    device count; survivors are few, ~m, so 32 CTAs of 8 warps)
    {
      const size_t rsm = ((size_t)p->he.k * p->he.h + p->he.k) * 8;
      if (rsm > 200 * 1024) return fail(MLT_EINVAL, "ensemble too large for the rescoring kernel (%zu B)", rsm);
      TRY(kernel_smem(c, k_rescore, 256, rsm));
      k_rescore<<<2 * c->sms, 256, rsm, c->stream>>>(p->de, ia, gs + 2, pa);
    }
    TRY(check_launch(c));
    // 3) sort by (prediction, index) in one CTA when small
    //    (sized for 4m survivors: the band keeps m + a few; more -> CUB below)
    const int scap = sort_small_cap(4 * m), ssmem = 16 * scap;
    TRY(kernel_smem(c, k_sort_small, 1024, ssmem));
    // the host-output step: the sort writes the result and the counters straight
    // into pinned host memory (mapped, UVA), so no copy follows the kernels
    const size_t res_bytes = 64 + (size_t)m * 16;
    if (!d_rec && c->res_cap < res_bytes) {
      if (c->res_pin) CU(cudaFreeHost(c->res_pin));
      c->res_pin = nullptr;
      c->res_cap = 0;
      CU(cudaHostAlloc(&c->res_pin, res_bytes, cudaHostAllocMapped));
      c->res_cap = res_bytes;
    }
    uint32_t* hres = d_rec ? nullptr : static_cast<uint32_t*>(c->res_pin);
    uint32_t* dres = nullptr;
    if (hres) CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dres), hres, 0));
    k_sort_small<<<1, 1024, ssmem, c->stream>>>(pa, ia, gs + 2, (int)m, tp, ti, gs + 3, scap, dres, gs, d_rec, cap);
    TRY(check_launch(c));
    if (d_rec) {   // device record (written by the sort): return without waiting
      local.group = B.G;
      local.delta = B.delta;
      local.launches = (int32_t)(c->launches - l0);
      if (st) *st = local;
      *out_n = -1;
      return MLT_OK;
    }
    double* rp = reinterpret_cast<double*>(hres + 16);
    int64_t* ri = reinterpret_cast<int64_t*>(rp + m);
    if (c->prof) CU(cudaEventRecord(c->ev[4], c->stream));   // device work of the step done
    CU(cudaStreamSynchronize(c->stream));
    const uint32_t count = hres[1];
    local.evaluated_frac = 1.0;
    if (prune) {
      uint64_t work;
      std::memcpy(&work, hres + 8, 8);
      local.evaluated_frac = (double)work / ((double)n_ob * n_ib * ngroups * (kThreads / 32));   // warp-groups
    }
    local.group = B.G;
    local.raw_candidates = count;
    local.delta = B.delta;
    if ((int64_t)count > c->cand_cap) {
      band = false;   // crowded guard band: fall back to the exact materialising path
    } else {
      const uint32_t n2 = hres[2], big = hres[3], take = hres[4];
      local.candidates = n2;
      if (!big) {   // the lists already landed in pinned memory with the counters
        const int64_t tk = std::min<int64_t>(m, take);
        int64_t cnt = 0;
        for (int64_t t = 0; t < tk; ++t) {
          if (ri[t] == INT64_MAX || ri[t] < 0) break;
          out_idx[cnt] = ri[t];
          out_pred[cnt] = rp[t];
          ++cnt;
        }
        *out_n = cnt;
      } else {
        double* pcur = pa;
        int64_t* icur = ia;
        TRY(sort_pairs(c, &pcur, &icur, pb, ib, n2, true));
        TRY(emit_top(c, pcur, icur, n2, m, out_idx, out_pred, out_n));
      }
    }
    if (c->prof) {
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]));
      local.sweep_ms = ms;
      if (std::getenv("MLT_STEP_TRACE")) {   // diagnostics: where the step's device time goes
        float pre = 0, post = 0;
        CU(cudaEventElapsedTime(&pre, c->ev[0], c->ev[1]));
        CU(cudaEventElapsedTime(&post, c->ev[2], c->ev[4]));
        std::fprintf(stderr, "{\"pre_sweep_ms\": %.4f, \"sweep_ms\": %.4f, \"band_stage_ms\": %.4f}\n", pre, ms, post);
      }
    }
  }
  if (!band) {
    local.path = 1;
    local.candidates = 0;
    const int64_t* dl = nullptr;
    if (idx_list) {
      int64_t* di;
      TRY(ws_t(c, S_IDX, n, &di));
      CU(cudaMemcpyAsync(di, idx_list, n * 8, cudaMemcpyHostToDevice, c->stream));
      dl = di;
    }
    if (c->prof) CU(cudaEventRecord(c->ev[1], c->stream));
    TRY(run_full(p, m, begin, end, dl, n, out_idx, out_pred, out_n));
    if (c->prof) {
      CU(cudaEventRecord(c->ev[2], c->stream));
      CU(cudaEventSynchronize(c->ev[2]));
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]));
      local.sweep_ms = ms;
    }
  }
  if (c->prof) {
    CU(cudaEventRecord(c->ev[3], c->stream));
    CU(cudaEventSynchronize(c->ev[3]));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, c->ev[0], c->ev[3]));
    local.total_ms = ms;
  }
  local.launches = (int32_t)(c->launches - l0);
  if (st) *st = local;
  return MLT_OK;
}

// Slices longer than kChunk configurations are swept chunk by chunk (bounded
// table and materialisation memory for spaces far beyond 10^8) and the
// per-chunk top-m lists merged by (prediction, index): exact, because every
// element of the global top-m is in its own chunk's top-m.
static int plan_top_m_range(mlt_plan* p, int64_t m, int64_t begin, int64_t end, int64_t* out_idx, double* out_pred,
                            int64_t* out_n, mlt_sweep_stats* st) {
  const int64_t kChunk = p->ctx->chunk;
  if (end - begin <= kChunk || m < 1 || begin < 0 || end > p->hs.card_i || begin > end)
    return plan_top_m_impl(p, m, begin, end, nullptr, 0, out_idx, out_pred, out_n, st);
  std::vector<std::pair<double, int64_t>> all;
  std::vector<int64_t> ci(m);
  std::vector<double> cp(m);
  mlt_sweep_stats tot;
  std::memset(&tot, 0, sizeof tot);
  tot.evaluated_frac = 0.0;
  for (int64_t lo = begin; lo < end; lo += kChunk) {
    const int64_t hi = std::min(end, lo + kChunk);
    int64_t n = 0;
    mlt_sweep_stats cs;
    std::memset(&cs, 0, sizeof cs);
    TRY(plan_top_m_impl(p, m, lo, hi, nullptr, 0, ci.data(), cp.data(), &n, &cs));
    for (int64_t q = 0; q < n; ++q) all.emplace_back(cp[q], ci[q]);
    tot.configs += cs.configs;
    tot.candidates += cs.candidates;
    tot.raw_candidates += cs.raw_candidates;
    tot.path = std::max(tot.path, cs.path);
    tot.group = cs.group;
    tot.split = cs.split;
    tot.delta = std::max(tot.delta, cs.delta);
    tot.sweep_ms += cs.sweep_ms;
    tot.total_ms += cs.total_ms;
    tot.launches += cs.launches;
    tot.evaluated_frac += cs.evaluated_frac * (double)(hi - lo);
  }
  std::sort(all.begin(), all.end());
  const int64_t take = std::min<int64_t>(m, (int64_t)all.size());
  for (int64_t q = 0; q < take; ++q) {
    out_pred[q] = all[q].first;
    out_idx[q] = all[q].second;
  }
  *out_n = take;
  tot.evaluated_frac /= (double)(end - begin);
  if (st) *st = tot;
  return MLT_OK;
}

int mlt_plan_top_m(mlt_plan* p, int64_t m, int64_t begin, int64_t end, int64_t* out_idx, double* out_pred,
                   int64_t* out_n, mlt_sweep_stats* st) {
  if (!p) return fail(MLT_EINVAL, "plan is NULL");
  CTX_GUARD(p->ctx);
  return plan_top_m_range(p, m, begin, end, out_idx, out_pred, out_n, st);
}

int mlt_plan_top_m_record(mlt_plan* p, int64_t m, int64_t begin, int64_t end, int64_t* d_rec) {
  if (!p) return fail(MLT_EINVAL, "plan is NULL");
  if (!d_rec) return fail(MLT_EINVAL, "record pointer is NULL");
  CTX_GUARD(p->ctx);
  if (m < 1) return fail(MLT_EINVAL, "m must be >= 1");
  std::vector<int64_t> hi(m);
  std::vector<double> hp(m);
  int64_t n = 0;
  if (end - begin <= p->ctx->chunk) {
    TRY(plan_top_m_impl(p, m, begin, end, nullptr, 0, hi.data(), hp.data(), &n, nullptr, d_rec));
    if (n < 0) return MLT_OK;   // enqueued on the device
  } else {
    TRY(plan_top_m_range(p, m, begin, end, hi.data(), hp.data(), &n, nullptr));
  }
  // host-side result (exact path, or a chunked slice): upload it as the record
  std::vector<int64_t> rec(2 * m + 1);
  for (int64_t t = 0; t < m; ++t) {
    const bool ok = t < n;
    rec[t] = ok ? hi[t] : -1;
    double v = ok ? hp[t] : INFINITY;
    std::memcpy(&rec[m + t], &v, 8);
  }
  rec[2 * m] = 0;
  return upload_pinned(p->ctx, d_rec, rec.data(), rec.size() * 8);
}

int mlt_merge_records(mlt_ctx* c, const int64_t* d_recs, int64_t n_rec, int64_t m, int64_t* out_idx,
                      double* out_pred, int64_t* out_n, int64_t* out_status) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  if (m < 1) return fail(MLT_EINVAL, "m must be >= 1");
  if (n_rec < 0 || !d_recs || !out_idx || !out_pred || !out_n || !out_status)
    return fail(MLT_EINVAL, "bad record merge arguments");
  CU(cudaSetDevice(c->dev));
  *out_n = 0;
  *out_status = 0;
  const int64_t n = n_rec * m;
  if (n == 0) return MLT_OK;
  if (n <= kMergeMaxEntries && n_rec <= kMergeMaxRec) {
    // one kernel: rank-merge of the sorted records straight into mapped host memory
    const size_t bytes = (2 + 2 * (size_t)m) * 8;
    if (c->merge_cap < bytes) {
      if (c->merge_pin) CU(cudaFreeHost(c->merge_pin));
      c->merge_pin = nullptr;
      c->merge_cap = 0;
      CU(cudaHostAlloc(&c->merge_pin, bytes, cudaHostAllocMapped));
      c->merge_cap = bytes;
    }
    int64_t* hres = static_cast<int64_t*>(c->merge_pin);
    int64_t* dres = nullptr;
    CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dres), hres, 0));
    const size_t smem = (size_t)n * 16;
    TRY(kernel_smem(c, k_merge_records, 1024, smem));
    k_merge_records<<<1, 1024, smem, c->stream>>>(d_recs, (int)n_rec, (int)m, dres);
    TRY(check_launch(c));
    CU(cudaStreamSynchronize(c->stream));
    const int64_t cnt = hres[0];
    const double* hp = reinterpret_cast<const double*>(hres + 2);
    const int64_t* hx = hres + 2 + m;
    for (int64_t t = 0; t < cnt; ++t) {
      out_idx[t] = hx[t];
      out_pred[t] = hp[t];
    }
    *out_n = cnt;
    *out_status = hres[1];
    return MLT_OK;
  }
  double *pa, *pb;
  int64_t *ia, *ib;
  uint32_t* gs;
  TRY(ws_t(c, S_OUT_A, n, &pa));
  TRY(ws_t(c, S_OUT_B, n, &pb));
  TRY(ws_t(c, S_OUT_C, n, &ia));
  TRY(ws_t(c, S_OUT_D, n, &ib));
  TRY(ws_t(c, S_GSCAL, 8, &gs));
  {
    uint32_t init[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    TRY(upload_pinned(c, gs, init, sizeof init));
  }
  unsigned long long* dstat = reinterpret_cast<unsigned long long*>(gs + 6);
  k_merge_rec_prep<<<grid_for(c, n, 256), 256, 0, c->stream>>>(d_recs, n_rec, (int)m, ia, pa, dstat);
  TRY(check_launch(c));
  int64_t* hst = reinterpret_cast<int64_t*>(static_cast<uint32_t*>(c->pinned) + 12);
  CU(cudaMemcpyAsync(hst, dstat, 8, cudaMemcpyDeviceToHost, c->stream));
  if (n <= kSmallSort) {
    double* tp;
    int64_t* ti;
    TRY(ws_t(c, S_TOPI, (size_t)std::min(m, n), &ti));
    TRY(ws_t(c, S_TOPP, (size_t)std::min(m, n), &tp));
    {
      const uint32_t cnt = (uint32_t)n;
      TRY(upload_pinned(c, gs + 2, &cnt, 4));
    }
    const int scap = sort_small_cap(n), ssmem = 16 * scap;
    TRY(kernel_smem(c, k_sort_small, 1024, ssmem));
    k_sort_small<<<1, 1024, ssmem, c->stream>>>(pa, ia, gs + 2, (int)std::min<int64_t>(m, n), tp, ti, gs + 3, scap);
    TRY(check_launch(c));
    TRY(emit_top(c, tp, ti, std::min(m, n), m, out_idx, out_pred, out_n));
  } else {
    TRY(sort_pairs(c, &pa, &ia, pb, ib, n, true));
    TRY(emit_top(c, pa, ia, n, m, out_idx, out_pred, out_n));
  }
  *out_status = *hst;   // landed before emit_top's host wait returned
  return MLT_OK;
}

int mlt_top_m(mlt_ctx* c, const mlt_space* space, const mlt_ensemble* ens, int64_t m, int64_t begin, int64_t end,
              const int64_t* idx_list, int64_t n_list, int64_t* out_idx, double* out_pred, int64_t* out_n,
              mlt_sweep_stats* st) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  if (m < 1) return fail(MLT_EINVAL, "m must be >= 1");
  mlt_plan* p = nullptr;
  TRY(mlt_plan_create(c, space, ens, &p));
  const int rc = idx_list ? plan_top_m_impl(p, m, begin, end, idx_list, n_list, out_idx, out_pred, out_n, st)
                          : plan_top_m_range(p, m, begin, end, out_idx, out_pred, out_n, st);
  mlt_plan_destroy(p);
  return rc;
}

// Single-process multi-GPU top-m (SURVEY §8(b) `mlt_sweep_topn_multi`): the
// slice (or the index list) is cut into n_ctx contiguous shards, one host
// thread per context sweeps its shard on its own device concurrently, and the
// per-shard top-m lists (exact over their shard) are merged on the host by
// (prediction, index) -- the union's top-m is the global top-m. No collective:
// the only exchange is n_ctx x m (index, prediction) pairs.
int mlt_top_m_multi(mlt_ctx* const* ctxs, int32_t n_ctx, const mlt_space* space, const mlt_ensemble* ens,
                    int64_t m, int64_t begin, int64_t end, const int64_t* idx_list, int64_t n_list,
                    int64_t* out_idx, double* out_pred, int64_t* out_n, mlt_sweep_stats* st) {
  if (!ctxs || n_ctx < 1) return fail(MLT_EINVAL, "need at least one context");
  for (int i = 0; i < n_ctx; ++i) {
    if (!ctxs[i]) return fail(MLT_EINVAL, "context %d is NULL", i);
    for (int j = 0; j < i; ++j)
      if (ctxs[j] == ctxs[i]) return fail(MLT_EINVAL, "context %d is passed twice (contexts are not re-entrant)", i);
  }
  if (m < 1) return fail(MLT_EINVAL, "m must be >= 1");
  if (!out_idx || !out_pred || !out_n) return fail(MLT_EINVAL, "output pointer is NULL");
  if (idx_list ? n_list < 0 : (begin < 0 || begin > end)) return fail(MLT_EINVAL, "bad slice or list length");
  struct Shard {
    int64_t lo = 0, hi = 0, n = 0;
    std::vector<int64_t> idx;
    std::vector<double> pred;
    mlt_sweep_stats st;
    int rc = MLT_OK;
    std::string err;
  };
  std::vector<Shard> sh(n_ctx);
  const int64_t total = idx_list ? n_list : end - begin;
  const int64_t q = total / n_ctx, r = total % n_ctx;
  for (int i = 0; i < n_ctx; ++i) {
    sh[i].lo = i * q + std::min<int64_t>(i, r);
    sh[i].hi = sh[i].lo + q + (i < r ? 1 : 0);
  }
  auto work = [&](int i) {
    Shard& s = sh[i];
    std::memset(&s.st, 0, sizeof s.st);
    if (s.hi == s.lo) return;
    s.idx.resize(m);
    s.pred.resize(m);
    s.rc = idx_list ? mlt_top_m(ctxs[i], space, ens, m, begin, end, idx_list + s.lo, s.hi - s.lo, s.idx.data(),
                                s.pred.data(), &s.n, &s.st)
                    : mlt_top_m(ctxs[i], space, ens, m, begin + s.lo, begin + s.hi, nullptr, 0, s.idx.data(),
                                s.pred.data(), &s.n, &s.st);
    if (s.rc != MLT_OK) s.err = g_err;   // the worker's thread-local message
  };
  std::vector<std::thread> th;
  for (int i = 1; i < n_ctx; ++i) th.emplace_back(work, i);
  work(0);
  for (auto& t : th) t.join();
  for (int i = 0; i < n_ctx; ++i)
    if (sh[i].rc != MLT_OK) return fail(sh[i].rc, "shard %d (device %d): %s", i, ctxs[i]->dev, sh[i].err.c_str());
  std::vector<std::pair<double, int64_t>> all;
  mlt_sweep_stats tot;
  std::memset(&tot, 0, sizeof tot);
  for (auto& s : sh) {
    for (int64_t k = 0; k < s.n; ++k) all.emplace_back(s.pred[k], s.idx[k]);
    tot.configs += s.st.configs;
    tot.candidates += s.st.candidates;
    tot.raw_candidates += s.st.raw_candidates;
    tot.path = std::max(tot.path, s.st.path);
    tot.group = std::max(tot.group, s.st.group);
    tot.split = std::max(tot.split, s.st.split);
    tot.delta = std::max(tot.delta, s.st.delta);
    tot.sweep_ms = std::max(tot.sweep_ms, s.st.sweep_ms);   // the devices run concurrently
    tot.total_ms = std::max(tot.total_ms, s.st.total_ms);
    tot.launches += s.st.launches;
    tot.evaluated_frac += s.st.evaluated_frac * (double)(s.hi - s.lo);
  }
  tot.evaluated_frac = total > 0 ? tot.evaluated_frac / (double)total : 1.0;
  std::sort(all.begin(), all.end());
  const int64_t take = std::min<int64_t>(m, (int64_t)all.size());
  for (int64_t k = 0; k < take; ++k) {
    out_pred[k] = all[k].first;
    out_idx[k] = all[k].second;
  }
  *out_n = take;
  if (st) *st = tot;
  return MLT_OK;
}

int mlt_merge_top_m(mlt_ctx* c, const int64_t* dev_idx, const double* dev_pred, int64_t n, int64_t m,
                    int64_t* out_idx, double* out_pred, int64_t* out_n) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  if (m < 1) return fail(MLT_EINVAL, "m must be >= 1");
  if (n < 0) return fail(MLT_EINVAL, "negative count");
  CU(cudaSetDevice(c->dev));
  *out_n = 0;
  if (n == 0) return MLT_OK;
  double *pa, *pb;
  int64_t *ia, *ib;
  TRY(ws_t(c, S_OUT_A, n, &pa));
  TRY(ws_t(c, S_OUT_B, n, &pb));
  TRY(ws_t(c, S_OUT_C, n, &ia));
  TRY(ws_t(c, S_OUT_D, n, &ib));
  k_merge_prep<<<grid_for(c, n, 256), 256, 0, c->stream>>>(dev_idx, dev_pred, n, ia, pa);
  TRY(check_launch(c));
  if (n <= kSmallSort) {   // typical: P ranks x m entries -> one-CTA bitonic sort
    uint32_t* gs;
    double* tp;
    int64_t* ti;
    TRY(ws_t(c, S_GSCAL, 8, &gs));
    TRY(ws_t(c, S_TOPI, (size_t)std::min(m, n), &ti));
    TRY(ws_t(c, S_TOPP, (size_t)std::min(m, n), &tp));
    uint32_t* hs = static_cast<uint32_t*>(c->pinned);
    hs[2] = (uint32_t)n;
    CU(cudaMemcpyAsync(gs + 2, hs + 2, 4, cudaMemcpyHostToDevice, c->stream));
    const int scap = sort_small_cap(n), ssmem = 16 * scap;
    TRY(kernel_smem(c, k_sort_small, 1024, ssmem));
    k_sort_small<<<1, 1024, ssmem, c->stream>>>(pa, ia, gs + 2, (int)std::min<int64_t>(m, n), tp, ti, gs + 3, scap);
    TRY(check_launch(c));
    return emit_top(c, tp, ti, std::min(m, n), m, out_idx, out_pred, out_n);
  }
  TRY(sort_pairs(c, &pa, &ia, pb, ib, n, true));
  return emit_top(c, pa, ia, n, m, out_idx, out_pred, out_n);
}

int mlt_train_members_impl(int dev, cudaStream_t stream, int64_t* launches, const mlt_train_desc* dd, double* w1,
                           double* b1, double* w2, double* b2, double* lf, double* ll, int32_t* div, const char** err);

int mlt_train_members(mlt_ctx* c, const mlt_train_desc* desc, double* w1, double* b1, double* w2, double* b2,
                      double* loss_first, double* loss_final, int32_t* diverged_epoch) {
  if (!c || !desc) return fail(MLT_EINVAL, "ctx/desc is NULL");
  CTX_GUARD(c);
  const char* err = "";
  const int rc = mlt_train_members_impl(c->dev, c->stream, &c->launches, desc, w1, b1, w2, b2, loss_first,
                                        loss_final, diverged_epoch, &err);
  if (rc != MLT_OK) return fail(rc, "%s", err);
  return MLT_OK;
}

}  // extern "C"

// ---- A12: surrogate device ---------------------------------------------------
namespace {

constexpr int kMaxTerms = 4096;

// The spec's launch rules as a second space (same parameters, its own rules);
// terms with their matched values mapped to digits (-1 = value not in the list).
int read_surrogate(const mlt_space* space, const mlt_surrogate* sp, const HostSpace& hs, HostSpace* lr,
                   std::vector<int>* tpos, std::vector<int>* tdig, std::vector<double>* tfac) {
  if (!sp) return fail(MLT_EINVAL, "surrogate spec is NULL");
  if (!(sp->base_time > 0)) return fail(MLT_EINVAL, "base_time must be strictly positive");
  if (sp->n_terms < 0 || sp->n_terms > kMaxTerms) return fail(MLT_EINVAL, "0..%d terms supported", kMaxTerms);
  if (!(sp->log_sigma >= 0)) return fail(MLT_EINVAL, "log_sigma must be non-negative");
  mlt_space ls = *space;
  ls.n_rules = sp->n_rules;
  ls.rule_kind = sp->rule_kind;
  ls.rule_nops = sp->rule_nops;
  ls.rule_pos = sp->rule_pos;
  ls.rule_coeff = sp->rule_coeff;
  ls.rule_bound = sp->rule_bound;
  TRY(read_space(&ls, lr));
  std::vector<int> voff(hs.P, 0);
  for (int p = 1; p < hs.P; ++p) voff[p] = voff[p - 1] + hs.radix[p - 1];
  auto digit_of = [&](int p, int64_t v) {
    for (int q = 0; q < hs.radix[p]; ++q)
      if (hs.values[voff[p] + q] == v) return q;
    return -1;
  };
  tpos->assign(2 * std::max(sp->n_terms, 1), -1);
  tdig->assign(2 * std::max(sp->n_terms, 1), -1);
  tfac->assign(std::max(sp->n_terms, 1), 1.0);
  for (int t = 0; t < sp->n_terms; ++t) {
    const int np = sp->term_nparams[t];
    if (np != 1 && np != 2) return fail(MLT_EINVAL, "term %d covers %d parameters (1 or 2 allowed)", t, np);
    if (!(sp->term_factor[t] > 0)) return fail(MLT_EINVAL, "term %d factor must be strictly positive", t);
    for (int j = 0; j < np; ++j) {
      const int p = sp->term_pos[2 * t + j];
      if (p < 0 || p >= hs.P) return fail(MLT_EINVAL, "term %d parameter position %d out of range", t, p);
      (*tpos)[2 * t + j] = p;
      (*tdig)[2 * t + j] = digit_of(p, sp->term_match[2 * t + j]);
    }
    if (np == 2 && ((*tdig)[2 * t] < 0 || (*tdig)[2 * t + 1] < 0)) (*tdig)[2 * t] = -1;
    if (np == 1) (*tdig)[2 * t + 1] = -1;
    (*tfac)[t] = sp->term_factor[t];
  }
  return MLT_OK;
}

// never-hitting terms keep their position but an impossible digit (-2 never equals a digit)
// Term-hit masks of the surrogate kernels (k_surr_best_runs, k_surr_times_masks):
// A[voff[p] + v] has bit t when term t's first (parameter, digit) is (p, v);
// B likewise for its second; one-parameter terms always pass B (b_ones).
// Terms whose value is not in the list never hit. Needs T <= 64.
void term_masks(const DSpace& d, int P, int T, const std::vector<int>& tpos, const std::vector<int>& tdig,
                std::vector<uint64_t>* masks, uint64_t* b_ones, int* nm) {
  *nm = d.voff[P - 1] + d.radix[P - 1];
  masks->assign(2 * (size_t)std::max(*nm, 1), 0);
  *b_ones = 0;
  for (int t = 0; t < T; ++t) {
    const int p1 = tpos[2 * t], d1 = tdig[2 * t], p2 = tpos[2 * t + 1], d2 = tdig[2 * t + 1];
    if (d1 < 0) continue;
    const uint64_t bit = 1ull << t;
    if (p2 < 0) {
      (*masks)[d.voff[p1] + d1] |= bit;
      *b_ones |= bit;
    } else if (d2 >= 0) {
      (*masks)[d.voff[p1] + d1] |= bit;
      (*masks)[*nm + d.voff[p2] + d2] |= bit;
    }
  }
}

int upload_surrogate(mlt_ctx* c, const mlt_surrogate* sp, int reps, std::vector<int>& tpos, std::vector<int>& tdig,
                     const std::vector<double>& tfac, DSurr* d, size_t* smem) {
  const int T = sp->n_terms;
  for (int t = 0; t < T; ++t)
    if (tdig[2 * t] < 0) tdig[2 * t] = -2;
  const size_t bytes = tfac.size() * 8 + tpos.size() * 4 * 2;
  char* buf;
  TRY(ws_t(c, S_SURR, bytes, &buf));
  CU(cudaMemcpyAsync(buf, tfac.data(), tfac.size() * 8, cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemcpyAsync(buf + tfac.size() * 8, tpos.data(), tpos.size() * 4, cudaMemcpyHostToDevice, c->stream));
  CU(cudaMemcpyAsync(buf + tfac.size() * 8 + tpos.size() * 4, tdig.data(), tdig.size() * 4, cudaMemcpyHostToDevice,
                     c->stream));
  d->base = sp->base_time;
  d->sigma = sp->log_sigma;
  d->seed = sp->seed;
  d->T = T;
  d->reps = reps;
  d->tfac = reinterpret_cast<const double*>(buf);
  d->tpos = reinterpret_cast<const int*>(buf + tfac.size() * 8);
  d->tdig = reinterpret_cast<const int*>(buf + tfac.size() * 8 + tpos.size() * 4);
  *smem = (size_t)T * (8 + 16);
  return MLT_OK;
}

}  // namespace

extern "C" {

int mlt_surrogate_times(mlt_ctx* c, const mlt_space* space, const mlt_surrogate* spec, const int64_t* idx, int64_t n,
                        int32_t reps, double* times, uint8_t* ok) {
  if (!c) return fail(MLT_EINVAL, "ctx is NULL");
  CTX_GUARD(c);
  if (n < 0) return fail(MLT_EINVAL, "negative count");
  if (reps < 0) return fail(MLT_EINVAL, "repetitions must be >= 0");
  CU(cudaSetDevice(c->dev));
  HostSpace hs, lr;
  TRY(read_space(space, &hs));
  std::vector<int> tpos, tdig;
  std::vector<double> tfac;
  TRY(read_surrogate(space, spec, hs, &lr, &tpos, &tdig, &tfac));
  if (n == 0) return MLT_OK;
  for (int64_t t = 0; t < n; ++t)
    if (idx[t] < 0 || idx[t] >= hs.card_i)
      return fail(MLT_EINVAL, "index %lld out of range for %lld configurations", (long long)idx[t],
                  (long long)hs.card_i);
  DSpace dl;
  TRY(upload_space(c, lr, &dl, S_L_VALUES, S_L_RPOS, S_L_RCOEFF));
  DSurr ds;
  size_t smem = 0;
  TRY(upload_surrogate(c, spec, reps, tpos, tdig, tfac, &ds, &smem));
  int64_t* di;
  double* dt;
  uint8_t* dok;
  TRY(ws_t(c, S_IDX, n, &di));
  TRY(ws_t(c, S_OUT_A, n, &dt));
  TRY(ws_t(c, S_OUT_C, n, &dok));
  CU(cudaMemcpyAsync(di, idx, n * 8, cudaMemcpyHostToDevice, c->stream));
  const int T = spec->n_terms;
  uint64_t* gmask = nullptr;
  if (T <= 64 && hs.P <= 16) {
    int nm = 0;
    std::vector<uint64_t> masks;
    uint64_t b_ones = 0;
    term_masks(dl, hs.P, T, tpos, tdig, &masks, &b_ones, &nm);
    CU(cudaMallocAsync(&gmask, masks.size() * 8, c->stream));
    TRY(upload_pinned(c, gmask, masks.data(), masks.size() * 8));
    const size_t smem_m = (size_t)T * 8 + (size_t)2 * nm * 8;
    if (smem_m > 48 * 1024)
      CU(cudaFuncSetAttribute(k_surr_times_masks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_m));
    k_surr_times_masks<<<grid_for(c, n, 256), 256, smem_m, c->stream>>>(dl, ds, gmask, nm, b_ones, di, n, dt, dok);
    CU(cudaFreeAsync(gmask, c->stream));
  } else {
    if (smem > 48 * 1024) CU(cudaFuncSetAttribute(k_surr_times, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_surr_times<<<grid_for(c, n, 256), 256, smem, c->stream>>>(dl, ds, di, n, dt, dok);
  }
  TRY(check_launch(c));
  CU(cudaMemcpyAsync(times, dt, n * 8, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaMemcpyAsync(ok, dok, n, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MLT_OK;
}

int mlt_surrogate_best(mlt_ctx* c, const mlt_space* space, const mlt_surrogate* spec, int64_t begin, int64_t end,
                       int32_t reps, double threshold, int64_t* best_idx, double* best_time, int64_t* n_valid,
                       int64_t* n_below) {
  if (!c || !best_idx || !best_time || !n_valid || !n_below) return fail(MLT_EINVAL, "NULL argument");
  CTX_GUARD(c);
  if (reps < 0) return fail(MLT_EINVAL, "repetitions must be >= 0");
  CU(cudaSetDevice(c->dev));
  HostSpace hs, lr;
  TRY(read_space(space, &hs));
  std::vector<int> tpos, tdig;
  std::vector<double> tfac;
  TRY(read_surrogate(space, spec, hs, &lr, &tpos, &tdig, &tfac));
  if (begin < 0 || end > hs.card_i || begin > end) return fail(MLT_EINVAL, "bad range [%lld, %lld)", (long long)begin,
                                                               (long long)end);
  *best_idx = -1;
  *best_time = std::nan("");
  *n_valid = *n_below = 0;
  if (begin == end) return MLT_OK;
  DSpace dsp, dl;
  TRY(upload_space(c, hs, &dsp));
  TRY(upload_space(c, lr, &dl, S_L_VALUES, S_L_RPOS, S_L_RCOEFF));
  DSurr ds;
  size_t smem = 0;
  TRY(upload_surrogate(c, spec, reps, tpos, tdig, tfac, &ds, &smem));
  const int threads = 256;
  const double thr = std::isnan(threshold) ? -HUGE_VAL : threshold;
  const int T = spec->n_terms;
  // <= 64 terms, <= 16 parameters: the odometer / hit-mask kernel
  const bool runs = T <= 64 && hs.P <= 16;
  const int run = 256;
  const int64_t units = runs ? (end - begin + run - 1) / run : end - begin;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((units + threads - 1) / threads, (int64_t)c->sms * 8));
  SurrPart* part;
  TRY(ws_t(c, S_PART, (size_t)grid + 1, &part));
  uint64_t* gmask = nullptr;
  if (runs) {
    int nm = 0;
    std::vector<uint64_t> masks;
    uint64_t b_ones = 0;
    term_masks(dsp, hs.P, T, tpos, tdig, &masks, &b_ones, &nm);
    CU(cudaMallocAsync(&gmask, masks.size() * 8, c->stream));
    TRY(upload_pinned(c, gmask, masks.data(), masks.size() * 8));
    const size_t smem_r = (size_t)T * 8 + (size_t)2 * nm * 8;
    if (smem_r > 48 * 1024)
      CU(cudaFuncSetAttribute(k_surr_best_runs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_r));
    k_surr_best_runs<<<grid, threads, smem_r, c->stream>>>(dsp, dl, ds, gmask, nm, b_ones, begin, end, run, thr, part);
    TRY(check_launch(c));
    CU(cudaFreeAsync(gmask, c->stream));
  } else {
    if (smem > 48 * 1024) CU(cudaFuncSetAttribute(k_surr_best, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_surr_best<<<grid, threads, smem, c->stream>>>(dsp, dl, ds, begin, end, thr, part);
    TRY(check_launch(c));
  }
  k_surr_best_final<<<1, 1024, 0, c->stream>>>(part, grid, part + grid);
  TRY(check_launch(c));
  SurrPart r;
  CU(cudaMemcpyAsync(&r, part + grid, sizeof r, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  *n_valid = r.n_valid;
  *n_below = r.n_below;
  if (r.n_valid > 0) {
    *best_idx = r.i;
    *best_time = r.t;
  }
  return MLT_OK;
}

}  // extern "C"
