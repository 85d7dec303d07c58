// bench_common.cuh — pieces shared by the sm_100a benchmark kernels (the
// devices under tuning: bench_conv.cu, bench_stereo.cu, bench_raycast.cu).
// The reference has only the seam for these (ExternalRunner / runner.measure,
// measurement.py:274-348): timing follows its rules —
// minimum over repetitions (measurement.py:337-348) — on CUDA events, with
// the L2 flushed before every repetition.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "mltune_b200.h"

namespace mlt {
namespace bench {

constexpr size_t kFlushBytes = size_t(256) << 20;   // > 126 MB L2
constexpr size_t kMaxSmem = 227 * 1024;              // opt-in dynamic smem per CTA on sm_100

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// hash of (seed, element q): the synthetic-input generator of every benchmark
__device__ __forceinline__ uint64_t hash_at(uint64_t seed, uint64_t q) {
  return splitmix64(seed + 0x9E3779B97F4A7C15ull * (q + 1));
}

// %globaltimer (ns): the budgeted measurement mode's clock
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// the launch time stamp a budgeted kernel measures its budget from
static __global__ void k_stamp(unsigned long long* t0) { *t0 = gtimer(); }

static __global__ void k_flush_l2(uint4* buf, size_t n, uint32_t v) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x)
    buf[q] = make_uint4(v, v, v, v);
}

// Per-benchmark error slot + CUDA check macro (int-returning C-ABI functions).
struct ErrSlot {
  std::string msg;
  int fail(int code, const std::string& m) {
    msg = m;
    return code;
  }
};

#define MLT_BENCH_CK(slot, expr)                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess) return (slot).fail(MLT_ECUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

// 2D texture over a cudaArray copy of a device image: point sampling, clamp
// addressing, unnormalised coordinates (hardware linear filtering would
// quantise the weights to 8 bits and break the output tolerance).
template <typename T>
static int make_texture_2d(ErrSlot& es, const T* src, int w, int h, cudaArray_t* arr, cudaTextureObject_t* tex,
                           cudaStream_t s) {
  cudaChannelFormatDesc cd = cudaCreateChannelDesc<T>();
  MLT_BENCH_CK(es, cudaMallocArray(arr, &cd, w, h));
  MLT_BENCH_CK(es, cudaMemcpy2DToArrayAsync(*arr, 0, 0, src, (size_t)w * sizeof(T), (size_t)w * sizeof(T), h,
                                            cudaMemcpyDeviceToDevice, s));
  cudaResourceDesc rd;
  std::memset(&rd, 0, sizeof rd);
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = *arr;
  cudaTextureDesc td;
  std::memset(&td, 0, sizeof td);
  td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  MLT_BENCH_CK(es, cudaCreateTextureObject(tex, &rd, &td, nullptr));
  return MLT_OK;
}

// Event-timed repetitions of one launch: min over `reps`, L2 flushed before
// each. `launch` returns the cudaError_t of its launch; configuration errors
// (too many threads / registers / smem) report invalid-launch via *status = 1.
struct Timer {
  cudaStream_t stream = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  void* flush = nullptr;
  size_t flush_n = 0;
  int64_t launches = 0;

  int init(ErrSlot& es, cudaStream_t s) {
    stream = s;
    flush_n = kFlushBytes / 16;
    MLT_BENCH_CK(es, cudaMalloc(&flush, flush_n * 16));
    MLT_BENCH_CK(es, cudaEventCreate(&e0));
    MLT_BENCH_CK(es, cudaEventCreate(&e1));
    return MLT_OK;
  }
  void release() {
    cudaFree(flush);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    flush = nullptr;
    e0 = e1 = nullptr;
  }
  template <typename F>
  int run(ErrSlot& es, int reps, F&& launch, double* seconds, int32_t* status) {
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
      k_flush_l2<<<1024, 256, 0, stream>>>(static_cast<uint4*>(flush), flush_n, (uint32_t)r);
      MLT_BENCH_CK(es, cudaEventRecord(e0, stream));
      const cudaError_t le = launch();
      if (le == cudaErrorInvalidConfiguration || le == cudaErrorLaunchOutOfResources) {
        *status = 1;
        *seconds = 0;
        return MLT_OK;
      }
      if (le != cudaSuccess) return es.fail(MLT_ECUDA, std::string("benchmark launch: ") + cudaGetErrorString(le));
      MLT_BENCH_CK(es, cudaEventRecord(e1, stream));
      MLT_BENCH_CK(es, cudaEventSynchronize(e1));
      float ms = 0;
      MLT_BENCH_CK(es, cudaEventElapsedTime(&ms, e0, e1));
      launches += 2;
      if (ms * 1e-3 < best) best = ms * 1e-3;
    }
    *status = 0;
    *seconds = best;
    return MLT_OK;
  }
};

}  // namespace bench
}  // namespace mlt
