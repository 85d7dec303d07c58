// bench_stereo.cu — the paper's tunable stereo-matching benchmark (SURVEY
// §8(a) A13, §8(f) next #1; Tables 1-2: disparity between two
// stereo images), written for sm_100a behind the runner protocol
// (measurement.py:250-258). The paper does not fix the matching cost, the
// disparity range or the window (SURVEY §7 "hard parts"); this benchmark
// uses, per output pixel (x, y),
//
//   disparity(x, y) = argmin_{0 <= d < D}  sum_{|dy|,|dx| <= R} |L(y+dy, x+dx) - R(y+dy, x+dx-d)|
//
// over 8-bit images with clamp-to-edge borders, ties to the smaller d
// (defaults D = 64, R = 4: a 9 x 9 window). Integer SAD, so every knob
// variant is bit-identical to the numpy golden of tests/.
//
//   knob               realisation on the B200
//   wg_x, wg_y         CTA shape (wg_x*wg_y > 1024 -> invalid-launch)
//   ppt_x, ppt_y       output pixels per thread in x / y (contiguous block per thread)
//   img_left/right     that image read through a u8 texture object (point, clamp)
//   local_left/right   that image's CTA tile (+ window halo, + D-1 columns for the right image)
//                      staged in shared memory (tiles > 227 KB -> invalid-launch)
//   unroll_disparity   unroll factor of the disparity loop (1, 2, 4, 8)
//   unroll_diff_x/y    unroll factors of the window loops (1, 2, 4); unroll_diff_x = 4 with
//                      both tiles in shared memory (9 x 9 window) compares 4 pixels per
//                      VABSDIFF4 with the left window rows held in registers
//
// 16 memory-placement combinations x 36 unroll combinations = 576 template
// instances (bench_stereo_kern.cuh, compiled in bench_stereo_p0..p7.cu); ppt
// and wg stay runtime values.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "bench_common.cuh"
#include "bench_stereo.cuh"
#include "mltune_b200.h"

namespace mlt {

static StereoKernel pick_stereo(int flags, int ud, int ux, int uy) {
  switch (flags) {
#define MLT_STEREO_CASE(f) \
  case f: return stereo_pick<((f) >> 3) & 1, ((f) >> 2) & 1, ((f) >> 1) & 1, (f) & 1>(ud, ux, uy);
    MLT_STEREO_CASE(0) MLT_STEREO_CASE(1) MLT_STEREO_CASE(2) MLT_STEREO_CASE(3)
    MLT_STEREO_CASE(4) MLT_STEREO_CASE(5) MLT_STEREO_CASE(6) MLT_STEREO_CASE(7)
    MLT_STEREO_CASE(8) MLT_STEREO_CASE(9) MLT_STEREO_CASE(10) MLT_STEREO_CASE(11)
    MLT_STEREO_CASE(12) MLT_STEREO_CASE(13) MLT_STEREO_CASE(14) MLT_STEREO_CASE(15)
#undef MLT_STEREO_CASE
  }
  return nullptr;
}

// Synthetic pair: a random 8-bit right image, and a left image that is the
// right image shifted by a piecewise-constant disparity field (4 x 4 blocks
// cycling through 4 levels within [D/8, D/8 + 3D/5]) plus +-2 noise.
__global__ void k_fill_right(uint8_t* right, int W, int H, uint64_t seed) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)W * H;
       q += (int64_t)gridDim.x * blockDim.x)
    right[q] = (uint8_t)(bench::hash_at(seed, (uint64_t)q) >> 56);
}

__global__ void k_fill_left(const uint8_t* right, uint8_t* left, int W, int H, int D, uint64_t seed) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)W * H;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(q / W), x = (int)(q % W);
    const int level = ((int)((int64_t)x * 4 / W) + (int)((int64_t)y * 4 / H)) & 3;
    const int disp = D / 8 + level * (D / 5);
    const int xs = min(max(x - disp, 0), W - 1);
    const int noise = (int)(bench::hash_at(seed ^ 0x5DEECE66Dull, (uint64_t)q) % 5) - 2;
    left[q] = (uint8_t)min(max((int)right[(size_t)y * W + xs] + noise, 0), 255);
  }
}

}  // namespace mlt

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
struct mlt_stereobench {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int W = 0, H = 0, D = 0, R = 0;
  uint8_t* left = nullptr;
  uint8_t* right = nullptr;
  uint8_t* out = nullptr;
  cudaArray_t arr_l = nullptr, arr_r = nullptr;
  cudaTextureObject_t tex_l = 0, tex_r = 0;
  mlt::bench::Timer timer;
  uint64_t budget_ns = 0;                  // mlt_stereobench_set_budget (0: normal measurement)
  unsigned long long* d_t0 = nullptr;      // its launch time stamp
};

namespace {
thread_local mlt::bench::ErrSlot g_serr;
#define CK(expr) MLT_BENCH_CK(g_serr, expr)
}  // namespace

extern "C" {

MLT_API const char* mlt_stereobench_last_error(void) { return g_serr.msg.c_str(); }

MLT_API int mlt_stereobench_create(int device, int32_t width, int32_t height, int32_t disparities, int32_t radius,
                                   const uint8_t* left, const uint8_t* right, uint64_t seed, mlt_stereobench** out) {
  using namespace mlt;
  if (!out) return g_serr.fail(MLT_EINVAL, "out is NULL");
  *out = nullptr;
  if (width < 1 || height < 1 || width > 32768 || height > 32768) return g_serr.fail(MLT_EINVAL, "bad image size");
  if (disparities < 1 || disparities > 256) return g_serr.fail(MLT_EINVAL, "disparities must be in [1, 256]");
  if (radius < 0 || radius > 32) return g_serr.fail(MLT_EINVAL, "window radius must be in [0, 32]");
  if ((left == nullptr) != (right == nullptr)) return g_serr.fail(MLT_EINVAL, "give both images or neither");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return g_serr.fail(MLT_ECUDA, "no CUDA device (no CPU fallback)");
  CK(cudaSetDevice(device));
  mlt_stereobench* b = new mlt_stereobench();
  b->dev = device;
  b->W = width;
  b->H = height;
  b->D = disparities;
  b->R = radius;
  CK(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
  const size_t px = (size_t)width * height;
  CK(cudaMalloc(&b->left, px));
  CK(cudaMalloc(&b->right, px));
  CK(cudaMalloc(&b->out, px));
  CK(cudaMemsetAsync(b->out, 0, px, b->stream));
  if (left) {
    CK(cudaMemcpyAsync(b->left, left, px, cudaMemcpyHostToDevice, b->stream));
    CK(cudaMemcpyAsync(b->right, right, px, cudaMemcpyHostToDevice, b->stream));
  } else {
    k_fill_right<<<1024, 256, 0, b->stream>>>(b->right, width, height, seed);
    k_fill_left<<<1024, 256, 0, b->stream>>>(b->right, b->left, width, height, disparities, seed);
    CK(cudaGetLastError());
  }
  int rc = bench::make_texture_2d(g_serr, b->left, width, height, &b->arr_l, &b->tex_l, b->stream);
  if (rc == MLT_OK) rc = bench::make_texture_2d(g_serr, b->right, width, height, &b->arr_r, &b->tex_r, b->stream);
  if (rc == MLT_OK) rc = b->timer.init(g_serr, b->stream);
  if (rc != MLT_OK) return rc;
  CK(cudaStreamSynchronize(b->stream));
  *out = b;
  return MLT_OK;
}

MLT_API int mlt_stereobench_destroy(mlt_stereobench* b) {
  if (!b) return MLT_OK;
  cudaSetDevice(b->dev);
  cudaStreamSynchronize(b->stream);
  cudaDestroyTextureObject(b->tex_l);
  cudaDestroyTextureObject(b->tex_r);
  cudaFreeArray(b->arr_l);
  cudaFreeArray(b->arr_r);
  cudaFree(b->left);
  cudaFree(b->right);
  cudaFree(b->out);
  if (b->d_t0) cudaFree(b->d_t0);
  b->timer.release();
  cudaStreamDestroy(b->stream);
  delete b;
  return MLT_OK;
}

// Budgeted screening for exhaustive sweeps (see mlt_raybench_set_budget).
MLT_API int mlt_stereobench_set_budget(mlt_stereobench* b, uint64_t budget_ns) {
  if (!b) return g_serr.fail(MLT_EINVAL, "NULL argument");
  CK(cudaSetDevice(b->dev));
  if (budget_ns && !b->d_t0) CK(cudaMalloc(&b->d_t0, sizeof(unsigned long long)));
  b->budget_ns = budget_ns;
  return MLT_OK;
}

// knobs = {wg_x, wg_y, ppt_x, ppt_y, img_left, img_right, local_left, local_right,
//          unroll_disparity, unroll_diff_x, unroll_diff_y}  (paramspace.py:320-329 order)
MLT_API int mlt_stereobench_run(mlt_stereobench* b, const int32_t* knobs, int32_t reps, double* seconds,
                                int32_t* status) {
  using namespace mlt;
  if (!b || !knobs || !seconds || !status) return g_serr.fail(MLT_EINVAL, "NULL argument");
  if (reps < 1) return g_serr.fail(MLT_EINVAL, "repetitions must be >= 1");
  CK(cudaSetDevice(b->dev));
  const int wgx = knobs[0], wgy = knobs[1], pptx = knobs[2], ppty = knobs[3];
  const int flags = ((knobs[4] != 0) << 3) | ((knobs[5] != 0) << 2) | ((knobs[6] != 0) << 1) | (knobs[7] != 0);
  const int ud = knobs[8], ux = knobs[9], uy = knobs[10];
  *status = 0;
  *seconds = 0;
  if (wgx < 1 || wgy < 1 || pptx < 1 || ppty < 1) return g_serr.fail(MLT_EINVAL, "non-positive knob");
  if ((ud != 1 && ud != 2 && ud != 4 && ud != 8) || (ux != 1 && ux != 2 && ux != 4) || (uy != 1 && uy != 2 && uy != 4))
    return g_serr.fail(MLT_EINVAL, "unroll factors: disparity in {1,2,4,8}, diff_x/diff_y in {1,2,4}");
  const int64_t bw = (int64_t)wgx * pptx, bh = (int64_t)wgy * ppty;
  const int64_t gx = (b->W + bw - 1) / bw, gy = (b->H + bh - 1) / bh;
  const int64_t th = bh + 2 * b->R;
  // (+16 bytes: the packed path reads up to one aligned word past the last row)
  const size_t smem = (size_t)(((flags >> 1) & 1) ? (bw + 2 * b->R) * th : 0) +
                      (size_t)((flags & 1) ? (bw + 2 * b->R + b->D - 1) * th : 0) + 16;
  if ((int64_t)wgx * wgy > 1024 || wgy > 1024 || smem > bench::kMaxSmem || gy > 65535) {
    *status = 1;
    return MLT_OK;
  }
  StereoKernel k = pick_stereo(flags, ud, ux, uy);
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  StereoArgs a;
  a.W = b->W;
  a.H = b->H;
  a.D = b->D;
  a.R = b->R;
  a.left = b->left;
  a.right = b->right;
  a.tex_left = b->tex_l;
  a.tex_right = b->tex_r;
  a.out = b->out;
  a.pptx = pptx;
  a.ppty = ppty;
  a.budget_ns = b->budget_ns;
  a.t0 = b->d_t0;
  return b->timer.run(g_serr, reps, [&]() {
    if (b->budget_ns) bench::k_stamp<<<1, 1, 0, b->stream>>>(b->d_t0);
    k<<<dim3((unsigned)gx, (unsigned)gy), dim3(wgx, wgy), smem, b->stream>>>(a);
    return cudaGetLastError();
  }, seconds, status);
}

MLT_API int mlt_stereobench_output(mlt_stereobench* b, uint8_t* host_disparity) {
  if (!b || !host_disparity) return g_serr.fail(MLT_EINVAL, "NULL argument");
  CK(cudaSetDevice(b->dev));
  CK(cudaMemcpyAsync(host_disparity, b->out, (size_t)b->W * b->H, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return MLT_OK;
}

MLT_API int mlt_stereobench_input(mlt_stereobench* b, uint8_t* host_left, uint8_t* host_right) {
  if (!b || !host_left || !host_right) return g_serr.fail(MLT_EINVAL, "NULL argument");
  CK(cudaSetDevice(b->dev));
  CK(cudaMemcpyAsync(host_left, b->left, (size_t)b->W * b->H, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaMemcpyAsync(host_right, b->right, (size_t)b->W * b->H, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return MLT_OK;
}

}  // extern "C"
