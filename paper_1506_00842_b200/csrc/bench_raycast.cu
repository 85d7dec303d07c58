// bench_raycast.cu — the paper's tunable volume raycasting benchmark (SURVEY
// §8(a) A13, §8(f) next #1; Tables 1-2: a 1024 x 1024 image from a
// 512^3 volume), written for sm_100a behind the runner protocol
// (measurement.py:250-258). The paper fixes neither the camera nor the
// transfer function; this benchmark casts one orthographic ray per pixel
// (RayCamera), steps it through the volume box at unit spacing from the slab
// entry, samples the nearest voxel (8-bit), maps it through a 256-entry RGBA
// transfer function and composites front to back until the opacity reaches
// `thr` (0.95). All arithmetic is round-to-nearest fp32 in a fixed order, so
// every knob variant is bit-identical to the numpy golden of tests/.
//
//   knob              realisation on the B200
//   wg_x, wg_y        CTA shape (wg_x*wg_y > 1024 -> invalid-launch)
//   ppt_x, ppt_y      output pixels per thread in x / y
//   img_data          volume read through a 3D u8 texture object (point sampling)
//   img_transfer      transfer function read through a 1D float4 texture
//   local_transfer    transfer function staged in shared memory by each CTA
//                     (from the texture / constant / global source selected by the other flags)
//   const_transfer    transfer function in the constant bank (a __grid_constant__
//                     kernel parameter; the texture wins when img_transfer is also set)
//   interleaved       a thread's pixels are strided by the CTA width instead of contiguous
//   unroll_ray        ray loop unrolled U = 1, 2, 4, 8, 16 steps: U independent
//                     voxel gathers issued before the U compositing steps
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

#include "bench_common.cuh"
#include "bench_raycast.cuh"
#include "mltune_b200.h"

namespace mlt {

static RayKernel pick_raycast(int flags, int unroll) {
  switch (unroll) {
    case 1: return ray_pick<1>(flags);
    case 2: return ray_pick<2>(flags);
    case 4: return ray_pick<4>(flags);
    case 8: return ray_pick<8>(flags);
    case 16: return ray_pick<16>(flags);
  }
  return nullptr;
}

// Synthetic volume: five soft blobs and a spherical shell over low-amplitude
// hash noise, quantised to 8 bits.
__global__ void k_fill_volume(uint8_t* vol, int VX, int VY, int VZ, uint64_t seed) {
  const float cx[5] = {0.30f, 0.70f, 0.50f, 0.35f, 0.68f}, cy[5] = {0.35f, 0.40f, 0.70f, 0.65f, 0.62f},
              cz[5] = {0.40f, 0.55f, 0.45f, 0.70f, 0.30f}, rr[5] = {0.12f, 0.10f, 0.14f, 0.08f, 0.09f},
              amp[5] = {0.9f, 0.7f, 0.6f, 1.0f, 0.8f};
  const int64_t n = (int64_t)VX * VY * VZ;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(q % VX), y = (int)((q / VX) % VY), z = (int)(q / ((int64_t)VX * VY));
    const float px = (x + 0.5f) / VX, py = (y + 0.5f) / VY, pz = (z + 0.5f) / VZ;
    float d = 0.f;
    for (int k = 0; k < 5; ++k) {
      const float dx = px - cx[k], dy = py - cy[k], dz = pz - cz[k];
      d += amp[k] * __expf(-(dx * dx + dy * dy + dz * dz) / (rr[k] * rr[k]));
    }
    const float rad = sqrtf((px - 0.5f) * (px - 0.5f) + (py - 0.5f) * (py - 0.5f) + (pz - 0.5f) * (pz - 0.5f));
    d += 0.5f * __expf(-(rad - 0.42f) * (rad - 0.42f) / 0.0004f);
    d += 0.12f * (float)(bench::hash_at(seed, (uint64_t)q) >> 40) * (1.0f / 16777216.0f);
    vol[q] = (uint8_t)fminf(255.f, d * 200.f);
  }
}

// Default transfer function: transparent below 15 % density, then a rising
// opacity ramp; colour runs blue -> green -> red with density.
static void default_transfer(float* tf) {
  for (int s = 0; s < 256; ++s) {
    const double x = s / 255.0;
    const double a = x < 0.15 ? 0.0 : 0.10 * std::pow((x - 0.15) / 0.85, 1.5);
    tf[4 * s + 0] = (float)x;
    tf[4 * s + 1] = (float)(0.5 + 0.5 * std::sin(6.283185307179586 * x));
    tf[4 * s + 2] = (float)(1.0 - x);
    tf[4 * s + 3] = (float)a;
  }
}

// Orthographic view from yaw 30 deg / pitch 20 deg, image plane covering the
// volume's diagonal; plane centre one diagonal away from the volume centre.
static RayCamera default_camera(int IW, int IH, int VX, int VY, int VZ) {
  const double yaw = 0.5235987755982988, pitch = 0.3490658503988659;
  const double w[3] = {std::sin(yaw) * std::cos(pitch), std::sin(pitch), std::cos(yaw) * std::cos(pitch)};
  const double u[3] = {std::cos(yaw), 0.0, -std::sin(yaw)};
  double v[3] = {w[1] * u[2] - w[2] * u[1], w[2] * u[0] - w[0] * u[2], w[0] * u[1] - w[1] * u[0]};
  const double vn = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  const double diag = std::sqrt((double)VX * VX + (double)VY * VY + (double)VZ * VZ);
  const double ctr[3] = {VX / 2.0, VY / 2.0, VZ / 2.0};
  RayCamera c;
  for (int i = 0; i < 3; ++i) {
    c.w[i] = (float)w[i];
    c.u[i] = (float)u[i];
    c.v[i] = (float)(v[i] / vn);
    c.c[i] = (float)(ctr[i] - w[i] * diag);
    c.inv[i] = 1.0f / c.w[i];
  }
  c.scale = (float)(diag / (IW < IH ? IW : IH));
  c.hw = IW * 0.5f;
  c.hh = IH * 0.5f;
  c.thr = 0.95f;
  return c;
}

}  // namespace mlt

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
struct mlt_raybench {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int IW = 0, IH = 0, VX = 0, VY = 0, VZ = 0;
  uint8_t* vol = nullptr;
  float4* tf = nullptr;
  float4* out = nullptr;
  cudaArray_t arr_vol = nullptr;
  cudaTextureObject_t tex_vol = 0, tex_tf = 0;
  float tf_host[1024];
  mlt::RayCamera cam;
  mlt::bench::Timer timer;
  uint64_t budget_ns = 0;                  // mlt_raybench_set_budget (0: normal measurement)
  unsigned long long* d_t0 = nullptr;      // its launch time stamp
};

namespace {
thread_local mlt::bench::ErrSlot g_rerr;
#define CK(expr) MLT_BENCH_CK(g_rerr, expr)
}  // namespace

extern "C" {

MLT_API const char* mlt_raybench_last_error(void) { return g_rerr.msg.c_str(); }

MLT_API int mlt_raybench_create(int device, int32_t image_w, int32_t image_h, int32_t vx, int32_t vy, int32_t vz,
                                const uint8_t* volume, const float* transfer, uint64_t seed, mlt_raybench** out) {
  using namespace mlt;
  if (!out) return g_rerr.fail(MLT_EINVAL, "out is NULL");
  *out = nullptr;
  if (image_w < 1 || image_h < 1 || image_w > 16384 || image_h > 16384) return g_rerr.fail(MLT_EINVAL, "bad image size");
  if (vx < 1 || vy < 1 || vz < 1 || vx > 2048 || vy > 2048 || vz > 2048) return g_rerr.fail(MLT_EINVAL, "bad volume size");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return g_rerr.fail(MLT_ECUDA, "no CUDA device (no CPU fallback)");
  CK(cudaSetDevice(device));
  mlt_raybench* b = new mlt_raybench();
  b->dev = device;
  b->IW = image_w;
  b->IH = image_h;
  b->VX = vx;
  b->VY = vy;
  b->VZ = vz;
  if (transfer) std::memcpy(b->tf_host, transfer, sizeof b->tf_host);
  else default_transfer(b->tf_host);
  b->cam = default_camera(image_w, image_h, vx, vy, vz);
  CK(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
  const size_t nv = (size_t)vx * vy * vz, px = (size_t)image_w * image_h;
  CK(cudaMalloc(&b->vol, nv));
  CK(cudaMalloc(&b->tf, 256 * sizeof(float4)));
  CK(cudaMalloc(&b->out, px * sizeof(float4)));
  CK(cudaMemsetAsync(b->out, 0, px * sizeof(float4), b->stream));
  CK(cudaMemcpyAsync(b->tf, b->tf_host, sizeof b->tf_host, cudaMemcpyHostToDevice, b->stream));
  if (volume) {
    CK(cudaMemcpyAsync(b->vol, volume, nv, cudaMemcpyHostToDevice, b->stream));
  } else {
    k_fill_volume<<<2048, 256, 0, b->stream>>>(b->vol, vx, vy, vz, seed);
    CK(cudaGetLastError());
  }
  // 3D texture over a cudaArray copy of the volume
  cudaChannelFormatDesc cd = cudaCreateChannelDesc<unsigned char>();
  CK(cudaMalloc3DArray(&b->arr_vol, &cd, make_cudaExtent(vx, vy, vz)));
  cudaMemcpy3DParms cp;
  std::memset(&cp, 0, sizeof cp);
  cp.srcPtr = make_cudaPitchedPtr(b->vol, (size_t)vx, (size_t)vx, (size_t)vy);
  cp.dstArray = b->arr_vol;
  cp.extent = make_cudaExtent(vx, vy, vz);
  cp.kind = cudaMemcpyDeviceToDevice;
  CK(cudaMemcpy3DAsync(&cp, b->stream));
  cudaResourceDesc rd;
  std::memset(&rd, 0, sizeof rd);
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = b->arr_vol;
  cudaTextureDesc td;
  std::memset(&td, 0, sizeof td);
  td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  CK(cudaCreateTextureObject(&b->tex_vol, &rd, &td, nullptr));
  // 1D float4 texture over the transfer function
  std::memset(&rd, 0, sizeof rd);
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = b->tf;
  rd.res.linear.desc = cudaCreateChannelDesc<float4>();
  rd.res.linear.sizeInBytes = 256 * sizeof(float4);
  std::memset(&td, 0, sizeof td);
  td.readMode = cudaReadModeElementType;
  CK(cudaCreateTextureObject(&b->tex_tf, &rd, &td, nullptr));
  const int rc = b->timer.init(g_rerr, b->stream);
  if (rc != MLT_OK) return rc;
  CK(cudaStreamSynchronize(b->stream));
  *out = b;
  return MLT_OK;
}

MLT_API int mlt_raybench_destroy(mlt_raybench* b) {
  if (!b) return MLT_OK;
  cudaSetDevice(b->dev);
  cudaStreamSynchronize(b->stream);
  cudaDestroyTextureObject(b->tex_vol);
  cudaDestroyTextureObject(b->tex_tf);
  cudaFreeArray(b->arr_vol);
  cudaFree(b->vol);
  cudaFree(b->tf);
  cudaFree(b->out);
  if (b->d_t0) cudaFree(b->d_t0);
  b->timer.release();
  cudaStreamDestroy(b->stream);
  delete b;
  return MLT_OK;
}

// Budgeted screening for exhaustive sweeps over the raycasting space: with
// budget_ns > 0 every launch stops starting new pixels budget_ns after it
// began, so a configuration slower than the budget costs about the budget
// (its measured time is then >= budget_ns: "slower than the budget", not a
// time); faster ones render completely and time as usual. 0 restores the
// normal measurement. The image is only complete for unaborted launches.
MLT_API int mlt_raybench_set_budget(mlt_raybench* b, uint64_t budget_ns) {
  if (!b) return g_rerr.fail(MLT_EINVAL, "NULL argument");
  CK(cudaSetDevice(b->dev));
  if (budget_ns && !b->d_t0) CK(cudaMalloc(&b->d_t0, sizeof(unsigned long long)));
  b->budget_ns = budget_ns;
  return MLT_OK;
}

// knobs = {wg_x, wg_y, ppt_x, ppt_y, img_data, img_transfer, local_transfer, const_transfer,
//          interleaved, unroll_ray}  (paramspace.py:311-319 order)
MLT_API int mlt_raybench_run(mlt_raybench* b, const int32_t* knobs, int32_t reps, double* seconds, int32_t* status) {
  using namespace mlt;
  if (!b || !knobs || !seconds || !status) return g_rerr.fail(MLT_EINVAL, "NULL argument");
  if (reps < 1) return g_rerr.fail(MLT_EINVAL, "repetitions must be >= 1");
  CK(cudaSetDevice(b->dev));
  const int wgx = knobs[0], wgy = knobs[1], pptx = knobs[2], ppty = knobs[3];
  int flags = 0;
  for (int i = 4; i < 9; ++i) flags = (flags << 1) | (knobs[i] != 0);
  const int unroll = knobs[9];
  *status = 0;
  *seconds = 0;
  if (wgx < 1 || wgy < 1 || pptx < 1 || ppty < 1) return g_rerr.fail(MLT_EINVAL, "non-positive knob");
  RayKernel k = pick_raycast(flags, unroll);
  if (!k) return g_rerr.fail(MLT_EINVAL, "unroll_ray must be one of 1, 2, 4, 8, 16");
  const int64_t bw = (int64_t)wgx * pptx, bh = (int64_t)wgy * ppty;
  const int64_t gx = (b->IW + bw - 1) / bw, gy = (b->IH + bh - 1) / bh;
  if ((int64_t)wgx * wgy > 1024 || wgy > 1024 || gy > 65535) {
    *status = 1;
    return MLT_OK;
  }
  RayArgs a;
  a.IW = b->IW;
  a.IH = b->IH;
  a.VX = b->VX;
  a.VY = b->VY;
  a.VZ = b->VZ;
  a.vol = b->vol;
  a.tex_vol = b->tex_vol;
  a.tf = b->tf;
  a.tex_tf = b->tex_tf;
  a.out = b->out;
  a.pptx = pptx;
  a.ppty = ppty;
  a.cam = b->cam;
  a.budget_ns = b->budget_ns;
  a.t0 = b->d_t0;
  RayConstTF ctf;
  std::memcpy(ctf.e, b->tf_host, sizeof ctf.e);
  return b->timer.run(g_rerr, reps, [&]() {
    if (b->budget_ns) bench::k_stamp<<<1, 1, 0, b->stream>>>(b->d_t0);
    k<<<dim3((unsigned)gx, (unsigned)gy), dim3(wgx, wgy), 0, b->stream>>>(a, ctf);
    return cudaGetLastError();
  }, seconds, status);
}

MLT_API int mlt_raybench_output(mlt_raybench* b, float* host_rgba) {
  if (!b || !host_rgba) return g_rerr.fail(MLT_EINVAL, "NULL argument");
  CK(cudaSetDevice(b->dev));
  CK(cudaMemcpyAsync(host_rgba, b->out, (size_t)b->IW * b->IH * sizeof(float4), cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return MLT_OK;
}

MLT_API int mlt_raybench_volume(mlt_raybench* b, uint8_t* host_volume) {
  if (!b || !host_volume) return g_rerr.fail(MLT_EINVAL, "NULL argument");
  CK(cudaSetDevice(b->dev));
  CK(cudaMemcpyAsync(host_volume, b->vol, (size_t)b->VX * b->VY * b->VZ, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return MLT_OK;
}

MLT_API int mlt_raybench_transfer(mlt_raybench* b, float* host_rgba256) {
  if (!b || !host_rgba256) return g_rerr.fail(MLT_EINVAL, "NULL argument");
  std::memcpy(host_rgba256, b->tf_host, sizeof b->tf_host);
  return MLT_OK;
}

// 19 floats: c[3], u[3], v[3], w[3], inv[3], scale, hw, hh, thr
MLT_API int mlt_raybench_camera(mlt_raybench* b, float* host_cam19) {
  if (!b || !host_cam19) return g_rerr.fail(MLT_EINVAL, "NULL argument");
  const mlt::RayCamera& c = b->cam;
  for (int i = 0; i < 3; ++i) {
    host_cam19[i] = c.c[i];
    host_cam19[3 + i] = c.u[i];
    host_cam19[6 + i] = c.v[i];
    host_cam19[9 + i] = c.w[i];
    host_cam19[12 + i] = c.inv[i];
  }
  host_cam19[15] = c.scale;
  host_cam19[16] = c.hw;
  host_cam19[17] = c.hh;
  host_cam19[18] = c.thr;
  return MLT_OK;
}

}  // extern "C"
