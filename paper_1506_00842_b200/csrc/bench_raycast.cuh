// bench_raycast.cuh — shared declarations of the raycasting benchmark
// (bench_raycast.cu). The 160 kernel instances are compiled in 5 translation
// units (bench_raycast_u{1,2,4,8,16}.cu, one ray-loop unroll factor each) so
// the build parallelises; each explicitly instantiates ray_pick<U>.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mlt {

// Orthographic camera; every per-pixel quantity is derived from these floats
// with round-to-nearest fp32 operations in a fixed order (no contraction), so
// the numpy golden reproduces the rays bit-for-bit.
struct RayCamera {
  float c[3];      // image-plane centre (outside the volume)
  float u[3], v[3];// image-plane axes (unit)
  float w[3];      // ray direction (unit, every component non-zero)
  float inv[3];    // 1 / w
  float scale;     // world units per pixel
  float hw, hh;    // image width / 2, height / 2
  float thr;       // early-termination opacity
};

struct RayArgs {
  int IW, IH;                       // image
  int VX, VY, VZ;                   // volume (x fastest)
  const uint8_t* vol;               // [VZ][VY][VX]
  cudaTextureObject_t tex_vol;      // 3D u8 texture over a copy of vol
  const float4* tf;                 // transfer function, 256 RGBA entries (global)
  cudaTextureObject_t tex_tf;       // 1D float4 texture over tf
  float4* out;                      // IW x IH RGBA
  int pptx, ppty;
  RayCamera cam;
  // budgeted screening (mlt_raybench_set_budget): threads stop starting new
  // pixels once budget_ns has passed since *t0 (k_stamp right before the
  // launch); 0 = the normal measurement, every pixel rendered
  unsigned long long budget_ns;
  const unsigned long long* t0;
};

// the transfer function as a kernel-parameter (constant-bank) array
struct RayConstTF {
  float4 e[256];
};

typedef void (*RayKernel)(RayArgs, const __grid_constant__ RayConstTF);

// flags = img_data<<4 | img_transfer<<3 | local_transfer<<2 | const_transfer<<1 | interleaved
template <int U>
RayKernel ray_pick(int flags);

}  // namespace mlt
