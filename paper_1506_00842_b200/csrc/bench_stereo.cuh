// bench_stereo.cuh — shared declarations of the stereo benchmark (bench_stereo.cu).
// The 576 kernel instances are compiled in 8 translation units
// (bench_stereo_p0..p7.cu, two memory-placement combinations each) so the
// build parallelises; each explicitly instantiates stereo_pick<> for its combos.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mlt {

struct StereoArgs {
  int W, H, D, R;
  const uint8_t* left;
  const uint8_t* right;
  cudaTextureObject_t tex_left, tex_right;
  uint8_t* out;
  int pptx, ppty;
  // budgeted screening (mlt_stereobench_set_budget): threads stop starting new
  // pixels once budget_ns has passed since *t0; 0 = the normal measurement
  unsigned long long budget_ns;
  const unsigned long long* t0;
};

typedef void (*StereoKernel)(StereoArgs);

// the k_stereo instance for (img_left, img_right, local_left, local_right) and the
// unroll factors (disparity 1/2/4/8, diff_x 1/2/4, diff_y 1/2/4)
template <bool IL, bool IR, bool LL, bool LR>
StereoKernel stereo_pick(int ud, int ux, int uy);

}  // namespace mlt
