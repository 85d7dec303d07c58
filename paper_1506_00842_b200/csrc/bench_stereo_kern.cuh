// bench_stereo_kern.cuh — the stereo-matching kernel template (see bench_stereo.cu
// for the cost function and the knob mapping). Included only by bench_stereo_p*.cu.
#pragma once

#include "bench_common.cuh"
#include "bench_stereo.cuh"

namespace mlt {

template <bool IMG>
__device__ __forceinline__ unsigned fetch_u8(const uint8_t* img, cudaTextureObject_t tex, int W, int H, int y, int x) {
  if (IMG) return tex2D<unsigned char>(tex, (float)x + 0.5f, (float)y + 0.5f);   // clamp addressing
  const int yy = min(max(y, 0), H - 1), xx = min(max(x, 0), W - 1);
  return __ldg(img + (size_t)yy * W + xx);
}

// Three 4-byte words of a shared-memory row starting at byte `p` (any
// alignment): four aligned 32-bit loads and three funnel shifts.
__device__ __forceinline__ void ld12(const uint8_t* p, unsigned& w0, unsigned& w1, unsigned& w2) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const unsigned* w = reinterpret_cast<const unsigned*>(a & ~uintptr_t(3));
  const unsigned sh = (unsigned)(a & 3) * 8;
  const unsigned x0 = w[0], x1 = w[1], x2 = w[2], x3 = w[3];
  w0 = __funnelshift_r(x0, x1, sh);
  w1 = __funnelshift_r(x1, x2, sh);
  w2 = __funnelshift_r(x2, x3, sh);
}

template <bool IL, bool IR, bool LL, bool LR, int UD, int UX, int UY>
__global__ void k_stereo(StereoArgs a) {
  extern __shared__ uint8_t smem[];
  const int wgx = blockDim.x, wgy = blockDim.y;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int bw = wgx * a.pptx, bh = wgy * a.ppty;
  const int X0 = blockIdx.x * bw, Y0 = blockIdx.y * bh;
  const int R = a.R, D = a.D;
  const int th = bh + 2 * R;
  const int twl = bw + 2 * R;                 // left tile: the window halo
  const int twr = bw + 2 * R + D - 1;         // right tile: halo + the disparity range
  uint8_t* tl = smem;
  uint8_t* tr = smem + (LL ? twl * th : 0);
  if (LL || LR) {
    const int nt = wgx * wgy;
    if (LL)
      for (int q = ty * wgx + tx; q < twl * th; q += nt) {
        const int r = q / twl, c = q - r * twl;
        tl[q] = (uint8_t)fetch_u8<IL>(a.left, a.tex_left, a.W, a.H, Y0 - R + r, X0 - R + c);
      }
    if (LR)
      for (int q = ty * wgx + tx; q < twr * th; q += nt) {
        const int r = q / twr, c = q - r * twr;
        tr[q] = (uint8_t)fetch_u8<IR>(a.right, a.tex_right, a.W, a.H, Y0 - R + r, X0 - R - (D - 1) + c);
      }
    __syncthreads();
  }
  const unsigned long long start = a.budget_ns ? *a.t0 : 0ull;
  for (int iy = 0; iy < a.ppty; ++iy) {
    const int ly = ty * a.ppty + iy;
    const int y = Y0 + ly;
    if (y >= a.H) break;
    for (int ix = 0; ix < a.pptx; ++ix) {
      const int lx = tx * a.pptx + ix;
      const int x = X0 + lx;
      if (x >= a.W) break;
      if (a.budget_ns && bench::gtimer() - start > a.budget_ns) return;   // screening: over budget
      unsigned best = 0xffffffffu;
      int bd = 0;
      if (LL && LR && UX == 4 && R == 4) {
        // unroll_diff_x = 4 with both tiles in shared memory (9 x 9 window):
        // each window row is 9 bytes = 2 packed words + 1 byte, compared with
        // VABSDIFF4 (4 pixels per instruction); the left rows are loaded once
        // per pixel, the right rows once per (disparity, row). Integer sums:
        // the same values as the byte-wise loop.
        unsigned lw[9][3];
#pragma unroll
        for (int r = 0; r < 9; ++r) {
          ld12(tl + (ly + r) * twl + lx, lw[r][0], lw[r][1], lw[r][2]);
          lw[r][2] &= 0xffu;
        }
        const uint8_t* rbase = tr + ly * twr + lx + D - 1;
#pragma unroll UD
        for (int d = 0; d < D; ++d) {
          unsigned s = 0;
#pragma unroll      // fully: the left words stay in registers (unroll_diff_y acts on the byte path)
          for (int r = 0; r < 9; ++r) {
            unsigned r0, r1, r2;
            ld12(rbase + r * twr - d, r0, r1, r2);
            s = __vsadu4(lw[r][0], r0) + s;
            s = __vsadu4(lw[r][1], r1) + s;
            s = __vsadu4(lw[r][2], r2 & 0xffu) + s;
          }
          if (s < best) {
            best = s;
            bd = d;
          }
        }
        a.out[(size_t)y * a.W + x] = (uint8_t)bd;
        continue;
      }
#pragma unroll UD
      for (int d = 0; d < D; ++d) {
        unsigned s = 0;
#pragma unroll UY
        for (int dy = -R; dy <= R; ++dy) {
#pragma unroll UX
          for (int dx = -R; dx <= R; ++dx) {
            const unsigned l = LL ? (unsigned)tl[(ly + R + dy) * twl + (lx + R + dx)]
                                  : fetch_u8<IL>(a.left, a.tex_left, a.W, a.H, y + dy, x + dx);
            const unsigned r = LR ? (unsigned)tr[(ly + R + dy) * twr + (lx + R + D - 1 + dx - d)]
                                  : fetch_u8<IR>(a.right, a.tex_right, a.W, a.H, y + dy, x + dx - d);
            s = __usad(l, r, s);
          }
        }
        if (s < best) {
          best = s;
          bd = d;
        }
      }
      a.out[(size_t)y * a.W + x] = (uint8_t)bd;
    }
  }
}

template <bool IL, bool IR, bool LL, bool LR, int UD>
struct StereoRow {   // the 9 (unroll_diff_x, unroll_diff_y) instances
  static constexpr StereoKernel k[9] = {
      k_stereo<IL, IR, LL, LR, UD, 1, 1>, k_stereo<IL, IR, LL, LR, UD, 1, 2>, k_stereo<IL, IR, LL, LR, UD, 1, 4>,
      k_stereo<IL, IR, LL, LR, UD, 2, 1>, k_stereo<IL, IR, LL, LR, UD, 2, 2>, k_stereo<IL, IR, LL, LR, UD, 2, 4>,
      k_stereo<IL, IR, LL, LR, UD, 4, 1>, k_stereo<IL, IR, LL, LR, UD, 4, 2>, k_stereo<IL, IR, LL, LR, UD, 4, 4>};
};

template <bool IL, bool IR, bool LL, bool LR>
StereoKernel stereo_pick(int ud, int ux, int uy) {
  const int j = (ux == 1 ? 0 : ux == 2 ? 1 : 2) * 3 + (uy == 1 ? 0 : uy == 2 ? 1 : 2);
  switch (ud) {
    case 1: return StereoRow<IL, IR, LL, LR, 1>::k[j];
    case 2: return StereoRow<IL, IR, LL, LR, 2>::k[j];
    case 4: return StereoRow<IL, IR, LL, LR, 4>::k[j];
    default: return StereoRow<IL, IR, LL, LR, 8>::k[j];
  }
}

}  // namespace mlt

#define MLT_STEREO_INSTANTIATE(f)                                                                  \
  template mlt::StereoKernel mlt::stereo_pick<((f) >> 3) & 1, ((f) >> 2) & 1, ((f) >> 1) & 1, (f) & 1>( \
      int, int, int);
