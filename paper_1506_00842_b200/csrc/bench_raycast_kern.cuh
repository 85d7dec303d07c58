// bench_raycast_kern.cuh — the raycasting kernel template (see bench_raycast.cu
// for the algorithm and the knob mapping). Included only by bench_raycast_u*.cu.
#pragma once

#include "bench_common.cuh"
#include "bench_raycast.cuh"

namespace mlt {

template <bool IMG>
__device__ __forceinline__ unsigned ray_voxel(const RayArgs& a, int ix, int iy, int iz) {
  if (IMG) return tex3D<unsigned char>(a.tex_vol, (float)ix + 0.5f, (float)iy + 0.5f, (float)iz + 0.5f);
  return __ldg(a.vol + ((size_t)iz * a.VY + iy) * a.VX + ix);
}

// transfer-function source: texture if img_transfer, else the constant bank if
// const_transfer, else global memory (local_transfer stages from that source)
template <bool ITF, bool CTF>
__device__ __forceinline__ float4 ray_tf(const RayArgs& a, const RayConstTF& ctf, unsigned s) {
  if (ITF) return tex1Dfetch<float4>(a.tex_tf, (int)s);
  if (CTF) return ctf.e[s];
  return __ldg(a.tf + s);
}

__device__ __forceinline__ int ray_cell(float p, int n) { return min(max((int)floorf(p), 0), n - 1); }

template <bool IMGD, bool ITF, bool LTF, bool CTF, bool INTER, int U>
__global__ void k_raycast(RayArgs a, const __grid_constant__ RayConstTF ctf) {
  __shared__ float4 stf[256];
  const int wgx = blockDim.x, wgy = blockDim.y;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (LTF) {
    for (int q = ty * wgx + tx; q < 256; q += wgx * wgy) stf[q] = ray_tf<ITF, CTF>(a, ctf, (unsigned)q);
    __syncthreads();
  }
  const RayCamera& cam = a.cam;
  const int bw = wgx * a.pptx, bh = wgy * a.ppty;
  const int X0 = blockIdx.x * bw, Y0 = blockIdx.y * bh;
  const float V[3] = {(float)a.VX, (float)a.VY, (float)a.VZ};
  const unsigned long long start = a.budget_ns ? *a.t0 : 0ull;
  for (int iy = 0; iy < a.ppty; ++iy) {
    const int py = Y0 + (INTER ? iy * wgy + ty : ty * a.ppty + iy);
    if (py >= a.IH) continue;
    for (int ix = 0; ix < a.pptx; ++ix) {
      const int px = X0 + (INTER ? ix * wgx + tx : tx * a.pptx + ix);
      if (px >= a.IW) continue;
      if (a.budget_ns && bench::gtimer() - start > a.budget_ns) return;   // screening: over budget
      const float sa = __fmul_rn(__fsub_rn(__fadd_rn((float)px, 0.5f), cam.hw), cam.scale);
      const float sb = __fmul_rn(__fsub_rn(__fadd_rn((float)py, 0.5f), cam.hh), cam.scale);
      float o[3], tn = -INFINITY, tf = INFINITY;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        o[i] = __fadd_rn(__fadd_rn(cam.c[i], __fmul_rn(cam.u[i], sa)), __fmul_rn(cam.v[i], sb));
        const float t0 = __fmul_rn(__fsub_rn(0.0f, o[i]), cam.inv[i]);
        const float t1 = __fmul_rn(__fsub_rn(V[i], o[i]), cam.inv[i]);
        tn = fmaxf(tn, fminf(t0, t1));
        tf = fminf(tf, fmaxf(t0, t1));
      }
      float r = 0.f, g = 0.f, bl = 0.f, al = 0.f;
      if (tf > tn) {
        const int n = (int)ceilf(__fsub_rn(tf, tn));
        bool live = true;
        for (int k = 0; live && k < n; k += U) {
          unsigned s[U];
#pragma unroll
          for (int j = 0; j < U; ++j) {            // U independent gathers in flight
            const float t = __fadd_rn(tn, __fadd_rn((float)(k + j), 0.5f));
            s[j] = ray_voxel<IMGD>(a, ray_cell(__fadd_rn(o[0], __fmul_rn(t, cam.w[0])), a.VX),
                                   ray_cell(__fadd_rn(o[1], __fmul_rn(t, cam.w[1])), a.VY),
                                   ray_cell(__fadd_rn(o[2], __fmul_rn(t, cam.w[2])), a.VZ));
          }
#pragma unroll
          for (int j = 0; j < U; ++j) {            // front-to-back compositing, in step order
            if (live && k + j < n) {
              const float4 c = LTF ? stf[s[j]] : ray_tf<ITF, CTF>(a, ctf, s[j]);
              const float f = __fmul_rn(__fsub_rn(1.0f, al), c.w);
              r = __fadd_rn(r, __fmul_rn(f, c.x));
              g = __fadd_rn(g, __fmul_rn(f, c.y));
              bl = __fadd_rn(bl, __fmul_rn(f, c.z));
              al = __fadd_rn(al, f);
              if (al >= cam.thr) live = false;
            }
          }
        }
      }
      a.out[(size_t)py * a.IW + px] = make_float4(r, g, bl, al);
    }
  }
}

template <int U>
RayKernel ray_pick(int flags) {
  switch (flags & 31) {
#define MLT_RAY_CASE(f) \
  case f: return k_raycast<((f) >> 4) & 1, ((f) >> 3) & 1, ((f) >> 2) & 1, ((f) >> 1) & 1, (f) & 1, U>;
    MLT_RAY_CASE(0) MLT_RAY_CASE(1) MLT_RAY_CASE(2) MLT_RAY_CASE(3) MLT_RAY_CASE(4) MLT_RAY_CASE(5)
    MLT_RAY_CASE(6) MLT_RAY_CASE(7) MLT_RAY_CASE(8) MLT_RAY_CASE(9) MLT_RAY_CASE(10) MLT_RAY_CASE(11)
    MLT_RAY_CASE(12) MLT_RAY_CASE(13) MLT_RAY_CASE(14) MLT_RAY_CASE(15) MLT_RAY_CASE(16) MLT_RAY_CASE(17)
    MLT_RAY_CASE(18) MLT_RAY_CASE(19) MLT_RAY_CASE(20) MLT_RAY_CASE(21) MLT_RAY_CASE(22) MLT_RAY_CASE(23)
    MLT_RAY_CASE(24) MLT_RAY_CASE(25) MLT_RAY_CASE(26) MLT_RAY_CASE(27) MLT_RAY_CASE(28) MLT_RAY_CASE(29)
    MLT_RAY_CASE(30) MLT_RAY_CASE(31)
#undef MLT_RAY_CASE
  }
  return nullptr;
}

}  // namespace mlt

#define MLT_RAY_INSTANTIATE(u) template mlt::RayKernel mlt::ray_pick<u>(int);
