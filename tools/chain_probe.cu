// Probe: the sweep's group arithmetic in isolation (LDS-fed exp(-A'), per-thread
// factors held in registers, no global loads) at the sweep's occupancy, to
// separate the dependency structure from memory latency.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) { f2 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void upk(f2 v, float& lo, float& hi) { asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) { f2 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ f2 fmul2(f2 a, f2 b) { f2 d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) { f2 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float rcpa(float x) { float r; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
constexpr int kOB = 16, kInner = 2, G = 3;
template <int LDG>
__global__ void __launch_bounds__(256, 2) k_probe(float* out, const float* __restrict__ gsrc, int ngroups, int stride) {
  __shared__ float4 s_ea[480 * kOB / 4];
  for (int q = threadIdx.x; q < 480 * kOB / 4; q += 256) s_ea[q] = make_float4(1e-3f * q, 2e-3f, 3e-3f, 4e-3f * q);
  __syncthreads();
  f2 acc[kInner][kOB / 2];
  for (int s = 0; s < kInner; ++s) for (int q = 0; q < kOB / 2; ++q) acc[s][q] = 0ull;
  float eb[kInner][G], uu[G];
  for (int x = 0; x < G; ++x) { uu[x] = 1.0f + x; for (int s = 0; s < kInner; ++s) eb[s][x] = 0.5f + threadIdx.x * 1e-4f + s + x; }
  const float* pe = gsrc + threadIdx.x;
  for (int rep = 0; rep < 8; ++rep) {
#pragma unroll 1
    for (int gi = 0; gi < ngroups; ++gi) {
      if (LDG) {
#pragma unroll
        for (int x = 0; x < G; ++x)
#pragma unroll
          for (int s = 0; s < kInner; ++s) eb[s][x] = __ldg(pe + (size_t)(gi * G + x) * stride + s * 256);
      }
      const float* E = reinterpret_cast<const float*>(s_ea) + (gi % 160) * G * kOB;
#pragma unroll
      for (int q = 0; q < kOB / 4; ++q) {
        float4 ea[G];
#pragma unroll
        for (int x = 0; x < G; ++x) ea[x] = *reinterpret_cast<const float4*>(E + x * kOB + 4 * q);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
          for (int s = 0; s < kInner; ++s) {
            f2 d[G];
#pragma unroll
            for (int x = 0; x < G; ++x) d[x] = ffma2(half ? pk(ea[x].z, ea[x].w) : pk(ea[x].x, ea[x].y), pk(eb[s][x], eb[s][x]), pk(uu[x], uu[x]));
            const f2 sm = fadd2(d[0], d[1]), pr = fmul2(d[0], d[1]);
            const f2 num = ffma2(d[2], sm, pr), den = fmul2(pr, d[2]);
            float dl, dh; upk(den, dl, dh);
            acc[s][2 * q + half] = ffma2(num, pk(rcpa(dl), rcpa(dh)), acc[s][2 * q + half]);
          }
        }
      }
    }
  }
  float t = 0; for (int s = 0; s < kInner; ++s) for (int q = 0; q < kOB / 2; ++q) { float a, b; upk(acc[s][q], a, b); t += a + b; }
  if (t == 1234.5f) out[0] = t;
}
template <int LDG>
void run(float* out, float* g, int ngroups) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 2;
  k_probe<LDG><<<blocks, 256>>>(out, g, ngroups, 12288); cudaDeviceSynchronize();
  cudaEventRecord(e0); k_probe<LDG><<<blocks, 256>>>(out, g, ngroups, 12288); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double pairs = (double)blocks * 256 * 8 * ngroups * kInner * (kOB / 2);    // pair-chains
  double lanefma = pairs * 2 * 8;     // 8 packed FP per pair chain, 2 lanes each
  double mufu = pairs * 2;
  printf("{\"ldg\": %d, \"ms\": %.3f, \"fma_frac\": %.3f, \"mufu_frac\": %.3f}\n", LDG, ms,
         lanefma / (ms * 1e-3) / (148.0 * 128 * 1.965e9), mufu / (ms * 1e-3) / (148.0 * 16 * 1.965e9));
}
int main() {
  float *out, *g; cudaMalloc(&out, 4); cudaMalloc(&g, 480 * 12288 * 4); cudaMemset(g, 0, 480 * 12288 * 4);
  run<0>(out, g, 160); run<1>(out, g, 160);
  return 0;
}
