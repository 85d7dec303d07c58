// Pipe-rate microbenchmark for the sweep kernel's roofline denominators.
// Measures, on the current device, the sustained per-GPU rate of:
//   FFMA (fp32 scalar), FFMA2 (fp32x2 packed), MUFU.RCP, MUFU.EX2, DFMA (fp64).
// Each kernel runs a long dependent-free unrolled loop on a persistent grid
// (148 SMs x 8 CTAs x 256 threads) and is timed with CUDA events (best of 5).
// Output: one JSON line on stdout.
#include <cstdio>
#include <cuda_runtime.h>

#define NCHAIN 8
#define ITERS 4096

__global__ void k_ffma(float* out, float s) {
  float a[NCHAIN];
  for (int c = 0; c < NCHAIN; ++c) a[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) a[c] = fmaf(a[c], s, 0.5f);
  }
  float r = 0; for (int c = 0; c < NCHAIN; ++c) r += a[c];
  if (r == 1234.5f) out[0] = r;
}

__global__ void k_ffma2(float* out, float s) {
  unsigned long long a[NCHAIN], sv, hv;
  asm("mov.b64 %0, {%1,%1};" : "=l"(sv) : "f"(s));
  asm("mov.b64 %0, {%1,%1};" : "=l"(hv) : "f"(0.5f));
  for (int c = 0; c < NCHAIN; ++c) { float x = threadIdx.x * 1e-3f + c; asm("mov.b64 %0, {%1,%1};" : "=l"(a[c]) : "f"(x)); }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[c]) : "l"(sv), "l"(hv));
  }
  float r = 0; for (int c = 0; c < NCHAIN; ++c) { float x, y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[c])); r += x + y; }
  if (r == 1234.5f) out[0] = r;
}

__global__ void k_rcp(float* out, float s) {
  float a[NCHAIN];
  for (int c = 0; c < NCHAIN; ++c) a[c] = 1.0f + threadIdx.x * 1e-3f + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) {
      asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a[c]));
      asm volatile("add.f32 %0, %0, 0f3F800000;" : "+f"(a[c]));   // defeats rcp(rcp(x)) folding
    }
  }
  float r = 0; for (int c = 0; c < NCHAIN; ++c) r += a[c];
  if (r == 1234.5f) out[0] = r;
}

__global__ void k_ex2(float* out, float s) {
  float a[NCHAIN];
  for (int c = 0; c < NCHAIN; ++c) a[c] = -1.0f - threadIdx.x * 1e-4f - c * 1e-2f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[c]));
  }
  float r = 0; for (int c = 0; c < NCHAIN; ++c) r += a[c];
  if (r == 1234.5f) out[0] = r;
}

__global__ void k_dfma(float* out, float s) {
  double a[NCHAIN]; double sd = s;
  for (int c = 0; c < NCHAIN; ++c) a[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) a[c] = fma(a[c], sd, 0.5);
  }
  double r = 0; for (int c = 0; c < NCHAIN; ++c) r += a[c];
  if (r == 1234.5) out[0] = (float)r;
}

typedef void (*kfn)(float*, float);

static double time_kernel(kfn f, int blocks, int threads, float* out) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f<<<blocks, threads>>>(out, 0.999f);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a); f<<<blocks, threads>>>(out, 0.999f); cudaEventRecord(b);
    cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best * 1e-3;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount; int blocks = sms * 8, threads = 256;
  float* out; cudaMalloc(&out, 4);
  double ops = (double)blocks * threads * ITERS * NCHAIN;   // lane-ops per kernel
  double t_ffma = time_kernel(k_ffma, blocks, threads, out);
  double t_ffma2 = time_kernel(k_ffma2, blocks, threads, out);
  double t_rcp = time_kernel(k_rcp, blocks, threads, out);
  double t_ex2 = time_kernel(k_ex2, blocks, threads, out);
  double t_dfma = time_kernel(k_dfma, blocks, threads, out);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f, "
         "\"fp32_ffma_tflops\": %.2f, \"fp32_ffma2_tflops\": %.2f, "
         "\"mufu_rcp_gops\": %.1f, \"mufu_ex2_gops\": %.1f, \"fp64_dfma_tflops\": %.2f}\n",
         p.name, sms, clk_khz / 1e3,
         2 * ops / t_ffma / 1e12, 4 * ops / t_ffma2 / 1e12,
         ops / t_rcp / 1e9, ops / t_ex2 / 1e9, 2 * ops / t_dfma / 1e12);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "cuda error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
