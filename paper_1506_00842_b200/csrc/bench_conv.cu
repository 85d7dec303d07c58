// bench_conv.cu — the paper's tunable 2D convolution benchmark (SURVEY §8(a)
// A13, §8(f) next #1; Tables 1-2: 5x5 box filter over a 2D image),
// written for sm_100a behind the runner protocol (measurement.py:250-258):
//
//   knob             realisation on the B200
//   wg_x, wg_y       CTA shape (wg_x*wg_y > 1024 -> invalid-launch)
//   ppt_x, ppt_y     output pixels per thread in x / y
//   use_image        input read through a texture object (point sampling, clamp addressing)
//   use_local        the CTA's input tile + 2-pixel halo staged in shared memory
//                    (tile > 227 KB -> invalid-launch); with padding and no image
//                    memory the tile arrives by TMA (cp.async.bulk.tensor + mbarrier)
//   padding          input pre-padded by 2 replicated pixels: no clamping in the kernel
//   interleaved      a thread's pixels are strided by the CTA width (coalesced) instead of contiguous
//   unroll           the 5x5 filter loops fully unrolled; with contiguous pixels (interleaved = 0)
//                    each thread also streams 8 input rows once for 4 vertically adjacent outputs
//
// Every variant sums the 25 taps in the same (dy, dx) order in fp32 and
// divides by 25 (correctly rounded), so all 32 variants produce bit-identical
// images, equal to the numpy float32 golden of tests/ (clamp-to-edge borders).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "bench_common.cuh"
#include "mltune_b200.h"

namespace mlt {

struct ConvArgs {
  int W, H;
  const float* in;        // W x H, or (W+4) x (H+4) when padded
  int pitch;              // row pitch (elements) of `in`
  cudaTextureObject_t tex;
  float* out;             // W x H
  int pptx, ppty;
};

template <bool IMG, bool PAD>
__device__ __forceinline__ float fetch(const ConvArgs& a, int y, int x) {
  // y, x may lie up to 2 pixels outside the image
  if (PAD) {
    if (IMG) return tex2D<float>(a.tex, (float)(x + 2) + 0.5f, (float)(y + 2) + 0.5f);
    return __ldg(a.in + (size_t)(y + 2) * a.pitch + (x + 2));
  }
  if (IMG) return tex2D<float>(a.tex, (float)x + 0.5f, (float)y + 0.5f);   // clamp addressing
  const int yy = min(max(y, 0), a.H - 1), xx = min(max(x, 0), a.W - 1);
  return __ldg(a.in + (size_t)yy * a.pitch + xx);
}

// s / 25 correctly rounded with two FMAs: exhaustively equal to the IEEE
// division for every finite float except -0 (tools/check_div25.cu), and a tap
// sum that starts from +0 is never -0.
__device__ __forceinline__ float div25(float s) {
  const float inv = 1.0f / 25.0f;
  const float q0 = __fmul_rn(s, inv);
  return __fmaf_rn(__fmaf_rn(-q0, 25.0f, s), inv, q0);
}

template <bool IMG, bool LOCAL, bool PAD, bool INTER, bool UNROLL>
__device__ __forceinline__ void conv_compute(const ConvArgs& a, const float* tile, int tw, int X0, int Y0, int bw,
                                             int bh, int tx, int ty, int wgx, int wgy) {
  int iy0 = 0;
  if (UNROLL && !INTER && LOCAL && (a.pptx & 3) == 0 && (tw & 3) == 0) {
    // 4 x 4 register block per step: 8 input rows x 8 columns (two aligned
    // 16-byte shared loads per row) feed 16 outputs, each still summing its
    // 25 taps in (dy, dx) order.
    for (; iy0 + 4 <= a.ppty; iy0 += 4) {
      const int ly = ty * a.ppty + iy0;
      const int y = Y0 + ly;
      if (y + 3 >= a.H) break;
      for (int ix = 0; ix < a.pptx; ix += 4) {
        const int lx = tx * a.pptx + ix;
        const int x = X0 + lx;
        if (x + 3 >= a.W) {     // right edge: the per-column path below finishes these
          if (x < a.W) {
            for (int c = 0; c < 4 && x + c < a.W; ++c)
              for (int k = 0; k < 4; ++k) {
                float sum = 0.0f;
#pragma unroll
                for (int dy = 0; dy < 5; ++dy)
#pragma unroll
                  for (int dx = 0; dx < 5; ++dx) sum += tile[(ly + k + dy) * tw + (lx + c + dx)];
                a.out[(size_t)(y + k) * a.W + x + c] = div25(sum);
              }
          }
          break;
        }
        float acc[4][4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[k][c] = 0.0f;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float4 u0 = *reinterpret_cast<const float4*>(tile + (ly + r) * tw + lx);
          const float4 u1 = *reinterpret_cast<const float4*>(tile + (ly + r) * tw + lx + 4);
          const float t[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (r - k >= 0 && r - k <= 4) {
#pragma unroll
              for (int dx = 0; dx < 5; ++dx)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[k][c] += t[c + dx];
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float* o = a.out + (size_t)(y + k) * a.W + x;
          if ((a.W & 3) == 0) {
            *reinterpret_cast<float4*>(o) = make_float4(div25(acc[k][0]), div25(acc[k][1]), div25(acc[k][2]),
                                                         div25(acc[k][3]));
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) o[c] = div25(acc[k][c]);
          }
        }
      }
    }
  } else if (UNROLL && !INTER) {
    // Unrolled + contiguous rows: 4 vertically adjacent outputs of a column
    // stream the 8 input rows they cover once (8 x 5 loads for 4 outputs
    // instead of 4 x 25); each output still adds its 25 taps in (dy, dx)
    // order. Adjacent lanes read adjacent columns (conflict-free when ppt_x = 1).
    for (; iy0 + 4 <= a.ppty; iy0 += 4) {
      const int ly = ty * a.ppty + iy0;
      const int y = Y0 + ly;
      if (y + 3 >= a.H) break;
      for (int ix = 0; ix < a.pptx; ++ix) {
        const int lx = tx * a.pptx + ix;
        const int x = X0 + lx;
        if (x >= a.W) break;
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          float t[5];
#pragma unroll
          for (int dx = 0; dx < 5; ++dx)
            t[dx] = LOCAL ? tile[(ly + r) * tw + (lx + dx)] : fetch<IMG, PAD>(a, y - 2 + r, x - 2 + dx);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (r - k >= 0 && r - k <= 4) {
#pragma unroll
              for (int dx = 0; dx < 5; ++dx) acc[k] += t[dx];
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) a.out[(size_t)(y + k) * a.W + x] = div25(acc[k]);
      }
    }
  }
  for (int iy = iy0; iy < a.ppty; ++iy) {
    const int ly = INTER ? iy * wgy + ty : ty * a.ppty + iy;   // row within the CTA's output block
    const int y = Y0 + ly;
    if (y >= a.H) continue;
    for (int ix = 0; ix < a.pptx; ++ix) {
      const int lx = INTER ? ix * wgx + tx : tx * a.pptx + ix;
      const int x = X0 + lx;
      if (x >= a.W) continue;
      float s = 0.0f;
      if (UNROLL) {
#pragma unroll
        for (int dy = -2; dy <= 2; ++dy)
#pragma unroll
          for (int dx = -2; dx <= 2; ++dx)
            s += LOCAL ? tile[(ly + 2 + dy) * tw + (lx + 2 + dx)] : fetch<IMG, PAD>(a, y + dy, x + dx);
      } else {
#pragma unroll 1
        for (int dy = -2; dy <= 2; ++dy)
#pragma unroll 1
          for (int dx = -2; dx <= 2; ++dx)
            s += LOCAL ? tile[(ly + 2 + dy) * tw + (lx + 2 + dx)] : fetch<IMG, PAD>(a, y + dy, x + dx);
      }
      a.out[(size_t)y * a.W + x] = div25(s);
    }
  }
}


template <bool IMG, bool LOCAL, bool PAD, bool INTER, bool UNROLL>
__global__ void k_conv5(ConvArgs a) {
  extern __shared__ float tile[];
  const int wgx = blockDim.x, wgy = blockDim.y;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int bw = wgx * a.pptx, bh = wgy * a.ppty;           // output pixels per CTA
  const int X0 = blockIdx.x * bw, Y0 = blockIdx.y * bh;
  const int tw = bw + 4;
  if (LOCAL) {
    const int th = bh + 4;
    // flat, evenly split over the CTA; (r, c) advanced incrementally (no division).
    // Rows/cols past the image's 2-pixel halo feed no valid output: clamp them in range.
    const int nt = wgx * wgy, step_r = nt / tw, step_c = nt - step_r * tw;
    int q = ty * wgx + tx;
    int r = q / tw, c = q - r * tw;
    for (; q < tw * th; q += nt) {
      tile[q] = fetch<IMG, PAD>(a, min(Y0 - 2 + r, a.H + 1), min(X0 - 2 + c, a.W + 1));
      r += step_r;
      c += step_c;
      if (c >= tw) {
        c -= tw;
        ++r;
      }
    }
    __syncthreads();
  }
  conv_compute<IMG, LOCAL, PAD, INTER, UNROLL>(a, tile, tw, X0, Y0, bw, bh, tx, ty, wgx, wgy);
}

// use_local + padding (no image memory), on a row pitch that is a multiple of
// 16 bytes: the CTA's tile + halo arrives by TMA (cp.async.bulk.tensor.2d,
// one elected thread, mbarrier completion) from the pre-padded image instead
// of per-thread loads; boxes of up to 256 rows stack into the row-major tile.
// The compute part is k_conv5's, so the output is bit-identical.
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(map), "r"(x), "r"(y), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

template <bool INTER, bool UNROLL>
__global__ void k_conv5_tma(ConvArgs a, const __grid_constant__ CUtensorMap map, int box_rows) {
  extern __shared__ __align__(128) float tile[];
  __shared__ __align__(8) uint64_t bar;
  const int wgx = blockDim.x, wgy = blockDim.y;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int bw = wgx * a.pptx, bh = wgy * a.ppty;
  const int X0 = blockIdx.x * bw, Y0 = blockIdx.y * bh;
  const int tw = bw + 4, th = bh + 4;
  const int nbox = (th + box_rows - 1) / box_rows;
  if (tx == 0 && ty == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&bar, (unsigned)(nbox * box_rows * tw * 4));
    // padded coordinates: tile column 0 = padded column X0 (= image column X0 - 2)
    for (int bx = 0; bx < nbox; ++bx) tma_load_2d(tile + (size_t)bx * box_rows * tw, &map, X0, Y0 + bx * box_rows, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  conv_compute<false, true, true, INTER, UNROLL>(a, tile, tw, X0, Y0, bw, bh, tx, ty, wgx, wgy);
}

typedef void (*ConvKernel)(ConvArgs);

#define MLT_CONV_ENTRY(i)                                                                              \
  k_conv5<((i) >> 4) & 1, ((i) >> 3) & 1, ((i) >> 2) & 1, ((i) >> 1) & 1, (i) & 1>
static const ConvKernel kConvKernels[32] = {
    MLT_CONV_ENTRY(0),  MLT_CONV_ENTRY(1),  MLT_CONV_ENTRY(2),  MLT_CONV_ENTRY(3),  MLT_CONV_ENTRY(4),
    MLT_CONV_ENTRY(5),  MLT_CONV_ENTRY(6),  MLT_CONV_ENTRY(7),  MLT_CONV_ENTRY(8),  MLT_CONV_ENTRY(9),
    MLT_CONV_ENTRY(10), MLT_CONV_ENTRY(11), MLT_CONV_ENTRY(12), MLT_CONV_ENTRY(13), MLT_CONV_ENTRY(14),
    MLT_CONV_ENTRY(15), MLT_CONV_ENTRY(16), MLT_CONV_ENTRY(17), MLT_CONV_ENTRY(18), MLT_CONV_ENTRY(19),
    MLT_CONV_ENTRY(20), MLT_CONV_ENTRY(21), MLT_CONV_ENTRY(22), MLT_CONV_ENTRY(23), MLT_CONV_ENTRY(24),
    MLT_CONV_ENTRY(25), MLT_CONV_ENTRY(26), MLT_CONV_ENTRY(27), MLT_CONV_ENTRY(28), MLT_CONV_ENTRY(29),
    MLT_CONV_ENTRY(30), MLT_CONV_ENTRY(31)};

// deterministic synthetic image: uniform [0, 1) from a splitmix64 hash of (seed, pixel)
__global__ void k_fill_image(float* img, int W, int H, uint64_t seed) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)W * H;
       q += (int64_t)gridDim.x * blockDim.x)
    img[q] = (float)((double)(bench::hash_at(seed, (uint64_t)q) >> 40) * (1.0 / 16777216.0));
}

// padded copy with 2 replicated border pixels
__global__ void k_pad_image(const float* img, float* pad, int W, int H) {
  const int pw = W + 4;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (int64_t)pw * (H + 4);
       q += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(q / pw), c = (int)(q % pw);
    const int y = min(max(r - 2, 0), H - 1), x = min(max(c - 2, 0), W - 1);
    pad[q] = img[(size_t)y * W + x];
  }
}

}  // namespace mlt

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
struct mlt_convbench {
  int dev = 0;
  cudaStream_t stream = nullptr;
  int W = 0, H = 0;
  float* img = nullptr;
  float* pad = nullptr;
  float* out = nullptr;
  cudaArray_t arr = nullptr, arr_pad = nullptr;
  cudaTextureObject_t tex = 0, tex_pad = 0;
  mlt::bench::Timer timer;
};

namespace {
thread_local mlt::bench::ErrSlot g_cerr;
#define CK(expr) MLT_BENCH_CK(g_cerr, expr)
}  // namespace

extern "C" {

MLT_API const char* mlt_convbench_last_error(void) { return g_cerr.msg.c_str(); }

MLT_API int mlt_convbench_create(int device, int32_t width, int32_t height, const float* image, uint64_t seed,
                                 mlt_convbench** out) {
  using namespace mlt;
  if (!out) return g_cerr.fail(MLT_EINVAL, "out is NULL");
  *out = nullptr;
  if (width < 1 || height < 1 || width > 32768 || height > 32768) return g_cerr.fail(MLT_EINVAL, "bad image size");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return g_cerr.fail(MLT_ECUDA, "no CUDA device (no CPU fallback)");
  CK(cudaSetDevice(device));
  mlt_convbench* b = new mlt_convbench();
  b->dev = device;
  b->W = width;
  b->H = height;
  CK(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking));
  const size_t px = (size_t)width * height;
  CK(cudaMalloc(&b->img, px * 4));
  CK(cudaMalloc(&b->out, px * 4));
  CK(cudaMalloc(&b->pad, (size_t)(width + 4) * (height + 4) * 4));
  if (image) {
    CK(cudaMemcpyAsync(b->img, image, px * 4, cudaMemcpyHostToDevice, b->stream));
  } else {
    k_fill_image<<<1024, 256, 0, b->stream>>>(b->img, width, height, seed);
  }
  k_pad_image<<<1024, 256, 0, b->stream>>>(b->img, b->pad, width, height);
  CK(cudaGetLastError());
  int rc = bench::make_texture_2d(g_cerr, b->img, width, height, &b->arr, &b->tex, b->stream);
  if (rc == MLT_OK) rc = bench::make_texture_2d(g_cerr, b->pad, width + 4, height + 4, &b->arr_pad, &b->tex_pad, b->stream);
  if (rc == MLT_OK) rc = b->timer.init(g_cerr, b->stream);
  if (rc != MLT_OK) return rc;
  CK(cudaStreamSynchronize(b->stream));
  *out = b;
  return MLT_OK;
}

MLT_API int mlt_convbench_destroy(mlt_convbench* b) {
  if (!b) return MLT_OK;
  cudaSetDevice(b->dev);
  cudaStreamSynchronize(b->stream);
  cudaDestroyTextureObject(b->tex);
  cudaDestroyTextureObject(b->tex_pad);
  cudaFreeArray(b->arr);
  cudaFreeArray(b->arr_pad);
  cudaFree(b->img);
  cudaFree(b->pad);
  cudaFree(b->out);
  b->timer.release();
  cudaStreamDestroy(b->stream);
  delete b;
  return MLT_OK;
}

// knobs = {wg_x, wg_y, ppt_x, ppt_y, use_image, use_local, padding, interleaved, unroll}
// (the convolution space's parameter order, paramspace.py:287-310). status: 0 = valid,
// 1 = invalid-launch. seconds = min over `reps` runs, each after an L2 flush.
MLT_API int mlt_convbench_run(mlt_convbench* b, const int32_t* knobs, int32_t reps, double* seconds, int32_t* status) {
  using namespace mlt;
  if (!b || !knobs || !seconds || !status) return g_cerr.fail(MLT_EINVAL, "NULL argument");
  if (reps < 1) return g_cerr.fail(MLT_EINVAL, "repetitions must be >= 1");
  CK(cudaSetDevice(b->dev));
  const int wgx = knobs[0], wgy = knobs[1], pptx = knobs[2], ppty = knobs[3];
  const bool img = knobs[4], local = knobs[5], pad = knobs[6], inter = knobs[7], unroll = knobs[8];
  *status = 0;
  *seconds = 0;
  if (wgx < 1 || wgy < 1 || pptx < 1 || ppty < 1) return g_cerr.fail(MLT_EINVAL, "non-positive knob");
  const int64_t bw = (int64_t)wgx * pptx, bh = (int64_t)wgy * ppty;
  const int64_t gx = (b->W + bw - 1) / bw, gy = (b->H + bh - 1) / bh;
  const size_t smem = local ? (size_t)(bw + 4) * (size_t)(bh + 4) * 4 : 0;
  if ((int64_t)wgx * wgy > 1024 || wgy > 1024 || smem > bench::kMaxSmem || gy > 65535) {
    *status = 1;                                     // cannot launch on this device
    return MLT_OK;
  }
  // use_local + padding without image memory: TMA-staged tile when the
  // tensor-map constraints hold (16-byte row pitch and box width, box <= 256 wide)
  const int tw = (int)bw + 4, th = (int)bh + 4;
  if (!img && local && pad && (b->W % 4) == 0 && (tw % 4) == 0 && tw <= 256) {
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }
    const int box_rows = th < 256 ? th : 256;
    const int nbox = (th + box_rows - 1) / box_rows;
    const size_t tsmem = (size_t)nbox * box_rows * tw * 4;
    if (encode && tsmem <= bench::kMaxSmem && (int64_t)wgx * wgy <= 1024 && gy <= 65535) {
      CUtensorMap map;
      const cuuint64_t gdim[2] = {(cuuint64_t)b->W + 4, (cuuint64_t)b->H + 4};
      const cuuint64_t gstride[1] = {(cuuint64_t)(b->W + 4) * 4};
      const cuuint32_t box[2] = {(cuuint32_t)tw, (cuuint32_t)box_rows};
      const cuuint32_t estride[2] = {1, 1};
      if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, b->pad, gdim, gstride, box, estride,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
        void (*tk)(ConvArgs, const CUtensorMap, int) =
            inter ? (unroll ? k_conv5_tma<true, true> : k_conv5_tma<true, false>)
                  : (unroll ? k_conv5_tma<false, true> : k_conv5_tma<false, false>);
        if (tsmem > 48 * 1024) CK(cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem));
        ConvArgs ta;
        ta.W = b->W;
        ta.H = b->H;
        ta.in = b->pad;
        ta.pitch = b->W + 4;
        ta.tex = b->tex_pad;
        ta.out = b->out;
        ta.pptx = pptx;
        ta.ppty = ppty;
        return b->timer.run(g_cerr, reps, [&]() {
          tk<<<dim3((unsigned)gx, (unsigned)gy), dim3(wgx, wgy), tsmem, b->stream>>>(ta, map, box_rows);
          return cudaGetLastError();
        }, seconds, status);
      }
    }
  }
  const int sel = (img << 4) | (local << 3) | (pad << 2) | (inter << 1) | (int)unroll;
  ConvKernel k = kConvKernels[sel];
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ConvArgs a;
  a.W = b->W;
  a.H = b->H;
  a.in = pad ? b->pad : b->img;
  a.pitch = pad ? b->W + 4 : b->W;
  a.tex = pad ? b->tex_pad : b->tex;
  a.out = b->out;
  a.pptx = pptx;
  a.ppty = ppty;
  return b->timer.run(g_cerr, reps, [&]() {
    k<<<dim3((unsigned)gx, (unsigned)gy), dim3(wgx, wgy), smem, b->stream>>>(a);
    return cudaGetLastError();
  }, seconds, status);
}

MLT_API int mlt_convbench_output(mlt_convbench* b, float* host_out) {
  if (!b || !host_out) return g_cerr.fail(MLT_EINVAL, "NULL argument");
  CK(cudaSetDevice(b->dev));
  CK(cudaMemcpyAsync(host_out, b->out, (size_t)b->W * b->H * 4, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return MLT_OK;
}

MLT_API int mlt_convbench_input(mlt_convbench* b, float* host_in) {
  if (!b || !host_in) return g_cerr.fail(MLT_EINVAL, "NULL argument");
  CK(cudaSetDevice(b->dev));
  CK(cudaMemcpyAsync(host_in, b->img, (size_t)b->W * b->H * 4, cudaMemcpyDeviceToHost, b->stream));
  CK(cudaStreamSynchronize(b->stream));
  return MLT_OK;
}

}  // extern "C"
