// Depthwise 3x3 convolution kernels (stride 1 / 2, pad 1, NHWC bf16) of the MobileNetV2 and ShuffleNetV2
// client engines: forward, data gradient, weight gradient (two-pass, deterministic) + SGD, and the small
// step-counter kernels of their per-step CUDA graphs.
#pragma once
#include "cifar_common.cuh"

namespace fedhc {
namespace mb {

using rn::bf;

// ---- depthwise 3x3 convolution (pad 1, stride S), NHWC bf16 ----
// Thread = (8-channel group cg, lane); a lane owns runs ("segments") of 4 consecutive output pixels of one row,
// so a row of the 3 x (3S + 3) input window is loaded once (16-byte vectors) and reused by the 4 outputs
// (sliding window along x: 4.5 / 6.75 loads per output instead of 9).  The 9 x 8 taps stay packed bf16 in
// registers and every product is one mixed-precision FHFMA (bf16 x bf16 + fp32 -> fp32: the exact product of
// the two bf16 values, so results equal fp32 math on the converted operands) -- no unpacking instructions.
// lanes = DW_THREADS / (C / 8) (C <= 1024).
constexpr int DW_SEG_PER_LANE = 2, DW_THREADS = 128;

__device__ __forceinline__ float fma_bf16(unsigned short a, unsigned short b, float c) {
  float d;
  asm("fma.rn.f32.bf16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}

// acc[e] += x[e] * w[e] for the 8 packed bf16 lanes of two uint4
__device__ __forceinline__ void fma8(const uint4& x, const uint4& w, float (&acc)[8]) {
  const unsigned xs[4] = {x.x, x.y, x.z, x.w}, ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    unsigned short xl, xh, wl, wh;
    asm("mov.b32 {%0, %1}, %2;" : "=h"(xl), "=h"(xh) : "r"(xs[q]));
    asm("mov.b32 {%0, %1}, %2;" : "=h"(wl), "=h"(wh) : "r"(ws[q]));
    acc[2 * q] = fma_bf16(xl, wl, acc[2 * q]);
    acc[2 * q + 1] = fma_bf16(xh, wh, acc[2 * q + 1]);
  }
}

__device__ __forceinline__ uint4 pack8(const float (&a)[8]) {
  __align__(16) __nv_bfloat16 v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = __float2bfloat16_rn(a[e]);
  return *reinterpret_cast<const uint4*>(v);
}

template <int S>
static __global__ void __launch_bounds__(DW_THREADS) dw_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                     const __nv_bfloat16* __restrict__ shadow, int64_t pstride,
                                                     int64_t woff, int Bp, int H, int C,
                                                     __nv_bfloat16* __restrict__ y) {
  constexpr int NC = 3 * S + 3;  // input columns of a 4-output segment
  const int c8 = C >> 3, lanes = DW_THREADS / c8, cg = threadIdx.x % c8, lane = threadIdx.x / c8;
  if (lane >= lanes) return;
  const int img = blockIdx.y, g = img / Bp, Ho = H / S, sw = Ho >> 2, nseg = Ho * sw;
  uint4 wt[9];
  const __nv_bfloat16* w = shadow + (int64_t)g * pstride + woff + cg * 8;
#pragma unroll
  for (int t = 0; t < 9; ++t) wt[t] = *reinterpret_cast<const uint4*>(w + t * C);
  const __nv_bfloat16* xi = x + (int64_t)img * H * H * C + cg * 8;
  __nv_bfloat16* yo = y + (int64_t)img * Ho * Ho * C + cg * 8;
  const int s0 = blockIdx.x * lanes * DW_SEG_PER_LANE, s1 = min(s0 + lanes * DW_SEG_PER_LANE, nseg);
  for (int sg = s0 + lane; sg < s1; sg += lanes) {
    const int oy = sg / sw, x0 = (sg - oy * sw) * 4;
    float acc[4][8];
#pragma unroll
    for (int o = 0; o < 4; ++o)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[o][e] = 0.f;
    // issue the whole 3 x NC window before any math (out-of-image taps read as zeros)
    uint4 xv[3][NC];
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int iy = oy * S + kh - 1;
      const bool rin = iy >= 0 && iy < H;
      const __nv_bfloat16* row = xi + (int64_t)iy * H * C;
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const int ix = x0 * S - 1 + j;
        xv[kh][j] = (rin && ix >= 0 && ix < H) ? *reinterpret_cast<const uint4*>(row + (int64_t)ix * C)
                                               : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll
      for (int j = 0; j < NC; ++j)
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          const int kw = j - o * S;
          if (kw >= 0 && kw <= 2) fma8(xv[kh][j], wt[kh * 3 + kw], acc[o]);
        }
#pragma unroll
    for (int o = 0; o < 4; ++o) *reinterpret_cast<uint4*>(yo + ((int64_t)oy * Ho + x0 + o) * C) = pack8(acc[o]);
  }
}

// dx (H x H) = transposed depthwise convolution of dy (Ho x Ho): dx[y][x] = sum dy[(y+1-kh)/S][(x+1-kw)/S] w[kh][kw]
template <int S>
static __global__ void __launch_bounds__(DW_THREADS) dw_dgrad_kernel(const __nv_bfloat16* __restrict__ dy,
                                                       const __nv_bfloat16* __restrict__ shadow, int64_t pstride,
                                                       int64_t woff, int Bp, int H, int C,
                                                       __nv_bfloat16* __restrict__ dx) {
  constexpr int NJ = S == 1 ? 6 : 3;  // gradient columns feeding a 4-output segment
  const int c8 = C >> 3, lanes = DW_THREADS / c8, cg = threadIdx.x % c8, lane = threadIdx.x / c8;
  if (lane >= lanes) return;
  const int img = blockIdx.y, g = img / Bp, Ho = H / S, sw = H >> 2, nseg = H * sw;
  uint4 wt[9];
  const __nv_bfloat16* w = shadow + (int64_t)g * pstride + woff + cg * 8;
#pragma unroll
  for (int t = 0; t < 9; ++t) wt[t] = *reinterpret_cast<const uint4*>(w + t * C);
  const __nv_bfloat16* di = dy + (int64_t)img * Ho * Ho * C + cg * 8;
  __nv_bfloat16* xo = dx + (int64_t)img * H * H * C + cg * 8;
  const int s0 = blockIdx.x * lanes * DW_SEG_PER_LANE, s1 = min(s0 + lanes * DW_SEG_PER_LANE, nseg);
  for (int sg = s0 + lane; sg < s1; sg += lanes) {
    const int yy = sg / sw, x0 = (sg - yy * sw) * 4;
    float acc[4][8];
#pragma unroll
    for (int o = 0; o < 4; ++o)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[o][e] = 0.f;
    uint4 dv[3][NJ];
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
      const int ny = yy + 1 - kh;
      const bool rin = ny >= 0 && !(S == 2 && (ny & 1)) && ny / S < Ho;
      const __nv_bfloat16* row = di + (int64_t)(ny / S) * Ho * C;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int dc = S == 1 ? x0 - 1 + j : (x0 >> 1) + j;  // gradient column
        dv[kh][j] = (rin && dc >= 0 && dc < Ho) ? *reinterpret_cast<const uint4*>(row + (int64_t)dc * C)
                                                : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int kh = 0; kh < 3; ++kh)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          const int kw = S == 1 ? o + 2 - j : o + 1 - 2 * j;  // x0 + o + 1 - dc * S
          if (kw >= 0 && kw <= 2) fma8(dv[kh][j], wt[kh * 3 + kw], acc[o]);
        }
#pragma unroll
    for (int o = 0; o < 4; ++o) *reinterpret_cast<uint4*>(xo + ((int64_t)yy * H + x0 + o) * C) = pack8(acc[o]);
  }
}

// weight gradient partials: part [G][DW_SPLIT][9][C] = this split's segments of sum x (*) dy.  grid (G, DW_SPLIT),
// 256 threads = (cg, lane) with 72 fp32 accumulators each; lanes reduced in a fixed order through dynamic
// shared memory (lanes x C/8 x 72 floats <= 72 KB).  Segments whose gradient is all zero (padding images) skip.
constexpr int DW_SPLIT = 64;
constexpr int DW_WGRAD_SMEM = DW_THREADS * 72 * 4;
template <int S>
static __global__ void __launch_bounds__(DW_THREADS, 3) dw_wgrad_kernel(const __nv_bfloat16* __restrict__ x,
                                                       const __nv_bfloat16* __restrict__ dy, int Bp, int H, int C,
                                                       float* __restrict__ part) {
  extern __shared__ float red[];
  constexpr int NC = 3 * S + 3;
  const int c8 = C >> 3, lanes = DW_THREADS / c8, cg = threadIdx.x % c8, lane = threadIdx.x / c8;
  const int g = blockIdx.x, sp = blockIdx.y, Ho = H / S, sw = Ho >> 2, segs_img = Ho * sw, nseg = Bp * segs_img;
  if (lane < lanes) {
    float acc[9][8];
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[t][e] = 0.f;
    const int q0 = (int)((int64_t)nseg * sp / DW_SPLIT), q1 = (int)((int64_t)nseg * (sp + 1) / DW_SPLIT);
    for (int q = q0 + lane; q < q1; q += lanes) {
      const int bi = q / segs_img, r = q - bi * segs_img, oy = r / sw, x0 = (r - oy * sw) * 4;
      const int64_t img = (int64_t)g * Bp + bi;
      const __nv_bfloat16* drow = dy + ((img * Ho + oy) * Ho + x0) * C + cg * 8;
      uint4 dv[4];
      unsigned any = 0;
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        dv[o] = *reinterpret_cast<const uint4*>(drow + (int64_t)o * C);
        any |= dv[o].x | dv[o].y | dv[o].z | dv[o].w;
      }
      if (!any) continue;
      const __nv_bfloat16* xi = x + img * H * H * C + cg * 8;
      uint4 xv[3][NC];
#pragma unroll
      for (int kh = 0; kh < 3; ++kh) {
        const int iy = oy * S + kh - 1;
        const bool rin = iy >= 0 && iy < H;
        const __nv_bfloat16* row = xi + (int64_t)iy * H * C;
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const int ix = x0 * S - 1 + j;
          xv[kh][j] = (rin && ix >= 0 && ix < H) ? *reinterpret_cast<const uint4*>(row + (int64_t)ix * C)
                                                 : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int kh = 0; kh < 3; ++kh)
#pragma unroll
        for (int j = 0; j < NC; ++j)
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            const int kw = j - o * S;
            if (kw >= 0 && kw <= 2) fma8(xv[kh][j], dv[o], acc[kh * 3 + kw]);
          }
    }
    float* rr = red + (lane * c8 + cg) * 72;
#pragma unroll
    for (int t = 0; t < 9; ++t)
#pragma unroll
      for (int e = 0; e < 8; ++e) rr[t * 8 + e] = acc[t][e];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < c8 * 72; i += blockDim.x) {
    const int cq = i / 72, rr = i - cq * 72;
    float sum = 0.f;
    for (int l = 0; l < lanes; ++l) sum += red[(l * c8 + cq) * 72 + rr];
    part[(((int64_t)g * DW_SPLIT + sp) * 9 + rr / 8) * C + cq * 8 + (rr & 7)] = sum;
  }
}

static int dw_blocks(int nseg, int C) {
  const int per = (DW_THREADS / (C / 8)) * DW_SEG_PER_LANE;
  return (nseg + per - 1) / per;
}

static void dw_fwd(const __nv_bfloat16* x, const __nv_bfloat16* shadow, int64_t pstride, int64_t woff, int n_img,
                   int Bp, int H, int C, int s, __nv_bfloat16* y, cudaStream_t st) {
  const int ho = H / s;
  const dim3 grid(dw_blocks(ho * (ho / 4), C), n_img);
  if (s == 1) dw_fwd_kernel<1><<<grid, DW_THREADS, 0, st>>>(x, shadow, pstride, woff, Bp, H, C, y);
  else dw_fwd_kernel<2><<<grid, DW_THREADS, 0, st>>>(x, shadow, pstride, woff, Bp, H, C, y);
}

static void dw_dgrad(const __nv_bfloat16* dy, const __nv_bfloat16* shadow, int64_t pstride, int64_t woff, int n_img,
                     int Bp, int H, int C, int s, __nv_bfloat16* dx, cudaStream_t st) {
  const dim3 grid(dw_blocks(H * (H / 4), C), n_img);
  if (s == 1) dw_dgrad_kernel<1><<<grid, DW_THREADS, 0, st>>>(dy, shadow, pstride, woff, Bp, H, C, dx);
  else dw_dgrad_kernel<2><<<grid, DW_THREADS, 0, st>>>(dy, shadow, pstride, woff, Bp, H, C, dx);
}

static void dw_wgrad(const __nv_bfloat16* x, const __nv_bfloat16* dy, int G, int Bp, int H, int C, int s, float* part,
                     cudaStream_t st) {
  const dim3 grid(G, DW_SPLIT);
  const size_t smem = (size_t)(DW_THREADS / (C / 8)) * (C / 8) * 72 * 4;
  if (s == 1) dw_wgrad_kernel<1><<<grid, DW_THREADS, smem, st>>>(x, dy, Bp, H, C, part);
  else dw_wgrad_kernel<2><<<grid, DW_THREADS, smem, st>>>(x, dy, Bp, H, C, part);
}

static int dw_setup() {
  FEDHC_CUDA_TRY(cudaFuncSetAttribute(dw_wgrad_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, DW_WGRAD_SMEM));
  FEDHC_CUDA_TRY(cudaFuncSetAttribute(dw_wgrad_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, DW_WGRAD_SMEM));
  return FEDHC_OK;
}

// master[9][C] -= lr * sum over splits (fixed order); shadow = bf16(master).  grid (ceil(9C / 256), G)
static __global__ void dw_sgd_kernel(const float* __restrict__ part, float* __restrict__ master,
                              __nv_bfloat16* __restrict__ shadow, int64_t pstride, int64_t woff, int C, float lr) {
  const int g = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 9 * C) return;
  float* m = master + (int64_t)g * pstride + woff;
  __nv_bfloat16* sh = shadow + (int64_t)g * pstride + woff;
  float s = 0.f;
  for (int sp = 0; sp < DW_SPLIT; ++sp) s += part[(((int64_t)g * DW_SPLIT + sp) * 9) * C + i];
  m[i] -= lr * s;
  sh[i] = __float2bfloat16_rn(m[i]);
}

static __global__ void step_inc_kernel(int* c) { *c += 1; }
static __global__ void add_count_kernel(unsigned long long* dst, const unsigned long long* src) { *dst += *src; }

}  // namespace mb
}  // namespace fedhc
