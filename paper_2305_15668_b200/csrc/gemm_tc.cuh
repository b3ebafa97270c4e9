// Grouped tcgen05 GEMM: plan once (tensor maps, kernel choice), launch many times.
// Used by the C-ABI entry fedhc_gemm and by the CNN client engine (cnn.cu), which
// builds every per-layer plan when its workspace is created so a training step
// is launches only (and can be captured into a CUDA graph).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"

namespace fedhc {
namespace tc {

struct Epilogue {
  int kind;             // FEDHC_EPI_*
  void* D;              // F32 / BF16 / BIAS_RELU_BF16 output
  int64_t ldd, d_gstride;
  const float* bias;    // BIAS_RELU_BF16
  int bias_per_row;
  int64_t bias_gstride;
  float* master;        // SGD: fp32 master, same indexing as D
  __nv_bfloat16* shadow;  // SGD: optional bf16 copy
  float lr;
  const __nv_bfloat16* mask;  // RELU_MASK_BF16: D = acc * (mask > 0), mask indexed like D
  float* rowsum;        // RELU_MASK_BF16 (optional, single N tile): rowsum[g*M + m] = sum_n D
};

// Implicit-GEMM convolution modes (see gemm_tc.cu conv_loads / nhwc_loads).
//   CONV_FWD/DGRAD/WGRAD: the FEMNIST CNN's conv2 (5x5 'same' on 14x14 maps, channel-pair layout).
//   NHWC_FWD/DGRAD/WGRAD: k x k (1 or 3) 'same' convolutions with stride s (1 or 2) on [img][H][W][C]
//   bf16 maps, C multiple of 64 (ResNet client models).  DGRAD is stride 1 only: a stride-2 data gradient
//   runs on the zero-upsampled output gradient.
enum { CONV_NONE = 0, CONV_FWD = 1, CONV_DGRAD = 2, CONV_WGRAD = 3, NHWC_FWD = 4, NHWC_DGRAD = 5, NHWC_WGRAD = 6 };
struct ConvSpec {
  int mode;   // CONV_* / NHWC_*
  int bp;     // images per group
  // NHWC_*: input map H x W x cin, kernel k, stride s, output (H / s) x (W / s) x cout
  int H, W, cin, cout, k, s;
  // derived (gemm_plan): 128-slot M tile = ib images x hb rows x wo columns; 64-slot WGRAD K block
  int ho, wo, hb, ib, khb, kib;
};

struct GemmPlan {
  CUtensorMap ma, mb;   // operands
  CUtensorMap mo;       // epilogue store target: D, or the SGD fp32 master
  CUtensorMap ms;       // SGD bf16 shadow (optional)
  CUtensorMap ml;       // epilogue load source: SGD master or ReLU-backward mask
  Epilogue ep;
  ConvSpec conv;
  int G, M, N, K;
  const void* kern;
  int grid, smem, stages, nst;
  int sms, tiles_per_g;  // persistent grid = min(G * tiles_per_g, sms)
};

// Validate a problem and build its plan (no launch).  Returns a FEDHC_* status.
// conv != nullptr: implicit-GEMM convolution (a.A / a.B / a.D are the activation / weight / output
// tensors of the mode, M / N / K its virtual GEMM shape; conv2 fwd: M = 256 * bp, N = 64, K = 960;
// dgrad: M = 256 * bp, N = 32, K = 1600; wgrad: M = 1024, N = 64, K = 256 * bp, SGD epilogue).
int gemm_plan(const fedhc_gemm_args& a, GemmPlan* plan, const ConvSpec* conv = nullptr);
// Launch a plan on a stream.
// G_run in [1, p.G]: run only the first G_run groups (same maps and buffers); <= 0: all of them
int gemm_run(const GemmPlan& p, cudaStream_t st, int G_run = 0);

}  // namespace tc
}  // namespace fedhc
