// Test-set accuracy -- fl_core.evaluate_accuracy (fl_core.py:154-160):
// mean(argmax(X @ W + b) == y) with numpy's first-max tie-break.
//
// Grid-stride over rows, one warp per row.  W^T (fp32) is staged once per
// CTA in shared memory; each lane streams 16-byte chunks of its row
// (coalesced) and accumulates 16 classes at a time; lane 0 keeps the first
// strict maximum.  One atomic per CTA for the correct-count.
#include <float.h>

#include <algorithm>

#include "common.cuh"

namespace fedhc {

constexpr int kEvalThreads = 512;
constexpr int kEvalCT = 16;

// GW = false: W^T staged in shared memory (every model the trainers' fast paths cover);
// GW = true: models too large for shared memory read W (fp64, L2-resident) from global memory.
template <bool GW>
__global__ void __launch_bounds__(kEvalThreads, 1)
    eval_kernel(const float* __restrict__ x, const int32_t* __restrict__ y, int64_t n, int F, int C, int Fs,
                const double* __restrict__ params, unsigned long long* correct) {
  extern __shared__ __align__(16) unsigned char smem[];
  float* Wt = reinterpret_cast<float*>(smem);  // [C][Fs]
  float* bias = GW ? Wt : Wt + (size_t)C * Fs;  // [C]
  __shared__ unsigned int s_count;
  if (threadIdx.x == 0) s_count = 0;
  if (!GW)
    for (int i = threadIdx.x; i < C * Fs; i += kEvalThreads) {
      const int c = i / Fs, f = i - c * Fs;
      Wt[i] = f < F ? static_cast<float>(params[(size_t)f * C + c]) : 0.f;
    }
  for (int c = threadIdx.x; c < C; c += kEvalThreads) bias[c] = static_cast<float>(params[(size_t)F * C + c]);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (kEvalThreads / 32);
  unsigned int mine = 0;
  const bool vec = (F % 4) == 0;
  for (int64_t r = (int64_t)blockIdx.x * (kEvalThreads / 32) + (threadIdx.x >> 5); r < n; r += warps_total) {
    const float* xr = x + r * F;
    float best = -FLT_MAX;
    int besti = 0;
    for (int c0 = 0; c0 < C; c0 += kEvalCT) {
      float acc[kEvalCT];
#pragma unroll
      for (int u = 0; u < kEvalCT; ++u) acc[u] = 0.f;
      if (GW) {
        for (int f = lane; f < F; f += 32) {
          const float xv = __ldg(xr + f);
#pragma unroll
          for (int u = 0; u < kEvalCT; ++u)
            if (c0 + u < C) acc[u] = fmaf(xv, static_cast<float>(__ldg(params + (size_t)f * C + c0 + u)), acc[u]);
        }
      } else if (vec) {
        for (int f = 4 * lane; f < F; f += 128) {
          const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + f));
#pragma unroll
          for (int u = 0; u < kEvalCT; ++u) {
            if (c0 + u < C) {
              const float4 w = *reinterpret_cast<const float4*>(Wt + (size_t)(c0 + u) * Fs + f);
              acc[u] = fmaf(xv.x, w.x, fmaf(xv.y, w.y, fmaf(xv.z, w.z, fmaf(xv.w, w.w, acc[u]))));
            }
          }
        }
      } else {
        for (int f = lane; f < F; f += 32) {
          const float xv = __ldg(xr + f);
#pragma unroll
          for (int u = 0; u < kEvalCT; ++u)
            if (c0 + u < C) acc[u] = fmaf(xv, Wt[(size_t)(c0 + u) * Fs + f], acc[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < kEvalCT; ++u) {
        if (c0 + u < C) {
          const float s = warp_sum(acc[u]) + bias[c0 + u];
          if (s > best) {  // strict: first maximum wins (np.argmax)
            best = s;
            besti = c0 + u;
          }
        }
      }
    }
    if (lane == 0 && besti == y[r]) ++mine;
  }
  if (lane == 0 && mine) atomicAdd(&s_count, mine);
  __syncthreads();
  if (threadIdx.x == 0 && s_count) atomicAdd(correct, static_cast<unsigned long long>(s_count));
}

}  // namespace fedhc

using namespace fedhc;

extern "C" int fedhc_eval_ctas(const float* x, const int32_t* y, int64_t n, int n_features, int n_classes,
                               const double* params, unsigned long long* correct, int max_ctas, void* stream) {
  if (n_features < 1 || n_classes < 1) return fail(FEDHC_ERR_VALUE, "eval: bad shape");
  if (n <= 0) return FEDHC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, max_smem = 0, sms = 0;
  FEDHC_CUDA_TRY(cudaGetDevice(&dev));
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int Fs = (n_features + 3) / 4 * 4;
  size_t smem = ((size_t)n_classes * Fs + n_classes) * 4;
  const bool gw = smem > (size_t)max_smem;
  if (gw) smem = (size_t)n_classes * 4;
  if (smem > (size_t)max_smem) return fail(FEDHC_ERR_UNSUPPORTED, "eval: too many classes");
  const int64_t need = (n + (kEvalThreads / 32) - 1) / (kEvalThreads / 32);
  const int cap = max_ctas > 0 ? std::min(max_ctas, sms) : sms;
  const int blocks = static_cast<int>(std::min<int64_t>(need, (int64_t)cap));
  if (gw) {
    if (smem > 48 * 1024) FEDHC_CUDA_TRY(smem_optin_max(reinterpret_cast<const void*>(eval_kernel<true>)));
    eval_kernel<true><<<blocks, kEvalThreads, smem, st>>>(x, y, n, n_features, n_classes, Fs, params, correct);
  } else {
    if (smem > 48 * 1024) FEDHC_CUDA_TRY(smem_optin_max(reinterpret_cast<const void*>(eval_kernel<false>)));
    eval_kernel<false><<<blocks, kEvalThreads, smem, st>>>(x, y, n, n_features, n_classes, Fs, params, correct);
  }
  FEDHC_CUDA_TRY(cudaGetLastError());
  return FEDHC_OK;
}

extern "C" int fedhc_eval(const float* x, const int32_t* y, int64_t n, int n_features, int n_classes,
                          const double* params, unsigned long long* correct, void* stream) {
  return fedhc_eval_ctas(x, y, n, n_features, n_classes, params, correct, 0, stream);
}
