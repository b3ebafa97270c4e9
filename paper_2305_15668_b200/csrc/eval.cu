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

// Fast path for F % 4 == 0, F <= 128 * NCH, C <= 16 NG (the logistic models of the round loop): a warp takes
// kER rows at a time and issues all of their 16-byte loads before any arithmetic (the warp-per-row loop
// above waited on one load per 128 features), each W^T float4 read from shared memory serves kER rows (W^T
// re-reads were the bound: 50 KB of shared-memory traffic per row), each 16-class group's sums are reduced
// with a halving butterfly (16 shuffles per row instead of 5 per class), every lane keeps its first-max
// candidate over the groups, and one (value, class) warp max ends the row.  Used by the round loop's
// accuracy, which runs on a few side SMs; NG = 4 covers FEMNIST's 62 classes (the per-class warp sums of
// eval_kernel made that 0.86 ms on 48 SMs for 16k rows).
constexpr int kRowsThreads = 256;
constexpr int kER = 4;
template <int NCH, int NG>
__global__ void __launch_bounds__(kRowsThreads, 1)
    eval_rows_kernel(const float* __restrict__ x, const int32_t* __restrict__ y, int64_t n, int F, int C, int Fs,
                     const double* __restrict__ params, unsigned long long* correct) {
  constexpr int CP = 16 * NG;  // padded classes
  extern __shared__ __align__(16) unsigned char smem[];
  float* Wt = reinterpret_cast<float*>(smem);  // [CP][Fs], classes >= C zero
  float* bias = Wt + (size_t)CP * Fs;          // [CP]
  __shared__ unsigned int s_count;
  if (threadIdx.x == 0) s_count = 0;
  for (int i = threadIdx.x; i < CP * Fs; i += kRowsThreads) {
    const int c = i / Fs, f = i - c * Fs;
    Wt[i] = (c < C && f < F) ? static_cast<float>(params[(size_t)f * C + c]) : 0.f;
  }
  for (int c = threadIdx.x; c < CP; c += kRowsThreads) bias[c] = c < C ? static_cast<float>(params[(size_t)F * C + c]) : 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int cls = 8 * ((lane >> 4) & 1) + 4 * ((lane >> 3) & 1) + 2 * ((lane >> 2) & 1) + ((lane >> 1) & 1);
  const int64_t warps_total = (int64_t)gridDim.x * (kRowsThreads / 32);
  unsigned int mine = 0;
  for (int64_t r0 = kER * ((int64_t)blockIdx.x * (kRowsThreads / 32) + (threadIdx.x >> 5)); r0 < n;
       r0 += kER * warps_total) {
    float4 xv[kER][NCH];
#pragma unroll
    for (int q = 0; q < kER; ++q) {
      const float* xr = x + min(r0 + q, n - 1) * F;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int f = 4 * lane + 128 * j;
        xv[q][j] = f < F ? __ldcs(reinterpret_cast<const float4*>(xr + f)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    int yr[kER];
#pragma unroll
    for (int q = 0; q < kER; ++q) yr[q] = r0 + q < n ? y[r0 + q] : -1;
    float best[kER];
    int bi[kER];
#pragma unroll
    for (int q = 0; q < kER; ++q) {
      best[q] = -FLT_MAX;
      bi[q] = CP;
    }
#pragma unroll 1
    for (int gi = 0; gi < NG; ++gi) {
      const float* Wg = Wt + (size_t)16 * gi * Fs;
      float v[kER][16];
#pragma unroll
      for (int q = 0; q < kER; ++q)
#pragma unroll
        for (int u = 0; u < 16; ++u) v[q][u] = 0.f;
#pragma unroll
      for (int j = 0; j < NCH; ++j) {
        const int f = 4 * lane + 128 * j;
        if (f < Fs) {
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const float4 w = *reinterpret_cast<const float4*>(Wg + (size_t)u * Fs + f);
#pragma unroll
            for (int q = 0; q < kER; ++q)
              v[q][u] = fmaf(xv[q][j].x, w.x, fmaf(xv[q][j].y, w.y, fmaf(xv[q][j].z, w.z, fmaf(xv[q][j].w, w.w, v[q][u]))));
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kER; ++q) {
        // halving butterfly: after offset o a lane keeps the half of its classes selected by (lane & o)
#pragma unroll
        for (int o = 16, h = 8; o >= 2; o >>= 1, h >>= 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int j = 0; j < h; ++j) {
            const float send = up ? v[q][j] : v[q][j + h];
            const float keep = up ? v[q][j + h] : v[q][j];
            v[q][j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        const int c = 16 * gi + cls;
        float s = v[q][0] + __shfl_xor_sync(0xffffffffu, v[q][0], 1);
        s = c < C ? s + bias[c] : -FLT_MAX;
        if (s > best[q]) {  // groups in class order: strict keeps the first maximum
          best[q] = s;
          bi[q] = c;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kER; ++q) {
      float bv = best[q];
      int bc = bi[q];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {  // (value, class) max; ties -> the smaller class (np.argmax)
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bc, o);
        if (ov > bv || (ov == bv && oi < bc)) {
          bv = ov;
          bc = oi;
        }
      }
      if (lane == 0 && bc == yr[q]) ++mine;
    }
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
  const int nch = (n_features + 127) / 128;
  const int ng = n_classes <= 16 ? 1 : n_classes <= 32 ? 2 : n_classes <= 64 ? 4 : 0;
  const size_t smemg = ((size_t)16 * ng * Fs + 16 * ng) * 4;
  if (n_features % 4 == 0 && ng > 0 && nch <= 8 && smemg <= (size_t)max_smem) {
    const int64_t need2 = (n + kER * (kRowsThreads / 32) - 1) / (kER * (kRowsThreads / 32));
    const int b2 = static_cast<int>(std::min<int64_t>(need2, (int64_t)cap));  // one CTA per SM (~215 registers)
#define FEDHC_EVAL_ROWS(N, G)                                                                                        \
  case N:                                                                                                           \
    if (smemg > 48 * 1024) FEDHC_CUDA_TRY(smem_optin_max(reinterpret_cast<const void*>(eval_rows_kernel<N, G>)));  \
    eval_rows_kernel<N, G><<<b2, kRowsThreads, smemg, st>>>(x, y, n, n_features, n_classes, Fs, params, correct);   \
    break;
#define FEDHC_EVAL_NCH(G)                                                                                            \
    switch (nch) {                                                                                                  \
      FEDHC_EVAL_ROWS(1, G) FEDHC_EVAL_ROWS(2, G) FEDHC_EVAL_ROWS(3, G) FEDHC_EVAL_ROWS(4, G)                       \
      FEDHC_EVAL_ROWS(5, G) FEDHC_EVAL_ROWS(6, G) FEDHC_EVAL_ROWS(7, G) FEDHC_EVAL_ROWS(8, G)                       \
    }
    if (ng == 1) {
      FEDHC_EVAL_NCH(1)
    } else if (ng == 2) {
      FEDHC_EVAL_NCH(2)
    } else {
      FEDHC_EVAL_NCH(4)
    }
#undef FEDHC_EVAL_NCH
#undef FEDHC_EVAL_ROWS
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }
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
