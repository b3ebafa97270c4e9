// Sample-weighted FedAvg -- fl_core.fedavg (fl_core.py:197-218).
//
// out[p] = base[p] + sum_k coef[k] * delta_k[p]
//
// HBM-bound streaming reduction.  Each thread owns 4 consecutive elements
// for the whole K loop, so every delta is read exactly once (16-byte loads
// for fp32, 2x16-byte for fp64), the base once and the output written once:
// algorithmic traffic (K * esize + 16) * n bytes.  Coefficients and delta
// pointers are staged through shared memory in blocks of kKTile.  The
// accumulation is fp64, in list order, with separately rounded multiply and
// add (no FMA contraction) -- the exact operation sequence of the
// reference's `out += (w / total) * d` loop, so fp64 inputs give
// bit-identical results.
//
// Short vectors (fewer than one 4-element thread per SM of the streaming
// kernel -- the logistic model has P = 7850) are latency-bound instead: a
// thread's K dependent loads cost ~K/8 memory round trips.  There
// `fedavg_tile_kernel` gives each CTA 128 elements, stages a [KT][128] tile of
// all its delta rows into shared memory with cp.async (every load in flight
// at once), then runs the same list-order fp64 chain from shared memory.
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"

namespace fedhc {

constexpr int kAvgThreads = 256;
constexpr int kKTile = 512;
constexpr int kUnroll = 8;

template <typename T>
struct Vec4;
template <>
struct Vec4<float> {
  static __device__ __forceinline__ void load(const float* p, double (&v)[4]) {
    const float4 q = __ldcs(reinterpret_cast<const float4*>(p));  // streaming: evict-first
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
  static __device__ __forceinline__ void load_tail(const float* p, int m, double (&v)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = i < m ? static_cast<double>(__ldcs(p + i)) : 0.0;
  }
};
template <>
struct Vec4<double> {
  static __device__ __forceinline__ void load(const double* p, double (&v)[4]) {
    const double2 a = __ldcs(reinterpret_cast<const double2*>(p));
    const double2 b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
  static __device__ __forceinline__ void load_tail(const double* p, int m, double (&v)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = i < m ? __ldcs(p + i) : 0.0;
  }
};

template <typename T>
__global__ void __launch_bounds__(kAvgThreads)
    fedavg_kernel(const T* const* __restrict__ ptrs, const T* __restrict__ packed, int64_t ld,
                  const double* __restrict__ coef, int K, const double* base, double* out, int64_t n) {
  __shared__ double s_coef[kKTile];
  __shared__ const T* s_ptr[kKTile];
  const int64_t p0 = ((int64_t)blockIdx.x * kAvgThreads + threadIdx.x) * 4;
  const bool active = p0 < n;
  const int m = active ? static_cast<int>(n - p0 < 4 ? n - p0 : 4) : 0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (base != nullptr && active) {
    for (int i = 0; i < m; ++i) acc[i] = base[p0 + i];
  }
  for (int k0 = 0; k0 < K; k0 += kKTile) {
    const int kt = min(kKTile, K - k0);
    __syncthreads();
    int misaligned = 0;
    for (int i = threadIdx.x; i < kt; i += kAvgThreads) {
      s_coef[i] = coef[k0 + i];
      const T* ptr = ptrs != nullptr ? ptrs[k0 + i] : packed + (int64_t)(k0 + i) * ld;
      s_ptr[i] = ptr;
      misaligned |= (reinterpret_cast<uintptr_t>(ptr) & 15) != 0;
    }
    // rows are 16-byte aligned (p0 % 4 == 0) -> 16-byte vector loads, else scalar
    const bool vec = (__syncthreads_or(misaligned) == 0) && m == 4;
    if (!active) continue;
    int k = 0;
    if (vec) {
      for (; k + kUnroll <= kt; k += kUnroll) {
        double v[kUnroll][4];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) Vec4<T>::load(s_ptr[k + u] + p0, v[u]);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const double c = s_coef[k + u];
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i] = __dadd_rn(acc[i], __dmul_rn(c, v[u][i]));
        }
      }
    }
    for (; k < kt; ++k) {
      double v[4];
      if (vec)
        Vec4<T>::load(s_ptr[k] + p0, v);
      else
        Vec4<T>::load_tail(s_ptr[k] + p0, m, v);
      const double c = s_coef[k];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = __dadd_rn(acc[i], __dmul_rn(c, v[i]));
    }
  }
  if (!active) return;
  if (m == 4 && (reinterpret_cast<uintptr_t>(out + p0) & 15) == 0) {
    reinterpret_cast<double2*>(out + p0)[0] = make_double2(acc[0], acc[1]);
    reinterpret_cast<double2*>(out + p0)[1] = make_double2(acc[2], acc[3]);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i < m) out[p0 + i] = acc[i];
  }
}

constexpr int kTileE = 128;          // elements (= threads) per CTA
constexpr int kTileBytes = 64 << 10;  // delta tile per K block

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(kTileE)
    fedavg_tile_kernel(const T* const* __restrict__ ptrs, const T* __restrict__ packed, int64_t ld,
                       const double* __restrict__ coef, int K, const double* base, double* out, int64_t n) {
  constexpr int KT = kTileBytes / (kTileE * (int)sizeof(T));  // delta rows per block
  constexpr int kPer = 16 / (int)sizeof(T);                   // elements per 16-byte chunk
  constexpr int kCpr = kTileE / kPer;                         // chunks per row
  extern __shared__ __align__(16) unsigned char smem[];
  T* tile = reinterpret_cast<T*>(smem);  // [KT][kTileE]
  __shared__ double s_coef[KT];
  __shared__ const T* s_ptr[KT];
  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * kTileE;
  const int64_t e = e0 + tid;
  double acc = (base != nullptr && e < n) ? base[e] : 0.0;
  for (int k0 = 0; k0 < K; k0 += KT) {
    const int kt = min(KT, K - k0);
    __syncthreads();  // previous block's tile fully consumed
    int misaligned = 0;
    for (int i = tid; i < kt; i += kTileE) {
      s_coef[i] = coef[k0 + i];
      const T* ptr = ptrs != nullptr ? ptrs[k0 + i] : packed + (int64_t)(k0 + i) * ld;
      s_ptr[i] = ptr;
      misaligned |= (reinterpret_cast<uintptr_t>(ptr) & 15) != 0;
    }
    const bool vec = __syncthreads_or(misaligned) == 0;
    if (vec) {
      for (int i = tid; i < kt * kCpr; i += kTileE) {
        const int r = i / kCpr, c = i - r * kCpr;
        const int64_t idx = e0 + (int64_t)c * kPer;
        const int64_t rem = n - idx;
        const int bytes = rem <= 0 ? 0 : (rem >= kPer ? 16 : static_cast<int>(rem) * (int)sizeof(T));
        cp_async16(tile + r * kTileE + c * kPer, bytes ? s_ptr[r] + idx : s_ptr[r], bytes);  // zero-fills
      }
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;\n" ::: "memory");
    } else {
      for (int r = 0; r < kt; ++r) tile[r * kTileE + tid] = e < n ? s_ptr[r][e] : T(0);
    }
    __syncthreads();
    if (e < n) {
      int k = 0;
      for (; k + 4 <= kt; k += 4) {
        const T v0 = tile[k * kTileE + tid], v1 = tile[(k + 1) * kTileE + tid];
        const T v2 = tile[(k + 2) * kTileE + tid], v3 = tile[(k + 3) * kTileE + tid];
        acc = __dadd_rn(acc, __dmul_rn(s_coef[k], static_cast<double>(v0)));
        acc = __dadd_rn(acc, __dmul_rn(s_coef[k + 1], static_cast<double>(v1)));
        acc = __dadd_rn(acc, __dmul_rn(s_coef[k + 2], static_cast<double>(v2)));
        acc = __dadd_rn(acc, __dmul_rn(s_coef[k + 3], static_cast<double>(v3)));
      }
      for (; k < kt; ++k) acc = __dadd_rn(acc, __dmul_rn(s_coef[k], static_cast<double>(tile[k * kTileE + tid])));
    }
  }
  if (e < n) out[e] = acc;
}

// Streaming FedAvg through the TMA engine: persistent CTAs walk 1024-element segments; a producer warp
// bulk-copies each delta row's segment (4 KB for fp32) into a ring of shared-memory stages, so one CTA keeps
// up to kBulkStages * kBulkRows rows in flight with one instruction per 4 KB (the per-thread vector loads of
// fedavg_kernel hold 128 B per thread and re-fetch a pointer per delta).  The 256 consumer threads run the
// same list-order fp64 chain on 4 elements each, so the result is bit-identical to fedavg_kernel.
constexpr int kBulkE = 1024;                       // elements per segment
constexpr int kBulkRows = 4, kBulkStages = 6;      // rows per stage, stages in the ring
constexpr int kBulkConsumers = kBulkE / 4;         // 256 threads x 4 elements
constexpr int kBulkThreads = kBulkConsumers + 32;  // + the producer warp

template <typename T>
__global__ void __launch_bounds__(kBulkThreads)
    fedavg_bulk_kernel(const T* const* __restrict__ ptrs, const T* __restrict__ packed, int64_t ld,
                       const double* __restrict__ coef, int K, const double* base, double* out, int64_t n) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int kRowBytes = kBulkE * (int)sizeof(T);
  T* ring = reinterpret_cast<T*>(smem);  // [stages][rows][kBulkE]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBulkStages * kBulkRows * kRowBytes);
  uint64_t* empty = full + kBulkStages;
  const int tid = threadIdx.x;
  const int64_t nseg = (n + kBulkE - 1) / kBulkE;
  const int groups = (K + kBulkRows - 1) / kBulkRows;  // stage fills per segment
  if (tid == 0) {
    for (int s = 0; s < kBulkStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBulkConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= kBulkConsumers) {
    // ---- producer warp: lane 0 issues the bulk copies of (segment, row group) in consumption order
    if (tid == kBulkConsumers) {
      int it = 0;
      for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
        const int64_t e0 = sg * kBulkE;
        // bytes of this segment (a ragged last segment rounded up to 16 bytes: rows are padded to that)
        const uint32_t bytes = (uint32_t)((min((int64_t)kBulkE, n - e0) * (int64_t)sizeof(T) + 15) & ~15);
        for (int gi = 0; gi < groups; ++gi, ++it) {
          const int s = it % kBulkStages, use = it / kBulkStages;
          if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
          const int k0 = gi * kBulkRows, kr = min(kBulkRows, K - k0);
          mbar_arrive_expect_tx(&full[s], bytes * kr);
          for (int r = 0; r < kr; ++r) {
            const T* row = ptrs != nullptr ? ptrs[k0 + r] : packed + (int64_t)(k0 + r) * ld;
            bulk_g2s(ring + ((size_t)s * kBulkRows + r) * kBulkE, row + e0, bytes, &full[s]);
          }
        }
      }
    }
    return;
  }
  // ---- consumers: element p = e0 + 4 tid .. + 3
  int it = 0;
  for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
    const int64_t p0 = sg * kBulkE + 4 * tid;
    const int m = p0 < n ? (int)min((int64_t)4, n - p0) : 0;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (base != nullptr)
      for (int i = 0; i < m; ++i) acc[i] = base[p0 + i];
    for (int gi = 0; gi < groups; ++gi, ++it) {
      const int s = it % kBulkStages, use = it / kBulkStages;
      mbar_wait(&full[s], use & 1);
      const int k0 = gi * kBulkRows, kr = min(kBulkRows, K - k0);
      for (int r = 0; r < kr; ++r) {
        double v[4];
        const T* q = ring + ((size_t)s * kBulkRows + r) * kBulkE + 4 * tid;
        if constexpr (sizeof(T) == 4) {
          const float4 f = *reinterpret_cast<const float4*>(q);
          v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
          const double2 a = reinterpret_cast<const double2*>(q)[0], b = reinterpret_cast<const double2*>(q)[1];
          v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
        }
        const double c = __ldg(coef + k0 + r);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = __dadd_rn(acc[i], __dmul_rn(c, v[i]));
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    }
    if (m == 4) {
      reinterpret_cast<double2*>(out + p0)[0] = make_double2(acc[0], acc[1]);
      reinterpret_cast<double2*>(out + p0)[1] = make_double2(acc[2], acc[3]);
    } else {
      for (int i = 0; i < m; ++i) out[p0 + i] = acc[i];
    }
  }
}

}  // namespace fedhc

using namespace fedhc;

extern "C" int fedhc_fedavg_coefficients(const double* weights, int n, double* coef_out) {
  // fl_core.py:201-209 (shape checks are the caller's: it owns the arrays)
  if (n <= 0) return fail(FEDHC_ERR_AGGREGATION, "no deltas to aggregate");
  for (int i = 0; i < n; ++i)
    if (weights[i] < 0) return fail(FEDHC_ERR_AGGREGATION, "weights must be non-negative");
  // CPython >= 3.12 float sum(): Neumaier compensated summation.
  double s = 0.0, comp = 0.0;
  for (int i = 0; i < n; ++i) {
    const double x = weights[i];
    const double t = s + x;
    if (fabs(s) >= fabs(x))
      comp += (s - t) + x;
    else
      comp += (x - t) + s;
    s = t;
  }
  if (comp != 0.0 && isfinite(comp)) s += comp;
  if (s == 0.0) return fail(FEDHC_ERR_AGGREGATION, "weights must not all be zero");
  for (int i = 0; i < n; ++i) coef_out[i] = weights[i] / s;
  return FEDHC_OK;
}

extern "C" int fedhc_fedavg(const void* const* deltas, const void* packed, int64_t ld, int dtype,
                            const double* coef, int n_deltas, const double* base, double* out, int64_t n,
                            void* stream) {
  if (n_deltas <= 0) return fail(FEDHC_ERR_AGGREGATION, "no deltas to aggregate");
  if (n < 0) return fail(FEDHC_ERR_VALUE, "fedavg: negative length");
  if (deltas == nullptr && packed == nullptr) return fail(FEDHC_ERR_VALUE, "fedavg: no delta storage given");
  if (coef == nullptr || out == nullptr) return fail(FEDHC_ERR_VALUE, "fedavg: null coefficient/output");
  if (n == 0) return FEDHC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = (n + 4LL * kAvgThreads - 1) / (4LL * kAvgThreads);
  if (blocks > 0x7fffffffLL) return fail(FEDHC_ERR_UNSUPPORTED, "fedavg: vector too long");
  if (dtype != FEDHC_F32 && dtype != FEDHC_F64)
    return fail(FEDHC_ERR_VALUE, "fedavg: dtype must be FEDHC_F32 or FEDHC_F64");
  int dev = 0;
  FEDHC_CUDA_TRY(cudaGetDevice(&dev));
  int sms = 0;
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (blocks < sms) {  // short vector: latency-bound, stage every delta row through shared memory at once
    FEDHC_CUDA_TRY(smem_optin_max(reinterpret_cast<const void*>(fedavg_tile_kernel<float>)));
    FEDHC_CUDA_TRY(smem_optin_max(reinterpret_cast<const void*>(fedavg_tile_kernel<double>)));
    const unsigned tb = static_cast<unsigned>((n + kTileE - 1) / kTileE);
    if (dtype == FEDHC_F32)
      fedavg_tile_kernel<float><<<tb, kTileE, kTileBytes, st>>>(
          reinterpret_cast<const float* const*>(deltas), static_cast<const float*>(packed), ld, coef, n_deltas,
          base, out, n);
    else
      fedavg_tile_kernel<double><<<tb, kTileE, kTileBytes, st>>>(
          reinterpret_cast<const double* const*>(deltas), static_cast<const double*>(packed), ld, coef, n_deltas,
          base, out, n);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }
  // packed rows with a 16-byte pitch, at the sweep points where it measured faster (short vectors: the
  // per-thread kernel runs few waves; many deltas: it re-fetches a pointer per delta): the TMA-fed persistent
  // kernel (bit-identical).  Pointer rows keep the per-thread streaming kernel (their alignment is only known on
  // the device).  profiles/r2c_fedavg.md has both kernels over the config-5 sweep.
  static const bool no_bulk = getenv("FEDHC_FEDAVG_NO_BULK") != nullptr;
  const int esz = dtype == FEDHC_F32 ? 4 : 8;
  if (!no_bulk && deltas == nullptr && (ld * esz) % 16 == 0 && (reinterpret_cast<uintptr_t>(packed) & 15) == 0 &&
      ((n <= (4LL << 20) && n_deltas >= 32) || n_deltas >= 500)) {
    const int smem = kBulkStages * kBulkRows * kBulkE * esz + 2 * kBulkStages * 8;
    const void* kern = dtype == FEDHC_F32 ? reinterpret_cast<const void*>(fedavg_bulk_kernel<float>)
                                          : reinterpret_cast<const void*>(fedavg_bulk_kernel<double>);
    static int per_sm_of[64][2] = {};  // resident CTAs per SM, per device and dtype (set once; benign race)
    int& per_sm = per_sm_of[dev & 63][dtype == FEDHC_F32 ? 0 : 1];
    if (per_sm == 0) {
      FEDHC_CUDA_TRY(smem_optin_max(kern));
      int v = 0;
      FEDHC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, kBulkThreads, smem));
      per_sm = std::max(v, 1);
    }
    const int64_t nseg = (n + kBulkE - 1) / kBulkE;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(nseg, (int64_t)per_sm * sms));
    if (dtype == FEDHC_F32)
      fedavg_bulk_kernel<float><<<grid, kBulkThreads, smem, st>>>(nullptr, static_cast<const float*>(packed), ld,
                                                                   coef, n_deltas, base, out, n);
    else
      fedavg_bulk_kernel<double><<<grid, kBulkThreads, smem, st>>>(nullptr, static_cast<const double*>(packed), ld,
                                                                    coef, n_deltas, base, out, n);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }
  if (dtype == FEDHC_F32) {
    fedavg_kernel<float><<<(unsigned)blocks, kAvgThreads, 0, st>>>(
        reinterpret_cast<const float* const*>(deltas), static_cast<const float*>(packed), ld, coef, n_deltas, base,
        out, n);
  } else if (dtype == FEDHC_F64) {
    fedavg_kernel<double><<<(unsigned)blocks, kAvgThreads, 0, st>>>(
        reinterpret_cast<const double* const*>(deltas), static_cast<const double*>(packed), ld, coef, n_deltas,
        base, out, n);
  } else {
    return fail(FEDHC_ERR_VALUE, "fedavg: dtype must be FEDHC_F32 or FEDHC_F64");
  }
  FEDHC_CUDA_TRY(cudaGetLastError());
  return FEDHC_OK;
}
