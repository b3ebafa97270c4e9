// Grouped GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   D_g[M x N] = epilogue( A_g[M x K] . B_g[N x K]^T ),  g = 0..G-1, bf16 operands, fp32 accumulate
//
// Operands may be K-major ([rows][K], e.g. activations, weights in forward) or
// MN-major ([K][rows], e.g. the transposed operands of dgrad / wgrad) so no
// transposes are materialised.  Epilogues: fp32 store, bf16 store,
// bias (+ per-row or per-column) + ReLU -> bf16, and an in-place SGD step on
// an fp32 master (W -= lr * acc) with an optional bf16 shadow copy.
//
// The per-client dense contraction of the FL client models (one GEMM per
// client per layer, all clients of a round in one launch): the foundation of
// the CNN / MLP client path (BASELINE.json configs 2-4).
//
// Structure (one persistent CTA per SM, 192 threads, warp-specialised):
//   warp 0  TMA producer: 3-D tensor maps {K, rows, G} with 128-byte swizzle
//           land BMx64 / BNx64 bf16 tiles in the canonical SW128 layouts
//           into a 4-8 stage ring (full/empty mbarriers, expect_tx bytes).
//   warp 1  MMA issuer: one elected thread issues tcgen05.mma.cta_group::1
//           .kind::f16 (M=BM in {64, 128}, N=BN in {32..256}, K=16) from
//           shared-memory descriptors into a double-buffered TMEM accumulator
//           (2 x BN fp32 columns; all 512 columns at BN=256).  M=64 keeps the
//           batch-sized (B=64) client GEMMs on the tensor pipe;
//           tcgen05.commit releases ring stages and signals the epilogue.
//   warps 2-5  epilogue: tcgen05.ld (32x32b.x32) TMEM -> registers -> global,
//           one TMEM lane quadrant per warp, then release the accumulator.
// Tile order: g-major, then M, then N, strided over CTAs.
#include <cuda.h>
#include <cuda_bf16.h>

#include <mutex>
#include <string>

#include "gemm_tc.cuh"

namespace fedhc {

namespace tc {

constexpr int BK = 64;
constexpr int kThreads = 192;

template <int BM, int BN>
struct Cfg {
  static constexpr int kTileABytes = BM * BK * 2;
  static constexpr int kTileBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kTileABytes + kTileBBytes;
  static constexpr int STAGES = (200 * 1024) / kStageBytes > 8 ? 8 : (200 * 1024) / kStageBytes;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered fp32 accumulator
  static constexpr int smem_bytes() { return STAGES * kStageBytes + 1024 + 256; }
};

// M=64 accumulators occupy TMEM lanes 0-15 of each 32-lane quadrant (row = 16*q + lane,
// CUTLASS cute/atom/mma_traits_sm100.hpp tmem_frg M_MMA == 64); M=128 uses all lanes.
template <int BM, int BN, bool A_MN, bool B_MN>
__host__ __device__ constexpr uint32_t idesc() {
  return (1u << 4)                    // D format: f32
         | (1u << 7)                  // A format: bf16
         | (1u << 10)                 // B format: bf16
         | ((A_MN ? 1u : 0u) << 15)   // A major (1 = MN)
         | ((B_MN ? 1u : 0u) << 16)   // B major (1 = MN)
         | ((uint32_t)(BN >> 3) << 17)  // N
         | ((uint32_t)(BM >> 4) << 24); // M
}

// Canonical 128-byte-swizzled layouts (CUTLASS make_umma_desc, cute/atom/mma_traits_sm100.hpp):
//   K-major : 8-row core groups 1024 B apart (SBO), LBO unused; +32 B per K=16 step.
//   MN-major: 64-element MN atoms 8 KB apart (LBO, one TMA box of 64 K-rows each),
//             8-row K groups 1024 B apart (SBO); +2048 B per K=16 step.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);       // start address
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16; // leading byte offset
  d |= (uint64_t)(1024 >> 4) << 32;                 // stride byte offset = 1024 B
  d |= (uint64_t)1 << 46;                           // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void tma_load_3d(uint32_t smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}



template <int BM, int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                        int G, int M, int N, int K, const Epilogue ep) {
  using CF = Cfg<BM, BN>;
  constexpr int STAGES = CF::STAGES, kStageBytes = CF::kStageBytes, kTmemCols = CF::kTmemCols;
  constexpr int kTileABytes = CF::kTileABytes;
  constexpr uint32_t kIdesc = idesc<BM, BN, A_MN, B_MN>();
  constexpr uint32_t kLboA = A_MN ? 64 * BK * 2 : 16, kLboB = B_MN ? 64 * BK * 2 : 16;
  constexpr uint32_t kStepA = A_MN ? 2048 : 32, kStepB = B_MN ? 2048 : 32;  // bytes per K=16
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;       // [2] accumulator drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = M / BM, tiles_n = N / BN;
  const int n_tiles = G * tiles_m * tiles_n;
  const int kblocks = K / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM allocation by one full warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int g = t / (tiles_m * tiles_n);
        const int r = t - g * tiles_m * tiles_n;
        const int m0 = (r / tiles_n) * BM, n0 = (r % tiles_n) * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], kStageBytes);
          const uint32_t sa = smem_u32(smem + s * kStageBytes), sb = sa + kTileABytes;
          if (A_MN) {
#pragma unroll
            for (int h = 0; h < BM / 64; ++h) tma_load_3d(sa + h * 64 * BK * 2, &map_a, &full[s], m0 + 64 * h, kb * BK, g);
          } else {
            tma_load_3d(sa, &map_a, &full[s], kb * BK, m0, g);
          }
          if (B_MN) {
#pragma unroll
            for (int h = 0; h < BN / 64; ++h) tma_load_3d(sb + h * 64 * BK * 2, &map_b, &full[s], n0 + 64 * h, kb * BK, g);
          } else {
            tma_load_3d(sb, &map_b, &full[s], kb * BK, n0, g);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * kStageBytes);
          const uint64_t da = sw128_desc(sa, kLboA), db = sw128_desc(sa + kTileABytes, kLboB);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(tmem_d, da + (kStepA >> 4) * k, db + (kStepB >> 4) * k, kIdesc, (kb | k) != 0);
          umma_commit(&empty[s]);  // ring stage free once these MMAs retire
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // epilogue warps 2..5 -> TMEM lane quadrant (warp % 4): thread = one output row
    // (M=64: lanes 0-15 of the quadrant hold rows 16*q + lane)
    const int q = warp & 3;
    constexpr int kRowsPerWarp = BM / 4;
    const bool active = lane < kRowsPerWarp;
    int it = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const int g = t / (tiles_m * tiles_n);
      const int r = t - g * tiles_m * tiles_n;
      const int m0 = (r / tiles_n) * BM, n0 = (r % tiles_n) * BN;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int row = m0 + kRowsPerWarp * q + (active ? lane : 0);
      const int64_t base = (int64_t)g * ep.d_gstride + (int64_t)row * ep.ldd + n0;
      const float rbias = (ep.kind == FEDHC_EPI_BIAS_RELU_BF16 && ep.bias_per_row)
                              ? ep.bias[(int64_t)g * ep.bias_gstride + row] : 0.f;
      float rsum = 0.f;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(32 * q) << 16) + acc * BN + 32 * c, v);
        if (!active) continue;
        const int64_t o = base + 32 * c;
        if (ep.kind == FEDHC_EPI_F32) {
          float* d = static_cast<float*>(ep.D) + o;
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(d + i) = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                                            __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
        } else if (ep.kind == FEDHC_EPI_SGD) {
          float* w = ep.master + o;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            float4 m4 = *reinterpret_cast<float4*>(w + i);
            m4.x -= ep.lr * __uint_as_float(v[i]);
            m4.y -= ep.lr * __uint_as_float(v[i + 1]);
            m4.z -= ep.lr * __uint_as_float(v[i + 2]);
            m4.w -= ep.lr * __uint_as_float(v[i + 3]);
            *reinterpret_cast<float4*>(w + i) = m4;
            if (ep.shadow) {
              __nv_bfloat162* sh = reinterpret_cast<__nv_bfloat162*>(ep.shadow + o + i);
              sh[0] = __floats2bfloat162_rn(m4.x, m4.y);
              sh[1] = __floats2bfloat162_rn(m4.z, m4.w);
            }
          }
        } else {
          const int kind = ep.kind;
          __nv_bfloat16* d = static_cast<__nv_bfloat16*>(ep.D) + o;
          const float* cb = (kind == FEDHC_EPI_BIAS_RELU_BF16 && !ep.bias_per_row)
                                ? ep.bias + (int64_t)g * ep.bias_gstride + n0 + 32 * c : nullptr;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            float f[8];
            uint4 mk = make_uint4(0, 0, 0, 0);
            if (kind == FEDHC_EPI_RELU_MASK_BF16) mk = *reinterpret_cast<const uint4*>(ep.mask + o + i);
            const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mk);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              float x = __uint_as_float(v[i + u]);
              if (kind == FEDHC_EPI_BIAS_RELU_BF16) x = fmaxf(x + (cb ? cb[i + u] : rbias), 0.f);
              if (kind == FEDHC_EPI_RELU_MASK_BF16) x = __bfloat162float(mb[u]) > 0.f ? x : 0.f;
              f[u] = x;
            }
            uint4 pk;
            __nv_bfloat162 t0 = __floats2bfloat162_rn(f[0], f[1]), t1 = __floats2bfloat162_rn(f[2], f[3]);
            __nv_bfloat162 t2 = __floats2bfloat162_rn(f[4], f[5]), t3 = __floats2bfloat162_rn(f[6], f[7]);
            pk.x = *reinterpret_cast<uint32_t*>(&t0);
            pk.y = *reinterpret_cast<uint32_t*>(&t1);
            pk.z = *reinterpret_cast<uint32_t*>(&t2);
            pk.w = *reinterpret_cast<uint32_t*>(&t3);
            *reinterpret_cast<uint4*>(d + i) = pk;
            // row sum of the stored (bf16-rounded) values, fixed order -> deterministic
            const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(&pk);
#pragma unroll
            for (int u = 0; u < 8; ++u) rsum += __bfloat162float(pb[u]);
          }
        }
      }
      if (ep.rowsum && active) ep.rowsum[(int64_t)g * M + row] = rsum;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols));
  }
}

// ---- host: tensor maps through the driver entry point --------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// bf16 tensor [G][outer][inner] (group stride gstride elements, 0 = dense) -> 3-D map,
// box {64, box_outer, 1}, 128-byte swizzle
static int make_map(CUtensorMap* map, const void* base, int G, int outer, int inner, int box_outer,
                    int64_t gstride) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(FEDHC_ERR_UNSUPPORTED, "gemm: cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)outer, (cuuint64_t)G};
  if (gstride <= 0) gstride = (int64_t)outer * inner;
  if (gstride % 8) return fail(FEDHC_ERR_VALUE, "gemm: operand group stride must be a multiple of 8 elements");
  cuuint64_t strides[2] = {(cuuint64_t)inner * 2, (cuuint64_t)gstride * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FEDHC_ERR_CUDA, "gemm: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return FEDHC_OK;
}

template <int BM, int BN, bool A_MN, bool B_MN>
static int plan_kernel(const fedhc_gemm_args& a, GemmPlan* p) {
  int rc = A_MN ? make_map(&p->ma, a.A, a.G, a.K, a.M, 64, a.a_gstride)
                 : make_map(&p->ma, a.A, a.G, a.M, a.K, BM, a.a_gstride);
  if (rc) return rc;
  rc = B_MN ? make_map(&p->mb, a.B, a.G, a.K, a.N, 64, a.b_gstride) : make_map(&p->mb, a.B, a.G, a.N, a.K, BN, a.b_gstride);
  if (rc) return rc;
  int dev = 0, sms = 0;
  FEDHC_CUDA_TRY(cudaGetDevice(&dev));
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int tiles = a.G * (a.M / BM) * (a.N / BN);
  p->smem = Cfg<BM, BN>::smem_bytes();
  auto kern = grouped_gemm_kernel<BM, BN, A_MN, B_MN>;
  FEDHC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, p->smem));
  p->kern = reinterpret_cast<const void*>(kern);
  p->grid = tiles < sms ? tiles : sms;
  return FEDHC_OK;
}

template <int BM, int BN>
static int plan_major(const fedhc_gemm_args& a, GemmPlan* p) {
  if constexpr (BN >= 64) {
    if (a.a_mn && a.b_mn) return plan_kernel<BM, BN, true, true>(a, p);
    if (a.b_mn) return plan_kernel<BM, BN, false, true>(a, p);
  } else {
    if (a.b_mn) return fail(FEDHC_ERR_UNSUPPORTED, "gemm: N = 32 tiles need a K-major B operand");
  }
  if (a.a_mn) return plan_kernel<BM, BN, true, false>(a, p);
  return plan_kernel<BM, BN, false, false>(a, p);
}

template <int BM>
static int plan_n(const fedhc_gemm_args& a, GemmPlan* p) {
  if (a.N % 256 == 0) return plan_major<BM, 256>(a, p);
  if (a.N % 128 == 0) return plan_major<BM, 128>(a, p);
  if (a.N % 64 == 0) return plan_major<BM, 64>(a, p);
  return plan_major<BM, 32>(a, p);
}

int gemm_plan(const fedhc_gemm_args& a, GemmPlan* p) {
  if (a.G < 1 || a.M < 1 || a.N < 1 || a.K < 1) return fail(FEDHC_ERR_VALUE, "gemm: empty problem");
  if (a.M % 64 || a.N % 32 || a.K % BK)
    return fail(FEDHC_ERR_UNSUPPORTED, "gemm: need M % 64 == 0, N % 32 == 0, K % 64 == 0");
  if ((reinterpret_cast<uintptr_t>(a.A) | reinterpret_cast<uintptr_t>(a.B)) & 15)
    return fail(FEDHC_ERR_VALUE, "gemm: operands must be 16-byte aligned");
  Epilogue ep{a.epilogue, a.D, a.ldd > 0 ? a.ldd : a.N, 0, a.bias, a.bias_per_row, a.bias_gstride, a.master,
              static_cast<__nv_bfloat16*>(a.shadow), a.lr, static_cast<const __nv_bfloat16*>(a.mask), a.rowsum};
  ep.d_gstride = a.d_gstride > 0 ? a.d_gstride : (int64_t)a.M * ep.ldd;
  if (ep.kind < FEDHC_EPI_F32 || ep.kind > FEDHC_EPI_RELU_MASK_BF16) return fail(FEDHC_ERR_VALUE, "gemm: unknown epilogue");
  if (ep.kind == FEDHC_EPI_SGD ? !ep.master : !ep.D) return fail(FEDHC_ERR_VALUE, "gemm: missing output");
  if (ep.kind == FEDHC_EPI_BIAS_RELU_BF16 && !ep.bias) return fail(FEDHC_ERR_VALUE, "gemm: missing bias");
  if (ep.kind == FEDHC_EPI_RELU_MASK_BF16 && !ep.mask) return fail(FEDHC_ERR_VALUE, "gemm: missing mask");
  if (ep.rowsum && (ep.kind == FEDHC_EPI_F32 || ep.kind == FEDHC_EPI_SGD))
    return fail(FEDHC_ERR_VALUE, "gemm: rowsum needs a bf16 epilogue");
  if (ep.ldd % 8 || ep.d_gstride % 8) return fail(FEDHC_ERR_VALUE, "gemm: ldd and d_gstride must be multiples of 8");
  const int bn = a.N % 256 == 0 ? 256 : a.N % 128 == 0 ? 128 : a.N % 64 == 0 ? 64 : 32;
  if (ep.rowsum && bn != a.N) return fail(FEDHC_ERR_UNSUPPORTED, "gemm: rowsum needs N to fit one tile (N <= 256)");
  p->ep = ep;
  p->G = a.G;
  p->M = a.M;
  p->N = a.N;
  p->K = a.K;
  return a.M % 128 == 0 ? plan_n<128>(a, p) : plan_n<64>(a, p);
}

int gemm_run(const GemmPlan& p, cudaStream_t st) {
  void* args[] = {const_cast<CUtensorMap*>(&p.ma), const_cast<CUtensorMap*>(&p.mb), const_cast<int*>(&p.G),
                  const_cast<int*>(&p.M), const_cast<int*>(&p.N), const_cast<int*>(&p.K),
                  const_cast<Epilogue*>(&p.ep)};
  FEDHC_CUDA_TRY(cudaLaunchKernel(p.kern, dim3(p.grid), dim3(kThreads), args, p.smem, st));
  return FEDHC_OK;
}

}  // namespace tc
}  // namespace fedhc

using namespace fedhc;

extern "C" int fedhc_gemm(const fedhc_gemm_args* args, void* stream) {
  if (!args) return fail(FEDHC_ERR_VALUE, "gemm: null args");
  tc::GemmPlan p;
  int rc = tc::gemm_plan(*args, &p);
  if (rc) return rc;
  return tc::gemm_run(p, static_cast<cudaStream_t>(stream));
}

extern "C" int fedhc_gemm_bf16_tn(int G, int M, int N, int K, const void* A, const void* B, float* D, void* stream) {
  fedhc_gemm_args a{};
  a.G = G;
  a.M = M;
  a.N = N;
  a.K = K;
  a.A = A;
  a.B = B;
  a.epilogue = FEDHC_EPI_F32;
  a.D = D;
  return fedhc_gemm(&a, stream);
}
