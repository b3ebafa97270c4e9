// Microbenchmark: per-SM ingress of gathered client rows on B200.
//   mode 0: TMA tile::gather4 of pre-split bf16 hi/mid rows into SW128 tiles
//           (13 chunks of 64 features x 64 rows per step), PASSES = 1 or 2
//   mode 1: 1-D bulk copies of whole fp32 rows (3136 B) into 16-row stages
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g4(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int c0, int r0, int r1, int r2, int r3) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
               ::"r"(dst), "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

constexpr int SLOT = 16384, NCH = 13, ROWS = 64, F = 784;

template <int LANES>
__global__ void __launch_bounds__(64, 1) k_gather(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mm,
                                                  const int* __restrict__ perm, int steps, int passes, int slots, int n_rows) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + slots * SLOT);
  uint64_t* empty = full + slots;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int* P = perm + (size_t)blockIdx.x * steps * ROWS;
  const int base = blockIdx.x * n_rows;
  const int total = steps * passes * NCH;
  if (warp == 0) {
    for (int it = 0; it < total; ++it) {
      const int slot = it % slots, use = it / slots;
      if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
      const int s = it / (passes * NCH), ch = it % NCH;
      if (lane == 0) mbar_expect(&full[slot], SLOT);
      __syncwarp();
      if (lane < LANES) {
        for (int j = lane; j < 32; j += LANES) {
          const int half = j / 16, g = j % 16;  // hi / mid, 4-row group
          const int* r = P + s * ROWS + g * 4;
          const uint32_t dst = su32(smem + slot * SLOT + half * 8192 + g * 512);
          g4(dst, half ? &mm : &mh, &full[slot], ch * 64, base + r[0], base + r[1], base + r[2], base + r[3]);
        }
      }
      __syncwarp();
    }
  } else if (lane == 0) {
    for (int it = 0; it < total; ++it) {
      const int slot = it % slots, use = it / slots;
      mbar_wait(&full[slot], use & 1);
      mbar_arrive(&empty[slot]);
    }
  }
}

__global__ void __launch_bounds__(64, 1) k_rows(const float* __restrict__ x, const int* __restrict__ perm, int steps, int stages, int n_rows) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int SB = 16 * F * 4;
  uint64_t* full = (uint64_t*)(smem + stages * SB);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int* P = perm + (size_t)blockIdx.x * steps * ROWS;
  const float* X = x + (size_t)blockIdx.x * n_rows * F;
  const int total = steps * 4;
  if (warp == 0) {
    for (int it = 0; it < total; ++it) {
      const int slot = it % stages, use = it / stages;
      if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
      if (lane == 0) mbar_expect(&full[slot], SB);
      __syncwarp();
      if (lane < 16) bulk(smem + slot * SB + lane * F * 4, X + (size_t)P[it * 16 + lane] * F, F * 4, &full[slot]);
      __syncwarp();
    }
  } else if (lane == 0) {
    for (int it = 0; it < total; ++it) {
      const int slot = it % stages, use = it / stages;
      mbar_wait(&full[slot], use & 1);
      mbar_arrive(&empty[slot]);
    }
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int clients = argc > 1 ? atoi(argv[1]) : 100;
  const int n_rows = 6400, steps = 100;
  void* p; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  EncFn enc = (EncFn)p;
  size_t n = (size_t)clients * n_rows * F;
  uint16_t *xh, *xm; float* xf; int* perm;
  CK(cudaMalloc(&xh, n * 2)); CK(cudaMalloc(&xm, n * 2)); CK(cudaMalloc(&xf, n * 4));
  CK(cudaMemset(xh, 0, n * 2)); CK(cudaMemset(xm, 0, n * 2)); CK(cudaMemset(xf, 0, n * 4));
  std::vector<int> hp((size_t)clients * steps * ROWS);
  srand(1);
  for (int c = 0; c < clients; ++c) {
    std::vector<int> pr(n_rows);
    for (int i = 0; i < n_rows; ++i) pr[i] = i;
    for (int i = n_rows - 1; i > 0; --i) { int j = rand() % (i + 1); int t = pr[i]; pr[i] = pr[j]; pr[j] = t; }
    for (int i = 0; i < steps * ROWS; ++i) hp[(size_t)c * steps * ROWS + i] = pr[i];
  }
  CK(cudaMalloc(&perm, hp.size() * 4));
  CK(cudaMemcpy(perm, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice));
  CUtensorMap mh, mm;
  cuuint64_t dims[2] = {(cuuint64_t)F, (cuuint64_t)clients * n_rows};
  cuuint64_t str[1] = {(cuuint64_t)F * 2};
  cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  CUresult r1 = enc(&mh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xh, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&mm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, xm, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r1 || r2) { printf("encode failed %d %d\n", r1, r2); return 1; }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int smem, auto... args) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int w = 0; w < 2; ++w) kern<<<clients, 64, smem>>>(args...);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int w = 0; w < 5; ++w) kern<<<clients, 64, smem>>>(args...);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
  };
  const double hbm_bytes = (double)clients * steps * ROWS * F * 4;
  for (int passes = 1; passes <= 2; ++passes)
    for (int slots : {4, 8, 12}) {
      int smem = slots * SLOT + 1024 + 2 * slots * 8;
      float t1 = run(k_gather<1>, smem, mh, mm, perm, steps, passes, slots, n_rows);
      float t4 = run(k_gather<4>, smem, mh, mm, perm, steps, passes, slots, n_rows);
      float t32 = run(k_gather<32>, smem, mh, mm, perm, steps, passes, slots, n_rows);
      printf("gather4 passes=%d slots=%2d : lanes1 %.3f ms  lanes4 %.3f ms  lanes32 %.3f ms  (%.0f GB/s unique @best, %.2f us/step)\n",
             passes, slots, t1, t4, t32, hbm_bytes / (fminf(t1, fminf(t4, t32)) * 1e6), fminf(t1, fminf(t4, t32)) * 1e3 / steps);
    }
  for (int st : {2, 3, 4}) {
    int smem = st * 16 * F * 4 + 1024 + 2 * st * 8;
    float t = run(k_rows, smem, (const float*)xf, (const int*)perm, steps, st, n_rows);
    printf("bulk rows stages=%d : %.3f ms (%.0f GB/s, %.2f us/step)\n", st, t, hbm_bytes / (t * 1e6), t * 1e3 / steps);
  }
  return 0;
}
