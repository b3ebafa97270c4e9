// Microbenchmark: per-SM ingress of gathered client rows stored PRE-SPLIT in HBM
// (row = 12 chunks x [hi 64 bf16 | mid 64 bf16] + tail [hi 16 | mid 16] = 3136 B,
// the same bytes as the fp32 row) into tcgen05 SW128 K-major tiles whose M rows
// interleave (row r hi, row r mid) -- one 4-D TMA box {64, 2, 1, 1} per (row, chunk)
// lands 256 contiguous bytes at tile offset 256 r, and the tail chunk is a SW32 tile.
//   1) checks that the hardware swizzle is a function of the shared-memory address
//      (a box landing mid-atom is swizzled by its own row index within the atom)
//   2) times 1 and 2 passes (forward + L2 re-read for the backward) per SGD step
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chunk_gather_bench chunk_gather_bench.cu
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
__device__ __forceinline__ void tma4(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
               ::"r"(dst), "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
               ::"r"(dst), "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}

constexpr int F = 784, NCH = 12, ROWS = 64, SLOT = ROWS * 256, TAIL = ROWS * 64;

// swizzle check: rows perm[0..63] of client 0, chunk ch -> slot; tail -> tail tile; dump smem
__global__ void k_check(const __grid_constant__ CUtensorMap mc, const __grid_constant__ CUtensorMap mt, const int* perm,
                        int ch, uint16_t* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(smem + SLOT + TAIL);
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (threadIdx.x == 0) mbar_expect(bar, SLOT + TAIL);
  __syncthreads();
  if (threadIdx.x < ROWS) {
    const int r = threadIdx.x;
    tma4(su32(smem + r * 256), &mc, bar, 0, 0, ch, perm[r]);
    tma3(su32(smem + SLOT + r * 64), &mt, bar, 0, 0, perm[r]);
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < (SLOT + TAIL) / 2; i += blockDim.x) out[i] = ((const uint16_t*)smem)[i];
}

template <int LANES>
__global__ void __launch_bounds__(64, 1) k_chunks(const __grid_constant__ CUtensorMap mc, const __grid_constant__ CUtensorMap mt,
                                                  const int* __restrict__ perm, int steps, int passes, int slots, int n_rows) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + slots * SLOT + TAIL);
  uint64_t* empty = full + slots;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int* P = perm + (size_t)blockIdx.x * steps * ROWS;
  const int base = blockIdx.x * n_rows;
  const int per = NCH + 1;  // 12 chunks + tail (the tail shares the slot ring)
  const int total = steps * passes * per;
  if (warp == 0) {
    for (int it = 0; it < total; ++it) {
      const int slot = it % slots, use = it / slots;
      if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
      const int s = it / (passes * per), ch = it % per;
      if (lane == 0) mbar_expect(&full[slot], ch < NCH ? SLOT : TAIL);
      __syncwarp();
      if (lane < LANES) {
        for (int r = lane; r < ROWS; r += LANES) {
          const int row = base + P[s * ROWS + r];
          if (ch < NCH) tma4(su32(smem + slot * SLOT + r * 256), &mc, &full[slot], 0, 0, ch, row);
          else tma3(su32(smem + slot * SLOT + r * 64), &mt, &full[slot], 0, 0, row);
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

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int clients = argc > 1 ? atoi(argv[1]) : 100;
  const int n_rows = 6400, steps = 100;
  void* p; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  EncFn enc = (EncFn)p;
  const size_t total_rows = (size_t)clients * n_rows;
  const size_t row_elems = F * 2;  // bf16 elements per row (hi + mid)
  std::vector<uint16_t> hx(total_rows * row_elems);
  for (size_t i = 0; i < hx.size(); ++i) hx[i] = (uint16_t)(i * 2654435761u >> 7);
  uint16_t* x; int* perm;
  CK(cudaMalloc(&x, hx.size() * 2));
  CK(cudaMemcpy(x, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
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
  CUtensorMap mc, mt;
  {
    cuuint64_t dims[4] = {64, 2, NCH, (cuuint64_t)total_rows};
    cuuint64_t str[3] = {128, 256, (cuuint64_t)row_elems * 2};
    cuuint32_t box[4] = {64, 2, 1, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&mc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode chunks failed %d\n", r); return 1; }
  }
  {
    cuuint64_t dims[3] = {16, 2, (cuuint64_t)total_rows};
    cuuint64_t str[2] = {32, (cuuint64_t)row_elems * 2};
    cuuint32_t box[3] = {16, 2, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&mt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, x + NCH * 128, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) { printf("encode tail failed %d\n", r); return 1; }
  }
  // ---- swizzle check ----
  {
    uint16_t* dout;
    CK(cudaMalloc(&dout, SLOT + TAIL));
    const int smem = SLOT + TAIL + 1024 + 64;
    CK(cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int bad = 0, checked = 0;
    for (int ch : {0, 5, 11}) {
      k_check<<<1, 128, smem>>>(mc, mt, perm, ch, dout);
      CK(cudaDeviceSynchronize());
      std::vector<uint16_t> o((SLOT + TAIL) / 2);
      CK(cudaMemcpy(o.data(), dout, SLOT + TAIL, cudaMemcpyDeviceToHost));
      for (int r = 0; r < ROWS; ++r)
        for (int pl = 0; pl < 2; ++pl) {
          const int m = 2 * r + pl;
          for (int e = 0; e < 64; ++e) {  // SW128 K-major: 16-byte unit u -> u ^ (m % 8)
            const size_t byte = (size_t)m * 128 + ((((e * 2) >> 4) ^ (m & 7)) << 4) + ((e * 2) & 15);
            const uint16_t want = hx[(size_t)hp[r] * row_elems + ch * 128 + pl * 64 + e];
            bad += o[byte / 2] != want;
            ++checked;
          }
          for (int e = 0; e < 16; ++e) {  // SW32: 16-byte unit u (0..1) -> u ^ ((m >> 2) & 1)
            const size_t byte = SLOT + (size_t)m * 32 + ((((e * 2) >> 4) ^ ((m >> 2) & 1)) << 4) + ((e * 2) & 15);
            const uint16_t want = hx[(size_t)hp[r] * row_elems + NCH * 128 + pl * 16 + e];
            bad += o[byte / 2] != want;
            ++checked;
          }
        }
    }
    printf("swizzle check: %d mismatches of %d\n", bad, checked);
  }
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
    for (int slots : {4, 6, 8, 12}) {
      int smem = slots * SLOT + TAIL + 1024 + 2 * slots * 8;
      float t1 = run(k_chunks<1>, smem, mc, mt, perm, steps, passes, slots, n_rows);
      float t8 = run(k_chunks<8>, smem, mc, mt, perm, steps, passes, slots, n_rows);
      float t32 = run(k_chunks<32>, smem, mc, mt, perm, steps, passes, slots, n_rows);
      float best = fminf(t1, fminf(t8, t32));
      printf("chunk boxes passes=%d slots=%2d : lanes1 %.3f ms  lanes8 %.3f  lanes32 %.3f  (%.0f GB/s unique, %.2f us/step)\n",
             passes, slots, t1, t8, t32, hbm_bytes / (best * 1e6), best * 1e3 / steps);
    }
  return 0;
}
