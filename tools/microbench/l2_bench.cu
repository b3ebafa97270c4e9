// (a) per-SM ingress from L2-resident data via 1-D bulk copies (each CTA re-reads its own 200 KB)
// (b) legacy mma.sync m16n8k16 bf16 throughput per SM
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}
constexpr int F = 784;
__global__ void __launch_bounds__(64, 1) k_rows(const float* __restrict__ x, int iters, int stages, int rows_region) {
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
  const float* X = x + (size_t)blockIdx.x * rows_region * F;
  if (warp == 0) {
    for (int it = 0; it < iters; ++it) {
      const int slot = it % stages, use = it / stages;
      if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
      if (lane == 0) mbar_expect(&full[slot], SB);
      __syncwarp();
      if (lane < 16) bulk(smem + slot * SB + lane * F * 4, X + (size_t)(((it * 16 + lane) * 37) % rows_region) * F, F * 4, &full[slot]);
      __syncwarp();
    }
  } else if (lane == 0) {
    for (int it = 0; it < iters; ++it) {
      const int slot = it % stages, use = it / stages;
      mbar_wait(&full[slot], use & 1);
      mbar_arrive(&empty[slot]);
    }
  }
}

__global__ void k_hmma(float* out, int iters) {
  uint32_t a[4] = {threadIdx.x, 2u, 3u, 4u}, b0 = 5, b1 = 6;
  float d[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  if (s == 123.f) out[0] = s;
}

int main() {
  float* x; float* o;
  const int clients = 100, region = 64;  // 64 rows = 200 KB per CTA, L2 resident
  CK(cudaMalloc(&x, (size_t)clients * region * F * 4)); CK(cudaMemset(x, 0, (size_t)clients * region * F * 4));
  CK(cudaMalloc(&o, 4));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int ncta : {100}) {
    for (int st : {2, 4}) {
      int smem = st * 16 * F * 4 + 1024 + 2 * st * 8;
      CK(cudaFuncSetAttribute(k_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      int iters = 4000;
      k_rows<<<ncta, 64, smem>>>(x, iters, st, region);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      k_rows<<<ncta, 64, smem>>>(x, iters, st, region);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      double bytes = (double)iters * 16 * F * 4;
      printf("L2 bulk rows: ctas=%3d stages=%d  %.1f GB/s per SM  %.0f GB/s total\n", ncta, st, bytes / (ms * 1e6), bytes * ncta / (ms * 1e6));
    }
  }
  for (int warps : {4, 8, 16}) {
    int iters = 20000;
    k_hmma<<<148, warps * 32>>>(o, iters);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    k_hmma<<<148, warps * 32>>>(o, iters);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double mac = (double)iters * 4 * warps * 16 * 8 * 16;
    printf("mma.sync m16n8k16 bf16: warps/SM=%2d  %.0f MAC/clk/SM (at 1.965 GHz)  %.1f TFLOP/s chip\n", warps,
           mac / (ms * 1e-3) / 1.965e9, 2 * mac * 148 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
