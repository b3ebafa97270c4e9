// Microbenchmark: the train_c64_kernel re-layout (staged rows, 1536-byte pitch -> swizzled SW128 chunk tiles),
// 6 warps x 16 KB per SM, with and without 10 warps polling an mbarrier.  Measured: ~2200 cycles per 16 KB
// per warp either way (~87 B/cycle of shared-memory traffic): bandwidth, not polling, bounds it.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o relayout_bench relayout_bench.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int iters, unsigned long long* out, int spin) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  const uint32_t sb = su32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  __syncthreads();
  if (warp >= 6) {  // "spinning" warps: poll an mbarrier that never completes until the end
    if (spin) {
      uint32_t ok = 0;
      while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
      }
    }
    return;
  }
  const int j = warp, u = lane & 7, p = (lane >> 3) & 1, r0 = lane >> 4;
  const uint32_t spitch = 1536, sbase = sb + 102400 + (8 * j + u) * 32 + p * 16, dst = sb + j * 16384 + p * 8192;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      uint4 v[8];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int row = r0 + 2 * (8 * b + kk);
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v[kk].x), "=r"(v[kk].y), "=r"(v[kk].z), "=r"(v[kk].w) : "r"(sbase + row * spitch));
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int row = r0 + 2 * (8 * b + kk);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + row * 128 + ((u ^ (row & 7)) << 4)), "r"(v[kk].x), "r"(v[kk].y), "r"(v[kk].z), "r"(v[kk].w) : "memory");
      }
    }
  }
  unsigned long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 6 + warp] = (t1 - t0) / iters;
  __syncwarp();
  if (warp == 0 && lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar)) : "memory");
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 148 * 6 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int spin : {0, 1}) {
    k<<<148, 512, 200 * 1024>>>(100, d, spin);
    unsigned long long h[148 * 6]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double a = 0; for (int i = 0; i < 148 * 6; ++i) a += h[i];
    printf("spin=%d relayout of 16 KB per warp (6 warps): %.0f cycles  err=%s\n", spin, a / (148 * 6), cudaGetErrorString(cudaGetLastError()));
  }
}
