// Microbenchmark: tcgen05.mma (kind::f16, bf16 -> fp32, cta_group::1, M = 128, K = 16) issue-to-completion rate
// per SM for the operand layouts of train_c64_kernel: cycles per MMA over 512 back-to-back MMAs into one
// accumulator, smem operands only (no other traffic).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2305_15668_b200/csrc -I../../include -o umma_rate umma_rate.cu
#include <cuda_runtime.h>
#include <stdio.h>

#include "tc5.cuh"

using namespace fedhc;
using namespace fedhc::tc5;

struct Cfg { int n, a_mn, b_mn, a_lbo, b_lbo, a_step, b_step; const char* name; int nch = 1, b_base = 32768, waits = 0; };

__global__ void k_rate(Cfg c, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t sb = (smem_u32(smem_raw) + 1023) & ~1023u;
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 198 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem_raw)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); fence_mbar_init(); mbar_arrive(&bar2); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = slot;
  const uint32_t id = idesc_f16(128, c.n, c.a_mn, c.b_mn);
  if (threadIdx.x < 32) {  // whole warp, elected issue; operands walk nch chunks of distinct shared memory
    const uint64_t da = smem_desc(sb, c.a_lbo, 1024, 2), db = smem_desc(sb + c.b_base, c.b_lbo, 1024, 2);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += 4 * c.nch)
      for (int ch = 0; ch < c.nch; ++ch) {
        if (c.waits) {
          mbar_wait(&bar2, 0);
          fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_ws(tm, da + ((ch * 16384 + kk * c.a_step) >> 4), db + ((ch * 16384 + kk * c.b_step) >> 4), id, i | ch | kk);
      }
    commit_ws(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  fence_after();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int main() {
  const int iters = 480;
  Cfg cfgs[] = {
      {128, 0, 1, 16, 8192, 32, 2048, "fwd  walk 6 chunks (A 96K | B 96K)", 6, 98304},
      {128, 0, 1, 16, 8192, 32, 2048, "fwd  walk 6 chunks + mbar wait per chunk", 6, 98304, 1},
      {64, 1, 1, 16384, 8192, 2048, 2048, "bwd  walk 6 chunks", 6, 98304},
      {128, 0, 1, 16, 8192, 32, 2048, "fwd  walk 1 chunk", 1, 98304},
      {128, 0, 1, 16, 8192, 32, 2048, "fwd  A K-major SW128, B MN-major N=128"},
      {64, 0, 1, 16, 8192, 32, 2048, "fwd2 A K-major SW128, B MN-major N=64"},
      {64, 1, 1, 16384, 8192, 2048, 2048, "bwd  A MN-major SW128 (LBO 16K), B MN-major N=64"},
      {128, 1, 1, 16384, 8192, 2048, 2048, "bwd2 A MN-major SW128, B MN-major N=128"},
      {64, 0, 0, 16, 16, 32, 32, "kk   A K-major, B K-major N=64"},
      {256, 0, 1, 16, 8192, 32, 2048, "big  A K-major, B MN-major N=256"},
  };
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(k_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (const Cfg& c : cfgs) {
    k_rate<<<148, 128, 200 * 1024>>>(c, iters, d);
    k_rate<<<148, 128, 200 * 1024>>>(c, iters, d);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("%-52s: %6.1f cycles / MMA (floor %d)  err=%s\n", c.name, avg / iters, 128 * c.n / 256,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
