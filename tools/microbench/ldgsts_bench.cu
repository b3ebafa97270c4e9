// Microbenchmark: per-SM ingress of gathered split rows by 16-byte LDGSTS (cp.async.cg) into SW128 chunk
// tiles, the train_c64_kernel loader pattern: W warps, warp w loads chunks j = w, w + W, ... of a 64-row step
// (chunk = 64 rows x 8 units x 2 planes x 16 B = 16 KB), wait_group 0 per chunk.  Rows gathered from a
// 2 GB array (HBM) or a 16 MB one (L2-resident).  Prints us per 7-chunk step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ldgsts_bench ldgsts_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int F = 784, NCH = 7, ROWS = 64;

__global__ void k_ldgsts(const char* __restrict__ x, const int* __restrict__ perm, int steps, int nwarps, int n_rows,
                         int prefetch, int mode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = lane & 7, p = (lane >> 3) & 1, r0 = lane >> 4;
  const int* P = perm + (size_t)blockIdx.x * steps * ROWS;
  const char* xs = x + p * 16 + u * 32;
  for (int s = 0; s < steps; ++s) {
    if (prefetch && warp == 0 && s + 1 < steps)
      for (int r = lane; r < ROWS; r += 32)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x + (size_t)P[(s + 1) * ROWS + r] * F * 4),
                     "r"(F * 2) : "memory");
    int idx[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) idx[i] = P[s * ROWS + r0 + 2 * i];
    if (mode == 1) {  // lane = 16-byte unit of one row: 512 B (two chunks) per instruction
      for (int jj = warp; jj < (NCH + 1) / 2; jj += nwarps) {
        const int j = 2 * jj + (lane >> 4), uu = lane & 7, pp = (lane >> 3) & 1;
        for (int row = 0; row < ROWS && j < NCH; ++row) {
          const int ix = P[s * ROWS + row];
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sb + j * 16384 + pp * 8192 + row * 128 + ((uu ^ (row & 7)) << 4)),
                       "l"(x + (size_t)ix * F * 4 + j * 256 + uu * 32 + pp * 16) : "memory");
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      continue;
    }
    if (mode == 2) {  // LDG.128 into registers (8 rows in flight per lane), then STS.128
      for (int j = warp; j < NCH; j += nwarps) {
        const uint32_t dst = sb + j * 16384 + p * 8192;
        for (int i0 = 0; i0 < 32; i0 += 8) {
          uint4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) v[k] = __ldcg(reinterpret_cast<const uint4*>(xs + (size_t)idx[i0 + k] * F * 4 + j * 256));
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int row = r0 + 2 * (i0 + k);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + row * 128 + ((u ^ (row & 7)) << 4)), "r"(v[k].x), "r"(v[k].y), "r"(v[k].z), "r"(v[k].w) : "memory");
          }
        }
      }
      __syncthreads();
      continue;
    }
    for (int j = warp; j < NCH; j += nwarps) {
      const uint32_t dst = sb + j * 16384 + p * 8192;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int row = r0 + 2 * i;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + row * 128 + ((u ^ (row & 7)) << 4)),
                     "l"(xs + (size_t)idx[i] * F * 4 + j * 256) : "memory");
      }
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
  }
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 148;
  const int steps = 100;
  for (size_t rows_total : {(size_t)100 * 6400, (size_t)5000}) {
    char* x;
    CK(cudaMalloc(&x, rows_total * F * 4));
    CK(cudaMemset(x, 1, rows_total * F * 4));
    std::vector<int> hp((size_t)ctas * steps * ROWS);
    srand(1);
    for (auto& v : hp) v = rand() % rows_total;
    int* perm;
    CK(cudaMalloc(&perm, hp.size() * 4));
    CK(cudaMemcpy(perm, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, NCH * 16384));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode : {0, 1, 2})
    for (int pf : {0})
      for (int nw : {4, 7, 14}) {
        k_ldgsts<<<ctas, 32 * nw, NCH * 16384>>>(x, perm, steps, nw, rows_total, pf, mode);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        k_ldgsts<<<ctas, 32 * nw, NCH * 16384>>>(x, perm, steps, nw, rows_total, pf, mode);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%s mode=%d ctas=%d warps=%d prefetch=%d: %.2f us/step (%.0f GB/s per SM)\n",
               rows_total > 100000 ? "HBM" : "L2 ", mode, ctas, nw, pf, ms * 1e3 / steps,
               NCH * 16384.0 * steps / (ms * 1e6));
      }
    cudaFree(x);
    cudaFree(perm);
  }
  return 0;
}
