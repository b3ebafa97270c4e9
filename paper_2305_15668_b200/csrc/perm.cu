// PCG64 batch permutations generated on the GPU (numpy-bit-exact).
//
// The batch order local_train walks (fl_core.py:181-187) is one sequential
// Fisher-Yates per client permutation; clients are independent, so the
// kernel runs one CTA per client: the permutation lives in shared memory,
// thread 0 walks the numpy random_interval / PCG64 stream (pcg64.cuh, shared
// with the host implementation), all threads initialise arange(n) and write
// the result out coalesced.  Launched on a side stream, it overlaps the
// previous round's training on the SMs the one-CTA-per-client train kernel
// leaves idle, so the host only ships 24 bytes per client (seed + sizes).
#include "common.cuh"
#include "pcg64.cuh"

namespace fedhc {

constexpr int kPermThreads = 128;

__global__ void __launch_bounds__(kPermThreads)
    perm_kernel(const uint64_t* __restrict__ seeds, const int32_t* __restrict__ n_rows,
                const int32_t* __restrict__ n_perms, const int64_t* __restrict__ offsets, int32_t* __restrict__ out,
                int smem_rows) {
  extern __shared__ int32_t a_s[];
  const int c = blockIdx.x;
  const int n = n_rows[c], k = n_perms[c];
  int32_t* dst = out + offsets[c];
  const bool in_smem = n <= smem_rows;
  fedhc_pcg::Pcg64 rng(threadIdx.x == 0 ? seeds[c] : 0ull);
  for (int p = 0; p < k; ++p) {
    int32_t* a = in_smem ? a_s : dst + (int64_t)p * n;
    for (int i = threadIdx.x; i < n; i += kPermThreads) a[i] = i;
    __syncthreads();
    if (threadIdx.x == 0) fedhc_pcg::fisher_yates(rng, a, n);
    __syncthreads();
    if (in_smem) {
      for (int i = threadIdx.x; i < n; i += kPermThreads) dst[(int64_t)p * n + i] = a[i];
      __syncthreads();
    }
  }
}

}  // namespace fedhc

using namespace fedhc;

extern "C" int fedhc_batch_permutations_device(const uint64_t* seeds, const int32_t* n_rows, const int32_t* n_perms,
                                               const int64_t* offsets, int n_clients, int32_t* out, int max_rows,
                                               void* stream) {
  if (n_clients < 0 || max_rows < 0) return fail(FEDHC_ERR_VALUE, "batch_permutations_device: negative size");
  if (n_clients == 0) return FEDHC_OK;
  int dev = 0, max_smem = 0;
  FEDHC_CUDA_TRY(cudaGetDevice(&dev));
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int smem_rows = max_rows * 4 <= max_smem ? max_rows : 0;  // larger shards permute in global memory
  const int smem = smem_rows * 4;
  static int smem_set = 48 * 1024;  // raise the opt-in only when needed (keeps launches graph-capturable)
  if (smem > smem_set) {
    FEDHC_CUDA_TRY(cudaFuncSetAttribute(perm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    smem_set = smem;
  }
  perm_kernel<<<n_clients, kPermThreads, smem, static_cast<cudaStream_t>(stream)>>>(seeds, n_rows, n_perms, offsets,
                                                                                   out, smem_rows);
  FEDHC_CUDA_TRY(cudaGetLastError());
  return FEDHC_OK;
}
