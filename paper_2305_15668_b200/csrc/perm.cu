// PCG64 batch permutations generated on the GPU (numpy-bit-exact).
//
// The batch order local_train walks (fl_core.py:181-187) is one sequential
// Fisher-Yates per client permutation; clients are independent, so the
// kernel runs one CTA per client: the permutation lives in shared memory,
// warp 0 generates the PCG64 stream in parallel (jump-ahead), thread 0 walks
// numpy's random_interval rejection + swaps over it, all threads initialise
// arange(n) and write the result out coalesced.  Launched on a side stream, it overlaps the
// previous round's training on the SMs the one-CTA-per-client train kernel
// leaves idle, so the host only ships 24 bytes per client (seed + sizes).
#include "common.cuh"
#include "pcg64.cuh"

namespace fedhc {

constexpr int kPermThreads = 128;
constexpr int kDrawChunk = 2048;  // 32-bit draws generated per refill (1024 PCG64 outputs)

// PCG64 jump-ahead: s_{j+32} = A32 s_j + inc * S32 (mod 2^128), A32 = mult^32, S32 = sum_{i<32} mult^i
struct PcgJump {
  uint64_t a_lo, a_hi, s_lo, s_hi;
};

__device__ __forceinline__ void mul128(uint64_t alo, uint64_t ahi, uint64_t blo, uint64_t bhi, uint64_t& lo,
                                       uint64_t& hi) {
  lo = alo * blo;
  hi = __umul64hi(alo, blo) + alo * bhi + ahi * blo;
}

// Consume draws from the chunk until it runs out or the permutation is complete.  The next draw is read
// ahead of the swap so the only dependent chain per step is draw -> index -> a[v] -> stores.
template <class Arr>
__device__ __forceinline__ void fy_walk(Arr a, const uint32_t* draws, int& s_i, int& s_pos, uint32_t& s_mask) {
  int i = s_i, pos = s_pos;
  uint32_t mask = s_mask;
  uint32_t next = draws[pos];
  while (i >= 1 && pos < kDrawChunk) {
    const uint32_t v = next & mask;
    ++pos;
    next = draws[pos & (kDrawChunk - 1)];
    if (v <= static_cast<uint32_t>(i)) {
      const int32_t t = a[i], u = a[v];
      a[v] = t;
      a[i] = u;
      --i;
      if ((mask >> 1) >= static_cast<uint32_t>(i)) mask >>= 1;  // i drops by one: at most one halving
    }
  }
  s_i = i;
  s_pos = pos;
  s_mask = mask;
}

// One CTA per client.  numpy's permutation is a sequential Fisher-Yates walk over the client's PCG64 stream
// (pcg64.cuh); the stream itself is not sequential work: warp 0 generates it 32 outputs at a time with a
// jump-ahead LCG (lane L owns outputs L, L + 32, ...) into a shared-memory chunk, and thread 0 only walks
// the chunk (mask, reject, swap in shared memory) -- the 128-bit multiply chain leaves the critical path.
// The 32-bit draws are the low then high halves of each 64-bit output (numpy's next_uint32 buffering);
// the stream continues across a client's successive permutations.
__global__ void __launch_bounds__(kPermThreads)
    perm_kernel(const uint64_t* __restrict__ seeds, const int32_t* __restrict__ n_rows,
                const int32_t* __restrict__ n_perms, const int64_t* __restrict__ offsets, int32_t* __restrict__ out,
                int smem_rows, PcgJump jump) {
  extern __shared__ int32_t a_s[];
  __shared__ uint32_t draws[kDrawChunk];
  __shared__ int s_pos, s_i;
  __shared__ uint32_t s_mask;
  const int c = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = n_rows[c], k = n_perms[c];
  int32_t* dst = out + offsets[c];
  const bool in_smem = n <= smem_rows;
  // producer lane state: s_{L+1} (the state whose output is out64[L]), then +32 per chunk column
  uint64_t lo = 0, hi = 0, clo = 0, chi = 0;
  if (warp == 0) {
    fedhc_pcg::Pcg64 rng(seeds[c]);
    for (int q = 0; q <= lane; ++q) rng.step();
    lo = static_cast<uint64_t>(rng.state);
    hi = static_cast<uint64_t>(rng.state >> 64);
    mul128(static_cast<uint64_t>(rng.inc), static_cast<uint64_t>(rng.inc >> 64), jump.s_lo, jump.s_hi, clo, chi);
  }
  auto refill = [&]() {  // warp 0: the next kDrawChunk draws
    if (warp != 0) return;
#pragma unroll 4
    for (int t = 0; t < kDrawChunk / 64; ++t) {
      const uint64_t x = hi ^ lo;
      const unsigned rot = static_cast<unsigned>(hi >> 58);
      const uint64_t o = (x >> rot) | (x << ((64 - rot) & 63));
      draws[(t * 32 + lane) * 2] = static_cast<uint32_t>(o);
      draws[(t * 32 + lane) * 2 + 1] = static_cast<uint32_t>(o >> 32);
      uint64_t nlo, nhi;
      mul128(lo, hi, jump.a_lo, jump.a_hi, nlo, nhi);
      lo = nlo + clo;
      hi = nhi + chi + (lo < nlo ? 1ull : 0ull);
    }
  };
  refill();
  if (threadIdx.x == 0) s_pos = 0;
  for (int p = 0; p < k; ++p) {
    int32_t* a = in_smem ? a_s : dst + (int64_t)p * n;
    for (int i = threadIdx.x; i < n; i += kPermThreads) a[i] = i;
    if (threadIdx.x == 0) {
      uint32_t mask = static_cast<uint32_t>(n > 1 ? n - 1 : 0);
      mask |= mask >> 1;
      mask |= mask >> 2;
      mask |= mask >> 4;
      mask |= mask >> 8;
      mask |= mask >> 16;
      s_mask = mask;
      s_i = n - 1;
    }
    __syncthreads();
    while (true) {
      if (threadIdx.x == 0) {  // walk the chunk: a = arange(n); for i = n-1..1: j = random_interval(i); swap
        if (in_smem)
          fy_walk(a_s, draws, s_i, s_pos, s_mask);  // shared-memory array: the compiler sees two arrays
        else
          fy_walk(a, draws, s_i, s_pos, s_mask);
      }
      __syncthreads();
      const bool done = s_i < 1;
      if (s_pos == kDrawChunk) {  // chunk used up (perm finished or not): generate the next one
        __syncthreads();
        refill();
        if (threadIdx.x == 0) s_pos = 0;
        __syncthreads();
      }
      if (done) break;
    }
    if (in_smem) {
      for (int i = threadIdx.x; i < n; i += kPermThreads) dst[(int64_t)p * n + i] = a[i];
    }
    __syncthreads();
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
  // the kernel also holds 8 KB of draws in static shared memory; larger shards permute in global memory
  const int smem_rows = max_rows * 4 + (int)sizeof(uint32_t) * kDrawChunk + 256 <= max_smem ? max_rows : 0;
  const int smem = smem_rows * 4;
  // shared-memory opt-in: once per device, to the maximum (thread-safe: the runner launches from two threads)
  if (smem > 48 * 1024) FEDHC_CUDA_TRY(smem_optin_max(reinterpret_cast<const void*>(perm_kernel)));
  static const PcgJump jump = [] {
    using fedhc_pcg::u128;
    const u128 m = FEDHC_PCG_MULT;
    u128 a = 1, sum = 0;
    for (int i = 0; i < 32; ++i) {
      sum += a;
      a *= m;
    }
    return PcgJump{static_cast<uint64_t>(a), static_cast<uint64_t>(a >> 64), static_cast<uint64_t>(sum),
                   static_cast<uint64_t>(sum >> 64)};
  }();
  perm_kernel<<<n_clients, kPermThreads, smem, static_cast<cudaStream_t>(stream)>>>(seeds, n_rows, n_perms, offsets,
                                                                                   out, smem_rows, jump);
  FEDHC_CUDA_TRY(cudaGetLastError());
  return FEDHC_OK;
}
