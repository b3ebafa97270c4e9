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
#include <stdlib.h>

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

// ---------------------------------------------------------------------------------------------------
// perm_fast_kernel: the same permutations without the sequential swap walk.
//
// Fisher-Yates (numpy shuffle) is: for i = n-1 .. 1: v_i = random_interval(i); swap(a[i], a[v_i]).  The
// accepted draws v_i depend only on the PCG64 stream (not on the array), and the final array follows from
// them in parallel: position i is final after step i, and receives the value that sat at position v_i just
// before step i.  A position p <= t was last written before step t by the smallest step j > t with
// v_j == p (which moved the value of position j there), else it still holds p.  With the steps grouped by
// their v (bucket p = {j : v_j = p}, ascending; every j in bucket p is >= p):
//   a[i] = v_i                               if bucket v_i has no element after i
//        = follow(next element after i)      otherwise,
//   follow(j) = j if bucket j has no element > j, else follow(that element)
// (a[0] reads bucket 0 from its start).  Chains are short (an element moves ~ln n times).
//   phase B (warp 0): the acceptance scan -- v = draw & mask accepted iff v <= i -- 32 draws per iteration:
//     a lane is surely accepted if v <= i - lane, surely rejected if v > i, else ambiguous; the lanes before
//     the first ambiguous one are resolved by a ballot, the ambiguous lane exactly, and the scan resumes
//     after it (single draws near a mask change and at the end of a draw chunk).
//   phase C (all threads): counting sort of the steps by v into buckets, per-bucket insertion sort, the
//     chain resolution above, coalesced writes.
// Shared memory: V [n] | bucket offsets [n + 1] | bucket lists [n] (+ the 8 KB draw chunk).
// ---------------------------------------------------------------------------------------------------
constexpr int kPermFastThreads = 256;

__device__ __forceinline__ void block_exclusive_scan(int32_t* a, int m, int32_t* warp_tot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kPermFastThreads / 32;
  const int per = (m + kPermFastThreads - 1) / kPermFastThreads;
  const int lo = min(m, tid * per), hi = min(m, lo + per);
  int sum = 0;
  for (int q = lo; q < hi; ++q) sum += a[q];
  int incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < NW ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    if (lane < NW) warp_tot[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int run = incl - sum + (warp ? warp_tot[warp - 1] : 0);
  for (int q = lo; q < hi; ++q) {
    const int v = a[q];
    a[q] = run;
    run += v;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kPermFastThreads)
    perm_fast_kernel(const uint64_t* __restrict__ seeds, const int32_t* __restrict__ n_rows,
                     const int32_t* __restrict__ n_perms, const int64_t* __restrict__ offsets,
                     int32_t* __restrict__ out, int cap_rows, PcgJump jump) {
  extern __shared__ int32_t sm[];
  __shared__ uint32_t draws[kDrawChunk];
  __shared__ int32_t warp_tot[kPermFastThreads / 32];
  const int c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = n_rows[c], k = n_perms[c];
  if (n <= 0) return;  // uniform per CTA
  int32_t* dst = out + offsets[c];
  int32_t* V = sm;           // V[i] = accepted v of step i (V[0] = 0)
  int32_t* bo = sm + n;      // bucket offsets
  int32_t* lst = bo + n + 1; // bucket lists
  uint64_t lo = 0, hi = 0, clo = 0, chi = 0;
  int pos = 0;
  if (warp == 0) {
    fedhc_pcg::Pcg64 rng(seeds[c]);
    for (int q = 0; q <= lane; ++q) rng.step();
    lo = static_cast<uint64_t>(rng.state);
    hi = static_cast<uint64_t>(rng.state >> 64);
    mul128(static_cast<uint64_t>(rng.inc), static_cast<uint64_t>(rng.inc >> 64), jump.s_lo, jump.s_hi, clo, chi);
  }
  auto refill = [&]() {  // warp 0: the next kDrawChunk draws (stream order)
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
    __syncwarp();
  };
  if (warp == 0) refill();
  if (n > cap_rows) {  // larger than the caller's max_rows: the sequential walk in global memory
    for (int p = 0; p < k; ++p) {
      int32_t* a = dst + (int64_t)p * n;
      for (int i = tid; i < n; i += kPermFastThreads) a[i] = i;
      __syncthreads();
      if (warp == 0) {
        int i = n - 1;
        uint32_t mask = static_cast<uint32_t>(n > 1 ? n - 1 : 0);
        mask |= mask >> 1;
        mask |= mask >> 2;
        mask |= mask >> 4;
        mask |= mask >> 8;
        mask |= mask >> 16;
        while (i >= 1) {
          if (pos == kDrawChunk) {
            refill();
            pos = 0;
          }
          if (lane == 0) fy_walk(a, draws, i, pos, mask);
          i = __shfl_sync(0xffffffffu, i, 0);
          pos = __shfl_sync(0xffffffffu, pos, 0);
          mask = __shfl_sync(0xffffffffu, mask, 0);
        }
      }
      __syncthreads();
    }
    return;
  }
  for (int p = 0; p < k; ++p) {
    // ---- phase B: accepted draws (warp 0) ----
    if (warp == 0) {
      int i = n - 1;
      uint32_t mask = static_cast<uint32_t>(n > 1 ? n - 1 : 0);
      mask |= mask >> 1;
      mask |= mask >> 2;
      mask |= mask >> 4;
      mask |= mask >> 8;
      mask |= mask >> 16;
      if (lane == 0) V[0] = 0;
      while (i >= 1) {
        if (pos == kDrawChunk) {
          refill();
          pos = 0;
        }
        // batch width: every lane's step index stays above mask >> 1 even if all lanes accept (no mask change
        // inside a batch); near a mask change the batches narrow instead of falling back to single draws
        const int wid = min(min(32, i - static_cast<int>(mask >> 1)), kDrawChunk - pos);
        if (wid >= 2) {
          const int d = lane < wid ? static_cast<int>(draws[pos + lane] & mask) : 0x7fffffff;
          const bool sure = d <= i - lane;
          const uint32_t bamb = __ballot_sync(0xffffffffu, !sure && d <= i);
          uint32_t bacc = __ballot_sync(0xffffffffu, sure);
          int consumed = wid;
          if (bamb) {
            const int L = __ffs(bamb) - 1;
            bacc &= (1u << L) - 1u;
            const int dl = __shfl_sync(0xffffffffu, d, L);
            if (dl <= i - __popc(bacc)) bacc |= 1u << L;
            consumed = L + 1;
          }
          if ((bacc >> lane) & 1u) V[i - __popc(bacc & ((1u << lane) - 1u))] = d;
          i -= __popc(bacc);
          pos += consumed;
          if ((mask >> 1) >= static_cast<uint32_t>(i)) mask >>= 1;  // the last acceptance may reach mask >> 1
        } else {
          const int d = static_cast<int>(draws[pos] & mask);
          ++pos;
          if (d <= i) {
            if (lane == 0) V[i] = d;
            --i;
            if ((mask >> 1) >= static_cast<uint32_t>(i)) mask >>= 1;
          }
        }
      }
    }
    __syncthreads();
    // ---- phase C: buckets of steps by v, then the chain resolution ----
    for (int v = tid; v <= n; v += kPermFastThreads) bo[v] = 0;
    __syncthreads();
    for (int j = 1 + tid; j < n; j += kPermFastThreads) atomicAdd(&bo[V[j]], 1);
    __syncthreads();
    block_exclusive_scan(bo, n + 1, warp_tot);
    for (int j = 1 + tid; j < n; j += kPermFastThreads) lst[atomicAdd(&bo[V[j]], 1)] = j;
    __syncthreads();  // bucket v = [v ? bo[v - 1] : 0, bo[v])
    for (int v = tid; v < n; v += kPermFastThreads) {
      const int b = v ? bo[v - 1] : 0, e = bo[v];
      for (int q = b + 1; q < e; ++q) {  // insertion sort (buckets hold ~1 element)
        const int x = lst[q];
        int r = q - 1;
        while (r >= b && lst[r] > x) {
          lst[r + 1] = lst[r];
          --r;
        }
        lst[r + 1] = x;
      }
    }
    __syncthreads();
    for (int i = tid; i < n; i += kPermFastThreads) {
      const int v = V[i];
      const int b = v ? bo[v - 1] : 0, e = bo[v];
      int nxt = -1;
      if (i == 0) {
        if (b < e) nxt = lst[b];
      } else {
        for (int q = b; q < e; ++q)
          if (lst[q] == i) {
            if (q + 1 < e) nxt = lst[q + 1];
            break;
          }
      }
      int res = v;
      if (nxt >= 0) {
        int j = nxt;
        while (true) {
          const int bb = bo[j - 1], ee = bo[j];  // j >= 1
          int f = -1;
          if (bb < ee) f = lst[bb] > j ? lst[bb] : (bb + 1 < ee ? lst[bb + 1] : -1);
          if (f < 0) break;
          j = f;
        }
        res = j;
      }
      dst[(int64_t)p * n + i] = res;
    }
    __syncthreads();
  }
}

size_t perm_fast_smem(int max_rows) { return (size_t)(3 * max_rows + 1) * 4; }

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
  static const bool legacy = getenv("FEDHC_PERM_LEGACY") != nullptr;
  const size_t fast_smem = perm_fast_smem(max_rows);  // clients with more rows walk in global memory
  if (!legacy && fast_smem + sizeof(uint32_t) * kDrawChunk + 256 <= (size_t)max_smem) {
    if (fast_smem > 48 * 1024) FEDHC_CUDA_TRY(smem_optin_max(reinterpret_cast<const void*>(perm_fast_kernel)));
    perm_fast_kernel<<<n_clients, kPermFastThreads, fast_smem, static_cast<cudaStream_t>(stream)>>>(
        seeds, n_rows, n_perms, offsets, out, max_rows, jump);
    FEDHC_CUDA_TRY(cudaGetLastError());
    return FEDHC_OK;
  }
  perm_kernel<<<n_clients, kPermThreads, smem, static_cast<cudaStream_t>(stream)>>>(seeds, n_rows, n_perms, offsets,
                                                                                   out, smem_rows, jump);
  FEDHC_CUDA_TRY(cudaGetLastError());
  return FEDHC_OK;
}
