// numpy Generator.standard_normal (float64) on the GPU, value-for-value: the reference's synthetic features
// (fl_core.py:47-55: means[labels] + rng.standard_normal((n_total, n_features))) at fleet scale.
//
// numpy draws one next_uint64 per ziggurat attempt (distributions.c random_standard_normal): idx = r & 0xff,
// sign = bit 8, rabs = bits 9..60, x = rabs * wi[idx], accepted at once when rabs < ki[idx] (99 %); otherwise the
// wedge test (idx > 0: one next_double, may reject and restart) or the tail loop (idx = 0: pairs of next_double).
// So the k-th normal sits at a data-dependent position of the PCG64 stream.  Three passes over the stream:
//   1. runs of kRun positions, one thread each: walk the attempt chain from entry offsets 0..kE-1 (entries that
//      fall on the offset-0 chain share its result), recording per entry the exit offset into the next run and
//      the number of accepted attempts;
//   2. host: chain the runs (run k's entry = run k-1's exit), giving each run its entry offset and the index of
//      its first normal (a rare exit >= kE is resolved by simulating that run);
//   3. runs again, from their true entries, writing the accepted values in place.
// Tables: tools/gen/numpy_ziggurat_tables.py (extracted from numpy by driving its PCG64).  Arithmetic is spelled
// out with round-to-nearest intrinsics so nvcc cannot contract it differently from numpy's (FMA-free) build.  The
// tail uses log1p exactly as the image's glibc computes it (glibc_log1p below), so tail values match bit for bit;
// the wedge test calls CUDA's exp where numpy calls libm's, so a wedge decision could flip only when the two sides
// meet within an ulp (probability ~1e-16 per wedge test).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "common.cuh"
#include "pcg64.cuh"
#include "ziggurat_tables.h"
#include "log1p_glibc.cuh"

namespace fedhc {
namespace zig {

using fedhc_pcg::u128;
constexpr double kR = 3.6541528853610087963519472518;       // ziggurat_nor_r
constexpr double kInvR = 0.27366123732975827203338247596;   // ziggurat_nor_inv_r
constexpr int kRun = 1024;                                   // stream positions per run
constexpr int kE = 16;                                       // precomputed entry offsets per run
constexpr int kThreads = 128;
constexpr uint64_t kMask52 = 0x000fffffffffffffull;

struct Tables {
  double wi[256], fi[256];
  uint64_t ki[256];
};

__device__ __forceinline__ void load_tables(Tables& t) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    t.wi[i] = wi[i];
    t.fi[i] = fi[i];
    t.ki[i] = ki[i];
  }
  __syncthreads();
}

// PCG64 positioned so that its next next64() returns the draw at stream position p.
struct Gen {
  u128 state, inc;
  __host__ __device__ uint64_t next64() {
    state = state * FEDHC_PCG_MULT + inc;
    const uint64_t x = static_cast<uint64_t>(state >> 64) ^ static_cast<uint64_t>(state);
    const unsigned rot = static_cast<unsigned>(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  __host__ __device__ double next_double() { return static_cast<double>(next64() >> 11) * (1.0 / 9007199254740992.0); }
};

// pcg_advance_lcg_128: the state `delta` steps later.
__host__ __device__ inline u128 advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = FEDHC_PCG_MULT, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// One ziggurat attempt whose first draw is r; g yields the draws after it.  Returns the draws consumed.
template <class T>
__host__ __device__ inline int attempt(const T& t, uint64_t r, Gen& g, bool& acc, double& val) {
  const int idx = static_cast<int>(r & 0xff);
  r >>= 8;
  const int sign = static_cast<int>(r & 1);
  const uint64_t rabs = (r >> 1) & kMask52;
  double x = mul_rn(static_cast<double>(rabs), t.wi[idx]);
  if (sign) x = -x;
  if (rabs < t.ki[idx]) {
    acc = true;
    val = x;
    return 1;
  }
  if (idx == 0) {
    int c = 1;
    for (;;) {
      const double xx = mul_rn(-kInvR, glibc_log1p(-g.next_double()));
      const double yy = -glibc_log1p(-g.next_double());
      c += 2;
      if (add_rn(yy, yy) > mul_rn(xx, xx)) {
        acc = true;
        val = ((rabs >> 8) & 1) ? -add_rn(kR, xx) : add_rn(kR, xx);
        return c;
      }
    }
  }
  acc = add_rn(mul_rn(sub_rn(t.fi[idx - 1], t.fi[idx]), g.next_double()), t.fi[idx]) < exp(mul_rn(mul_rn(-0.5, x), x));
  val = x;
  return 2;
}

// Walk run-relative positions [e, kRun) from entry e: accepted attempts and the exit offset into the next run.
template <class T>
__host__ __device__ inline void walk(const T& t, u128 s0, u128 inc, int64_t p0, int e, int& count, int& exit) {
  Gen g{advance(s0, inc, static_cast<uint64_t>(p0 + e)), inc};
  int q = e, cnt = 0;
  while (q < kRun) {
    bool acc;
    double v;
    q += attempt(t, g.next64(), g, acc, v);
    cnt += acc ? 1 : 0;
  }
  count = cnt;
  exit = q - kRun;
}

__global__ void __launch_bounds__(kThreads) runs_kernel(u128 s0, u128 inc, int64_t n_runs, int16_t* exit_tab,
                                                       int16_t* count_tab) {
  __shared__ Tables t;
  __shared__ uint32_t starts[kRun / 32][kThreads];  // offset-0 chain: attempt starts (thread-major: no conflicts)
  __shared__ uint32_t accs[kRun / 32][kThreads];    // ... and the accepted ones
  load_tables(t);
  const int64_t k = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (k >= n_runs) return;
  auto st = [&](int w) -> uint32_t& { return starts[w][threadIdx.x]; };
  auto ac = [&](int w) -> uint32_t& { return accs[w][threadIdx.x]; };
  for (int i = 0; i < kRun / 32; ++i) st(i) = ac(i) = 0;
  const int64_t p0 = k * kRun;
  Gen g{advance(s0, inc, static_cast<uint64_t>(p0)), inc};
  int q = 0, cnt = 0;
  while (q < kRun) {
    bool acc;
    double v;
    const int c = attempt(t, g.next64(), g, acc, v);
    st(q >> 5) |= 1u << (q & 31);
    if (acc) {
      ac(q >> 5) |= 1u << (q & 31);
      ++cnt;
    }
    q += c;
  }
  const int exit0 = q - kRun;
  int16_t* ex = exit_tab + k * kE;
  int16_t* co = count_tab + k * kE;
  ex[0] = static_cast<int16_t>(exit0);
  co[0] = static_cast<int16_t>(cnt);
  int before = 0;  // accepted attempts of the offset-0 chain before offset e
  for (int e = 1; e < kE; ++e) {
    before += (ac((e - 1) >> 5) >> ((e - 1) & 31)) & 1;
    if ((st(e >> 5) >> (e & 31)) & 1) {  // e is on the offset-0 chain: same suffix
      ex[e] = static_cast<int16_t>(exit0);
      co[e] = static_cast<int16_t>(cnt - before);
    } else {  // inside an earlier attempt's extra draws: walk until the chains meet
      Gen h{advance(s0, inc, static_cast<uint64_t>(p0 + e)), inc};
      int qe = e, ce = 0;
      while (qe < kRun && !((st(qe >> 5) >> (qe & 31)) & 1)) {
        bool acc;
        double v;
        qe += attempt(t, h.next64(), h, acc, v);
        ce += acc ? 1 : 0;
      }
      if (qe < kRun) {
        int b = 0;  // accepted attempts of the offset-0 chain before qe
        for (int i = 0; i < (qe >> 5); ++i) b += __popc(ac(i));
        b += __popc(ac(qe >> 5) & ((1u << (qe & 31)) - 1u));
        ex[e] = static_cast<int16_t>(exit0);
        co[e] = static_cast<int16_t>(ce + cnt - b);
      } else {
        ex[e] = static_cast<int16_t>(qe - kRun);
        co[e] = static_cast<int16_t>(ce);
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads) emit_kernel(u128 s0, u128 inc, int64_t n_runs, const int16_t* entry,
                                                       const int64_t* first, int64_t n, double* out) {
  __shared__ Tables t;
  load_tables(t);
  const int64_t k = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (k >= n_runs || first[k] >= n) return;
  const int64_t p0 = k * kRun;
  const int e = entry[k];
  Gen g{advance(s0, inc, static_cast<uint64_t>(p0 + e)), inc};
  int q = e;
  int64_t o = first[k];
  while (q < kRun && o < n) {
    bool acc;
    double v;
    q += attempt(t, g.next64(), g, acc, v);
    if (acc) out[o++] = v;
  }
}

// host copies of the tables for the rare chain resolution on the host
struct HostTables {
  double wi[256], fi[256];
  uint64_t ki[256];
};

}  // namespace zig
}  // namespace fedhc

using namespace fedhc;

// n standard normals of numpy's Generator.standard_normal from the PCG64 stream whose state BEFORE the first
// draw is (state, inc) = (state_hi:state_lo, inc_hi:inc_lo) -- rng.bit_generator.state["state"] of the
// reference's generator.  out: device fp64 [n].  state_after (host, optional): the stream state after the last
// draw numpy would have taken (for chaining further draws).  Synchronous on `stream`.
extern "C" int fedhc_pcg64_standard_normal(const uint64_t* state_words, int64_t n, double* out, uint64_t* state_after,
                                           void* stream) {
  using namespace zig;
  if (n < 0 || state_words == nullptr || (n > 0 && out == nullptr)) return fail(FEDHC_ERR_VALUE, "standard_normal: bad arguments");
  const u128 s0 = (static_cast<u128>(state_words[0]) << 64) | state_words[1];
  const u128 inc = (static_cast<u128>(state_words[2]) << 64) | state_words[3];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HostTables ht;
  FEDHC_CUDA_TRY(cudaMemcpyFromSymbol(ht.wi, wi, sizeof(ht.wi)));
  FEDHC_CUDA_TRY(cudaMemcpyFromSymbol(ht.fi, fi, sizeof(ht.fi)));
  FEDHC_CUDA_TRY(cudaMemcpyFromSymbol(ht.ki, ki, sizeof(ht.ki)));
  // positions: n accepted attempts need ~1.01 n draws; extend and redo in the (never seen) case of a shortfall
  int64_t n_runs = (n + n / 32) / kRun + 2;
  for (;;) {
    int16_t *d_exit = nullptr, *d_count = nullptr, *d_entry = nullptr;
    int64_t* d_first = nullptr;
    const size_t tab = (size_t)n_runs * kE * sizeof(int16_t);
    FEDHC_CUDA_TRY(cudaMallocAsync(&d_exit, tab, st));
    FEDHC_CUDA_TRY(cudaMallocAsync(&d_count, tab, st));
    FEDHC_CUDA_TRY(cudaMallocAsync(&d_entry, n_runs * sizeof(int16_t), st));
    FEDHC_CUDA_TRY(cudaMallocAsync(&d_first, n_runs * sizeof(int64_t), st));
    const unsigned grid = static_cast<unsigned>((n_runs + kThreads - 1) / kThreads);
    runs_kernel<<<grid, kThreads, 0, st>>>(s0, inc, n_runs, d_exit, d_count);
    FEDHC_CUDA_TRY(cudaGetLastError());
    std::vector<int16_t> h_exit((size_t)n_runs * kE), h_count((size_t)n_runs * kE), h_entry(n_runs);
    std::vector<int64_t> h_first(n_runs);
    FEDHC_CUDA_TRY(cudaMemcpyAsync(h_exit.data(), d_exit, tab, cudaMemcpyDeviceToHost, st));
    FEDHC_CUDA_TRY(cudaMemcpyAsync(h_count.data(), d_count, tab, cudaMemcpyDeviceToHost, st));
    FEDHC_CUDA_TRY(cudaStreamSynchronize(st));
    // chain the runs: run 0 starts with an attempt at offset 0
    int entry = 0;
    int64_t total = 0, last_pos = 0;
    bool enough = false;
    for (int64_t k = 0; k < n_runs; ++k) {
      h_entry[k] = static_cast<int16_t>(entry);
      h_first[k] = total;
      int cnt, ex;
      if (entry < kE) {
        cnt = h_count[k * kE + entry];
        ex = h_exit[k * kE + entry];
      } else {
        walk(ht, s0, inc, k * (int64_t)kRun, entry, cnt, ex);
      }
      if (!enough && total + cnt >= n) {
        enough = true;
        // the stream position right after the n-th normal's attempt (for state_after)
        Gen g{advance(s0, inc, static_cast<uint64_t>(k * (int64_t)kRun + entry)), inc};
        int64_t pos = k * (int64_t)kRun + entry, got = total;
        while (got < n) {
          bool acc;
          double v;
          pos += attempt(ht, g.next64(), g, acc, v);
          got += acc ? 1 : 0;
        }
        last_pos = pos;
      }
      total += cnt;
      entry = ex;
    }
    if (enough || n == 0) {
      FEDHC_CUDA_TRY(cudaMemcpyAsync(d_entry, h_entry.data(), n_runs * sizeof(int16_t), cudaMemcpyHostToDevice, st));
      FEDHC_CUDA_TRY(cudaMemcpyAsync(d_first, h_first.data(), n_runs * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      if (n > 0) emit_kernel<<<grid, kThreads, 0, st>>>(s0, inc, n_runs, d_entry, d_first, n, out);
      FEDHC_CUDA_TRY(cudaGetLastError());
      FEDHC_CUDA_TRY(cudaFreeAsync(d_exit, st));
      FEDHC_CUDA_TRY(cudaFreeAsync(d_count, st));
      FEDHC_CUDA_TRY(cudaFreeAsync(d_entry, st));
      FEDHC_CUDA_TRY(cudaFreeAsync(d_first, st));
      FEDHC_CUDA_TRY(cudaStreamSynchronize(st));
      if (state_after) {
        const u128 sa = advance(s0, inc, static_cast<uint64_t>(n == 0 ? 0 : last_pos));
        state_after[0] = static_cast<uint64_t>(sa >> 64);
        state_after[1] = static_cast<uint64_t>(sa);
      }
      return FEDHC_OK;
    }
    FEDHC_CUDA_TRY(cudaFreeAsync(d_exit, st));
    FEDHC_CUDA_TRY(cudaFreeAsync(d_count, st));
    FEDHC_CUDA_TRY(cudaFreeAsync(d_entry, st));
    FEDHC_CUDA_TRY(cudaFreeAsync(d_first, st));
    n_runs *= 2;
  }
}
