// Batch-order generator: the PCG64 permutations local_train draws
// (fl_core.py:181-187: `rng = np.random.default_rng(seed); rng.permutation(n)`),
// re-implemented natively and multi-threaded.
//
// Bit-exact with numpy >= 1.17 for integer seeds:
//   SeedSequence(seed).generate_state(4, uint64)      (numpy bit_generator.pyx)
//   PCG64 XSL-RR 128/64, pcg64_set_seed(state, inc)    (numpy pcg64.h/.c)
//   Generator.permutation(n) = arange(n) + Fisher-Yates from the top with
//   random_interval(i) on buffered 32-bit halves       (numpy distributions.c)
// Verified against numpy in tests/test_host_parity.py.
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fedhc.h"

namespace fedhc {
int fail(int code, const std::string& msg);
}

#include "pcg64.cuh"

namespace {

using fedhc_pcg::Pcg64;

void permutations_for(uint64_t seed, int32_t n, int32_t count, int32_t* out) {
  Pcg64 rng(seed);
  for (int32_t p = 0; p < count; ++p) {
    int32_t* a = out + static_cast<int64_t>(p) * n;
    for (int32_t i = 0; i < n; ++i) a[i] = i;
    fedhc_pcg::fisher_yates(rng, a, n);
  }
}

}  // namespace
extern "C" int fedhc_pcg64_state(uint64_t seed, uint64_t* state_hi, uint64_t* state_lo, uint64_t* inc_hi,
                                 uint64_t* inc_lo) {
  Pcg64 r(seed);
  *state_hi = static_cast<uint64_t>(r.state >> 64);
  *state_lo = static_cast<uint64_t>(r.state);
  *inc_hi = static_cast<uint64_t>(r.inc >> 64);
  *inc_lo = static_cast<uint64_t>(r.inc);
  return FEDHC_OK;
}

extern "C" int fedhc_batch_permutations(const uint64_t* seeds, const int32_t* n_rows, const int32_t* n_perms,
                                        const int64_t* offsets, int n_clients, int32_t* out, int n_threads) {
  if (n_clients < 0) return fedhc::fail(FEDHC_ERR_VALUE, "batch_permutations: negative client count");
  for (int c = 0; c < n_clients; ++c)
    if (n_rows[c] < 0 || n_perms[c] < 0) return fedhc::fail(FEDHC_ERR_VALUE, "batch_permutations: negative size");
  int threads = n_threads > 0 ? n_threads : static_cast<int>(std::thread::hardware_concurrency());
  threads = std::max(1, std::min(threads, n_clients));
  if (threads == 1) {
    for (int c = 0; c < n_clients; ++c) permutations_for(seeds[c], n_rows[c], n_perms[c], out + offsets[c]);
    return FEDHC_OK;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  pool.reserve(threads);
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (int c = next.fetch_add(1); c < n_clients; c = next.fetch_add(1))
        permutations_for(seeds[c], n_rows[c], n_perms[c], out + offsets[c]);
    });
  for (auto& th : pool) th.join();
  return FEDHC_OK;
}
