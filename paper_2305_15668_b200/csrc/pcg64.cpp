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
#include <string>
#include <thread>
#include <vector>

#include "../../include/fedhc.h"

namespace fedhc {
int fail(int code, const std::string& msg);
}

namespace {

typedef unsigned __int128 u128;

// ---- numpy SeedSequence (pool size 4) --------------------------------------
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kXShift = 16;

inline uint32_t hashmix(uint32_t v, uint32_t& h) {
  v ^= h;
  h *= kMultA;
  v *= h;
  v ^= v >> kXShift;
  return v;
}

inline uint32_t mixw(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> kXShift;
  return r;
}

// entropy = little-endian 32-bit words of the non-negative integer seed
void seed_sequence_state(uint64_t seed, uint64_t out[4]) {
  uint32_t ent[2];
  int n_ent = 0;
  if (seed == 0) {
    ent[n_ent++] = 0;
  } else {
    while (seed) {
      ent[n_ent++] = static_cast<uint32_t>(seed & 0xffffffffu);
      seed >>= 32;
    }
  }
  uint32_t pool[4];
  uint32_t h = kInitA;
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u, h);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mixw(pool[d], hashmix(pool[s], h));
  for (int s = 4; s < n_ent; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mixw(pool[d], hashmix(ent[s], h));
  uint32_t st[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> kXShift;
    st[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = static_cast<uint64_t>(st[2 * i]) | (static_cast<uint64_t>(st[2 * i + 1]) << 32);
}

// ---- numpy PCG64 ----------------------------------------------------------------
// (n < 2^31 always here, so random_interval takes its 32-bit branch)
const u128 kMult = (static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;

struct Pcg64 {
  u128 state, inc;
  bool has32 = false;
  uint32_t buf32 = 0;

  explicit Pcg64(uint64_t seed) {
    uint64_t v[4];
    seed_sequence_state(seed, v);
    const u128 initstate = (static_cast<u128>(v[0]) << 64) | v[1];
    const u128 initseq = (static_cast<u128>(v[2]) << 64) | v[3];
    state = 0;
    inc = (initseq << 1) | 1;
    step();
    state += initstate;
    step();
  }
  inline void step() { state = state * kMult + inc; }
  inline uint64_t next64() {
    step();
    const uint64_t x = static_cast<uint64_t>(state >> 64) ^ static_cast<uint64_t>(state);
    const unsigned rot = static_cast<unsigned>(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  inline uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    const uint64_t n = next64();
    has32 = true;
    buf32 = static_cast<uint32_t>(n >> 32);
    return static_cast<uint32_t>(n & 0xffffffffu);
  }
  // numpy random_interval(max): smallest all-ones mask >= max, rejection.
  inline uint64_t interval(uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t value;
    if (max <= 0xffffffffull) {
      while ((value = (next32() & mask)) > max) {
      }
    } else {
      while ((value = (next64() & mask)) > max) {
      }
    }
    return value;
  }
};

void permutations_for(uint64_t seed, int32_t n, int32_t count, int32_t* out) {
  Pcg64 rng(seed);
  for (int32_t p = 0; p < count; ++p) {
    int32_t* a = out + static_cast<int64_t>(p) * n;
    for (int32_t i = 0; i < n; ++i) a[i] = i;
    if (n < 2) continue;
    // random_interval(i) for i = n-1 .. 1 with the mask hoisted out of the
    // loop (it only changes when i drops below a power of two)
    uint32_t mask = static_cast<uint32_t>(n - 1);
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    for (int32_t i = n - 1; i >= 1; --i) {
      while ((mask >> 1) >= static_cast<uint32_t>(i)) mask >>= 1;
      uint32_t v;
      do {
        v = rng.next32() & mask;
      } while (v > static_cast<uint32_t>(i));
      const int32_t t = a[i];
      a[i] = a[v];
      a[v] = t;
    }
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
