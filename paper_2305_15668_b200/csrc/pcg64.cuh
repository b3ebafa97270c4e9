// numpy-compatible SeedSequence + PCG64 (XSL-RR 128/64), usable on host and
// device.  Bit-exact with numpy >= 1.17 (bit_generator.pyx SeedSequence,
// pcg64.h pcg64_set_seed / pcg64_next32, distributions.c random_interval).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define FEDHC_HD __host__ __device__
#else
#define FEDHC_HD
#endif

namespace fedhc_pcg {

typedef unsigned __int128 u128;

// ---- numpy SeedSequence (pool size 4) --------------------------------------
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kXShift = 16;

FEDHC_HD inline uint32_t hashmix(uint32_t v, uint32_t& h) {
  v ^= h;
  h *= kMultA;
  v *= h;
  v ^= v >> kXShift;
  return v;
}

FEDHC_HD inline uint32_t mixw(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> kXShift;
  return r;
}

// entropy = little-endian 32-bit words of the non-negative integer seed
FEDHC_HD inline void seed_sequence_state(uint64_t seed, uint64_t out[4]) {
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
#define FEDHC_PCG_MULT ((static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull)

struct Pcg64 {
  u128 state, inc;
  bool has32 = false;
  uint32_t buf32 = 0;

  FEDHC_HD explicit Pcg64(uint64_t seed) {
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
  FEDHC_HD inline void step() {
#ifdef __CUDA_ARCH__
    // 128-bit LCG step from four 64-bit products (the generic u128 multiply compiles to a longer chain)
    constexpr uint64_t MH = 0x2360ED051FC65DA4ull, ML = 0x4385DF649FCCF645ull;
    const uint64_t lo = static_cast<uint64_t>(state), hi = static_cast<uint64_t>(state >> 64);
    const uint64_t ilo = static_cast<uint64_t>(inc), ihi = static_cast<uint64_t>(inc >> 64);
    const uint64_t p_lo = lo * ML;
    uint64_t p_hi = __umul64hi(lo, ML) + hi * ML + lo * MH;
    const uint64_t n_lo = p_lo + ilo;
    p_hi += ihi + (n_lo < p_lo ? 1ull : 0ull);
    state = (static_cast<u128>(p_hi) << 64) | n_lo;
#else
    state = state * FEDHC_PCG_MULT + inc;
#endif
  }
  FEDHC_HD inline uint64_t next64() {
    step();
    const uint64_t x = static_cast<uint64_t>(state >> 64) ^ static_cast<uint64_t>(state);
    const unsigned rot = static_cast<unsigned>(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  FEDHC_HD inline uint32_t next32() {
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
  FEDHC_HD inline uint64_t interval(uint64_t max) {
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


// Fisher-Yates from the top with random_interval(i), exactly Generator.permutation(n):
// a = arange(n); for i = n-1 .. 1: j = random_interval(i); swap(a[i], a[j]).
template <class Array>
FEDHC_HD inline void fisher_yates(Pcg64& rng, Array& a, int32_t n) {
  if (n < 2) return;
  uint32_t mask = static_cast<uint32_t>(n - 1);
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  for (int32_t i = n - 1; i >= 1; --i) {
    while ((mask >> 1) >= static_cast<uint32_t>(i)) mask >>= 1;  // smallest all-ones mask >= i
    uint32_t v;
    do {
      v = rng.next32() & mask;
    } while (v > static_cast<uint32_t>(i));
    const int32_t t = a[i];
    a[i] = a[v];
    a[v] = t;
  }
}

}  // namespace fedhc_pcg
