// Per-round client seeds -- fl_core.stable_seed (fl_core.py:21-24) as used by
// engine.run_experiment (engine.py:336-347) and local_train (fl_core.py:181):
//
//   train_seed = stable_seed("train", seed, r, cid)
//              = LE uint32 of sha256(repr(("train", seed, r, cid)))[:4]
//   rng_seed   = stable_seed("local_train", train_seed)
//
// The caller passes repr(cid) (Python's quoting rules), so the hashed byte
// strings are exactly Python's repr of the tuples.  SHA-256 per FIPS 180-4.
#include <stdint.h>
#include <string.h>

#include <string>

#include "../../include/fedhc.h"

namespace fedhc {
int fail(int code, const std::string& msg);
}

namespace {

constexpr uint32_t kK[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

inline uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

void compress(uint32_t h[8], const uint8_t* blk) {
  uint32_t w[64];
  for (int i = 0; i < 16; ++i)
    w[i] = (uint32_t)blk[4 * i] << 24 | (uint32_t)blk[4 * i + 1] << 16 | (uint32_t)blk[4 * i + 2] << 8 | blk[4 * i + 3];
  for (int i = 16; i < 64; ++i) {
    const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
    const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
    w[i] = w[i - 16] + s0 + w[i - 7] + s1;
  }
  uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
  for (int i = 0; i < 64; ++i) {
    const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + kK[i] + w[i];
    const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
    hh = g;
    g = f;
    f = e;
    e = d + t1;
    d = c;
    c = b;
    b = a;
    a = t1 + t2;
  }
  h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// first 4 digest bytes, little-endian (int.from_bytes(digest[:4], "little"))
uint32_t sha256_le32(const std::string& msg) {
  uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  const size_t n = msg.size();
  size_t i = 0;
  for (; i + 64 <= n; i += 64) compress(h, reinterpret_cast<const uint8_t*>(msg.data()) + i);
  uint8_t tail[128] = {0};
  const size_t rem = n - i;
  memcpy(tail, msg.data() + i, rem);
  tail[rem] = 0x80;
  const size_t tl = rem + 9 <= 64 ? 64 : 128;
  const uint64_t bits = static_cast<uint64_t>(n) * 8;
  for (int k = 0; k < 8; ++k) tail[tl - 1 - k] = static_cast<uint8_t>(bits >> (8 * k));
  compress(h, tail);
  if (tl == 128) compress(h, tail + 64);
  const uint32_t d0 = h[0];  // digest bytes 0..3 = big-endian h[0]
  return (d0 >> 24) | ((d0 >> 8) & 0xff00u) | ((d0 << 8) & 0xff0000u) | (d0 << 24);
}

}  // namespace

extern "C" uint32_t fedhc_sha256_le32(const char* data, int64_t n) { return sha256_le32(std::string(data, n)); }

extern "C" int fedhc_round_seeds(int64_t seed, int64_t round_index, const char* const* cid_reprs, int n,
                                 uint64_t* train_seeds, uint64_t* rng_seeds) {
  if (n < 0) return fedhc::fail(FEDHC_ERR_VALUE, "round_seeds: negative count");
  const std::string head = "('train', " + std::to_string(seed) + ", " + std::to_string(round_index) + ", ";
  for (int i = 0; i < n; ++i) {
    const uint32_t ts = sha256_le32(head + cid_reprs[i] + ")");
    train_seeds[i] = ts;
    rng_seeds[i] = sha256_le32("('local_train', " + std::to_string(ts) + ")");
  }
  return FEDHC_OK;
}
