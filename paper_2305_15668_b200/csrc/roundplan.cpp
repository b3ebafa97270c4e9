// Host round planning in native code (the serving loop's per-round host work, FederatedRunner.plan):
//
//   fedhc_mt_sample   CPython 3.12's random.Random.sample(range(n), k) on an MT19937 state taken from
//                     Random.getstate() -- the reference's participant selection (engine.py:302, :327),
//                     bit-exact (same _randbelow rejection draws, same pool / set branches).
//   fedhc_round_pack  the rest of a round's plan for this rank's participants in one call: per-client seeds
//                     (stable_seed("train", ...) -> stable_seed("local_train", ...), fl_core.py:21-24, :181),
//                     the device batch-order block (PCG64 seeds, shard sizes, permutation counts, offsets),
//                     the local_train descriptors and the FedAvg coefficients w_i / W, written straight into
//                     the pinned staging block that is copied to the GPU in one transfer.
//
// ctypes releases the GIL for the duration of these calls, so the planner thread no longer competes with
// the launching thread for the interpreter.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/fedhc.h"

namespace fedhc {
int fail(int code, const std::string& msg);
}

namespace {

constexpr int kN = 624, kM = 397;

// CPython Modules/_randommodule.c genrand_uint32 on the (state[624], index) pair of Random.getstate()
uint32_t genrand(uint32_t* mt, uint32_t& index) {
  static const uint32_t mag01[2] = {0x0u, 0x9908b0dfu};
  uint32_t y;
  if (index >= (uint32_t)kN) {
    int kk;
    for (kk = 0; kk < kN - kM; kk++) {
      y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
      mt[kk] = mt[kk + kM] ^ (y >> 1) ^ mag01[y & 0x1u];
    }
    for (; kk < kN - 1; kk++) {
      y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
      mt[kk] = mt[kk + (kM - kN)] ^ (y >> 1) ^ mag01[y & 0x1u];
    }
    y = (mt[kN - 1] & 0x80000000u) | (mt[0] & 0x7fffffffu);
    mt[kN - 1] = mt[kM - 1] ^ (y >> 1) ^ mag01[y & 0x1u];
    index = 0;
  }
  y = mt[index++];
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= (y >> 18);
  return y;
}

int bit_length(uint32_t n) {
  int k = 0;
  while (n) {
    ++k;
    n >>= 1;
  }
  return k;
}

// Random._randbelow_with_getrandbits(n), n in [1, 2^31)
uint32_t randbelow(uint32_t* mt, uint32_t& index, uint32_t n) {
  const int k = bit_length(n);
  uint32_t r = genrand(mt, index) >> (32 - k);
  while (r >= n) r = genrand(mt, index) >> (32 - k);
  return r;
}

// CPython >= 3.12 sum() over floats (Neumaier), as in des.cpp
struct PySum {
  double s = 0.0, c = 0.0;
  void add(double x) {
    const double t = s + x;
    if (fabs(s) >= fabs(x))
      c += (s - t) + x;
    else
      c += (x - t) + s;
    s = t;
  }
  double value() const { return (c != 0.0 && isfinite(c)) ? s + c : s; }
};

}  // namespace

extern "C" uint32_t fedhc_sha256_le32(const char* data, int64_t n);

extern "C" int fedhc_mt_sample(uint32_t* state, int n, int k, int32_t* out) {
  if (state == nullptr || (k > 0 && out == nullptr)) return fedhc::fail(FEDHC_ERR_VALUE, "mt_sample: null pointer");
  if (!(0 <= k && k <= n)) return fedhc::fail(FEDHC_ERR_VALUE, "Sample larger than population or is negative");
  uint32_t* mt = state;
  uint32_t index = state[kN];
  if (index > (uint32_t)kN) return fedhc::fail(FEDHC_ERR_VALUE, "mt_sample: bad MT19937 state index");
  // setsize = 21; if k > 5: setsize += 4 ** ceil(log(k * 3, 4))  (math.log(x, b) = log(x) / log(b))
  double setsize = 21.0;
  if (k > 5) setsize += pow(4.0, ceil(log((double)k * 3.0) / log(4.0)));
  if ((double)n <= setsize) {
    std::vector<int32_t> pool(n);
    for (int i = 0; i < n; ++i) pool[i] = i;
    for (int i = 0; i < k; ++i) {
      const uint32_t j = randbelow(mt, index, (uint32_t)(n - i));
      out[i] = pool[j];
      pool[j] = pool[n - i - 1];
    }
  } else {
    std::unordered_set<uint32_t> selected;
    selected.reserve(2 * (size_t)k);
    for (int i = 0; i < k; ++i) {
      uint32_t j = randbelow(mt, index, (uint32_t)n);
      while (selected.count(j)) j = randbelow(mt, index, (uint32_t)n);
      selected.insert(j);
      out[i] = (int32_t)j;
    }
  }
  state[kN] = index;
  return FEDHC_OK;
}

extern "C" double fedhc_py_float_sum(const double* x, int n) {
  PySum s;
  for (int i = 0; i < n; ++i) s.add(x[i]);
  return s.value();
}

extern "C" int fedhc_round_pack(int64_t seed, int64_t round_index, int k, const int64_t* mine,
                                const char* const* reprs, const int32_t* rows, const int32_t* n_perms,
                                const int32_t* n_batches, const int32_t* batch_size, const uint64_t* xptr,
                                const uint64_t* yptr, const double* weight, double total, float lr,
                                uint64_t perm_base, uint64_t delta_base, int64_t delta_stride, uint8_t* staging,
                                int64_t* perm_words, int32_t* max_rows) {
  if (k < 0) return fedhc::fail(FEDHC_ERR_VALUE, "round_pack: negative count");
  if (k > 0 && (mine == nullptr || staging == nullptr))
    return fedhc::fail(FEDHC_ERR_VALUE, "round_pack: null pointer");
  static_assert(sizeof(fedhc_client) == 48, "descriptor layout");
  uint64_t* m_seed = reinterpret_cast<uint64_t*>(staging);
  int32_t* m_rows = reinterpret_cast<int32_t*>(staging + 8 * (size_t)k);
  int32_t* m_perm = reinterpret_cast<int32_t*>(staging + 12 * (size_t)k);
  int64_t* m_off = reinterpret_cast<int64_t*>(staging + 16 * (size_t)k);
  uint8_t* desc = staging + 24 * (size_t)k;
  double* coef = reinterpret_cast<double*>(desc + sizeof(fedhc_client) * (size_t)k);
  const std::string head = "('train', " + std::to_string(seed) + ", " + std::to_string(round_index) + ", ";
  int64_t at = 0;
  int32_t mr = 0;
  for (int i = 0; i < k; ++i) {
    const int64_t c = mine[i];
    const std::string msg = head + reprs[c] + ")";
    const uint32_t ts = fedhc_sha256_le32(msg.data(), (int64_t)msg.size());
    const std::string msg2 = "('local_train', " + std::to_string(ts) + ")";
    m_seed[i] = fedhc_sha256_le32(msg2.data(), (int64_t)msg2.size());
    m_rows[i] = rows[c];
    m_perm[i] = n_perms[c];
    m_off[i] = at;
    fedhc_client d{};
    d.x = reinterpret_cast<const float*>(xptr[c]);
    d.y = reinterpret_cast<const int32_t*>(yptr[c]);
    d.perm = reinterpret_cast<const int32_t*>(perm_base + (uint64_t)at * 4);
    d.n_rows = rows[c];
    d.n_batches = n_batches[c];
    d.batch_size = batch_size[c];
    d.lr = lr;
    d.delta = reinterpret_cast<float*>(delta_base + (uint64_t)i * (uint64_t)delta_stride);
    memcpy(desc + sizeof(fedhc_client) * (size_t)i, &d, sizeof(fedhc_client));
    coef[i] = weight[c] / total;
    at += (int64_t)rows[c] * n_perms[c];
    if (rows[c] > mr) mr = rows[c];
  }
  if (perm_words) *perm_words = at;
  if (max_rows) *max_rows = mr;
  return FEDHC_OK;
}
