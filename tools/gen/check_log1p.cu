// Pins log1p_glibc.cuh (host instantiation: the same source, FMA-explicit) against this image's libm log1p
// on the inputs numpy's ziggurat tail feeds it (x = -u, u = m / 2^53).  Build + run:
//   nvcc -O2 -std=c++17 tools/gen/check_log1p.cu -o /tmp/check_log1p && /tmp/check_log1p
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../paper_2305_15668_b200/csrc/log1p_glibc.cuh"

int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 300000000L;
  uint64_t st = 88172645463325252ull;
  long bad = 0;
  for (long i = 0; i < n; ++i) {
    st ^= st << 13;
    st ^= st >> 7;
    st ^= st << 17;
    uint64_t m = st >> 11;
    if (i % 4 == 1) m >>= (st & 63) % 53;                          // small u
    if (i % 1000 == 7) m = (st >> 11) >> (25 + (st & 31) % 28);   // |x| < 2^-29
    const double x = -static_cast<double>(m) * (1.0 / 9007199254740992.0);
    const double want = log1p(x), got = fedhc::zig::glibc_log1p(x);
    if (memcmp(&want, &got, sizeof got) != 0) {
      if (bad < 5) printf("x=%a libm=%a ours=%a\n", x, want, got);
      ++bad;
    }
  }
  printf("glibc_log1p: %ld mismatches against libm log1p in %ld inputs\n", bad, n);
  return bad != 0;
}
