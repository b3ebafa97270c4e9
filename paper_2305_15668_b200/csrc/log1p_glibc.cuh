// log1p bit-identical to the image's glibc, plus round-to-nearest arithmetic helpers that keep nvcc from
// contracting host-ordered expressions into FMAs.  Used by normal.cu (numpy's ziggurat tail) and pinned by
// tools/gen/check_log1p.cu.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

namespace fedhc {
namespace zig {

__host__ __device__ __forceinline__ long long as_bits(double x) {
#ifdef __CUDA_ARCH__
  return __double_as_longlong(x);
#else
  long long b;
  memcpy(&b, &x, sizeof b);
  return b;
#endif
}
__host__ __device__ __forceinline__ double from_bits(long long b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(b);
#else
  double x;
  memcpy(&x, &b, sizeof x);
  return x;
#endif
}
__host__ __device__ __forceinline__ double add_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
__host__ __device__ __forceinline__ double sub_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
__host__ __device__ __forceinline__ double mul_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
__host__ __device__ __forceinline__ double div_rn(double a, double b) {
#ifdef __CUDA_ARCH__
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
__host__ __device__ __forceinline__ double fma_rn(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return fma(a, b, c);
#endif
}
__host__ __device__ __forceinline__ int32_t high_word(double x) {
  return static_cast<int32_t>(static_cast<uint64_t>(as_bits(x)) >> 32);
}

// log1p(x) for -1 < x <= 0 as glibc 2.39 computes it on x86-64 (its FMA ifunc build of the fdlibm-derived
// s_log1p.c: Estrin-split polynomial, with the multiply-adds the compiler fused written as fma_rn).  Pinned
// against the image's libm on 3e8 inputs by tools/gen/check_log1p.cu; numpy's random_standard_normal tail calls
// it through npy_log1p.
__host__ __device__ inline double glibc_log1p(double x) {
  constexpr double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  constexpr double two54 = 1.80143985094819840000e+16;
  constexpr double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
                   Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                   Lp7 = 1.479819860511658591e-01;
  const int32_t hx = high_word(x), ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;
    if (ax < 0x3e200000) {
      if (add_rn(two54, x) > 0.0 && ax < 0x3c900000) return x;
      return fma_rn(-mul_rn(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= static_cast<int32_t>(0xbfd2bec3)) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (k != 0) {
    double u = add_rn(1.0, x);
    hu = high_word(u);
    k = (hu >> 20) - 1023;
    c = k > 0 ? sub_rn(1.0, sub_rn(u, x)) : sub_rn(x, sub_rn(u, 1.0));
    c = div_rn(c, u);
    hu &= 0x000fffff;
    const uint64_t lo = static_cast<uint64_t>(as_bits(u)) & 0xffffffffull;
    if (hu < 0x6a09e) {
      u = from_bits(static_cast<long long>((static_cast<uint64_t>(hu | 0x3ff00000) << 32) | lo));
    } else {
      k += 1;
      u = from_bits(static_cast<long long>((static_cast<uint64_t>(hu | 0x3fe00000) << 32) | lo));
      hu = (0x00100000 - hu) >> 2;
    }
    f = sub_rn(u, 1.0);
  }
  const double hfsq = mul_rn(mul_rn(0.5, f), f), dk = static_cast<double>(k);
  if (hu == 0) {
    if (f == 0.0) return k == 0 ? 0.0 : fma_rn(dk, ln2_hi, fma_rn(dk, ln2_lo, c));
    const double R = mul_rn(hfsq, fma_rn(-0.66666666666666666, f, 1.0));
    if (k == 0) return sub_rn(f, R);
    return fma_rn(dk, ln2_hi, -sub_rn(sub_rn(R, fma_rn(dk, ln2_lo, c)), f));
  }
  const double s = div_rn(f, add_rn(2.0, f)), z = mul_rn(s, s);
  const double z2 = mul_rn(z, z), z4 = mul_rn(z2, z2), z6 = mul_rn(z4, z2);
  const double R2 = fma_rn(z, Lp3, Lp2), R3 = fma_rn(z, Lp5, Lp4), R4 = fma_rn(z, Lp7, Lp6);
  const double R = fma_rn(z6, R4, fma_rn(z4, R3, fma_rn(z, Lp1, mul_rn(z2, R2))));
  const double st = mul_rn(s, add_rn(hfsq, R));
  if (k == 0) return sub_rn(f, sub_rn(hfsq, st));
  return fma_rn(dk, ln2_hi, -sub_rn(sub_rn(hfsq, add_rn(fma_rn(dk, ln2_lo, c), st)), f));
}

}  // namespace zig
}  // namespace fedhc
