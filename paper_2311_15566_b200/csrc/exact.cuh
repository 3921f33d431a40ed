// exact.cuh -- correctly rounded integer-ratio -> double conversion, shared by
// the host planner (planner.cpp) and the device kernels (spotkm.cu).
//
// The reference converts exact Fractions with float() (domain.py:320,
// migration.py's byte counts); float(Fraction(n, d)) is the correctly rounded
// (round-half-even) value of n / d.  rat_to_double reproduces it for any
// 0 <= n < 2^127 and 0 < d < 2^63.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define SK_HD __host__ __device__ __forceinline__
#else
#define SK_HD inline
#endif

namespace sk_exact {

typedef __int128 i128;

SK_HD int bitlen(i128 x) {
  const uint64_t hi = (uint64_t)((unsigned __int128)x >> 64), lo = (uint64_t)x;
#if defined(__CUDA_ARCH__)
  return hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
#else
  return hi ? 128 - __builtin_clzll(hi) : (lo ? 64 - __builtin_clzll(lo) : 0);
#endif
}

SK_HD double scale2(double x, int e) {
#if defined(__CUDA_ARCH__)
  return ldexp(x, e);
#else
  return __builtin_ldexp(x, e);
#endif
}

// correctly rounded num / den (num >= 0, den > 0)
SK_HD double rat_to_double(i128 num, int64_t den) {
  if (num == 0) return 0.0;
  const i128 lim = (i128)1 << 53;
  if (num < lim && den < ((int64_t)1 << 53)) {
    // both exact in double: one IEEE division is correctly rounded
#if defined(__CUDA_ARCH__)
    return __ddiv_rn((double)(int64_t)num, (double)den);
#else
    return (double)(int64_t)num / (double)den;
#endif
  }
  // scale so that the integer quotient has 54 bits, then round half-even
  int s = 54 - (bitlen(num) - bitlen((i128)den));
  i128 n = num, d = den;
  if (s >= 0)
    n <<= s;
  else
    d <<= -s;
  i128 q = n / d, r = n % d;
  while (q >= ((i128)1 << 54)) {  // the estimate was one bit long
    r += (q & 1) * d;
    q >>= 1;
    d <<= 1;
    --s;
  }
  while (q < ((i128)1 << 53)) {
    n = r * 2;
    q = q * 2 + n / d;
    r = n % d;
    ++s;
  }
  // q has 54 bits: keep 53, round half-even with the dropped bit and r
  const bool half = (q & 1) != 0;
  q >>= 1;
  const bool sticky = r != 0;
  if (half && (sticky || (q & 1))) ++q;
  return scale2((double)(int64_t)q, -(s - 1));
}

}  // namespace sk_exact
