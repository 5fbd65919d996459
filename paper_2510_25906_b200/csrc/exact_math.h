// Exact-arithmetic helpers shared by the device kernels and the host-side
// tests (tests/test_exact_math.py compiles this header with g++ and checks it
// against the plain expressions on adversarial inputs). Every function returns
// bit-for-bit what the reference expression returns; only the work differs.
// Compile with FMA contraction off (nvcc --fmad=false, g++ -ffp-contract=off):
// the explicit fma() calls are the only fused operations.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define UCFVB_HD __host__ __device__ __forceinline__
#else
#define UCFVB_HD inline
#endif

namespace ucfvb {

using std::fabs;
using std::fma;

// pressure / is_physical (euler.hpp:30-36)
UCFVB_HD double pressure(const double* s, double g) {
  return (g - 1.0) * (s[3] - 0.5 * (s[1] * s[1] + s[2] * s[2]) / s[0]);
}
// is_physical = s0 > 0 && pressure > 0, decided without the division in the
// common case: with s0 > 0, g - 1 >= 2^-60 and P = RN(s3*s0) in [2^-900,
// 2^900], A = 0.5*(s1^2 + s2^2) below RN(P*(1 - 2^-46)) puts A/s0 below
// s3*(1 - 2^-47) (P and the product carry <= 2^-53 each), so RN(A/s0) < s3
// strictly and the pressure is positive (s3 >= 2^-900 keeps it clear of
// underflow); above RN(P*(1 + 2^-46)) it is negative. s3 <= 0 gives p <= 0
// outright. Inside the margin, and for non-finite inputs, the reference
// expression decides -- the result is always the reference's.
UCFVB_HD bool is_physical(const double* s, double g) {
  const double gm1 = g - 1.0;
  const double A = 0.5 * (s[1] * s[1] + s[2] * s[2]);
  const double P = s[3] * s[0];
  const bool pos = s[0] > 0.0;
  const bool gok = gm1 >= 0x1p-60;
  const bool neg_e = gok && s[3] <= 0.0;  // p <= 0 whatever A / s0 is
  const bool range = gok && s[3] >= 0x1p-900 && P >= 0x1p-900 && P <= 0x1p900;
  const bool below = range && A < P * (1.0 - 0x1p-46);
  const bool above = range && A > P * (1.0 + 0x1p-46);
  bool r = pos && below;
  if (pos && !neg_e && !below && !above) r = pressure(s, g) > 0.0;  // rare: inside the margin / non-finite
  return r;
}

// RN(x / d) from r = RN(1 / d) (d in [2^-60, 2^60]): q = RN(x r) and two
// remainder corrections e = fma(-q, d, x) (exact once q is within an ulp),
// q = fma(e, r, q); the last one is Markstein's correctly rounded step. Valid
// when div_rn_ok(x): x = +-0 (returned as is: x / d keeps the sign of a zero)
// or 2^-960 <= |x| < 2^960; callers test a batch of numerators once and take
// the IEEE division for the whole batch otherwise (tiny, huge, non-finite).
UCFVB_HD bool div_rn_ok(double x) {
  uint64_t b;
  std::memcpy(&b, &x, sizeof b);
  const uint32_t e = static_cast<uint32_t>(b >> 52) & 0x7ffu;  // biased exponent
  return (e - 63u) < 1920u || (b << 1) == 0;
}
UCFVB_HD double div_rn_unchecked(double x, double d, double r) {
  double q = x * r;
  double e = fma(-q, d, x);
  q = fma(e, r, q);
  e = fma(-q, d, x);
  q = fma(e, r, q);
  return x == 0.0 ? x : q;
}
UCFVB_HD double div_rn(double x, double d, double r) {
  return div_rn_ok(x) ? div_rn_unchecked(x, d, r) : x / d;
}

}  // namespace ucfvb
