"""csrc/exact_math.h -- the shortcuts the kernels take for the reference's
is_physical (euler.hpp:34-36) and for divisions by a value whose reciprocal is
known (CWENOZ weights, reconstruct.cpp:104-147) -- compiled with g++ exactly
as shipped and compared bit-for-bit with the plain expressions on random and
adversarial inputs (quotients next to rounding boundaries, pressures within a
few ulps of zero, divisors with all-ones significands, zeros, subnormals,
infinities, NaNs)."""
import shutil
import subprocess
from pathlib import Path

import pytest

CSRC = Path(__file__).resolve().parents[1] / "paper_2510_25906_b200" / "csrc"

PROG = r"""
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <limits>
#include "exact_math.h"
using namespace ucfvb;
static uint64_t st = 0x9E3779B97F4A7C15ULL;
static inline uint64_t rnd() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }
static inline double mk(int e) {  // random significand, exponent e
  uint64_t b = ((uint64_t)(e + 1023) << 52) | (rnd() & ((1ULL << 52) - 1));
  double x; std::memcpy(&x, &b, 8); return x;
}
static inline bool same(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }
static bool ref_phys(const double* s, double g) { return s[0] > 0.0 && pressure(s, g) > 0.0; }
int main(int argc, char** argv) {
  const long n = atol(argv[1]);
  long bad_div = 0, bad_phys = 0, fast_hits = 0;
  const double specials[] = {0.0, -0.0, 5e-324, -5e-324, 1e-310, std::numeric_limits<double>::infinity(),
                             -std::numeric_limits<double>::infinity(), std::nan(""), 1.0, -1.0};
  double ds[9] = {1.0 - 1.0 / 1e3, 1.0 - 1.0 / 1e4, 1.0 - 1.0 / 1e2, 3.0, 4.0, 1.0 / 3.0,
                  std::nextafter(1.0, 0.0), 1.0 + 0x1p-52, 0x1.fffffffffffffp+1};
  for (long it = 0; it < n; ++it) {
    // ---- div_rn
    double d = (it % 4 != 3) ? ds[it % 9] : mk((int)(rnd() % 120) - 60);
    if (it % 16 == 7) { uint64_t b = 0x3ff0000000000000ULL | ((1ULL << 52) - 1 - (rnd() % 64)); std::memcpy(&d, &b, 8); }
    const double r = 1.0 / d;
    double x;
    switch (rnd() % 4) {
      case 0: x = mk((int)(rnd() % 1940) - 970); break;
      case 1: { double q = mk((int)(rnd() % 1800) - 900); x = std::nextafter(q * d, (rnd() & 1) ? 1e308 : -1e308); break; }
      case 2: { double q = mk((int)(rnd() % 1800) - 900); double h = std::nextafter(q, 1e308) - q;
                x = (q + 0.5 * h) * d; x = std::nextafter(x, (rnd() & 1) ? 1e308 : -1e308); break; }
      default: x = specials[rnd() % 10];
    }
    if (rnd() & 1) x = -x;
    if (!same(div_rn(x, d, r), x / d) || (div_rn_ok(x) && !same(div_rn_unchecked(x, d, r), x / d))) { if (bad_div < 5) std::printf("div x=%a d=%a\n", x, d); ++bad_div; }
    // ---- is_physical
    double s[4];
    s[0] = (rnd() % 8) ? mk((int)(rnd() % 40) - 20) : specials[rnd() % 10];
    s[1] = mk((int)(rnd() % 40) - 20) * ((rnd() & 1) ? 1 : -1);
    s[2] = mk((int)(rnd() % 40) - 20) * ((rnd() & 1) ? 1 : -1);
    const double A = 0.5 * (s[1] * s[1] + s[2] * s[2]);
    const int mode = rnd() % 5;
    if (mode == 0) s[3] = mk((int)(rnd() % 80) - 40);
    else if (mode == 4) s[3] = specials[rnd() % 10];
    else {  // s3 within a few ulps / within the 2^-46 band of A/s0: pressure near zero
      double t = A / s[0];
      if (mode == 2) t = t * (1.0 + (double)((int)(rnd() % 2001) - 1000) * 0x1p-53);
      if (mode == 3) t = t * (1.0 + (double)((int)(rnd() % 2001) - 1000) * 0x1p-46);
      for (int k = (int)(rnd() % 7) - 3; k != 0; k += (k > 0 ? -1 : 1)) t = std::nextafter(t, k > 0 ? 1e308 : -1e308);
      s[3] = t;
    }
    const double g = (it % 7 == 0) ? 1.0 + 0x1p-70 : 1.4;
    if (is_physical(s, g) != ref_phys(s, g)) {
      if (bad_phys < 5) std::printf("phys %a %a %a %a\n", s[0], s[1], s[2], s[3]); ++bad_phys;
    }
  }
  std::printf("%ld %ld\n", bad_div, bad_phys);
  return 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="no host compiler")
def test_exact_math_matches_plain_expressions(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(PROG)
    exe = tmp_path / "t"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", f"-I{CSRC}", str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe), "20000000"], capture_output=True, text=True, check=True).stdout
    assert out.strip().splitlines()[-1] == "0 0", out
