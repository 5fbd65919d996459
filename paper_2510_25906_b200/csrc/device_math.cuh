// Point functions of the stage pass as __device__ code. Every function keeps
// the reference's fp64 operation order; the kernels are compiled with
// --fmad=false so no multiply-add is contracted (the reference's x86-64 -O3
// build has no FMA). IEEE division and sqrt are the
// nvcc defaults (-prec-div=true -prec-sqrt=true).
#pragma once

#include <cstdint>

#include "exact_math.h"

namespace ucfvb {

constexpr int NV = 4;

// std::min / std::max semantics (NaN and signed-zero behaviour included)
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

struct d4 {
  double v[4];
};

__device__ __forceinline__ d4 ld4(const double4* p) {
  const double4 t = *p;
  return d4{{t.x, t.y, t.z, t.w}};
}
__device__ __forceinline__ void st4(double4* p, const d4& a) {
  *p = make_double4(a.v[0], a.v[1], a.v[2], a.v[3]);
}
__device__ __forceinline__ void st4(double4* p, const double* a) {
  *p = make_double4(a[0], a[1], a[2], a[3]);
}



// cons_to_prim (euler.hpp:38-45): returns false where the reference throws
__device__ __forceinline__ bool cons_to_prim(const double* s, double g, double& rho, double& u, double& v,
                                             double& p) {
  if (!(s[0] > 0.0)) return false;
  u = s[1] / s[0];
  v = s[2] / s[0];
  p = (g - 1.0) * (s[3] - 0.5 * s[0] * (u * u + v * v));
  if (!(p > 0.0)) return false;
  rho = s[0];
  return true;
}

struct Frame {
  double rho, un, ut, p, E, a;
};

// rotate_in (euler.cpp:13-23)
__device__ __forceinline__ bool rotate_in(const double* s, double nx, double ny, double g, Frame& f) {
  double rho, u, v, p;
  if (!cons_to_prim(s, g, rho, u, v, p)) return false;
  f.rho = rho;
  f.un = u * nx + v * ny;
  f.ut = -u * ny + v * nx;
  f.p = p;
  f.E = s[3];
  f.a = sqrt(g * p / rho);
  return true;
}

__device__ __forceinline__ void frame_flux(const Frame& f, double* o) {  // euler.cpp:26-28
  o[0] = f.rho * f.un;
  o[1] = f.rho * f.un * f.un + f.p;
  o[2] = f.rho * f.un * f.ut;
  o[3] = (f.E + f.p) * f.un;
}
__device__ __forceinline__ void frame_cons(const Frame& f, double* o) {  // euler.cpp:30-32
  o[0] = f.rho;
  o[1] = f.rho * f.un;
  o[2] = f.rho * f.ut;
  o[3] = f.E;
}
__device__ __forceinline__ void rotate_out(const double* ff, double nx, double ny, double* o) {  // :34-36
  o[0] = ff[0];
  o[1] = ff[1] * nx - ff[2] * ny;
  o[2] = ff[1] * ny + ff[2] * nx;
  o[3] = ff[3];
}

// hllc_flux (euler.cpp:40-69) when hll == false, hll_flux (euler.cpp:71-89)
// otherwise. Returns false where cons_to_prim throws NonPhysicalError.
__device__ __forceinline__ bool riemann_flux(bool hll, const double* UL, const double* UR, double nx, double ny,
                                             double g, double* out) {
  Frame L, R;
  if (!rotate_in(UL, nx, ny, g, L)) return false;
  if (!rotate_in(UR, nx, ny, g, R)) return false;
  const double SL = smin(L.un - L.a, R.un - R.a);
  const double SR = smax(L.un + L.a, R.un + R.a);
  double ff[4];
  if (SL >= 0.0) {
    frame_flux(L, ff);
  } else if (SR <= 0.0) {
    frame_flux(R, ff);
  } else if (!hll) {
    const double dL = L.rho * (SL - L.un);
    const double dR = R.rho * (SR - R.un);
    const double Sstar = (R.p - L.p + L.un * dL - R.un * dR) / (dL - dR);
    const bool left = Sstar >= 0.0;
    const Frame& K = left ? L : R;
    const double SK = left ? SL : SR;
    double WK[4], FK[4], Ws[4];
    frame_cons(K, WK);
    frame_flux(K, FK);
    const double coef = K.rho * (SK - K.un) / (SK - Sstar);
    Ws[0] = coef;
    Ws[1] = coef * Sstar;
    Ws[2] = coef * K.ut;
    Ws[3] = coef * (WK[3] / K.rho + (Sstar - K.un) * (Sstar + K.p / (K.rho * (SK - K.un))));
#pragma unroll
    for (int v = 0; v < NV; ++v) ff[v] = FK[v] + SK * (Ws[v] - WK[v]);
  } else {
    double FL[4], FR[4], WL[4], WR[4];
    frame_flux(L, FL);
    frame_flux(R, FR);
    frame_cons(L, WL);
    frame_cons(R, WR);
#pragma unroll
    for (int v = 0; v < NV; ++v) ff[v] = (SR * FL[v] - SL * FR[v] + SL * SR * (WR[v] - WL[v])) / (SR - SL);
  }
  rotate_out(ff, nx, ny, out);
  return true;
}

// mirror_state (euler.hpp:67-70)
__device__ __forceinline__ void mirror_state(const double* s, double nx, double ny, double* o) {
  const double mn = s[1] * nx + s[2] * ny;
  o[0] = s[0];
  o[1] = s[1] - 2.0 * mn * nx;
  o[2] = s[2] - 2.0 * mn * ny;
  o[3] = s[3];
}

struct MarginParams {
  double alpha_m, beta_m, alpha_w, beta_w, kappa, deact_n;
};

// compute_margins (detector.cpp:18-24)
__device__ __forceinline__ void compute_margins(const MarginParams& m, double du, double& dm, double& dw) {
  dm = smax(m.alpha_m, m.beta_m * du);
  const double sgn = (m.beta_w > 0.0) ? 1.0 : (m.beta_w < 0.0 ? -1.0 : 0.0);
  dw = sgn * smax(m.alpha_w, fabs(m.beta_w * du));
}

// classify_violation (detector.cpp:26-30) as a severity 0/1/2
__device__ __forceinline__ int violation_severity(double v, double dm, double dw) {
  if (v > dm) return 2;
  if (v > dw) return 1;
  return 0;
}

// x^b for the CWENOZ tau (reconstruct.cpp:135). b == 4 (the default) and
// b == 2 are evaluated correctly rounded through an exact double-double
// square; other exponents use CUDA's pow (<= 2 ulp). glibc's pow is within
// 0.52 ulp, so results agree with the reference to 1 ulp (not bit-exact).
__device__ __forceinline__ double tau_pow(double x, double b) {
  if (b == 4.0) {
    const double h = x * x;
    const double l = __fma_rn(x, x, -h);
    const double H = h * h;
    const double L = __fma_rn(h, h, -H);
    const double cross = 2.0 * h * l;
    return H + (L + cross + l * l);
  }
  if (b == 2.0) return x * x;
  if (b == 1.0) return x;
  return pow(x, b);
}

// limiter_barth_jespersen (reconstruct.cpp:59-71), one q at a time
__device__ __forceinline__ double bj_update(double theta, double u0, double umin, double umax, double uq) {
  const double d = uq - u0;
  if (d > 0.0)
    theta = smin(theta, smin(1.0, (umax - u0) / d));
  else if (d < 0.0)
    theta = smin(theta, smin(1.0, (umin - u0) / d));
  return theta;
}

// limiter_venkatakrishnan (reconstruct.cpp:73-86), one q at a time
__device__ __forceinline__ double venkat_update(double theta, double u0, double umin, double umax, double uq,
                                                double eps2) {
  const double dm = uq - u0;
  if (dm == 0.0) return theta;
  const double dp = (dm > 0.0) ? (umax - u0) : (umin - u0);
  const double num = (dp * dp + eps2) * dm + 2.0 * dm * dm * dp;
  const double den = dm * (dp * dp + 2.0 * dm * dm + dm * dp + eps2);
  const double phi = (den != 0.0) ? num / den : 1.0;
  const double cl = phi < 0.0 ? 0.0 : (1.0 < phi ? 1.0 : phi);  // std::clamp(phi, 0, 1)
  return smin(theta, cl);
}

}  // namespace ucfvb
