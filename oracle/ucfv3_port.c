/*
 * ORACLE TEST INFRASTRUCTURE -- not product code. Only tests/, the smoke
 * check and bench.py's CPU legs load this library (as the checker).
 *
 * Plain-C restatement of the reference's per-stage hot path in THREE
 * dimensions with five conserved variables (rho, rho u, rho v, rho w, E),
 * over the flat views of include/ucfvb3.h. The reference (/root/reference/
 * proj) is 2D only, so this restatement is "parity unpinned" for 3D: each
 * function is the reference's 2D function with the dimension changed, in the
 * reference's operation order (built with -ffp-contract=off):
 *
 *   compute_residual    solver.cpp:316-379
 *   solve_dofs          reconstruct.cpp:9-28          (K x M, 5 accumulators)
 *   evaluate_cell       solver.cpp:76-89, reconstruct.hpp:26-36
 *   classify_cells      solver.cpp:113-149            (checked vars rho, E = 0, 4)
 *   spread_flags        detector.cpp:37-53
 *   apply_troubled      solver.cpp:151-227            (nf directional r=1 solves, 3 dofs each)
 *   cwenoz_blend_scalar reconstruct.cpp:99-150        (SI of a zero-padded r=1 vector: 3x3 block of OI)
 *   limiters            reconstruct.cpp:59-86
 *   fallback_check      solver.cpp:229-264            (pressure with three momenta)
 *   assemble_fluxes     solver.cpp:266-314            (per-qp normal and weight x area element)
 *   hllc_flux/hll_flux  euler.cpp:40-89               (Cartesian form: star momentum coef*(S* n + u_t))
 *   max_stable_dt       solver.cpp:103-111            (|u|+|v|+|w|+a)
 *   SSP-RK3 / SSPRK(5,4) time_integrator.cpp:31-74
 * The 2D restatement of the same functions (oracle/ucfv_port.c) is pinned
 * bit-exactly to the compiled reference.
 *
 * Arithmetic: the 2D path keeps the reference's unfused x86-64 arithmetic
 * (no FMA) for bit parity. The 3D discretisation has no reference
 * arithmetic to match, so its least-squares solves, polynomial
 * evaluations and the K x K smoothness-indicator form (the contractions)
 * accumulate with fused multiply-adds, acc = fma(a, b, acc) in the same term
 * order -- one rounding
 * per term and half the fp64 instructions on the device; every other
 * operation is unfused as in 2D. C's fma() and CUDA's __fma_rn are both the
 * correctly rounded fused operation, so the device matches this restatement
 * bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ucfvb3.h"

#define NV 5

static _Thread_local char g_err[512];
const char* port3_last_error(void) { return g_err; }

static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }

typedef struct port3 {
  ucfvb3_mesh_view m;
  ucfvb3_stencil_view s;
  ucfvb_options o;
  int n, nF, nf, nq, Q, K, M, MD;
  double *dofs, *fp, *ff, *bounds, *thr, *eps2;
  uint8_t *labels, *step_labels;
  int64_t bad_face;
  double *ua, *ub, *uc, *ud, *rhs, *rhs3;
} port3;

/* ---- euler.hpp in 3D ------------------------------------------------------ */
static inline double pressure3(const double* s, double g) {
  return (g - 1.0) * (s[4] - 0.5 * (s[1] * s[1] + s[2] * s[2] + s[3] * s[3]) / s[0]);
}
static inline int is_physical3(const double* s, double g) { return s[0] > 0.0 && pressure3(s, g) > 0.0; }
static inline int cons_to_prim3(const double* s, double g, double* w) {
  if (!(s[0] > 0.0)) return 1;
  const double u = s[1] / s[0], v = s[2] / s[0], ww = s[3] / s[0];
  const double p = (g - 1.0) * (s[4] - 0.5 * s[0] * (u * u + v * v + ww * ww));
  if (!(p > 0.0)) return 2;
  w[0] = s[0], w[1] = u, w[2] = v, w[3] = ww, w[4] = p;
  return 0;
}

typedef struct { double rho, u, v, w, un, p, E, a; } state3_t;

static int prep(const double* s, const double* n, double g, state3_t* f) {
  double w[5];
  const int rc = cons_to_prim3(s, g, w);
  if (rc) return rc;
  f->rho = w[0], f->u = w[1], f->v = w[2], f->w = w[3], f->p = w[4];
  f->un = w[1] * n[0] + w[2] * n[1] + w[3] * n[2];
  f->E = s[4];
  f->a = sqrt(g * w[4] / w[0]);
  return 0;
}
static inline void phys_flux(const state3_t* f, const double* n, double* o) {
  o[0] = f->rho * f->un;
  o[1] = f->rho * f->u * f->un + f->p * n[0];
  o[2] = f->rho * f->v * f->un + f->p * n[1];
  o[3] = f->rho * f->w * f->un + f->p * n[2];
  o[4] = (f->E + f->p) * f->un;
}
static inline void cons_of(const state3_t* f, double* o) {
  o[0] = f->rho, o[1] = f->rho * f->u, o[2] = f->rho * f->v, o[3] = f->rho * f->w, o[4] = f->E;
}

/* hllc_flux / hll_flux (euler.cpp:40-89) in Cartesian form */
static int riemann3(int kind, const double* UL, const double* UR, const double* n, double g, double* out) {
  state3_t L, R;
  if (prep(UL, n, g, &L) || prep(UR, n, g, &R)) return 1;
  const double SL = smin(L.un - L.a, R.un - R.a);
  const double SR = smax(L.un + L.a, R.un + R.a);
  if (SL >= 0.0) {
    phys_flux(&L, n, out);
    return 0;
  }
  if (SR <= 0.0) {
    phys_flux(&R, n, out);
    return 0;
  }
  if (kind == UCFVB_HLLC) {
    const double dL = L.rho * (SL - L.un);
    const double dR = R.rho * (SR - R.un);
    const double Ss = (R.p - L.p + L.un * dL - R.un * dR) / (dL - dR);
    const state3_t* K = (Ss >= 0.0) ? &L : &R;
    const double SK = (Ss >= 0.0) ? SL : SR;
    double WK[5], FK[5], Ws[5];
    cons_of(K, WK);
    phys_flux(K, n, FK);
    const double coef = K->rho * (SK - K->un) / (SK - Ss);
    Ws[0] = coef;
    Ws[1] = coef * (Ss * n[0] + (K->u - K->un * n[0]));
    Ws[2] = coef * (Ss * n[1] + (K->v - K->un * n[1]));
    Ws[3] = coef * (Ss * n[2] + (K->w - K->un * n[2]));
    Ws[4] = coef * (WK[4] / K->rho + (Ss - K->un) * (Ss + K->p / (K->rho * (SK - K->un))));
    for (int v = 0; v < NV; ++v) out[v] = FK[v] + SK * (Ws[v] - WK[v]);
  } else {
    double FL[5], FR[5], WL[5], WR[5];
    phys_flux(&L, n, FL);
    phys_flux(&R, n, FR);
    cons_of(&L, WL);
    cons_of(&R, WR);
    for (int v = 0; v < NV; ++v) out[v] = (SR * FL[v] - SL * FR[v] + SL * SR * (WR[v] - WL[v])) / (SR - SL);
  }
  return 0;
}

/* ---- detector.cpp ------------------------------------------------------------ */
static void compute_margins(const ucfvb_margins* m, double du, double* dm, double* dw) {
  *dm = smax(m->alpha_m, m->beta_m * du);
  const double sgn = (m->beta_w > 0.0) ? 1.0 : (m->beta_w < 0.0 ? -1.0 : 0.0);
  *dw = sgn * smax(m->alpha_w, fabs(m->beta_w * du));
}
static int classify_violation(double v, double dm, double dw) {
  if (v > dm) return UCFVB_SCHEME_MUSCL;
  if (v > dw) return UCFVB_SCHEME_CWENOZ;
  return UCFVB_SCHEME_LINEAR;
}
static inline int severity(int s) { return s == 0 ? 0 : (s == 1 ? 1 : 2); }

/* ---- accessors ----------------------------------------------------------------- */
static inline int opi(const port3* P, int c) { return P->s.op_index[c]; }
static inline const int32_t* central(const port3* P, int c) { return &P->s.central[(int64_t)c * (P->M + 1)]; }
static inline const int32_t* nbrs(const port3* P, int c) { return &P->m.cell_nbr[(int64_t)c * P->nf]; }
static inline double* slot_ptr(port3* P, int slot) { return &P->fp[(int64_t)slot * NV]; }

/* solve_dofs (reconstruct.cpp:9-28) */
static void solve_dofs(const port3* P, int c, const double* u, double* dofs) {
  const int K = P->K, M = P->M;
  const int32_t* st = central(P, c);
  const double* u0 = &u[(int64_t)st[0] * NV];
  const double* pinv = &P->s.pinv[(int64_t)opi(P, c) * K * M];
  for (int k = 0; k < K; ++k) {
    const double* row = &pinv[k * M];
    double s[NV] = {0, 0, 0, 0, 0};
    for (int m = 0; m < M; ++m) {
      const double* um = &u[(int64_t)st[m + 1] * NV];
      const double w = row[m];
      for (int v = 0; v < NV; ++v) s[v] = fma(w, um[v] - u0[v], s[v]);
    }
    for (int v = 0; v < NV; ++v) dofs[k * NV + v] = s[v];
  }
}

/* evaluate_cell (solver.cpp:76-89) with eval_poly (reconstruct.hpp:26-36) over
 * the first ke dofs (ke = K; MUSCL's limited r = 1 polynomial passes ke = 3:
 * its dofs k >= 3 are zero and those terms are left out) */
static void evaluate_cell_n(port3* P, const double* u, int c, const double* dofs, int ke) {
  const int K = P->K, Q = P->Q;
  const double* phi = &P->s.phi[(int64_t)opi(P, c) * Q * K];
  const int32_t* slots = &P->s.qp_slot[(int64_t)c * Q];
  const double* u0 = &u[(int64_t)c * NV];
  for (int q = 0; q < Q; ++q) {
    double out[NV];
    for (int v = 0; v < NV; ++v) out[v] = u0[v];
    for (int k = 0; k < ke; ++k) {
      const double p = phi[q * K + k];
      for (int v = 0; v < NV; ++v) out[v] = fma(dofs[k * NV + v], p, out[v]);
    }
    memcpy(slot_ptr(P, slots[q]), out, sizeof out);
  }
}
static void evaluate_cell(port3* P, const double* u, int c, const double* dofs) { evaluate_cell_n(P, u, c, dofs, P->K); }
static void evaluate_constant(port3* P, const double* u, int c) {
  const int32_t* slots = &P->s.qp_slot[(int64_t)c * P->Q];
  for (int q = 0; q < P->Q; ++q) memcpy(slot_ptr(P, slots[q]), &u[(int64_t)c * NV], sizeof(double) * NV);
}

static const int kChecked[2] = {0, 4};

static void cell_bounds(const port3* P, const double* u, int c, double* bnd) {
  for (int t = 0; t < 2; ++t) {
    const int v = kChecked[t];
    double lo = u[(int64_t)c * NV + v], hi = lo;
    for (int i = 0; i < P->nf; ++i) {
      const double x = u[(int64_t)nbrs(P, c)[i] * NV + v];
      lo = smin(lo, x);
      hi = smax(hi, x);
    }
    bnd[2 * t] = lo;
    bnd[2 * t + 1] = hi;
  }
}

/* classify_cells (solver.cpp:113-149) + spread_flags (detector.cpp:37-53) */
static void classify_cells(port3* P, const double* u) {
  const int n = P->n;
  uint8_t* raw = (uint8_t*)malloc((size_t)n);
  for (int c = 0; c < n; ++c) {
    double* bnd = &P->bounds[(int64_t)c * 4];
    cell_bounds(P, u, c, bnd);
    const int32_t* slots = &P->s.qp_slot[(int64_t)c * P->Q];
    int sev = 0;
    for (int t = 0; t < 2 && sev < 2; ++t) {
      const double du = bnd[2 * t + 1] - bnd[2 * t];
      if (P->o.margins.kappa > 0.0 && du < P->thr[c]) continue; /* deactivate_smooth, detector.cpp:32-35 */
      double v = -1e300;
      for (int q = 0; q < P->Q; ++q) {
        const double uq = slot_ptr(P, slots[q])[kChecked[t]];
        v = smax(v, smax(bnd[2 * t] - uq, uq - bnd[2 * t + 1]));
      }
      double dm, dw;
      compute_margins(&P->o.margins, du, &dm, &dw);
      const int vs = severity(classify_violation(v, dm, dw));
      sev = vs > sev ? vs : sev;
    }
    raw[c] = (uint8_t)(sev == 0 ? UCFVB_SCHEME_LINEAR : (sev == 1 ? UCFVB_SCHEME_CWENOZ : UCFVB_SCHEME_MUSCL));
  }
  memcpy(P->labels, raw, (size_t)n);
  for (int c = 0; c < n; ++c) {
    const int s = raw[c];
    if (severity(s) == 0) continue;
    for (int i = 0; i < P->nf; ++i) {
      const int nb = nbrs(P, c)[i];
      if (severity(P->labels[nb]) < severity(s)) P->labels[nb] = (uint8_t)s;
    }
  }
  free(raw);
}

/* limiter_barth_jespersen / limiter_venkatakrishnan (reconstruct.cpp:59-86) */
static double limiter_bj(double u0, double umin, double umax, const double* q, int nq) {
  double theta = 1.0;
  for (int i = 0; i < nq; ++i) {
    const double d = q[i] - u0;
    if (d > 0.0)
      theta = smin(theta, smin(1.0, (umax - u0) / d));
    else if (d < 0.0)
      theta = smin(theta, smin(1.0, (umin - u0) / d));
  }
  return smax(theta, 0.0);
}
static double limiter_venkat(double u0, double umin, double umax, const double* q, int nq, double eps2) {
  double theta = 1.0;
  for (int i = 0; i < nq; ++i) {
    const double dm = q[i] - u0;
    if (dm == 0.0) continue;
    const double dp = (dm > 0.0) ? (umax - u0) : (umin - u0);
    const double num = (dp * dp + eps2) * dm + 2.0 * dm * dm * dp;
    const double den = dm * (dp * dp + 2.0 * dm * dm + dm * dp + eps2);
    double phi = (den != 0.0) ? num / den : 1.0;
    phi = phi < 0.0 ? 0.0 : (1.0 < phi ? 1.0 : phi); /* std::clamp */
    theta = smin(theta, phi);
  }
  return theta;
}

/* smoothness_indicator (reconstruct.cpp:88-97): row then dot, each a fused
 * accumulation in the reference's order (the 3D contraction rule of the header) */
static double smoothness_indicator(const double* oi, const double* a, int K) {
  double s = 0.0;
  for (int k = 0; k < K; ++k) {
    const double* row = &oi[(int64_t)k * K];
    double t = 0.0;
    for (int q = 0; q < K; ++q) t = fma(row[q], a[q], t);
    s = fma(a[k], t, s);
  }
  return s;
}

/* cwenoz_blend_scalar (reconstruct.cpp:99-150); dir is [nd][3] */
static int cwenoz_blend3(const double* oi, int K, const double* cen, const double (*dir)[3], int nd, double lambda1p,
                         double eps, double b, double* blended) {
  if (!(lambda1p > 1.0)) {
    snprintf(g_err, sizeof g_err, "cwenoz: central linear weight lambda1' must exceed 1");
    return UCFVB_INVALID;
  }
  const int st = nd + 1;
  double lambda[8], si[8], omega[8], p1[128];
  lambda[0] = 1.0 - 1.0 / lambda1p;
  for (int s = 1; s < st; ++s) lambda[s] = (1.0 - lambda[0]) / (st - 1);
  for (int k = 0; k < K; ++k) p1[k] = cen[k];
  for (int s = 1; s < st; ++s) {
    p1[0] -= lambda[s] * dir[s - 1][0];
    p1[1] -= lambda[s] * dir[s - 1][1];
    p1[2] -= lambda[s] * dir[s - 1][2];
  }
  for (int k = 0; k < K; ++k) p1[k] /= lambda[0];
  si[0] = smoothness_indicator(oi, p1, K);
  for (int s = 1; s < st; ++s) {
    const double a0 = dir[s - 1][0], a1 = dir[s - 1][1], a2 = dir[s - 1][2];
    double t = oi[0] * a0 * a0;
    t = t + (oi[1] + oi[K]) * a0 * a1;
    t = t + (oi[2] + oi[2 * K]) * a0 * a2;
    t = t + oi[K + 1] * a1 * a1;
    t = t + (oi[K + 2] + oi[2 * K + 1]) * a1 * a2;
    t = t + oi[2 * K + 2] * a2 * a2;
    si[s] = t;
  }
  double tau = 0.0;
  for (int s = 1; s < st; ++s) tau += fabs(si[s] - si[0]);
  tau /= (st - 1);
  tau = pow(tau, b);
  double wsum = 0.0;
  for (int s = 0; s < st; ++s) {
    omega[s] = lambda[s] * (1.0 + tau / (eps + si[s]));
    wsum += omega[s];
  }
  for (int s = 0; s < st; ++s) omega[s] /= wsum;
  for (int k = 0; k < K; ++k) blended[k] = omega[0] * p1[k];
  for (int s = 1; s < st; ++s) {
    blended[0] += omega[s] * dir[s - 1][0];
    blended[1] += omega[s] * dir[s - 1][1];
    blended[2] += omega[s] * dir[s - 1][2];
  }
  return 0;
}

/* apply_troubled (solver.cpp:151-227) */
static int apply_troubled(port3* P, const double* u) {
  const int K = P->K, M = P->M, MD = P->MD, nf = P->nf, Q = P->Q;
  double dir[8][NV][3], dd[8][3], cen[128], bl[128], lin[3][NV], qv[64 * NV], vv[64];
  for (int c = 0; c < P->n; ++c) {
    const int lab = P->labels[c];
    if (lab == UCFVB_SCHEME_LINEAR) continue;
    double* dofs = &P->dofs[(int64_t)c * K * NV];
    const int op = opi(P, c);
    const int32_t* st = central(P, c);
    const double* u0 = &u[(int64_t)c * NV];
    if (lab == UCFVB_SCHEME_CWENOZ) {
      for (int s = 0; s < nf; ++s) { /* solve_dofs_directional (reconstruct.cpp:43-57) */
        const int32_t* mem = &P->s.dir_members[((int64_t)op * nf + s) * MD];
        const double* pd = &P->s.pinv_dir[(((int64_t)op * nf + s) * 3) * MD];
        for (int k = 0; k < 3; ++k)
          for (int v = 0; v < NV; ++v) {
            double acc = 0.0;
            for (int m = 0; m < MD; ++m) acc = fma(pd[k * MD + m], u[(int64_t)st[mem[m]] * NV + v] - u0[v], acc);
            dir[s][v][k] = acc;
          }
      }
      const double* oi = &P->s.oi[(int64_t)op * K * K];
      for (int v = 0; v < NV; ++v) {
        for (int k = 0; k < K; ++k) cen[k] = dofs[k * NV + v];
        for (int s = 0; s < nf; ++s)
          for (int k = 0; k < 3; ++k) dd[s][k] = dir[s][v][k];
        const int rc = cwenoz_blend3(oi, K, cen, (const double(*)[3])dd, nf, P->o.lambda1p, P->o.weno_eps, P->o.weno_b,
                                     bl);
        if (rc) return rc;
        for (int k = 0; k < K; ++k) dofs[k * NV + v] = bl[k];
      }
      evaluate_cell(P, u, c, dofs);
    } else if (lab == UCFVB_SCHEME_MUSCL) {
      const double* pl = &P->s.pinv_lin[(int64_t)op * 3 * M];
      for (int k = 0; k < 3; ++k) /* solve_dofs_linear (reconstruct.cpp:30-41) */
        for (int v = 0; v < NV; ++v) {
          double s = 0.0;
          for (int m = 0; m < M; ++m) s = fma(pl[k * M + m], u[(int64_t)st[m + 1] * NV + v] - u0[v], s);
          lin[k][v] = s;
        }
      const double* phi = &P->s.phi[(int64_t)op * Q * K];
      for (int q = 0; q < Q; ++q) {
        const double p0 = phi[q * K], p1 = phi[q * K + 1], p2 = phi[q * K + 2];
        for (int v = 0; v < NV; ++v) qv[q * NV + v] = fma(lin[2][v], p2, fma(lin[1][v], p1, fma(lin[0][v], p0, u0[v])));
      }
      for (int v = 0; v < NV; ++v) {
        double lo = u0[v], hi = u0[v];
        for (int i = 0; i < nf; ++i) {
          const double x = u[(int64_t)nbrs(P, c)[i] * NV + v];
          lo = smin(lo, x);
          hi = smax(hi, x);
        }
        for (int q = 0; q < Q; ++q) vv[q] = qv[q * NV + v];
        const double th = (P->o.limiter == UCFVB_BARTH_JESPERSEN) ? limiter_bj(u0[v], lo, hi, vv, Q)
                                                                  : limiter_venkat(u0[v], lo, hi, vv, Q, P->eps2[c]);
        for (int k = 0; k < 3; ++k) dofs[k * NV + v] = th * lin[k][v];
        for (int k = 3; k < K; ++k) dofs[k * NV + v] = 0.0;
      }
      evaluate_cell_n(P, u, c, dofs, 3);
    } else {
      for (int k = 0; k < K * NV; ++k) dofs[k] = 0.0;
      evaluate_constant(P, u, c);
    }
  }
  return 0;
}

/* fallback_check (solver.cpp:229-264) */
static void fallback_check(port3* P, const double* u) {
  const int K = P->K;
  for (int c = 0; c < P->n; ++c) {
    const int32_t* slots = &P->s.qp_slot[(int64_t)c * P->Q];
    const double* bnd = &P->bounds[(int64_t)c * 4];
    int demote = 0;
    for (int q = 0; q < P->Q && !demote; ++q)
      if (!is_physical3(slot_ptr(P, slots[q]), P->o.gamma)) demote = 1;
    for (int t = 0; t < 2 && !demote; ++t) {
      const double du = bnd[2 * t + 1] - bnd[2 * t];
      double dm, dw;
      compute_margins(&P->o.margins, du, &dm, &dw);
      for (int q = 0; q < P->Q; ++q) {
        const double uq = slot_ptr(P, slots[q])[kChecked[t]];
        if (smax(bnd[2 * t] - uq, uq - bnd[2 * t + 1]) > dm) {
          demote = 1;
          break;
        }
      }
    }
    if (demote) {
      P->labels[c] = UCFVB_SCHEME_FIRST;
      double* dofs = &P->dofs[(int64_t)c * K * NV];
      for (int k = 0; k < K * NV; ++k) dofs[k] = 0.0;
      evaluate_constant(P, u, c);
    }
  }
}

/* assemble_fluxes (solver.cpp:266-314) */
static int assemble_fluxes(port3* P, double* out) {
  const int nq = P->nq;
  for (int f = 0; f < P->nF; ++f) {
    double total[NV] = {0, 0, 0, 0, 0};
    /* subdomain boundary faces (decompose3.cpp: both sides the same halo cell)
     * carry no flux; they never touch an owned residual */
    if (P->m.face_left[f] == P->m.face_right[f]) {
      memcpy(&P->ff[(int64_t)f * NV], total, sizeof total);
      continue;
    }
    for (int q = 0; q < nq; ++q) {
      const double* UL = slot_ptr(P, (f * nq + q) * 2);
      const double* UR = slot_ptr(P, (f * nq + q) * 2 + 1);
      double fl[NV];
      if (riemann3(P->o.riemann, UL, UR, &P->m.face_normal[((int64_t)f * nq + q) * 3], P->o.gamma, fl)) {
        P->bad_face = f;
        snprintf(g_err, sizeof g_err, "non-physical state at face %d", f);
        return UCFVB_NONPHYSICAL;
      }
      const double w = P->m.face_wa[(int64_t)f * nq + q];
      for (int v = 0; v < NV; ++v) total[v] += w * fl[v];
    }
    memcpy(&P->ff[(int64_t)f * NV], total, sizeof total);
  }
  for (int c = 0; c < P->n; ++c) {
    double acc[NV] = {0, 0, 0, 0, 0};
    for (int i = 0; i < P->nf; ++i) {
      const int64_t j = (int64_t)c * P->nf + i;
      const double sgn = P->m.cell_side[j] == 0 ? 1.0 : -1.0;
      const double* fl = &P->ff[(int64_t)P->m.cell_faces[j] * NV];
      for (int v = 0; v < NV; ++v) acc[v] += sgn * fl[v];
    }
    const double inv_vol = 1.0 / P->m.cell_volume[c];
    for (int v = 0; v < NV; ++v) out[(int64_t)c * NV + v] = -acc[v] * inv_vol;
  }
  return 0;
}

/* compute_residual (solver.cpp:316-379) */
/* one stage; `first` = first stage of a step (stage_is_first_, solver.cpp:371-374):
 * with detect_every_stage = 0 the later stages keep the labels and only
 * refresh the bounds (solver.cpp:343-361) */
static int stage3(port3* P, const double* u, double t, double* out, int first) {
  (void)t;
  const int n = P->n, K = P->K, mode = P->o.mode;
  if (mode == UCFVB_FIRST) memset(P->labels, UCFVB_SCHEME_FIRST, (size_t)n);
  if (mode == UCFVB_MUSCL) memset(P->labels, UCFVB_SCHEME_MUSCL, (size_t)n);
  if (mode == UCFVB_CWENOZ) memset(P->labels, UCFVB_SCHEME_CWENOZ, (size_t)n);
  if (mode == UCFVB_LINEAR || mode == UCFVB_CWENOZ || mode == UCFVB_HYBRID)
    for (int c = 0; c < n; ++c) {
      double* dofs = &P->dofs[(int64_t)c * K * NV];
      solve_dofs(P, c, u, dofs);
      if (mode != UCFVB_CWENOZ) evaluate_cell(P, u, c, dofs);
    }
  if (mode == UCFVB_HYBRID) {
    if (first || P->o.detect_every_stage)
      classify_cells(P, u);
    else
      for (int c = 0; c < n; ++c) cell_bounds(P, u, c, &P->bounds[(int64_t)c * 4]);
  }
  if (mode != UCFVB_LINEAR) {
    const int rc = apply_troubled(P, u);
    if (rc) return rc;
  }
  if (mode == UCFVB_HYBRID) fallback_check(P, u);
  if (first) memcpy(P->step_labels, P->labels, (size_t)n);
  return assemble_fluxes(P, out);
}

/* compute_residual (solver.cpp:316-379) called on its own: a first stage */
int port3_compute_residual(port3* P, const double* u, double t, double* out) { return stage3(P, u, t, out, 1); }

/* max_stable_dt (solver.cpp:103-111) */
int port3_max_stable_dt(port3* P, const double* u, double* out) {
  double dt = 1e300;
  for (int c = 0; c < P->n; ++c) {
    double w[5];
    if (cons_to_prim3(&u[(int64_t)c * NV], P->o.gamma, w)) {
      snprintf(g_err, sizeof g_err, "non-physical state in cell %d", c);
      return UCFVB_NONPHYSICAL;
    }
    const double speed = fabs(w[1]) + fabs(w[2]) + fabs(w[3]) + sqrt(P->o.gamma * w[4] / w[0]);
    dt = smin(dt, P->m.cell_h[c] / speed);
  }
  *out = P->o.cfl * dt;
  return 0;
}

static void combine2(int64_t n, double* out, double wa, const double* ua, double wb, const double* ub, double wr,
                     const double* r, double dt) {
  const double wrdt = wr * dt;
  for (int64_t i = 0; i < NV * n; ++i) out[i] = wa * ua[i] + wb * ub[i] + wrdt * r[i];
}

/* ssp_rk4_step (time_integrator.cpp:42-74) or SSP-RK3 (Shu-Osher, stage times t, t+dt, t+dt/2) */
int port3_advance(port3* P, double* u, double dt, double t, int rk) {
  const int64_t n = P->n;
  int rc;
  if (rk == UCFVB_RK3) {
    if ((rc = stage3(P, u, t, P->rhs, 1))) return rc;
    combine2(n, P->ua, 1.0, u, 0.0, u, 1.0, P->rhs, dt);
    if ((rc = stage3(P, P->ua, t + dt, P->rhs, 0))) return rc;
    combine2(n, P->ub, 0.75, u, 0.25, P->ua, 0.25, P->rhs, dt);
    if ((rc = stage3(P, P->ub, t + 0.5 * dt, P->rhs, 0))) return rc;
    combine2(n, u, 1.0 / 3.0, u, 2.0 / 3.0, P->ub, 2.0 / 3.0, P->rhs, dt);
    return 0;
  }
  const double a10 = 0.391752226571890;
  const double b20 = 0.444370493651235, b21 = 0.555629506348765, a21 = 0.368410593050371;
  const double b30 = 0.620101851488403, b32 = 0.379898148511597, a32 = 0.251891774271694;
  const double b40 = 0.178079954393132, b43 = 0.821920045606868, a43 = 0.544974750228521;
  const double c52 = 0.517231671970585, c53 = 0.096059710526147, a53 = 0.063692468666290;
  const double c54 = 0.386708617503269, a54 = 0.226007483236906;
  if ((rc = stage3(P, u, t, P->rhs, 1))) return rc;
  combine2(n, P->ua, 1.0, u, 0.0, u, a10, P->rhs, dt);
  if ((rc = stage3(P, P->ua, t, P->rhs, 0))) return rc;
  combine2(n, P->ub, b20, u, b21, P->ua, a21, P->rhs, dt);
  if ((rc = stage3(P, P->ub, t, P->rhs, 0))) return rc;
  combine2(n, P->uc, b30, u, b32, P->ub, a32, P->rhs, dt);
  if ((rc = stage3(P, P->uc, t, P->rhs3, 0))) return rc;
  combine2(n, P->ud, b40, u, b43, P->uc, a43, P->rhs3, dt);
  if ((rc = stage3(P, P->ud, t, P->rhs, 0))) return rc;
  for (int64_t i = 0; i < NV * n; ++i)
    u[i] = c52 * P->ub[i] + c53 * P->uc[i] + a53 * dt * P->rhs3[i] + c54 * P->ud[i] + a54 * dt * P->rhs[i];
  return 0;
}

int port3_create(const ucfvb3_mesh_view* m, const ucfvb3_stencil_view* s, const ucfvb_options* o, port3** out) {
  if (m->n_cells != s->n_cells || m->nf != s->nf || m->nq != s->nq) {
    snprintf(g_err, sizeof g_err, "port3: stencils do not match the mesh");
    return UCFVB_INVALID;
  }
  if (s->K > 120 || m->nf > 7 || s->Q > 64) {
    snprintf(g_err, sizeof g_err, "port3: sizes out of range");
    return UCFVB_INVALID;
  }
  port3* P = (port3*)calloc(1, sizeof *P);
  P->m = *m;
  P->s = *s;
  P->o = *o;
  P->n = m->n_cells, P->nF = m->n_faces, P->nf = m->nf, P->nq = m->nq, P->Q = s->Q;
  P->K = s->K, P->M = s->M, P->MD = s->MD;
  const int64_t n = P->n;
  P->dofs = (double*)calloc((size_t)n * P->K * NV, sizeof(double));
  P->fp = (double*)calloc((size_t)P->nF * P->nq * 2 * NV, sizeof(double));
  P->ff = (double*)calloc((size_t)P->nF * NV, sizeof(double));
  P->bounds = (double*)calloc((size_t)n * 4, sizeof(double));
  P->thr = (double*)calloc((size_t)n, sizeof(double));
  P->eps2 = (double*)calloc((size_t)n, sizeof(double));
  for (int64_t c = 0; c < n; ++c) {
    P->thr[c] = pow(o->margins.kappa * m->cell_h[c], o->margins.deact_n);
    P->eps2[c] = pow(o->venkat_kappa * m->cell_h[c], 3);
  }
  P->labels = (uint8_t*)calloc((size_t)n, 1);
  P->step_labels = (uint8_t*)calloc((size_t)n, 1);
  double** ws[] = {&P->ua, &P->ub, &P->uc, &P->ud, &P->rhs, &P->rhs3};
  for (int i = 0; i < 6; ++i) *ws[i] = (double*)calloc((size_t)n * NV, sizeof(double));
  P->bad_face = -1;
  *out = P;
  return 0;
}

void port3_free(port3* P) {
  if (!P) return;
  free(P->dofs); free(P->fp); free(P->ff); free(P->bounds); free(P->thr); free(P->eps2);
  free(P->labels); free(P->step_labels);
  free(P->ua); free(P->ub); free(P->uc); free(P->ud); free(P->rhs); free(P->rhs3);
  free(P);
}

void port3_get_labels(const port3* P, uint8_t* out, int step) { memcpy(out, step ? P->step_labels : P->labels, (size_t)P->n); }
void port3_get_face_values(const port3* P, double* out) {
  memcpy(out, P->fp, sizeof(double) * (size_t)P->nF * P->nq * 2 * NV);
}
void port3_get_dofs(const port3* P, double* out) { memcpy(out, P->dofs, sizeof(double) * (size_t)P->n * P->K * NV); }
int64_t port3_bad_face(const port3* P) { return P->bad_face; }
int port3_flux(const double* ul, const double* ur, const double* n, double g, int kind, double* out) {
  return riemann3(kind, ul, ur, n, g, out);
}
