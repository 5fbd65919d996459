/*
 * ORACLE TEST INFRASTRUCTURE -- not product code. Only tests/, the smoke
 * check and bench.py's CPU legs load this library (as the checker).
 *
 * Plain-C restatement of the reference's per-stage hot path over the flat
 * views of include/ucfvb.h. Every function names the reference lines it
 * restates; the arithmetic follows the reference's operation order (built
 * with -ffp-contract=off) so that it is bit-identical to the compiled
 * reference (pinned by tests/test_oracle_pin.py against oracle/_ref and
 * tests/golden/).
 *
 *   compute_residual   solver.cpp:316-379
 *   solve_dofs         reconstruct.cpp:9-28
 *   evaluate_cell      solver.cpp:76-89 (+ eval_poly reconstruct.hpp:26-36)
 *   classify_cells     solver.cpp:113-149, detector.cpp:18-35
 *   spread_flags       detector.cpp:37-53
 *   apply_troubled     solver.cpp:151-227, reconstruct.cpp:30-150
 *   fallback_check     solver.cpp:229-264, euler.hpp:30-36
 *   assemble_fluxes    solver.cpp:266-314, euler.cpp:1-89
 *   max_stable_dt      solver.cpp:103-111
 *   ssp_rk4_step       time_integrator.cpp:10-74 ; SSP-RK3 per oracle/ref_harness.cpp
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ucfvb.h"

#define NV 4

static _Thread_local char g_err[512];

/* std::min / std::max semantics: min(a,b) = (b < a) ? b : a */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }

typedef struct {
  int kind;
  double state[4];
} port_bc;

typedef struct port_solver {
  ucfvb_mesh_view m;
  ucfvb_stencil_view s;
  ucfvb_options o;
  int n, nf, nq, K;
  int* nb_ptr; /* face neighbours incl. periodic (mesh.cpp:19-30) */
  int* nb;
  port_bc* patch_bc;
  double* dofs;        /* n*K*4 */
  double* val_left;    /* nf*nq*4 */
  double* val_right;
  double* face_flux;   /* nf*4 */
  uint8_t* labels;
  uint8_t* step_labels;
  double* bounds;      /* n*4 */
  int stage_is_first;
  /* rk workspaces */
  double *ua, *ub, *uc, *ud, *rhs, *rhs3;
} port_solver;

const char* port_last_error(void) { return g_err; }

/* ---- euler.hpp --------------------------------------------------------- */
static inline double pressure(const double* s, double g) {
  return (g - 1.0) * (s[3] - 0.5 * (s[1] * s[1] + s[2] * s[2]) / s[0]); /* euler.hpp:30-32 */
}
static inline int is_physical(const double* s, double g) { /* euler.hpp:34-36 */
  return s[0] > 0.0 && pressure(s, g) > 0.0;
}
/* cons_to_prim (euler.hpp:38-45); returns 0 ok, 1 rho, 2 p */
static inline int cons_to_prim(const double* s, double g, double* w) {
  if (!(s[0] > 0.0)) return 1;
  const double u = s[1] / s[0];
  const double v = s[2] / s[0];
  const double p = (g - 1.0) * (s[3] - 0.5 * s[0] * (u * u + v * v));
  if (!(p > 0.0)) {
    w[3] = p;
    return 2;
  }
  w[0] = s[0];
  w[1] = u;
  w[2] = v;
  w[3] = p;
  return 0;
}

typedef struct { double rho, un, ut, p, E, a; } frame_t;

/* rotate_in (euler.cpp:13-23) */
static int rotate_in(const double* s, double nx, double ny, double g, frame_t* f, double* bad) {
  double w[4];
  const int rc = cons_to_prim(s, g, w);
  if (rc) {
    *bad = rc == 1 ? s[0] : w[3];
    return rc;
  }
  f->rho = w[0];
  f->un = w[1] * nx + w[2] * ny;
  f->ut = -w[1] * ny + w[2] * nx;
  f->p = w[3];
  f->E = s[3];
  f->a = sqrt(g * w[3] / w[0]);
  return 0;
}
static inline void frame_flux(const frame_t* f, double* o) { /* euler.cpp:26-28 */
  o[0] = f->rho * f->un;
  o[1] = f->rho * f->un * f->un + f->p;
  o[2] = f->rho * f->un * f->ut;
  o[3] = (f->E + f->p) * f->un;
}
static inline void frame_cons(const frame_t* f, double* o) { /* euler.cpp:30-32 */
  o[0] = f->rho;
  o[1] = f->rho * f->un;
  o[2] = f->rho * f->ut;
  o[3] = f->E;
}
static inline void rotate_out(const double* ff, double nx, double ny, double* o) { /* euler.cpp:34-36 */
  o[0] = ff[0];
  o[1] = ff[1] * nx - ff[2] * ny;
  o[2] = ff[1] * ny + ff[2] * nx;
  o[3] = ff[3];
}

/* hllc_flux (euler.cpp:40-69) / hll_flux (euler.cpp:71-89) */
static int riemann_flux(int kind, const double* UL, const double* UR, double nx, double ny, double g,
                        double* out, int* which, double* bad) {
  frame_t L, R;
  int rc = rotate_in(UL, nx, ny, g, &L, bad);
  if (rc) {
    *which = rc;
    return 1;
  }
  rc = rotate_in(UR, nx, ny, g, &R, bad);
  if (rc) {
    *which = rc;
    return 1;
  }
  const double SL = smin(L.un - L.a, R.un - R.a);
  const double SR = smax(L.un + L.a, R.un + R.a);
  double ff[4];
  if (SL >= 0.0) {
    frame_flux(&L, ff);
    rotate_out(ff, nx, ny, out);
    return 0;
  }
  if (SR <= 0.0) {
    frame_flux(&R, ff);
    rotate_out(ff, nx, ny, out);
    return 0;
  }
  if (kind == UCFVB_HLLC) {
    const double dL = L.rho * (SL - L.un);
    const double dR = R.rho * (SR - R.un);
    const double Sstar = (R.p - L.p + L.un * dL - R.un * dR) / (dL - dR);
    const frame_t* K = (Sstar >= 0.0) ? &L : &R;
    const double SK = (Sstar >= 0.0) ? SL : SR;
    double WK[4], FK[4], Ws[4];
    frame_cons(K, WK);
    frame_flux(K, FK);
    const double coef = K->rho * (SK - K->un) / (SK - Sstar);
    Ws[0] = coef;
    Ws[1] = coef * Sstar;
    Ws[2] = coef * K->ut;
    Ws[3] = coef * (WK[3] / K->rho + (Sstar - K->un) * (Sstar + K->p / (K->rho * (SK - K->un))));
    for (int v = 0; v < NV; ++v) ff[v] = FK[v] + SK * (Ws[v] - WK[v]);
  } else {
    double FL[4], FR[4], WL[4], WR[4];
    frame_flux(&L, FL);
    frame_flux(&R, FR);
    frame_cons(&L, WL);
    frame_cons(&R, WR);
    for (int v = 0; v < NV; ++v) ff[v] = (SR * FL[v] - SL * FR[v] + SL * SR * (WR[v] - WL[v])) / (SR - SL);
  }
  rotate_out(ff, nx, ny, out);
  return 0;
}

/* ---- detector.cpp ------------------------------------------------------ */
static void compute_margins(const ucfvb_margins* m, double du, double* dm, double* dw) {
  *dm = smax(m->alpha_m, m->beta_m * du); /* detector.cpp:18-24 */
  const double sgn = (m->beta_w > 0.0) ? 1.0 : (m->beta_w < 0.0 ? -1.0 : 0.0);
  *dw = sgn * smax(m->alpha_w, fabs(m->beta_w * du));
}
static int classify_violation(double v, double dm, double dw) { /* detector.cpp:26-30 */
  if (v > dm) return UCFVB_SCHEME_MUSCL;
  if (v > dw) return UCFVB_SCHEME_CWENOZ;
  return UCFVB_SCHEME_LINEAR;
}
static int deactivate_smooth(double du, double h, double kappa, double n) { /* detector.cpp:32-35 */
  if (kappa <= 0.0) return 0;
  return du < pow(kappa * h, n);
}
static inline int severity(int s) { return s == 0 ? 0 : (s == 1 ? 1 : 2); } /* detector.hpp:16-22 */

/* ---- reconstruct.cpp --------------------------------------------------- */
/* solve_dofs (reconstruct.cpp:9-28) */
static void solve_dofs(const port_solver* P, int c, const double* u, double* dofs) {
  const int64_t c0 = P->s.central_ptr[c];
  const int M = (int)(P->s.central_ptr[c + 1] - c0) - 1;
  const double* u0 = &u[4 * (int64_t)P->s.central[3 * c0]];
  const double* pinv = &P->s.pinv[P->s.pinv_off[c]];
  for (int k = 0; k < P->K; ++k) {
    const double* row = &pinv[(int64_t)k * M];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int m = 0; m < M; ++m) {
      const double* um = &u[4 * (int64_t)P->s.central[3 * (c0 + m + 1)]];
      const double w = row[m];
      s0 += w * (um[0] - u0[0]);
      s1 += w * (um[1] - u0[1]);
      s2 += w * (um[2] - u0[2]);
      s3 += w * (um[3] - u0[3]);
    }
    dofs[k * NV + 0] = s0;
    dofs[k * NV + 1] = s1;
    dofs[k * NV + 2] = s2;
    dofs[k * NV + 3] = s3;
  }
}

/* solve_dofs_linear (reconstruct.cpp:30-41) */
static void solve_dofs_linear(const port_solver* P, int c, const double* u, double* dofs) {
  const int64_t c0 = P->s.central_ptr[c];
  const int M = (int)(P->s.central_ptr[c + 1] - c0) - 1;
  const double* u0 = &u[4 * (int64_t)P->s.central[3 * c0]];
  const double* pl = &P->s.pinv_lin[P->s.pinv_lin_off[c]];
  for (int k = 0; k < 2; ++k) {
    const double* row = &pl[(int64_t)k * M];
    for (int v = 0; v < NV; ++v) {
      double s = 0.0;
      for (int m = 0; m < M; ++m) s += row[m] * (u[4 * (int64_t)P->s.central[3 * (c0 + m + 1)] + v] - u0[v]);
      dofs[k * NV + v] = s;
    }
  }
}

/* solve_dofs_directional (reconstruct.cpp:43-57); s is a global stencil index */
static void solve_dofs_directional(const port_solver* P, int c, int64_t s, const double* u, double* dofs) {
  const int64_t c0 = P->s.central_ptr[c];
  const int64_t m0 = P->s.dir_member_ptr[s];
  const int M = (int)(P->s.dir_member_ptr[s + 1] - m0) - 1;
  const double* u0 = &u[4 * (int64_t)P->s.central[3 * c0]];
  const double* pd = &P->s.pinv_dir[P->s.pinv_dir_off[s]];
  for (int k = 0; k < 2; ++k) {
    const double* row = &pd[(int64_t)k * M];
    for (int v = 0; v < NV; ++v) {
      double acc = 0.0;
      for (int m = 0; m < M; ++m) {
        const int mem = P->s.dir_members[m0 + m + 1];
        acc += row[m] * (u[4 * (int64_t)P->s.central[3 * (c0 + mem)] + v] - u0[v]);
      }
      dofs[k * NV + v] = acc;
    }
  }
}

/* limiter_barth_jespersen (reconstruct.cpp:59-71) */
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

/* limiter_venkatakrishnan (reconstruct.cpp:73-86) */
static double limiter_venkat(double u0, double umin, double umax, const double* q, int nq, double eps2) {
  double theta = 1.0;
  for (int i = 0; i < nq; ++i) {
    const double dm = q[i] - u0;
    if (dm == 0.0) continue;
    const double dp = (dm > 0.0) ? (umax - u0) : (umin - u0);
    const double num = (dp * dp + eps2) * dm + 2.0 * dm * dm * dp;
    const double den = dm * (dp * dp + 2.0 * dm * dm + dm * dp + eps2);
    const double phi = (den != 0.0) ? num / den : 1.0;
    const double cl = phi < 0.0 ? 0.0 : (1.0 < phi ? 1.0 : phi); /* std::clamp */
    theta = smin(theta, cl);
  }
  return theta;
}

/* smoothness_indicator (reconstruct.cpp:88-97) */
static double smoothness_indicator(const double* oi, const double* a, int K) {
  double s = 0.0;
  for (int k = 0; k < K; ++k) {
    const double* row = &oi[(int64_t)k * K];
    double t = 0.0;
    for (int q = 0; q < K; ++q) t += row[q] * a[q];
    s += a[k] * t;
  }
  return s;
}

/* cwenoz_blend_scalar (reconstruct.cpp:99-150); dir is [nd][2] */
static int cwenoz_blend(const double* oi, int K, const double* central, const double (*dir)[2], int nd,
                        double lambda1p, double eps, double b, double* blended) {
  if (!(lambda1p > 1.0)) {
    snprintf(g_err, sizeof g_err, "cwenoz: central linear weight lambda1' must exceed 1");
    return UCFVB_INVALID;
  }
  const int st = nd + 1;
  if (st > 8) {
    snprintf(g_err, sizeof g_err, "cwenoz: too many directional stencils");
    return UCFVB_INVALID;
  }
  double lambda[8], si[8], omega[8], p1[64];
  lambda[0] = 1.0 - 1.0 / lambda1p;
  for (int s = 1; s < st; ++s) lambda[s] = (1.0 - lambda[0]) / (st - 1);
  for (int k = 0; k < K; ++k) p1[k] = central[k];
  for (int s = 1; s < st; ++s) {
    p1[0] -= lambda[s] * dir[s - 1][0];
    p1[1] -= lambda[s] * dir[s - 1][1];
  }
  for (int k = 0; k < K; ++k) p1[k] /= lambda[0];
  si[0] = smoothness_indicator(oi, p1, K);
  for (int s = 1; s < st; ++s) {
    const double a0 = dir[s - 1][0], a1 = dir[s - 1][1];
    si[s] = oi[0] * a0 * a0 + (oi[1] + oi[K]) * a0 * a1 + oi[K + 1] * a1 * a1;
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
  }
  return 0;
}

/* ---- solver.cpp --------------------------------------------------------- */
static inline double* slot_ptr(port_solver* P, int slot) {
  return (slot & 1) ? &P->val_right[4 * (int64_t)(slot >> 1)] : &P->val_left[4 * (int64_t)(slot >> 1)];
}

/* evaluate_cell (solver.cpp:76-89) */
static void evaluate_cell(port_solver* P, const double* u, int c, const double* dofs) {
  const int64_t q0 = P->s.qp_ptr[c], q1 = P->s.qp_ptr[c + 1];
  const double* phi = &P->s.phi[P->s.phi_off[c]];
  const int K = P->K;
  const double* u0 = &u[4 * (int64_t)c];
  for (int64_t q = 0; q < q1 - q0; ++q) {
    double out[4] = {u0[0], u0[1], u0[2], u0[3]};
    const double* ph = &phi[q * K];
    for (int k = 0; k < K; ++k) {
      const double p = ph[k];
      out[0] += dofs[k * NV + 0] * p;
      out[1] += dofs[k * NV + 1] * p;
      out[2] += dofs[k * NV + 2] * p;
      out[3] += dofs[k * NV + 3] * p;
    }
    memcpy(slot_ptr(P, P->s.qp_slot[q0 + q]), out, sizeof out);
  }
}

/* evaluate_constant (solver.cpp:91-101) */
static void evaluate_constant(port_solver* P, const double* u, int c) {
  for (int64_t q = P->s.qp_ptr[c]; q < P->s.qp_ptr[c + 1]; ++q)
    memcpy(slot_ptr(P, P->s.qp_slot[q]), &u[4 * (int64_t)c], 4 * sizeof(double));
}

static const int kChecked[2] = {0, 3}; /* solver.cpp:18 */

static void cell_bounds(const port_solver* P, const double* u, int c, double* bnd) {
  for (int t = 0; t < 2; ++t) {
    const double u0 = u[4 * (int64_t)c + kChecked[t]];
    double lo = u0, hi = u0;
    for (int i = P->nb_ptr[c]; i < P->nb_ptr[c + 1]; ++i) {
      lo = smin(lo, u[4 * (int64_t)P->nb[i] + kChecked[t]]);
      hi = smax(hi, u[4 * (int64_t)P->nb[i] + kChecked[t]]);
    }
    bnd[2 * t] = lo;
    bnd[2 * t + 1] = hi;
  }
}

/* classify_cells (solver.cpp:113-149) + spread_flags (detector.cpp:37-53) */
static void classify_cells(port_solver* P, const double* u) {
  const int n = P->n;
  uint8_t* raw = (uint8_t*)malloc((size_t)n);
  for (int c = 0; c < n; ++c) {
    double* bnd = &P->bounds[4 * (int64_t)c];
    cell_bounds(P, u, c, bnd);
    int sev = 0;
    for (int t = 0; t < 2 && sev < 2; ++t) {
      const double du = bnd[2 * t + 1] - bnd[2 * t];
      if (deactivate_smooth(du, P->m.cell_h[c], P->o.margins.kappa, P->o.margins.deact_n)) continue;
      double v = -1e300;
      for (int64_t q = P->s.qp_ptr[c]; q < P->s.qp_ptr[c + 1]; ++q) {
        const double uq = slot_ptr(P, P->s.qp_slot[q])[kChecked[t]];
        v = smax(v, smax(bnd[2 * t] - uq, uq - bnd[2 * t + 1]));
      }
      double dm, dw;
      compute_margins(&P->o.margins, du, &dm, &dw);
      const int vote = classify_violation(v, dm, dw);
      sev = sev < severity(vote) ? severity(vote) : sev;
    }
    raw[c] = (uint8_t)(sev == 0 ? UCFVB_SCHEME_LINEAR : (sev == 1 ? UCFVB_SCHEME_CWENOZ : UCFVB_SCHEME_MUSCL));
  }
  /* spread_flags: one pass reading `raw` only */
  memcpy(P->labels, raw, (size_t)n);
  for (int c = 0; c < n; ++c) {
    const int s = raw[c];
    if (severity(s) == 0) continue;
    for (int i = P->m.cell_face_ptr[c]; i < P->m.cell_face_ptr[c + 1]; ++i) {
      const int fid = P->m.cell_faces[i];
      int nb = -1;
      if (P->m.face_right[fid] >= 0)
        nb = (P->m.face_left[fid] == c) ? P->m.face_right[fid] : P->m.face_left[fid];
      else if (P->m.face_partner[fid] >= 0)
        nb = P->m.face_left[P->m.face_partner[fid]];
      if (nb >= 0 && severity(P->labels[nb]) < severity(s)) P->labels[nb] = (uint8_t)s;
    }
  }
  free(raw);
}

/* apply_troubled (solver.cpp:151-227) */
static int apply_troubled(port_solver* P, const double* u) {
  const int n = P->n, K = P->K;
  for (int c = 0; c < n; ++c) {
    const int lab = P->labels[c];
    if (lab == UCFVB_SCHEME_LINEAR) continue;
    double* dofs = &P->dofs[(int64_t)c * K * NV];
    if (lab == UCFVB_SCHEME_CWENOZ) {
      const int64_t s0 = P->s.dir_ptr[c];
      const int nd = (int)(P->s.dir_ptr[c + 1] - s0);
      double dir_all[8][NV][2];
      double tmp[2 * NV];
      for (int s = 0; s < nd; ++s) {
        solve_dofs_directional(P, c, s0 + s, u, tmp);
        for (int v = 0; v < NV; ++v) {
          dir_all[s][v][0] = tmp[0 * NV + v];
          dir_all[s][v][1] = tmp[1 * NV + v];
        }
      }
      for (int v = 0; v < NV; ++v) {
        double sc[64], bl[64], dv[8][2];
        for (int k = 0; k < K; ++k) sc[k] = dofs[k * NV + v];
        for (int s = 0; s < nd; ++s) {
          dv[s][0] = dir_all[s][v][0];
          dv[s][1] = dir_all[s][v][1];
        }
        const int rc = cwenoz_blend(&P->s.oi[(int64_t)c * K * K], K, sc, (const double(*)[2])dv, nd,
                                    P->o.lambda1p, P->o.weno_eps, P->o.weno_b, bl);
        if (rc) return rc;
        for (int k = 0; k < K; ++k) dofs[k * NV + v] = bl[k];
      }
      evaluate_cell(P, u, c, dofs);
    } else if (lab == UCFVB_SCHEME_MUSCL) {
      double lin[2 * NV];
      solve_dofs_linear(P, c, u, lin);
      const double* phi = &P->s.phi[P->s.phi_off[c]];
      const int nq = (int)(P->s.qp_ptr[c + 1] - P->s.qp_ptr[c]);
      double qpv[64 * NV];
      for (int q = 0; q < nq; ++q) {
        const double p0 = phi[(int64_t)q * K];
        const double p1 = phi[(int64_t)q * K + 1];
        for (int v = 0; v < NV; ++v)
          qpv[q * NV + v] = u[4 * (int64_t)c + v] + lin[0 * NV + v] * p0 + lin[1 * NV + v] * p1;
      }
      const double eps2 = pow(P->o.venkat_kappa * P->m.cell_h[c], 3);
      for (int v = 0; v < NV; ++v) {
        const double u0 = u[4 * (int64_t)c + v];
        double lo = u0, hi = u0;
        for (int i = P->nb_ptr[c]; i < P->nb_ptr[c + 1]; ++i) {
          lo = smin(lo, u[4 * (int64_t)P->nb[i] + v]);
          hi = smax(hi, u[4 * (int64_t)P->nb[i] + v]);
        }
        double vv[64];
        for (int q = 0; q < nq; ++q) vv[q] = qpv[q * NV + v];
        const double theta = (P->o.limiter == UCFVB_BARTH_JESPERSEN) ? limiter_bj(u0, lo, hi, vv, nq)
                                                                    : limiter_venkat(u0, lo, hi, vv, nq, eps2);
        dofs[0 * NV + v] = theta * lin[0 * NV + v];
        dofs[1 * NV + v] = theta * lin[1 * NV + v];
        for (int k = 2; k < K; ++k) dofs[k * NV + v] = 0.0;
      }
      evaluate_cell(P, u, c, dofs);
    } else {
      for (int k = 0; k < K * NV; ++k) dofs[k] = 0.0;
      evaluate_constant(P, u, c);
    }
  }
  return 0;
}

/* fallback_check (solver.cpp:229-264) */
static void fallback_check(port_solver* P, const double* u) {
  const int n = P->n, K = P->K;
  const double g = P->o.gamma;
  for (int c = 0; c < n; ++c) {
    const double* bnd = &P->bounds[4 * (int64_t)c];
    const int64_t q0 = P->s.qp_ptr[c], q1 = P->s.qp_ptr[c + 1];
    int demote = 0;
    for (int64_t q = q0; q < q1; ++q)
      if (!is_physical(slot_ptr(P, P->s.qp_slot[q]), g)) {
        demote = 1;
        break;
      }
    if (!demote) {
      for (int t = 0; t < 2 && !demote; ++t) {
        const double du = bnd[2 * t + 1] - bnd[2 * t];
        double dm, dw;
        compute_margins(&P->o.margins, du, &dm, &dw);
        for (int64_t q = q0; q < q1; ++q) {
          const double uq = slot_ptr(P, P->s.qp_slot[q])[kChecked[t]];
          if (smax(bnd[2 * t] - uq, uq - bnd[2 * t + 1]) > dm) {
            demote = 1;
            break;
          }
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
static int assemble_fluxes(port_solver* P, double t, double* out) {
  const int nf = P->nf, nq = P->nq;
  (void)t;
  for (int fid = 0; fid < nf; ++fid) {
    const int partner = P->m.face_partner[fid];
    if (partner >= 0 && partner < fid) continue;
    const double nx = P->m.face_normal[2 * fid], ny = P->m.face_normal[2 * fid + 1];
    double total[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = 0; q < nq; ++q) {
      const double* UL = &P->val_left[4 * ((int64_t)fid * nq + q)];
      double UR[4];
      if (P->m.face_right[fid] >= 0) {
        memcpy(UR, &P->val_right[4 * ((int64_t)fid * nq + q)], sizeof UR);
      } else if (partner >= 0) {
        memcpy(UR, &P->val_left[4 * ((int64_t)partner * nq + P->m.face_partner_qp[fid * nq + q])], sizeof UR);
      } else {
        const port_bc* bc = &P->patch_bc[P->m.face_patch[fid]];
        if (bc->kind == UCFVB_BC_OUTFLOW) {
          memcpy(UR, UL, sizeof UR);
        } else if (bc->kind == UCFVB_BC_WALL) { /* mirror_state euler.hpp:67-70 */
          const double mn = UL[1] * nx + UL[2] * ny;
          UR[0] = UL[0];
          UR[1] = UL[1] - 2.0 * mn * nx;
          UR[2] = UL[2] - 2.0 * mn * ny;
          UR[3] = UL[3];
        } else {
          memcpy(UR, bc->state, sizeof UR);
        }
      }
      double fl[4], bad = 0.0;
      int which = 0;
      if (riemann_flux(P->o.riemann, UL, UR, nx, ny, P->o.gamma, fl, &which, &bad)) {
        snprintf(g_err, sizeof g_err, "non-physical state: %s = %f at face %d (midpoint %f, %f)",
                 which == 1 ? "rho" : "p", bad, fid, P->m.face_midpoint[2 * fid], P->m.face_midpoint[2 * fid + 1]);
        return UCFVB_NONPHYSICAL;
      }
      for (int v = 0; v < NV; ++v) total[v] += P->m.face_qw[fid * nq + q] * fl[v];
    }
    for (int v = 0; v < NV; ++v) P->face_flux[4 * (int64_t)fid + v] = total[v] * P->m.face_length[fid];
  }
  for (int c = 0; c < P->n; ++c) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = P->m.cell_face_ptr[c]; i < P->m.cell_face_ptr[c + 1]; ++i) {
      const int fid = P->m.cell_faces[i];
      double sgn = (P->m.face_left[fid] == c) ? 1.0 : -1.0;
      int src = fid;
      const int partner = P->m.face_partner[fid];
      if (partner >= 0 && partner < fid) {
        src = partner;
        sgn = -1.0;
      }
      for (int v = 0; v < NV; ++v) acc[v] += sgn * P->face_flux[4 * (int64_t)src + v];
    }
    const double inv_vol = 1.0 / P->m.cell_area[c];
    for (int v = 0; v < NV; ++v) out[4 * (int64_t)c + v] = -acc[v] * inv_vol;
  }
  return 0;
}

/* compute_residual (solver.cpp:316-379) */
int port_compute_residual(port_solver* P, const double* u, double t, int stage_first, double* out) {
  const int n = P->n, K = P->K, mode = P->o.mode;
  if (stage_first >= 0) P->stage_is_first = stage_first != 0;
  if (mode == UCFVB_FIRST)
    memset(P->labels, UCFVB_SCHEME_FIRST, (size_t)n);
  else if (mode == UCFVB_MUSCL)
    memset(P->labels, UCFVB_SCHEME_MUSCL, (size_t)n);
  else if (mode == UCFVB_CWENOZ)
    memset(P->labels, UCFVB_SCHEME_CWENOZ, (size_t)n);
  if (mode == UCFVB_LINEAR || mode == UCFVB_CWENOZ || mode == UCFVB_HYBRID) {
    for (int c = 0; c < n; ++c) {
      double* dofs = &P->dofs[(int64_t)c * K * NV];
      solve_dofs(P, c, u, dofs);
      if (mode != UCFVB_CWENOZ) evaluate_cell(P, u, c, dofs);
    }
  }
  if (mode == UCFVB_HYBRID && (P->stage_is_first || P->o.detect_every_stage)) classify_cells(P, u);
  if (mode != UCFVB_LINEAR) {
    const int rc = apply_troubled(P, u);
    if (rc) return rc;
  }
  if (mode == UCFVB_HYBRID) {
    if (!P->stage_is_first && !P->o.detect_every_stage)
      for (int c = 0; c < n; ++c) cell_bounds(P, u, c, &P->bounds[4 * (int64_t)c]);
    fallback_check(P, u);
  }
  if (P->stage_is_first) {
    memcpy(P->step_labels, P->labels, (size_t)n);
    P->stage_is_first = 0;
  }
  return assemble_fluxes(P, t, out);
}

/* max_stable_dt (solver.cpp:103-111) */
int port_max_stable_dt(port_solver* P, const double* u, double* out) {
  double dt = 1e300;
  const double g = P->o.gamma;
  for (int c = 0; c < P->n; ++c) {
    double w[4];
    const int rc = cons_to_prim(&u[4 * (int64_t)c], g, w);
    if (rc) {
      snprintf(g_err, sizeof g_err, "non-physical state: %s = %f", rc == 1 ? "rho" : "p",
               rc == 1 ? u[4 * (int64_t)c] : w[3]);
      return UCFVB_NONPHYSICAL;
    }
    const double speed = fabs(w[1]) + fabs(w[2]) + sqrt(g * w[3] / w[0]);
    dt = smin(dt, P->m.cell_h[c] / speed);
  }
  *out = P->o.cfl * dt;
  return 0;
}

/* combine2 (time_integrator.cpp:31-38) */
static void combine2(int n, double* out, double wa, const double* ua, double wb, const double* ub, double wr,
                     const double* r, double dt) {
  const double wrdt = wr * dt;
  for (int64_t i = 0; i < 4 * (int64_t)n; ++i) out[i] = wa * ua[i] + wb * ub[i] + wrdt * r[i];
}

/* ssp_rk4_step (time_integrator.cpp:42-74) or SSP-RK3; u in/out */
int port_advance(port_solver* P, double* u, double dt, double t, int rk) {
  const int n = P->n;
  int rc;
  P->stage_is_first = 1;
  if (rk == UCFVB_RK3) {
    if ((rc = port_compute_residual(P, u, t, -1, P->rhs))) return rc;
    combine2(n, P->ua, 1.0, u, 0.0, u, 1.0, P->rhs, dt);
    if ((rc = port_compute_residual(P, P->ua, t + dt, -1, P->rhs))) return rc;
    combine2(n, P->ub, 0.75, u, 0.25, P->ua, 0.25, P->rhs, dt);
    if ((rc = port_compute_residual(P, P->ub, t + 0.5 * dt, -1, P->rhs))) return rc;
    combine2(n, u, 1.0 / 3.0, u, 2.0 / 3.0, P->ub, 2.0 / 3.0, P->rhs, dt);
    return 0;
  }
  const double a10 = 0.391752226571890;
  const double b20 = 0.444370493651235, b21 = 0.555629506348765, a21 = 0.368410593050371;
  const double b30 = 0.620101851488403, b32 = 0.379898148511597, a32 = 0.251891774271694;
  const double b40 = 0.178079954393132, b43 = 0.821920045606868, a43 = 0.544974750228521;
  const double c52 = 0.517231671970585, c53 = 0.096059710526147, a53 = 0.063692468666290;
  const double c54 = 0.386708617503269, a54 = 0.226007483236906;
  const double t1 = t + a10 * dt;
  const double t2 = t + (b21 * a10 + a21) * dt;
  const double t3 = t + (b32 * (b21 * a10 + a21) + a32) * dt;
  const double t4 = t + (b43 * (b32 * (b21 * a10 + a21) + a32) + a43) * dt;
  if ((rc = port_compute_residual(P, u, t, -1, P->rhs))) return rc;
  combine2(n, P->ua, 1.0, u, 0.0, u, a10, P->rhs, dt);
  if ((rc = port_compute_residual(P, P->ua, t1, -1, P->rhs))) return rc;
  combine2(n, P->ub, b20, u, b21, P->ua, a21, P->rhs, dt);
  if ((rc = port_compute_residual(P, P->ub, t2, -1, P->rhs))) return rc;
  combine2(n, P->uc, b30, u, b32, P->ub, a32, P->rhs, dt);
  if ((rc = port_compute_residual(P, P->uc, t3, -1, P->rhs3))) return rc;
  combine2(n, P->ud, b40, u, b43, P->uc, a43, P->rhs3, dt);
  if ((rc = port_compute_residual(P, P->ud, t4, -1, P->rhs))) return rc;
  for (int64_t i = 0; i < 4 * (int64_t)n; ++i)
    u[i] = c52 * P->ub[i] + c53 * P->uc[i] + a53 * dt * P->rhs3[i] + c54 * P->ud[i] + a54 * dt * P->rhs[i];
  return 0;
}

/* ---- lifecycle ------------------------------------------------------------ */
int port_create(const ucfvb_mesh_view* m, const ucfvb_stencil_view* s, const ucfvb_options* o,
                const ucfvb_bc* bcs, int n_bcs, port_solver** out) {
  port_solver* P = (port_solver*)calloc(1, sizeof *P);
  P->m = *m;
  P->s = *s;
  P->o = *o;
  P->n = m->n_cells;
  P->nf = m->n_faces;
  P->nq = s->n_qp;
  P->K = s->K;
  P->patch_bc = (port_bc*)calloc((size_t)(m->n_patches > 0 ? m->n_patches : 1), sizeof(port_bc));
  for (int i = 0; i < n_bcs; ++i)
    for (int p = 0; p < m->n_patches; ++p)
      if (strcmp(m->patch_names[p], bcs[i].patch) == 0) {
        P->patch_bc[p].kind = bcs[i].kind;
        memcpy(P->patch_bc[p].state, bcs[i].state, sizeof(double) * 4);
      }
  for (int f = 0; f < m->n_faces; ++f)
    if (m->face_right[f] < 0 && m->face_partner[f] < 0 &&
        (m->face_patch[f] < 0 || P->patch_bc[m->face_patch[f]].kind == UCFVB_BC_NONE)) {
      snprintf(g_err, sizeof g_err, "solver: boundary face %d has no boundary condition", f);
      free(P->patch_bc);
      free(P);
      return UCFVB_INVALID;
    }
  const int n = P->n;
  P->nb_ptr = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  P->nb = (int*)malloc(sizeof(int) * (size_t)(m->cell_face_ptr[n] + 1));
  int w = 0;
  for (int c = 0; c < n; ++c) {
    P->nb_ptr[c] = w;
    for (int i = m->cell_face_ptr[c]; i < m->cell_face_ptr[c + 1]; ++i) {
      const int fid = m->cell_faces[i];
      if (m->face_right[fid] >= 0)
        P->nb[w++] = (m->face_left[fid] == c) ? m->face_right[fid] : m->face_left[fid];
      else if (m->face_partner[fid] >= 0)
        P->nb[w++] = m->face_left[m->face_partner[fid]];
    }
  }
  P->nb_ptr[n] = w;
  const size_t nK = (size_t)n * (size_t)P->K * NV;
  P->dofs = (double*)calloc(nK, sizeof(double));
  P->val_left = (double*)calloc((size_t)P->nf * P->nq * NV, sizeof(double));
  P->val_right = (double*)calloc((size_t)P->nf * P->nq * NV, sizeof(double));
  P->face_flux = (double*)calloc((size_t)P->nf * NV, sizeof(double));
  P->labels = (uint8_t*)calloc((size_t)n, 1);
  P->step_labels = (uint8_t*)calloc((size_t)n, 1);
  P->bounds = (double*)calloc((size_t)n * 4, sizeof(double));
  double** ws[] = {&P->ua, &P->ub, &P->uc, &P->ud, &P->rhs, &P->rhs3};
  for (int i = 0; i < 6; ++i) *ws[i] = (double*)calloc((size_t)n * NV, sizeof(double));
  P->stage_is_first = 1;
  *out = P;
  return 0;
}

void port_free(port_solver* P) {
  if (!P) return;
  free(P->nb_ptr); free(P->nb); free(P->patch_bc); free(P->dofs); free(P->val_left);
  free(P->val_right); free(P->face_flux); free(P->labels); free(P->step_labels); free(P->bounds);
  free(P->ua); free(P->ub); free(P->uc); free(P->ud); free(P->rhs); free(P->rhs3);
  free(P);
}

/* taps */
void port_get_labels(const port_solver* P, uint8_t* out, int step) {
  memcpy(out, step ? P->step_labels : P->labels, (size_t)P->n);
}
void port_get_face_values(const port_solver* P, double* L, double* R) {
  memcpy(L, P->val_left, sizeof(double) * (size_t)P->nf * P->nq * NV);
  memcpy(R, P->val_right, sizeof(double) * (size_t)P->nf * P->nq * NV);
}
void port_get_dofs(const port_solver* P, double* d) { memcpy(d, P->dofs, sizeof(double) * (size_t)P->n * P->K * NV); }
void port_get_bounds(const port_solver* P, double* b) { memcpy(b, P->bounds, sizeof(double) * (size_t)P->n * 4); }

/* ---- exported point functions (known-answer tests, tests/test_kat.py) ---- */
void port_compute_margins(const ucfvb_margins* m, double du, double* dm, double* dw) { compute_margins(m, du, dm, dw); }
int port_classify_violation(double v, double dm, double dw) { return classify_violation(v, dm, dw); }
int port_deactivate_smooth(double du, double h, double kappa, double n) { return deactivate_smooth(du, h, kappa, n); }
double port_limiter_bj(double u0, double lo, double hi, const double* q, int nq) { return limiter_bj(u0, lo, hi, q, nq); }
double port_limiter_venkat(double u0, double lo, double hi, const double* q, int nq, double eps2) {
  return limiter_venkat(u0, lo, hi, q, nq, eps2);
}
int port_flux(const double* ul, const double* ur, double nx, double ny, double g, int kind, double* out) {
  int which = 0;
  double bad = 0.0;
  return riemann_flux(kind, ul, ur, nx, ny, g, out, &which, &bad) ? UCFVB_NONPHYSICAL : 0;
}
int port_cwenoz_blend(const double* oi, int K, const double* central, const double* dir, int nd, double lambda1p,
                      double eps, double b, double* blended) {
  return cwenoz_blend(oi, K, central, (const double(*)[2])dir, nd, lambda1p, eps, b, blended);
}
