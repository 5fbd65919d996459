// sm_100a fp64 kernels of the hybrid NAD stage pass (arXiv 2510.25906).
//
// Data layout: per-cell operator data is stored in 32-cell
// AoSoA chunks, element e of cell c at ((c>>5)*E + e)*32 + (c&31), so the 32
// threads of a warp (32 consecutive cells) read one contiguous 256 B line per
// element. The state U is AoS double4 (one 32 B sector per gathered stencil
// member, same layout as the reference's std::array<double,4>). Face-point
// values are stored per cell-local quadrature point (the reference's
// val_left_/val_right_ slots re-indexed by owning cell) as double4 chunks.
//
// Kernels (one RK stage):
//   k_central   central LSQ solve + face-point eval + NAD raw label + fallback
//               pre-check (reference solver.cpp:333-337, 113-149, 229-264)
//   k_spread    von Neumann spread + linear-cell demotion + warp-ballot
//               compaction into the CWENOZ / MUSCL lists (detector.cpp:37-53)
//   k_cwenoz    directional solves + SI + weights + blend + eval + fallback
//               epilogue on the CWENOZ list (solver.cpp:167-188, reconstruct.cpp:43-150)
//   k_muscl     r=1 solve + BJ/Venkat limiter + eval + fallback epilogue on the
//               MUSCL list (solver.cpp:189-221, reconstruct.cpp:30-86)
//   k_flux      per-cell HLLC/HLL at every face Gauss point, owner-ordered
//               face-to-cell gather (no atomics) and the RK stage update
//               (solver.cpp:266-314, time_integrator.cpp:31-38,70-73)
//   k_dt        max_stable_dt min-reduction (solver.cpp:103-111) + device-side t/dt
#pragma once

#include <cstdint>

#include "device_math.cuh"

namespace ucfvb {

enum : int { FL_DOFS = 1, FL_EVAL = 2, FL_NAD = 4, FL_PRECHECK = 8, FL_TAPS = 16, FL_FALLBACK = 32,
             FL_CENSUS = 64, FL_STEP_LABELS = 128 };

constexpr int kMaxPatches = 16;
constexpr int kBlock = 128;

struct BcEntry {
  int kind;
  double state[4];
};

// everything a stage kernel reads; passed by value (fits the 32 KB param space)
struct Layout {
  int n;       // cells
  int MM;      // padded central stencil size (excluding self)
  int MD;      // padded directional stencil size (excluding self)
  const int* st_idx;        // E = MM           central member cell ids
  const double* pinv;       // E = MM*K  [m][k]
  const double* phi;        // E = Q*K   [lq][k]
  const double* pinv_lin;   // E = MM*2  [m][k]
  const int* dir_idx;       // E = NF*MD [s][m] member cell ids
  const double* pinv_dir;   // E = NF*MD*2 [s][m][k]
  const double* oi;         // E = K*K
  const int* nbr;           // E = NF    face neighbour (-1: none)
  const int* other_ref;     // E = NF*NQ fv index of the other face-point value, or -(1+patch)
  const uint8_t* self_lq;   // E = NF*NQ own local qp feeding canonical qp q
  const double* fgeom;      // E = NF*3  canonical normal x, y, length
  const int8_t* fsgn;       // E = NF    +1: own value is UL, -1: own value is UR
  const int* face_id;       // E = NF    canonical face id (error reports)
  const uint8_t* nfc;       // [n] faces per cell
  const double* deact_thr;  // [n] (kappa*h)^n or -inf
  const double* eps2;       // [n] (venkat_kappa*h)^3
  const double* h;          // [n]
  const double* inv_vol;    // [n] 1/area
};

struct Physics {
  MarginParams mp;
  double gamma, lambda1p, weno_eps, weno_b;
  int limiter;  // 0 BJ, 1 Venkat
  int hll;      // 0 HLLC, 1 HLL
  double qw[4];  // face quadrature weights (identical on every face)
  BcEntry bc[kMaxPatches];
};

struct Scratch {
  double4* fv;       // face-point values [chunk][Q][lane]
  double4* dofs;     // [chunk][K][lane]
  uint8_t* raw;      // raw NAD label | demote-if-linear << 2
  uint8_t* labels;
  uint8_t* step_labels;
  int* list_c;
  int* list_m;
  int* counts;       // [0] CWENOZ list length, [1] MUSCL list length
  unsigned long long* ties;
  unsigned long long* census;  // base of [steps][4]; row selected by *step
  const int* step;
  int* err;          // [0] error kind bits, [1] min failing face, [2] min failing cell, [3] min failing step
};

// RK stage epilogue: out = sum_i coef_i * term_i, accumulated left to right
// (combine2 time_integrator.cpp:31-38, final SSPRK(5,4) line :70-73).
struct RkEpilogue {
  int nterms;
  const double4* term[5];  // nullptr: this stage's residual
  double coef[5];
  int dt_scaled[5];        // coef * dt (dt read from the device)
  double4* out;            // nullable
  double4* rhs_out;        // nullable: store the residual itself
  const double* dt;        // device dt
};

__device__ __forceinline__ size_t aos(int c, int e, int E) {
  return ((static_cast<size_t>(c >> 5) * E) + e) * 32 + (c & 31);
}

__device__ __forceinline__ void record_error(int* err, int face, const int* step) {
  atomicOr(&err[0], 1);
  atomicMin(&err[1], face);
  atomicMin(&err[3], *step);
}

// ---------------------------------------------------------------------------
// k_central: solve_dofs (reconstruct.cpp:9-28) with the m-loop outermost (each
// accumulator still sums in m order), evaluate_cell (solver.cpp:76-89),
// classify_cells raw severity (solver.cpp:113-149) and the fallback pre-check
// a Linear cell needs (solver.cpp:229-264).
template <int K, int NQ, int NF>
__global__ void __launch_bounds__(kBlock) k_central(Layout L, Physics ph, Scratch S, const double4* __restrict__ U,
                                                    int flags) {
  constexpr int Q = NF * NQ;
  const int c = blockIdx.x * kBlock + threadIdx.x;
  if (c >= L.n) return;
  if (*(volatile int*)S.err) return;
  const d4 u0 = ld4(&U[c]);
  double acc[K][NV];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[k][v] = 0.0;

  const int MM = L.MM;
  const int* ip = L.st_idx + aos(c, 0, MM);
  const double* pp = L.pinv + aos(c, 0, MM * K);
#pragma unroll 2
  for (int m = 0; m < MM; ++m) {
    const int nb = __ldg(ip + m * 32);
    const d4 um = ld4(&U[nb]);
    double d[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) d[v] = um.v[v] - u0.v[v];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const double w = __ldg(pp + (m * K + k) * 32);
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[k][v] += w * d[v];
    }
  }
  if (flags & FL_DOFS) {
#pragma unroll
    for (int k = 0; k < K; ++k) st4(&S.dofs[aos(c, k, K)], acc[k]);
  }
  if (!(flags & FL_EVAL)) return;

  const int nf = L.nfc[c];
  const bool detect = (flags & (FL_NAD | FL_PRECHECK)) != 0;
  // neighbourhood bounds of rho and E (solver.cpp:120-129)
  double lo0 = u0.v[0], hi0 = u0.v[0], lo3 = u0.v[3], hi3 = u0.v[3];
  if (detect) {
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int nb = __ldg(L.nbr + aos(c, j, NF));
      if (nb >= 0) {
        const double r = __ldg(&U[nb].x), e = __ldg(&U[nb].w);
        lo0 = smin(lo0, r);
        hi0 = smax(hi0, r);
        lo3 = smin(lo3, e);
        hi3 = smax(hi3, e);
      }
    }
  }
  const double du0 = hi0 - lo0, du3 = hi3 - lo3;
  double dm0, dw0, dm3, dw3;
  compute_margins(ph.mp, du0, dm0, dw0);
  compute_margins(ph.mp, du3, dm3, dw3);
  double v0 = -1e300, v3 = -1e300;
  bool bad = false;
  const double* fp = L.phi + aos(c, 0, Q * K);
#pragma unroll
  for (int lq = 0; lq < Q; ++lq) {
    if (lq < nf * NQ) {
      double val[NV] = {u0.v[0], u0.v[1], u0.v[2], u0.v[3]};
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const double p = __ldg(fp + (lq * K + k) * 32);
#pragma unroll
        for (int v = 0; v < NV; ++v) val[v] += acc[k][v] * p;
      }
      st4(&S.fv[aos(c, lq, Q)], val);
      if (detect) {
        const double x0 = smax(lo0 - val[0], val[0] - hi0);
        const double x3 = smax(lo3 - val[3], val[3] - hi3);
        v0 = smax(v0, x0);
        v3 = smax(v3, x3);
        bad |= (x0 > dm0) || (x3 > dm3) || !is_physical(val, ph.gamma);
      }
    }
  }
  if (!detect) return;
  int sev = 0;
  bool tie = false;
  if (flags & FL_NAD) {
    const double thr = L.deact_thr[c];
    if (!(du0 < thr)) {
      sev = violation_severity(v0, dm0, dw0);
      const double sc = smax(smax(fabs(u0.v[0]), du0), 1e-300);
      tie |= fabs(v0 - dm0) <= 1e-12 * smax(sc, fabs(dm0)) || fabs(v0 - dw0) <= 1e-12 * smax(sc, fabs(dw0));
    }
    if (sev < 2 && !(du3 < thr)) {
      const int s3 = violation_severity(v3, dm3, dw3);
      sev = sev < s3 ? s3 : sev;
      const double sc = smax(smax(fabs(u0.v[3]), du3), 1e-300);
      tie |= fabs(v3 - dm3) <= 1e-12 * smax(sc, fabs(dm3)) || fabs(v3 - dw3) <= 1e-12 * smax(sc, fabs(dw3));
    }
    if (thr > 0.0) tie |= fabs(du0 - thr) <= 1e-12 * thr || fabs(du3 - thr) <= 1e-12 * thr;
    const unsigned tm = __ballot_sync(__activemask(), tie);
    if (tm && (threadIdx.x & 31) == __ffs(tm) - 1) atomicAdd(S.ties, static_cast<unsigned long long>(__popc(tm)));
  }
  S.raw[c] = static_cast<uint8_t>(sev | (bad ? 4 : 0));
}

// ---------------------------------------------------------------------------
// k_spread: labels = spread_flags(raw) as a pull-max over face neighbours
// (detector.cpp:37-53 reads `in` only, so push == pull); Linear cells whose
// pre-check failed become FirstOrder (fallback_check); the troubled classes
// are compacted into lists with one atomic per warp (ballot + popc).
template <int NQ, int NF>
__global__ void __launch_bounds__(kBlock) k_spread(Layout L, Scratch S, const double4* __restrict__ U, int flags,
                                                   int detect) {
  constexpr int Q = NF * NQ;
  const int c = blockIdx.x * kBlock + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int lab = -1;
  if (c < L.n && !*(volatile int*)S.err) {
    const int r = S.raw[c];
    if (detect) {
      lab = r & 3;
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int nb = __ldg(L.nbr + aos(c, j, NF));
        if (nb >= 0) {
          const int rn = S.raw[nb] & 3;
          lab = lab < rn ? rn : lab;
        }
      }
    } else {
      lab = S.labels[c];  // frozen classification (detect_every_stage = false)
    }
    if (lab == 0 && (r & 4)) lab = 3;
    if (lab == 3) {
      const d4 u0 = ld4(&U[c]);
      const int nf = L.nfc[c];
#pragma unroll
      for (int lq = 0; lq < Q; ++lq)
        if (lq < nf * NQ) st4(&S.fv[aos(c, lq, Q)], u0);
    }
    S.labels[c] = static_cast<uint8_t>(lab);
  }
  const unsigned full = 0xffffffffu;
  const unsigned mc = __ballot_sync(full, lab == 1);
  const unsigned mm = __ballot_sync(full, lab == 2);
  const unsigned lt = (1u << lane) - 1u;
  if (mc) {
    int base = 0;
    if (lane == __ffs(mc) - 1) base = atomicAdd(&S.counts[0], __popc(mc));
    base = __shfl_sync(full, base, __ffs(mc) - 1);
    if (lab == 1) S.list_c[base + __popc(mc & lt)] = c;
  }
  if (mm) {
    int base = 0;
    if (lane == __ffs(mm) - 1) base = atomicAdd(&S.counts[1], __popc(mm));
    base = __shfl_sync(full, base, __ffs(mm) - 1);
    if (lab == 2) S.list_m[base + __popc(mm & lt)] = c;
  }
}

// fallback_check epilogue for a reconstructed (CWENOZ/MUSCL) cell: returns
// true when the cell must drop to first order (solver.cpp:229-264).
template <int NQ, int NF>
__device__ __forceinline__ bool fallback_demote(const Layout& L, const Physics& ph, const double4* __restrict__ U,
                                                int c, const d4& u0, const double (*vals)[NV], int nq_cell) {
  double lo0 = u0.v[0], hi0 = u0.v[0], lo3 = u0.v[3], hi3 = u0.v[3];
#pragma unroll
  for (int j = 0; j < NF; ++j) {
    const int nb = __ldg(L.nbr + aos(c, j, NF));
    if (nb >= 0) {
      const double r = __ldg(&U[nb].x), e = __ldg(&U[nb].w);
      lo0 = smin(lo0, r);
      hi0 = smax(hi0, r);
      lo3 = smin(lo3, e);
      hi3 = smax(hi3, e);
    }
  }
  double dm0, dw0, dm3, dw3;
  compute_margins(ph.mp, hi0 - lo0, dm0, dw0);
  compute_margins(ph.mp, hi3 - lo3, dm3, dw3);
  bool bad = false;
#pragma unroll
  for (int lq = 0; lq < NF * NQ; ++lq) {
    if (lq < nq_cell) {
      const double* val = vals[lq];
      bad |= !is_physical(val, ph.gamma) || smax(lo0 - val[0], val[0] - hi0) > dm0 ||
             smax(lo3 - val[3], val[3] - hi3) > dm3;
    }
  }
  return bad;
}

// ---------------------------------------------------------------------------
// k_cwenoz: one thread per listed cell, all four variables in registers.
template <int K, int NQ, int NF>
__global__ void __launch_bounds__(kBlock) k_cwenoz(Layout L, Physics ph, Scratch S, const double4* __restrict__ U,
                                                   int flags) {
  constexpr int Q = NF * NQ;
  const bool all = (flags & FL_NAD) == 0;  // forced CWENOZ mode: every cell, no list
  const int count = all ? L.n : S.counts[0];
  if (*(volatile int*)S.err) return;
  for (int i = blockIdx.x * kBlock + threadIdx.x; i < count; i += gridDim.x * kBlock) {
    const int c = all ? i : S.list_c[i];
    const d4 u0 = ld4(&U[c]);
    const int nf = L.nfc[c];
    // directional r=1 solves (reconstruct.cpp:43-57)
    double dir[NF][2][NV];
#pragma unroll
    for (int s = 0; s < NF; ++s)
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int v = 0; v < NV; ++v) dir[s][k][v] = 0.0;
    const int MD = L.MD;
#pragma unroll
    for (int s = 0; s < NF; ++s) {
      if (s < nf) {
        for (int m = 0; m < MD; ++m) {
          const int nb = __ldg(L.dir_idx + aos(c, s * MD + m, NF * MD));
          const d4 um = ld4(&U[nb]);
          const double w0 = __ldg(L.pinv_dir + aos(c, (s * MD + m) * 2 + 0, NF * MD * 2));
          const double w1 = __ldg(L.pinv_dir + aos(c, (s * MD + m) * 2 + 1, NF * MD * 2));
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const double d = um.v[v] - u0.v[v];
            dir[s][0][v] += w0 * d;
            dir[s][1][v] += w1 * d;
          }
        }
      }
    }
    // cwenoz_blend_scalar (reconstruct.cpp:99-150) for the four variables at once
    if (!(ph.lambda1p > 1.0)) {  // cwenoz_blend_scalar throws (reconstruct.cpp:102-103)
      atomicOr(&S.err[0], 4);
      return;
    }
    const int st = nf + 1;
    const double lam0 = 1.0 - 1.0 / ph.lambda1p;
    const double lams = (1.0 - lam0) / (st - 1);
    double p1[K][NV];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const d4 a = ld4(&S.dofs[aos(c, k, K)]);
#pragma unroll
      for (int v = 0; v < NV; ++v) p1[k][v] = a.v[v];
    }
#pragma unroll
    for (int s = 0; s < NF; ++s)
      if (s < nf) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          p1[0][v] -= lams * dir[s][0][v];
          p1[1][v] -= lams * dir[s][1][v];
        }
      }
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int v = 0; v < NV; ++v) p1[k][v] /= lam0;
    // SI_0 = p1^T OI p1, row then dot (reconstruct.cpp:88-97)
    const double* oi = L.oi + aos(c, 0, K * K);
    double si0[NV] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t[NV] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const double o = __ldg(oi + (k * K + q) * 32);
#pragma unroll
        for (int v = 0; v < NV; ++v) t[v] += o * p1[q][v];
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) si0[v] += p1[k][v] * t[v];
    }
    const double o00 = __ldg(oi + 0 * 32), o01 = __ldg(oi + 1 * 32);
    const double o10 = __ldg(oi + K * 32), o11 = __ldg(oi + (K + 1) * 32);
    double tau[NV] = {0.0, 0.0, 0.0, 0.0};
    double sis[NF][NV];
#pragma unroll
    for (int s = 0; s < NF; ++s)
      if (s < nf) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double a0 = dir[s][0][v], a1 = dir[s][1][v];
          sis[s][v] = o00 * a0 * a0 + (o01 + o10) * a0 * a1 + o11 * a1 * a1;
          tau[v] += fabs(sis[s][v] - si0[v]);
        }
      }
    double om0[NV], oms[NF][NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      tau[v] /= (st - 1);
      tau[v] = tau_pow(tau[v], ph.weno_b);
      om0[v] = lam0 * (1.0 + tau[v] / (ph.weno_eps + si0[v]));
      double wsum = om0[v];
#pragma unroll
      for (int s = 0; s < NF; ++s)
        if (s < nf) {
          oms[s][v] = lams * (1.0 + tau[v] / (ph.weno_eps + sis[s][v]));
          wsum += oms[s][v];
        }
      om0[v] /= wsum;
#pragma unroll
      for (int s = 0; s < NF; ++s)
        if (s < nf) oms[s][v] /= wsum;
    }
    // blended = omega_0 p1 + sum_s omega_s p_s (zero-padded directional dofs)
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int v = 0; v < NV; ++v) p1[k][v] = om0[v] * p1[k][v];
#pragma unroll
    for (int s = 0; s < NF; ++s)
      if (s < nf) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          p1[0][v] += oms[s][v] * dir[s][0][v];
          p1[1][v] += oms[s][v] * dir[s][1][v];
        }
      }
    // evaluate_cell + fallback epilogue
    const double* fp = L.phi + aos(c, 0, Q * K);
    double vals[Q][NV];
#pragma unroll
    for (int lq = 0; lq < Q; ++lq) {
      if (lq < nf * NQ) {
#pragma unroll
        for (int v = 0; v < NV; ++v) vals[lq][v] = u0.v[v];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const double p = __ldg(fp + (lq * K + k) * 32);
#pragma unroll
          for (int v = 0; v < NV; ++v) vals[lq][v] += p1[k][v] * p;
        }
      }
    }
    bool demote = false;
    if (flags & FL_FALLBACK) demote = fallback_demote<NQ, NF>(L, ph, U, c, u0, vals, nf * NQ);
#pragma unroll
    for (int lq = 0; lq < Q; ++lq)
      if (lq < nf * NQ) {
        if (demote)
          st4(&S.fv[aos(c, lq, Q)], u0);
        else
          st4(&S.fv[aos(c, lq, Q)], vals[lq]);
      }
    if (demote) S.labels[c] = 3;
    if (flags & FL_TAPS) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (demote) {
          const double z[NV] = {0.0, 0.0, 0.0, 0.0};
          st4(&S.dofs[aos(c, k, K)], z);
        } else {
          st4(&S.dofs[aos(c, k, K)], p1[k]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_muscl: r=1 LSQ gradient, BJ (or Venkatakrishnan) limiter per variable,
// limited evaluation and fallback epilogue.
template <int K, int NQ, int NF>
__global__ void __launch_bounds__(kBlock) k_muscl(Layout L, Physics ph, Scratch S, const double4* __restrict__ U,
                                                  int flags) {
  constexpr int Q = NF * NQ;
  const bool all = (flags & FL_NAD) == 0;  // forced MUSCL mode
  const int count = all ? L.n : S.counts[1];
  if (*(volatile int*)S.err) return;
  for (int i = blockIdx.x * kBlock + threadIdx.x; i < count; i += gridDim.x * kBlock) {
    const int c = all ? i : S.list_m[i];
    const d4 u0 = ld4(&U[c]);
    const int nf = L.nfc[c];
    double lin[2][NV];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int v = 0; v < NV; ++v) lin[k][v] = 0.0;
    const int MM = L.MM;
#pragma unroll 2
    for (int m = 0; m < MM; ++m) {
      const int nb = __ldg(L.st_idx + aos(c, m, MM));
      const d4 um = ld4(&U[nb]);
      const double w0 = __ldg(L.pinv_lin + aos(c, m * 2 + 0, MM * 2));
      const double w1 = __ldg(L.pinv_lin + aos(c, m * 2 + 1, MM * 2));
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const double d = um.v[v] - u0.v[v];
        lin[0][v] += w0 * d;
        lin[1][v] += w1 * d;
      }
    }
    // neighbourhood bounds of all four variables (solver.cpp:207-211)
    double lo[NV], hi[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) lo[v] = hi[v] = u0.v[v];
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int nb = __ldg(L.nbr + aos(c, j, NF));
      if (nb >= 0) {
        const d4 un = ld4(&U[nb]);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          lo[v] = smin(lo[v], un.v[v]);
          hi[v] = smax(hi[v], un.v[v]);
        }
      }
    }
    const double* fp = L.phi + aos(c, 0, Q * K);
    double p0s[Q], p1s[Q];
    double theta[NV] = {1.0, 1.0, 1.0, 1.0};
    const bool venkat = ph.limiter == 1;
    const double eps2 = venkat ? L.eps2[c] : 0.0;
#pragma unroll
    for (int lq = 0; lq < Q; ++lq) {
      if (lq < nf * NQ) {
        p0s[lq] = __ldg(fp + (lq * K + 0) * 32);
        p1s[lq] = __ldg(fp + (lq * K + 1) * 32);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double qv = u0.v[v] + lin[0][v] * p0s[lq] + lin[1][v] * p1s[lq];
          theta[v] = venkat ? venkat_update(theta[v], u0.v[v], lo[v], hi[v], qv, eps2)
                            : bj_update(theta[v], u0.v[v], lo[v], hi[v], qv);
        }
      }
    }
    double d0[NV], d1[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const double th = venkat ? theta[v] : smax(theta[v], 0.0);
      d0[v] = th * lin[0][v];
      d1[v] = th * lin[1][v];
    }
    double vals[Q][NV];
#pragma unroll
    for (int lq = 0; lq < Q; ++lq)
      if (lq < nf * NQ) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          double o = u0.v[v];
          o += d0[v] * p0s[lq];
          o += d1[v] * p1s[lq];
          vals[lq][v] = o;  // dofs k >= 2 are zero: adding 0*phi leaves o unchanged
        }
      }
    bool demote = false;
    if (flags & FL_FALLBACK) demote = fallback_demote<NQ, NF>(L, ph, U, c, u0, vals, nf * NQ);
#pragma unroll
    for (int lq = 0; lq < Q; ++lq)
      if (lq < nf * NQ) {
        if (demote)
          st4(&S.fv[aos(c, lq, Q)], u0);
        else
          st4(&S.fv[aos(c, lq, Q)], vals[lq]);
      }
    if (demote) S.labels[c] = 3;
    if (flags & FL_TAPS) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double z[NV] = {0.0, 0.0, 0.0, 0.0};
        if (!demote && k == 0)
          st4(&S.dofs[aos(c, k, K)], d0);
        else if (!demote && k == 1)
          st4(&S.dofs[aos(c, k, K)], d1);
        else
          st4(&S.dofs[aos(c, k, K)], z);
      }
    }
  }
}

// first-order cells everywhere (SchemeMode::First; evaluate_constant solver.cpp:91-101)
template <int NQ, int NF>
__global__ void __launch_bounds__(kBlock) k_constant(Layout L, Scratch S, const double4* __restrict__ U) {
  constexpr int Q = NF * NQ;
  const int c = blockIdx.x * kBlock + threadIdx.x;
  if (c >= L.n) return;
  const d4 u0 = ld4(&U[c]);
  const int nf = L.nfc[c];
#pragma unroll
  for (int lq = 0; lq < Q; ++lq)
    if (lq < nf * NQ) st4(&S.fv[aos(c, lq, Q)], u0);
}

// ---------------------------------------------------------------------------
// k_flux: per cell, the integrated flux of each of its faces is recomputed
// from the two sides' face-point values in the face's canonical (left ->
// right, primary) orientation, so both owners obtain the bit-identical value
// the reference stores once in face_flux_; the gather then adds +-flux in the
// cell's face order and scales by 1/area (solver.cpp:294-311). No atomics, no
// face_flux_ round trip through HBM. The RK combination is fused.
template <int NQ, int NF>
__global__ void __launch_bounds__(kBlock) k_flux(Layout L, Physics ph, Scratch S, const double4* __restrict__ U,
                                                 RkEpilogue rk, int flags) {
  constexpr int Q = NF * NQ;
  const int c = blockIdx.x * kBlock + threadIdx.x;
  const int lane = threadIdx.x & 31;
  bool live = c < L.n;
  if (*(volatile int*)S.err) return;
  if (flags & (FL_CENSUS | FL_STEP_LABELS)) {
    const int lab = live ? S.labels[c] : -1;
    if ((flags & FL_STEP_LABELS) && live) S.step_labels[c] = static_cast<uint8_t>(lab);
    if (flags & FL_CENSUS) {
      unsigned long long* row = S.census + 4 * static_cast<size_t>(*S.step);
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const unsigned m = __ballot_sync(0xffffffffu, lab == l);
        if (m && lane == __ffs(m) - 1) atomicAdd(&row[l], static_cast<unsigned long long>(__popc(m)));
      }
    }
  }
  if (!live) return;
  const int nf = L.nfc[c];
  double acc[NV] = {0.0, 0.0, 0.0, 0.0};
  const size_t base = static_cast<size_t>(c >> 5) * Q * 32 + lane;
#pragma unroll
  for (int j = 0; j < NF; ++j) {
    if (j < nf) {
      const double nx = __ldg(L.fgeom + aos(c, j * 3 + 0, NF * 3));
      const double ny = __ldg(L.fgeom + aos(c, j * 3 + 1, NF * 3));
      const double len = __ldg(L.fgeom + aos(c, j * 3 + 2, NF * 3));
      const bool own_left = __ldg(L.fsgn + aos(c, j, NF)) > 0;
      double total[NV] = {0.0, 0.0, 0.0, 0.0};
      bool ok = true;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int slq = __ldg(L.self_lq + aos(c, j * NQ + q, Q));
        const int ref = __ldg(L.other_ref + aos(c, j * NQ + q, Q));
        const d4 own = ld4(&S.fv[base + static_cast<size_t>(slq) * 32]);
        d4 oth;
        if (ref >= 0) {
          oth = ld4(&S.fv[ref]);
        } else {
          const BcEntry& bc = ph.bc[-ref - 1];
          if (bc.kind == 2) {
            mirror_state(own.v, nx, ny, oth.v);
          } else if (bc.kind == 3) {
#pragma unroll
            for (int v = 0; v < NV; ++v) oth.v[v] = bc.state[v];
          } else {
            oth = own;
          }
        }
        double F[NV];
        ok &= own_left ? riemann_flux(ph.hll, own.v, oth.v, nx, ny, ph.gamma, F)
                       : riemann_flux(ph.hll, oth.v, own.v, nx, ny, ph.gamma, F);
#pragma unroll
        for (int v = 0; v < NV; ++v) total[v] += ph.qw[q] * F[v];
      }
      if (!ok) record_error(S.err, __ldg(L.face_id + aos(c, j, NF)), S.step);
      const double sgn = own_left ? 1.0 : -1.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] += sgn * (total[v] * len);
    }
  }
  const double inv_vol = L.inv_vol[c];
  double r[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) r[v] = -acc[v] * inv_vol;
  if (rk.rhs_out) st4(&rk.rhs_out[c], r);
  if (rk.out) {
    const double dt = rk.nterms ? *rk.dt : 0.0;
    double o[NV];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      if (i < rk.nterms) {
        const double w = rk.dt_scaled[i] ? rk.coef[i] * dt : rk.coef[i];
        double x[NV];
        if (rk.term[i]) {
          const d4 t = ld4(&rk.term[i][c]);
#pragma unroll
          for (int v = 0; v < NV; ++v) x[v] = t.v[v];
        } else {
#pragma unroll
          for (int v = 0; v < NV; ++v) x[v] = r[v];
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) o[v] = (i == 0) ? w * x[v] : o[v] + w * x[v];
      }
    }
    st4(&rk.out[c], o);
  }
}

// ---------------------------------------------------------------------------
// k_dt: max_stable_dt (solver.cpp:103-111) as a min-reduction over cells; the
// last block turns it into this step's dt = min(cfl*min, t_end - t)
// (run.cpp:100) and advances the device clock by the previous dt.
struct DtState {
  unsigned long long dmin_bits;  // running min of h/speed (positive doubles order as integers)
  unsigned int blocks_done;
  int step;     // steps completed in this run (census row)
  double t;     // time at the start of the current step
  double dt;    // dt of the current step
  double t_end;
  double cfl;
};

__global__ void __launch_bounds__(256) k_dt(Layout L, const double4* __restrict__ U, double gamma, DtState* ds,
                                            int* err) {
  __shared__ double red[8];
  __shared__ bool last;
  if (*(volatile int*)err) return;  // a previous kernel failed: freeze the run
  const int c = blockIdx.x * 256 + threadIdx.x;
  double x = 1e300;
  if (c < L.n) {
    const d4 s = ld4(&U[c]);
    double rho, u, v, p;
    if (cons_to_prim(s.v, gamma, rho, u, v, p)) {
      const double speed = fabs(u) + fabs(v) + sqrt(gamma * p / rho);
      x = L.h[c] / speed;
    } else {
      atomicOr(&err[0], 2);
      atomicMin(&err[2], c);
      atomicMin(&err[3], ds->step + 1);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = smin(x, __shfl_xor_sync(0xffffffffu, x, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = red[0];
    for (int i = 1; i < 8; ++i) b = smin(b, red[i]);
    atomicMin(&ds->dmin_bits, static_cast<unsigned long long>(__double_as_longlong(b)));
    __threadfence();
    const unsigned done = atomicAdd(&ds->blocks_done, 1u);
    last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    const double dmin = __longlong_as_double(static_cast<long long>(atomicAdd(&ds->dmin_bits, 0ull)));
    // run.cpp:97-132: t advances by the previous dt (0 before the first step)
    ds->t = ds->t + ds->dt;
    ds->step += 1;
    const double dt = ds->cfl * dmin;
    ds->dt = smin(dt, ds->t_end - ds->t);
    ds->dmin_bits = static_cast<unsigned long long>(__double_as_longlong(1e300));
    ds->blocks_done = 0;
  }
}

}  // namespace ucfvb
