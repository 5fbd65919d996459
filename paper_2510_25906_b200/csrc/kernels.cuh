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
//   k_face_flux HLLC/HLL at every face Gauss point, integrated face flux
//               (solver.cpp:266-292)
//   k_gather_rk owner-ordered face-to-cell gather (no atomics) fused with the
//               RK stage update (solver.cpp:294-311, time_integrator.cpp:31-38,70-73)
//   k_dt        max_stable_dt min-reduction (solver.cpp:103-111) for a run's first
//               step; later steps reduce it inside the previous final k_gather_rk;
//               k_dt_finalize turns it into the step's dt (device-side t/dt)
#pragma once

#include <cstdint>

#include "device_math.cuh"

namespace ucfvb {

enum : int { FL_DOFS = 1, FL_EVAL = 2, FL_NAD = 4, FL_PRECHECK = 8, FL_TAPS = 16, FL_FALLBACK = 32,
             FL_CENSUS = 64, FL_STEP_LABELS = 128, FL_CHUNKS = 256, FL_DT = 512 };

constexpr int kMaxPatches = 16;

// Programmatic dependent launch: every stage kernel is launched while its
// predecessor drains (cudaLaunchAttributeProgrammaticStreamSerialization, no
// explicit trigger, so the predecessor's blocks have all exited when we run).
// Work on static data may precede pdl_wait(); anything the predecessor wrote
// (and the error word) is read only after it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
constexpr int kBlock = 128;

struct BcEntry {
  int kind;
  double state[4];
};

// everything a stage kernel reads; passed by value (fits the 32 KB param space)
struct Layout {
  int n;       // cells (local: owned + halo on a subdomain)
  int n_owned; // cells whose residual / RK update / dt this solver owns
  int MM;      // padded central stencil size (excluding self)
  int MD;      // padded directional stencil size (excluding self)
  const int* st_idx;        // E = MM           central member cell ids
  const double* pinv;       // E = MM*K  [m][k]
  const double* phi;        // E = Q*K   [lq][k]
  const double* phi01;      // E = Q*2   [lq][k<2] (MUSCL needs only the linear basis values)
  const double* pinv_lin;   // E = MM*2  [m][k]
  const int* dir_idx;       // E = NF*MD [s][m] member cell ids
  const double* pinv_dir;   // E = NF*MD*2 [s][m][k]
  const double* oi;         // E = K*K
  const int* nbr;           // E = NF    face neighbour (-1: none)
  const int* dest;          // E = Q     face-point slot (double4 index into fp) of each cell-local qp
  const int* cface;         // E = NF    (canonical face << 1) | (cell sits on its right / periodic secondary)
  int n_faces;
  const double* fnx;        // [n_faces] canonical unit normal (left -> right)
  const double* fny;
  const double* flen;       // [n_faces] length
  const int8_t* fkind;      // [n_faces] 0: two-sided flux face, 1: boundary condition, 2: periodic secondary (skipped)
  const int8_t* fpatch;     // [n_faces] boundary patch
  const int* fslot;         // [n_faces][2] residual slot (aos(cell, j, NF)) of the left / right owner, -1 none
  const uint8_t* nfc;       // [n] faces per cell
  const double* deact_thr;  // [n] (kappa*h)^n or -inf
  const double* eps2;       // [n] (venkat_kappa*h)^3
  const double* h;          // [n]
  const double* inv_vol;    // [n] 1/area
  // per-cell records of the troubled-cell operator rows (kernels_cells.cuh, CellRec)
  const unsigned char* rec_ca;  // CWENOZ records [n][GC]: group A at 0
  const unsigned char* rec_cb;  //   group B at CA (= rec_ca + CA)
  const unsigned char* rec_ma;  // MUSCL records [n][GM]: group A at 0
  const unsigned char* rec_mb;  //   group B at MA (= rec_ma + MA)
};

struct Physics {
  MarginParams mp;
  double gamma, lambda1p, weno_eps, weno_b;
  // CWENOZ linear weights (reconstruct.cpp:104-106), host-computed with the
  // same IEEE operations: lam0 = 1 - 1/lambda1', lams[nd] = (1 - lam0)/nd, and
  // the correctly rounded reciprocals div_rn needs (nd = directional stencils)
  double lam0, inv_lam0;
  double lams[5], nd_d[5], inv_nd[5];
  int limiter;  // 0 BJ, 1 Venkat
  int hll;      // 0 HLLC, 1 HLL
  double qw[4];  // face quadrature weights (identical on every face)
  BcEntry bc[kMaxPatches];
};

struct Scratch {
  double4* fp;       // face-point values [face][q][side]: the reference's val_left_/val_right_
                     // slots (periodic partners' values land in the primary face's right slot)
  double4* rs;       // +-face_flux_ per cell-face slot [chunk][NF][lane] (the gather's terms, in face order)
  double4* dofs;     // [chunk][K][lane]
  uint8_t* raw;      // raw NAD label | demote-if-linear << 2
  uint8_t* labels;
  uint8_t* step_labels;
  int* list_c;
  int* list_m;
  int* counts;       // [0]/[1] CWENOZ/MUSCL cells (per-cell list lengths), [2]/[3] CWENOZ/MUSCL chunks (chunk-list lengths)
  int2* chunks_c;    // (chunk, lane mask) of 32-cell chunks holding CWENOZ cells
  int2* chunks_m;    // ... MUSCL cells
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
  int c_begin, c_end;      // owned cells [c_begin, c_end) of this launch (c_end 0: all owned cells)
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
// Reconstruction kernels map FOUR lanes to one cell, lane v = lane & 3 owning
// conserved variable v (the reference solves the four variables with the same
// operator, reconstruct.cpp:9-28). Per-cell operator loads are broadcast to
// the four lanes (8 cells x 8 B = 64 B per warp load in the 32-cell chunk
// layout), face-point stores of a cell's double4 are one 32 B sector, and
// each lane keeps only its variable's accumulators in registers.
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ double grp_get(double x, int j) {
  return __shfl_sync(kFull, x, ((threadIdx.x & 31) & ~3) | j);
}
__device__ __forceinline__ bool grp_any(bool b) {
  unsigned x = b ? 1u : 0u;
  x |= __shfl_xor_sync(kFull, x, 1);
  x |= __shfl_xor_sync(kFull, x, 2);
  return x != 0;
}
__device__ __forceinline__ int grp_max(int s) {
  s = max(s, __shfl_xor_sync(kFull, s, 1));
  s = max(s, __shfl_xor_sync(kFull, s, 2));
  return s;
}

// is_physical (euler.hpp:34-36) of the cell's Q face points without the 4x
// redundancy: lane v holds variable v of every point; a 4x4 butterfly
// transpose (shfl_xor 2, then shfl_xor 1, with selects on the lane's two
// index bits) hands lane v all four variables of points v, v+4, ... and each
// lane checks only those. Returns this lane's verdict (OR over the group with
// grp_any).
template <int Q>
__device__ __forceinline__ bool group_nonphysical(const double* vals, int nq_cell, double gamma) {
  const int v = threadIdx.x & 3;
  const bool b0 = v & 1, b1 = v & 2;
  bool bad = false;
#pragma unroll
  for (int r = 0; r < (Q + 3) / 4; ++r) {
    double row[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) row[j] = 4 * r + j < Q ? vals[4 * r + j] : 1.0;
    // step 1 (lane v^2): keep the two points whose bit 1 equals ours, trade the other two
    const double k0 = b1 ? row[2] : row[0], k1 = b1 ? row[3] : row[1];
    const double c0 = __shfl_xor_sync(kFull, b1 ? row[0] : row[2], 2);
    const double c1 = __shfl_xor_sync(kFull, b1 ? row[1] : row[3], 2);
    // step 2 (lane v^1): keep point v, trade point v^1 (own and the v^2 row's values)
    const double A = b0 ? k1 : k0, C = b0 ? c1 : c0;  // variables v, v^2 of point v
    const double B = __shfl_xor_sync(kFull, b0 ? k0 : k1, 1);  // variable v^1
    const double D = __shfl_xor_sync(kFull, b0 ? c0 : c1, 1);  // variable v^3
    const double P0 = b0 ? B : A, Q0 = b0 ? D : C, P1 = b0 ? A : B, Q1 = b0 ? C : D;
    const double st[NV] = {b1 ? Q0 : P0, b1 ? Q1 : P1, b1 ? P0 : Q0, b1 ? P1 : Q1};
    if (4 * r + v < nq_cell) bad |= !is_physical(st, gamma);
  }
  return bad;
}

// NAD detector value (solver.cpp:136-141): v = max over the cell's face points
// q of max(lo - u_q, u_q - hi), starting from v0 = -1e300, from the running
// min / max of u_q. Exact: RN(lo - u) is non-increasing and RN(u - hi)
// non-decreasing in u, so the per-point maxima are attained at min_q u_q and
// max_q u_q; std::max ignores NaN points in both forms (a NaN point leaves
// the running value unchanged), and the sign of a zero v is never observed
// (v only enters comparisons and |v - delta|). The fallback pre-check's
// "some q with max(lo - u_q, u_q - hi) > delta_m" is then v > delta_m.
__device__ __forceinline__ double nad_violation(double v0, double lo, double hi, double qmin, double qmax) {
  return smax(v0, smax(lo - qmin, qmax - hi));
}

// neighbourhood bounds of this lane's variable over {c} U face neighbours
// (solver.cpp:120-129, 207-211)
template <int NF>
__device__ __forceinline__ void var_bounds(const Layout& L, const double* __restrict__ Ud, int c, int v, double u0,
                                           double& lo, double& hi) {
  lo = u0;
  hi = u0;
#pragma unroll
  for (int j = 0; j < NF; ++j) {
    const int nb = __ldg(L.nbr + aos(c, j, NF));
    if (nb >= 0) {
      const double x = __ldg(Ud + 4 * static_cast<size_t>(nb) + v);
      lo = smin(lo, x);
      hi = smax(hi, x);
    }
  }
}

// fallback_check's verdict for one cell (solver.cpp:229-264): positivity of
// the first nq_cell face points spread over the group (group_nonphysical) and
// the relaxed DMP of rho (lane 0) and E (lane 3) against delta_m.
template <int Q>
__device__ __forceinline__ bool group_demote(const Physics& ph, int v, double lo, double hi, const double* vals,
                                             int nq_cell) {
  double dm, dw;
  compute_margins(ph.mp, hi - lo, dm, dw);
  bool bad = group_nonphysical<Q>(vals, nq_cell, ph.gamma);
  if (v == 0 || v == 3) {
#pragma unroll
    for (int lq = 0; lq < Q; ++lq)
      if (lq < nq_cell) bad |= smax(lo - vals[lq], vals[lq] - hi) > dm;
  }
  return grp_any(bad);
}

// ---------------------------------------------------------------------------
// k_central: solve_dofs (reconstruct.cpp:9-28) with the m-loop outermost (each
// accumulator still sums in m order), evaluate_cell (solver.cpp:76-89), the
// raw NAD severity (classify_cells, solver.cpp:113-149) and the fallback
// pre-check a cell that ends Linear needs (solver.cpp:229-264).
template <int K, int NQ, int NF, int MMT, int MDT, bool UNI>
__global__ void __launch_bounds__(kBlock) k_central(Layout L, Physics ph, Scratch S, const double4* __restrict__ U,
                                                    int flags) {
  constexpr int Q = NF * NQ;
  const double* __restrict__ Ud = reinterpret_cast<const double*>(U);
  const int g = blockIdx.x * kBlock + threadIdx.x;
  const int v = g & 3;
  const int c0 = g >> 2;
  pdl_wait();
  if (g == 0) {  // this stage's class-list counters and tie count (read only by later kernels)
    for (int i = 0; i < 4; ++i) S.counts[i] = 0;
  }
  if (*(volatile int*)S.err) return;
  const bool live = c0 < L.n;
  const int c = live ? c0 : L.n - 1;  // dead groups shadow a real cell so the group shuffles stay uniform
  const double u0 = __ldg(Ud + 4 * static_cast<size_t>(c) + v);
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  const int MM = MMT ? MMT : L.MM;
  const int* ip = L.st_idx + aos(c, 0, MM);
  const double* pp = L.pinv + aos(c, 0, MM * K);
#pragma unroll
  for (int m = 0; m < MM; ++m) {
    const int nb = __ldg(ip + m * 32);
    const double d = __ldg(Ud + 4 * static_cast<size_t>(nb) + v) - u0;
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] += __ldg(pp + (m * K + k) * 32) * d;
  }
  double* dofs = reinterpret_cast<double*>(S.dofs);
  if ((flags & FL_DOFS) && live) {
#pragma unroll
    for (int k = 0; k < K; ++k) dofs[4 * aos(c, k, K) + v] = acc[k];
  }
  if (!(flags & FL_EVAL)) return;
  const int nf = UNI ? NF : L.nfc[c];
  const bool detect = (flags & (FL_NAD | FL_PRECHECK)) != 0;
  double lo = u0, hi = u0;
  if (detect) var_bounds<NF>(L, Ud, c, v, u0, lo, hi);
  const double du = hi - lo;
  double dm, dw;
  compute_margins(ph.mp, du, dm, dw);
  double vmax = -1e300, qmin = INFINITY, qmax = -INFINITY;
  bool bad = false;
  const double* fp = L.phi + aos(c, 0, Q * K);
  double* fv = reinterpret_cast<double*>(S.fp);
  double vals[Q];
#pragma unroll
  for (int lq = 0; lq < Q; ++lq) {
    vals[lq] = u0;
    if (lq < nf * NQ) {
      double val = u0;
#pragma unroll
      for (int k = 0; k < K; ++k) val += acc[k] * __ldg(fp + (lq * K + k) * 32);
      vals[lq] = val;
      if (detect) {
        qmin = smin(qmin, val);
        qmax = smax(qmax, val);
      }
    }
  }
  if (detect) {
    vmax = nad_violation(vmax, lo, hi, qmin, qmax);
    if (v == 0 || v == 3) bad |= vmax > dm;
    bad |= group_nonphysical<Q>(vals, nf * NQ, ph.gamma);
  }
  int sev = 0;
  bool tie = false;
  if (detect && (flags & FL_NAD) && (v == 0 || v == 3)) {
    const double thr = L.deact_thr[c];
    if (!(du < thr)) {  // deactivate_smooth (detector.cpp:32-35)
      sev = violation_severity(vmax, dm, dw);
      const double sc = smax(smax(fabs(u0), du), 1e-300);
      tie = fabs(vmax - dm) <= 1e-12 * smax(sc, fabs(dm)) || fabs(vmax - dw) <= 1e-12 * smax(sc, fabs(dw));
    }
    if (thr > 0.0) tie |= fabs(du - thr) <= 1e-12 * thr;
  }
  if (detect) {
    sev = grp_max(sev);
    bad = grp_any(bad);
    tie = grp_any(tie);
    if (flags & FL_NAD) {
      const unsigned tm = __ballot_sync(kFull, tie && v == 0 && live);
      if (tm && (threadIdx.x & 31) == __ffs(tm) - 1) atomicAdd(S.ties, static_cast<unsigned long long>(__popc(tm)));
    }
    if (v == 0 && live) S.raw[c] = static_cast<uint8_t>(sev | (bad ? 4 : 0));
  }
  // a raw label >= CWENOZ survives the spread: the troubled kernels rewrite these face points
  if (live && !((flags & FL_NAD) && sev >= 1)) {
#pragma unroll
    for (int lq = 0; lq < Q; ++lq)
      if (lq < nf * NQ) fv[4 * static_cast<size_t>(__ldg(L.dest + aos(c, lq, Q))) + v] = vals[lq];
  }
}

// ---------------------------------------------------------------------------
// k_spread: labels = spread_flags(raw) as a pull-max over face neighbours
// (detector.cpp:37-53 reads `in` only, so push == pull); Linear cells whose
// pre-check failed become FirstOrder (fallback_check); the troubled classes
// are compacted into lists with one atomic per warp (ballot + popc).
// CPT cells per thread (cell = block base + i * kBlock + thread): on large
// meshes the one-cell form is bound by its per-block latency chain (neighbour
// ids -> raw labels -> block barrier -> returning global atomic -> list
// store) and by ~n/128 same-address atomics per counter; CPT = 8 keeps eight
// independent chains per thread in flight and issues one atomic per 1024 cells.
template <int K, int NQ, int NF, int MMT, int MDT, bool UNI, int CPT>
__global__ void __launch_bounds__(kBlock) k_spread(Layout L, Scratch S, const double4* __restrict__ U, int flags,
                                                   int detect) {
  constexpr int Q = NF * NQ;
  constexpr int NW = kBlock / 32;
  const int base = blockIdx.x * (kBlock * CPT) + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  pdl_wait();
  const bool ok = !*(volatile int*)S.err;
  int lab[CPT], raw[CPT], nb[CPT][NF];
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = base + i * kBlock;
    const bool live = ok && c < L.n;
    raw[i] = live ? S.raw[c] : 0;
    lab[i] = -1;
    if (detect) {
#pragma unroll
      for (int j = 0; j < NF; ++j) nb[i][j] = live ? __ldg(L.nbr + aos(c, j, NF)) : -1;
    } else if (live) {
      lab[i] = S.labels[c];  // frozen classification (detect_every_stage = false)
    }
  }
  if (detect) {
    int rn[CPT][NF];
#pragma unroll
    for (int i = 0; i < CPT; ++i)
#pragma unroll
      for (int j = 0; j < NF; ++j) rn[i][j] = nb[i][j] >= 0 ? S.raw[nb[i][j]] & 3 : 0;
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      int l = raw[i] & 3;
#pragma unroll
      for (int j = 0; j < NF; ++j) l = l < rn[i][j] ? rn[i][j] : l;
      lab[i] = (ok && base + i * kBlock < L.n) ? l : -1;
    }
  }
  unsigned mc[CPT], mm[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = base + i * kBlock;
    if (lab[i] == 0 && (raw[i] & 4)) lab[i] = 3;
    if (lab[i] == 3) {
      const d4 u0 = ld4(&U[c]);
      const int nf = UNI ? NF : L.nfc[c];
#pragma unroll
      for (int lq = 0; lq < Q; ++lq)
        if (lq < nf * NQ) st4(&S.fp[__ldg(L.dest + aos(c, lq, Q))], u0);
      if (flags & FL_TAPS) {
        const double z[NV] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < K; ++k) st4(&S.dofs[aos(c, k, K)], z);
      }
    }
    if (lab[i] >= 0) S.labels[c] = static_cast<uint8_t>(lab[i]);
    mc[i] = __ballot_sync(kFull, lab[i] == 1);
    mm[i] = __ballot_sync(kFull, lab[i] == 2);
  }
  const unsigned lt = (1u << lane) - 1u;
  // per (i, warp) counts -> block-exclusive offsets in cell order; one global
  // atomic per block and class (the lists are unordered across blocks;
  // per-cell results do not depend on the order)
  __shared__ int s_c[CPT * NW], s_m[CPT * NW], s_bc, s_bm;
  const bool chunks = (flags & FL_CHUNKS) != 0;  // one entry per 32-cell chunk (= one warp iteration)
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      s_c[i * NW + w] = chunks ? (mc[i] ? 1 : 0) | (__popc(mc[i]) << 8) : __popc(mc[i]) | ((mc[i] ? 1 : 0) << 8);
      s_m[i * NW + w] = chunks ? (mm[i] ? 1 : 0) | (__popc(mm[i]) << 8) : __popc(mm[i]) | ((mm[i] ? 1 : 0) << 8);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // low byte: list entries (cells, or chunks under FL_CHUNKS); high bits: the
    // other total (list statistics only)
    int tc = 0, tm = 0, xc = 0, xm = 0;
#pragma unroll
    for (int i = 0; i < CPT * NW; ++i) {
      const int a = s_c[i], b = s_m[i];
      s_c[i] = tc;
      s_m[i] = tm;
      tc += a & 255;
      tm += b & 255;
      xc += a >> 8;
      xm += b >> 8;
    }
    const int ic = chunks ? 2 : 0, is = chunks ? 0 : 2;
    s_bc = tc ? atomicAdd(&S.counts[ic], tc) : 0;
    s_bm = tm ? atomicAdd(&S.counts[ic + 1], tm) : 0;
    if (xc) atomicAdd(&S.counts[is], xc);
    if (xm) atomicAdd(&S.counts[is + 1], xm);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    const int c = base + i * kBlock;
    if (chunks) {
      if (lane == 0 && mc[i]) S.chunks_c[s_bc + s_c[i * NW + w]] = make_int2(c >> 5, static_cast<int>(mc[i]));
      if (lane == 0 && mm[i]) S.chunks_m[s_bm + s_m[i * NW + w]] = make_int2(c >> 5, static_cast<int>(mm[i]));
    } else {
      if (lab[i] == 1) S.list_c[s_bc + s_c[i * NW + w] + __popc(mc[i] & lt)] = c;
      if (lab[i] == 2) S.list_m[s_bm + s_m[i * NW + w] + __popc(mm[i] & lt)] = c;
    }
  }
}

// ---------------------------------------------------------------------------
// k_cwenoz: directional r=1 solves (reconstruct.cpp:43-57), SI via OI, tau,
// nonlinear weights, blend (cwenoz_blend_scalar reconstruct.cpp:99-150),
// evaluation and fallback epilogue. The blend is per variable in the
// reference, so lane v owns variable v end to end.
template <int K, int NQ, int NF, int MMT, int MDT, bool UNI>
__global__ void __launch_bounds__(kBlock) k_cwenoz(Layout L, Physics ph, Scratch S, const double4* __restrict__ U,
                                                   int flags) {
  constexpr int Q = NF * NQ;
  constexpr int CPB = kBlock / 4;  // cells per block iteration
  const double* __restrict__ Ud = reinterpret_cast<const double*>(U);
  const bool all = (flags & FL_NAD) == 0;  // forced CWENOZ mode: every cell, no list
  pdl_wait();
  const int count = all ? L.n : S.counts[0];
  if (*(volatile int*)S.err) return;
  if (!(ph.lambda1p > 1.0)) {  // cwenoz_blend_scalar throws (reconstruct.cpp:102-103)
    if (count > 0 && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&S.err[0], 4);
    return;
  }
  const int v = threadIdx.x & 3;
  double* dofs = reinterpret_cast<double*>(S.dofs);
  double* fv = reinterpret_cast<double*>(S.fp);
  for (int base = blockIdx.x * CPB; base < count; base += gridDim.x * CPB) {
    const int i = base + (threadIdx.x >> 2);
    const bool live = i < count;
    const int c = all ? (live ? i : count - 1) : S.list_c[live ? i : count - 1];
    const double u0 = __ldg(Ud + 4 * static_cast<size_t>(c) + v);
    const int nf = UNI ? NF : L.nfc[c];
    double dir[NF][2];
    const int MD = MDT ? MDT : L.MD;
#pragma unroll
    for (int s = 0; s < NF; ++s) {
      dir[s][0] = 0.0;
      dir[s][1] = 0.0;
      if (s < nf) {
#pragma unroll
        for (int m = 0; m < MD; ++m) {
          const int nb = __ldg(L.dir_idx + aos(c, s * MD + m, NF * MD));
          const double d = __ldg(Ud + 4 * static_cast<size_t>(nb) + v) - u0;
          dir[s][0] += __ldg(L.pinv_dir + aos(c, (s * MD + m) * 2 + 0, NF * MD * 2)) * d;
          dir[s][1] += __ldg(L.pinv_dir + aos(c, (s * MD + m) * 2 + 1, NF * MD * 2)) * d;
        }
      }
    }
    const int st = nf + 1;
    const double lam0 = 1.0 - 1.0 / ph.lambda1p;
    const double lams = (1.0 - lam0) / (st - 1);
    double p1[K];
#pragma unroll
    for (int k = 0; k < K; ++k) p1[k] = dofs[4 * aos(c, k, K) + v];
#pragma unroll
    for (int s = 0; s < NF; ++s)
      if (s < nf) {
        p1[0] -= lams * dir[s][0];
        p1[1] -= lams * dir[s][1];
      }
#pragma unroll
    for (int k = 0; k < K; ++k) p1[k] /= lam0;
    // SI_0 = p1^T OI p1, row then dot (smoothness_indicator reconstruct.cpp:88-97)
    const double* oi = L.oi + aos(c, 0, K * K);
    double si0 = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < K; ++q) t += __ldg(oi + (k * K + q) * 32) * p1[q];
      si0 += p1[k] * t;
    }
    const double o00 = __ldg(oi), o01 = __ldg(oi + 32), o10 = __ldg(oi + K * 32), o11 = __ldg(oi + (K + 1) * 32);
    double sis[NF];
    double tau = 0.0;
#pragma unroll
    for (int s = 0; s < NF; ++s)
      if (s < nf) {
        const double a0 = dir[s][0], a1 = dir[s][1];
        sis[s] = o00 * a0 * a0 + (o01 + o10) * a0 * a1 + o11 * a1 * a1;
        tau += fabs(sis[s] - si0);
      }
    tau /= (st - 1);
    tau = tau_pow(tau, ph.weno_b);
    double om0 = lam0 * (1.0 + tau / (ph.weno_eps + si0));
    double oms[NF];
    double wsum = om0;
#pragma unroll
    for (int s = 0; s < NF; ++s)
      if (s < nf) {
        oms[s] = lams * (1.0 + tau / (ph.weno_eps + sis[s]));
        wsum += oms[s];
      }
    om0 /= wsum;
#pragma unroll
    for (int k = 0; k < K; ++k) p1[k] = om0 * p1[k];
#pragma unroll
    for (int s = 0; s < NF; ++s)
      if (s < nf) {
        const double w = oms[s] / wsum;
        p1[0] += w * dir[s][0];
        p1[1] += w * dir[s][1];
      }
    // evaluate_cell + fallback epilogue
    const double* fp = L.phi + aos(c, 0, Q * K);
    double vals[Q];
#pragma unroll
    for (int lq = 0; lq < Q; ++lq) {
      vals[lq] = u0;
      if (lq < nf * NQ) {
#pragma unroll
        for (int k = 0; k < K; ++k) vals[lq] += p1[k] * __ldg(fp + (lq * K + k) * 32);
      }
    }
    bool demote = false;
    if (flags & FL_FALLBACK) {
      double lo, hi;
      var_bounds<NF>(L, Ud, c, v, u0, lo, hi);
      demote = group_demote<Q>(ph, v, lo, hi, vals, nf * NQ);
    }
    if (live) {
#pragma unroll
      for (int lq = 0; lq < Q; ++lq)
        if (lq < nf * NQ) fv[4 * static_cast<size_t>(__ldg(L.dest + aos(c, lq, Q))) + v] = demote ? u0 : vals[lq];
      if (demote && v == 0) S.labels[c] = 3;
      if (flags & FL_TAPS) {
#pragma unroll
        for (int k = 0; k < K; ++k) dofs[4 * aos(c, k, K) + v] = demote ? 0.0 : p1[k];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// k_muscl: r=1 LSQ gradient (solve_dofs_linear reconstruct.cpp:30-41), BJ or
// Venkatakrishnan limiter per variable (reconstruct.cpp:59-86), limited
// evaluation (solver.cpp:189-221) and fallback epilogue; lane v owns variable v.
template <int K, int NQ, int NF, int MMT, int MDT, bool UNI>
__global__ void __launch_bounds__(kBlock) k_muscl(Layout L, Physics ph, Scratch S, const double4* __restrict__ U,
                                                  int flags) {
  constexpr int Q = NF * NQ;
  constexpr int CPB = kBlock / 4;
  const double* __restrict__ Ud = reinterpret_cast<const double*>(U);
  const bool all = (flags & FL_NAD) == 0;  // forced MUSCL mode
  pdl_wait();
  const int count = all ? L.n : S.counts[1];
  if (*(volatile int*)S.err) return;
  const int v = threadIdx.x & 3;
  double* dofs = reinterpret_cast<double*>(S.dofs);
  double* fv = reinterpret_cast<double*>(S.fp);
  const bool venkat = ph.limiter == 1;
  for (int base = blockIdx.x * CPB; base < count; base += gridDim.x * CPB) {
    const int i = base + (threadIdx.x >> 2);
    const bool live = i < count;
    const int c = all ? (live ? i : count - 1) : S.list_m[live ? i : count - 1];
    const double u0 = __ldg(Ud + 4 * static_cast<size_t>(c) + v);
    const int nf = UNI ? NF : L.nfc[c];
    double l0 = 0.0, l1 = 0.0;
    const int MM = MMT ? MMT : L.MM;
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      const int nb = __ldg(L.st_idx + aos(c, m, MM));
      const double d = __ldg(Ud + 4 * static_cast<size_t>(nb) + v) - u0;
      l0 += __ldg(L.pinv_lin + aos(c, m * 2 + 0, MM * 2)) * d;
      l1 += __ldg(L.pinv_lin + aos(c, m * 2 + 1, MM * 2)) * d;
    }
    double lo, hi;
    var_bounds<NF>(L, Ud, c, v, u0, lo, hi);
    const double* fp = L.phi + aos(c, 0, Q * K);
    double p0s[Q], p1s[Q];
    double theta = 1.0;
    const double eps2 = venkat ? L.eps2[c] : 0.0;
#pragma unroll
    for (int lq = 0; lq < Q; ++lq) {
      p0s[lq] = 0.0;
      p1s[lq] = 0.0;
      if (lq < nf * NQ) {
        p0s[lq] = __ldg(fp + (lq * K + 0) * 32);
        p1s[lq] = __ldg(fp + (lq * K + 1) * 32);
        const double qv = u0 + l0 * p0s[lq] + l1 * p1s[lq];
        theta = venkat ? venkat_update(theta, u0, lo, hi, qv, eps2) : bj_update(theta, u0, lo, hi, qv);
      }
    }
    if (!venkat) theta = smax(theta, 0.0);
    const double d0 = theta * l0, d1 = theta * l1;
    double vals[Q];
#pragma unroll
    for (int lq = 0; lq < Q; ++lq) {
      double o = u0;
      o += d0 * p0s[lq];
      o += d1 * p1s[lq];
      vals[lq] = o;  // dofs k >= 2 are zero: adding 0*phi leaves o unchanged
    }
    bool demote = false;
    if (flags & FL_FALLBACK) {
      // the fallback DMP uses the rho/E bounds, which lanes 0 and 3 hold already
      demote = group_demote<Q>(ph, v, lo, hi, vals, nf * NQ);
    }
    if (live) {
#pragma unroll
      for (int lq = 0; lq < Q; ++lq)
        if (lq < nf * NQ) fv[4 * static_cast<size_t>(__ldg(L.dest + aos(c, lq, Q))) + v] = demote ? u0 : vals[lq];
      if (demote && v == 0) S.labels[c] = 3;
      if (flags & FL_TAPS) {
#pragma unroll
        for (int k = 0; k < K; ++k)
          dofs[4 * aos(c, k, K) + v] = demote ? 0.0 : (k == 0 ? d0 : (k == 1 ? d1 : 0.0));
      }
    }
  }
}

// first-order cells everywhere (SchemeMode::First; evaluate_constant solver.cpp:91-101)
template <int NQ, int NF, bool UNI>
__global__ void __launch_bounds__(kBlock) k_constant(Layout L, Scratch S, const double4* __restrict__ U) {
  constexpr int Q = NF * NQ;
  const int c = blockIdx.x * kBlock + threadIdx.x;
  pdl_wait();
  if (c >= L.n) return;
  const d4 u0 = ld4(&U[c]);
  const int nf = UNI ? NF : L.nfc[c];
#pragma unroll
  for (int lq = 0; lq < Q; ++lq)
    if (lq < nf * NQ) st4(&S.fp[__ldg(L.dest + aos(c, lq, Q))], u0);
}

// ---------------------------------------------------------------------------
// max_stable_dt support (solver.cpp:103-111) + device-side t/dt of run_steps
struct DtState {
  unsigned long long dmin_bits;  // running min of h/speed (positive doubles order as integers)
  int dt_bad;   // a cell's state was non-physical when its h/speed was taken
  int step;     // steps completed in this run (census row)
  double t;     // time at the start of the current step
  double dt;    // dt of the current step
  double t_end;
  double cfl;
  double dmin;  // collected min(h/speed) (all-reduced across ranks before k_dt_finalize)
  double* dt_log;  // nullable [steps]: each step's dt (run.cpp:111 CensusRow::dt)
  int until;       // 1: stop at run_simulation's loop condition t < t_end - 1e-14 t_end (run.cpp:96)
};

// err[0] bit set when an `until` run reached t_end: every later kernel of the
// batch exits early (like after an error); the host does not report it
constexpr int kErrDone = 8;

// max_stable_dt's per-cell term (solver.cpp:103-111): h_c / (|u| + |v| + a)
__device__ __forceinline__ bool dt_term(const double* s, double gamma, double h, double& x) {
  double rho, u, v, p;
  if (!cons_to_prim(s, gamma, rho, u, v, p)) return false;
  const double speed = fabs(u) + fabs(v) + sqrt(gamma * p / rho);
  x = h / speed;
  return true;
}

// block-wide min of x folded into ds->dmin_bits (every thread of the block must call)
__device__ __forceinline__ void block_min_into(double x, DtState* ds) {
  __shared__ double red[kBlock / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = smin(x, __shfl_xor_sync(0xffffffffu, x, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = red[0];
    for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) b = smin(b, red[i]);
    if (b < 1e300) atomicMin(&ds->dmin_bits, static_cast<unsigned long long>(__double_as_longlong(b)));
  }
}

// min over owned cells of h/speed into ds->dmin_bits (the first step of a run;
// later steps get it from the previous step's final k_gather_rk)
__global__ void __launch_bounds__(kBlock) k_dt(Layout L, const double4* __restrict__ U, double gamma, DtState* ds,
                                               int* err) {
  pdl_wait();
  if (*(volatile int*)err) return;  // block-uniform
  const int c = blockIdx.x * kBlock + threadIdx.x;
  double x = 1e300;
  if (c < L.n_owned) {
    const d4 s = ld4(&U[c]);
    if (!dt_term(s.v, gamma, L.h[c], x)) {
      x = 1e300;
      ds->dt_bad = 1;
      atomicMin(&err[2], c);
    }
  }
  block_min_into(x, ds);
}

// collect the reduced min (and reset the accumulator)
__device__ __forceinline__ void dt_collect(DtState* ds) {
  ds->dmin = __longlong_as_double(static_cast<long long>(ds->dmin_bits));
  ds->dmin_bits = static_cast<unsigned long long>(__double_as_longlong(1e300));
}

// start of a step: raise a pending dt failure (max_stable_dt throws before the
// step touches the state) or advance t by the previous dt and set this step's
// dt = min(cfl * dmin, t_end - t) (run.cpp:97-132, solver.cpp:110)
__device__ __forceinline__ void dt_finalize(DtState* ds, int* err) {
  if (ds->until) {
    const double t = ds->t + ds->dt;
    if (!(t < ds->t_end - 1e-14 * ds->t_end)) {  // the loop ends before max_stable_dt is taken
      ds->t = t;
      ds->dt = 0.0;
      atomicOr(&err[0], kErrDone);
      return;
    }
  }
  if (ds->dt_bad) {
    atomicOr(&err[0], 2);
    atomicMin(&err[3], ds->step + 1);
    return;
  }
  ds->t = ds->t + ds->dt;  // 0 before the first step
  ds->step += 1;
  const double dt = ds->cfl * ds->dmin;
  ds->dt = smin(dt, ds->t_end - ds->t);
  if (ds->dt_log) ds->dt_log[ds->step] = ds->dt;
}

__global__ void k_dt_collect(DtState* ds) {
  pdl_wait();
  dt_collect(ds);
}

__global__ void k_dt_finalize(DtState* ds, int* err, int collect) {
  pdl_wait();
  if (*(volatile int*)err) return;
  if (collect) dt_collect(ds);
  dt_finalize(ds, err);
}

// ---------------------------------------------------------------------------
// k_face_flux: assemble_fluxes pass 1 (solver.cpp:266-292). One lane per
// (face, Gauss point), NQ consecutive lanes per face: UL/UR are read as one
// contiguous 64 B pair from the face-major fp array, the Riemann flux is
// weighted, and the face's lanes sum total = (0 + w_0 F_0) + w_1 F_1 ... in q
// order; face_flux = total * length. Periodic secondaries are skipped (their
// flux lives on the primary, solver.cpp:272); boundary faces evaluate the
// patch's BC from UL (solver.cpp:22-34, 283).
template <int NQ>
__global__ void __launch_bounds__(kBlock) k_face_flux(Layout L, Physics ph, Scratch S) {
  constexpr int FPW = 32 / NQ;  // faces per warp
  const int lane = threadIdx.x & 31;
  const int fs = lane / NQ;
  const int q = lane - fs * NQ;
  const int warp = (blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int f0 = warp * FPW + fs;
  const bool in = fs < FPW && f0 < L.n_faces;
  const int f = in ? f0 : 0;
  const int kind = in ? L.fkind[f] : 2;
  const double nx = L.fnx[f], ny = L.fny[f];  // static geometry: fetched while the predecessor drains
  pdl_wait();
  const int err0 = *(volatile int*)S.err;
  double t[NV] = {0.0, 0.0, 0.0, 0.0};
  if (kind != 2) {
    const d4 UL = ld4(&S.fp[(static_cast<size_t>(f) * NQ + q) * 2 + 0]);
    d4 UR;
    if (kind == 0) {
      UR = ld4(&S.fp[(static_cast<size_t>(f) * NQ + q) * 2 + 1]);
    } else {
      const BcEntry& bc = ph.bc[L.fpatch[f]];
      if (bc.kind == 2) {
        mirror_state(UL.v, nx, ny, UR.v);
      } else if (bc.kind == 3) {
#pragma unroll
        for (int v = 0; v < NV; ++v) UR.v[v] = bc.state[v];
      } else {
        UR = UL;
      }
    }
    double F[NV];
    if (!riemann_flux(ph.hll, UL.v, UR.v, nx, ny, ph.gamma, F) && !err0) record_error(S.err, f, S.step);
    const double w = ph.qw[q];
#pragma unroll
    for (int v = 0; v < NV; ++v) t[v] = w * F[v];
  }
  double total[NV] = {0.0, 0.0, 0.0, 0.0};
  const int g0 = fs * NQ;
#pragma unroll
  for (int qq = 0; qq < NQ; ++qq)
#pragma unroll
    for (int v = 0; v < NV; ++v) total[v] += __shfl_sync(kFull, t[v], min(g0 + qq, 31));
  if (kind == 2 || q != 0 || err0) return;
  const double len = L.flen[f];
  double o[NV], m[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    o[v] = total[v] * len;  // face_flux_ (solver.cpp:292)
    m[v] = -1.0 * o[v];     // sgn * face_flux_ for the right / periodic-secondary owner (solver.cpp:301-306)
  }
  const int sl = L.fslot[2 * f], sr = L.fslot[2 * f + 1];
  if (sl >= 0) st4(&S.rs[sl], o);
  if (sr >= 0) st4(&S.rs[sr], m);
}

// ---------------------------------------------------------------------------
// k_gather_rk: assemble_fluxes pass 2 (solver.cpp:294-311) fused with the RK
// stage combination, one thread per cell (all four variables, 32 B loads and
// stores: the pass is latency-bound and this keeps 3 + nterms independent
// loads in flight per thread). acc = sum over the cell's faces, in the cell's
// face order, of +-face_flux (scattered into the cell's slots by k_face_flux);
// residual = -acc * (1/area); out = sum_i coef_i * term_i left to right
// (combine2, time_integrator.cpp:31-38; final SSPRK(5,4) line :70-73).
// Owner-ordered: no atomics.
template <int NF, bool UNI, int NT>  // NT >= rk.nterms: registers for the prefetched RK terms
__global__ void __launch_bounds__(kBlock) k_gather_rk(Layout L, Scratch S, RkEpilogue rk, int flags, DtState* ds,
                                                      double gamma) {
  const int cend = rk.c_end ? rk.c_end : L.n_owned;
  const int c0 = rk.c_begin + blockIdx.x * kBlock + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool live = c0 < cend;
  const int c = live ? c0 : cend - 1;
  // RK terms were written by earlier stages and 1/area is static: fetched while the face kernel drains
  d4 term[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    if (i < rk.nterms && rk.term[i]) {
      term[i] = ld4(rk.term[i] + c);
    } else {
      term[i] = d4{{0.0, 0.0, 0.0, 0.0}};
    }
  }
  const double inv_vol = L.inv_vol[c];
  pdl_wait();
  const int err0 = *(volatile int*)S.err;
  const int nf = UNI ? NF : L.nfc[c];
  double acc[NV] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < NF; ++j)
    if (j < nf) {
      const d4 r = ld4(&S.rs[aos(c, j, NF)]);
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] += r.v[v];
    }
  if (flags & (FL_CENSUS | FL_STEP_LABELS)) {
    const int lab = live ? S.labels[c] : -1;
    if ((flags & FL_STEP_LABELS) && live && !err0) S.step_labels[c] = static_cast<uint8_t>(lab);
    if ((flags & FL_CENSUS) && !err0) {
      unsigned long long* row = S.census + 4 * static_cast<size_t>(*S.step);
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const unsigned m = __ballot_sync(kFull, lab == l);
        if (m && lane == __ffs(m) - 1) atomicAdd(&row[l], static_cast<unsigned long long>(__popc(m)));
      }
    }
  }
  double r[NV], o[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    r[v] = -acc[v] * inv_vol;
    o[v] = 0.0;
  }
  if (rk.out) {
    const double dt = rk.nterms ? *rk.dt : 0.0;
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      if (i < rk.nterms) {
        const double w = rk.dt_scaled[i] ? rk.coef[i] * dt : rk.coef[i];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const double x = rk.term[i] ? term[i].v[v] : r[v];
          o[v] = (i == 0) ? w * x : o[v] + w * x;
        }
      }
    }
  }
  if (live && !err0) {
    if (rk.rhs_out) st4(rk.rhs_out + c, r);
    if (rk.out) st4(rk.out + c, o);
  }
  if (flags & FL_DT) {  // max_stable_dt of the new state, for the next step (block-uniform branch)
    double x = 1e300;
    if (live && !err0 && !dt_term(o, gamma, L.h[c], x)) {
      x = 1e300;
      ds->dt_bad = 1;
      atomicMin(&S.err[2], c);
    }
    block_min_into(x, ds);
  }
}

// ---------------------------------------------------------------------------
// pack the owned cells a peer needs into a contiguous send buffer
__global__ void __launch_bounds__(256) k_halo_pack(const double4* __restrict__ U, const int* __restrict__ idx, int n,
                                                   double4* __restrict__ out) {
  const int i = blockIdx.x * 256 + threadIdx.x;
  pdl_wait();
  if (i < n) out[i] = U[idx[i]];
}

}  // namespace ucfvb
