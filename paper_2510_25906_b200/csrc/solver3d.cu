// 3D stage pass on B200 (BASELINE configs 4-5).
//
// Five conserved variables per cell. Reconstruction kernels run one WARP PER
// CONSERVED VARIABLE over a chunk of 32 cells (block = 5 warps = 160
// threads): lane = cell, warp = variable, so every per-cell operator load is
// a coalesced 256 B line (32-cell AoSoA chunks, as the 2D path), the five
// warps of a block read the same operator lines (L1 hits after the first),
// and each thread keeps only its variable's K accumulators. The cross-variable
// steps (NAD severity over rho and E, positivity of the face values) meet in
// shared memory. Op orders follow oracle/ucfv3_port.c (the 3D restatement of
// the reference's 2D functions); kernels are compiled with --fmad=false and
// the K x M / Q x K contractions use explicit __fma_rn, as the restatement
// does with fma() (no reference arithmetic exists in 3D; see its header).
// Stencil values arrive by 8-byte cp.async (all in flight at once).
// Lattice-class meshes (config 5) number their cells type-blocked, so a block
// sees one operator row: it is staged in shared memory once per kernel
// (STAGED) and the contractions run as fp64 tensor-core tiles (DMMA
// m8n8k4, bit-identical to the fma chain in k order; dmma884 below).
//
//   k3_central   solve_dofs + evaluate_cell + NAD raw label + fallback pre-check  (solver.cpp:336-349, 113-149, 229-264)
//   k3_spread    spread_flags (pull form) + class lists + Linear-cell demotion    (detector.cpp:37-53)
//   k3_cwenoz    directional solves + CWENOZ blend + evaluate + fallback          (solver.cpp:167-188, reconstruct.cpp:43-150)
//   k3_muscl     r=1 solve + BJ/Venkatakrishnan limiter + evaluate + fallback    (solver.cpp:189-221)
//   k3_face_flux HLLC/HLL at every face Gauss point, summed in qp order          (solver.cpp:266-295)
//                (k3_face_flux_lanes: one lane per point, shuffle sum, for power-of-two point counts)
//   k3_gather_rk owner-ordered face->cell sum + SSP-RK combination               (solver.cpp:296-311, time_integrator.cpp:31-38)
//   k3_dt        max_stable_dt                                                   (solver.cpp:103-111)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "device_math.cuh"
#include "layout.hpp"
#include "solver3d.hpp"
#include "decompose3.hpp"
#include "nccl_dl.hpp"
#include "tma.cuh"

namespace ucfvb {
namespace {

constexpr int V5 = 5;
constexpr int MD3 = 6;
constexpr int kCwList = 0, kMuList = 1, kBadFace = 2, kBadCell = 3, kCnt0 = 4;
// counters[kHalt] != 0 once a recorded failure has been seen by a later
// kernel: every state-writing kernel and every error-recording kernel after
// that exits, so the failing kernel's min face / cell stays deterministic and
// U stays at the failing step's input (the reference throws before touching state_)
constexpr int kHalt = 0;

#define CK3(x)                                                                                      \
  do {                                                                                              \
    cudaError_t e_ = (x);                                                                           \
    if (e_ != cudaSuccess) throw ApiError(UCFVB_CUDA, std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x); \
  } while (0)

__device__ __forceinline__ size_t ao(int c, int e, int E) {
  return (static_cast<size_t>(c >> 5) * E + e) * 32 + (c & 31);
}

// pressure / is_physical / cons_to_prim with three momenta (euler.hpp:30-45)
__device__ __forceinline__ double pressure3(const double* s, double g) {
  return (g - 1.0) * (s[4] - 0.5 * (s[1] * s[1] + s[2] * s[2] + s[3] * s[3]) / s[0]);
}
__device__ __forceinline__ bool is_physical3(const double* s, double g) { return s[0] > 0.0 && pressure3(s, g) > 0.0; }

struct P3 {
  double rho, u, v, w, un, p, E, a;
};
__device__ __forceinline__ bool prep3(const double* s, const double* n, double g, P3& f) {
  if (!(s[0] > 0.0)) return false;
  const double u = s[1] / s[0], v = s[2] / s[0], w = s[3] / s[0];
  const double p = (g - 1.0) * (s[4] - 0.5 * s[0] * (u * u + v * v + w * w));
  if (!(p > 0.0)) return false;
  f.rho = s[0], f.u = u, f.v = v, f.w = w, f.p = p;
  f.un = u * n[0] + v * n[1] + w * n[2];
  f.E = s[4];
  f.a = sqrt(g * p / s[0]);
  return true;
}
__device__ __forceinline__ void phys_flux3(const P3& f, const double* n, double* o) {
  o[0] = f.rho * f.un;
  o[1] = f.rho * f.u * f.un + f.p * n[0];
  o[2] = f.rho * f.v * f.un + f.p * n[1];
  o[3] = f.rho * f.w * f.un + f.p * n[2];
  o[4] = (f.E + f.p) * f.un;
}
__device__ __forceinline__ void cons3(const P3& f, double* o) {
  o[0] = f.rho, o[1] = f.rho * f.u, o[2] = f.rho * f.v, o[3] = f.rho * f.w, o[4] = f.E;
}
// hllc_flux / hll_flux (euler.cpp:40-89), Cartesian form of oracle/ucfv3_port.c
__device__ __forceinline__ bool riemann3(bool hll, const double* UL, const double* UR, const double* n, double g,
                                         double* out) {
  P3 L, R;
  if (!prep3(UL, n, g, L) || !prep3(UR, n, g, R)) return false;
  const double SL = smin(L.un - L.a, R.un - R.a);
  const double SR = smax(L.un + L.a, R.un + R.a);
  if (SL >= 0.0) {
    phys_flux3(L, n, out);
  } else if (SR <= 0.0) {
    phys_flux3(R, n, out);
  } else if (!hll) {
    const double dL = L.rho * (SL - L.un);
    const double dR = R.rho * (SR - R.un);
    const double Ss = (R.p - L.p + L.un * dL - R.un * dR) / (dL - dR);
    const bool left = Ss >= 0.0;
    const P3& K = left ? L : R;
    const double SK = left ? SL : SR;
    double WK[5], FK[5], Ws[5];
    cons3(K, WK);
    phys_flux3(K, n, FK);
    const double coef = K.rho * (SK - K.un) / (SK - Ss);
    Ws[0] = coef;
    Ws[1] = coef * (Ss * n[0] + (K.u - K.un * n[0]));
    Ws[2] = coef * (Ss * n[1] + (K.v - K.un * n[1]));
    Ws[3] = coef * (Ss * n[2] + (K.w - K.un * n[2]));
    Ws[4] = coef * (WK[4] / K.rho + (Ss - K.un) * (Ss + K.p / (K.rho * (SK - K.un))));
#pragma unroll
    for (int v = 0; v < V5; ++v) out[v] = FK[v] + SK * (Ws[v] - WK[v]);
  } else {
    double FL[5], FR[5], WL[5], WR[5];
    phys_flux3(L, n, FL);
    phys_flux3(R, n, FR);
    cons3(L, WL);
    cons3(R, WR);
#pragma unroll
    for (int v = 0; v < V5; ++v) out[v] = (SR * FL[v] - SL * FR[v] + SL * SR * (WR[v] - WL[v])) / (SR - SL);
  }
  return true;
}

struct Dev3 {
  int n, nF, n_ops, n_owned;
  // per cell, 32-cell AoSoA
  const int32_t* central;  // [M+1]
  const int32_t* nbr;      // [NF]
  const int32_t* slot;     // [Q]
  const int32_t* cface;    // [NF] (face << 1) | side
  const int32_t* opi;      // [n]
  const double *thr, *eps2, *inv_vol, *h;
  // per operator row, 32-row AoSoA
  const double* pinv;      // [M][K]
  const double* pinv_lin;  // [M][3]
  const int32_t* dirm;     // [NF][MD]
  const double* pinv_dir;  // [NF][3][MD]
  const double* oi;        // [K][K]
  const double* phi;       // [Q][K]
  // faces
  const double* fnrm;  // [nF][NQ][3]
  const double* fwa;   // [nF][NQ]
  const uint8_t* fown; // subdomains: 1 for faces of owned cells (the only ones that may report errors)
};

struct Phys3 {
  double gamma, cfl, lambda1p, weno_eps, weno_b, lam0, lams;
  double inv_lam0;  // RN(1 / lam0) for div_rn (exact_math.h)
  MarginParams mg;
  int mode, limiter, hll;
};

struct Work3 {
  double* fp;        // [nF][NQ][2][5]
  double* ff;        // [nF][5]
  double* bounds;    // AoSoA [4]
  uint8_t* raw;      // raw label | prefail << 2
  uint8_t* labels;
  int32_t* lists;    // [2][ntl][cap] class lists (ntl = 1, or one per lattice type when staged)
  int32_t* counters; // [0] halt, [1] unused, bad face, bad cell, then [4 + L*ntl + t] list lengths
  int ntl, cap;
  unsigned long long* dtmin;
  double* dt;        // device dt of the current step
  double* t;         // device time
  unsigned long long* ties;
};
__device__ __forceinline__ int cnt_idx(const Work3& W, int L, int t) { return kCnt0 + L * W.ntl + t; }
__device__ __forceinline__ bool halted(const Work3& W) { return *(volatile int32_t*)&W.counters[kHalt] != 0; }
// a failure recorded by an earlier kernel: raise the halt flag (idempotent)
__device__ __forceinline__ bool failed_before(const Work3& W) {
  const volatile int32_t* c = W.counters;
  if (c[kBadFace] != 0x7fffffff || c[kBadCell] != 0x7fffffff) {
    if (threadIdx.x == 0) W.counters[kHalt] = 1;
    return true;
  }
  return c[kHalt] != 0;
}
__device__ __forceinline__ int32_t* list_of(const Work3& W, int L, int t) {
  return W.lists + (static_cast<size_t>(L) * W.ntl + t) * W.cap;
}


// fp64 tensor-core tile D(8x8) += A(8x4) B(4x8) (DMMA). Measured on B200
// (scripts/dmma_order.cu, profiles/dmma_order.json): every element equals the
// sequential chain fma(a3,b3,fma(a2,b2,fma(a1,b1,fma(a0,b0,c)))), i.e. the
// oracle's fma accumulation in k order, so tensor-core solves stay bit-exact.
// Fragments (lane l): a = A[l/4][l%4], b = B[l%4][l/4], d = D[l/4][2(l%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// dynamic shared memory of the reconstruction kernels: the cp.async stencil
// gather [G][160] and, after the solve, the face values [Q][5][33] (union)
__host__ __device__ constexpr size_t smem3_bytes(int G, int Q) {
  return 8 * static_cast<size_t>((G * 160 > Q * V5 * 33) ? G * 160 : Q * V5 * 33);
}

// Shared-memory strides of the lattice-class tensor-core (DMMA) kernels, all in
// doubles. An m8n8k4 fragment load has lane (fr = lane / 4, fc = lane % 4) read
// element (row 4*ks + fc, column fr) or (row fr, column fc): with a row stride
// = 4 (mod 16) the 16 lanes of a half warp fall into 16 distinct 8-byte banks
// (strides 160 / 32 / K = 19 gave 2- to 8-way conflicts: 47 % of the central
// kernel's shared-memory wavefronts were replays).
//   gather buffer  xs[row g][variable v][cell l] = g * kXS + v * kVS + l
//   operator rows  pinv [M][KP], phi [Q][KP], OI [K][KP], KP = kpad(K)
//   dofs           sd[v][k][cell] = (v * K + k) * kRS + cell
// The gather itself is issued transposed: thread t copies (cell t / 5,
// variable t % 5), so the five variables of a stencil member are one
// contiguous 40-byte read and a warp's request touches 2-3 cache lines instead
// of 10 (lane = cell at a 40-byte stride); kVS = 35 spreads the five
// variables of a cell over different banks for those writes.
constexpr int kXS = 180, kVS = 35, kRS = 36;
__host__ __device__ constexpr int kpad(int K) {
  int p = K;
  while (p % 16 != 4 && p % 16 != 12) ++p;
  return p;
}
// lattice-class MUSCL: gather rows of kMS doubles (5 variables at kVS), then the face values
constexpr int kMS = 5 * kVS;
__host__ __device__ constexpr size_t muscl_union(int G, int Q) {
  const size_t u = (static_cast<size_t>(G) * kMS > static_cast<size_t>(Q * V5 * 33)) ? static_cast<size_t>(G) * kMS
                                                                                    : static_cast<size_t>(Q * V5 * 33);
  return (u + 1) & ~static_cast<size_t>(1);  // the operator rows behind it are read as double2
}
// union buffer of a DMMA kernel: the gather [G][kXS], later face values [Q][5][33] + dofs [5][K][kRS]
__host__ __device__ constexpr size_t dm_union(int G, int Q, int K) {
  return (static_cast<size_t>(G) * kXS > static_cast<size_t>(Q * V5 * 33 + V5 * K * kRS))
             ? static_cast<size_t>(G) * kXS
             : static_cast<size_t>(Q * V5 * 33 + V5 * K * kRS);
}

// evaluate the reconstruction of (cell, var) at its Q face points, stage the
// values for the positivity check, and report the bounds failure (fallback_check)
// KE: number of leading dofs evaluated (MUSCL's limited r = 1 polynomial: 3, the
// rest are zero; oracle evaluate_cell_n)
// STORE = false: only the staged values (the troubled kernels store the final
// face values cooperatively in troubled_fallback)
// phc: the chunk's per-cell phi rows staged in shared memory ([Q*K][32], lane = cell)
template <int K, int NQ, int NF, int KE = K, bool STORE = true>
__device__ __forceinline__ void eval_store(const Dev3& D, const Work3& W, int c, int op, int v, int lane, bool act,
                                           double u0, const double* a, double (*sval)[V5][33], bool chk,
                                           double blo, double bhi, double& viol, const int* sl,
                                           const double* phs = nullptr, const double* phc = nullptr) {
  constexpr int Q = NF * NQ;
  constexpr int QG = (Q % 4 == 0) ? 4 : ((Q % 3 == 0) ? 3 : 1);  // independent fma chains in flight
  auto group = [&](int q0) {
    int gs[QG];  // this group's slots (issued before the fma chains)
#pragma unroll
    for (int j = 0; j < QG; ++j) gs[j] = !STORE ? 0 : (sl ? sl[q0 + j] : D.slot[ao(c, q0 + j, Q)]);
    double val[QG];
#pragma unroll
    for (int j = 0; j < QG; ++j) val[j] = u0;
    if (phs) {  // the block's operator row staged in shared memory (broadcast 16-byte reads)
      double2 w[QG];
#pragma unroll
      for (int k = 0; k < KE; ++k)
#pragma unroll
        for (int j = 0; j < QG; ++j) {
          const int e = (q0 + j) * K + k;
          if ((e & 1) == 0 || k == 0) w[j] = reinterpret_cast<const double2*>(phs)[e >> 1];
          val[j] = __fma_rn(a[k], (e & 1) ? w[j].y : w[j].x, val[j]);
        }
    } else if (phc) {
#pragma unroll
      for (int k = 0; k < KE; ++k)
#pragma unroll
        for (int j = 0; j < QG; ++j) val[j] = __fma_rn(a[k], phc[((q0 + j) * K + k) * 32 + lane], val[j]);
    } else {
#pragma unroll
      for (int k = 0; k < KE; ++k)
#pragma unroll
        for (int j = 0; j < QG; ++j) val[j] = __fma_rn(a[k], D.phi[ao(op, (q0 + j) * K + k, Q * K)], val[j]);
    }
#pragma unroll
    for (int j = 0; j < QG; ++j) {
      if (STORE && act) W.fp[static_cast<size_t>(gs[j]) * V5 + v] = val[j];
      sval[q0 + j][v][lane] = val[j];
      if (chk) viol = smax(viol, smax(blo - val[j], val[j] - bhi));
    }
  };
  // p = 3: fully unrolled (the slot array stays in registers); p <= 2: rolled
  // (measured faster there: fewer live registers, slots from L1-resident stack)
  if (K >= 19) {
#pragma unroll
    for (int q0 = 0; q0 < Q; q0 += QG) group(q0);
  } else {
#pragma unroll 1
    for (int q0 = 0; q0 < Q; q0 += QG) group(q0);
  }
}

// fallback (solver.cpp:229-264) after a troubled reconstruction; demoted cells
// get first-order values. COOP (lattice-class kernels): the reconstruction
// only staged its face values in shared memory, and the block now stores the
// chunk's final values, five consecutive threads per face point (one
// contiguous 40-byte record instead of scattered 8-byte stores per variable):
// config 5 weights 26.4 -> 22.8 ms/stage; per-cell-row kernels (config 4c)
// keep the per-thread stores (cooperative measured 4.76 vs 4.65 ms).
// scell: (COOP) the cell this thread stores for, thread t <-> (list entry t / 5,
// variable t % 5), or -1: its face-point slots are requested on entry, so their
// latency is covered by the bounds / positivity votes (L1 prefetch; loaded cold group by group
// between the stores they were 25 % of the lattice-class CWENOZ kernel's stall samples)
template <int NF, int NQ, bool COOP>
__device__ __forceinline__ void troubled_fallback(const Dev3& D, const Phys3& P, const Work3& W, int c, int v,
                                                  int lane, bool act, double u0, bool chk, double blo, double bhi,
                                                  double viol, double (*sval)[V5][33], int* s_fail, int scell = -1) {
  constexpr int Q = NF * NQ;
  __shared__ double s_u0[V5][32];
  if (COOP && scell >= 0) {  // the five threads of a cell touch its Q slot lines between them (no registers held)
#pragma unroll
    for (int q = threadIdx.x % V5; q < Q; q += V5) prefetch_l1(&D.slot[ao(scell, q, Q)]);
  }
  if (v == 0) s_fail[lane] = 0;
  if (COOP) s_u0[v][lane] = u0;
  __syncthreads();
  if (P.mode == UCFVB_HYBRID) {
    if (chk) {
      double dm, dw;
      compute_margins(P.mg, bhi - blo, dm, dw);
      if (viol > dm) s_fail[lane] = 1;
    }
    for (int p = threadIdx.x; p < Q * 32; p += 160) {
      const int q = p >> 5, l = p & 31;
      double s[5];
#pragma unroll
      for (int w = 0; w < V5; ++w) s[w] = sval[q][w][l];
      if (!is_physical3(s, P.gamma)) s_fail[l] = 1;
    }
  }
  __syncthreads();
  if constexpr (COOP) {
    if (act && v == 0 && s_fail[lane]) W.labels[c] = UCFVB_SCHEME_FIRST;
    const int l = threadIdx.x / V5, w = threadIdx.x - l * V5;  // thread (cell l, variable w)
    if (scell >= 0) {
      const bool fail = s_fail[l] != 0;
      constexpr int G = 4;  // slot loads (L1 hits after the prefetch) a group at a time: register pressure
#pragma unroll 1
      for (int q0 = 0; q0 < Q; q0 += G) {
        int sl[G];
#pragma unroll
        for (int j = 0; j < G; ++j) sl[j] = q0 + j < Q ? __ldg(&D.slot[ao(scell, q0 + j, Q)]) : 0;
#pragma unroll
        for (int j = 0; j < G; ++j)
          if (q0 + j < Q) W.fp[static_cast<size_t>(sl[j]) * V5 + w] = fail ? s_u0[w][l] : sval[q0 + j][w][l];
      }
    }
  } else {
    if (act && s_fail[lane]) {
      if (v == 0) W.labels[c] = UCFVB_SCHEME_FIRST;
      for (int q = 0; q < Q; ++q) W.fp[static_cast<size_t>(D.slot[ao(c, q, Q)]) * V5 + v] = u0;
    }
  }
  __syncthreads();
}

// The block stores a chunk's staged face values run by run: with side-major
// face points the NQ points a cell owns on one face are NQ * 40 contiguous
// bytes, so consecutive threads take consecutive doubles of a (cell, face) run
// and a warp's store covers whole sectors (per-thread stores of one variable
// hit one 8-byte piece of 32 different sectors).
template <int NF, int NQ>
__device__ __forceinline__ void coop_store_runs(const Dev3& D, const Work3& W, int cb, double (*sval)[V5][33]) {
  constexpr int Q = NF * NQ, RL = NQ * V5, RPI = 160 / RL;  // run length (doubles), runs per pass
  const int r_in = threadIdx.x / RL, j = threadIdx.x - r_in * RL;
  const int q = j / V5, w = j - q * V5;
  if (r_in >= RPI) return;
#pragma unroll 4
  for (int r0 = 0; r0 < 32 * NF; r0 += RPI) {
    const int r = r0 + r_in;
    const int l = r / NF, lf = r - l * NF;
    if (r < 32 * NF && cb + l < D.n) {
      const int sl = __ldg(&D.slot[ao(cb + l, lf * NQ + q, Q)]);
      W.fp[static_cast<size_t>(sl) * V5 + w] = sval[lf * NQ + q][w][l];
    }
  }
}

// per-cell-row central kernel: store the candidates cooperatively (coop_store_runs)
#ifndef UCFVB_C3_COOP
#define UCFVB_C3_COOP 1
#endif

// ---- central: solve + evaluate + NAD + fallback pre-check -----------------------------
// STAGED: lattice-class operators on a type-blocked mesh (every chunk one
// type): the grid is a multiple of the type count, so block b only ever sees
// chunks of type b % 6 and stages that type's pinv and phi rows in shared
// memory once, read as broadcast 16-byte loads
// nad bit 0: NAD classification (hybrid); bit 1: this stage detects (first
// stage or detect_every_stage), so the raw label decides the final one
// TMA staging of the phi block as well (pinv + phi: 1 block/SM, config 4
// central 3.85 ms/stage; pinv only: 3 blocks/SM, 3.51 ms; cp.async pinv at the
// chunk start: 3.61 ms). UCFVB_TMA3_PHI=1 builds the pinv + phi variant.
// UCFVB_C3_RING=1: the phi block streams through a ring of kRingSlots
// shared-memory slots, one slot = the rows of QG = 4 face points (4 K 32
// doubles), bulk-copied three pieces ahead: the five variable-warps read each
// phi line from shared memory instead of five times through L1 (the L1 tag
// stage was the busiest unit of this kernel), and the footprint stays at two
// blocks per SM (whole-block staging, UCFVB_TMA3_PHI, leaves one).
#ifndef UCFVB_C3_RING
#define UCFVB_C3_RING 1
#endif
constexpr int kRingSlots = 3;
#ifndef UCFVB_TMA3_PHI
#define UCFVB_TMA3_PHI 0
#endif
// TMA: per-cell operator rows (config 4): the chunk's pinv block (group A)
// and phi block (group B) are bulk-copied into shared memory one chunk ahead,
// each refilled as soon as the solve / the evaluation has consumed it
// (split-phase, as the 2D k_central_tma)
// lattice-class central kernel: L1 prefetch of the next chunk's stencil-id lines
#ifndef UCFVB_C5_PFID
#define UCFVB_C5_PFID 1
#endif
// resident blocks per SM asked of the p = 3 central kernels (register bound; shared memory allows three)
#ifndef UCFVB_C5_MINB
#define UCFVB_C5_MINB 4
#endif
// resident blocks per SM asked of the per-cell-row (p <= 2) central kernels
#ifndef UCFVB_C3_MINB
#define UCFVB_C3_MINB 2
#endif
// TMA variant: bulk L2 prefetch of the next chunk's phi block (read through L1 by the evaluation)
#ifndef UCFVB_C3_PFPHI
#define UCFVB_C3_PFPHI 1
#endif
template <int K, int M, int NF, int NQ, bool STAGED, bool TMA = false>
__global__ void __launch_bounds__(160, (K * M <= 200) ? UCFVB_C3_MINB : UCFVB_C5_MINB) k3_central(Dev3 D, Phys3 P, Work3 W, const double* __restrict__ U, int eval,
                                                   int nad) {
  constexpr int Q = NF * NQ;
  // staged path on a detecting stage: the candidate face values are stored
  // after the NAD vote, only for cells that stay Linear (a raw label >=
  // CWENOZ survives the spread and a failed pre-check demotes the cell: the
  // troubled kernels / the spread rewrite those cells' face points)
  const bool detect = STAGED && K >= 8 && eval && (nad & 2);
  nad &= 1;
  constexpr int G = M + NF;  // stencil members + face neighbours
  extern __shared__ __align__(16) double smem3[];
  double* xs = smem3;
  auto sval = reinterpret_cast<double (*)[V5][33]>(smem3);
  // STAGED: pinv row [M][K], phi row [Q][K] and the centre values [5][32] past the union buffer
  constexpr bool DM = STAGED && K >= 8;  // tensor-core path (strides: see kXS)
  constexpr int KP = DM ? kpad(K) : K;
  constexpr size_t kUnion = DM ? dm_union(G, Q, K) : smem3_bytes(G, Q) / 8;
  double* sp = smem3 + kUnion;
  // per-cell operator rows (p <= 2): the chunk's pinv block is copied to shared
  // memory with 16-byte cp.async at the chunk start (all in flight at once)
  constexpr bool PCS = !STAGED && !TMA && K * M <= 200;
  double* spc = smem3 + kUnion;
  double* sphc = spc + M * K * 32;  // TMA: the chunk's phi block
  constexpr bool kRing = TMA && UCFVB_C3_RING && !UCFVB_TMA3_PHI && (Q % 4 == 0);
  constexpr int kPiece = 4 * K * 32, kPieces = Q / 4;  // doubles per ring slot; pieces per chunk
  // TMA: [0] pinv, [1] phi (whole block) or [1 .. kRingSlots] the ring's full barriers
  uint64_t* bar = reinterpret_cast<uint64_t*>(sphc + (UCFVB_TMA3_PHI ? Q * K * 32 : (kRing ? kRingSlots * kPiece : 0)));
  __shared__ int s_sev[2][32], s_bf[2][32], s_pos[32];
  const int lane = threadIdx.x & 31, v = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x < 2 * W.ntl) W.counters[kCnt0 + threadIdx.x] = 0;  // list lengths of this stage
  const int nch = (D.n + 31) >> 5;
  constexpr bool kTmaPhi = TMA && UCFVB_TMA3_PHI;  // phi staged too (else read through L1)
  constexpr uint32_t kPinvBytes = M * K * 32 * 8, kPhiBytes = Q * K * 32 * 8;
  auto issue_pinv = [&](int ch) {
    mbar_arrive_expect_tx(&bar[0], kPinvBytes);
    bulk_g2s(spc, D.pinv + static_cast<size_t>(ch) * M * K * 32, kPinvBytes, &bar[0]);
  };
  auto issue_phi = [&](int ch) {
    mbar_arrive_expect_tx(&bar[1], kPhiBytes);
    bulk_g2s(sphc, D.phi + static_cast<size_t>(ch) * Q * K * 32, kPhiBytes, &bar[1]);
  };
  // ring piece gp of this block's chunk sequence: chunk blockIdx.x + (gp / kPieces) * gridDim.x, piece gp % kPieces
  auto issue_piece = [&](int gp) {
    const int chp = blockIdx.x + (gp / kPieces) * static_cast<int>(gridDim.x);
    if (chp >= nch) return;
    const int slot = gp % kRingSlots;
    mbar_arrive_expect_tx(&bar[1 + slot], kPiece * 8);
    bulk_g2s(sphc + slot * kPiece, D.phi + static_cast<size_t>(chp) * Q * K * 32 + static_cast<size_t>(gp % kPieces) * kPiece,
             kPiece * 8, &bar[1 + slot]);
  };
  if (TMA) {
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      if (kRing)
        for (int i = 1; i < kRingSlots; ++i) mbar_init(&bar[1 + i], 1);
      mbar_fence_init();
      if (static_cast<int>(blockIdx.x) < nch) {
        issue_pinv(blockIdx.x);
        if (kTmaPhi) issue_phi(blockIdx.x);
        if (kRing)
          for (int i = 0; i < kRingSlots; ++i) issue_piece(i);
      }
    }
    __syncthreads();
  }
  int it = 0;
  if (STAGED) {
    const int t = blockIdx.x % D.n_ops;
    for (int e = threadIdx.x; e < M * K; e += 160) sp[(e / K) * KP + e % K] = D.pinv[ao(t, e, M * K)];
    for (int e = threadIdx.x; e < Q * K; e += 160) sp[M * KP + (e / K) * KP + e % K] = D.phi[ao(t, e, Q * K)];
    __syncthreads();
  }
  for (int ch = blockIdx.x; ch < nch; ch += gridDim.x, ++it) {
    const int c = (ch << 5) + lane;
    const bool act = c < D.n;
    const int cc = act ? c : (D.n - 1);
    if (v == 0) s_pos[lane] = 0;  // read last before the previous iteration's final barrier
    const int op = D.opi[cc];
    const int nxt = ch + static_cast<int>(gridDim.x);
    if (!TMA && D.n_ops == D.n && threadIdx.x == 0 && ch + static_cast<int>(gridDim.x) < nch) {
      // this block's next chunk's pinv rows and stencil ids -> L2 (TMA prefetch;
      // measured: prefetching phi as well thrashes L2 and is slower)
      const int nx = ch + gridDim.x;
      bulk_prefetch_l2(D.pinv + static_cast<size_t>(nx) * M * K * 32, M * K * 32 * 8);
      bulk_prefetch_l2(D.central + static_cast<size_t>(nx) * (M + 1) * 32, (M + 1) * 32 * 4);
    }
    if (TMA && UCFVB_C3_PFPHI && !kTmaPhi && !kRing && threadIdx.x == 32 && nxt < nch)
      bulk_prefetch_l2(D.phi + static_cast<size_t>(nxt) * Q * K * 32, Q * K * 32 * 8);
    const bool pcs = PCS && D.n_ops == D.n;
    if (pcs) {
      const double* src = D.pinv + static_cast<size_t>(ch) * M * K * 32;
      for (int e = threadIdx.x; e < M * K * 32 / 2; e += 160) cp_async16(spc + 2 * e, src + 2 * e);
    }
    // every stencil and neighbour value of this (cell, variable) in flight at
    // once: G fire-and-forget 8-byte cp.async copies into shared memory
    if constexpr (DM) {
      if (UCFVB_C5_PFID && nxt < nch && threadIdx.x < M + 1 + NF) {
        // the next chunk's stencil-id and neighbour lines (one 128-byte line per member) into L1:
        // their round trip leaves the head of that chunk's ids -> gather dependency chain
        const int e = threadIdx.x;
        prefetch_l1(e <= M ? &D.central[ao(nxt << 5, e, M + 1)] : &D.nbr[ao(nxt << 5, e - M - 1, NF)]);
      }
      // transposed: thread (cell gl, variable gv) -- one member's five variables are one 40-byte read
      const int gl = threadIdx.x / V5, gv = threadIdx.x - gl * V5;
      const int gc = min((ch << 5) + gl, D.n - 1);
      int id[G];
#pragma unroll
      for (int m = 0; m < M; ++m) id[m] = D.central[ao(gc, m + 1, M + 1)];
#pragma unroll
      for (int i = 0; i < NF; ++i) id[M + i] = D.nbr[ao(gc, i, NF)];
#pragma unroll
      for (int g = 0; g < G; ++g) cp_async8(&xs[g * kXS + gv * kVS + gl], &U[static_cast<size_t>(id[g]) * V5 + gv]);
      cp_async_commit();
    } else {
      int id[G];
#pragma unroll
      for (int m = 0; m < M; ++m) id[m] = D.central[ao(cc, m + 1, M + 1)];
#pragma unroll
      for (int i = 0; i < NF; ++i) id[M + i] = D.nbr[ao(cc, i, NF)];
#pragma unroll
      for (int g = 0; g < G; ++g) cp_async8(&xs[g * 160 + threadIdx.x], &U[static_cast<size_t>(id[g]) * V5 + v]);
      cp_async_commit();
    }
    // face-point slots: loaded up front while the gather is in flight for small
    // stencils, per face-point group for p = 3 (register pressure; measured)
    constexpr bool kHoist = K * M <= 200;
    int slh[kHoist ? NF * NQ : 1];
    if (kHoist) {
#pragma unroll
      for (int q = 0; q < (kHoist ? NF * NQ : 0); ++q) slh[q] = D.slot[ao(c, q, NF * NQ)];
    }
    const int* sl = kHoist ? slh : nullptr;
    const double u0 = U[static_cast<size_t>(cc) * V5 + v];
    cp_async_wait_all();  // this thread's own copies
    if (pcs) __syncthreads();  // the pinv block is copied by all threads
    if (TMA) mbar_wait(&bar[0], it & 1);
    double lo = u0, hi = u0;
    if constexpr (!DM) {
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        const double x = xs[(M + i) * 160 + threadIdx.x];
        lo = smin(lo, x);
        hi = smax(hi, x);
      }
    }
    double a[K];
#pragma unroll
    for (int k = 0; k < K; ++k) a[k] = 0.0;
    if constexpr (STAGED && K >= 8) {
      // the block's 32 cells share one operator row: the K x M solve of warp v
      // (variable v) is the GEMM a(K x 32) = pinv(K x M) . dU(M x 32) on the
      // fp64 tensor cores, m in k-steps of 4 (the oracle's fma order)
      constexpr int MT = (K + 7) / 8, KS = (M + 3) / 4;
      double* su0 = sp + M * KP + Q * KP;  // [5][32] centre values
      su0[threadIdx.x] = u0;
      __syncthreads();  // every thread's gather landed (each value was copied by another thread)
#pragma unroll
      for (int i = 0; i < NF; ++i) {
        const double x = xs[(M + i) * kXS + v * kVS + lane];
        lo = smin(lo, x);
        hi = smax(hi, x);
      }
      double dacc[MT][4][2];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int t = 0; t < 4; ++t) dacc[i][t][0] = dacc[i][t][1] = 0.0;
      const int fr = lane >> 2, fc = lane & 3;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int m = 4 * ks + fc;
        double af[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int k = 8 * i + fr;
          af[i] = (k < K && m < M) ? sp[m * KP + k] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int cl = 8 * t + fr;
          const double bf = m < M ? xs[m * kXS + v * kVS + cl] - su0[v * 32 + cl] : 0.0;
#pragma unroll
          for (int i = 0; i < MT; ++i) dmma884(dacc[i][t][0], dacc[i][t][1], af[i], bf);
        }
      }
      __syncthreads();  // gather buffer consumed: it carries the dofs back to their lanes
      double* sd = xs + Q * V5 * 33;  // [5][K][kRS], past the face-value buffer
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int k = 8 * i + fr;
          if (k < K) {
            sd[(v * K + k) * kRS + 8 * t + 2 * fc] = dacc[i][t][0];
            sd[(v * K + k) * kRS + 8 * t + 2 * fc + 1] = dacc[i][t][1];
          }
        }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < K; ++k) a[k] = sd[(v * K + k) * kRS + lane];
    } else {
      double2 w = make_double2(0.0, 0.0);
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const double x = xs[m * 160 + threadIdx.x] - u0;
        if (STAGED) {
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const int e = m * K + k;
            if ((e & 1) == 0) w = reinterpret_cast<const double2*>(sp)[e >> 1];
            a[k] = __fma_rn((e & 1) ? w.y : w.x, x, a[k]);
          }
        } else if (PCS || TMA) {
#pragma unroll
          for (int k = 0; k < K; ++k)
            a[k] = __fma_rn((TMA || pcs) ? spc[(m * K + k) * 32 + lane] : D.pinv[ao(op, m * K + k, M * K)], x, a[k]);
        } else {
#pragma unroll
          for (int k = 0; k < K; ++k) a[k] = __fma_rn(D.pinv[ao(op, m * K + k, M * K)], x, a[k]);
        }
      }
    }
    // the gather buffer becomes the face-value buffer (DM: every gather read precedes the
    // barrier after the solve, and until the barrier behind the evaluation each warp only
    // touches its own dofs rows)
    if (!DM) __syncthreads();
    if (TMA && threadIdx.x == 0 && nxt < nch) {  // pinv consumed: the next chunk's
      fence_proxy_async_smem();
      issue_pinv(nxt);
    }
    const bool chk = (v == 0 || v == 4);
    double viol = -1e300;
    if constexpr (STAGED && K >= 8) {
      if (eval) {
        // face values of warp v's 32 cells: F(Q x 32) = u0 + phi(Q x K) . a(K x 32) on
        // the tensor cores, k in steps of 4 from C = u0 (evaluate_cell's fma order)
        constexpr int QT = (Q + 7) / 8, KS2 = (K + 3) / 4;
        const double* sd = xs + Q * V5 * 33;
        const double* sph = sp + M * KP;
        const double* su0 = sp + M * KP + Q * KP;
        const int fr = lane >> 2, fc = lane & 3;
        double f[QT][4][2];
#pragma unroll
        for (int i = 0; i < QT; ++i)
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            f[i][t][0] = su0[v * 32 + 8 * t + 2 * fc];
            f[i][t][1] = su0[v * 32 + 8 * t + 2 * fc + 1];
          }
#pragma unroll
        for (int ks = 0; ks < KS2; ++ks) {
          const int k = 4 * ks + fc;
          double af[QT];
#pragma unroll
          for (int i = 0; i < QT; ++i) {
            const int q = 8 * i + fr;
            af[i] = (q < Q && k < K) ? sph[q * KP + k] : 0.0;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const double bf = k < K ? sd[(v * K + k) * kRS + 8 * t + fr] : 0.0;
#pragma unroll
            for (int i = 0; i < QT; ++i) dmma884(f[i][t][0], f[i][t][1], af[i], bf);
          }
        }
        const int cb = ch << 5;
#pragma unroll
        for (int i = 0; i < QT; ++i)
#pragma unroll
          for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int q = 8 * i + fr, cl = 8 * t + 2 * fc + j;
              if (q < Q) {
                sval[q][v][cl] = f[i][t][j];
                if (!detect && cb + cl < D.n) W.fp[static_cast<size_t>(D.slot[ao(cb + cl, q, Q)]) * V5 + v] = f[i][t][j];
              }
            }
        __syncthreads();  // every face value of the block in sval
        if (chk)
          for (int q = 0; q < Q; ++q) {
            const double val = sval[q][v][lane];
            viol = smax(viol, smax(lo - val, val - hi));
          }
      }
    } else {
      if (kTmaPhi) mbar_wait(&bar[1], it & 1);
      if constexpr (kRing) {
        // phi by pieces of four face points through the ring (every chunk consumes its
        // kPieces pieces whether or not it evaluates, so the ring's order is fixed)
#pragma unroll
        for (int g = 0; g < kPieces; ++g) {
          const int gp = it * kPieces + g, slot = gp % kRingSlots;
          mbar_wait(&bar[1 + slot], (gp / kRingSlots) & 1);
          if (eval) {
            const double* ph = sphc + slot * kPiece;
            int gs[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) gs[j] = UCFVB_C3_COOP ? 0 : (sl ? sl[4 * g + j] : D.slot[ao(c, 4 * g + j, Q)]);
            double val[4] = {u0, u0, u0, u0};
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
              for (int j = 0; j < 4; ++j) val[j] = __fma_rn(a[k], ph[(j * K + k) * 32 + lane], val[j]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (!UCFVB_C3_COOP && act) W.fp[static_cast<size_t>(gs[j]) * V5 + v] = val[j];
              sval[4 * g + j][v][lane] = val[j];
              if (chk) viol = smax(viol, smax(lo - val[j], val[j] - hi));
            }
          }
          __syncthreads();  // every warp is done with this slot: refill it three pieces ahead
          if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            issue_piece(gp + kRingSlots);
          }
        }
      } else if (eval) {
        if constexpr (TMA && UCFVB_C3_COOP)
          eval_store<K, NQ, NF, K, false>(D, W, c, op, v, lane, act, u0, a, sval, chk, lo, hi, viol, sl,
                                          nullptr, kTmaPhi ? sphc : nullptr);
        else
          eval_store<K, NQ, NF>(D, W, c, op, v, lane, act, u0, a, sval, chk, lo, hi, viol, sl,
                                STAGED ? sp + M * KP : nullptr, kTmaPhi ? sphc : nullptr);
      }
    }
    // per checked variable: deactivation, severity vote and bounds failure
    if (chk && eval) {
      const int t = v == 0 ? 0 : 1;
      const double du = hi - lo;
      double dm, dw;
      compute_margins(P.mg, du, dm, dw);
      int sev = 0;
      if (nad) {
        const double thr = D.thr[cc];
        const bool deact = P.mg.kappa > 0.0 && du < thr;
        if (!deact) sev = violation_severity(viol, dm, dw);
        const double sc = 1e-12 * smax(fabs(u0), smax(du, fabs(dm)));
        const bool tie = (P.mg.kappa > 0.0 && fabs(du - thr) <= 1e-12 * thr) ||
                         (!deact && (fabs(viol - dm) <= sc || fabs(viol - dw) <= 1e-12 * smax(fabs(u0), smax(du, fabs(dw)))));
        if (tie && act) atomicAdd(W.ties, 1ull);
        if (act) {
          W.bounds[ao(c, 2 * t, 4)] = lo;
          W.bounds[ao(c, 2 * t + 1, 4)] = hi;
        }
      }
      s_sev[t][lane] = sev;
      s_bf[t][lane] = viol > dm;
    }
    // the face values are visible (DM: the barrier behind the evaluation; s_pos was cleared
    // at the top of the iteration)
    if (!DM) __syncthreads();
    if (eval && nad) {
      // positivity of every face value of the 32 cells, spread over the block
      for (int p = threadIdx.x; p < Q * 32; p += 160) {
        const int q = p >> 5, l = p & 31;
        double s[5];
#pragma unroll
        for (int w = 0; w < V5; ++w) s[w] = sval[q][w][l];
        if (!is_physical3(s, P.gamma)) s_pos[l] = 1;
      }
    }
    __syncthreads();
    if (v == 0 && act && nad) {
      const int sev = max(s_sev[0][lane], s_sev[1][lane]);
      const int fail = s_pos[lane] | s_bf[0][lane] | s_bf[1][lane];
      W.raw[c] = static_cast<uint8_t>(sev | (fail << 2));
    }
    if (detect) {  // the surviving candidates, five contiguous variables per face point
      if (v == 0) s_pos[lane] = !(max(s_sev[0][lane], s_sev[1][lane]) | s_pos[lane] | s_bf[0][lane] | s_bf[1][lane]);
      __syncthreads();
      const int cb = ch << 5;
      const int l = threadIdx.x / V5, w = threadIdx.x - l * V5;  // thread (cell l, variable w)
      if (s_pos[l] && cb + l < D.n) {  // every slot load in flight before the stores (end of the iteration: registers are free)
        int sl[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) sl[q] = __ldg(&D.slot[ao(cb + l, q, Q)]);
#pragma unroll
        for (int q = 0; q < Q; ++q) W.fp[static_cast<size_t>(sl[q]) * V5 + w] = sval[q][w][l];
      }
    }
    if constexpr (TMA && UCFVB_C3_COOP) {
      if (eval) coop_store_runs<NF, NQ>(D, W, ch << 5, sval);
    }
    __syncthreads();
    if (kTmaPhi && threadIdx.x == 0 && nxt < nch) {  // phi consumed: the next chunk's
      fence_proxy_async_smem();
      issue_phi(nxt);
    }
  }
}

__device__ __forceinline__ int sev_of(int s) { return s == 0 ? 0 : (s == 1 ? 1 : 2); }

// ---- spread + lists (hybrid detection stage) ------------------------------------------
template <int NF, int NQ>
// detect = 0: frozen classification (detect_every_stage = false, later stages
// of a step): the labels stay as the previous stage left them (solver.cpp:343-361)
__global__ void __launch_bounds__(256) k3_spread(Dev3 D, Work3 W, const double* __restrict__ U, int detect) {
  constexpr int Q = NF * NQ;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int lab = 0;
  bool ok = c < D.n;
  if (ok) {
    const int r = W.raw[c];
    if (detect) {
      int sev = r & 3;
#pragma unroll
      for (int i = 0; i < NF; ++i) sev = max(sev, static_cast<int>(W.raw[D.nbr[ao(c, i, NF)]] & 3));
      lab = sev == 0 ? UCFVB_SCHEME_LINEAR : (sev == 1 ? UCFVB_SCHEME_CWENOZ : UCFVB_SCHEME_MUSCL);
    } else {
      lab = W.labels[c];
    }
    if ((lab == UCFVB_SCHEME_LINEAR && (r >> 2)) || lab == UCFVB_SCHEME_FIRST) {
      // fallback_check demotes the Linear candidate (solver.cpp:256-262), or a
      // frozen FirstOrder label (apply_troubled's constant branch): first-order values
      lab = UCFVB_SCHEME_FIRST;
    }
    W.labels[c] = static_cast<uint8_t>(lab);
  }
  {
    // first-order face values, written by the whole warp per demoted cell: lane e of pass j
    // stores value (point e / 5, variable e % 5), so a face's points go out as contiguous runs
    // (one thread per cell wrote 120 scattered 8-byte stores with 4 of 5 lanes idle)
    unsigned fo = __ballot_sync(0xffffffffu, ok && lab == UCFVB_SCHEME_FIRST);
    const int c0 = c - lane;
    while (fo) {
      const int l = __ffs(fo) - 1;
      fo &= fo - 1;
      const int cc = c0 + l;
#pragma unroll
      for (int e = lane; e < Q * V5; e += 32) {
        const int q = e / V5, v = e - q * V5;
        W.fp[static_cast<size_t>(D.slot[ao(cc, q, Q)]) * V5 + v] = U[static_cast<size_t>(cc) * V5 + v];
      }
    }
  }
  // warp-aggregated appends to the CWENOZ / MUSCL lists
  for (int L = 0; L < 2; ++L) {
    const bool mine = ok && lab == (L == 0 ? UCFVB_SCHEME_CWENOZ : UCFVB_SCHEME_MUSCL);
    const unsigned b = __ballot_sync(0xffffffffu, mine);
    if (!b) continue;
    int base = 0;
    // type-blocked meshes: the warp's 32 cells share one lattice type
    const int t = W.ntl > 1 ? ((c >> 5) % W.ntl) : 0;
    if (lane == 0) base = atomicAdd(&W.counters[cnt_idx(W, L, t)], __popc(b));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (mine) list_of(W, L, t)[base + __popc(b & ((1u << lane) - 1u))] = c;
  }
}

// forced modes: every cell in one list (SchemeMode::Cwenoz / Muscl, solver.cpp:322-328)
__global__ void k3_fill_list(int n, int which, uint8_t lab, Work3 W) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c == 0)
    for (int t = 0; t < W.ntl; ++t) W.counters[cnt_idx(W, which, t)] = n / W.ntl;
  if (c < n) {
    const int t = W.ntl > 1 ? ((c >> 5) % W.ntl) : 0;
    const int i = W.ntl > 1 ? ((c >> 5) / W.ntl) * 32 + (c & 31) : c;
    list_of(W, which, t)[i] = c;
    W.labels[c] = lab;
  }
}

// lattice-class CWENOZ / MUSCL kernels: L1 prefetch of the next tile's stencil-id lines
#ifndef UCFVB_W5_PFID
#define UCFVB_W5_PFID 0
#endif
// ---- CWENOZ (solver.cpp:167-188; reconstruct.cpp:43-57, 99-150) -------------------------
#ifndef UCFVB_W5_MINB
#define UCFVB_W5_MINB 3
#endif
// lattice-class p = 3 (config 5): three resident blocks per SM (<= 136
// registers; 168 unbounded) measured faster despite a few spills (22.3 vs
// 25.2 ms/stage of weights); per-cell rows keep the unbounded allocation
template <int K, int M, int NF, int NQ, bool STAGED>
__global__ void __launch_bounds__(160, (STAGED && K >= 19) ? UCFVB_W5_MINB : 0) k3_cwenoz(Dev3 D, Phys3 P, Work3 W, const double* __restrict__ U) {
  constexpr int Q = NF * NQ;
  constexpr int G = M;  // the central stencil (the directional members are a subset of it)
  // DM: lattice-class chunks (one operator row per block) run the central
  // solve and the face evaluation on the fp64 tensor cores (see k3_central; strides: kXS)
  constexpr bool DM = STAGED && K >= 8;
  constexpr int KP = DM ? kpad(K) : K;  // row stride of the staged pinv / OI / phi rows
  constexpr int EPG = M * K;            // pinv elements per operator row in global memory
  constexpr int EP = M * KP, ED = NF * 3 * MD3, EO = (K * KP + 1) & ~1;  // region sizes (even: phi is read as double2)
  constexpr size_t kUnion = DM ? dm_union(G, Q, K) : smem3_bytes(G, Q) / 8;
  extern __shared__ __align__(16) double smem3[];
  double* xs = smem3;
  auto sval = reinterpret_cast<double (*)[V5][33]>(smem3);
  double* sd = xs + Q * V5 * 33;  // DM: dofs [5][K][32] past the face values
  // STAGED: this block's lattice type's rows: pinv | pinv_dir | OI | phi | (DM: centre values [5][32]) | dir members
  double* sp = smem3 + kUnion;
  double* su0 = sp + EP + ED + EO + Q * KP;
  int* sdm = reinterpret_cast<int*>(su0 + (DM ? 160 : 0));
  int* scell = sdm + NF * MD3;  // DM: the chunk's cells
  // forced CWENOZ on per-cell rows (p <= 2): the list is the identity, so each
  // item is one AoSoA chunk whose pinv block is copied to shared memory first
  constexpr bool PCS = !STAGED && K * M <= 200;
  double* spc = smem3 + kUnion;
  __shared__ int s_fail[32];
  const int lane = threadIdx.x & 31, v = threadIdx.x >> 5;
  const int t = STAGED ? blockIdx.x % W.ntl : 0;
  const int b0 = STAGED ? blockIdx.x / W.ntl : blockIdx.x, nb = STAGED ? gridDim.x / W.ntl : gridDim.x;
  const int cnt = W.counters[cnt_idx(W, kCwList, t)];
  const int32_t* list = list_of(W, kCwList, t);
  if (STAGED) {
    for (int e = threadIdx.x; e < EPG; e += 160) sp[(e / K) * KP + e % K] = D.pinv[ao(t, e, EPG)];
    for (int e = threadIdx.x; e < ED; e += 160) sp[EP + e] = D.pinv_dir[ao(t, e, ED)];
    for (int e = threadIdx.x; e < K * K; e += 160) sp[EP + ED + (e / K) * KP + e % K] = D.oi[ao(t, e, K * K)];
    for (int e = threadIdx.x; e < Q * K; e += 160) sp[EP + ED + EO + (e / K) * KP + e % K] = D.phi[ao(t, e, Q * K)];
    for (int e = threadIdx.x; e < NF * MD3; e += 160) sdm[e] = D.dirm[ao(t, e, NF * MD3)];
    __syncthreads();
  }
  for (int base = b0 * 32; base < cnt; base += nb * 32) {
    const bool act = base + lane < cnt;
    const int c = list[act ? base + lane : base];
    const int op = D.opi[c];
    const double u0 = U[static_cast<size_t>(c) * V5 + v];
    const bool pcs = PCS && P.mode == UCFVB_CWENOZ && D.n_ops == D.n && (base & 31) == 0;
    if (pcs) {
      const double* src = D.pinv + static_cast<size_t>(base >> 5) * M * K * 32;
      for (int e = threadIdx.x; e < M * K * 32 / 2; e += 160) cp_async16(spc + 2 * e, src + 2 * e);
    }
    // the M central-stencil values in flight at once (cp.async); the central
    // solve is recomputed here (bit-identical to k3_central's) instead of
    // storing K x 5 dofs for every cell
    if constexpr (DM) {
      // transposed: thread (cell gl, variable gv) -- one member's five variables are one 40-byte read
      const int gl = threadIdx.x / V5, gv = threadIdx.x - gl * V5;
      const int gc = list[base + gl < cnt ? base + gl : base];
      int id[M];
#pragma unroll
      for (int m = 0; m < M; ++m) id[m] = D.central[ao(gc, m + 1, M + 1)];
#pragma unroll
      for (int m = 0; m < M; ++m) cp_async8(&xs[m * kXS + gv * kVS + gl], &U[static_cast<size_t>(id[m]) * V5 + gv]);
      cp_async_commit();
    } else {
      int id[M];
#pragma unroll
      for (int m = 0; m < M; ++m) id[m] = D.central[ao(c, m + 1, M + 1)];
#pragma unroll
      for (int m = 0; m < M; ++m) cp_async8(&xs[m * 160 + threadIdx.x], &U[static_cast<size_t>(id[m]) * V5 + v]);
      cp_async_commit();
    }
    // face-point slots, loaded while the gather is in flight (p <= 2; for p = 3
    // per face-point group: register pressure)
    constexpr bool kHoist = K * M <= 200;
    int slh[kHoist ? NF * NQ : 1];
    if (kHoist) {
#pragma unroll
      for (int q = 0; q < (kHoist ? NF * NQ : 0); ++q) slh[q] = D.slot[ao(c, q, NF * NQ)];
    }
    const int* sl = kHoist ? slh : nullptr;
    cp_async_wait_all();
    double p1[K];
#pragma unroll
    for (int k = 0; k < K; ++k) p1[k] = 0.0;
    if constexpr (!DM) {
      if (pcs) __syncthreads();  // the pinv block is copied by all threads
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const double x = xs[m * 160 + threadIdx.x] - u0;
#pragma unroll
        for (int k = 0; k < K; ++k)
          p1[k] = __fma_rn(STAGED ? sp[m * KP + k]
                                  : (pcs ? spc[(m * K + k) * 32 + lane] : D.pinv[ao(op, m * K + k, M * K)]),
                           x, p1[k]);
      }
    } else {
      su0[threadIdx.x] = u0;
      if (v == 0) scell[lane] = act ? c : -1;
      __syncthreads();  // every gather landed and the centre values are shared
    }
    double dir[NF][3];
#pragma unroll
    for (int s = 0; s < NF; ++s) {
      double x[MD3];
#pragma unroll
      for (int m = 0; m < MD3; ++m)
        x[m] = (DM ? xs[(sdm[s * MD3 + m] - 1) * kXS + v * kVS + lane]
                   : xs[((STAGED ? sdm[s * MD3 + m] : D.dirm[ao(op, s * MD3 + m, NF * MD3)]) - 1) * 160 + threadIdx.x]) - u0;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < MD3; ++m)
          acc = __fma_rn(STAGED ? sp[EP + (s * 3 + k) * MD3 + m] : D.pinv_dir[ao(op, (s * 3 + k) * MD3 + m, ED)],
                         x[m], acc);
        dir[s][k] = acc;
      }
    }
    const int fr = lane >> 2, fc = lane & 3;
    if constexpr (DM) {
      // central solve p1(K x 32) = pinv(K x M) . dU(M x 32) for warp v's variable
      constexpr int MT = (K + 7) / 8, KS = (M + 3) / 4;
      double dacc[MT][4][2];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) dacc[i][tt][0] = dacc[i][tt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int m = 4 * ks + fc;
        double af[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int k = 8 * i + fr;
          af[i] = (k < K && m < M) ? sp[m * KP + k] : 0.0;
        }
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
          const int cl = 8 * tt + fr;
          const double bf = m < M ? xs[m * kXS + v * kVS + cl] - su0[v * 32 + cl] : 0.0;
#pragma unroll
          for (int i = 0; i < MT; ++i) dmma884(dacc[i][tt][0], dacc[i][tt][1], af[i], bf);
        }
      }
      __syncthreads();  // the gather buffer is dead: the dofs travel through sd
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
          const int k = 8 * i + fr;
          if (k < K) {
            sd[(v * K + k) * kRS + 8 * tt + 2 * fc] = dacc[i][tt][0];
            sd[(v * K + k) * kRS + 8 * tt + 2 * fc + 1] = dacc[i][tt][1];
          }
        }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < K; ++k) p1[k] = sd[(v * K + k) * kRS + lane];
      __syncwarp();
    }
#pragma unroll
    for (int s = 0; s < NF; ++s) {
      p1[0] -= P.lams * dir[s][0];
      p1[1] -= P.lams * dir[s][1];
      p1[2] -= P.lams * dir[s][2];
    }
    // x / lam0 and x / wsum as div_rn (correctly rounded from the rounded reciprocal,
    // exact_math.h: the same bits as the IEEE division, a fifth of its instructions)
    const bool rl = P.lam0 >= 0x1p-60;
#pragma unroll
    for (int k = 0; k < K; ++k) p1[k] = rl ? div_rn(p1[k], P.lam0, P.inv_lam0) : p1[k] / P.lam0;
    // SI_0 = p1' OI p1 (row then dot) and the directional SI from the 3x3 block
    // SI_0 = p1' OI p1: t_k = sum_q OI_kq p1_q, si0 = sum_k p1_k t_k, fused, in the oracle's order
    double si0 = 0.0;
    if constexpr (DM) {
      // t(K x 32) = OI(K x K) . p1(K x 32) on the tensor cores (warp v's variable)
      constexpr int MT = (K + 7) / 8, KS3 = (K + 3) / 4;
#pragma unroll
      for (int k = 0; k < K; ++k) sd[(v * K + k) * kRS + lane] = p1[k];
      __syncwarp();
      double tacc[MT][4][2];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) tacc[i][tt][0] = tacc[i][tt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS3; ++ks) {
        const int q = 4 * ks + fc;
        double af[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) {
          const int k = 8 * i + fr;
          af[i] = (k < K && q < K) ? sp[EP + ED + k * KP + q] : 0.0;
        }
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
          const double bf = q < K ? sd[(v * K + q) * kRS + 8 * tt + fr] : 0.0;
#pragma unroll
          for (int i = 0; i < MT; ++i) dmma884(tacc[i][tt][0], tacc[i][tt][1], af[i], bf);
        }
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
          const int k = 8 * i + fr;
          if (k < K) {
            sd[(v * K + k) * kRS + 8 * tt + 2 * fc] = tacc[i][tt][0];
            sd[(v * K + k) * kRS + 8 * tt + 2 * fc + 1] = tacc[i][tt][1];
          }
        }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < K; ++k) si0 = __fma_rn(p1[k], sd[(v * K + k) * kRS + lane], si0);
      __syncwarp();
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < K; ++q) t = __fma_rn(STAGED ? sp[EP + ED + k * KP + q] : D.oi[ao(op, k * K + q, K * K)], p1[q], t);
        si0 = __fma_rn(p1[k], t, si0);
      }
    }
    const double o00 = (STAGED ? sp[EP + ED + (0)] : D.oi[ao(op, 0, K * K)]), o01 = (STAGED ? sp[EP + ED + (1)] : D.oi[ao(op, 1, K * K)]), o02 = (STAGED ? sp[EP + ED + (2)] : D.oi[ao(op, 2, K * K)]);
    const double o10 = (STAGED ? sp[EP + ED + (KP)] : D.oi[ao(op, K, K * K)]), o11 = (STAGED ? sp[EP + ED + (KP + 1)] : D.oi[ao(op, K + 1, K * K)]), o12 = (STAGED ? sp[EP + ED + (KP + 2)] : D.oi[ao(op, K + 2, K * K)]);
    const double o20 = (STAGED ? sp[EP + ED + (2 * KP)] : D.oi[ao(op, 2 * K, K * K)]), o21 = (STAGED ? sp[EP + ED + (2 * KP + 1)] : D.oi[ao(op, 2 * K + 1, K * K)]),
                 o22 = (STAGED ? sp[EP + ED + (2 * KP + 2)] : D.oi[ao(op, 2 * K + 2, K * K)]);
    double si[NF];
    double tau = 0.0;
#pragma unroll
    for (int s = 0; s < NF; ++s) {
      const double a0 = dir[s][0], a1 = dir[s][1], a2 = dir[s][2];
      double t = o00 * a0 * a0;
      t = t + (o01 + o10) * a0 * a1;
      t = t + (o02 + o20) * a0 * a2;
      t = t + o11 * a1 * a1;
      t = t + (o12 + o21) * a1 * a2;
      t = t + o22 * a2 * a2;
      si[s] = t;
      tau += fabs(t - si0);
    }
    tau /= NF;
    tau = tau_pow(tau, P.weno_b);
    double om0 = P.lam0 * (1.0 + tau / (P.weno_eps + si0));
    double om[NF];
    double wsum = om0;
#pragma unroll
    for (int s = 0; s < NF; ++s) {
      om[s] = P.lams * (1.0 + tau / (P.weno_eps + si[s]));
      wsum += om[s];
    }
    const double rw = 1.0 / wsum;  // wsum >= lam0 > 0
    const bool rwok = rl && wsum <= 0x1p60;
    om0 = rwok ? div_rn(om0, wsum, rw) : om0 / wsum;
#pragma unroll
    for (int s = 0; s < NF; ++s) om[s] = rwok ? div_rn(om[s], wsum, rw) : om[s] / wsum;
    double* bl = p1;  // blended in place (same operations; saves K registers)
#pragma unroll
    for (int k = 0; k < K; ++k) bl[k] = om0 * p1[k];
#pragma unroll
    for (int s = 0; s < NF; ++s) {
      bl[0] += om[s] * dir[s][0];
      bl[1] += om[s] * dir[s][1];
      bl[2] += om[s] * dir[s][2];
    }
    const bool chk = (v == 0 || v == 4);
    double blo = 0.0, bhi = 0.0, viol = -1e300;
    if (chk && P.mode == UCFVB_HYBRID) {
      blo = W.bounds[ao(c, v == 0 ? 0 : 2, 4)];
      bhi = W.bounds[ao(c, v == 0 ? 1 : 3, 4)];
    }
    if constexpr (DM) {
      // face values F(Q x 32) = u0 + phi(Q x K) . bl(K x 32) on the tensor cores
      constexpr int QT = (Q + 7) / 8, KS2 = (K + 3) / 4;
#pragma unroll
      for (int k = 0; k < K; ++k) sd[(v * K + k) * kRS + lane] = bl[k];
      __syncwarp();
      const double* sph = sp + EP + ED + EO;
      double f[QT][4][2];
#pragma unroll
      for (int i = 0; i < QT; ++i)
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
          f[i][tt][0] = su0[v * 32 + 8 * tt + 2 * fc];
          f[i][tt][1] = su0[v * 32 + 8 * tt + 2 * fc + 1];
        }
#pragma unroll
      for (int ks = 0; ks < KS2; ++ks) {
        const int k = 4 * ks + fc;
        double af[QT];
#pragma unroll
        for (int i = 0; i < QT; ++i) {
          const int q = 8 * i + fr;
          af[i] = (q < Q && k < K) ? sph[q * KP + k] : 0.0;
        }
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
          const double bf = k < K ? sd[(v * K + k) * kRS + 8 * tt + fr] : 0.0;
#pragma unroll
          for (int i = 0; i < QT; ++i) dmma884(f[i][tt][0], f[i][tt][1], af[i], bf);
        }
      }
#pragma unroll
      for (int i = 0; i < QT; ++i)
#pragma unroll
        for (int tt = 0; tt < 4; ++tt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int q = 8 * i + fr, cl = 8 * tt + 2 * fc + j;
            if (q < Q) {
              sval[q][v][cl] = f[i][tt][j];
              const int cc2 = scell[cl];
              if (!STAGED && cc2 >= 0) W.fp[static_cast<size_t>(D.slot[ao(cc2, q, Q)]) * V5 + v] = f[i][tt][j];
            }
          }
      __syncthreads();  // every face value of the chunk in sval
      if (chk)
        for (int q = 0; q < Q; ++q) {
          const double val = sval[q][v][lane];
          viol = smax(viol, smax(blo - val, val - bhi));
        }
    } else {
      __syncthreads();  // the gather buffer becomes the face-value buffer
      eval_store<K, NQ, NF, K, !STAGED>(D, W, c, op, v, lane, act, u0, bl, sval, chk, blo, bhi, viol, sl,
                                             STAGED ? sp + EP + ED + EO : nullptr);
    }
    const int sl_l = threadIdx.x / V5;  // cooperative stores: thread <-> (list entry sl_l, variable)
    if (STAGED && UCFVB_W5_PFID) {
      // this block's next tile: the stencil-id lines of its cells into L1 while the fallback votes
      // and the stores run (the five threads of a cell share its M + 1 + NF lines)
      const int nbase = base + nb * 32;
      if (nbase + sl_l < cnt) {
        const int ncell = list[nbase + sl_l];
#pragma unroll
        for (int e = threadIdx.x % V5; e < M + 1 + NF; e += V5)
          prefetch_l1(e <= M ? &D.central[ao(ncell, e, M + 1)] : &D.nbr[ao(ncell, e - M - 1, NF)]);
      }
    }
    troubled_fallback<NF, NQ, STAGED>(D, P, W, c, v, lane, act, u0, chk, blo, bhi, viol, sval, s_fail,
                                      (STAGED && base + sl_l < cnt) ? list[base + sl_l] : -1);
  }
}

// ---- MUSCL (solver.cpp:189-221; reconstruct.cpp:30-86) ---------------------------------
// resident blocks per SM asked of the lattice-class MUSCL kernel: five (72 registers, what its
// shared memory allows) measured 15.87 -> 15.29 ms/stage of config-5 weights against four (96)
#ifndef UCFVB_M3_MINB
#define UCFVB_M3_MINB 5
#endif
template <int K, int M, int NF, int NQ, bool STAGED>
__global__ void __launch_bounds__(160, STAGED ? UCFVB_M3_MINB : 0) k3_muscl(Dev3 D, Phys3 P, Work3 W, const double* __restrict__ U) {
  constexpr int Q = NF * NQ;
  constexpr int H1 = M / 2, H2 = M - H1 + NF;  // the two gathers
  constexpr int G = H2;
  extern __shared__ __align__(16) double smem3[];
  double* xs = smem3;
  auto sval = reinterpret_cast<double (*)[V5][33]>(smem3);
  // STAGED (lattice classes): the gathers are issued transposed (thread = (cell t / 5, variable
  // t % 5): a member's five variables are one 40-byte read) into rows of kMS doubles
  constexpr int XS = STAGED ? kMS : 160, VS = STAGED ? kVS : 32;
  double* sp = smem3 + (STAGED ? muscl_union(G, Q) : smem3_bytes(G, Q) / 8);  // STAGED: pinv_lin [3][M] | phi [Q][K]
  __shared__ int s_fail[32];
  const int lane = threadIdx.x & 31, v = threadIdx.x >> 5;
  const int t = STAGED ? blockIdx.x % W.ntl : 0;
  const int b0 = STAGED ? blockIdx.x / W.ntl : blockIdx.x, nb = STAGED ? gridDim.x / W.ntl : gridDim.x;
  const int cnt = W.counters[cnt_idx(W, kMuList, t)];
  const int32_t* list = list_of(W, kMuList, t);
  if (STAGED) {
    for (int e = threadIdx.x; e < 3 * M; e += 160) sp[e] = D.pinv_lin[ao(t, e, 3 * M)];
    for (int e = threadIdx.x; e < Q * K; e += 160) sp[3 * M + e] = D.phi[ao(t, e, Q * K)];
    __syncthreads();
  }
  for (int base = b0 * 32; base < cnt; base += nb * 32) {
    const bool act = base + lane < cnt;
    const int c = list[act ? base + lane : base];
    const int op = D.opi[c];
    const double u0 = U[static_cast<size_t>(c) * V5 + v];
    // two gathers of H1 and H2 values (all of each in flight), so the gather
    // buffer fits inside the face-value buffer: twice the resident blocks
    const int gl = STAGED ? threadIdx.x / V5 : lane, gv = STAGED ? threadIdx.x - gl * V5 : v;  // gather mapping
    const int gc = STAGED ? list[base + gl < cnt ? base + gl : base] : c;
    {
      int id[H1];
#pragma unroll
      for (int m = 0; m < H1; ++m) id[m] = D.central[ao(gc, m + 1, M + 1)];
#pragma unroll
      for (int g = 0; g < H1; ++g) cp_async8(&xs[g * XS + gv * VS + gl], &U[static_cast<size_t>(id[g]) * V5 + gv]);
      cp_async_commit();
    }
    // face-point slots, loaded while the gather is in flight (p <= 2; for p = 3
    // per face-point group: register pressure)
    constexpr bool kHoist = K * M <= 200;
    int slh[kHoist ? NF * NQ : 1];
    if (kHoist) {
#pragma unroll
      for (int q = 0; q < (kHoist ? NF * NQ : 0); ++q) slh[q] = D.slot[ao(c, q, NF * NQ)];
    }
    const int* sl = kHoist ? slh : nullptr;
    // the second half's ids, in flight during the first wait
    int id2[H2];
#pragma unroll
    for (int m = H1; m < M; ++m) id2[m - H1] = D.central[ao(gc, m + 1, M + 1)];
#pragma unroll
    for (int i = 0; i < NF; ++i) id2[M - H1 + i] = D.nbr[ao(gc, i, NF)];
    cp_async_wait_all();
    if (STAGED) __syncthreads();  // each value was copied by another thread
    double l0 = 0.0, l1 = 0.0, l2 = 0.0;
    double xv[H1];  // first half consumed into registers before the buffer is reused
#pragma unroll
    for (int m = 0; m < H1; ++m) xv[m] = xs[m * XS + v * VS + lane];
    if (STAGED) __syncthreads(); else __syncwarp();
    {
#pragma unroll
      for (int g = 0; g < H2; ++g) cp_async8(&xs[g * XS + gv * VS + gl], &U[static_cast<size_t>(id2[g]) * V5 + gv]);
      cp_async_commit();
    }
#pragma unroll
    for (int m = 0; m < H1; ++m) {
      const double x = xv[m] - u0;
      l0 = __fma_rn((STAGED ? sp[0 * M + m] : D.pinv_lin[ao(op, 0 * M + m, 3 * M)]), x, l0);
      l1 = __fma_rn((STAGED ? sp[1 * M + m] : D.pinv_lin[ao(op, 1 * M + m, 3 * M)]), x, l1);
      l2 = __fma_rn((STAGED ? sp[2 * M + m] : D.pinv_lin[ao(op, 2 * M + m, 3 * M)]), x, l2);
    }
    cp_async_wait_all();
    if (STAGED) __syncthreads();
#pragma unroll
    for (int m = H1; m < M; ++m) {
      const double x = xs[(m - H1) * XS + v * VS + lane] - u0;
      l0 = __fma_rn((STAGED ? sp[0 * M + m] : D.pinv_lin[ao(op, 0 * M + m, 3 * M)]), x, l0);
      l1 = __fma_rn((STAGED ? sp[1 * M + m] : D.pinv_lin[ao(op, 1 * M + m, 3 * M)]), x, l1);
      l2 = __fma_rn((STAGED ? sp[2 * M + m] : D.pinv_lin[ao(op, 2 * M + m, 3 * M)]), x, l2);
    }
    double lo = u0, hi = u0;
#pragma unroll
    for (int i = 0; i < NF; ++i) {
      const double x = xs[(M - H1 + i) * XS + v * VS + lane];
      lo = smin(lo, x);
      hi = smax(hi, x);
    }
    __syncthreads();  // the gather buffer becomes the face-value buffer
    double th = 1.0;
    const double e2 = D.eps2[c];
    for (int q = 0; q < Q; ++q) {
      const double uq = __fma_rn(l2, (STAGED ? sp[3 * M + q * K + 2] : D.phi[ao(op, q * K + 2, Q * K)]),
                                 __fma_rn(l1, (STAGED ? sp[3 * M + q * K + 1] : D.phi[ao(op, q * K + 1, Q * K)]),
                                          __fma_rn(l0, (STAGED ? sp[3 * M + q * K + 0] : D.phi[ao(op, q * K + 0, Q * K)]), u0)));
      th = (P.limiter == UCFVB_BARTH_JESPERSEN) ? bj_update(th, u0, lo, hi, uq) : venkat_update(th, u0, lo, hi, uq, e2);
    }
    if (P.limiter == UCFVB_BARTH_JESPERSEN) th = smax(th, 0.0);
    double a[K];
    a[0] = th * l0;
    a[1] = th * l1;
    a[2] = th * l2;
#pragma unroll
    for (int k = 3; k < K; ++k) a[k] = 0.0;
    const bool chk = (v == 0 || v == 4);
    double blo = 0.0, bhi = 0.0, viol = -1e300;
    if (chk && P.mode == UCFVB_HYBRID) {
      blo = W.bounds[ao(c, v == 0 ? 0 : 2, 4)];
      bhi = W.bounds[ao(c, v == 0 ? 1 : 3, 4)];
    }
    eval_store<K, NQ, NF, 3, !STAGED>(D, W, c, op, v, lane, act, u0, a, sval, chk, blo, bhi, viol, sl,
                                           STAGED ? sp + 3 * M : nullptr);
    const int sl_l = threadIdx.x / V5;  // cooperative stores: thread <-> (list entry sl_l, variable)
    if (STAGED && UCFVB_W5_PFID) {
      // this block's next tile: the stencil-id lines of its cells into L1 while the fallback votes
      // and the stores run (the five threads of a cell share its M + 1 + NF lines)
      const int nbase = base + nb * 32;
      if (nbase + sl_l < cnt) {
        const int ncell = list[nbase + sl_l];
#pragma unroll
        for (int e = threadIdx.x % V5; e < M + 1 + NF; e += V5)
          prefetch_l1(e <= M ? &D.central[ao(ncell, e, M + 1)] : &D.nbr[ao(ncell, e - M - 1, NF)]);
      }
    }
    troubled_fallback<NF, NQ, STAGED>(D, P, W, c, v, lane, act, u0, chk, blo, bhi, viol, sval, s_fail,
                                      (STAGED && base + sl_l < cnt) ? list[base + sl_l] : -1);
  }
}

// first-order everywhere (SchemeMode::First)
template <int NF, int NQ>
__global__ void k3_constant(Dev3 D, Work3 W, const double* __restrict__ U) {
  constexpr int Q = NF * NQ;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= D.n) return;
  W.labels[c] = UCFVB_SCHEME_FIRST;
  for (int q = 0; q < Q; ++q)
#pragma unroll
    for (int v = 0; v < V5; ++v) W.fp[static_cast<size_t>(D.slot[ao(c, q, Q)]) * V5 + v] = U[static_cast<size_t>(c) * V5 + v];
}

// ---- fluxes (solver.cpp:266-295) ----------------------------------------------------------
// resident 128-thread blocks per SM asked of the lane-per-point flux kernels: eight (64 registers)
// measured -6.6 % against the unbounded 72 (config 5 flux 4.96 -> 4.63 ms, config 4 773 -> 722 us)
#ifndef UCFVB_F3_MINB
#define UCFVB_F3_MINB 8
#endif
template <int NQ>
__global__ void __launch_bounds__(128) k3_face_flux(Dev3 D, Phys3 P, Work3 W) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= D.nF || halted(W)) return;
  double tot[V5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  bool ok = true;
  if (D.fown && D.fown[f] == 2) {  // subdomain boundary face of a halo cell: no flux, never owned
#pragma unroll
    for (int v = 0; v < V5; ++v) W.ff[static_cast<size_t>(f) * V5 + v] = 0.0;
    return;
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double* UL = &W.fp[(static_cast<size_t>(f) * 2 * NQ + q) * V5];  // [face][side][q][5]
    double ul[5], ur[5], n[3], fl[5];
#pragma unroll
    for (int v = 0; v < V5; ++v) ul[v] = UL[v], ur[v] = UL[NQ * V5 + v];
#pragma unroll
    for (int d = 0; d < 3; ++d) n[d] = D.fnrm[(static_cast<size_t>(f) * NQ + q) * 3 + d];
    ok = riemann3(P.hll, ul, ur, n, P.gamma, fl) && ok;
    const double w = D.fwa[static_cast<size_t>(f) * NQ + q];
#pragma unroll
    for (int v = 0; v < V5; ++v) tot[v] += w * fl[v];
  }
  if (!ok && (!D.fown || D.fown[f] == 1)) atomicMin(&W.counters[kBadFace], f);
#pragma unroll
  for (int v = 0; v < V5; ++v) W.ff[static_cast<size_t>(f) * V5 + v] = tot[v];
}

// NQ lanes per face (NQ a power of two): lane q evaluates the Riemann flux at
// point q, then every lane of the face sums the NQ weighted fluxes in q order
// through shuffles (the same total += w_q F_q sequence as one thread would)
template <int NQ>
__global__ void __launch_bounds__(128, UCFVB_F3_MINB) k3_face_flux_lanes(Dev3 D, Phys3 P, Work3 W) {
  constexpr int LP = NQ <= 1 ? 1 : (NQ <= 2 ? 2 : (NQ <= 4 ? 4 : 8));  // lanes per face (NQ <= 8)
  static_assert(NQ <= 8, "at most 8 points per face");
  if (halted(W)) return;  // block-uniform
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  const int f0 = g / LP, q0 = g % LP;
  const bool in = f0 < D.nF;
  const int f = in ? f0 : D.nF - 1;
  const int q = q0 < NQ ? q0 : 0;  // idle lanes recompute point 0 and are not summed
  const bool skip = D.fown && D.fown[f] == 2;  // subdomain boundary face of a halo cell
  double t[V5];
  bool ok = true;
  {
    const double* UL = &W.fp[(static_cast<size_t>(f) * 2 * NQ + q) * V5];  // [face][side][q][5]
    double ul[5], ur[5], n[3], fl[5];
#pragma unroll
    for (int v = 0; v < V5; ++v) ul[v] = UL[v], ur[v] = UL[NQ * V5 + v];
#pragma unroll
    for (int d = 0; d < 3; ++d) n[d] = D.fnrm[(static_cast<size_t>(f) * NQ + q) * 3 + d];
    ok = skip || riemann3(P.hll, ul, ur, n, P.gamma, fl);
    const double w = D.fwa[static_cast<size_t>(f) * NQ + q];
#pragma unroll
    for (int v = 0; v < V5; ++v) t[v] = w * fl[v];
  }
  const int lane = threadIdx.x & 31, base = lane & ~(LP - 1);
  double tot[V5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < NQ; ++j)
#pragma unroll
    for (int v = 0; v < V5; ++v) tot[v] += __shfl_sync(0xffffffffu, t[v], base + j);
  const bool fail = ((__ballot_sync(0xffffffffu, !ok && in) >> base) & ((1u << LP) - 1u)) != 0;
  if (!in || q0 != 0) return;
  if (fail && (!D.fown || D.fown[f] == 1)) atomicMin(&W.counters[kBadFace], f);
#pragma unroll
  for (int v = 0; v < V5; ++v) W.ff[static_cast<size_t>(f) * V5 + v] = skip ? 0.0 : tot[v];
}

// Point counts that are not a power of two (6-point triangle faces): 32 / NQ
// faces per warp, lane = (face, point), the warp's last 32 % NQ lanes idle
// (2 of 32 for NQ = 6). A warp reads its faces' points as one contiguous run
// of side-major rows, every lane carries one Riemann problem (a sixth of the
// registers and latency chain of the thread-per-face form), and the face's
// lanes sum the weighted fluxes in q order through shuffles.
#ifndef UCFVB_FLUX3_PACK
#define UCFVB_FLUX3_PACK 1
#endif
template <int NQ>
__global__ void __launch_bounds__(128, UCFVB_F3_MINB) k3_face_flux_pack(Dev3 D, Phys3 P, Work3 W) {
  constexpr int FPW = 32 / NQ;  // faces per warp
  if (halted(W)) return;        // block-uniform
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int fl0 = lane / NQ;
  const bool lane_on = fl0 < FPW;
  const int fl = lane_on ? fl0 : FPW - 1, q0 = lane_on ? lane - fl0 * NQ : 0;
  const int64_t f0 = warp * FPW + fl;
  const bool in = lane_on && f0 < D.nF;
  const int f = f0 < D.nF ? static_cast<int>(f0) : D.nF - 1;
  const int q = q0;
  const bool skip = D.fown && D.fown[f] == 2;  // subdomain boundary face of a halo cell
  double t[V5];
  bool ok = true;
  {
    const double* UL = &W.fp[(static_cast<size_t>(f) * 2 * NQ + q) * V5];  // [face][side][q][5]
    double ul[5], ur[5], n[3], fl5[5];
#pragma unroll
    for (int v = 0; v < V5; ++v) ul[v] = UL[v], ur[v] = UL[NQ * V5 + v];
#pragma unroll
    for (int d = 0; d < 3; ++d) n[d] = D.fnrm[(static_cast<size_t>(f) * NQ + q) * 3 + d];
    ok = skip || riemann3(P.hll, ul, ur, n, P.gamma, fl5);
    const double w = D.fwa[static_cast<size_t>(f) * NQ + q];
#pragma unroll
    for (int v = 0; v < V5; ++v) t[v] = w * fl5[v];
  }
  const int base = fl * NQ;
  double tot[V5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < NQ; ++j)
#pragma unroll
    for (int v = 0; v < V5; ++v) tot[v] += __shfl_sync(0xffffffffu, t[v], base + j);
  const bool fail = ((__ballot_sync(0xffffffffu, !ok && in) >> base) & ((1u << NQ) - 1u)) != 0;
  if (!in || q0 != 0) return;
  if (fail && (!D.fown || D.fown[f] == 1)) atomicMin(&W.counters[kBadFace], f);
#pragma unroll
  for (int v = 0; v < V5; ++v) W.ff[static_cast<size_t>(f) * V5 + v] = skip ? 0.0 : tot[v];
}

// ---- gather + RK combination (solver.cpp:296-311, time_integrator.cpp:31-38) --------------
// out = wa*ua + wb*ub + (wr*dt)*res, res = -acc*(1/vol); store_res keeps res (compute_residual tap / RK54)
// cells: nullable list of the cells to update (n_cells of them); else cells [0, D.n)
template <int NF>
__global__ void __launch_bounds__(256) k3_gather_rk(Dev3 D, Work3 W, const double* __restrict__ ua,
                                                    const double* __restrict__ ub, double* __restrict__ out,
                                                    double* __restrict__ res_out, double wa, double wb, double wr,
                                                    int combine, const int32_t* __restrict__ cells, int n_cells) {
  if (failed_before(W)) return;  // block-uniform
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (cells ? n_cells : D.n)) return;
  const int c = cells ? cells[i] : i;
  double acc[V5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < NF; ++i) {
    const int cf = D.cface[ao(c, i, NF)];
    const double sgn = (cf & 1) ? -1.0 : 1.0;
    const double* fl = &W.ff[static_cast<size_t>(cf >> 1) * V5];
#pragma unroll
    for (int v = 0; v < V5; ++v) acc[v] += sgn * fl[v];
  }
  const double iv = D.inv_vol[c];
  double r[V5];
#pragma unroll
  for (int v = 0; v < V5; ++v) r[v] = -acc[v] * iv;
  if (res_out) {
#pragma unroll
    for (int v = 0; v < V5; ++v) res_out[static_cast<size_t>(c) * V5 + v] = r[v];
  }
  if (combine) {
    const double wrdt = wr * W.dt[0];
#pragma unroll
    for (int v = 0; v < V5; ++v) {
      const size_t i = static_cast<size_t>(c) * V5 + v;
      out[i] = wa * ua[i] + wb * ub[i] + wrdt * r[v];
    }
  }
}

// SSPRK(5,4) final combination (time_integrator.cpp:66-73)
__global__ void k3_rk54_final(Work3 W, int64_t N, double* u, const double* ub, const double* uc, const double* rhs3,
                              const double* ud, const double* rhs, const double* dtp) {
  if (failed_before(W)) return;  // block-uniform: U keeps the failing step's input
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= N) return;
  const double dt = dtp[0];
  const double c52 = 0.517231671970585, c53 = 0.096059710526147, a53 = 0.063692468666290;
  const double c54 = 0.386708617503269, a54 = 0.226007483236906;
  u[i] = c52 * ub[i] + c53 * uc[i] + a53 * dt * rhs3[i] + c54 * ud[i] + a54 * dt * rhs[i];
}

// SSP-RK3 final stage result (written out of place) -> U, owned cells, when no failure was recorded
// (one failure check per block, 16-byte copies, four per thread: the one-double-per-thread
// form with three volatile counter loads in every thread ran at 0.6 TB/s)
__global__ void __launch_bounds__(256) k3_commit(Work3 W, int64_t N, double* __restrict__ u,
                                                 const double* __restrict__ src) {
  __shared__ int s_fail;
  if (threadIdx.x == 0) s_fail = failed_before(W) ? 1 : 0;
  __syncthreads();
  if (s_fail) return;
  const int64_t n2 = N >> 1;  // both arrays are cudaMalloc-aligned
  const double2* s2 = reinterpret_cast<const double2*>(src);
  double2* u2 = reinterpret_cast<double2*>(u);
  const int64_t b = static_cast<int64_t>(blockIdx.x) * 1024 + threadIdx.x;
  double2 x[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (b + j * 256 < n2) x[j] = s2[b + j * 256];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (b + j * 256 < n2) u2[b + j * 256] = x[j];
  if ((N & 1) && blockIdx.x == 0 && threadIdx.x == 0) u[N - 1] = src[N - 1];
}

// ---- max_stable_dt (solver.cpp:103-111) ----------------------------------------------------
__global__ void __launch_bounds__(256) k3_dt(Dev3 D, Phys3 P, Work3 W, const double* __restrict__ U) {
  if (halted(W)) return;  // block-uniform
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  double dt = 1e300;
  if (c < D.n_owned) {
    const double* s = &U[static_cast<size_t>(c) * V5];
    bool ok = s[0] > 0.0;
    if (ok) {
      const double u = s[1] / s[0], v = s[2] / s[0], w = s[3] / s[0];
      const double p = (P.gamma - 1.0) * (s[4] - 0.5 * s[0] * (u * u + v * v + w * w));
      ok = p > 0.0;
      if (ok) {
        const double speed = fabs(u) + fabs(v) + fabs(w) + sqrt(P.gamma * p / s[0]);
        dt = D.h[c] / speed;
      }
    }
    if (!ok) atomicMin(&W.counters[kBadCell], c);
  }
  // one atomic per block (min is order-free; per warp it was 393 k same-address atomics on config 5)
  for (int o = 16; o; o >>= 1) dt = smin(dt, __shfl_xor_sync(0xffffffffu, dt, o));
  __shared__ double s_dt[8];
  if ((threadIdx.x & 31) == 0) s_dt[threadIdx.x >> 5] = dt;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 1; i < 8; ++i) dt = smin(dt, s_dt[i]);
    atomicMin(W.dtmin, static_cast<unsigned long long>(__double_as_longlong(dt)));
  }
}

// halo exchange: owned values a peer holds as halo, packed in its order
__global__ void k3_halo_pack(const double* __restrict__ U, const int32_t* __restrict__ idx, int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * V5) return;
  out[i] = U[static_cast<size_t>(idx[i / V5]) * V5 + i % V5];
}

__global__ void k3_dt_init(Work3 W) { *W.dtmin = static_cast<unsigned long long>(__double_as_longlong(1e300)); }

__global__ void k3_dt_finalize(Work3 W, double cfl) {
  if (failed_before(W)) return;
  W.dt[0] = cfl * __longlong_as_double(static_cast<long long>(*W.dtmin));
}

__global__ void k3_time_add(Work3 W) {
  if (failed_before(W)) return;
  *W.t += W.dt[0];
}

// ---- dispatch ----------------------------------------------------------------------------------
struct Kern3 {
  size_t smem_central, smem_cwenoz, smem_muscl, smem_central_staged;
  void (*central)(Dev3, Phys3, Work3, const double*, int, int);
  void (*central_staged)(Dev3, Phys3, Work3, const double*, int, int);
  void (*central_tma)(Dev3, Phys3, Work3, const double*, int, int) = nullptr;  // per-cell rows, K*M <= 200
  size_t smem_central_tma = 0;
  void (*spread)(Dev3, Work3, const double*, int);
  void (*cwenoz)(Dev3, Phys3, Work3, const double*);
  void (*muscl)(Dev3, Phys3, Work3, const double*);
  void (*cwenoz_staged)(Dev3, Phys3, Work3, const double*);
  void (*muscl_staged)(Dev3, Phys3, Work3, const double*);
  size_t smem_cwenoz_staged, smem_muscl_staged, smem_cwenoz_base;
  void (*constant)(Dev3, Work3, const double*);
  void (*flux)(Dev3, Phys3, Work3);
  int flux_lanes = 1;
  void (*gather)(Dev3, Work3, const double*, const double*, double*, double*, double, double, double, int,
                 const int32_t*, int);
};

template <int K, int M, int NF, int NQ>
Kern3 kern3() {
  constexpr int Q = NF * NQ;
  Kern3 k{};
  k.smem_central = smem3_bytes(M + NF, Q) + (K * M <= 200 ? 8 * static_cast<size_t>(M * K * 32) : 0);
  k.smem_cwenoz_base = smem3_bytes(M, Q);
  k.smem_cwenoz = smem3_bytes(M, Q) + (K * M <= 200 ? 8 * static_cast<size_t>(M * K * 32) : 0);
  k.smem_muscl = smem3_bytes(M - M / 2 + NF, Q);
  // STAGED: the union buffer also holds the dofs [5][K][32] past the face values (K >= 8)
  constexpr int KP = K >= 8 ? kpad(K) : K;
  k.smem_central_staged = (K >= 8 ? 8 * dm_union(M + NF, Q, K) : smem3_bytes(M + NF, Q)) +
                          8 * static_cast<size_t>(M * KP + Q * KP + 160);
  k.smem_cwenoz_staged = (K >= 8 ? 8 * dm_union(M, Q, K) : smem3_bytes(M, Q)) +
                         8 * static_cast<size_t>(M * KP + NF * 3 * MD3 + ((K * KP + 1) & ~1) + Q * KP +
                                                 (K >= 8 ? 160 : 0)) +
                         4 * static_cast<size_t>(NF * MD3 + 32);
  k.smem_muscl_staged = 8 * muscl_union(M - M / 2 + NF, Q) + 8 * static_cast<size_t>(3 * M + Q * K);
  k.central = k3_central<K, M, NF, NQ, false>;
  if constexpr (K * M <= 200) {
    k.central_tma = k3_central<K, M, NF, NQ, false, true>;
    k.smem_central_tma = smem3_bytes(M + NF, Q) +
                         8 * static_cast<size_t>(M * K * 32 + (UCFVB_TMA3_PHI ? Q * K * 32
                                                                               : (UCFVB_C3_RING && Q % 4 == 0 ? kRingSlots * 4 * K * 32 : 0))) +
                         8 * (1 + kRingSlots);
  }
  k.central_staged = k3_central<K, M, NF, NQ, true>;
  k.spread = k3_spread<NF, NQ>;
  k.cwenoz = k3_cwenoz<K, M, NF, NQ, false>;
  k.muscl = k3_muscl<K, M, NF, NQ, false>;
  k.cwenoz_staged = k3_cwenoz<K, M, NF, NQ, true>;
  k.muscl_staged = k3_muscl<K, M, NF, NQ, true>;
  k.constant = k3_constant<NF, NQ>;
  // lanes per face when NQ is a power of two (config 4: flux 376 -> 316 us/stage at 96^3);
  // 6-point triangle faces keep one thread per face (8 lanes with 2 idle measured slower)
  if constexpr ((NQ & (NQ - 1)) == 0) {
    k.flux = k3_face_flux_lanes<NQ>;
    k.flux_lanes = NQ;
  } else if (UCFVB_FLUX3_PACK && NQ <= 16) {
    k.flux = k3_face_flux_pack<NQ>;
    k.flux_lanes = -(32 / NQ);  // negative: faces per warp
  } else {
    k.flux = k3_face_flux<NQ>;
    k.flux_lanes = 1;
  }
  k.gather = k3_gather_rk<NF>;
  return k;
}

bool pick3(int K, int M, int NF, int NQ, Kern3& k) {
#define PICK3(k_, m_, nf_, nq_) \
  if (K == k_ && M == m_ && NF == nf_ && NQ == nq_) return k = kern3<k_, m_, nf_, nq_>(), true;
  PICK3(3, 6, 6, 1)
  PICK3(9, 18, 6, 4)
  PICK3(19, 38, 6, 4)
  PICK3(3, 6, 4, 3)
  PICK3(9, 18, 4, 6)
  PICK3(19, 38, 4, 6)
#undef PICK3
  return false;
}

template <typename T>
T* dalloc(size_t count, std::vector<void*>& owned) {
  void* p = nullptr;
  CK3(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)));
  owned.push_back(p);
  return static_cast<T*>(p);
}

// 32-row AoSoA of a row-major [rows][E] host array
template <typename T>
std::vector<T> to_aosoa(const T* src, int64_t rows, int E, int n_threads) {
  const int64_t nch = (rows + 31) / 32;
  std::vector<T> out(static_cast<size_t>(nch) * 32 * E, T{});
  parallel_for(rows, n_threads, [&](int64_t a0, int64_t a1) {
    for (int64_t r = a0; r < a1; ++r)
      for (int e = 0; e < E; ++e) out[((r >> 5) * E + e) * 32 + (r & 31)] = src[r * E + e];
  });
  return out;
}

}  // namespace

struct GpuSolver3::Impl {
  int device = 0, n = 0, nF = 0, K = 0, M = 0, NF = 0, NQ = 0, Q = 0;
  ucfvb_options o{};
  Kern3 kern{};
  Dev3 D{};
  Phys3 P{};
  Work3 W{};
  cudaStream_t st = nullptr;
  std::vector<void*> owned;
  double *U = nullptr, *ua = nullptr, *ub = nullptr, *uc = nullptr, *ud = nullptr, *rhs = nullptr, *rhs3 = nullptr;
  uint8_t* step_labels = nullptr;
  int32_t* h_counters = nullptr;
  double* h_dt = nullptr;
  // advance_host_batch: device staging per direction, copy streams, events, pinned per-entry results
  double* pipe_up[2] = {nullptr, nullptr};
  double* pipe_down[2] = {nullptr, nullptr};
  cudaStream_t up_st = nullptr, down_st = nullptr;
  cudaEvent_t pipe_ev[8] = {};
  char* pipe_host = nullptr;
  int pipe_slots = 0;
  void free_pipe() {
    if (pipe_host) cudaFreeHost(pipe_host);
    for (auto& e : pipe_ev)
      if (e) cudaEventDestroy(e);
    if (up_st) cudaStreamDestroy(up_st);
    if (down_st) cudaStreamDestroy(down_st);
  }
  int64_t launches = 0, graph_launches = 0;
  int central_grid = 0, cw_grid = 0, mu_grid = 0;
  // decomposition: owned cells first; NCCL halo exchange after every stage
  int n_owned = 0;
  struct DevPeer {
    int rank, n_send, n_recv, recv_begin;
    size_t send_off;
    int32_t* send_idx;
  };
  std::vector<DevPeer> peers;
  double* sendbuf = nullptr;
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
  // owned cells some peer holds (updated first each stage) and the rest
  int32_t *sent_cells = nullptr, *interior_cells = nullptr;
  int n_sent = 0, n_interior = 0;
  cudaStream_t comm_st = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void exchange(double* buf, cudaStream_t s = nullptr) {
    if (!comm || peers.empty()) return;
    if (!s) s = st;
    for (const DevPeer& p : peers)
      if (p.n_send) {
        k3_halo_pack<<<(p.n_send * V5 + 255) / 256, 256, 0, s>>>(buf, p.send_idx, p.n_send, sendbuf + p.send_off);
        ++launches;
      }
    NK(nccl().GroupStart());
    for (const DevPeer& p : peers) {
      if (p.n_send) NK(nccl().Send(sendbuf + p.send_off, V5 * static_cast<size_t>(p.n_send), ncclDouble, p.rank, comm, s));
      if (p.n_recv)
        NK(nccl().Recv(buf + static_cast<size_t>(p.recv_begin) * V5, V5 * static_cast<size_t>(p.n_recv), ncclDouble,
                       p.rank, comm, s));
    }
    NK(nccl().GroupEnd());
  }
  bool staged = false;  // lattice-class operators on a type-blocked mesh
  cudaGraphExec_t step_graph = nullptr;
  int graph_rk = -1;
  // per-kernel-group timing (central, detect, weights, flux, gather+RK) with
  // events between the groups of un-graphed stages
  bool timing = false;
  cudaEvent_t ev[6] = {};
  double phase_s[5] = {0, 0, 0, 0, 0};
  void mark(int i) {
    if (timing) CK3(cudaEventRecord(ev[i], st));
  }
  void collect() {
    if (!timing) return;
    CK3(cudaEventSynchronize(ev[5]));
    for (int i = 0; i < 5; ++i) {
      float ms = 0.f;
      CK3(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
      phase_s[i] += 1e-3 * ms;
    }
  }

  void launch_stage(const double* Us, bool first, double* out, const double* wa_src, const double* wb_src,
                    double wa, double wb, double wr, double* res, int combine, bool xchg = true) {
    const int mode = o.mode;
    const bool nad = mode == UCFVB_HYBRID;
    const int nblk = (n + 255) / 256;
    mark(0);
    if (mode == UCFVB_LINEAR || mode == UCFVB_HYBRID) {  // forced CWENOZ solves inside k3_cwenoz
      if (staged)
        kern.central_staged<<<central_grid, 160, kern.smem_central_staged, st>>>(
            D, P, W, Us, 1, nad ? (1 | ((first || o.detect_every_stage) ? 2 : 0)) : 0);
      else
        kern.central<<<central_grid, 160, kern.smem_central, st>>>(D, P, W, Us, 1, nad ? 1 : 0);
      ++launches;
    }
    mark(1);
    if (nad) {
      kern.spread<<<nblk, 256, 0, st>>>(D, W, Us, (first || o.detect_every_stage) ? 1 : 0);
      ++launches;
    } else if (mode == UCFVB_CWENOZ || mode == UCFVB_MUSCL) {
      k3_fill_list<<<nblk, 256, 0, st>>>(n, mode == UCFVB_CWENOZ ? kCwList : kMuList,
                                         mode == UCFVB_CWENOZ ? UCFVB_SCHEME_CWENOZ : UCFVB_SCHEME_MUSCL, W);
      ++launches;
    } else if (mode == UCFVB_FIRST) {
      kern.constant<<<nblk, 256, 0, st>>>(D, W, Us);
      ++launches;
    } else {
      CK3(cudaMemsetAsync(W.labels, UCFVB_SCHEME_LINEAR, n, st));
    }
    mark(2);
    if (mode == UCFVB_HYBRID || mode == UCFVB_CWENOZ) {
      if (staged)
        kern.cwenoz_staged<<<cw_grid, 160, kern.smem_cwenoz_staged, st>>>(D, P, W, Us);
      else
        kern.cwenoz<<<cw_grid, 160, kern.smem_cwenoz, st>>>(D, P, W, Us);
      ++launches;
    }
    if (mode == UCFVB_HYBRID || mode == UCFVB_MUSCL) {
      if (staged)
        kern.muscl_staged<<<mu_grid, 160, kern.smem_muscl_staged, st>>>(D, P, W, Us);
      else
        kern.muscl<<<mu_grid, 160, kern.smem_muscl, st>>>(D, P, W, Us);
      ++launches;
    }
    mark(3);
    if (first) CK3(cudaMemcpyAsync(step_labels, W.labels, n, cudaMemcpyDeviceToDevice, st));
    {
      // threads: one per face, flux_lanes per face, or (flux_lanes < 0) a warp per -flux_lanes faces
      const int64_t thr = kern.flux_lanes > 0 ? static_cast<int64_t>(nF) * kern.flux_lanes
                                              : (static_cast<int64_t>(nF) + (-kern.flux_lanes) - 1) / (-kern.flux_lanes) * 32;
      kern.flux<<<static_cast<unsigned>((thr + 127) / 128), 128, 0, st>>>(D, P, W);
    }
    mark(4);
    if (sent_cells) {
      // subdomain: owned cells only, the cells peers hold first; with NCCL the
      // halo exchange then runs on the exchange stream (forked / joined with
      // events, inside the step graph) while the interior cells are updated
      const bool fork = combine && out && xchg && comm && !peers.empty();
      if (n_sent > 0)
        kern.gather<<<(n_sent + 255) / 256, 256, 0, st>>>(D, W, wa_src, wb_src, out, res, wa, wb, wr, combine,
                                                          sent_cells, n_sent);
      if (fork) {
        CK3(cudaEventRecord(ev_fork, st));
        CK3(cudaStreamWaitEvent(comm_st, ev_fork, 0));
        exchange(out, comm_st);
      }
      if (n_interior > 0)
        kern.gather<<<(n_interior + 255) / 256, 256, 0, st>>>(D, W, wa_src, wb_src, out, res, wa, wb, wr, combine,
                                                             interior_cells, n_interior);
      if (fork) {
        CK3(cudaEventRecord(ev_join, comm_st));
        CK3(cudaStreamWaitEvent(st, ev_join, 0));
      }
      launches += 3;
    } else {
      kern.gather<<<nblk, 256, 0, st>>>(D, W, wa_src, wb_src, out, res, wa, wb, wr, combine, nullptr, 0);
      launches += 2;
      if (combine && out && xchg) exchange(out);
    }
    mark(5);
    collect();
  }

  // one RK step on the device state U with the device dt W.dt
  // The step's result reaches U only through a final kernel gated on the
  // (all-reduced) error counters: k3_commit (RK3, last stage written out of
  // place into uc) or k3_rk54_final.
  void step(int rk) {
    const int64_t NO = static_cast<int64_t>(n_owned) * V5;
    if (rk == UCFVB_RK3) {
      launch_stage(U, true, ua, U, U, 1.0, 0.0, 1.0, nullptr, 1);
      launch_stage(ua, false, ub, U, ua, 0.75, 0.25, 0.25, nullptr, 1);
      launch_stage(ub, false, uc, U, ub, 1.0 / 3.0, 2.0 / 3.0, 2.0 / 3.0, nullptr, 1, false);
      allreduce_errors();
      k3_commit<<<static_cast<unsigned>((NO / 2 + 1023) / 1024 + 1), 256, 0, st>>>(W, NO, U, uc);
      ++launches;
      exchange(U);
      return;
    }
    const double a10 = 0.391752226571890;
    const double b20 = 0.444370493651235, b21 = 0.555629506348765, a21 = 0.368410593050371;
    const double b30 = 0.620101851488403, b32 = 0.379898148511597, a32 = 0.251891774271694;
    const double b40 = 0.178079954393132, b43 = 0.821920045606868, a43 = 0.544974750228521;
    launch_stage(U, true, ua, U, U, 1.0, 0.0, a10, nullptr, 1);
    launch_stage(ua, false, ub, U, ua, b20, b21, a21, nullptr, 1);
    launch_stage(ub, false, uc, U, ub, b30, b32, a32, nullptr, 1);
    launch_stage(uc, false, ud, U, uc, b40, b43, a43, rhs3, 1);
    launch_stage(ud, false, nullptr, nullptr, nullptr, 0, 0, 0, rhs, 0);
    allreduce_errors();
    k3_rk54_final<<<static_cast<unsigned>((NO + 255) / 256), 256, 0, st>>>(W, NO, U, ub, uc, rhs3, ud, rhs, W.dt);
    ++launches;
    exchange(U);
  }

  // every rank learns the job's failures (min face / cell) before any rank
  // commits the step, so all ranks keep the failing step's input
  void allreduce_errors() {
    if (comm) NK(nccl().AllReduce(W.counters + kBadFace, W.counters + kBadFace, 2, ncclInt32, ncclMin, comm, st));
  }

  void dt_kernels() {
    k3_dt_init<<<1, 1, 0, st>>>(W);
    k3_dt<<<(n + 255) / 256, 256, 0, st>>>(D, P, W, U);
    if (comm) NK(nccl().AllReduce(W.dtmin, W.dtmin, 1, ncclUint64, ncclMin, comm, st));  // positive doubles order as bits
    k3_dt_finalize<<<1, 1, 0, st>>>(W, o.cfl);
    launches += 3;
  }

  // one RK step (device dt, time advance) captured as a CUDA graph
  void capture(int rk) {
    if (step_graph) cudaGraphExecDestroy(step_graph);
    step_graph = nullptr;
    cudaGraph_t g = nullptr;
    const int64_t before = launches;
    CK3(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    dt_kernels();
    step(rk);
    k3_time_add<<<1, 1, 0, st>>>(W);
    ++launches;
    CK3(cudaStreamEndCapture(st, &g));
    CK3(cudaGraphInstantiate(&step_graph, g, 0));
    CK3(cudaGraphDestroy(g));
    graph_launches = launches - before;
    launches = before;
    graph_rk = rk;
  }

  void reset_errors() {
    const int32_t init[4] = {0, 0, 0x7fffffff, 0x7fffffff};  // halt, -, bad face, bad cell
    std::memcpy(h_counters, init, sizeof init);
    CK3(cudaMemcpyAsync(W.counters, h_counters, sizeof init, cudaMemcpyHostToDevice, st));
  }

  void check_errors() {
    CK3(cudaMemcpyAsync(h_counters, W.counters, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK3(cudaStreamSynchronize(st));
    CK3(cudaGetLastError());
    if (h_counters[kBadFace] != 0x7fffffff)
      throw ApiError(UCFVB_NONPHYSICAL, "non-physical state at face " + std::to_string(h_counters[kBadFace]));
    if (h_counters[kBadCell] != 0x7fffffff)
      throw ApiError(UCFVB_NONPHYSICAL, "non-physical state in cell " + std::to_string(h_counters[kBadCell]));
  }
};

GpuSolver3::GpuSolver3(const ucfvb3_mesh_view& m, const ucfvb3_stencil_view& s, const ucfvb_options& o, int device,
                       const ucfvb3_subdomain* sub)
    : p_(new Impl) {
  Impl& I = *p_;
  try {
    if (m.n_cells != s.n_cells || m.nf != s.nf || m.nq != s.nq || s.MD != MD3)
      throw ApiError(UCFVB_INVALID, "solver3d: stencils do not match the mesh");
    if (o.mode < UCFVB_LINEAR || o.mode > UCFVB_FIRST) throw ApiError(UCFVB_INVALID, "solver3d: unknown mode");
    if (!(o.lambda1p > 1.0)) throw ApiError(UCFVB_INVALID, "cwenoz: central linear weight lambda1' must exceed 1");
    if (o.margins.alpha_m < 0.0 || o.margins.beta_m < 0.0)
      throw ApiError(UCFVB_INVALID, "NAD margins: alpha_m and beta_m must be non-negative");
    if (o.margins.beta_w > 0.0 && (o.margins.beta_w > o.margins.beta_m || o.margins.alpha_w > o.margins.alpha_m))
      throw ApiError(UCFVB_INVALID, "NAD margins: delta_w <= delta_m requires beta_w <= beta_m and alpha_w <= alpha_m");
    if (o.margins.kappa < 0.0) throw ApiError(UCFVB_INVALID, "NAD margins: kappa must be >= 0");
    I.o = o;
    I.n = m.n_cells, I.nF = m.n_faces, I.K = s.K, I.M = s.M, I.NF = m.nf, I.NQ = m.nq, I.Q = s.Q;
    if (!pick3(I.K, I.M, I.NF, I.NQ, I.kern))
      throw ApiError(UCFVB_UNSUPPORTED, "solver3d: no kernel instance for K=" + std::to_string(I.K) +
                                            " M=" + std::to_string(I.M) + " nf=" + std::to_string(I.NF) +
                                            " nq=" + std::to_string(I.NQ));
    I.device = device;
    CK3(cudaSetDevice(device));
    CK3(cudaStreamCreateWithFlags(&I.st, cudaStreamNonBlocking));
    const int n = I.n, K = I.K, M = I.M, NF = I.NF, NQ = I.NQ, Q = I.Q, nops = s.n_ops;
    const int nth = 0;
    auto up = [&](auto* dst, const auto& host) {
      CK3(cudaMemcpy(dst, host.data(), host.size() * sizeof(host[0]), cudaMemcpyHostToDevice));
    };
    auto upload_ao = [&](auto ptr, int64_t rows, int E) {
      using T = std::remove_const_t<std::remove_pointer_t<decltype(ptr)>>;
      auto h = to_aosoa<T>(ptr, rows, E, nth);
      T* d = dalloc<T>(h.size(), I.owned);
      up(d, h);
      return static_cast<const T*>(d);
    };
    Dev3& D = I.D;
    D.n = n, D.nF = I.nF, D.n_ops = nops;
    I.n_owned = D.n_owned = sub ? sub->n_owned : n;
    D.fown = nullptr;
    if (sub) {
      std::vector<uint8_t> fo(I.nF, 0);
      for (int f = 0; f < I.nF; ++f)
        fo[f] = m.face_left[f] == m.face_right[f] ? 2 : ((m.face_left[f] < I.n_owned || m.face_right[f] < I.n_owned) ? 1 : 0);
      uint8_t* d = dalloc<uint8_t>(fo.size(), I.owned);
      up(d, fo);
      D.fown = d;
      size_t off = 0;
      for (const auto& pr : sub->peers) {
        Impl::DevPeer dp{pr.rank, static_cast<int>(pr.send.size()), pr.n_recv, pr.recv_begin, off, nullptr};
        if (dp.n_send) {
          dp.send_idx = dalloc<int32_t>(pr.send.size(), I.owned);
          up(dp.send_idx, pr.send);
        }
        off += static_cast<size_t>(dp.n_send) * V5;
        I.peers.push_back(dp);
      }
      I.sendbuf = dalloc<double>(std::max<size_t>(off, 1), I.owned);
      std::vector<uint8_t> is_sent(I.n_owned, 0);
      for (const auto& pr : sub->peers)
        for (int32_t c : pr.send) is_sent[c] = 1;
      std::vector<int32_t> sent, interior;
      for (int c = 0; c < I.n_owned; ++c) (is_sent[c] ? sent : interior).push_back(c);
      I.n_sent = static_cast<int>(sent.size());
      I.n_interior = static_cast<int>(interior.size());
      I.sent_cells = dalloc<int32_t>(std::max<size_t>(sent.size(), 1), I.owned);
      I.interior_cells = dalloc<int32_t>(std::max<size_t>(interior.size(), 1), I.owned);
      if (!sent.empty()) up(I.sent_cells, sent);
      if (!interior.empty()) up(I.interior_cells, interior);
      CK3(cudaStreamCreateWithFlags(&I.comm_st, cudaStreamNonBlocking));
      CK3(cudaEventCreateWithFlags(&I.ev_fork, cudaEventDisableTiming));
      CK3(cudaEventCreateWithFlags(&I.ev_join, cudaEventDisableTiming));
    }
    D.central = upload_ao(s.central, n, M + 1);
    D.nbr = upload_ao(m.cell_nbr, n, NF);
    {
      // device face-point order [face][side][q] (the view's slot is (face*nq + q)*2 + side): the
      // points a cell writes on one face are one contiguous run of nq*40 bytes (config 4: five
      // whole sectors, config 5: 7.5) instead of nq 40-byte pieces interleaved with the other side's
      std::vector<int32_t> ds(static_cast<size_t>(n) * Q);
      for (size_t i = 0; i < ds.size(); ++i) {
        const int32_t sl = s.qp_slot[i];
        const int32_t side = sl & 1, fq = sl >> 1, f = fq / NQ, q = fq - f * NQ;
        ds[i] = (f * 2 + side) * NQ + q;
      }
      D.slot = upload_ao(ds.data(), n, Q);
    }
    {
      std::vector<int32_t> cf(static_cast<size_t>(n) * NF);
      for (size_t i = 0; i < cf.size(); ++i) cf[i] = (m.cell_faces[i] << 1) | (m.cell_side[i] ? 1 : 0);
      D.cface = upload_ao(cf.data(), n, NF);
    }
    {
      int32_t* d = dalloc<int32_t>(n, I.owned);
      CK3(cudaMemcpy(d, s.op_index, sizeof(int32_t) * n, cudaMemcpyHostToDevice));
      D.opi = d;
    }
    std::vector<double> thr(n), eps2(n), iv(n), hh(n);
    for (int c = 0; c < n; ++c) {
      thr[c] = std::pow(o.margins.kappa * m.cell_h[c], o.margins.deact_n);  // deactivate_smooth (detector.cpp:34)
      eps2[c] = std::pow(o.venkat_kappa * m.cell_h[c], 3);                   // solver.cpp:203
      iv[c] = 1.0 / m.cell_volume[c];
      hh[c] = m.cell_h[c];
    }
    auto upd = [&](const std::vector<double>& h) {
      double* d = dalloc<double>(h.size(), I.owned);
      up(d, h);
      return static_cast<const double*>(d);
    };
    D.thr = upd(thr), D.eps2 = upd(eps2), D.inv_vol = upd(iv), D.h = upd(hh);
    {
      // pinv [K][M] -> [M][K] (m-major), then AoSoA
      std::vector<double> t(static_cast<size_t>(nops) * K * M);
      for (int64_t r = 0; r < nops; ++r)
        for (int k = 0; k < K; ++k)
          for (int mm = 0; mm < M; ++mm) t[(r * M + mm) * K + k] = s.pinv[(r * K + k) * M + mm];
      D.pinv = upload_ao(t.data(), nops, M * K);
    }
    D.pinv_lin = upload_ao(s.pinv_lin, nops, 3 * M);
    D.dirm = upload_ao(s.dir_members, nops, NF * MD3);
    D.pinv_dir = upload_ao(s.pinv_dir, nops, NF * 3 * MD3);
    D.oi = upload_ao(s.oi, nops, K * K);
    D.phi = upload_ao(s.phi, nops, Q * K);
    {
      double* fn = dalloc<double>(static_cast<size_t>(I.nF) * NQ * 3, I.owned);
      double* fw = dalloc<double>(static_cast<size_t>(I.nF) * NQ, I.owned);
      CK3(cudaMemcpy(fn, m.face_normal, sizeof(double) * I.nF * NQ * 3, cudaMemcpyHostToDevice));
      CK3(cudaMemcpy(fw, m.face_wa, sizeof(double) * I.nF * NQ, cudaMemcpyHostToDevice));
      D.fnrm = fn, D.fwa = fw;
    }
    Phys3& P = I.P;
    P.gamma = o.gamma, P.cfl = o.cfl, P.lambda1p = o.lambda1p, P.weno_eps = o.weno_eps, P.weno_b = o.weno_b;
    P.lam0 = 1.0 - 1.0 / o.lambda1p;            // reconstruct.cpp:113
    P.lams = (1.0 - P.lam0) / (I.NF + 1 - 1);   // reconstruct.cpp:114
    P.inv_lam0 = 1.0 / P.lam0;
    P.mg = MarginParams{o.margins.alpha_m, o.margins.beta_m, o.margins.alpha_w, o.margins.beta_w, o.margins.kappa,
                        o.margins.deact_n};
    P.mode = o.mode, P.limiter = o.limiter, P.hll = o.riemann == UCFVB_HLL ? 1 : 0;
    Work3& W = I.W;
    const int64_t nch = (n + 31) / 32;
    W.fp = dalloc<double>(static_cast<size_t>(I.nF) * NQ * 2 * V5, I.owned);
    W.ff = dalloc<double>(static_cast<size_t>(I.nF) * V5, I.owned);
    W.bounds = dalloc<double>(static_cast<size_t>(nch) * 32 * 4, I.owned);
    W.raw = dalloc<uint8_t>(n, I.owned);
    W.labels = dalloc<uint8_t>(n, I.owned);
    const bool staged_lists = (nops == m.n_types && m.cell_order == 1 && nops > 1);
    W.ntl = staged_lists ? nops : 1;
    W.cap = staged_lists ? n / nops : n;
    W.lists = dalloc<int32_t>(static_cast<size_t>(2) * W.ntl * W.cap, I.owned);
    W.counters = dalloc<int32_t>(kCnt0 + 2 * W.ntl, I.owned);
    W.dtmin = dalloc<unsigned long long>(1, I.owned);
    W.dt = dalloc<double>(1, I.owned);
    W.t = dalloc<double>(1, I.owned);
    W.ties = dalloc<unsigned long long>(1, I.owned);
    CK3(cudaMemset(W.fp, 0, sizeof(double) * static_cast<size_t>(I.nF) * NQ * 2 * V5));
    CK3(cudaMemset(W.labels, 0, n));
    CK3(cudaMemset(W.counters, 0, (kCnt0 + 2 * W.ntl) * sizeof(int32_t)));
    CK3(cudaMemset(W.ties, 0, sizeof(unsigned long long)));
    I.step_labels = dalloc<uint8_t>(n, I.owned);
    CK3(cudaMemset(I.step_labels, 0, n));
    const size_t sz = static_cast<size_t>(n) * V5;
    I.U = dalloc<double>(sz, I.owned);
    I.ua = dalloc<double>(sz, I.owned);
    I.ub = dalloc<double>(sz, I.owned);
    I.uc = dalloc<double>(sz, I.owned);
    I.ud = dalloc<double>(sz, I.owned);
    I.rhs = dalloc<double>(sz, I.owned);
    I.rhs3 = dalloc<double>(sz, I.owned);
    CK3(cudaMemset(I.U, 0, sz * sizeof(double)));
    CK3(cudaMallocHost(&I.h_counters, 4 * sizeof(int32_t)));
    CK3(cudaMallocHost(&I.h_dt, 2 * sizeof(double)));
    int sms = 148;
    CK3(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    auto grid_for = [&](auto fn, size_t smem) {
      CK3(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      int per = 1;
      CK3(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 160, smem));
      return std::max(1, static_cast<int>(std::min<int64_t>(nch, static_cast<int64_t>(sms) * std::max(1, per))));
    };
    I.staged = (nops == m.n_types && m.cell_order == 1 && nops > 1);
    if (I.staged) {
      I.central_grid = grid_for(I.kern.central_staged, I.kern.smem_central_staged);
      I.central_grid = std::max(nops, I.central_grid - I.central_grid % nops);  // block b <-> type b % n_ops
    } else {
      // per-cell rows: the TMA-staged central kernel (UCFVB_CENTRAL3_TMA=0: the cp.async one, diagnostics)
      const char* e = std::getenv("UCFVB_CENTRAL3_TMA");
      if (I.kern.central_tma && nops == n && !(e && e[0] == '0')) {
        I.kern.central = I.kern.central_tma;
        I.kern.smem_central = I.kern.smem_central_tma;
      }
      I.central_grid = grid_for(I.kern.central, I.kern.smem_central);
    }
    if (I.staged) {
      I.cw_grid = grid_for(I.kern.cwenoz_staged, I.kern.smem_cwenoz_staged);
      I.cw_grid = std::max(nops, I.cw_grid - I.cw_grid % nops);
      I.mu_grid = grid_for(I.kern.muscl_staged, I.kern.smem_muscl_staged);
      I.mu_grid = std::max(nops, I.mu_grid - I.mu_grid % nops);
    } else {
      // the per-cell pinv staging region is only used by forced CWENOZ (identity list)
      if (o.mode != UCFVB_CWENOZ) I.kern.smem_cwenoz = I.kern.smem_cwenoz_base;
      I.cw_grid = grid_for(I.kern.cwenoz, I.kern.smem_cwenoz);
      I.mu_grid = grid_for(I.kern.muscl, I.kern.smem_muscl);
    }
    I.reset_errors();
    CK3(cudaStreamSynchronize(I.st));
  } catch (...) {
    for (void* q : I.owned) cudaFree(q);
    if (I.h_counters) cudaFreeHost(I.h_counters);
    if (I.h_dt) cudaFreeHost(I.h_dt);
    if (I.st) cudaStreamDestroy(I.st);
    if (I.comm_st) cudaStreamDestroy(I.comm_st);
    if (I.ev_fork) cudaEventDestroy(I.ev_fork);
    if (I.ev_join) cudaEventDestroy(I.ev_join);
    for (auto& e : I.ev)
      if (e) cudaEventDestroy(e);
    delete p_;
    throw;
  }
}

GpuSolver3::~GpuSolver3() {
  Impl& I = *p_;
  cudaSetDevice(I.device);
  if (I.step_graph) cudaGraphExecDestroy(I.step_graph);
  if (I.st) cudaStreamSynchronize(I.st);
  for (auto& e : I.ev)
    if (e) cudaEventDestroy(e);
  if (I.comm) nccl().CommDestroy(I.comm);
  for (void* q : I.owned) cudaFree(q);
  if (I.h_counters) cudaFreeHost(I.h_counters);
  if (I.h_dt) cudaFreeHost(I.h_dt);
  I.free_pipe();
  if (I.st) cudaStreamDestroy(I.st);
  if (I.comm_st) cudaStreamDestroy(I.comm_st);
  if (I.ev_fork) cudaEventDestroy(I.ev_fork);
  if (I.ev_join) cudaEventDestroy(I.ev_join);
  delete p_;
}

void GpuSolver3::set_state(const double* u) {
  CK3(cudaSetDevice(p_->device));
  CK3(cudaMemcpyAsync(p_->U, u, sizeof(double) * p_->n * V5, cudaMemcpyHostToDevice, p_->st));
  CK3(cudaStreamSynchronize(p_->st));
}
void GpuSolver3::get_state(double* u) {
  CK3(cudaSetDevice(p_->device));
  CK3(cudaMemcpyAsync(u, p_->U, sizeof(double) * p_->n * V5, cudaMemcpyDeviceToHost, p_->st));
  CK3(cudaStreamSynchronize(p_->st));
}

double GpuSolver3::max_stable_dt() {
  Impl& I = *p_;
  CK3(cudaSetDevice(I.device));
  I.reset_errors();
  I.dt_kernels();
  CK3(cudaMemcpyAsync(I.h_dt, I.W.dt, sizeof(double), cudaMemcpyDeviceToHost, I.st));
  I.check_errors();
  return I.h_dt[0];
}

void GpuSolver3::advance(double dt, double t, int rk) {
  Impl& I = *p_;
  (void)t;
  if (rk != UCFVB_RK3 && rk != UCFVB_RK54) throw ApiError(UCFVB_INVALID, "advance: unknown integrator");
  CK3(cudaSetDevice(I.device));
  I.reset_errors();
  I.h_dt[1] = dt;
  CK3(cudaMemcpyAsync(I.W.dt, &I.h_dt[1], sizeof(double), cudaMemcpyHostToDevice, I.st));
  I.step(rk);
  I.check_errors();
}

double GpuSolver3::run_steps(int n_steps, double t0, int rk) {
  Impl& I = *p_;
  if (rk != UCFVB_RK3 && rk != UCFVB_RK54) throw ApiError(UCFVB_INVALID, "run_steps: unknown integrator");
  CK3(cudaSetDevice(I.device));
  I.reset_errors();
  I.h_dt[1] = t0;
  CK3(cudaMemcpyAsync(I.W.t, &I.h_dt[1], sizeof(double), cudaMemcpyHostToDevice, I.st));
  if (I.timing) {
    for (int i = 0; i < n_steps; ++i) {
      I.dt_kernels();
      I.step(rk);
      k3_time_add<<<1, 1, 0, I.st>>>(I.W);
      ++I.launches;
    }
    CK3(cudaMemcpyAsync(I.h_dt, I.W.t, sizeof(double), cudaMemcpyDeviceToHost, I.st));
    I.check_errors();
    return I.h_dt[0];
  }
  if (!I.step_graph || I.graph_rk != rk) I.capture(rk);
  for (int i = 0; i < n_steps; ++i) {
    CK3(cudaGraphLaunch(I.step_graph, I.st));
    I.launches += I.graph_launches;
  }
  CK3(cudaMemcpyAsync(I.h_dt, I.W.t, sizeof(double), cudaMemcpyDeviceToHost, I.st));
  I.check_errors();
  return I.h_dt[0];
}

// host state in -> n_steps graph-replayed steps -> host state out, one synchronisation
double GpuSolver3::advance_host(const double* u_in, double* u_out, int n_steps, int rk, double t0) {
  Impl& I = *p_;
  if (rk != UCFVB_RK3 && rk != UCFVB_RK54) throw ApiError(UCFVB_INVALID, "advance_host: unknown integrator");
  if (n_steps <= 0) throw ApiError(UCFVB_INVALID, "advance_host: n_steps must be >= 1");
  CK3(cudaSetDevice(I.device));
  const size_t bytes = sizeof(double) * static_cast<size_t>(I.n) * V5;
  CK3(cudaMemcpyAsync(I.U, u_in, bytes, cudaMemcpyHostToDevice, I.st));
  I.reset_errors();
  I.h_dt[1] = t0;
  CK3(cudaMemcpyAsync(I.W.t, &I.h_dt[1], sizeof(double), cudaMemcpyHostToDevice, I.st));
  if (!I.timing && (!I.step_graph || I.graph_rk != rk)) I.capture(rk);
  for (int i = 0; i < n_steps; ++i) {
    if (I.timing) {
      I.dt_kernels();
      I.step(rk);
      k3_time_add<<<1, 1, 0, I.st>>>(I.W);
      ++I.launches;
    } else {
      CK3(cudaGraphLaunch(I.step_graph, I.st));
      I.launches += I.graph_launches;
    }
  }
  CK3(cudaMemcpyAsync(I.h_dt, I.W.t, sizeof(double), cudaMemcpyDeviceToHost, I.st));
  CK3(cudaMemcpyAsync(I.h_counters, I.W.counters, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, I.st));
  CK3(cudaMemcpyAsync(u_out, I.U, bytes, cudaMemcpyDeviceToHost, I.st));
  CK3(cudaStreamSynchronize(I.st));
  CK3(cudaGetLastError());
  if (I.h_counters[kBadFace] != 0x7fffffff)
    throw ApiError(UCFVB_NONPHYSICAL, "non-physical state at face " + std::to_string(I.h_counters[kBadFace]));
  if (I.h_counters[kBadCell] != 0x7fffffff)
    throw ApiError(UCFVB_NONPHYSICAL, "non-physical state in cell " + std::to_string(I.h_counters[kBadCell]));
  return I.h_dt[0];
}

// advance_host over independent states, pipelined as the 2D ucfvb_advance_host_batch: the upload
// of entry i+1 and the download of entry i-1 run on copy streams while entry i is stepped (two
// device staging buffers per direction, device-to-device copies into and out of U).
void GpuSolver3::advance_host_batch(int n_batch, const double* const* u_in, double* const* u_out, int n_steps, int rk,
                                    double t0, double* t_out) {
  Impl& I = *p_;
  if (rk != UCFVB_RK3 && rk != UCFVB_RK54) throw ApiError(UCFVB_INVALID, "advance_host_batch: unknown integrator");
  if (n_steps <= 0) throw ApiError(UCFVB_INVALID, "advance_host_batch: n_steps must be >= 1");
  if (n_batch <= 0) throw ApiError(UCFVB_INVALID, "advance_host_batch: n_batch must be >= 1");
  for (int i = 0; i < n_batch; ++i)
    if (!u_in[i] || !u_out[i]) throw ApiError(UCFVB_INVALID, "advance_host_batch: null state pointer");
  CK3(cudaSetDevice(I.device));
  const size_t count = static_cast<size_t>(I.n) * V5, bytes = sizeof(double) * count;
  if (!I.pipe_up[0]) {
    for (int i = 0; i < 2; ++i) {
      I.pipe_up[i] = dalloc<double>(count, I.owned);
      I.pipe_down[i] = dalloc<double>(count, I.owned);
    }
    CK3(cudaStreamCreateWithFlags(&I.up_st, cudaStreamNonBlocking));
    CK3(cudaStreamCreateWithFlags(&I.down_st, cudaStreamNonBlocking));
    for (auto& e : I.pipe_ev) CK3(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // pinned per entry: t0 (in), final t (out), the four error counters (out), the counters' reset values (in)
  const size_t slot = 2 * sizeof(double) + 8 * sizeof(int32_t);
  if (I.pipe_slots < n_batch) {
    if (I.pipe_host) CK3(cudaFreeHost(I.pipe_host));
    I.pipe_host = nullptr;
    CK3(cudaMallocHost(&I.pipe_host, slot * n_batch));
    I.pipe_slots = n_batch;
  }
  auto h_t = [&](int i) { return reinterpret_cast<double*>(I.pipe_host + slot * i); };
  auto h_c = [&](int i) { return reinterpret_cast<int32_t*>(I.pipe_host + slot * i + 2 * sizeof(double)); };
  if (!I.timing && (!I.step_graph || I.graph_rk != rk)) I.capture(rk);
  // events: [0..1] upload landed, [2..3] upload buffer consumed, [4..5] result staged, [6..7] download done
  cudaEvent_t* ev = I.pipe_ev;
  for (int i = 0; i < n_batch; ++i) {
    const int b = i & 1;
    if (i >= 2) CK3(cudaStreamWaitEvent(I.up_st, ev[2 + b], 0));
    CK3(cudaMemcpyAsync(I.pipe_up[b], u_in[i], bytes, cudaMemcpyHostToDevice, I.up_st));
    CK3(cudaEventRecord(ev[b], I.up_st));
    CK3(cudaStreamWaitEvent(I.st, ev[b], 0));
    CK3(cudaMemcpyAsync(I.U, I.pipe_up[b], bytes, cudaMemcpyDeviceToDevice, I.st));
    CK3(cudaEventRecord(ev[2 + b], I.st));
    const int32_t init[4] = {0, 0, 0x7fffffff, 0x7fffffff};  // halt, -, bad face, bad cell (reset_errors)
    std::memcpy(h_c(i) + 4, init, sizeof init);
    CK3(cudaMemcpyAsync(I.W.counters, h_c(i) + 4, sizeof init, cudaMemcpyHostToDevice, I.st));
    h_t(i)[0] = t0;
    CK3(cudaMemcpyAsync(I.W.t, &h_t(i)[0], sizeof(double), cudaMemcpyHostToDevice, I.st));
    for (int s = 0; s < n_steps; ++s) {
      if (I.timing) {
        I.dt_kernels();
        I.step(rk);
        k3_time_add<<<1, 1, 0, I.st>>>(I.W);
        ++I.launches;
      } else {
        CK3(cudaGraphLaunch(I.step_graph, I.st));
        I.launches += I.graph_launches;
      }
    }
    CK3(cudaMemcpyAsync(&h_t(i)[1], I.W.t, sizeof(double), cudaMemcpyDeviceToHost, I.st));
    CK3(cudaMemcpyAsync(h_c(i), I.W.counters, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, I.st));
    if (i >= 2) CK3(cudaStreamWaitEvent(I.st, ev[6 + b], 0));
    CK3(cudaMemcpyAsync(I.pipe_down[b], I.U, bytes, cudaMemcpyDeviceToDevice, I.st));
    CK3(cudaEventRecord(ev[4 + b], I.st));
    CK3(cudaStreamWaitEvent(I.down_st, ev[4 + b], 0));
    CK3(cudaMemcpyAsync(u_out[i], I.pipe_down[b], bytes, cudaMemcpyDeviceToHost, I.down_st));
    CK3(cudaEventRecord(ev[6 + b], I.down_st));
  }
  CK3(cudaStreamSynchronize(I.st));
  CK3(cudaStreamSynchronize(I.down_st));
  CK3(cudaGetLastError());
  I.reset_errors();
  for (int i = 0; i < n_batch; ++i) {
    // every entry starts from reset counters: a failing entry (its result is its failing step's
    // input) leaves the others untouched; the first one is reported
    if (h_c(i)[kBadFace] != 0x7fffffff)
      throw ApiError(UCFVB_NONPHYSICAL, "non-physical state at face " + std::to_string(h_c(i)[kBadFace]) +
                                            " (batch entry " + std::to_string(i) + ")");
    if (h_c(i)[kBadCell] != 0x7fffffff)
      throw ApiError(UCFVB_NONPHYSICAL, "non-physical state in cell " + std::to_string(h_c(i)[kBadCell]) +
                                            " (batch entry " + std::to_string(i) + ")");
    if (t_out) t_out[i] = h_t(i)[1];
  }
}

void GpuSolver3::compute_residual(const double* u, double t, double* out) {
  Impl& I = *p_;
  (void)t;
  CK3(cudaSetDevice(I.device));
  I.reset_errors();
  CK3(cudaMemcpyAsync(I.ua, u, sizeof(double) * I.n * V5, cudaMemcpyHostToDevice, I.st));
  I.launch_stage(I.ua, true, nullptr, nullptr, nullptr, 0, 0, 0, I.rhs, 0);
  CK3(cudaMemcpyAsync(out, I.rhs, sizeof(double) * I.n * V5, cudaMemcpyDeviceToHost, I.st));
  I.check_errors();
}

void GpuSolver3::set_phase_timing(bool on) {
  Impl& I = *p_;
  CK3(cudaSetDevice(I.device));
  if (on && !I.ev[0])
    for (auto& e : I.ev) CK3(cudaEventCreate(&e));
  if (on && I.step_graph) {  // graphs bypass the per-group events
    cudaGraphExecDestroy(I.step_graph);
    I.step_graph = nullptr;
  }
  I.timing = on;
}

void GpuSolver3::phase_times(double out[5]) {
  for (int i = 0; i < 5; ++i) out[i] = p_->phase_s[i];
}

void GpuSolver3::get_labels(int which, uint8_t* out) {
  CK3(cudaSetDevice(p_->device));
  CK3(cudaMemcpyAsync(out, which ? p_->step_labels : p_->W.labels, p_->n, cudaMemcpyDeviceToHost, p_->st));
  CK3(cudaStreamSynchronize(p_->st));
}

void GpuSolver3::get_face_values(double* out) {
  CK3(cudaSetDevice(p_->device));
  const int NQ = p_->NQ;
  std::vector<double> dev(static_cast<size_t>(p_->nF) * NQ * 2 * V5);
  CK3(cudaMemcpyAsync(dev.data(), p_->W.fp, sizeof(double) * dev.size(), cudaMemcpyDeviceToHost, p_->st));
  CK3(cudaStreamSynchronize(p_->st));
  // device order [face][side][q] -> the view's slot order [face][q][side]
  for (int64_t f = 0; f < p_->nF; ++f)
    for (int q = 0; q < NQ; ++q)
      for (int side = 0; side < 2; ++side)
        for (int v = 0; v < V5; ++v)
          out[((f * NQ + q) * 2 + side) * V5 + v] = dev[((f * 2 + side) * NQ + q) * V5 + v];
}

void GpuSolver3::census(int64_t out[4]) {
  std::vector<uint8_t> l(p_->n);
  get_labels(1, l.data());
  for (int i = 0; i < 4; ++i) out[i] = 0;
  for (int c = 0; c < p_->n_owned; ++c) ++out[l[c] & 3];  // owned cells (the whole mesh on one domain)
}

void GpuSolver3::attach_nccl(const uint8_t id[128], int rank, int world) {
  Impl& I = *p_;
  CK3(cudaSetDevice(I.device));
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof u);
  if (I.comm) NK(nccl().CommDestroy(I.comm));
  I.comm = nullptr;
  NK(nccl().CommInitRank(&I.comm, world, u, rank));
  I.world = world, I.rank = rank;
  if (I.step_graph) cudaGraphExecDestroy(I.step_graph);
  I.step_graph = nullptr;
}

int64_t GpuSolver3::nad_ties() {
  unsigned long long t = 0;
  CK3(cudaSetDevice(p_->device));
  CK3(cudaMemcpyAsync(&t, p_->W.ties, sizeof t, cudaMemcpyDeviceToHost, p_->st));
  CK3(cudaStreamSynchronize(p_->st));
  return static_cast<int64_t>(t);
}

int64_t GpuSolver3::launches() const { return p_->launches; }
void* GpuSolver3::stream() const { return p_->st; }

}  // namespace ucfvb
