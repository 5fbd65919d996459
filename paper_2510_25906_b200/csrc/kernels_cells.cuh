// Per-cell troubled-cell reconstruction (fast path): CWENOZ and MUSCL over
// the dense per-class cell lists k_spread builds, with each listed cell's
// operator rows fetched as ONE contiguous record per group by cp.async.bulk.
//
// Why: on salt-and-pepper class maps (config 3: 60 % CWENOZ / 40 % MUSCL
// scattered over every 32-cell chunk) the chunk-list kernel stages a whole
// chunk of rows per list entry and runs every lane of it, so it moves ~1.8x
// the algorithmic bytes and does ~2x the lane work. Here a 32-cell tile of a
// class list is staged with 32 per-cell bulk copies (one per lane of warp 0),
// so the staged bytes are exactly the listed cells' rows.
//
// Records (built once on the device from the AoSoA arrays by k_pack_records;
// the arithmetic reads the same operator bytes in the same order):
//   CWENOZ  A:  pinv_dir [s][m][k<2] (f64), directional member ids [s][m], face neighbours [j] (i32)
//           B1: OI [k][q] (f64)
//           B2: phi [lq][k] (f64), face-point slots [lq] (i32)
//   MUSCL   A:  pinv_linear [m][k<2] (f64), central member ids [m], face neighbours [j] (i32)
//           B2: phi01 [lq][k<2] (f64), face-point slots [lq] (i32)
// Split-phase refill, one shared-memory slot per group and an mbarrier each:
// group A (directional / r=1 solves, fallback bounds) is refilled with the
// next tile as soon as the solves are done, group B = B1 | B2 (one copy) after
// the evaluation. (Refilling B1 on its own as soon as the smoothness
// indicators were done measured neutral and cost a third bulk copy per cell --
// a bulk copy with per-lane addresses is ~9 issued instructions, 12 % of this
// kernel's instructions with three copies per cell: profiles/round2.md.)
#pragma once

#include "kernels_tma.cuh"

namespace ucfvb {

// smallest 16-byte multiple >= x whose 16-byte count is odd: a shared-memory
// slot stride of 16*odd bytes puts the 8 cells one warp reads (4 lanes per
// cell) into 8 distinct bank pairs
__host__ __device__ constexpr uint32_t odd16(uint32_t x) { return ((x >> 4) & 1u) ? x : x + 16u; }

template <int K, int NQ, int NF, int MM, int MD, int TC = 32>
struct CellRec {
  static constexpr int Q = NF * NQ;
  static constexpr uint32_t CA_PD = 0, CA_ID = NF * MD * 2 * 8, CA_NBR = CA_ID + NF * MD * 4;
  static constexpr uint32_t CA = round16(CA_NBR + NF * 4);
  static constexpr uint32_t CB_OI = 0, CB1 = round16(K * K * 8);  // B1 = [0, CB1)
  static constexpr uint32_t CB_PHI = CB1, CB_DST = CB_PHI + Q * K * 8;
  static constexpr uint32_t CB = round16(CB_DST + Q * 4);         // B2 = [CB1, CB)
  static constexpr uint32_t MA_PL = 0, MA_ID = MM * 2 * 8, MA_NBR = MA_ID + MM * 4;
  static constexpr uint32_t MA = round16(MA_NBR + NF * 4);
  static constexpr uint32_t MB_PHI = 0, MB_DST = Q * 2 * 8;
  static constexpr uint32_t MB = round16(MB_DST + Q * 4);
  // in HBM a cell's CWENOZ groups A | B1 | B2 share one record, and so do its MUSCL
  // groups, each record a whole number of 64-byte lines (the L2's DRAM fetch
  // granularity): p = 3 CWENOZ 256 + 1120 -> 22 lines, MUSCL 384 + 128 = 8
  // lines exactly; unaligned separate records touched ~1.5 more lines per cell
  static constexpr uint32_t GC = (CA + CB + 63u) & ~63u, GM = (MA + MB + 63u) & ~63u;
  static constexpr uint32_t SCA = odd16(CA), SCB = odd16(CB), SMA = odd16(MA), SMB = odd16(MB);
  static constexpr uint32_t TILE_A = TC * (SCA > SMA ? SCA : SMA);  // TC cells per tile
  static constexpr uint32_t TILE_B = TC * (SCB > SMB ? SCB : SMB);
  static constexpr uint32_t BYTES = TILE_A + TILE_B;
};

// one thread per cell: AoSoA element e of cell c -> the cell's records
template <int K, int NQ, int NF, int MM, int MD>
__global__ void k_pack_records(Layout L, unsigned char* rc, unsigned char* rm) {
  using R = CellRec<K, NQ, NF, MM, MD>;
  constexpr int Q = R::Q;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L.n) return;
  {
    double* pd = reinterpret_cast<double*>(rc + static_cast<size_t>(c) * R::GC + R::CA_PD);
    int* id = reinterpret_cast<int*>(rc + static_cast<size_t>(c) * R::GC + R::CA_ID);
    for (int e = 0; e < NF * MD * 2; ++e) pd[e] = L.pinv_dir[aos(c, e, NF * MD * 2)];
    for (int e = 0; e < NF * MD; ++e) id[e] = L.dir_idx[aos(c, e, NF * MD)];
    for (int e = 0; e < NF; ++e) id[NF * MD + e] = L.nbr[aos(c, e, NF)];
  }
  {
    unsigned char* r = rc + static_cast<size_t>(c) * R::GC + R::CA;
    double* oi = reinterpret_cast<double*>(r + R::CB_OI);
    double* ph = reinterpret_cast<double*>(r + R::CB_PHI);
    int* ds = reinterpret_cast<int*>(r + R::CB_DST);
    for (int e = 0; e < K * K; ++e) oi[e] = L.oi[aos(c, e, K * K)];
    for (int e = 0; e < Q * K; ++e) ph[e] = L.phi[aos(c, e, Q * K)];
    for (int e = 0; e < Q; ++e) ds[e] = L.dest[aos(c, e, Q)];
  }
  {
    double* pl = reinterpret_cast<double*>(rm + static_cast<size_t>(c) * R::GM + R::MA_PL);
    int* id = reinterpret_cast<int*>(rm + static_cast<size_t>(c) * R::GM + R::MA_ID);
    for (int e = 0; e < MM * 2; ++e) pl[e] = L.pinv_lin[aos(c, e, MM * 2)];
    for (int e = 0; e < MM; ++e) id[e] = L.st_idx[aos(c, e, MM)];
    for (int e = 0; e < NF; ++e) id[MM + e] = L.nbr[aos(c, e, NF)];
  }
  {
    unsigned char* r = rm + static_cast<size_t>(c) * R::GM + R::MA;
    double* p01 = reinterpret_cast<double*>(r + R::MB_PHI);
    int* ds = reinterpret_cast<int*>(r + R::MB_DST);
    for (int e = 0; e < Q * 2; ++e) p01[e] = L.phi01[aos(c, e, Q * 2)];
    for (int e = 0; e < Q; ++e) ds[e] = L.dest[aos(c, e, Q)];
  }
}

// fallback_check's verdict for the cells of a single-warp tile (group_demote,
// kernels.cuh): the positivity check needs the four variables of a face point
// in one lane. Each lane writes its variable of the cell's Q points to a
// [point][variable] scratch row (the tile's dead group-B region), and lane v
// reads points v, v + 4, ... as two 16-byte loads -- ~15 instructions where the
// shuffle transpose (group_nonphysical) took ~90 (12 % of this kernel's).
// All 32 lanes of the warp call it; the scratch is free again on return.
__host__ __device__ constexpr uint32_t demote_stride(int Q) { return odd16(32u * Q); }  // bytes per cell
template <int Q>
__device__ __forceinline__ bool tile_demote(const Physics& ph, int v, int slot, double lo, double hi,
                                            const double* vals, unsigned char* scratch) {
  double dm, dw;
  compute_margins(ph.mp, hi - lo, dm, dw);
  double* sc = reinterpret_cast<double*>(scratch + slot * demote_stride(Q));
#pragma unroll
  for (int lq = 0; lq < Q; ++lq) sc[lq * 4 + v] = vals[lq];
  __syncwarp();
  bool bad = false;
#pragma unroll
  for (int r = 0; r < (Q + 3) / 4; ++r) {
    const int q = 4 * r + v;
    if (q < Q) {
      const double2 a = *reinterpret_cast<const double2*>(sc + q * 4);
      const double2 b = *reinterpret_cast<const double2*>(sc + q * 4 + 2);
      const double st[NV] = {a.x, a.y, b.x, b.y};
      bad |= !is_physical(st, ph.gamma);
    }
  }
  if (v == 0 || v == 3) {
#pragma unroll
    for (int lq = 0; lq < Q; ++lq) bad |= smax(lo - vals[lq], vals[lq] - hi) > dm;
  }
  bad = grp_any(bad);
  __syncwarp();
  return bad;
}

// Work items: tiles of 32 list entries, CWENOZ tiles [0, tc) then MUSCL tiles.
// Four lanes per cell (lane v = conserved variable v); arithmetic identical
// to k_troubled_split / k_cwenoz / k_muscl.
#ifndef UCFVB_CELLS_MINB
#define UCFVB_CELLS_MINB 16
#endif
#ifndef UCFVB_CELLS_PF
#define UCFVB_CELLS_PF 0
#endif
#ifndef UCFVB_CELLS_TILE
#define UCFVB_CELLS_TILE 8
#endif
#ifndef UCFVB_CELLS_CN
#define UCFVB_CELLS_CN 1
#endif

// cells per tile; a block is 4 * kCellTile threads
constexpr int kCellTile = UCFVB_CELLS_TILE;
// WHICH: 0 both classes in one launch, 1 the CWENOZ tiles only, 2 the MUSCL tiles only
// (UCFVB_CELLS_SPLIT: two launches; the MUSCL one needs ~half the registers and a third of
// the shared memory, so it runs at a higher occupancy)
#ifndef UCFVB_CELLS_SPLIT
#define UCFVB_CELLS_SPLIT 1
#endif
#ifndef UCFVB_CELLS_MINB_M
#define UCFVB_CELLS_MINB_M 24
#endif
template <int K, int NQ, int NF, int MM, int MD, int TC, int WHICH>
struct CellTile {
  using R = CellRec<K, NQ, NF, MM, MD, TC>;
  static constexpr uint32_t SB = R::SMB > demote_stride(NF * NQ) ? R::SMB : demote_stride(NF * NQ);
  static constexpr uint32_t TILE_A = WHICH == 2 ? TC * R::SMA : R::TILE_A;
  static constexpr uint32_t TILE_B = WHICH == 2 ? TC * SB : R::TILE_B;
  static constexpr uint32_t BYTES = TILE_A + TILE_B;
};
template <int K, int NQ, int NF, int MM, int MD, int WHICH = 0>
__global__ void __launch_bounds__(4 * kCellTile, WHICH == 2 ? UCFVB_CELLS_MINB_M : UCFVB_CELLS_MINB)
    k_troubled_cells(Layout L, Physics ph, Scratch S, const double4* __restrict__ U, int flags) {
  constexpr int TC = kCellTile;
  using R = CellRec<K, NQ, NF, MM, MD, TC>;
  using T = CellTile<K, NQ, NF, MM, MD, TC, WHICH>;
  constexpr int Q = R::Q;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + T::BYTES);  // [0] group A, [1] group B
  unsigned char* const ga = smem;
  unsigned char* const gb = smem + T::TILE_A;
  const double* __restrict__ Ud = reinterpret_cast<const double*>(U);
  const int tid = threadIdx.x;
  const int slot = tid >> 2;
  const int v = tid & 3;
  __shared__ int s_err, s_nc, s_nm;
  pdl_wait();
  if (tid == 0) {
    s_err = *(volatile int*)S.err;
    s_nc = S.counts[0];
    s_nm = S.counts[1];
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (s_err) return;
  const int nc = s_nc, nm = s_nm;
  const int tc = (nc + TC - 1) / TC;
  const int first = WHICH == 2 ? tc : 0;                               // this launch's items [first, nitems)
  const int nitems = WHICH == 1 ? tc : tc + (nm + TC - 1) / TC;
  if (WHICH != 2 && nc > 0 && !(ph.lambda1p > 1.0)) {  // cwenoz_blend_scalar throws (reconstruct.cpp:102-103)
    if (blockIdx.x == 0 && tid == 0) atomicOr(&S.err[0], 4);
    return;
  }
  // list entry j of tile i; lanes past the list's end repeat its last cell
  // (their records are staged and computed but never stored)
  auto tile_cell = [&](int i, int j) {
    return i < tc ? __ldg(S.list_c + min(i * TC + j, nc - 1)) : __ldg(S.list_m + min((i - tc) * TC + j, nm - 1));
  };
  // lanes j < TC of warp 0 only: lane j fetches slot j's record
  auto issue_a = [&](int i) {
    const int c = tile_cell(i, tid);
    if (tid == 0) mbar_arrive_expect_tx(&bar[0], TC * (i < tc ? R::CA : R::MA));
    __syncwarp(TC == 32 ? 0xffffffffu : (1u << TC) - 1u);
    if (i < tc)
      bulk_g2s(ga + tid * R::SCA, L.rec_ca + static_cast<size_t>(c) * R::GC, R::CA, &bar[0]);
    else
      bulk_g2s(ga + tid * R::SMA, L.rec_ma + static_cast<size_t>(c) * R::GM, R::MA, &bar[0]);
  };
  auto issue_b = [&](int i) {
    const int c = tile_cell(i, tid);
    if (tid == 0) mbar_arrive_expect_tx(&bar[1], TC * (i < tc ? R::CB : R::MB));
    __syncwarp(TC == 32 ? 0xffffffffu : (1u << TC) - 1u);
    if (i < tc)
      bulk_g2s(gb + tid * R::SCB, L.rec_cb + static_cast<size_t>(c) * R::GC, R::CB, &bar[1]);
    else
      bulk_g2s(gb + tid * R::SMB, L.rec_mb + static_cast<size_t>(c) * R::GM, R::MB, &bar[1]);
  };
  if (tid < TC && first + static_cast<int>(blockIdx.x) < nitems) {
    issue_a(first + blockIdx.x);
    issue_b(first + blockIdx.x);
  }
  double* dofs = reinterpret_cast<double*>(S.dofs);
  double* fv = reinterpret_cast<double*>(S.fp);
  const bool venkat = ph.limiter == 1;
  int it = 0;
  int c_next = (UCFVB_CELLS_CN && first + static_cast<int>(blockIdx.x) < nitems) ? tile_cell(first + blockIdx.x, slot) : 0;
  for (int i = first + blockIdx.x; i < nitems; i += gridDim.x, ++it) {
    const uint32_t par = it & 1;
    const int next = i + gridDim.x;
    const bool cw = WHICH == 1 ? true : (WHICH == 2 ? false : i < tc);
    const bool mine = cw ? i * TC + slot < nc : (i - tc) * TC + slot < nm;
    // the next tile's list entry is requested a tile ahead (UCFVB_CELLS_CN): its
    // L2 round trip leaves the head of that tile's dependency chain
    const int c = UCFVB_CELLS_CN ? c_next : tile_cell(i, slot);
    if (UCFVB_CELLS_CN && next < nitems) c_next = tile_cell(next, slot);
    const double u0 = __ldg(Ud + 4 * static_cast<size_t>(c) + v);
    double vals[Q];
    double lo = u0, hi = u0;
    double kd[K];  // dofs to keep for the tap
    int dst[Q];
    if (cw) {
      // ---- CWENOZ (solver.cpp:167-188, reconstruct.cpp:43-150)
      double p1[K];  // central dofs (k_central), issued before the record wait
#pragma unroll
      for (int k = 0; k < K; ++k) p1[k] = dofs[4 * aos(c, k, K) + v];
      mbar_wait(&bar[0], par);
      const unsigned char* ra = ga + slot * R::SCA;
      const double* spd = reinterpret_cast<const double*>(ra + R::CA_PD);
      const int* sdi = reinterpret_cast<const int*>(ra + R::CA_ID);
      const int* snb = reinterpret_cast<const int*>(ra + R::CA_NBR);
      int nbv[NF];
#pragma unroll
      for (int j = 0; j < NF; ++j) nbv[j] = snb[j];
      double um[NF][MD];
#pragma unroll
      for (int s = 0; s < NF; ++s)
#pragma unroll
        for (int m = 0; m < MD; ++m) um[s][m] = __ldg(Ud + 4 * static_cast<size_t>(sdi[s * MD + m]) + v);
      double dir[NF][2];
#pragma unroll
      for (int s = 0; s < NF; ++s) {
        dir[s][0] = 0.0;
        dir[s][1] = 0.0;
#pragma unroll
        for (int m = 0; m < MD; ++m) {
          const double d = um[s][m] - u0;
          dir[s][0] += spd[(s * MD + m) * 2 + 0] * d;
          dir[s][1] += spd[(s * MD + m) * 2 + 1] * d;
        }
      }
      __syncthreads();  // group A consumed: request the next tile's
      if (tid < TC && next < nitems) {
        fence_proxy_async_smem();
        issue_a(next);
      }
      // lam0 = 1 - 1/lambda1', lams = (1 - lam0)/(st - 1) (reconstruct.cpp:104-106), host-computed;
      // the divisions by lam0, st - 1 and wsum are div_rn (correctly rounded, as x / d)
      const double lam0 = ph.lam0;
      const double lams = ph.lams[NF];
      const bool rl = lam0 >= 0x1p-60;
#pragma unroll
      for (int s = 0; s < NF; ++s) {
        p1[0] -= lams * dir[s][0];
        p1[1] -= lams * dir[s][1];
      }
      {
        // one range test for the batch (exact_math.h): all numerators in range ->
        // the reciprocal form for all, else the IEEE division for all (same bits)
        bool okb = rl;
#pragma unroll
        for (int k = 0; k < K; ++k) okb = okb && div_rn_ok(p1[k]);
        if (okb) {
#pragma unroll
          for (int k = 0; k < K; ++k) p1[k] = div_rn_unchecked(p1[k], lam0, ph.inv_lam0);
        } else {
#pragma unroll
          for (int k = 0; k < K; ++k) p1[k] = p1[k] / lam0;
        }
      }
      double xn[NF];  // fallback bounds' neighbour values, in flight during the blend
#pragma unroll
      for (int j = 0; j < NF; ++j) xn[j] = nbv[j] >= 0 ? __ldg(Ud + 4 * static_cast<size_t>(nbv[j]) + v) : 0.0;
      mbar_wait(&bar[1], par);
      const unsigned char* rb = gb + slot * R::SCB;
      const double* soi = reinterpret_cast<const double*>(rb + R::CB_OI);
      const double* sph = reinterpret_cast<const double*>(rb + R::CB_PHI);
      const int* sdst = reinterpret_cast<const int*>(rb + R::CB_DST);
      double si0 = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < K; ++q) t += soi[k * K + q] * p1[q];
        si0 += p1[k] * t;
      }
      const double o00 = soi[0], o01 = soi[1], o10 = soi[K], o11 = soi[K + 1];
      double sis[NF];
      double tau = 0.0;
#pragma unroll
      for (int s = 0; s < NF; ++s) {
        const double a0 = dir[s][0], a1 = dir[s][1];
        sis[s] = o00 * a0 * a0 + (o01 + o10) * a0 * a1 + o11 * a1 * a1;
        tau += fabs(sis[s] - si0);
      }
      tau = div_rn(tau, ph.nd_d[NF], ph.inv_nd[NF]);
      tau = tau_pow(tau, ph.weno_b);
      double om0 = lam0 * (1.0 + tau / (ph.weno_eps + si0));
      double oms[NF];
      double wsum = om0;
#pragma unroll
      for (int s = 0; s < NF; ++s) {
        oms[s] = lams * (1.0 + tau / (ph.weno_eps + sis[s]));
        wsum += oms[s];
      }
      const double rw = 1.0 / wsum;  // wsum >= lam0 > 0
      const bool rwok = rl && wsum <= 0x1p60;
      {
        bool okb = rwok && div_rn_ok(om0);
#pragma unroll
        for (int s = 0; s < NF; ++s) okb = okb && div_rn_ok(oms[s]);
        if (okb) {
          om0 = div_rn_unchecked(om0, wsum, rw);
#pragma unroll
          for (int s = 0; s < NF; ++s) oms[s] = div_rn_unchecked(oms[s], wsum, rw);
        } else {
          om0 = om0 / wsum;
#pragma unroll
          for (int s = 0; s < NF; ++s) oms[s] = oms[s] / wsum;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) p1[k] = om0 * p1[k];
#pragma unroll
      for (int s = 0; s < NF; ++s) {
        const double w = oms[s];  // oms[s] / wsum
        p1[0] += w * dir[s][0];
        p1[1] += w * dir[s][1];
      }
#pragma unroll
      for (int lq = 0; lq < Q; ++lq) {
        vals[lq] = u0;
#pragma unroll
        for (int k = 0; k < K; ++k) vals[lq] += p1[k] * sph[lq * K + k];
      }
#pragma unroll
      for (int k = 0; k < K; ++k) kd[k] = p1[k];
      if (flags & FL_FALLBACK) {
#pragma unroll
        for (int j = 0; j < NF; ++j)
          if (nbv[j] >= 0) {
            lo = smin(lo, xn[j]);
            hi = smax(hi, xn[j]);
          }
      }
#pragma unroll
      for (int lq = 0; lq < Q; ++lq) dst[lq] = sdst[lq];
    } else {
      // ---- MUSCL (solver.cpp:189-221, reconstruct.cpp:30-86)
      mbar_wait(&bar[0], par);
      const unsigned char* ra = ga + slot * R::SMA;
      const double* spl = reinterpret_cast<const double*>(ra + R::MA_PL);
      const int* sid = reinterpret_cast<const int*>(ra + R::MA_ID);
      int nbm[NF];  // face neighbours (read before group A is refilled)
#pragma unroll
      for (int j = 0; j < NF; ++j) nbm[j] = reinterpret_cast<const int*>(ra + R::MA_NBR)[j];
      double um[MM];
#pragma unroll
      for (int m = 0; m < MM; ++m) um[m] = __ldg(Ud + 4 * static_cast<size_t>(sid[m]) + v);
      double l0 = 0.0, l1 = 0.0;
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        const double d = um[m] - u0;
        l0 += spl[m * 2 + 0] * d;
        l1 += spl[m * 2 + 1] * d;
      }
      __syncthreads();  // group A consumed: request the next tile's
      if (tid < TC && next < nitems) {
        fence_proxy_async_smem();
        issue_a(next);
      }
      mbar_wait(&bar[1], par);
      const unsigned char* rb = gb + slot * R::SMB;
      const double* sp01 = reinterpret_cast<const double*>(rb + R::MB_PHI);
      const int* sdst = reinterpret_cast<const int*>(rb + R::MB_DST);
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int nb = nbm[j];
        if (nb >= 0) {
          const double x = __ldg(Ud + 4 * static_cast<size_t>(nb) + v);
          lo = smin(lo, x);
          hi = smax(hi, x);
        }
      }
      double theta = 1.0;
      const double eps2 = venkat ? L.eps2[c] : 0.0;
#pragma unroll
      for (int lq = 0; lq < Q; ++lq) {
        const double p0 = sp01[lq * 2 + 0], pq1 = sp01[lq * 2 + 1];
        const double qv = u0 + l0 * p0 + l1 * pq1;
        theta = venkat ? venkat_update(theta, u0, lo, hi, qv, eps2) : bj_update(theta, u0, lo, hi, qv);
      }
      if (!venkat) theta = smax(theta, 0.0);
      const double d0 = theta * l0, d1 = theta * l1;
#pragma unroll
      for (int lq = 0; lq < Q; ++lq) {
        double o = u0;
        o += d0 * sp01[lq * 2 + 0];
        o += d1 * sp01[lq * 2 + 1];
        vals[lq] = o;  // dofs k >= 2 are zero: adding 0*phi leaves o unchanged
      }
#pragma unroll
      for (int k = 0; k < K; ++k) kd[k] = k == 0 ? d0 : (k == 1 ? d1 : 0.0);
#pragma unroll
      for (int lq = 0; lq < Q; ++lq) dst[lq] = sdst[lq];
    }
    __syncthreads();  // group B consumed (its face-point slots are in registers)
    // fallback verdict first: the positivity check transposes the tile's face
    // values through the dead group-B region (tile_demote), then the refill
    bool demote = false;
    constexpr bool kScratchFits = TC * demote_stride(Q) <= T::TILE_B;  // (not for p = 1 quadrilaterals)
    if (flags & FL_FALLBACK)
      demote = kScratchFits ? tile_demote<Q>(ph, v, slot, lo, hi, vals, gb) : group_demote<Q>(ph, v, lo, hi, vals, Q);
    if (4 * TC > 32) __syncthreads();  // multi-warp tiles: every warp's scratch reads precede the refill
    if (tid < TC && next < nitems) {
      fence_proxy_async_smem();
      issue_b(next);
    }
    if (UCFVB_CELLS_PF && next < nitems && v == 0) {
      // the next tile's member rows of U into L2 while this tile finishes
      mbar_wait(&bar[0], par ^ 1u);
      if (next < tc) {
        const int* nid = reinterpret_cast<const int*>(ga + slot * R::SCA + R::CA_ID);
#pragma unroll
        for (int m = 0; m < NF * MD; ++m) prefetch_l2(U + nid[m]);
      } else {
        const int* nid = reinterpret_cast<const int*>(ga + slot * R::SMA + R::MA_ID);
#pragma unroll
        for (int m = 0; m < MM; ++m) prefetch_l2(U + nid[m]);
      }
    }
    if (mine) {
#pragma unroll
      for (int lq = 0; lq < Q; ++lq) fv[4 * static_cast<size_t>(dst[lq]) + v] = demote ? u0 : vals[lq];
      if (demote && v == 0) S.labels[c] = 3;
      if (flags & FL_TAPS) {
#pragma unroll
        for (int k = 0; k < K; ++k) dofs[4 * aos(c, k, K) + v] = demote ? 0.0 : kd[k];
      }
    }
  }
}

}  // namespace ucfvb
