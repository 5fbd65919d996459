// TMA-staged (cp.async.bulk + mbarrier) persistent variants of the streaming
// kernels, used on the fast path (uniform face count, nominal stencil sizes).
//
// One 128-thread block processes one 32-cell chunk per iteration (four lanes
// per cell, lane v = variable v). Because the operator data is stored in
// 32-cell AoSoA chunks, every per-chunk array is ONE contiguous range in HBM
// (e.g. pinv: MM*K*32 doubles), so a single elected thread moves the whole
// chunk with a handful of bulk copies into a double-buffered shared-memory
// stage while the block computes the previous chunk. Per-thread registers are
// left for the stencil gathers of U (L2-served).
#pragma once

#include "kernels.cuh"
#include "tma.cuh"

namespace ucfvb {

__host__ __device__ constexpr uint32_t round16(uint32_t x) { return (x + 15u) & ~15u; }

// blocks per SM the shared-memory footprint allows (capped at 8): passed to
// __launch_bounds__ so that registers never become the tighter occupancy limit
__host__ __device__ constexpr int smem_min_blocks(uint32_t bytes) {
  const uint32_t per_block = bytes + 1024;  // + the per-block reservation
  const uint32_t b = (227u * 1024u) / per_block;
  return b < 1 ? 1 : (b > 8 ? 8 : static_cast<int>(b));
}

// cp.async prefetch of the stencil-member values one chunk ahead (p = 3). Off: without its
// 18 KB the p = 3 kernel fits three resident blocks instead of two, which measured central
// 3.39 -> 2.90 ms/stage on config 3 (three blocks WITH the prefetch and a slimmer group B:
// 3.53 ms; four blocks with only pinv and phi staged: 3.25 ms; profiles/round2.md)
#ifndef UCFVB_CENTRAL_PF
#define UCFVB_CENTRAL_PF 0
#endif
template <int K, int NQ, int NF, int MM>
struct CentralStage {
  static constexpr int Q = NF * NQ;
  // group A: consumed by the LSQ solve
  static constexpr uint32_t PINV = MM * K * 32 * 8;
  static constexpr uint32_t IDX = round16(MM * 32 * 4);
  static constexpr uint32_t A_BYTES = PINV + IDX;
  // group B: consumed by evaluation, NAD and the scatter
  static constexpr uint32_t PHI = Q * K * 32 * 8;
  static constexpr uint32_t THR = 32 * 8;
  static constexpr uint32_t NBR = round16(NF * 32 * 4);
  static constexpr uint32_t DEST = round16(Q * 32 * 4);
  static constexpr uint32_t B_BYTES = PHI + THR + NBR + DEST;
  // UCFVB_CENTRAL_PF (off): the U values of the chunk's central-stencil members
  // gathered with cp.async (8 B per lane and member) one chunk ahead, for the
  // larger stencils (p = 3: 18 members). At two resident blocks it hid the gather
  // latency (round 1: central -8 %); its 18 KB are what keeps the third block out.
  static constexpr bool PREFETCH = UCFVB_CENTRAL_PF && MM >= 16;
  static constexpr uint32_t UG = PREFETCH ? MM * 128 * 8 : 0;
  static constexpr uint32_t BYTES = A_BYTES + B_BYTES + UG;  // one stage
};

// k_central on the fast path: same arithmetic as k_central (kernels.cuh).
// One shared-memory stage split into two TMA groups with their own
// mbarriers: group A (pinv, stencil ids) is refilled with the next chunk as
// soon as the solve has consumed it, group B (phi, thresholds, neighbours,
// face-point slots) after the evaluation -- the copies of chunk i+1 overlap
// the second half of chunk i without doubling the footprint (NS = 2 keeps
// two such stages).
template <int K, int NQ, int NF, int MM, int NS>
__global__ void __launch_bounds__(kBlock, smem_min_blocks(NS * CentralStage<K, NQ, NF, MM>::BYTES + 16 * NS))
    k_central_tma(Layout L, Physics ph, Scratch S,
                                                        const double4* __restrict__ U, int flags) {
  using St = CentralStage<K, NQ, NF, MM>;
  constexpr int Q = St::Q;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + NS * St::BYTES);  // [2*NS]: A, B per stage
  const double* __restrict__ Ud = reinterpret_cast<const double*>(U);
  const int tid = threadIdx.x;
  const int slot = tid >> 2;  // cell within the chunk
  const int v = tid & 3;
  const int nchunks = (L.n + 31) >> 5;
  __shared__ int s_err;
  if (tid == 0) {
    for (int i = 0; i < 2 * NS; ++i) mbar_init(&bar[i], 1);
    mbar_fence_init();
  }
  auto issue_a = [&](int chunk, int st) {
    unsigned char* b = smem + st * St::BYTES;
    mbar_arrive_expect_tx(&bar[2 * st], St::A_BYTES);
    bulk_g2s(b, L.pinv + static_cast<size_t>(chunk) * MM * K * 32, St::PINV, &bar[2 * st]);
    bulk_g2s(b + St::PINV, L.st_idx + static_cast<size_t>(chunk) * MM * 32, St::IDX, &bar[2 * st]);
  };
  auto issue_b = [&](int chunk, int st) {
    unsigned char* b = smem + st * St::BYTES + St::A_BYTES;
    mbar_arrive_expect_tx(&bar[2 * st + 1], St::B_BYTES);
    bulk_g2s(b, L.phi + static_cast<size_t>(chunk) * Q * K * 32, St::PHI, &bar[2 * st + 1]);
    bulk_g2s(b + St::PHI, L.deact_thr + static_cast<size_t>(chunk) * 32, St::THR, &bar[2 * st + 1]);
    bulk_g2s(b + St::PHI + St::THR, L.nbr + static_cast<size_t>(chunk) * NF * 32, St::NBR, &bar[2 * st + 1]);
    bulk_g2s(b + St::PHI + St::THR + St::NBR, L.dest + static_cast<size_t>(chunk) * Q * 32, St::DEST,
             &bar[2 * st + 1]);
  };
  // the operator data is static: the first chunks' bulk copies are in flight
  // before the wait for the previous kernel (programmatic dependent launch)
  if (tid == 0)
    for (int p = 0; p < NS; ++p)
      if (static_cast<int>(blockIdx.x + p * gridDim.x) < nchunks) {
        issue_a(blockIdx.x + p * gridDim.x, p);
        issue_b(blockIdx.x + p * gridDim.x, p);
      }
  pdl_wait();
  if (tid == 0) {
    s_err = *(volatile int*)S.err;
    if (blockIdx.x == 0) {  // this stage's class-list counters and tie count
      for (int i = 0; i < 4; ++i) S.counts[i] = 0;
    }
  }
  __syncthreads();
  if (s_err) {  // block-uniform; drain the copies in flight before leaving
    for (int p = 0; p < NS; ++p)
      if (static_cast<int>(blockIdx.x + p * gridDim.x) < nchunks) {
        mbar_wait(&bar[2 * p], 0);
        mbar_wait(&bar[2 * p + 1], 0);
      }
    return;
  }
  // cp.async of this lane's stencil-member values of `chunk` (stage st, group A landed)
  auto gather_ahead = [&](int chunk, int st) {
    const unsigned char* b = smem + st * St::BYTES;
    const int* si = reinterpret_cast<const int*>(b + St::PINV);
    double* ug = reinterpret_cast<double*>(smem + st * St::BYTES + St::A_BYTES + St::B_BYTES);
#pragma unroll
    for (int m = 0; m < MM; ++m)
      cp_async8(ug + m * 128 + tid, Ud + 4 * static_cast<size_t>(si[m * 32 + slot]) + v);
    cp_async_commit();
  };
  if constexpr (St::PREFETCH) {
    if (static_cast<int>(blockIdx.x) < nchunks) {
      mbar_wait(&bar[0], 0);
      gather_ahead(blockIdx.x, 0);
    }
  }
  double* dofs = reinterpret_cast<double*>(S.dofs);
  double* fv = reinterpret_cast<double*>(S.fp);
  const bool detect = (flags & (FL_NAD | FL_PRECHECK)) != 0;
  int it = 0;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it) {
    const int st = it % NS;
    const uint32_t par = (it / NS) & 1;
    const int refill = chunk + NS * gridDim.x;  // the chunk this stage holds next
    const unsigned char* b = smem + st * St::BYTES;
    const double* sp = reinterpret_cast<const double*>(b);
    const int* si = reinterpret_cast<const int*>(b + St::PINV);
    const double* sf = reinterpret_cast<const double*>(b + St::A_BYTES);
    const double* sthr = reinterpret_cast<const double*>(b + St::A_BYTES + St::PHI);
    const int* sn = reinterpret_cast<const int*>(b + St::A_BYTES + St::PHI + St::THR);
    const int* sdst = reinterpret_cast<const int*>(b + St::A_BYTES + St::PHI + St::THR + St::NBR);

    const int c0 = chunk * 32 + slot;
    const bool live = c0 < L.n;
    const int c = live ? c0 : L.n - 1;
    const double u0 = __ldg(Ud + 4 * static_cast<size_t>(c) + v);
    mbar_wait(&bar[2 * st], par);
    // solve_dofs (reconstruct.cpp:9-28), m outermost, per-accumulator m order kept
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0.0;
    double um[MM];
    if constexpr (St::PREFETCH) {
      cp_async_wait_all();  // this lane's own prefetched member values
      const double* ug = reinterpret_cast<const double*>(b + St::A_BYTES + St::B_BYTES);
#pragma unroll
      for (int m = 0; m < MM; ++m) um[m] = ug[m * 128 + tid];
    } else {
#pragma unroll
      for (int m = 0; m < MM; ++m) um[m] = __ldg(Ud + 4 * static_cast<size_t>(si[m * 32 + slot]) + v);
    }
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      const double d = um[m] - u0;
#pragma unroll
      for (int k = 0; k < K; ++k) acc[k] += sp[(m * K + k) * 32 + slot] * d;
    }
    __syncthreads();  // group A of this stage consumed: refill it with the next chunk
    if (tid == 0 && refill < nchunks) {
      fence_proxy_async_smem();
      issue_a(refill, st);
    }
    // dofs feed the CWENOZ kernel; a raw MUSCL label survives the spread (it
    // only raises labels), so on detecting stages those cells' dofs are dead
    bool keep_dofs = (flags & FL_DOFS) && live;
    if (keep_dofs && !((flags & FL_NAD) && (flags & FL_EVAL))) {
#pragma unroll
      for (int k = 0; k < K; ++k) dofs[4 * aos(c, k, K) + v] = acc[k];
      keep_dofs = false;
    }
    mbar_wait(&bar[2 * st + 1], par);
    if (flags & FL_EVAL) {
      double lo = u0, hi = u0;
      if (detect) {
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int nb = sn[j * 32 + slot];
          if (nb >= 0) {
            const double x = __ldg(Ud + 4 * static_cast<size_t>(nb) + v);
            lo = smin(lo, x);
            hi = smax(hi, x);
          }
        }
      }
      const double du = hi - lo;
      double dm, dw;
      compute_margins(ph.mp, du, dm, dw);
      double vmax = -1e300, qmin = INFINITY, qmax = -INFINITY;
      bool bad = false;
      bool store = true;
      double vals[Q];
#pragma unroll
      for (int lq = 0; lq < Q; ++lq) {
        double val = u0;
#pragma unroll
        for (int k = 0; k < K; ++k) val += acc[k] * sf[(lq * K + k) * 32 + slot];
        vals[lq] = val;
        if (detect) {
          qmin = smin(qmin, val);
          qmax = smax(qmax, val);
        }
      }
      if (detect) {
        vmax = nad_violation(vmax, lo, hi, qmin, qmax);
        if (v == 0 || v == 3) bad |= vmax > dm;
        bad |= group_nonphysical<Q>(vals, Q, ph.gamma);
        int sev = 0;
        bool tie = false;
        if ((flags & FL_NAD) && (v == 0 || v == 3)) {
          const double thr = sthr[slot];
          if (!(du < thr)) {
            sev = violation_severity(vmax, dm, dw);
            const double sc = smax(smax(fabs(u0), du), 1e-300);
            tie = fabs(vmax - dm) <= 1e-12 * smax(sc, fabs(dm)) || fabs(vmax - dw) <= 1e-12 * smax(sc, fabs(dw));
          }
          if (thr > 0.0) tie |= fabs(du - thr) <= 1e-12 * thr;
        }
        sev = grp_max(sev);
        bad = grp_any(bad);
        tie = grp_any(tie);
        if (flags & FL_NAD) {
          const unsigned tm = __ballot_sync(kFull, tie && v == 0 && live);
          if (tm && (tid & 31) == __ffs(tm) - 1) atomicAdd(S.ties, static_cast<unsigned long long>(__popc(tm)));
        }
        if (v == 0 && live) S.raw[c] = static_cast<uint8_t>(sev | (bad ? 4 : 0));
#ifndef UCFVB_NO_DOFS_SKIP
        if (keep_dofs && (flags & FL_NAD) && sev == 2 && !(flags & FL_TAPS)) keep_dofs = false;
#endif
        // a raw label >= CWENOZ survives the spread (it only raises labels): the
        // troubled kernel rewrites this cell's face points, so the candidates are dead
        store = !((flags & FL_NAD) && sev >= 1);
      }
      if (live && store) {
#pragma unroll
        for (int lq = 0; lq < Q; ++lq) fv[4 * static_cast<size_t>(sdst[lq * 32 + slot]) + v] = vals[lq];
      }
    }
    if (keep_dofs) {
#pragma unroll
      for (int k = 0; k < K; ++k) dofs[4 * aos(c, k, K) + v] = acc[k];
    }
    __syncthreads();  // group B consumed
    if (tid == 0 && refill < nchunks) {
      fence_proxy_async_smem();
      issue_b(refill, st);
    }
    if constexpr (St::PREFETCH) {  // gather the next chunk's member values while the other warps finish this one
      const int nxt = chunk + static_cast<int>(gridDim.x);
      if (nxt < nchunks) {
        const int st2 = (it + 1) % NS;
        mbar_wait(&bar[2 * st2], ((it + 1) / NS) & 1);
        gather_ahead(nxt, st2);
      }
    }
  }
}

template <int K, int NQ, int NF, int MM, int MD>
struct TroubledStage {
  static constexpr int Q = NF * NQ;
  // CWENOZ chunk: member ids, directional pinv, OI, phi, neighbours, central dofs
  static constexpr uint32_t C_DIDX = round16(NF * MD * 32 * 4);
  static constexpr uint32_t C_PDIR = NF * MD * 2 * 32 * 8;
  static constexpr uint32_t C_OI = K * K * 32 * 8;
  static constexpr uint32_t C_PHI = Q * K * 32 * 8;
  static constexpr uint32_t C_NBR = round16(NF * 32 * 4);
  static constexpr uint32_t C_DOFS = K * 32 * 32;
  static constexpr uint32_t C_BYTES = C_DIDX + C_PDIR + C_OI + C_PHI + C_NBR + C_DOFS;
  // MUSCL chunk: central member ids, r=1 pinv, linear basis values, neighbours
  static constexpr uint32_t M_IDX = round16(MM * 32 * 4);
  static constexpr uint32_t M_PLIN = MM * 2 * 32 * 8;
  static constexpr uint32_t M_PHI = Q * 2 * 32 * 8;
  static constexpr uint32_t M_NBR = round16(NF * 32 * 4);
  static constexpr uint32_t M_BYTES = M_IDX + M_PLIN + M_PHI + M_NBR;
  static constexpr uint32_t BYTES = C_BYTES > M_BYTES ? C_BYTES : M_BYTES;
  // split-phase groups (k_troubled_split): A = what the directional / linear
  // solves read, B = what the blend, evaluation and fallback read
  static constexpr uint32_t DEST = round16(Q * 32 * 4);  // face-point destinations (the stores' addresses)
  static constexpr uint32_t CA = C_DIDX + C_PDIR + C_DOFS;
  static constexpr uint32_t CB = C_OI + C_PHI + C_NBR + DEST;
  static constexpr uint32_t MA = M_IDX + M_PLIN;
  static constexpr uint32_t MB = M_PHI + M_NBR + DEST;
  static constexpr uint32_t A_BYTES = CA > MA ? CA : MA;
  static constexpr uint32_t B_BYTES = CB > MB ? CB : MB;
  static constexpr uint32_t SPLIT_BYTES = A_BYTES + B_BYTES;
};

// k_troubled_split: the CWENOZ and MUSCL reconstructions of one stage in one
// persistent launch over the chunk lists built by k_spread (FL_CHUNKS): items
// [0, nC) are CWENOZ chunks, [nC, nC + nM) MUSCL chunks; the scheme is uniform
// per block iteration, lanes of cells outside the chunk's mask idle through
// the (shuffle-synchronous) math and store nothing. Split-phase refill (one
// stage, two mbarriers). Group A of the next work item is requested as soon as the
// directional (CWENOZ) or linear (MUSCL) solves of the current item have read
// it, so its copy overlaps the blend / limiter / evaluation / fallback; group
// B is requested once the evaluation and the fallback bounds are done.
// Arithmetic is identical to k_cwenoz / k_muscl (kernels.cuh).
template <int K, int NQ, int NF, int MM, int MD>
__global__ void __launch_bounds__(kBlock) k_troubled_split(Layout L, Physics ph, Scratch S,
                                                           const double4* __restrict__ U, int flags) {
  using St = TroubledStage<K, NQ, NF, MM, MD>;
  constexpr int Q = St::Q;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + St::SPLIT_BYTES);  // [0] group A, [1] group B
  unsigned char* const ga = smem;
  unsigned char* const gb = smem + St::A_BYTES;
  const double* __restrict__ Ud = reinterpret_cast<const double*>(U);
  const int tid = threadIdx.x;
  const int slot = tid >> 2;
  const int v = tid & 3;
  __shared__ int s_err, s_nc, s_nm;
  pdl_wait();
  if (tid == 0) {
    s_err = *(volatile int*)S.err;
    s_nc = S.counts[2];
    s_nm = S.counts[3];
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (s_err) return;
  const int nc = s_nc, nitems = s_nc + s_nm;
  if (nc > 0 && !(ph.lambda1p > 1.0)) {  // cwenoz_blend_scalar throws (reconstruct.cpp:102-103)
    if (blockIdx.x == 0 && tid == 0) atomicOr(&S.err[0], 4);
    return;
  }
  auto item_chunk = [&](int i) { return i < nc ? S.chunks_c[i] : S.chunks_m[i - nc]; };
  auto issue_a = [&](int i) {
    const size_t ch = static_cast<size_t>(item_chunk(i).x);
    unsigned char* p = ga;
    if (i < nc) {
      mbar_arrive_expect_tx(&bar[0], St::CA);
      bulk_g2s(p, L.dir_idx + ch * NF * MD * 32, St::C_DIDX, &bar[0]);
      p += St::C_DIDX;
      bulk_g2s(p, L.pinv_dir + ch * NF * MD * 2 * 32, St::C_PDIR, &bar[0]);
      p += St::C_PDIR;
      bulk_g2s(p, S.dofs + ch * K * 32, St::C_DOFS, &bar[0]);
    } else {
      mbar_arrive_expect_tx(&bar[0], St::MA);
      bulk_g2s(p, L.st_idx + ch * MM * 32, St::M_IDX, &bar[0]);
      p += St::M_IDX;
      bulk_g2s(p, L.pinv_lin + ch * MM * 2 * 32, St::M_PLIN, &bar[0]);
    }
  };
  auto issue_b = [&](int i) {
    const size_t ch = static_cast<size_t>(item_chunk(i).x);
    unsigned char* p = gb;
    if (i < nc) {
      mbar_arrive_expect_tx(&bar[1], St::CB);
      bulk_g2s(p, L.oi + ch * K * K * 32, St::C_OI, &bar[1]);
      p += St::C_OI;
      bulk_g2s(p, L.phi + ch * Q * K * 32, St::C_PHI, &bar[1]);
      p += St::C_PHI;
      bulk_g2s(p, L.nbr + ch * NF * 32, St::C_NBR, &bar[1]);
      p += St::C_NBR;
    } else {
      mbar_arrive_expect_tx(&bar[1], St::MB);
      bulk_g2s(p, L.phi01 + ch * Q * 2 * 32, St::M_PHI, &bar[1]);
      p += St::M_PHI;
      bulk_g2s(p, L.nbr + ch * NF * 32, St::M_NBR, &bar[1]);
      p += St::M_NBR;
    }
    bulk_g2s(p, L.dest + ch * Q * 32, St::DEST, &bar[1]);
  };
  if (tid == 0 && static_cast<int>(blockIdx.x) < nitems) {
    issue_a(blockIdx.x);
    issue_b(blockIdx.x);
  }
  double* dofs = reinterpret_cast<double*>(S.dofs);
  double* fv = reinterpret_cast<double*>(S.fp);
  const bool venkat = ph.limiter == 1;
  int it = 0;
  for (int i = blockIdx.x; i < nitems; i += gridDim.x, ++it) {
    const uint32_t par = it & 1;
    const int next = i + gridDim.x;
    const int2 e = item_chunk(i);
    const bool mine = (static_cast<unsigned>(e.y) >> slot) & 1u;
    const int c = e.x * 32 + slot;  // chunks are full-size in the padded layout; cells past n are never in a mask
    const int cc = c < L.n ? c : L.n - 1;
    const double u0 = __ldg(Ud + 4 * static_cast<size_t>(cc) + v);
    double vals[Q];
    double lo = u0, hi = u0;
    double kd[K];  // dofs to keep for the tap
    mbar_wait(&bar[0], par);
    if (i < nc) {
      // ---- CWENOZ (solver.cpp:167-188, reconstruct.cpp:43-150)
      const int* sdi = reinterpret_cast<const int*>(ga);
      const double* spd = reinterpret_cast<const double*>(ga + St::C_DIDX);
      const double* sdo = reinterpret_cast<const double*>(ga + St::C_DIDX + St::C_PDIR);
      double um[NF][MD];
#pragma unroll
      for (int s = 0; s < NF; ++s)
#pragma unroll
        for (int m = 0; m < MD; ++m) um[s][m] = __ldg(Ud + 4 * static_cast<size_t>(sdi[(s * MD + m) * 32 + slot]) + v);
      double dir[NF][2];
#pragma unroll
      for (int s = 0; s < NF; ++s) {
        dir[s][0] = 0.0;
        dir[s][1] = 0.0;
#pragma unroll
        for (int m = 0; m < MD; ++m) {
          const double d = um[s][m] - u0;
          dir[s][0] += spd[((s * MD + m) * 2 + 0) * 32 + slot] * d;
          dir[s][1] += spd[((s * MD + m) * 2 + 1) * 32 + slot] * d;
        }
      }
      double p1[K];
#pragma unroll
      for (int k = 0; k < K; ++k) p1[k] = sdo[(k * 32 + slot) * 4 + v];
      __syncthreads();  // group A consumed: request the next item's
      if (tid == 0 && next < nitems) {
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
        // one range test for the batch (exact_math.h), as k_troubled_cells
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
      mbar_wait(&bar[1], par);
      const double* soi = reinterpret_cast<const double*>(gb);
      const double* sph = reinterpret_cast<const double*>(gb + St::C_OI);
      const int* snb = reinterpret_cast<const int*>(gb + St::C_OI + St::C_PHI);
      double si0 = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < K; ++q) t += soi[(k * K + q) * 32 + slot] * p1[q];
        si0 += p1[k] * t;
      }
      const double o00 = soi[slot], o01 = soi[32 + slot], o10 = soi[K * 32 + slot], o11 = soi[(K + 1) * 32 + slot];
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
        for (int k = 0; k < K; ++k) vals[lq] += p1[k] * sph[(lq * K + k) * 32 + slot];
      }
#pragma unroll
      for (int k = 0; k < K; ++k) kd[k] = p1[k];
      if (flags & FL_FALLBACK) {
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int nb = snb[j * 32 + slot];
          if (nb >= 0) {
            const double x = __ldg(Ud + 4 * static_cast<size_t>(nb) + v);
            lo = smin(lo, x);
            hi = smax(hi, x);
          }
        }
      }
    } else {
      // ---- MUSCL (solver.cpp:189-221, reconstruct.cpp:30-86)
      const int* sid = reinterpret_cast<const int*>(ga);
      const double* spl = reinterpret_cast<const double*>(ga + St::M_IDX);
      double um[MM];
#pragma unroll
      for (int m = 0; m < MM; ++m) um[m] = __ldg(Ud + 4 * static_cast<size_t>(sid[m * 32 + slot]) + v);
      double l0 = 0.0, l1 = 0.0;
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        const double d = um[m] - u0;
        l0 += spl[(m * 2 + 0) * 32 + slot] * d;
        l1 += spl[(m * 2 + 1) * 32 + slot] * d;
      }
      __syncthreads();  // group A consumed: request the next item's
      if (tid == 0 && next < nitems) {
        fence_proxy_async_smem();
        issue_a(next);
      }
      mbar_wait(&bar[1], par);
      const double* sp01 = reinterpret_cast<const double*>(gb);
      const int* snb = reinterpret_cast<const int*>(gb + St::M_PHI);
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const int nb = snb[j * 32 + slot];
        if (nb >= 0) {
          const double x = __ldg(Ud + 4 * static_cast<size_t>(nb) + v);
          lo = smin(lo, x);
          hi = smax(hi, x);
        }
      }
      double theta = 1.0;
      const double eps2 = venkat ? L.eps2[cc] : 0.0;
#pragma unroll
      for (int lq = 0; lq < Q; ++lq) {
        const double p0 = sp01[(lq * 2 + 0) * 32 + slot], pq1 = sp01[(lq * 2 + 1) * 32 + slot];
        const double qv = u0 + l0 * p0 + l1 * pq1;
        theta = venkat ? venkat_update(theta, u0, lo, hi, qv, eps2) : bj_update(theta, u0, lo, hi, qv);
      }
      if (!venkat) theta = smax(theta, 0.0);
      const double d0 = theta * l0, d1 = theta * l1;
#pragma unroll
      for (int lq = 0; lq < Q; ++lq) {
        double o = u0;
        o += d0 * sp01[(lq * 2 + 0) * 32 + slot];
        o += d1 * sp01[(lq * 2 + 1) * 32 + slot];
        vals[lq] = o;  // dofs k >= 2 are zero: adding 0*phi leaves o unchanged
      }
#pragma unroll
      for (int k = 0; k < K; ++k) kd[k] = k == 0 ? d0 : (k == 1 ? d1 : 0.0);
    }
    int dst[Q];  // face-point destinations, staged with group B
    {
      const int* sdst = reinterpret_cast<const int*>(gb + (i < nc ? St::C_OI + St::C_PHI + St::C_NBR
                                                                  : St::M_PHI + St::M_NBR));
#pragma unroll
      for (int lq = 0; lq < Q; ++lq) dst[lq] = sdst[lq * 32 + slot];
    }
    __syncthreads();  // group B consumed: request the next item's
    if (tid == 0 && next < nitems) {
      fence_proxy_async_smem();
      issue_b(next);
    }
    bool demote = false;
    if (flags & FL_FALLBACK) demote = group_demote<Q>(ph, v, lo, hi, vals, Q);
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
