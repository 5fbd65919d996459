// Flat reference views -> device layout (see kernels.cuh for the consumers).
#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <thread>

#include "layout.hpp"

namespace ucfvb {

void parallel_for(int64_t n, int n_threads, const std::function<void(int64_t, int64_t)>& body) {
  if (n_threads <= 0) n_threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  if (n < 4096 || n_threads == 1) {
    body(0, n);
    return;
  }
  const int T = static_cast<int>(std::min<int64_t>(n_threads, (n + 1023) / 1024));
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> errs(T);
  for (int t = 0; t < T; ++t) {
    const int64_t a = n * t / T, b = n * (t + 1) / T;
    th.emplace_back([&, a, b, t] {
      try {
        body(a, b);
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  }
  for (auto& x : th) x.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

namespace {

int local_face_index(const ucfvb_mesh_view& m, int cell, int fid) {
  for (int i = m.cell_face_ptr[cell]; i < m.cell_face_ptr[cell + 1]; ++i)
    if (m.cell_faces[i] == fid) return i - m.cell_face_ptr[cell];
  throw ApiError(UCFVB_INVALID, "mesh: face " + std::to_string(fid) + " not listed by cell " + std::to_string(cell));
}

}  // namespace

HostLayout build_layout(const ucfvb_mesh_view& m, const ucfvb_stencil_view& s, const ucfvb_options& o,
                        int n_threads, int n_owned, int halo_patch) {
  HostLayout L;
  const int n = m.n_cells;
  if (n <= 0) throw ApiError(UCFVB_INVALID, "solver: empty mesh");
  if (s.n_cells != n) throw ApiError(UCFVB_INVALID, "solver: stencil set does not match the mesh");
  // solver.cpp:39-44
  if (m.n_faces > 0 && m.n_qp != s.n_qp)
    throw ApiError(UCFVB_INVALID, "solver: mesh was built with " + std::to_string(m.n_qp) +
                                      " face quadrature points but order " + std::to_string(o.order) + " needs " +
                                      std::to_string(s.n_qp));
  L.n = n;
  L.n_owned = n_owned;
  if (n_owned < 1 || n_owned > n) throw ApiError(UCFVB_INVALID, "solver: owned cell count out of range");
  L.n_pad = (n + 31) / 32 * 32;
  L.K = s.K;
  L.NQ = s.n_qp;
  L.n_faces = m.n_faces;
  int nfmax = 0;
  for (int c = 0; c < n; ++c) nfmax = std::max(nfmax, m.cell_face_ptr[c + 1] - m.cell_face_ptr[c]);
  if (nfmax > 4) throw ApiError(UCFVB_UNSUPPORTED, "solver: cells with more than 4 faces are not supported on the device");
  L.NF = nfmax <= 3 ? 3 : 4;
  L.Q = L.NF * L.NQ;
  if (L.NQ > 4) throw ApiError(UCFVB_UNSUPPORTED, "solver: more than 4 face quadrature points");
  int mm = 0, md = 0;
  for (int c = 0; c < n; ++c) mm = std::max<int>(mm, static_cast<int>(s.central_ptr[c + 1] - s.central_ptr[c]) - 1);
  for (int d = 0; d < s.n_dir_stencils; ++d)
    md = std::max<int>(md, static_cast<int>(s.dir_member_ptr[d + 1] - s.dir_member_ptr[d]) - 1);
  L.MM = mm;
  L.MD = md;
  // quadrature weights are identical on every face (segment_quadrature, quadrature.cpp:93-104)
  for (int q = 0; q < L.NQ; ++q) L.qw[q] = m.n_faces ? m.face_qw[q] : 0.0;
  for (int f = 0; f < m.n_faces; ++f)
    for (int q = 0; q < L.NQ; ++q)
      if (m.face_qw[f * L.NQ + q] != L.qw[q])
        throw ApiError(UCFVB_UNSUPPORTED, "solver: face quadrature weights differ between faces");

  const int K = L.K, NQ = L.NQ, NF = L.NF, Q = L.Q, MM = L.MM, MD = L.MD;
  const size_t nch = static_cast<size_t>(L.n_pad / 32);
  L.st_idx.assign(nch * MM * 32, 0);
  L.pinv.assign(nch * MM * K * 32, 0.0);
  L.phi.assign(nch * Q * K * 32, 0.0);
  L.phi01.assign(nch * Q * 2 * 32, 0.0);
  L.pinv_lin.assign(nch * MM * 2 * 32, 0.0);
  L.dir_idx.assign(nch * NF * MD * 32, 0);
  L.pinv_dir.assign(nch * NF * MD * 2 * 32, 0.0);
  L.oi.assign(nch * K * K * 32, 0.0);
  L.nbr.assign(nch * NF * 32, -1);
  // pad slots of cells with fewer faces point at a scratch slot past the faces
  L.dest.assign(nch * Q * 32, static_cast<int32_t>(2 * static_cast<int64_t>(m.n_faces) * NQ));
  L.cface.assign(nch * NF * 32, 0);
  L.fnx.assign(m.n_faces, 0.0);
  L.fny.assign(m.n_faces, 0.0);
  L.flen.assign(m.n_faces, 0.0);
  L.fkind.assign(m.n_faces, 0);
  L.fslot.assign(2 * static_cast<size_t>(m.n_faces), -1);
  L.fpatch.assign(m.n_faces, 0);
  for (int f = 0; f < m.n_faces; ++f) {
    L.fnx[f] = m.face_normal[2 * f];
    L.fny[f] = m.face_normal[2 * f + 1];
    L.flen[f] = m.face_length[f];
    const int partner = m.face_partner[f];
    if (m.face_right[f] >= 0) {
      L.fkind[f] = 0;
    } else if (partner >= 0) {
      L.fkind[f] = partner > f ? 0 : 2;  // the primary of a periodic pair carries the flux (solver.cpp:272)
    } else if (m.face_patch[f] == halo_patch && halo_patch >= 0) {
      L.fkind[f] = 2;  // leaves a subdomain's local set: never integrated
    } else {
      const int patch = m.face_patch[f];
      if (patch < 0 || patch >= 16)
        throw ApiError(UCFVB_INVALID, "solver: boundary face " + std::to_string(f) + " has no boundary condition");
      L.fkind[f] = 1;
      L.fpatch[f] = static_cast<int8_t>(patch);
    }
    // on a subdomain only faces touching an owned cell are integrated
    const bool touches_owned = m.face_left[f] < n_owned || (m.face_right[f] >= 0 && m.face_right[f] < n_owned) ||
                               (partner >= 0 && m.face_left[partner] < n_owned);
    if (!touches_owned) L.fkind[f] = 2;
  }
  L.nfc.assign(L.n_pad, 0);
  L.deact_thr.assign(L.n_pad, 0.0);
  L.eps2.assign(L.n_pad, 0.0);
  L.h.assign(L.n_pad, 1.0);
  L.inv_vol.assign(L.n_pad, 0.0);
  L.qp_ptr.assign(s.qp_ptr, s.qp_ptr + n + 1);
  L.qp_slot.assign(s.qp_slot, s.qp_slot + s.qp_ptr[n]);

  // face-point slot of (face, q, side) in the face-major fp array (double4 units)
  auto fp_slot = [&](int f, int q, int side) -> int64_t { return (static_cast<int64_t>(f) * NQ + q) * 2 + side; };
  if (2 * static_cast<int64_t>(m.n_faces) * NQ + 1 >= (int64_t{1} << 31))
    throw ApiError(UCFVB_UNSUPPORTED, "solver: mesh too large for 32-bit face-point indices");

  parallel_for(n, n_threads, [&](int64_t a, int64_t b) {
    for (int c = static_cast<int>(a); c < static_cast<int>(b); ++c) {
      const int nf = m.cell_face_ptr[c + 1] - m.cell_face_ptr[c];
      L.nfc[c] = static_cast<uint8_t>(nf);
      const double hc = m.cell_h[c];
      L.h[c] = hc;
      L.inv_vol[c] = 1.0 / m.cell_area[c];
      // deactivate_smooth threshold (detector.cpp:32-35) and Venkatakrishnan eps2
      // (solver.cpp:203) with the host's std::pow, exactly as the reference
      L.deact_thr[c] = (o.margins.kappa <= 0.0) ? -std::numeric_limits<double>::infinity()
                                                : std::pow(o.margins.kappa * hc, o.margins.deact_n);
      L.eps2[c] = std::pow(o.venkat_kappa * hc, 3);
      // central stencil
      const int64_t c0 = s.central_ptr[c];
      const int M = static_cast<int>(s.central_ptr[c + 1] - c0) - 1;
      if (s.central[3 * c0] != c) throw ApiError(UCFVB_INVALID, "stencil: central stencil must start with the cell");
      if (s.pinv_off[c + 1] - s.pinv_off[c] != static_cast<int64_t>(K) * M ||
          s.pinv_lin_off[c + 1] - s.pinv_lin_off[c] != 2LL * M)
        throw ApiError(UCFVB_INVALID, "stencil: pseudo-inverse sizes do not match the stencil");
      const double* pv = s.pinv + s.pinv_off[c];
      const double* pl = s.pinv_lin + s.pinv_lin_off[c];
      for (int mi = 0; mi < MM; ++mi) {
        const bool real = mi < M;
        L.st_idx[aos_index(c, mi, MM)] = real ? s.central[3 * (c0 + 1 + mi)] : c;
        for (int k = 0; k < K; ++k) L.pinv[aos_index(c, mi * K + k, MM * K)] = real ? pv[k * M + mi] : 0.0;
        for (int k = 0; k < 2; ++k) L.pinv_lin[aos_index(c, mi * 2 + k, MM * 2)] = real ? pl[k * M + mi] : 0.0;
      }
      // phi tables
      const int64_t q0 = s.qp_ptr[c];
      const int qc = static_cast<int>(s.qp_ptr[c + 1] - q0);
      if (qc != nf * NQ || s.phi_off[c + 1] - s.phi_off[c] != static_cast<int64_t>(qc) * K)
        throw ApiError(UCFVB_INVALID, "stencil: phi table does not match the cell's faces");
      const double* ph = s.phi + s.phi_off[c];
      for (int lq = 0; lq < qc; ++lq) {
        for (int k = 0; k < K; ++k) L.phi[aos_index(c, lq * K + k, Q * K)] = ph[lq * K + k];
        for (int k = 0; k < 2; ++k) L.phi01[aos_index(c, lq * 2 + k, Q * 2)] = ph[lq * K + k];
      }
      // directional stencils
      const int64_t d0 = s.dir_ptr[c];
      const int nd = static_cast<int>(s.dir_ptr[c + 1] - d0);
      if (nd != nf) throw ApiError(UCFVB_UNSUPPORTED, "stencil: expected one directional stencil per face");
      for (int sd = 0; sd < nd; ++sd) {
        const int64_t g = d0 + sd;
        const int64_t mb = s.dir_member_ptr[g];
        const int Md = static_cast<int>(s.dir_member_ptr[g + 1] - mb) - 1;
        if (s.pinv_dir_off[g + 1] - s.pinv_dir_off[g] != 2LL * Md)
          throw ApiError(UCFVB_INVALID, "stencil: directional pseudo-inverse size mismatch");
        const double* pd = s.pinv_dir + s.pinv_dir_off[g];
        for (int mi = 0; mi < MD; ++mi) {
          const bool real = mi < Md;
          const int cell = real ? s.central[3 * (c0 + s.dir_members[mb + 1 + mi])] : c;
          L.dir_idx[aos_index(c, sd * MD + mi, NF * MD)] = cell;
          for (int k = 0; k < 2; ++k)
            L.pinv_dir[aos_index(c, (sd * MD + mi) * 2 + k, NF * MD * 2)] = real ? pd[k * Md + mi] : 0.0;
        }
      }
      for (int e = 0; e < K * K; ++e) L.oi[aos_index(c, e, K * K)] = s.oi[static_cast<int64_t>(c) * K * K + e];
      // faces: neighbours (face_neighbors mesh.cpp:19-30), where each face-point
      // value goes (val_left_/val_right_ slot; a periodic secondary writes the
      // primary's right slot, which is what solver.cpp:280-281 reads) and the
      // signed canonical face of the owner-ordered gather (solver.cpp:298-307)
      for (int j = 0; j < nf; ++j) {
        const int f = m.cell_faces[m.cell_face_ptr[c] + j];
        const int right = m.face_right[f], left = m.face_left[f], partner = m.face_partner[f];
        int nb = -1;
        if (right >= 0)
          nb = (left == c) ? right : left;
        else if (partner >= 0)
          nb = m.face_left[partner];
        L.nbr[aos_index(c, j, NF)] = nb;
        int canon = f, neg = 0;
        for (int q = 0; q < NQ; ++q) {
          int64_t slot;
          if (right >= 0) {
            slot = fp_slot(f, q, left == c ? 0 : 1);
            neg = left == c ? 0 : 1;
          } else if (partner >= 0 && partner < f) {  // periodic secondary
            canon = partner;
            neg = 1;
            slot = fp_slot(partner, m.face_partner_qp[f * NQ + q], 1);
          } else {  // periodic primary or boundary: this cell is the left side
            slot = fp_slot(f, q, 0);
          }
          L.dest[aos_index(c, j * NQ + q, Q)] = static_cast<int32_t>(slot);
        }
        L.cface[aos_index(c, j, NF)] = (canon << 1) | neg;
        // the canonical face's flux lands in this cell's slot j with the gather's sign
        L.fslot[2 * static_cast<size_t>(canon) + neg] = static_cast<int32_t>(aos_index(c, j, NF));
      }
    }
  });
  return L;
}

}  // namespace ucfvb
