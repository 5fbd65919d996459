// Domain decomposition for the multi-GPU stage pass: recursive
// coordinate bisection of the cell centroids, and per-rank subdomains with the
// stencil-depth halo every owned residual depends on.
//
// Dependency radius: an owned cell's residual needs the final
// face values of its face neighbours (layer 1); their labels need the raw NAD
// labels of layer 2 (one spread pass, detector.cpp:37-53); a raw label needs
// the central-stencil candidate values and face-neighbour bounds of its cell.
// So the classification set is layers 0-2 and the local cell set is the
// classification set plus the central stencils and face neighbours of its
// cells. Cells outside the classification set only provide U: they get inert
// stencils (self members, zero weights) so every kernel can run over all local
// cells without branching; nothing they produce reaches an owned residual.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "decompose.hpp"
#include "layout.hpp"
#include "ucfvb.h"

namespace ucfvb {
namespace {

void face_neighbors(const ucfvb_mesh_view& m, int c, std::vector<int>& out) {
  out.clear();
  for (int i = m.cell_face_ptr[c]; i < m.cell_face_ptr[c + 1]; ++i) {
    const int f = m.cell_faces[i];
    if (m.face_right[f] >= 0)
      out.push_back(m.face_left[f] == c ? m.face_right[f] : m.face_left[f]);
    else if (m.face_partner[f] >= 0)
      out.push_back(m.face_left[m.face_partner[f]]);
  }
}

void rcb(const ucfvb_mesh_view& m, std::vector<int>& cells, int first_part, int n_parts, int32_t* part) {
  if (n_parts == 1) {
    for (int c : cells) part[c] = first_part;
    return;
  }
  double lo[2] = {1e300, 1e300}, hi[2] = {-1e300, -1e300};
  for (int c : cells)
    for (int d = 0; d < 2; ++d) {
      lo[d] = std::min(lo[d], m.cell_centroid[2 * c + d]);
      hi[d] = std::max(hi[d], m.cell_centroid[2 * c + d]);
    }
  const int axis = (hi[0] - lo[0]) >= (hi[1] - lo[1]) ? 0 : 1;
  const int pa = n_parts / 2, pb = n_parts - pa;
  const size_t na = cells.size() * pa / n_parts;
  // deterministic split: order by (coordinate, cell id)
  std::nth_element(cells.begin(), cells.begin() + na, cells.end(), [&](int a, int b) {
    const double xa = m.cell_centroid[2 * a + axis], xb = m.cell_centroid[2 * b + axis];
    return xa != xb ? xa < xb : a < b;
  });
  std::vector<int> A(cells.begin(), cells.begin() + na), B(cells.begin() + na, cells.end());
  std::vector<int>().swap(cells);
  rcb(m, A, first_part, pa, part);
  rcb(m, B, first_part + pa, pb, part);
}

// owned cells, classification set (layers 0..2) and local (U) set of rank r
struct Sets {
  std::vector<int> owned, classify, local;
};

Sets rank_sets(const ucfvb_mesh_view& m, const ucfvb_stencil_view& s, const int32_t* part, int r) {
  const int n = m.n_cells;
  Sets S;
  std::vector<int8_t> level(n, -1);
  for (int c = 0; c < n; ++c)
    if (part[c] == r) {
      S.owned.push_back(c);
      level[c] = 0;
    }
  std::vector<int> frontier = S.owned, next, nb;
  S.classify = S.owned;
  for (int l = 1; l <= 2; ++l) {
    next.clear();
    for (int c : frontier) {
      face_neighbors(m, c, nb);
      for (int x : nb)
        if (level[x] < 0) {
          level[x] = static_cast<int8_t>(l);
          next.push_back(x);
        }
    }
    S.classify.insert(S.classify.end(), next.begin(), next.end());
    frontier.swap(next);
  }
  std::vector<int8_t> in_local(n, 0);
  for (int c : S.classify) in_local[c] = 1;
  S.local = S.classify;
  for (int c : S.classify) {
    for (int64_t j = s.central_ptr[c]; j < s.central_ptr[c + 1]; ++j) {
      const int x = s.central[3 * j];
      if (!in_local[x]) {
        in_local[x] = 1;
        S.local.push_back(x);
      }
    }
    face_neighbors(m, c, nb);
    for (int x : nb)
      if (!in_local[x]) {
        in_local[x] = 1;
        S.local.push_back(x);
      }
  }
  return S;
}

}  // namespace

void partition_rcb(const ucfvb_mesh_view& m, int n_parts, int32_t* part) {
  if (n_parts < 1) throw ApiError(UCFVB_INVALID, "partition: n_parts must be >= 1");
  std::vector<int> cells(m.n_cells);
  std::iota(cells.begin(), cells.end(), 0);
  rcb(m, cells, 0, n_parts, part);
}

ucfvb_subdomain* build_subdomain(const ucfvb_mesh_view& m, const ucfvb_stencil_view& s, const int32_t* part,
                                 int n_parts, int r) {
  if (r < 0 || r >= n_parts) throw ApiError(UCFVB_INVALID, "subdomain: rank out of range");
  if (s.n_cells != m.n_cells) throw ApiError(UCFVB_INVALID, "subdomain: stencil set does not match the mesh");
  const int n = m.n_cells, nq = m.n_qp, K = s.K;
  auto* D = new ucfvb_subdomain;
  try {
    D->rank = r;
    D->n_parts = n_parts;
    Sets S = rank_sets(m, s, part, r);
    std::vector<int8_t> is_classify(n, 0);
    for (int c : S.classify) is_classify[c] = 1;
    // the owned cells some peer holds in its local set (they are sent every stage)
    std::vector<std::vector<int>> send_g(n_parts);
    std::vector<int8_t> sent(n, 0);
    for (int q = 0; q < n_parts; ++q) {
      if (q == r) continue;
      Sets Sq = rank_sets(m, s, part, q);
      for (int c : Sq.local)
        if (part[c] == r) {
          send_g[q].push_back(c);
          sent[c] = 1;
        }
      std::sort(send_g[q].begin(), send_g[q].end());
    }
    // local order: owned interior (global order) | owned sent cells (global
    // order) | halo by (owner, global id). The solver updates the sent cells
    // first each stage, so the halo exchange overlaps the interior's update.
    std::vector<int> owned, owned_sent, halo;
    for (int c : S.owned) (sent[c] ? owned_sent : owned).push_back(c);
    std::sort(owned.begin(), owned.end());
    std::sort(owned_sent.begin(), owned_sent.end());
    D->n_interior = static_cast<int>(owned.size());
    owned.insert(owned.end(), owned_sent.begin(), owned_sent.end());
    {
      std::vector<int8_t> own(n, 0);
      for (int c : owned) own[c] = 1;
      for (int c : S.local)
        if (!own[c]) halo.push_back(c);
    }
    std::sort(halo.begin(), halo.end(), [&](int a, int b) { return part[a] != part[b] ? part[a] < part[b] : a < b; });
    D->n_owned = static_cast<int>(owned.size());
    D->gid = owned;
    D->gid.insert(D->gid.end(), halo.begin(), halo.end());
    D->n_local = static_cast<int>(D->gid.size());
    const int nl = D->n_local;
    std::vector<int32_t> lid(n, -1);
    for (int l = 0; l < nl; ++l) lid[D->gid[l]] = l;
    D->part_of_local.resize(nl);
    for (int l = 0; l < nl; ++l) D->part_of_local[l] = part[D->gid[l]];

    // ---- local faces (global order) and mesh arrays
    std::vector<int32_t> lface(m.n_faces, -1);
    std::vector<int> faces;
    for (int g : D->gid)
      for (int i = m.cell_face_ptr[g]; i < m.cell_face_ptr[g + 1]; ++i) faces.push_back(m.cell_faces[i]);
    std::sort(faces.begin(), faces.end());
    faces.erase(std::unique(faces.begin(), faces.end()), faces.end());
    for (size_t i = 0; i < faces.size(); ++i) lface[faces[i]] = static_cast<int32_t>(i);
    D->patch_names.clear();
    for (int p = 0; p < m.n_patches; ++p) D->patch_names.push_back(m.patch_names[p]);
    const int halo_patch = m.n_patches;
    D->patch_names.push_back("__halo__");
    D->cvp = {0};
    D->cfp = {0};
    for (int l = 0; l < nl; ++l) {
      const int g = D->gid[l];
      for (int i = m.cell_vtx_ptr[g]; i < m.cell_vtx_ptr[g + 1]; ++i) D->cv.push_back(m.cell_vtx[i]);
      D->cvp.push_back(static_cast<int32_t>(D->cv.size()));
      for (int i = m.cell_face_ptr[g]; i < m.cell_face_ptr[g + 1]; ++i) D->cf.push_back(lface[m.cell_faces[i]]);
      D->cfp.push_back(static_cast<int32_t>(D->cf.size()));
      D->centroid.push_back(m.cell_centroid[2 * g]);
      D->centroid.push_back(m.cell_centroid[2 * g + 1]);
      D->area.push_back(m.cell_area[g]);
      D->h.push_back(m.cell_h[g]);
    }
    for (int f : faces) {
      const int gl = m.face_left[f], gr = m.face_right[f], gp = m.face_partner[f];
      int L = lid[gl], R = gr >= 0 ? lid[gr] : -1, P = -1, patch = m.face_patch[f];
      bool ghost = false;
      if (gr >= 0) {
        if (L < 0 || R < 0) {  // interior face leaving the local set
          ghost = true;
          L = L >= 0 ? L : R;
          R = -1;
        }
      } else if (gp >= 0) {
        if (lid[m.face_left[gp]] >= 0 && lface[gp] >= 0)
          P = lface[gp];
        else
          ghost = true;
      }
      if (ghost) patch = halo_patch;
      D->fvtx.push_back(m.face_vtx[2 * f]);
      D->fvtx.push_back(m.face_vtx[2 * f + 1]);
      D->fl.push_back(L);
      D->fr.push_back(R);
      D->normal.push_back(m.face_normal[2 * f]);
      D->normal.push_back(m.face_normal[2 * f + 1]);
      D->length.push_back(m.face_length[f]);
      D->midpoint.push_back(m.face_midpoint[2 * f]);
      D->midpoint.push_back(m.face_midpoint[2 * f + 1]);
      for (int q = 0; q < nq; ++q) {
        D->qp.push_back(m.face_qp[2 * (f * nq + q)]);
        D->qp.push_back(m.face_qp[2 * (f * nq + q) + 1]);
        D->qw.push_back(m.face_qw[f * nq + q]);
        D->pqp.push_back(P >= 0 ? m.face_partner_qp[f * nq + q] : -1);
      }
      D->patch.push_back(patch);
      D->partner.push_back(P);
      D->shift.push_back(P >= 0 ? m.face_shift[2 * f] : 0);
      D->shift.push_back(P >= 0 ? m.face_shift[2 * f + 1] : 0);
    }

    // ---- local stencils
    D->central_ptr = {0};
    D->pinv_off = {0};
    D->pinv_lin_off = {0};
    D->dir_ptr = {0};
    D->dir_member_ptr = {0};
    D->pinv_dir_off = {0};
    D->qp_ptr = {0};
    D->phi_off = {0};
    const int Mdummy = 2 * K, MDdummy = 4;
    for (int l = 0; l < nl; ++l) {
      const int g = D->gid[l];
      const int nfc = m.cell_face_ptr[g + 1] - m.cell_face_ptr[g];
      const int Qc = nfc * nq;
      if (is_classify[g]) {
        for (int64_t j = s.central_ptr[g]; j < s.central_ptr[g + 1]; ++j) {
          D->central.push_back(lid[s.central[3 * j]]);
          D->central.push_back(s.central[3 * j + 1]);
          D->central.push_back(s.central[3 * j + 2]);
        }
        D->pinv.insert(D->pinv.end(), s.pinv + s.pinv_off[g], s.pinv + s.pinv_off[g + 1]);
        D->pinv_lin.insert(D->pinv_lin.end(), s.pinv_lin + s.pinv_lin_off[g], s.pinv_lin + s.pinv_lin_off[g + 1]);
        for (int64_t d = s.dir_ptr[g]; d < s.dir_ptr[g + 1]; ++d) {
          D->dir_members.insert(D->dir_members.end(), s.dir_members + s.dir_member_ptr[d],
                                s.dir_members + s.dir_member_ptr[d + 1]);
          D->dir_member_ptr.push_back(static_cast<int64_t>(D->dir_members.size()));
          D->pinv_dir.insert(D->pinv_dir.end(), s.pinv_dir + s.pinv_dir_off[d], s.pinv_dir + s.pinv_dir_off[d + 1]);
          D->pinv_dir_off.push_back(static_cast<int64_t>(D->pinv_dir.size()));
        }
        D->oi.insert(D->oi.end(), s.oi + static_cast<int64_t>(g) * K * K, s.oi + static_cast<int64_t>(g + 1) * K * K);
        D->phi.insert(D->phi.end(), s.phi + s.phi_off[g], s.phi + s.phi_off[g + 1]);
      } else {  // inert stencil: only provides U to the layers inside
        for (int j = 0; j <= Mdummy; ++j) {
          D->central.push_back(l);
          D->central.push_back(0);
          D->central.push_back(0);
        }
        D->pinv.insert(D->pinv.end(), static_cast<size_t>(K) * Mdummy, 0.0);
        D->pinv_lin.insert(D->pinv_lin.end(), 2 * static_cast<size_t>(Mdummy), 0.0);
        for (int d = 0; d < nfc; ++d) {
          D->dir_members.insert(D->dir_members.end(), MDdummy + 1, 0);
          D->dir_member_ptr.push_back(static_cast<int64_t>(D->dir_members.size()));
          D->pinv_dir.insert(D->pinv_dir.end(), 2 * MDdummy, 0.0);
          D->pinv_dir_off.push_back(static_cast<int64_t>(D->pinv_dir.size()));
        }
        D->oi.insert(D->oi.end(), static_cast<size_t>(K) * K, 0.0);
        D->phi.insert(D->phi.end(), static_cast<size_t>(Qc) * K, 0.0);
      }
      D->central_ptr.push_back(static_cast<int64_t>(D->central.size() / 3));
      D->pinv_off.push_back(static_cast<int64_t>(D->pinv.size()));
      D->pinv_lin_off.push_back(static_cast<int64_t>(D->pinv_lin.size()));
      D->dir_ptr.push_back(static_cast<int64_t>(D->dir_member_ptr.size() - 1));
      D->phi_off.push_back(static_cast<int64_t>(D->phi.size()));
      // value slots with local face ids and local sides
      for (int j = 0; j < nfc; ++j) {
        const int lf = D->cf[D->cfp[l] + j];
        const int side = D->fl[lf] == l ? 0 : 1;
        for (int q = 0; q < nq; ++q) D->qp_slot.push_back((lf * nq + q) * 2 + side);
      }
      D->qp_ptr.push_back(static_cast<int64_t>(D->qp_slot.size()));
    }

    // ---- exchange plan: receive ranges (halo grouped by owner) and send lists
    std::vector<int> recv_begin(n_parts, 0), recv_count(n_parts, 0);
    for (int l = D->n_owned; l < nl; ++l) {
      const int q = part[D->gid[l]];
      if (recv_count[q] == 0) recv_begin[q] = l;
      ++recv_count[q];
    }
    std::vector<std::vector<int32_t>> send(n_parts);
    for (int q = 0; q < n_parts; ++q)
      for (int c : send_g[q]) send[q].push_back(lid[c]);
    for (int q = 0; q < n_parts; ++q) {
      if (q == r || (recv_count[q] == 0 && send[q].empty())) continue;
      ucfvb_subdomain::Peer p;
      p.rank = q;
      p.send = std::move(send[q]);
      p.recv_begin = recv_begin[q];
      p.n_recv = recv_count[q];
      D->peers.push_back(std::move(p));
    }

    // ---- views
    for (const auto& x : D->patch_names) D->pnames.push_back(x.c_str());
    ucfvb_mesh_view& v = D->mv;
    v.n_vertices = m.n_vertices;
    v.n_cells = nl;
    v.n_faces = static_cast<int32_t>(faces.size());
    v.n_qp = nq;
    v.n_patches = static_cast<int32_t>(D->patch_names.size());
    v.period_x = m.period_x;
    v.period_y = m.period_y;
    v.vertices = m.vertices;
    v.cell_vtx_ptr = D->cvp.data();
    v.cell_vtx = D->cv.data();
    v.cell_face_ptr = D->cfp.data();
    v.cell_faces = D->cf.data();
    v.cell_centroid = D->centroid.data();
    v.cell_area = D->area.data();
    v.cell_h = D->h.data();
    v.face_vtx = D->fvtx.data();
    v.face_left = D->fl.data();
    v.face_right = D->fr.data();
    v.face_normal = D->normal.data();
    v.face_length = D->length.data();
    v.face_midpoint = D->midpoint.data();
    v.face_qp = D->qp.data();
    v.face_qw = D->qw.data();
    v.face_patch = D->patch.data();
    v.face_partner = D->partner.data();
    v.face_shift = D->shift.data();
    v.face_partner_qp = D->pqp.data();
    v.patch_names = D->pnames.data();
    ucfvb_stencil_view& w = D->sv;
    w.order = s.order;
    w.K = K;
    w.n_qp = s.n_qp;
    w.si_exponent = s.si_exponent;
    w.n_cells = nl;
    w.n_dir_stencils = static_cast<int32_t>(D->dir_member_ptr.size() - 1);
    w.central_ptr = D->central_ptr.data();
    w.central = D->central.data();
    w.pinv_off = D->pinv_off.data();
    w.pinv = D->pinv.data();
    w.pinv_lin_off = D->pinv_lin_off.data();
    w.pinv_lin = D->pinv_lin.data();
    w.dir_ptr = D->dir_ptr.data();
    w.dir_member_ptr = D->dir_member_ptr.data();
    w.dir_members = D->dir_members.data();
    w.pinv_dir_off = D->pinv_dir_off.data();
    w.pinv_dir = D->pinv_dir.data();
    w.oi = D->oi.data();
    w.qp_ptr = D->qp_ptr.data();
    w.phi_off = D->phi_off.data();
    w.phi = D->phi.data();
    w.qp_slot = D->qp_slot.data();
  } catch (...) {
    delete D;
    throw;
  }
  return D;
}

}  // namespace ucfvb

