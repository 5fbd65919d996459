// Domain decomposition of the 3D stage pass (BASELINE configs 4-5 on 1/2/4/8
// GPUs): recursive coordinate bisection of the cell centroids and per-rank
// subdomains with the stencil-depth halo every owned residual depends on --
// the 3D counterpart of decompose.cpp (same dependency radius):
// classification set = layers 0..2 around the owned cells, local set =
// classification set + the central stencils and face neighbours of its cells.
// Local cells outside the classification set only provide U; their stencils
// and neighbours point at themselves (zero differences), so every kernel runs
// over all local cells and nothing they produce reaches an owned residual.
// Local faces are all faces of local cells; a side that is not local is
// replaced by the local side, and such faces never carry an owned residual.
#include <algorithm>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "decompose3.hpp"
#include "layout.hpp"
#include "ucfvb3.h"

namespace ucfvb {
namespace {

void rcb3(const ucfvb3_mesh_view& m, std::vector<int>& cells, int first, int n_parts, int32_t* part) {
  if (n_parts == 1) {
    for (int c : cells) part[c] = first;
    return;
  }
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int c : cells)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], m.cell_centroid[3 * c + d]);
      hi[d] = std::max(hi[d], m.cell_centroid[3 * c + d]);
    }
  int axis = 0;
  for (int d = 1; d < 3; ++d)
    if (hi[d] - lo[d] > hi[axis] - lo[axis]) axis = d;
  const int pa = n_parts / 2, pb = n_parts - pa;
  const size_t na = cells.size() * pa / n_parts;
  std::nth_element(cells.begin(), cells.begin() + na, cells.end(), [&](int a, int b) {
    const double xa = m.cell_centroid[3 * a + axis], xb = m.cell_centroid[3 * b + axis];
    return xa != xb ? xa < xb : a < b;
  });
  std::vector<int> A(cells.begin(), cells.begin() + na), B(cells.begin() + na, cells.end());
  std::vector<int>().swap(cells);
  rcb3(m, A, first, pa, part);
  rcb3(m, B, first + pa, pb, part);
}

struct Sets3 {
  std::vector<int> owned, classify, local;
};

Sets3 rank_sets3(const ucfvb3_mesh_view& m, const ucfvb3_stencil_view& s, const int32_t* part, int r) {
  const int n = m.n_cells, nf = m.nf, M = s.M;
  Sets3 S;
  std::vector<int8_t> level(n, -1);
  for (int c = 0; c < n; ++c)
    if (part[c] == r) {
      S.owned.push_back(c);
      level[c] = 0;
    }
  std::vector<int> frontier = S.owned, next;
  S.classify = S.owned;
  for (int l = 1; l <= 2; ++l) {
    next.clear();
    for (int c : frontier)
      for (int i = 0; i < nf; ++i) {
        const int x = m.cell_nbr[static_cast<size_t>(c) * nf + i];
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
  auto add = [&](int x) {
    if (!in_local[x]) {
      in_local[x] = 1;
      S.local.push_back(x);
    }
  };
  for (int c : S.classify) {
    for (int j = 1; j <= M; ++j) add(s.central[static_cast<size_t>(c) * (M + 1) + j]);
    for (int i = 0; i < nf; ++i) add(m.cell_nbr[static_cast<size_t>(c) * nf + i]);
  }
  return S;
}

// halo of rank r in its local order: (owner, global id)
std::vector<int> halo_of(const Sets3& S, const int32_t* part, int r) {
  std::vector<int> h;
  for (int c : S.local)
    if (part[c] != r) h.push_back(c);
  std::sort(h.begin(), h.end(), [&](int a, int b) { return part[a] != part[b] ? part[a] < part[b] : a < b; });
  return h;
}

}  // namespace

void partition_rcb3(const ucfvb3_mesh_view& m, int n_parts, int32_t* part) {
  if (n_parts < 1) throw ApiError(UCFVB_INVALID, "partition: n_parts must be >= 1");
  std::vector<int> cells(m.n_cells);
  std::iota(cells.begin(), cells.end(), 0);
  rcb3(m, cells, 0, n_parts, part);
}

ucfvb3_subdomain* build_subdomain3(const ucfvb3_mesh_view& m, const ucfvb3_stencil_view& s, const int32_t* part,
                                   int n_parts, int r) {
  if (r < 0 || r >= n_parts) throw ApiError(UCFVB_INVALID, "subdomain: rank out of range");
  if (s.n_cells != m.n_cells) throw ApiError(UCFVB_INVALID, "subdomain: stencil set does not match the mesh");
  const int n = m.n_cells, nf = m.nf, nq = m.nq, M = s.M, K = s.K, Q = s.Q, MD = s.MD, nvc = m.nvc;
  auto D = std::make_unique<ucfvb3_subdomain>();
  D->rank = r;
  D->n_parts = n_parts;
  const Sets3 S = rank_sets3(m, s, part, r);
  std::vector<int> owned = S.owned;
  std::sort(owned.begin(), owned.end());
  const std::vector<int> halo = halo_of(S, part, r);
  D->n_owned = static_cast<int>(owned.size());
  D->gid = owned;
  D->gid.insert(D->gid.end(), halo.begin(), halo.end());
  const int nl = D->n_local = static_cast<int>(D->gid.size());
  std::vector<int32_t> lid(n, -1);
  for (int l = 0; l < nl; ++l) lid[D->gid[l]] = l;
  std::vector<int8_t> classify(n, 0);
  for (int c : S.classify) classify[c] = 1;
  // local faces: every face of a local cell, in global face order
  std::vector<int32_t> lface(m.n_faces, -1);
  std::vector<int> gfaces;
  for (int l = 0; l < nl; ++l)
    for (int i = 0; i < nf; ++i) {
      const int f = m.cell_faces[static_cast<size_t>(D->gid[l]) * nf + i];
      if (lface[f] < 0) {
        lface[f] = 0;
        gfaces.push_back(f);
      }
    }
  std::sort(gfaces.begin(), gfaces.end());
  for (size_t i = 0; i < gfaces.size(); ++i) lface[gfaces[i]] = static_cast<int32_t>(i);
  const int nF = D->n_faces = static_cast<int>(gfaces.size());
  // mesh arrays
  D->cell_vtx.resize(static_cast<size_t>(nl) * nvc * 3);
  D->centroid.resize(static_cast<size_t>(nl) * 3);
  D->volume.resize(nl);
  D->h.resize(nl);
  D->cell_faces.resize(static_cast<size_t>(nl) * nf);
  D->cell_nbr.resize(static_cast<size_t>(nl) * nf);
  D->cell_nbr_shift.resize(static_cast<size_t>(nl) * nf * 3);
  D->cell_side.resize(static_cast<size_t>(nl) * nf);
  for (int l = 0; l < nl; ++l) {
    const size_t g = D->gid[l];
    std::copy_n(&m.cell_vtx[g * nvc * 3], nvc * 3, &D->cell_vtx[static_cast<size_t>(l) * nvc * 3]);
    std::copy_n(&m.cell_centroid[g * 3], 3, &D->centroid[static_cast<size_t>(l) * 3]);
    D->volume[l] = m.cell_volume[g];
    D->h[l] = m.cell_h[g];
    for (int i = 0; i < nf; ++i) {
      const size_t gi = g * nf + i, li = static_cast<size_t>(l) * nf + i;
      D->cell_faces[li] = lface[m.cell_faces[gi]];
      const int x = lid[m.cell_nbr[gi]];
      D->cell_nbr[li] = x >= 0 ? x : l;  // classification cells have every neighbour local
      for (int d = 0; d < 3; ++d) D->cell_nbr_shift[li * 3 + d] = m.cell_nbr_shift[gi * 3 + d];
      D->cell_side[li] = m.cell_side[gi];
    }
  }
  D->face_left.resize(nF);
  D->face_right.resize(nF);
  D->face_qp.resize(static_cast<size_t>(nF) * nq * 3);
  D->face_n.resize(static_cast<size_t>(nF) * nq * 3);
  D->face_wa.resize(static_cast<size_t>(nF) * nq);
  D->face_vtx.resize(static_cast<size_t>(nF) * 12);
  for (int lf = 0; lf < nF; ++lf) {
    const size_t f = gfaces[lf];
    int a = lid[m.face_left[f]], b = lid[m.face_right[f]];
    if (a < 0) a = b;
    if (b < 0) b = a;
    D->face_left[lf] = a;
    D->face_right[lf] = b;
    std::copy_n(&m.face_qp[f * nq * 3], nq * 3, &D->face_qp[static_cast<size_t>(lf) * nq * 3]);
    std::copy_n(&m.face_normal[f * nq * 3], nq * 3, &D->face_n[static_cast<size_t>(lf) * nq * 3]);
    std::copy_n(&m.face_wa[f * nq], nq, &D->face_wa[static_cast<size_t>(lf) * nq]);
    std::copy_n(&m.face_vtx[f * 12], 12, &D->face_vtx[static_cast<size_t>(lf) * 12]);
  }
  // stencils: classification cells keep theirs (all members are local), the
  // others get inert self stencils
  const bool per_cell = s.n_ops == n;
  D->central.resize(static_cast<size_t>(nl) * (M + 1));
  D->op_index.resize(nl);
  D->qp_slot.resize(static_cast<size_t>(nl) * Q);
  for (int l = 0; l < nl; ++l) {
    const size_t g = D->gid[l];
    for (int j = 0; j <= M; ++j) {
      const int x = lid[s.central[g * (M + 1) + j]];
      D->central[static_cast<size_t>(l) * (M + 1) + j] = classify[g] ? x : l;
      if (classify[g] && x < 0) throw ApiError(UCFVB_INVALID, "subdomain: stencil member outside the local set");
    }
    D->op_index[l] = per_cell ? l : s.op_index[g];
    for (int i = 0; i < nf; ++i)
      for (int q = 0; q < nq; ++q)
        D->qp_slot[static_cast<size_t>(l) * Q + i * nq + q] =
            (D->cell_faces[static_cast<size_t>(l) * nf + i] * nq + q) * 2 + D->cell_side[static_cast<size_t>(l) * nf + i];
  }
  if (per_cell) {
    auto rows = [&](const double* src, size_t E, std::vector<double>& dst) {
      dst.resize(static_cast<size_t>(nl) * E);
      for (int l = 0; l < nl; ++l) std::copy_n(&src[static_cast<size_t>(D->gid[l]) * E], E, &dst[l * E]);
    };
    rows(s.pinv, static_cast<size_t>(K) * M, D->pinv);
    rows(s.pinv_lin, static_cast<size_t>(3) * M, D->pinv_lin);
    rows(s.pinv_dir, static_cast<size_t>(nf) * 3 * MD, D->pinv_dir);
    rows(s.oi, static_cast<size_t>(K) * K, D->oi);
    rows(s.phi, static_cast<size_t>(Q) * K, D->phi);
    D->dir_members.resize(static_cast<size_t>(nl) * nf * MD);
    for (int l = 0; l < nl; ++l)
      std::copy_n(&s.dir_members[static_cast<size_t>(D->gid[l]) * nf * MD], nf * MD,
                  &D->dir_members[static_cast<size_t>(l) * nf * MD]);
  }
  // peers: receive = my halo block owned by p; send = my owned cells in p's halo (p's order)
  for (int p = 0; p < n_parts; ++p) {
    if (p == r) continue;
    ucfvb3_subdomain::Peer P;
    P.rank = p;
    int b = -1, cnt = 0;
    for (int l = D->n_owned; l < nl; ++l)
      if (part[D->gid[l]] == p) {
        if (b < 0) b = l;
        ++cnt;
      }
    P.recv_begin = b < 0 ? D->n_owned : b;
    P.n_recv = cnt;
    const Sets3 Sp = rank_sets3(m, s, part, p);
    for (int c : halo_of(Sp, part, p))
      if (part[c] == r) P.send.push_back(lid[c]);
    if (P.n_recv || !P.send.empty()) D->peers.push_back(std::move(P));
  }
  // views
  ucfvb3_mesh_view& v = D->mv;
  v = m;
  v.n_cells = nl;
  v.n_faces = nF;
  v.cell_order = 0;
  v.cell_vtx = D->cell_vtx.data();
  v.cell_centroid = D->centroid.data();
  v.cell_volume = D->volume.data();
  v.cell_h = D->h.data();
  v.cell_faces = D->cell_faces.data();
  v.cell_nbr = D->cell_nbr.data();
  v.cell_nbr_shift = D->cell_nbr_shift.data();
  v.cell_side = D->cell_side.data();
  v.face_left = D->face_left.data();
  v.face_right = D->face_right.data();
  v.face_qp = D->face_qp.data();
  v.face_normal = D->face_n.data();
  v.face_wa = D->face_wa.data();
  v.face_vtx = D->face_vtx.data();
  ucfvb3_stencil_view& w = D->sv;
  w = s;
  w.n_cells = nl;
  w.central = D->central.data();
  w.op_index = D->op_index.data();
  w.qp_slot = D->qp_slot.data();
  if (per_cell) {
    w.n_ops = nl;
    w.pinv = D->pinv.data();
    w.pinv_lin = D->pinv_lin.data();
    w.dir_members = D->dir_members.data();
    w.pinv_dir = D->pinv_dir.data();
    w.oi = D->oi.data();
    w.phi = D->phi.data();
  }
  return D.release();
}

}  // namespace ucfvb

namespace {
thread_local std::string g_err3d;
template <typename F>
int32_t guard3d(F&& f) {
  try {
    f();
    return UCFVB_OK;
  } catch (const ucfvb::ApiError& e) {
    g_err3d = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err3d = e.what();
    return UCFVB_INVALID;
  }
}
}  // namespace

extern "C" {

const char* ucfvb3_decomp_last_error(void) { return g_err3d.c_str(); }

int32_t ucfvb3_partition_rcb(const ucfvb3_mesh_view* mesh, int32_t n_parts, int32_t* part) {
  return guard3d([&] { ucfvb::partition_rcb3(*mesh, n_parts, part); });
}
int32_t ucfvb3_subdomain_build(const ucfvb3_mesh_view* mesh, const ucfvb3_stencil_view* stencils, const int32_t* part,
                               int32_t n_parts, int32_t rank, ucfvb3_subdomain** out) {
  return guard3d([&] { *out = ucfvb::build_subdomain3(*mesh, *stencils, part, n_parts, rank); });
}
int32_t ucfvb3_subdomain_views(const ucfvb3_subdomain* s, ucfvb3_mesh_view* mesh, ucfvb3_stencil_view* stencils) {
  return guard3d([&] {
    *mesh = s->mv;
    *stencils = s->sv;
  });
}
int32_t ucfvb3_subdomain_info(const ucfvb3_subdomain* s, int32_t* n_owned, int32_t* n_local, int32_t* n_peers) {
  return guard3d([&] {
    *n_owned = s->n_owned;
    *n_local = s->n_local;
    *n_peers = static_cast<int32_t>(s->peers.size());
  });
}
int32_t ucfvb3_subdomain_global_ids(const ucfvb3_subdomain* s, int32_t* gid) {
  return guard3d([&] { std::copy(s->gid.begin(), s->gid.end(), gid); });
}
int32_t ucfvb3_subdomain_peer(const ucfvb3_subdomain* s, int32_t i, int32_t* rank, int32_t* n_send, int32_t* n_recv,
                              int32_t* recv_begin) {
  return guard3d([&] {
    if (i < 0 || i >= static_cast<int>(s->peers.size())) throw ucfvb::ApiError(UCFVB_INVALID, "peer index out of range");
    const auto& p = s->peers[i];
    *rank = p.rank;
    *n_send = static_cast<int32_t>(p.send.size());
    *n_recv = p.n_recv;
    *recv_begin = p.recv_begin;
  });
}
int32_t ucfvb3_subdomain_send_list(const ucfvb3_subdomain* s, int32_t i, int32_t* local_ids) {
  return guard3d([&] {
    if (i < 0 || i >= static_cast<int>(s->peers.size())) throw ucfvb::ApiError(UCFVB_INVALID, "peer index out of range");
    std::copy(s->peers[i].send.begin(), s->peers[i].send.end(), local_ids);
  });
}
void ucfvb3_subdomain_free(ucfvb3_subdomain* s) { delete s; }

}  // extern "C"
