// Mesh side of the host setup: structured tri/quad generation with seeded
// interior-vertex jitter, connectivity + geometry (assemble_mesh,
// /root/reference/proj/src/mesh.cpp:32-97), rectangle patch tags
// (mesh.cpp:119-135) and translational periodic pairing (mesh.cpp:368-446).
// Flat storage matching ucfvb_mesh_view; the arithmetic of every geometric
// quantity follows the reference so meshes compare bitwise.
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "geom.hpp"
#include "layout.hpp"
#include "setup.hpp"

struct ucfvb_mesh {
  std::vector<double> vertices, centroid, area, h, normal, length, midpoint, qp, qw;
  std::vector<int32_t> cvp, cv, cfp, cf, fvtx, fl, fr, patch, partner, shift, pqp;
  std::vector<std::string> patch_names;
  std::vector<const char*> pnames;
  double period_x = 0.0, period_y = 0.0;
  int nqp = 1;
};

namespace ucfvb {

double uniform01(uint64_t seed, uint64_t stream, uint64_t idx) {
  uint64_t z = seed + stream * 0xD1B54A32D192ED03ULL + (idx + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

namespace {

// edge -> face lookup keyed on the smaller vertex id
struct EdgeTable {
  std::vector<std::vector<std::pair<int, int>>> by_min;
  explicit EdgeTable(size_t nv) : by_min(nv) {}
  int find(int a, int b) const {
    const int lo = std::min(a, b), hi = std::max(a, b);
    for (const auto& e : by_min[lo])
      if (e.first == hi) return e.second;
    return -1;
  }
  void add(int a, int b, int f) { by_min[std::min(a, b)].push_back({std::max(a, b), f}); }
};

void assemble(ucfvb_mesh& M, const std::vector<std::vector<int>>& cells) {
  const int nv = static_cast<int>(M.vertices.size() / 2);
  const int nc = static_cast<int>(cells.size());
  const int nq = M.nqp;
  const GaussRule g = gauss_legendre(nq);
  M.cvp.assign(1, 0);
  M.cfp.assign(1, 0);
  M.area.resize(nc);
  M.h.resize(nc);
  M.centroid.resize(2 * static_cast<size_t>(nc));
  EdgeTable edges(nv);
  for (int c = 0; c < nc; ++c) {
    const auto& vid = cells[c];
    if (vid.size() < 3) throw ApiError(UCFVB_INVALID, "cell " + std::to_string(c) + ": fewer than 3 vertices");
    std::vector<Vec2> poly;
    for (int v : vid) {
      if (v < 0 || v >= nv) throw ApiError(UCFVB_INVALID, "cell " + std::to_string(c) + ": dangling vertex id");
      poly.push_back({M.vertices[2 * v], M.vertices[2 * v + 1]});
      M.cv.push_back(v);
    }
    M.cvp.push_back(static_cast<int32_t>(M.cv.size()));
    const double a = polygon_signed_area(poly);
    if (!(a > 0.0))
      throw ApiError(UCFVB_INVALID, "cell " + std::to_string(c) + ": non-positive area (vertices must be counter-clockwise)");
    M.area[c] = a;
    M.h[c] = std::sqrt(a);
    const Vec2 ctr = polygon_centroid(poly);
    M.centroid[2 * c] = ctr.x;
    M.centroid[2 * c + 1] = ctr.y;
    const int k = static_cast<int>(vid.size());
    for (int e = 0; e < k; ++e) {
      const int a0 = vid[e], b0 = vid[(e + 1) % k];
      const int f = edges.find(a0, b0);
      if (f < 0) {
        const int fid = static_cast<int>(M.fl.size());
        const Vec2 va{M.vertices[2 * a0], M.vertices[2 * a0 + 1]};
        const Vec2 vb{M.vertices[2 * b0], M.vertices[2 * b0 + 1]};
        const Vec2 d = vb - va;
        const double len = norm(d);
        if (!(len > 0.0)) throw ApiError(UCFVB_INVALID, "cell " + std::to_string(c) + ": zero-length edge");
        const Vec2 nrm = Vec2{d.y, -d.x} / len;
        const Vec2 mid = 0.5 * (va + vb);
        M.fvtx.push_back(a0);
        M.fvtx.push_back(b0);
        M.fl.push_back(c);
        M.fr.push_back(-1);
        M.normal.push_back(nrm.x);
        M.normal.push_back(nrm.y);
        M.length.push_back(len);
        M.midpoint.push_back(mid.x);
        M.midpoint.push_back(mid.y);
        for (int q = 0; q < nq; ++q) {
          const double t = 0.5 * (g.nodes[q] + 1.0);
          const Vec2 p = va + t * (vb - va);
          M.qp.push_back(p.x);
          M.qp.push_back(p.y);
          M.qw.push_back(0.5 * g.weights[q]);
          M.pqp.push_back(-1);
        }
        M.patch.push_back(-1);
        M.partner.push_back(-1);
        M.shift.push_back(0);
        M.shift.push_back(0);
        edges.add(a0, b0, fid);
        M.cf.push_back(fid);
      } else {
        if (M.fr[f] >= 0)
          throw ApiError(UCFVB_INVALID, "non-conforming connectivity: edge shared by more than two cells");
        M.fr[f] = c;
        M.cf.push_back(f);
      }
    }
    M.cfp.push_back(static_cast<int32_t>(M.cf.size()));
  }
}

void tag_rect(ucfvb_mesh& M, double x0, double y0, double x1, double y1) {
  M.patch_names = {"left", "right", "bottom", "top"};
  const double tol = 1e-9 * std::max(x1 - x0, y1 - y0);
  const int nf = static_cast<int>(M.fl.size());
  for (int f = 0; f < nf; ++f) {
    if (M.fr[f] >= 0) continue;
    const double mx = M.midpoint[2 * f], my = M.midpoint[2 * f + 1];
    if (std::abs(mx - x0) < tol)
      M.patch[f] = 0;
    else if (std::abs(mx - x1) < tol)
      M.patch[f] = 1;
    else if (std::abs(my - y0) < tol)
      M.patch[f] = 2;
    else if (std::abs(my - y1) < tol)
      M.patch[f] = 3;
  }
}

// one axis of pair_periodic (mesh.cpp:368-446); axis 0 = x, 1 = y
void pair_axis(ucfvb_mesh& M, int axis, double tol) {
  double lo = 1e300, hi = -1e300;
  const size_t nv = M.vertices.size() / 2;
  for (size_t v = 0; v < nv; ++v) {
    const double c = M.vertices[2 * v + axis];
    lo = std::min(lo, c);
    hi = std::max(hi, c);
  }
  const double period = hi - lo;
  (axis == 0 ? M.period_x : M.period_y) = period;
  const int nf = static_cast<int>(M.fl.size());
  std::vector<int> low, high;
  for (int f = 0; f < nf; ++f) {
    if (M.fr[f] >= 0 || M.partner[f] >= 0) continue;
    const double c = M.midpoint[2 * f + axis];
    if (std::abs(c - lo) < tol)
      low.push_back(f);
    else if (std::abs(c - hi) < tol)
      high.push_back(f);
  }
  if (low.size() != high.size())
    throw ApiError(UCFVB_INVALID, "pair_periodic: side face counts differ (" + std::to_string(low.size()) + " vs " +
                                      std::to_string(high.size()) + ")");
  const Vec2 offset = axis == 0 ? Vec2{period, 0.0} : Vec2{0.0, period};
  // candidates sorted along the other coordinate: the first within tol in
  // list order (what the reference's linear scan returns) is found by
  // scanning the tol-window of the sorted order and keeping the smallest
  // position in `high`.
  const int other = 1 - axis;
  std::vector<int> order(high.size());
  for (size_t i = 0; i < high.size(); ++i) order[i] = static_cast<int>(i);
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    return M.midpoint[2 * high[a] + other] < M.midpoint[2 * high[b] + other];
  });
  std::vector<double> keys(order.size());
  for (size_t i = 0; i < order.size(); ++i) keys[i] = M.midpoint[2 * high[order[i]] + other];
  const int nq = M.nqp;
  for (int lf : low) {
    const Vec2 want = Vec2{M.midpoint[2 * lf], M.midpoint[2 * lf + 1]} + offset;
    const double key = want.y * (axis == 0) + want.x * (axis == 1);
    auto it = std::lower_bound(keys.begin(), keys.end(), key - tol);
    int best = -1;
    for (; it != keys.end() && *it <= key + tol; ++it) {
      const int hi_pos = order[it - keys.begin()];
      const int hf = high[hi_pos];
      if (M.partner[hf] >= 0) continue;
      const Vec2 mb{M.midpoint[2 * hf], M.midpoint[2 * hf + 1]};
      if (norm(mb - want) < tol && (best < 0 || hi_pos < best)) best = hi_pos;
    }
    if (best < 0)
      throw ApiError(UCFVB_INVALID, "pair_periodic: unmatched boundary face at centroid (" +
                                        std::to_string(M.midpoint[2 * lf]) + ", " +
                                        std::to_string(M.midpoint[2 * lf + 1]) + ")");
    const int match = high[best];
    if (std::abs(M.length[lf] - M.length[match]) > 1e-10)
      throw ApiError(UCFVB_INVALID, "pair_periodic: paired faces differ in length");
    M.partner[lf] = match;
    M.partner[match] = lf;
    M.shift[2 * lf + axis] = -1;
    M.shift[2 * match + axis] = +1;
    for (int i = 0; i < nq; ++i) {
      const Vec2 target = Vec2{M.qp[2 * (lf * nq + i)], M.qp[2 * (lf * nq + i) + 1]} + offset;
      int found = -1;
      for (int j = 0; j < nq; ++j) {
        const Vec2 pb{M.qp[2 * (match * nq + j)], M.qp[2 * (match * nq + j) + 1]};
        if (norm(pb - target) < tol) {
          found = j;
          break;
        }
      }
      if (found < 0) throw ApiError(UCFVB_INVALID, "pair_periodic: quadrature points of paired faces do not align");
      M.pqp[lf * nq + i] = found;
      M.pqp[match * nq + found] = i;
    }
  }
}

}  // namespace

ucfvb_mesh* mesh_structured(int nx, int ny, double x0, double y0, double x1, double y1, bool quads, int diagonal,
                            double jitter, uint64_t seed, int periodic_axis, double tol, int n_qp) {
  if (nx < 1 || ny < 1) throw ApiError(UCFVB_INVALID, "mesh generator: nx, ny must be >= 1");
  if (!(x1 - x0 > 0.0) || !(y1 - y0 > 0.0)) throw ApiError(UCFVB_INVALID, "mesh generator: zero-size domain");
  if (n_qp < 1) throw ApiError(UCFVB_INVALID, "mesh generator: n_qp must be >= 1");
  auto* M = new ucfvb_mesh;
  try {
    M->nqp = n_qp;
    const double w = x1 - x0, hgt = y1 - y0;
    M->vertices.reserve(2 * static_cast<size_t>(nx + 1) * (ny + 1));
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        M->vertices.push_back(x0 + w * i / nx);
        M->vertices.push_back(y0 + hgt * j / ny);
      }
    if (jitter != 0.0) {
      const double hx = w / nx, hy = hgt / ny;
      for (int j = 1; j < ny; ++j)
        for (int i = 1; i < nx; ++i) {
          const uint64_t v = static_cast<uint64_t>(j) * (nx + 1) + i;
          M->vertices[2 * v] += jitter * hx * (2.0 * uniform01(seed, 0, 2 * v) - 1.0);
          M->vertices[2 * v + 1] += jitter * hy * (2.0 * uniform01(seed, 0, 2 * v + 1) - 1.0);
        }
    }
    auto vid = [&](int i, int j) { return j * (nx + 1) + i; };
    std::vector<std::vector<int>> cells;
    cells.reserve((quads ? 1 : 2) * static_cast<size_t>(nx) * ny);
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int v00 = vid(i, j), v10 = vid(i + 1, j), v11 = vid(i + 1, j + 1), v01 = vid(i, j + 1);
        if (quads) {
          cells.push_back({v00, v10, v11, v01});
        } else if (!(diagonal == 1 && (i + j) % 2 == 1)) {
          cells.push_back({v00, v10, v11});
          cells.push_back({v00, v11, v01});
        } else {
          cells.push_back({v00, v10, v01});
          cells.push_back({v10, v11, v01});
        }
      }
    assemble(*M, cells);
    tag_rect(*M, x0, y0, x1, y1);
    if (periodic_axis == 1 || periodic_axis == 3) pair_axis(*M, 0, tol);
    if (periodic_axis == 2 || periodic_axis == 3) pair_axis(*M, 1, tol);
  } catch (...) {
    delete M;
    throw;
  }
  return M;
}

ucfvb_mesh_view mesh_view(const ucfvb_mesh* mc) {
  auto* M = const_cast<ucfvb_mesh*>(mc);
  M->pnames.clear();
  for (const auto& s : M->patch_names) M->pnames.push_back(s.c_str());
  ucfvb_mesh_view v{};
  v.n_vertices = static_cast<int32_t>(M->vertices.size() / 2);
  v.n_cells = static_cast<int32_t>(M->area.size());
  v.n_faces = static_cast<int32_t>(M->fl.size());
  v.n_qp = M->nqp;
  v.n_patches = static_cast<int32_t>(M->patch_names.size());
  v.period_x = M->period_x;
  v.period_y = M->period_y;
  v.vertices = M->vertices.data();
  v.cell_vtx_ptr = M->cvp.data();
  v.cell_vtx = M->cv.data();
  v.cell_face_ptr = M->cfp.data();
  v.cell_faces = M->cf.data();
  v.cell_centroid = M->centroid.data();
  v.cell_area = M->area.data();
  v.cell_h = M->h.data();
  v.face_vtx = M->fvtx.data();
  v.face_left = M->fl.data();
  v.face_right = M->fr.data();
  v.face_normal = M->normal.data();
  v.face_length = M->length.data();
  v.face_midpoint = M->midpoint.data();
  v.face_qp = M->qp.data();
  v.face_qw = M->qw.data();
  v.face_patch = M->patch.data();
  v.face_partner = M->partner.data();
  v.face_shift = M->shift.data();
  v.face_partner_qp = M->pqp.data();
  v.patch_names = M->pnames.data();
  return v;
}

void mesh_free(ucfvb_mesh* m) { delete m; }

}  // namespace ucfvb
