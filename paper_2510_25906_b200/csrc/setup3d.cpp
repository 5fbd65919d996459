// 3D host setup: periodic hexahedral / tetrahedral box
// meshes, cell and face geometry, and the per-cell operator precompute of the
// hybrid scheme generalised to three dimensions. The reference is 2D only;
// every step restates its 2D counterpart with the dimension changed:
//   lattice mesh + periodic pairing   mesh.cpp:137-170, 368-446 (torus: all faces interior)
//   Legendre-product basis            basis.cpp:12-68 (P_i(x) P_j(y) P_k(z), 1 <= i+j+k <= r)
//   central BFS stencil               stencil.cpp:31-71
//   directional stencils              stencil.cpp:73-117 (face cones instead of 2D sectors)
//   LSQ rows / QR pseudo-inverse      stencil.cpp:129-166 (qr_pinv = the ColPivHouseholderQR restatement)
//   oscillation matrix                stencil.cpp:168-190
//   phi tables + qp slots             stencil.cpp:262-281
//   initial-condition projection      cases.cpp:62-76
// Cells are processed in parallel; each cell's arithmetic is sequential and
// deterministic, so the output does not depend on the thread count.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "layout.hpp"
#include "setup.hpp"
#include "setup3d.hpp"
#include "ucfvb3.h"

struct ucfvb3_mesh {
  int kind = 0, nx = 0, ny = 0, nz = 0, nt = 1, n = 0, nF = 0, nf = 0, nq = 0, nvc = 0, blocked = 0;
  double L[3] = {0, 0, 0};
  std::vector<double> cell_vtx, centroid, volume, h;
  std::vector<int32_t> cell_faces, cell_nbr, cell_nbr_shift;
  std::vector<int8_t> cell_side;
  std::vector<int32_t> face_left, face_right;
  std::vector<double> face_qp, face_n, face_wa, face_vtx;
};

struct ucfvb3_stencils {
  int order = 1, K = 0, M = 0, MD = 6, nf = 0, nq = 0, Q = 0, n = 0, n_ops = 0, si = 0;
  std::vector<int32_t> central, op_index, dir_members, qp_slot;
  std::vector<double> pinv, pinv_lin, pinv_dir, oi, phi;
};

namespace ucfvb {

double uniform01(uint64_t seed, uint64_t stream, uint64_t idx);

namespace {

using V3 = std::array<double, 3>;
inline V3 operator+(const V3& a, const V3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
inline V3 operator-(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline V3 operator*(double s, const V3& a) { return {s * a[0], s * a[1], s * a[2]}; }
inline double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
inline double norm(const V3& a) { return std::sqrt(dot(a, a)); }

// ---- quadrature ---------------------------------------------------------------
// Gauss-Legendre nodes/weights on [0,1] (Newton on P_n, as quadrature.cpp:12-41 on [-1,1])
void gauss01(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.5);
  w.assign(n, 1.0);
  if (n == 1) return;
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::abs(dz) < 1e-16) break;
    }
    x[n - 1 - i] = 0.5 * (z + 1.0);
    w[n - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);
  }
}

struct QP3 {
  V3 x;
  double w;
};

// volume rule of degree `deg` on a cell given by its corners (hex: trilinear
// map of 8 corners, index a + 2b + 4c; tet: affine map, collapsed Gauss rule)
void volume_rule(int kind, const double* corners, int deg, std::vector<QP3>& out) {
  const int n = std::max(1, (deg + 4) / 2);
  std::vector<double> gx, gw;
  gauss01(n, gx, gw);
  out.clear();
  auto C = [&](int i) { return V3{corners[3 * i], corners[3 * i + 1], corners[3 * i + 2]}; };
  if (kind == UCFVB3_HEX) {
    V3 X[8];
    for (int i = 0; i < 8; ++i) X[i] = C(i);
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b)
        for (int c = 0; c < n; ++c) {
          const double s[3] = {gx[a], gx[b], gx[c]};
          V3 x{0, 0, 0}, J[3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
          for (int v = 0; v < 8; ++v) {
            const int bit[3] = {v & 1, (v >> 1) & 1, (v >> 2) & 1};
            double N = 1.0, dN[3] = {1.0, 1.0, 1.0};
            for (int d = 0; d < 3; ++d) {
              const double f = bit[d] ? s[d] : 1.0 - s[d];
              const double df = bit[d] ? 1.0 : -1.0;
              N *= f;
              for (int e = 0; e < 3; ++e) dN[e] *= (e == d) ? df : f;
            }
            x = x + N * X[v];
            for (int e = 0; e < 3; ++e) J[e] = J[e] + dN[e] * X[v];
          }
          const double det = dot(J[0], cross(J[1], J[2]));
          out.push_back({x, gw[a] * gw[b] * gw[c] * std::abs(det)});
        }
  } else {
    const V3 p0 = C(0), e1 = C(1) - p0, e2 = C(2) - p0, e3 = C(3) - p0;
    const double det = std::abs(dot(e1, cross(e2, e3)));
    for (int a = 0; a < n; ++a)
      for (int b = 0; b < n; ++b)
        for (int c = 0; c < n; ++c) {
          const double u = gx[a], v = gx[b], t = gx[c];
          const double l1 = u, l2 = v * (1.0 - u), l3 = t * (1.0 - u) * (1.0 - v);
          const V3 x = p0 + l1 * e1 + l2 * e2 + l3 * e3;
          out.push_back({x, gw[a] * gw[b] * gw[c] * (1.0 - u) * (1.0 - u) * (1.0 - v) * det});
        }
  }
}

// face rule: quads Gauss ng x ng on the bilinear patch, triangles 3- or 6-point
int face_nq(int kind, int order) {
  if (kind == UCFVB3_HEX) {
    const int ng = (order + 2) / 2;
    return ng * ng;
  }
  return order <= 1 ? 3 : 6;
}

void face_rule(int nv, const V3* v, int order, V3* qp, V3* nrm, double* wa) {
  if (nv == 4) {
    const int ng = (order + 2) / 2;
    std::vector<double> gx, gw;
    gauss01(ng, gx, gw);
    int q = 0;
    for (int i = 0; i < ng; ++i)
      for (int j = 0; j < ng; ++j, ++q) {
        const double s = gx[i], t = gx[j];
        qp[q] = ((1 - s) * (1 - t)) * v[0] + (s * (1 - t)) * v[1] + (s * t) * v[2] + ((1 - s) * t) * v[3];
        const V3 ds = (1 - t) * (v[1] - v[0]) + t * (v[2] - v[3]);
        const V3 dt = (1 - s) * (v[3] - v[0]) + s * (v[2] - v[1]);
        const V3 J = cross(ds, dt);
        const double a = norm(J);
        nrm[q] = (1.0 / a) * J;
        wa[q] = gw[i] * gw[j] * a;
      }
    return;
  }
  const V3 A = 0.5 * cross(v[1] - v[0], v[2] - v[0]);
  const double area = norm(A);
  const V3 n = (1.0 / area) * A;
  if (order <= 1) {
    const double l[3][3] = {{0.5, 0.5, 0.0}, {0.0, 0.5, 0.5}, {0.5, 0.0, 0.5}};
    for (int q = 0; q < 3; ++q) {
      qp[q] = l[q][0] * v[0] + l[q][1] * v[1] + l[q][2] * v[2];
      nrm[q] = n;
      wa[q] = area / 3.0;
    }
    return;
  }
  // 6-point degree-4 rule (Dunavant)
  const double a = 0.445948490915965, wa_ = 0.223381589678011;
  const double b = 0.091576213509771, wb = 0.109951743655322;
  const double l[6][3] = {{a, a, 1 - 2 * a}, {a, 1 - 2 * a, a}, {1 - 2 * a, a, a},
                          {b, b, 1 - 2 * b}, {b, 1 - 2 * b, b}, {1 - 2 * b, b, b}};
  for (int q = 0; q < 6; ++q) {
    qp[q] = l[q][0] * v[0] + l[q][1] * v[1] + l[q][2] * v[2];
    nrm[q] = n;
    wa[q] = (q < 3 ? wa_ : wb) * area;
  }
}

// ---- lattice cell topology -------------------------------------------------------
const int kPerm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
const int kHexFace[6][4] = {{0, 4, 6, 2}, {1, 3, 7, 5}, {0, 1, 5, 4}, {2, 6, 7, 3}, {0, 2, 3, 1}, {4, 5, 7, 6}};
const int kTetFace[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};

struct Topo {
  int kind, nt, nf, nvc, fv;  // types, faces/cell, corners/cell, vertices/face
  // corner lattice offsets [type][corner]
  std::vector<std::array<std::array<int, 3>, 8>> corner;
  // face table [type][lf]: corner list, neighbour (dcube, type, lf), left flag
  struct FaceInfo {
    int cs[4];
    int d[3], nt, nlf;
    bool left;
  };
  std::vector<std::array<FaceInfo, 6>> face;
  int left_faces_per_cube = 0;
  std::vector<std::array<int, 6>> left_rank;  // face id offset within the cube (or -1)

  explicit Topo(int k) : kind(k) {
    nt = (k == UCFVB3_HEX) ? 1 : 6;
    nf = (k == UCFVB3_HEX) ? 6 : 4;
    nvc = (k == UCFVB3_HEX) ? 8 : 4;
    fv = (k == UCFVB3_HEX) ? 4 : 3;
    corner.resize(nt);
    for (int t = 0; t < nt; ++t) {
      if (k == UCFVB3_HEX) {
        for (int v = 0; v < 8; ++v) corner[t][v] = {v & 1, (v >> 1) & 1, (v >> 2) & 1};
      } else {
        std::array<int, 3> p{0, 0, 0};
        corner[t][0] = p;
        for (int s = 0; s < 2; ++s) {
          p[kPerm[t][s]] = 1;
          corner[t][s + 1] = p;
        }
        corner[t][3] = {1, 1, 1};
      }
    }
    face.resize(nt);
    left_rank.resize(nt);
    auto key = [&](int t, int lf, const int* d) {
      std::vector<std::array<int, 3>> s;
      for (int i = 0; i < fv; ++i) {
        const int c = (k == UCFVB3_HEX) ? kHexFace[lf][i] : kTetFace[lf][i];
        s.push_back({corner[t][c][0] + d[0], corner[t][c][1] + d[1], corner[t][c][2] + d[2]});
      }
      std::sort(s.begin(), s.end());
      return s;
    };
    for (int t = 0; t < nt; ++t)
      for (int lf = 0; lf < nf; ++lf) {
        FaceInfo& F = face[t][lf];
        for (int i = 0; i < fv; ++i) F.cs[i] = (k == UCFVB3_HEX) ? kHexFace[lf][i] : kTetFace[lf][i];
        const int zero[3] = {0, 0, 0};
        const auto mine = key(t, lf, zero);
        bool found = false;
        for (int dx = -1; dx <= 1 && !found; ++dx)
          for (int dy = -1; dy <= 1 && !found; ++dy)
            for (int dz = -1; dz <= 1 && !found; ++dz)
              for (int t2 = 0; t2 < nt && !found; ++t2)
                for (int lf2 = 0; lf2 < nf && !found; ++lf2) {
                  if (dx == 0 && dy == 0 && dz == 0 && t2 == t) continue;
                  const int d[3] = {dx, dy, dz};
                  if (key(t2, lf2, d) == mine) {
                    F.d[0] = dx, F.d[1] = dy, F.d[2] = dz, F.nt = t2, F.nlf = lf2;
                    found = true;
                  }
                }
        if (!found) throw ApiError(UCFVB_INVALID, "mesh3d: unmatched lattice face");
        // left rule: the face on the cube's low plane belongs to this cube's
        // cell; interior faces to the lower type (translation invariant)
        int plane = -1;
        for (int a = 0; a < 3; ++a) {
          bool same = true;
          for (int i = 1; i < fv; ++i) same = same && corner[t][F.cs[i]][a] == corner[t][F.cs[0]][a];
          if (same) plane = 2 * a + corner[t][F.cs[0]][a];
        }
        F.left = (plane >= 0) ? (plane % 2 == 0) : (t < F.nt);
      }
    int r = 0;
    for (int t = 0; t < nt; ++t)
      for (int lf = 0; lf < nf; ++lf) left_rank[t][lf] = face[t][lf].left ? r++ : -1;
    left_faces_per_cube = r;
  }
};

}  // namespace

// ---- Legendre-product basis in 3D (basis.cpp:34-68 with a third factor) --------
Family3::Family3(int order) : r(order) {
  leg.resize(r + 1);
  std::vector<std::vector<double>> p(r + 1);
  p[0] = {1.0};
  if (r >= 1) p[1] = {0.0, 1.0};
  for (int m = 1; m < r; ++m) {
    std::vector<double> nx(m + 2, 0.0);
    for (int i = 0; i <= m; ++i) nx[i + 1] += (2.0 * m + 1.0) * p[m][i] / (m + 1.0);
    for (int i = 0; i < m; ++i) nx[i] -= m * p[m - 1][i] / (m + 1.0);
    p[m + 1] = std::move(nx);
  }
  // leg[n][d] = coefficients of the d-th derivative of P_n
  for (int n = 0; n <= r; ++n) {
    leg[n].resize(r + 1);
    leg[n][0] = p[n];
    for (int d = 1; d <= r; ++d) {
      const auto& prev = leg[n][d - 1];
      std::vector<double> q(prev.size() > 1 ? prev.size() - 1 : 1, 0.0);
      for (size_t i = 1; i < prev.size(); ++i) q[i - 1] = prev[i] * static_cast<double>(i);
      leg[n][d] = q;
    }
  }
  for (int t = 1; t <= r; ++t)
    for (int i = t; i >= 0; --i)
      for (int j = t - i; j >= 0; --j) deg.push_back({i, j, t - i - j});
  K = static_cast<int>(deg.size());
  for (int t = 1; t <= r; ++t)
    for (int bx = t; bx >= 0; --bx)
      for (int by = t - bx; by >= 0; --by) beta.push_back({bx, by, t - bx - by});
}

void Family3::tables(const double* xi, int dmax, double* P) const {
  // P[(axis*(r+1) + d)*(r+1) + n] = d-th derivative of P_n at xi[axis] (Horner)
  for (int a = 0; a < 3; ++a)
    for (int d = 0; d <= dmax; ++d)
      for (int n = 0; n <= r; ++n) {
        const auto& c = leg[n][d];
        double acc = 0.0;
        for (int i = static_cast<int>(c.size()) - 1; i >= 0; --i) acc = acc * xi[a] + c[i];
        P[(a * (r + 1) + d) * (r + 1) + n] = acc;
      }
}

void Family3::eval_all(const double* xi, double* out) const {
  double P[3 * 9 * 9];
  tables(xi, 0, P);
  const int s = (r + 1) * (r + 1);
  for (int k = 0; k < K; ++k) out[k] = P[deg[k][0]] * P[s + deg[k][1]] * P[2 * s + deg[k][2]];
}

void Family3::eval_deriv(int b, const double* xi, double* out) const {
  double P[3 * 9 * 9];
  tables(xi, r, P);
  const int R = r + 1;
  for (int k = 0; k < K; ++k)
    out[k] = P[(0 * R + beta[b][0]) * R + deg[k][0]] * P[(1 * R + beta[b][1]) * R + deg[k][1]] *
             P[(2 * R + beta[b][2]) * R + deg[k][2]];
}

// ---- mesh --------------------------------------------------------------------------
ucfvb3_mesh* mesh3_periodic_box(int nx, int ny, int nz, double lx, double ly, double lz, int kind, double jitter,
                                uint64_t seed, int order, int n_threads) {
  if (nx < 3 || ny < 3 || nz < 3) throw ApiError(UCFVB_INVALID, "mesh3d: need at least 3 cubes per direction");
  if (kind != UCFVB3_HEX && kind != UCFVB3_TET) throw ApiError(UCFVB_INVALID, "mesh3d: unknown cell kind");
  if (order < 1 || order > 6) throw ApiError(UCFVB_INVALID, "mesh3d: order must be in [1, 6]");
  if (!(jitter >= 0.0 && jitter < 0.25)) throw ApiError(UCFVB_INVALID, "mesh3d: jitter must be in [0, 0.25)");
  const Topo T(kind);
  auto M = std::make_unique<ucfvb3_mesh>();
  M->kind = kind, M->nx = nx, M->ny = ny, M->nz = nz, M->nt = T.nt, M->nf = T.nf, M->nvc = T.nvc;
  M->nq = face_nq(kind, order);
  M->L[0] = lx, M->L[1] = ly, M->L[2] = lz;
  const int64_t ncube = static_cast<int64_t>(nx) * ny * nz;
  const int64_t n64 = ncube * T.nt;
  const int64_t nF64 = ncube * T.left_faces_per_cube;
  if (nF64 * M->nq * 2 >= (int64_t(1) << 31)) throw ApiError(UCFVB_INVALID, "mesh3d: too many faces for int32 slots");
  const int n = static_cast<int>(n64), nF = static_cast<int>(nF64);
  M->n = n, M->nF = nF;
  // tetrahedra of 32 consecutive cubes are numbered type-major, so every
  // 32-cell chunk holds one type (one shared operator row under lattice classes)
  M->blocked = (T.nt == 6 && ncube % 32 == 0) ? 1 : 0;
  const CellOrder ord{T.nt, M->blocked};
  const double hh[3] = {lx / nx, ly / ny, lz / nz};
  // wrapped vertex positions
  std::vector<double> vpos(static_cast<size_t>(ncube) * 3);
  parallel_for(ncube, n_threads, [&](int64_t a0, int64_t a1) {
    for (int64_t v = a0; v < a1; ++v) {
      const int64_t ijk[3] = {v % nx, (v / nx) % ny, v / (static_cast<int64_t>(nx) * ny)};
      for (int d = 0; d < 3; ++d)
        vpos[3 * v + d] = ijk[d] * hh[d] + jitter * hh[d] * (2.0 * uniform01(seed, 3, 3 * static_cast<uint64_t>(v) + d) - 1.0);
    }
  });
  const int nf = T.nf, nq = M->nq, nvc = T.nvc;
  M->cell_vtx.resize(static_cast<size_t>(n) * nvc * 3);
  M->centroid.resize(static_cast<size_t>(n) * 3);
  M->volume.resize(n);
  M->h.resize(n);
  M->cell_faces.resize(static_cast<size_t>(n) * nf);
  M->cell_nbr.resize(static_cast<size_t>(n) * nf);
  M->cell_nbr_shift.resize(static_cast<size_t>(n) * nf * 3);
  M->cell_side.resize(static_cast<size_t>(n) * nf);
  M->face_left.resize(nF);
  M->face_right.resize(nF);
  M->face_qp.resize(static_cast<size_t>(nF) * nq * 3);
  M->face_n.resize(static_cast<size_t>(nF) * nq * 3);
  M->face_wa.resize(static_cast<size_t>(nF) * nq);
  M->face_vtx.assign(static_cast<size_t>(nF) * 12, 0.0);
  const int N3[3] = {nx, ny, nz};
  auto cube_of = [&](int64_t c, int* ijk) {
    const int64_t q = ord.cube(c);
    ijk[0] = static_cast<int>(q % nx);
    ijk[1] = static_cast<int>((q / nx) % ny);
    ijk[2] = static_cast<int>(q / (static_cast<int64_t>(nx) * ny));
  };
  // pass 1: cell geometry, neighbours, left-face ids
  parallel_for(n, n_threads, [&](int64_t a0, int64_t a1) {
    std::vector<QP3> qp;
    for (int64_t c = a0; c < a1; ++c) {
      int ijk[3];
      cube_of(c, ijk);
      const int t = ord.type(c);
      double* cv = &M->cell_vtx[static_cast<size_t>(c) * nvc * 3];
      for (int v = 0; v < nvc; ++v) {
        int64_t w[3];
        double sh[3];
        for (int d = 0; d < 3; ++d) {
          const int g = ijk[d] + T.corner[t][v][d];
          w[d] = g % N3[d];
          sh[d] = (g >= N3[d]) ? M->L[d] : 0.0;
        }
        const int64_t vid = (w[2] * ny + w[1]) * nx + w[0];
        for (int d = 0; d < 3; ++d) cv[3 * v + d] = vpos[3 * vid + d] + sh[d];
      }
      volume_rule(kind, cv, 1, qp);
      double vol = 0.0;
      V3 xc{0, 0, 0};
      for (const QP3& p : qp) {
        vol += p.w;
        xc = xc + p.w * p.x;
      }
      M->volume[c] = vol;
      M->h[c] = std::cbrt(vol);
      for (int d = 0; d < 3; ++d) M->centroid[3 * c + d] = xc[d] / vol;
      const int64_t cube = ord.cube(c);
      for (int lf = 0; lf < nf; ++lf) {
        const auto& F = T.face[t][lf];
        int nb[3];
        int32_t* sh = &M->cell_nbr_shift[(static_cast<size_t>(c) * nf + lf) * 3];
        for (int d = 0; d < 3; ++d) {
          const int g = ijk[d] + F.d[d];
          nb[d] = (g + N3[d]) % N3[d];
          sh[d] = (g < 0) ? -1 : (g >= N3[d] ? 1 : 0);
        }
        M->cell_nbr[static_cast<size_t>(c) * nf + lf] =
            static_cast<int32_t>(ord.cell((static_cast<int64_t>(nb[2]) * ny + nb[1]) * nx + nb[0], F.nt));
        M->cell_side[static_cast<size_t>(c) * nf + lf] = F.left ? 0 : 1;
        if (F.left)
          M->cell_faces[static_cast<size_t>(c) * nf + lf] =
              static_cast<int32_t>(cube * T.left_faces_per_cube + T.left_rank[t][lf]);
      }
    }
  });
  // pass 2: right-face ids and face geometry (computed by the left cell)
  parallel_for(n, n_threads, [&](int64_t a0, int64_t a1) {
    for (int64_t c = a0; c < a1; ++c) {
      const int t = ord.type(c);
      for (int lf = 0; lf < nf; ++lf) {
        const auto& F = T.face[t][lf];
        const size_t i = static_cast<size_t>(c) * nf + lf;
        if (!F.left) {
          const int nbc = M->cell_nbr[i];
          M->cell_faces[i] = M->cell_faces[static_cast<size_t>(nbc) * nf + F.nlf];
          continue;
        }
        const int f = M->cell_faces[i];
        M->face_left[f] = static_cast<int32_t>(c);
        M->face_right[f] = M->cell_nbr[i];
        const double* cv = &M->cell_vtx[static_cast<size_t>(c) * nvc * 3];
        V3 v[4];
        for (int k = 0; k < T.fv; ++k) v[k] = {cv[3 * F.cs[k]], cv[3 * F.cs[k] + 1], cv[3 * F.cs[k] + 2]};
        // outward orientation for the left cell
        V3 fc{0, 0, 0};
        for (int k = 0; k < T.fv; ++k) fc = fc + (1.0 / T.fv) * v[k];
        const V3 cc{M->centroid[3 * c], M->centroid[3 * c + 1], M->centroid[3 * c + 2]};
        const V3 an = (T.fv == 4) ? cross(v[1] - v[0] + (v[2] - v[3]), v[3] - v[0] + (v[2] - v[1]))
                                  : cross(v[1] - v[0], v[2] - v[0]);
        if (dot(an, fc - cc) < 0.0) std::swap(v[1], v[T.fv - 1]);
        V3 qp[8], nr[8];
        double wa[8];
        face_rule(T.fv, v, order, qp, nr, wa);
        for (int q = 0; q < nq; ++q) {
          for (int d = 0; d < 3; ++d) {
            M->face_qp[(static_cast<size_t>(f) * nq + q) * 3 + d] = qp[q][d];
            M->face_n[(static_cast<size_t>(f) * nq + q) * 3 + d] = nr[q][d];
          }
          M->face_wa[static_cast<size_t>(f) * nq + q] = wa[q];
        }
        for (int k = 0; k < T.fv; ++k)
          for (int d = 0; d < 3; ++d) M->face_vtx[static_cast<size_t>(f) * 12 + 3 * k + d] = v[k][d];
      }
    }
  });
  return M.release();
}

ucfvb3_mesh_view mesh3_view(const ucfvb3_mesh* M) {
  ucfvb3_mesh_view v{};
  v.kind = M->kind, v.nx = M->nx, v.ny = M->ny, v.nz = M->nz, v.n_types = M->nt;
  v.cell_order = M->blocked;
  v.n_cells = M->n, v.n_faces = M->nF, v.nf = M->nf, v.nq = M->nq, v.nvc = M->nvc;
  for (int d = 0; d < 3; ++d) v.period[d] = M->L[d];
  v.cell_vtx = M->cell_vtx.data();
  v.cell_centroid = M->centroid.data();
  v.cell_volume = M->volume.data();
  v.cell_h = M->h.data();
  v.cell_faces = M->cell_faces.data();
  v.cell_nbr = M->cell_nbr.data();
  v.cell_nbr_shift = M->cell_nbr_shift.data();
  v.cell_side = M->cell_side.data();
  v.face_left = M->face_left.data();
  v.face_right = M->face_right.data();
  v.face_qp = M->face_qp.data();
  v.face_normal = M->face_n.data();
  v.face_wa = M->face_wa.data();
  v.face_vtx = M->face_vtx.data();
  return v;
}

void mesh3_free(ucfvb3_mesh* m) { delete m; }

// ---- operator precompute ------------------------------------------------------------
namespace {

struct E3 {
  int cell, s[3];
  bool operator==(const E3& o) const {
    return cell == o.cell && s[0] == o.s[0] && s[1] == o.s[1] && s[2] == o.s[2];
  }
};

struct Builder3 {
  const ucfvb3_mesh_view& m;
  const Family3& fam;
  int order, K, M, MD, si;

  V3 centroid(int c) const { return {m.cell_centroid[3 * c], m.cell_centroid[3 * c + 1], m.cell_centroid[3 * c + 2]}; }
  V3 shift(const int* s) const { return {s[0] * m.period[0], s[1] * m.period[1], s[2] * m.period[2]}; }
  V3 entry_centroid(const E3& e) const { return centroid(e.cell) + shift(e.s); }

  void corners(const E3& e, std::vector<double>& cv) const {
    const V3 sh = shift(e.s);
    cv.resize(static_cast<size_t>(m.nvc) * 3);
    for (int v = 0; v < m.nvc; ++v)
      for (int d = 0; d < 3; ++d) cv[3 * v + d] = m.cell_vtx[(static_cast<size_t>(e.cell) * m.nvc + v) * 3 + d] + sh[d];
  }

  // stencil.cpp:31-71 in 3D
  void central_stencil(int cell, std::vector<E3>& st) const {
    const V3 origin = centroid(cell);
    const E3 self{cell, {0, 0, 0}};
    st.assign(1, self);
    std::vector<E3> visited{self}, ring{self}, next;
    std::vector<std::pair<double, E3>> keyed;
    while (static_cast<int>(st.size()) < M + 1) {
      next.clear();
      for (const E3& e : ring)
        for (int lf = 0; lf < m.nf; ++lf) {
          const size_t i = static_cast<size_t>(e.cell) * m.nf + lf;
          E3 nb{m.cell_nbr[i], {e.s[0] + m.cell_nbr_shift[3 * i], e.s[1] + m.cell_nbr_shift[3 * i + 1],
                                e.s[2] + m.cell_nbr_shift[3 * i + 2]}};
          if (std::find(visited.begin(), visited.end(), nb) == visited.end()) {
            visited.push_back(nb);
            next.push_back(nb);
          }
        }
      if (next.empty()) throw ApiError(UCFVB_INVALID, "stencil3d: mesh too small");
      keyed.clear();
      for (const E3& e : next) keyed.push_back({norm(entry_centroid(e) - origin), e});
      std::sort(keyed.begin(), keyed.end(), [](const auto& a, const auto& b) {
        if (a.first != b.first) return a.first < b.first;
        if (a.second.cell != b.second.cell) return a.second.cell < b.second.cell;
        for (int d = 0; d < 3; ++d)
          if (a.second.s[d] != b.second.s[d]) return a.second.s[d] < b.second.s[d];
        return false;
      });
      for (size_t i = 0; i < keyed.size(); ++i) {
        next[i] = keyed[i].second;
        if (static_cast<int>(st.size()) < M + 1) st.push_back(keyed[i].second);
      }
      ring.swap(next);
    }
  }

  struct CellOps {
    std::vector<E3> central;
    std::vector<double> pinv, pinv_lin, pinv_dir, oi, phi;
    std::vector<int32_t> dir;
  };

  void build(int c, CellOps& out) const {
    const V3 origin = centroid(c);
    const double h = m.cell_h[c];
    std::vector<double> cv;
    std::vector<QP3> qp;
    double psi[128];
    // basis means over the cell at degree 2r (basis.cpp:125-137)
    corners({c, {0, 0, 0}}, cv);
    volume_rule(m.kind, cv.data(), 2 * order, qp);
    std::vector<double> mean(K, 0.0);
    double vol = 0.0;
    for (const QP3& p : qp) vol += p.w;
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (const QP3& p : qp) {
        const double xi[3] = {(p.x[0] - origin[0]) / h, (p.x[1] - origin[1]) / h, (p.x[2] - origin[2]) / h};
        fam.eval_all(xi, psi);
        s += p.w * psi[k];
      }
      mean[k] = s / vol;
    }
    // central stencil and LSQ rows (stencil.cpp:129-150)
    central_stencil(c, out.central);
    std::vector<double> A(static_cast<size_t>(M) * K, 0.0);
    for (int r = 0; r < M; ++r) {
      corners(out.central[r + 1], cv);
      volume_rule(m.kind, cv.data(), order, qp);
      double* row = &A[static_cast<size_t>(r) * K];
      double w = 0.0;
      for (const QP3& p : qp) {
        const double xi[3] = {(p.x[0] - origin[0]) / h, (p.x[1] - origin[1]) / h, (p.x[2] - origin[2]) / h};
        fam.eval_all(xi, psi);
        for (int k = 0; k < K; ++k) row[k] += p.w * (psi[k] - mean[k]);
        w += p.w;
      }
      for (int k = 0; k < K; ++k) row[k] /= w;
    }
    if (!qr_pinv(A, M, K, out.pinv))
      throw ApiError(UCFVB_INVALID, "stencil3d: cell " + std::to_string(c) + " central system is rank-deficient");
    std::vector<double> A1(static_cast<size_t>(M) * 3);
    for (int r = 0; r < M; ++r)
      for (int k = 0; k < 3; ++k) A1[r * 3 + k] = A[static_cast<size_t>(r) * K + k];
    if (!qr_pinv(A1, M, 3, out.pinv_lin))
      throw ApiError(UCFVB_INVALID, "stencil3d: cell " + std::to_string(c) + " r=1 system is rank-deficient");
    // directional cones, one per face (stencil.cpp:73-117)
    std::vector<V3> dir(M);
    std::vector<double> dist(M);
    for (int i = 0; i < M; ++i) {
      dir[i] = entry_centroid(out.central[i + 1]) - origin;
      dist[i] = norm(dir[i]);
    }
    std::vector<int> by(M);
    for (int i = 0; i < M; ++i) by[i] = i;
    std::sort(by.begin(), by.end(), [&](int a, int b) {
      if (dist[a] != dist[b]) return dist[a] < dist[b];
      return a < b;
    });
    const int fv = (m.kind == UCFVB3_HEX) ? 4 : 3;
    out.dir.clear();
    out.pinv_dir.clear();
    for (int lf = 0; lf < m.nf; ++lf) {
      const size_t i = static_cast<size_t>(c) * m.nf + lf;
      const int f = m.cell_faces[i];
      V3 sh{0, 0, 0};
      if (m.cell_side[i]) sh = shift(&m.cell_nbr_shift[3 * i]);
      V3 v[4], fc{0, 0, 0};
      for (int k = 0; k < fv; ++k) {
        v[k] = V3{m.face_vtx[static_cast<size_t>(f) * 12 + 3 * k], m.face_vtx[static_cast<size_t>(f) * 12 + 3 * k + 1],
                  m.face_vtx[static_cast<size_t>(f) * 12 + 3 * k + 2]} + sh - origin;
        fc = fc + (1.0 / fv) * v[k];
      }
      // side planes of the cone through the face; members on a side plane
      // count as inside (relative tolerance 1e-10 so lattice-aligned members
      // are not lost to rounding; the 2D sector test is inclusive too)
      double sgn[4], tol[4];
      for (int k = 0; k < fv; ++k) {
        const V3 pn = cross(v[k], v[(k + 1) % fv]);
        sgn[k] = dot(pn, fc) >= 0.0 ? 1.0 : -1.0;
        tol[k] = -1e-10 * norm(pn);
      }
      std::vector<int> mem;
      for (int idx : by) {
        if (static_cast<int>(mem.size()) >= MD) break;
        bool in = true;
        for (int k = 0; k < fv && in; ++k)
          in = sgn[k] * dot(cross(v[k], v[(k + 1) % fv]), dir[idx]) >= tol[k] * dist[idx];
        if (in) mem.push_back(idx + 1);
      }
      for (int idx : by) {
        if (static_cast<int>(mem.size()) >= MD) break;
        if (std::find(mem.begin(), mem.end(), idx + 1) == mem.end()) mem.push_back(idx + 1);
      }
      std::vector<double> Ad(static_cast<size_t>(MD) * 3), pd;
      for (int r = 0; r < MD; ++r)
        for (int k = 0; k < 3; ++k) Ad[r * 3 + k] = A[static_cast<size_t>(mem[r] - 1) * K + k];
      if (!qr_pinv(Ad, MD, 3, pd)) {
        std::string msg = "stencil3d: cell " + std::to_string(c) + " face " + std::to_string(lf) +
                          " directional system is rank-deficient; rows:";
        for (int r = 0; r < MD; ++r)
          msg += " [" + std::to_string(Ad[r * 3]) + "," + std::to_string(Ad[r * 3 + 1]) + "," +
                 std::to_string(Ad[r * 3 + 2]) + "]";
        throw ApiError(UCFVB_INVALID, msg);
      }
      out.dir.insert(out.dir.end(), mem.begin(), mem.end());
      out.pinv_dir.insert(out.pinv_dir.end(), pd.begin(), pd.end());
    }
    // oscillation matrix (stencil.cpp:168-190), reference-frame weights w / h^3
    corners({c, {0, 0, 0}}, cv);
    volume_rule(m.kind, cv.data(), 2 * order, qp);
    out.oi.assign(static_cast<size_t>(K) * K, 0.0);
    double d[128];
    for (size_t b = 0; b < fam.beta.size(); ++b) {
      const int bt = fam.beta[b][0] + fam.beta[b][1] + fam.beta[b][2];
      const double hpow = (si == UCFVB_SI_PAPER) ? std::pow(std::abs(h), bt - 1) : std::pow(std::abs(h), 2 * bt - 2);
      for (const QP3& p : qp) {
        const double xi[3] = {(p.x[0] - origin[0]) / h, (p.x[1] - origin[1]) / h, (p.x[2] - origin[2]) / h};
        fam.eval_deriv(static_cast<int>(b), xi, d);
        const double w = (p.w / (h * h * h)) * hpow;
        for (int k = 0; k < K; ++k) {
          const double wk = w * d[k];
          for (int l = 0; l < K; ++l) out.oi[static_cast<size_t>(k) * K + l] += wk * d[l];
        }
      }
    }
    // phi at the cell's face quadrature points (stencil.cpp:262-281)
    out.phi.assign(static_cast<size_t>(m.nf) * m.nq * K, 0.0);
    for (int lf = 0; lf < m.nf; ++lf) {
      const size_t i = static_cast<size_t>(c) * m.nf + lf;
      const int f = m.cell_faces[i];
      V3 sh{0, 0, 0};
      if (m.cell_side[i]) sh = shift(&m.cell_nbr_shift[3 * i]);
      for (int q = 0; q < m.nq; ++q) {
        const double* x = &m.face_qp[(static_cast<size_t>(f) * m.nq + q) * 3];
        const double xi[3] = {(x[0] + sh[0] - origin[0]) / h, (x[1] + sh[1] - origin[1]) / h,
                              (x[2] + sh[2] - origin[2]) / h};
        fam.eval_all(xi, psi);
        double* dst = &out.phi[(static_cast<size_t>(lf) * m.nq + q) * K];
        for (int k = 0; k < K; ++k) dst[k] = psi[k] - mean[k];
      }
    }
  }
};

}  // namespace

ucfvb3_stencils* build_stencils3(const ucfvb3_mesh_view& m, int order, int si, int classes, int n_threads) {
  if (order < 1 || order > 6) throw ApiError(UCFVB_INVALID, "build_stencils3: order must be in [1, 6]");
  const Family3 fam(order);
  const int K = fam.K;
  if (m.nq != face_nq(m.kind, order))
    throw ApiError(UCFVB_INVALID, "build_stencils3: mesh was built for a different order (face rule)");
  auto S = std::make_unique<ucfvb3_stencils>();
  const int n = m.n_cells, nf = m.nf;
  S->order = order, S->K = K, S->M = 2 * K, S->MD = 6, S->nf = nf, S->nq = m.nq, S->Q = nf * m.nq;
  S->n = n, S->si = si;
  const int M = S->M, MD = S->MD, Q = S->Q;
  Builder3 B{m, fam, order, K, M, MD, si};
  S->central.resize(static_cast<size_t>(n) * (M + 1));
  S->op_index.resize(n);
  S->qp_slot.resize(static_cast<size_t>(n) * Q);
  // qp slots (per cell in every mode)
  parallel_for(n, n_threads, [&](int64_t a0, int64_t a1) {
    for (int64_t c = a0; c < a1; ++c)
      for (int lf = 0; lf < nf; ++lf) {
        const size_t i = static_cast<size_t>(c) * nf + lf;
        for (int q = 0; q < m.nq; ++q)
          S->qp_slot[static_cast<size_t>(c) * Q + lf * m.nq + q] =
              (m.cell_faces[i] * m.nq + q) * 2 + m.cell_side[i];
      }
  });
  auto alloc_ops = [&](int nops) {
    S->n_ops = nops;
    S->pinv.resize(static_cast<size_t>(nops) * K * M);
    S->pinv_lin.resize(static_cast<size_t>(nops) * 3 * M);
    S->dir_members.resize(static_cast<size_t>(nops) * nf * MD);
    S->pinv_dir.resize(static_cast<size_t>(nops) * nf * 3 * MD);
    S->oi.resize(static_cast<size_t>(nops) * K * K);
    S->phi.resize(static_cast<size_t>(nops) * Q * K);
  };
  auto store_ops = [&](int op, const Builder3::CellOps& o) {
    std::copy(o.pinv.begin(), o.pinv.end(), S->pinv.begin() + static_cast<size_t>(op) * K * M);
    std::copy(o.pinv_lin.begin(), o.pinv_lin.end(), S->pinv_lin.begin() + static_cast<size_t>(op) * 3 * M);
    std::copy(o.dir.begin(), o.dir.end(), S->dir_members.begin() + static_cast<size_t>(op) * nf * MD);
    std::copy(o.pinv_dir.begin(), o.pinv_dir.end(), S->pinv_dir.begin() + static_cast<size_t>(op) * nf * 3 * MD);
    std::copy(o.oi.begin(), o.oi.end(), S->oi.begin() + static_cast<size_t>(op) * K * K);
    std::copy(o.phi.begin(), o.phi.end(), S->phi.begin() + static_cast<size_t>(op) * Q * K);
  };
  if (!classes) {
    alloc_ops(n);
    parallel_for(n, n_threads, [&](int64_t a0, int64_t a1) {
      Builder3::CellOps o;
      for (int64_t c = a0; c < a1; ++c) {
        B.build(static_cast<int>(c), o);
        for (int j = 0; j <= M; ++j) S->central[static_cast<size_t>(c) * (M + 1) + j] = o.central[j].cell;
        S->op_index[c] = static_cast<int32_t>(c);
        store_ops(static_cast<int>(c), o);
      }
    });
    return S.release();
  }
  // lattice classes: every cell of a type is a translate of the canonical
  // cell of that type (checked), so it shares its operator row and its
  // stencil as lattice offsets
  const int nt = m.n_types, nx = m.nx, ny = m.ny, nz = m.nz;
  const int ci[3] = {nx / 2, ny / 2, nz / 2};
  const double hx[3] = {m.period[0] / nx, m.period[1] / ny, m.period[2] / nz};
  const CellOrder ord{nt, m.cell_order};
  auto cell_id = [&](int64_t i, int64_t j, int64_t k, int t) {
    return static_cast<int32_t>(ord.cell((k * ny + j) * nx + i, t));
  };
  {
    // translation check on the corner coordinates (unjittered lattice only)
    std::vector<int> bad(1, 0);
    parallel_for(n, n_threads, [&](int64_t a0, int64_t a1) {
      for (int64_t c = a0; c < a1; ++c) {
        const int64_t q = ord.cube(c);
        const int64_t ijk[3] = {q % nx, (q / nx) % ny, q / (static_cast<int64_t>(nx) * ny)};
        const int64_t c0 = cell_id(0, 0, 0, ord.type(c));
        for (int v = 0; v < m.nvc; ++v)
          for (int d = 0; d < 3; ++d) {
            const double a = m.cell_vtx[(static_cast<size_t>(c) * m.nvc + v) * 3 + d] - ijk[d] * hx[d];
            const double b = m.cell_vtx[(static_cast<size_t>(c0) * m.nvc + v) * 3 + d];
            if (std::abs(a - b) > 1e-9 * hx[d]) bad[0] = 1;
          }
      }
    });
    if (bad[0]) throw ApiError(UCFVB_INVALID, "build_stencils3: lattice classes need an unjittered lattice mesh");
  }
  alloc_ops(nt);
  std::vector<std::vector<std::array<int, 4>>> offs(nt);  // per type: (di, dj, dk, type) of each central entry
  for (int t = 0; t < nt; ++t) {
    Builder3::CellOps o;
    const int c0 = cell_id(ci[0], ci[1], ci[2], t);
    B.build(c0, o);
    store_ops(t, o);
    for (const E3& e : o.central) {
      const int64_t q = ord.cube(e.cell);
      const int64_t ijk[3] = {q % nx, (q / nx) % ny, q / (static_cast<int64_t>(nx) * ny)};
      std::array<int, 4> d{};
      const int N3[3] = {nx, ny, nz};
      for (int a = 0; a < 3; ++a) d[a] = static_cast<int>(ijk[a] + static_cast<int64_t>(e.s[a]) * N3[a] - ci[a]);
      d[3] = ord.type(e.cell);
      offs[t].push_back(d);
    }
  }
  parallel_for(n, n_threads, [&](int64_t a0, int64_t a1) {
    for (int64_t c = a0; c < a1; ++c) {
      const int t = ord.type(c);
      const int64_t q = ord.cube(c);
      const int64_t ijk[3] = {q % nx, (q / nx) % ny, q / (static_cast<int64_t>(nx) * ny)};
      S->op_index[c] = t;
      for (int j = 0; j <= M; ++j) {
        const auto& d = offs[t][j];
        const int64_t i2 = ((ijk[0] + d[0]) % nx + nx) % nx, j2 = ((ijk[1] + d[1]) % ny + ny) % ny,
                      k2 = ((ijk[2] + d[2]) % nz + nz) % nz;
        S->central[static_cast<size_t>(c) * (M + 1) + j] = cell_id(i2, j2, k2, d[3]);
      }
    }
  });
  return S.release();
}

ucfvb3_stencil_view stencils3_view(const ucfvb3_stencils* S) {
  ucfvb3_stencil_view v{};
  v.order = S->order, v.K = S->K, v.M = S->M, v.MD = S->MD, v.nf = S->nf, v.nq = S->nq, v.Q = S->Q;
  v.n_cells = S->n, v.n_ops = S->n_ops, v.si_exponent = S->si;
  v.central = S->central.data();
  v.op_index = S->op_index.data();
  v.pinv = S->pinv.data();
  v.pinv_lin = S->pinv_lin.data();
  v.dir_members = S->dir_members.data();
  v.pinv_dir = S->pinv_dir.data();
  v.oi = S->oi.data();
  v.phi = S->phi.data();
  v.qp_slot = S->qp_slot.data();
  return v;
}

void stencils3_free(ucfvb3_stencils* s) { delete s; }

// ---- initial conditions --------------------------------------------------------------
namespace {

void prim_to_cons5(double rho, double u, double v, double w, double p, double g, double* s) {
  s[0] = rho;
  s[1] = rho * u;
  s[2] = rho * v;
  s[3] = rho * w;
  s[4] = p / (g - 1.0) + 0.5 * rho * (u * u + v * v + w * w);
}

}  // namespace

void project_initial3(const ucfvb3_mesh_view& m, int ic, const double* prm, int n_prm, uint64_t seed, int degree,
                      double g, int n_threads, double* u_out) {
  const int n = m.n_cells;
  if (ic == UCFVB3_IC_TGV || ic == UCFVB3_IC_UNIFORM || ic == UCFVB3_IC_BLAST) {
    if (ic == UCFVB3_IC_TGV && n_prm < 1) throw ApiError(UCFVB_INVALID, "TGV IC needs {Mach}");
    if (ic == UCFVB3_IC_UNIFORM && n_prm < 5) throw ApiError(UCFVB_INVALID, "uniform IC needs 5 parameters");
    if (ic == UCFVB3_IC_BLAST && n_prm < 8) throw ApiError(UCFVB_INVALID, "blast IC needs 8 parameters");
    parallel_for(n, n_threads, [&](int64_t a0, int64_t a1) {
      std::vector<QP3> qp;
      for (int64_t c = a0; c < a1; ++c) {
        volume_rule(m.kind, &m.cell_vtx[static_cast<size_t>(c) * m.nvc * 3], degree, qp);
        double acc[5] = {0, 0, 0, 0, 0}, vol = 0.0;
        for (const QP3& q : qp) {
          double s[5];
          const double x = q.x[0], y = q.x[1], z = q.x[2];
          if (ic == UCFVB3_IC_TGV) {
            const double p0 = 1.0 / (g * prm[0] * prm[0]);
            const double p = p0 + (std::cos(2 * x) + std::cos(2 * y)) * (std::cos(2 * z) + 2.0) / 16.0;
            prim_to_cons5(1.0, std::sin(x) * std::cos(y) * std::cos(z), -std::cos(x) * std::sin(y) * std::cos(z), 0.0,
                          p, g, s);
          } else if (ic == UCFVB3_IC_UNIFORM) {
            prim_to_cons5(prm[0], prm[1], prm[2], prm[3], prm[4], g, s);
          } else {
            const double dx = x - prm[0], dy = y - prm[1], dz = z - prm[2];
            const bool in = dx * dx + dy * dy + dz * dz < prm[3] * prm[3];
            prim_to_cons5(in ? prm[4] : prm[6], 0.0, 0.0, 0.0, in ? prm[5] : prm[7], g, s);
          }
          for (int v = 0; v < 5; ++v) acc[v] += q.w * s[v];
          vol += q.w;
        }
        for (int v = 0; v < 5; ++v) u_out[5 * c + v] = acc[v] / vol;
      }
    });
    return;
  }
  if (ic != UCFVB3_IC_RANDOM_PHASE) throw ApiError(UCFVB_INVALID, "unknown 3D initial condition " + std::to_string(ic));
  if (n_prm < 3) throw ApiError(UCFVB_INVALID, "random-phase IC needs {rms Mach, k0, kmax}");
  const double mach = prm[0], k0 = prm[1];
  const int km = static_cast<int>(prm[2]);
  if (km < 1 || km > 32) throw ApiError(UCFVB_INVALID, "random-phase IC: kmax must be in [1, 32]");
  // solenoidal modes: u(x) = sum_k a(|k|) (e1 cos(k.x + f1) + e2 cos(k.x + f2)), e1, e2 unit and orthogonal to k
  struct Mode {
    int k[3];
    double e1[3], e2[3], c1, s1, c2, s2;
  };
  std::vector<Mode> modes;
  uint64_t idx = 0;
  const double kw[3] = {2 * M_PI / m.period[0], 2 * M_PI / m.period[1], 2 * M_PI / m.period[2]};
  for (int kx = 0; kx <= km; ++kx)
    for (int ky = -km; ky <= km; ++ky)
      for (int kz = -km; kz <= km; ++kz) {
        if (kx * kx + ky * ky + kz * kz > km * km) continue;
        if (!(kx > 0 || (kx == 0 && ky > 0) || (kx == 0 && ky == 0 && kz > 0))) continue;
        Mode md{};
        md.k[0] = kx, md.k[1] = ky, md.k[2] = kz;
        const V3 kv{kx * kw[0], ky * kw[1], kz * kw[2]};
        const double kk = norm(kv);
        const double E = std::pow(kk, 4) * std::exp(-2.0 * (kk / k0) * (kk / k0));
        const double a = std::sqrt(E / (4.0 * M_PI * kk * kk));
        const V3 kh = (1.0 / kk) * kv;
        V3 r{2 * uniform01(seed, 5, idx) - 1, 2 * uniform01(seed, 5, idx + 1) - 1, 2 * uniform01(seed, 5, idx + 2) - 1};
        V3 e1 = r - dot(r, kh) * kh;
        if (norm(e1) < 1e-6) e1 = cross(kh, V3{0.6, 0.0, 0.8});
        e1 = (a / norm(e1)) * e1;
        const V3 e2 = cross(kh, e1);
        const double f1 = 2 * M_PI * uniform01(seed, 5, idx + 3), f2 = 2 * M_PI * uniform01(seed, 5, idx + 4);
        idx += 5;
        for (int d = 0; d < 3; ++d) md.e1[d] = e1[d], md.e2[d] = e2[d];
        md.c1 = std::cos(f1), md.s1 = std::sin(f1), md.c2 = std::cos(f2), md.s2 = std::sin(f2);
        modes.push_back(md);
      }
  std::vector<double> vel(static_cast<size_t>(n) * 3);
  parallel_for(n, n_threads, [&](int64_t a0, int64_t a1) {
    std::vector<double> cr(3 * (2 * km + 1)), ci(3 * (2 * km + 1));
    for (int64_t c = a0; c < a1; ++c) {
      for (int d = 0; d < 3; ++d)
        for (int k = -km; k <= km; ++k) {
          const double ph = k * kw[d] * m.cell_centroid[3 * c + d];
          cr[d * (2 * km + 1) + k + km] = std::cos(ph);
          ci[d * (2 * km + 1) + k + km] = std::sin(ph);
        }
      double u[3] = {0, 0, 0};
      for (const Mode& md : modes) {
        const int ix = md.k[0] + km, iy = (2 * km + 1) + md.k[1] + km, iz = 2 * (2 * km + 1) + md.k[2] + km;
        const double xr = cr[ix] * cr[iy] - ci[ix] * ci[iy], xi = cr[ix] * ci[iy] + ci[ix] * cr[iy];
        const double zr = xr * cr[iz] - xi * ci[iz], zi = xr * ci[iz] + xi * cr[iz];
        const double a1 = zr * md.c1 - zi * md.s1, a2 = zr * md.c2 - zi * md.s2;  // cos(k.x + f)
        for (int d = 0; d < 3; ++d) u[d] += md.e1[d] * a1 + md.e2[d] * a2;
      }
      for (int d = 0; d < 3; ++d) vel[3 * c + d] = u[d];
    }
  });
  double s2 = 0.0, sv = 0.0;
  for (int64_t c = 0; c < n; ++c) {
    s2 += m.cell_volume[c] * (vel[3 * c] * vel[3 * c] + vel[3 * c + 1] * vel[3 * c + 1] + vel[3 * c + 2] * vel[3 * c + 2]);
    sv += m.cell_volume[c];
  }
  const double p0 = 1.0 / g;  // rho = 1, sound speed 1
  const double scale = mach / std::sqrt(s2 / sv);
  parallel_for(n, n_threads, [&](int64_t a0, int64_t a1) {
    for (int64_t c = a0; c < a1; ++c)
      prim_to_cons5(1.0, scale * vel[3 * c], scale * vel[3 * c + 1], scale * vel[3 * c + 2], p0, g, &u_out[5 * c]);
  });
}

}  // namespace ucfvb
