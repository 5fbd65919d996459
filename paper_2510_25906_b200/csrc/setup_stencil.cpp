// Operator precompute on the host: per cell the central
// BFS stencil, least-squares pseudo-inverses (full and r=1), directional
// sector stencils with their r=1 pseudo-inverses, the oscillation-indicator
// matrix and the basis values at the cell's face quadrature points.
// Restates /root/reference/proj/src/stencil.cpp:31-284 and basis.cpp:12-137
// with the same arithmetic; cells are processed in parallel with
// per-thread scratch. The QR is a column-pivoting Householder
// factorisation (the algorithm of Eigen's ColPivHouseholderQR, which the
// reference calls at stencil.cpp:152-166).
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "geom.hpp"
#include "layout.hpp"
#include "setup.hpp"

struct ucfvb_stencils {
  int order = 1, K = 0, nq = 1, si = 0, n = 0;
  std::vector<int64_t> central_ptr, pinv_off, pinv_lin_off, dir_ptr, dir_member_ptr, pinv_dir_off, qp_ptr, phi_off;
  std::vector<int32_t> central, dir_members, qp_slot;
  std::vector<double> pinv, pinv_lin, pinv_dir, oi, phi;
};

namespace ucfvb {

double uniform01(uint64_t seed, uint64_t stream, uint64_t idx);

namespace {

// ---- Legendre-product basis (basis.cpp) -------------------------------------
std::vector<double> legendre(int n) {
  std::vector<std::vector<double>> p(n + 1);
  p[0] = {1.0};
  if (n >= 1) p[1] = {0.0, 1.0};
  for (int m = 1; m < n; ++m) {
    std::vector<double> nx(m + 2, 0.0);
    for (int i = 0; i <= m; ++i) nx[i + 1] += (2.0 * m + 1.0) * p[m][i] / (m + 1.0);
    for (int i = 0; i < m; ++i) nx[i] -= m * p[m - 1][i] / (m + 1.0);
    p[m + 1] = std::move(nx);
  }
  return p[n];
}

struct Family {
  int r = 1, K = 0, nm = 0;         // order, functions, monomials (r+1)^2
  std::vector<double> c;            // K x nm dense coefficients, c[k][i*(r+1)+j] on xi^i eta^j
  std::vector<std::array<int, 2>> beta;
  std::vector<double> dc;           // nbeta x K x nm derivative coefficients

  explicit Family(int order) : r(order), nm((order + 1) * (order + 1)) {
    std::vector<std::vector<double>> leg(r + 1);
    for (int i = 0; i <= r; ++i) leg[i] = legendre(i);
    for (int t = 1; t <= r; ++t)
      for (int i = t; i >= 0; --i) {
        const int j = t - i;
        std::vector<double> f(nm, 0.0);
        for (size_t a = 0; a < leg[i].size(); ++a)
          for (size_t b = 0; b < leg[j].size(); ++b) f[a * (r + 1) + b] += leg[i][a] * leg[j][b];
        c.insert(c.end(), f.begin(), f.end());
        ++K;
      }
    for (int t = 1; t <= r; ++t)
      for (int bx = t; bx >= 0; --bx) beta.push_back({bx, t - bx});
    dc.assign(beta.size() * K * nm, 0.0);
    for (size_t b = 0; b < beta.size(); ++b)
      for (int k = 0; k < K; ++k)
        for (int i = beta[b][0]; i <= r; ++i)
          for (int j = beta[b][1]; j <= r; ++j) {
            double f = 1.0;
            for (int t = 0; t < beta[b][0]; ++t) f *= static_cast<double>(i - t);
            for (int t = 0; t < beta[b][1]; ++t) f *= static_cast<double>(j - t);
            dc[(b * K + k) * nm + (i - beta[b][0]) * (r + 1) + (j - beta[b][1])] = c[k * nm + i * (r + 1) + j] * f;
          }
  }

  void monomials(const Vec2& p, double* mono) const {
    double xp = 1.0;
    for (int i = 0; i <= r; ++i) {
      double yp = xp;
      for (int j = 0; j <= r; ++j) {
        mono[i * (r + 1) + j] = yp;
        yp *= p.y;
      }
      xp *= p.x;
    }
  }
  // dense evaluation of every psi_k (MonomialFamily::eval_all)
  void eval_all(const Vec2& p, double* out) const {
    double mono[100];
    monomials(p, mono);
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (int m = 0; m < nm; ++m) s += c[k * nm + m] * mono[m];
      out[k] = s;
    }
  }
  void eval_all_derivative(int b, const Vec2& p, double* out) const {
    double mono[100];
    monomials(p, mono);
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (int m = 0; m < nm; ++m) s += dc[(b * K + k) * nm + m] * mono[m];
      out[k] = s;
    }
  }
  // Horner evaluation of one psi_k (Poly2::eval, polynomial.hpp:19-27)
  double horner(int k, const Vec2& p) const {
    double acc = 0.0;
    for (int i = r; i >= 0; --i) {
      double row = 0.0;
      for (int j = r; j >= 0; --j) row = row * p.y + c[k * nm + i * (r + 1) + j];
      acc = acc * p.x + row;
    }
    return acc;
  }
};

// ---- least squares ---------------------------------------------------------
// Column-pivoting Householder QR of the row-major rows x cols matrix `A`;
// returns false when rank < cols (stencil.cpp:157-160), else writes the
// cols x rows least-squares pseudo-inverse (solution of A X = I) to `pinv`.
bool lsq_pinv(const std::vector<double>& A, int rows, int cols, std::vector<double>& pinv) {
  // column-major working copy
  std::vector<double> q(static_cast<size_t>(rows) * cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) q[j * rows + i] = A[static_cast<size_t>(i) * cols + j];
  auto at = [&](int i, int j) -> double& { return q[static_cast<size_t>(j) * rows + i]; };
  const int size = std::min(rows, cols);
  std::vector<double> tau(size, 0.0), nu(cols), nd(cols);
  std::vector<int> perm(cols);
  auto colnorm = [&](int j, int r0) {
    double s = 0.0;
    for (int i = r0; i < rows; ++i) s += at(i, j) * at(i, j);
    return std::sqrt(s);
  };
  for (int j = 0; j < cols; ++j) {
    perm[j] = j;
    nd[j] = nu[j] = colnorm(j, 0);
  }
  double maxn = 0.0;
  for (int j = 0; j < cols; ++j) maxn = nu[j] > maxn ? nu[j] : maxn;
  const double eps = std::numeric_limits<double>::epsilon();
  const double thr_help = (maxn * eps) * (maxn * eps) / static_cast<double>(rows);
  const double downdate = std::sqrt(eps);
  int nzp = size;
  double maxpiv = 0.0;
  auto reflect = [&](int k, int j0, int j1, std::vector<double>& m, int mrows) {
    // m is column-major with mrows rows
    auto mm = [&](int i, int j) -> double& { return m[static_cast<size_t>(j) * mrows + i]; };
    const double t = tau[k];
    if (rows - k == 1) {
      for (int j = j0; j < j1; ++j) mm(k, j) *= (1.0 - t);
      return;
    }
    if (t == 0.0) return;
    for (int j = j0; j < j1; ++j) {
      double s = 0.0;
      for (int i = k + 1; i < rows; ++i) s += at(i, k) * mm(i, j);
      s += mm(k, j);
      mm(k, j) -= t * s;
      for (int i = k + 1; i < rows; ++i) mm(i, j) -= t * at(i, k) * s;
    }
  };
  for (int k = 0; k < size; ++k) {
    int big = k;
    for (int j = k + 1; j < cols; ++j)
      if (nu[j] > nu[big]) big = j;
    if (nzp == size && nu[big] * nu[big] < thr_help * static_cast<double>(rows - k)) nzp = k;
    if (big != k) {
      for (int i = 0; i < rows; ++i) std::swap(at(i, k), at(i, big));
      std::swap(nu[k], nu[big]);
      std::swap(nd[k], nd[big]);
      std::swap(perm[k], perm[big]);
    }
    double tail = 0.0;
    for (int i = k + 1; i < rows; ++i) tail += at(i, k) * at(i, k);
    const double c0 = at(k, k);
    double beta;
    if (tail <= std::numeric_limits<double>::min()) {
      tau[k] = 0.0;
      beta = c0;
      for (int i = k + 1; i < rows; ++i) at(i, k) = 0.0;
    } else {
      beta = std::sqrt(c0 * c0 + tail);
      if (c0 >= 0.0) beta = -beta;
      for (int i = k + 1; i < rows; ++i) at(i, k) /= (c0 - beta);
      tau[k] = (beta - c0) / beta;
    }
    at(k, k) = beta;
    if (std::abs(beta) > maxpiv) maxpiv = std::abs(beta);
    reflect(k, k + 1, cols, q, rows);
    for (int j = k + 1; j < cols; ++j) {
      if (nu[j] != 0.0) {
        double t = std::abs(at(k, j)) / nu[j];
        t = (1.0 + t) * (1.0 - t);
        if (t < 0.0) t = 0.0;
        const double rr = nu[j] / nd[j];
        if (t * rr * rr <= downdate) {
          nd[j] = colnorm(j, k + 1);
          nu[j] = nd[j];
        } else {
          nu[j] *= std::sqrt(t);
        }
      }
    }
  }
  // rank with Eigen's default threshold (diag size * eps * |max pivot|)
  const double premult = std::abs(maxpiv) * (static_cast<double>(size) * eps);
  int rank = 0;
  for (int i = 0; i < nzp; ++i) rank += std::abs(at(i, i)) > premult;
  if (rank < cols) return false;
  // X = P R^-1 Q^T I
  std::vector<double> b(static_cast<size_t>(rows) * rows, 0.0);  // column-major identity
  for (int i = 0; i < rows; ++i) b[static_cast<size_t>(i) * rows + i] = 1.0;
  for (int k = 0; k < nzp; ++k) reflect(k, 0, rows, b, rows);
  auto bb = [&](int i, int j) -> double& { return b[static_cast<size_t>(j) * rows + i]; };
  for (int j = 0; j < rows; ++j)
    for (int i = nzp - 1; i >= 0; --i) {
      double s = bb(i, j);
      for (int t = i + 1; t < nzp; ++t) s -= at(i, t) * bb(t, j);
      bb(i, j) = s / at(i, i);
    }
  pinv.assign(static_cast<size_t>(cols) * rows, 0.0);
  for (int i = 0; i < nzp; ++i)
    for (int j = 0; j < rows; ++j) pinv[static_cast<size_t>(perm[i]) * rows + j] = bb(i, j);
  return true;
}

struct Entry {
  int cell, px, py;
};

struct Builder {
  const ucfvb_mesh_view& m;
  const Family& fam;
  int order, K, nq, si;

  Vec2 centroid(int c) const { return {m.cell_centroid[2 * c], m.cell_centroid[2 * c + 1]}; }
  Vec2 vertex(int v) const { return {m.vertices[2 * v], m.vertices[2 * v + 1]}; }
  Vec2 entry_centroid(const Entry& e) const {
    return centroid(e.cell) + Vec2{e.px * m.period_x, e.py * m.period_y};
  }

  // member polygon in the target cell's reference frame (stencil.cpp:119-127)
  void member_poly(int target, const Entry& e, std::vector<Vec2>& poly) const {
    const Vec2 shift{e.px * m.period_x, e.py * m.period_y};
    const Vec2 ct = centroid(target);
    const double h = m.cell_h[target];
    poly.clear();
    for (int i = m.cell_vtx_ptr[e.cell]; i < m.cell_vtx_ptr[e.cell + 1]; ++i)
      poly.push_back((vertex(m.cell_vtx[i]) + shift - ct) / h);
  }

  // breadth-first central stencil, rings sorted by centroid distance (stencil.cpp:31-71)
  void central_stencil(int cell, int M, std::vector<Entry>& st) const {
    const Vec2 origin = centroid(cell);
    st.assign(1, {cell, 0, 0});
    std::vector<Entry> visited{{cell, 0, 0}}, ring{{cell, 0, 0}}, next;
    std::vector<std::pair<double, Entry>> keyed;
    auto seen = [&](const Entry& e) {
      for (const Entry& v : visited)
        if (v.cell == e.cell && v.px == e.px && v.py == e.py) return true;
      return false;
    };
    while (static_cast<int>(st.size()) < M + 1) {
      next.clear();
      for (const Entry& e : ring) {
        for (int i = m.cell_face_ptr[e.cell]; i < m.cell_face_ptr[e.cell + 1]; ++i) {
          const int f = m.cell_faces[i];
          Entry nb;
          if (m.face_right[f] >= 0) {
            nb = {m.face_left[f] == e.cell ? m.face_right[f] : m.face_left[f], e.px, e.py};
          } else if (m.face_partner[f] >= 0) {
            nb = {m.face_left[m.face_partner[f]], e.px + m.face_shift[2 * f], e.py + m.face_shift[2 * f + 1]};
          } else {
            continue;
          }
          if (!seen(nb)) {
            visited.push_back(nb);
            next.push_back(nb);
          }
        }
      }
      if (next.empty())
        throw ApiError(UCFVB_INVALID, "stencil for cell " + std::to_string(cell) + ": mesh too small for " +
                                          std::to_string(M + 1) + " cells");
      keyed.clear();
      for (const Entry& e : next) keyed.push_back({norm(entry_centroid(e) - origin), e});
      std::sort(keyed.begin(), keyed.end(), [](const auto& a, const auto& b) {
        if (a.first != b.first) return a.first < b.first;
        if (a.second.cell != b.second.cell) return a.second.cell < b.second.cell;
        if (a.second.px != b.second.px) return a.second.px < b.second.px;
        return a.second.py < b.second.py;
      });
      for (size_t i = 0; i < keyed.size(); ++i) {
        next[i] = keyed[i].second;
        if (static_cast<int>(st.size()) < M + 1) st.push_back(keyed[i].second);
      }
      ring.swap(next);
    }
  }

  // one directional stencil per face (stencil.cpp:73-117)
  void directional(int cell, const std::vector<Entry>& central, int m_dir, std::vector<std::vector<int>>& out) const {
    const Vec2 origin = centroid(cell);
    const int M = static_cast<int>(central.size()) - 1;
    std::vector<Vec2> dir(M);
    std::vector<double> dist(M);
    for (int i = 0; i < M; ++i) {
      dir[i] = entry_centroid(central[i + 1]) - origin;
      dist[i] = norm(dir[i]);
    }
    std::vector<int> by(M);
    for (int i = 0; i < M; ++i) by[i] = i;
    std::sort(by.begin(), by.end(), [&](int a, int b) {
      if (dist[a] != dist[b]) return dist[a] < dist[b];
      return a < b;
    });
    out.clear();
    for (int i = m.cell_face_ptr[cell]; i < m.cell_face_ptr[cell + 1]; ++i) {
      const int f = m.cell_faces[i];
      Vec2 a = vertex(m.face_vtx[2 * f]) - origin;
      Vec2 b = vertex(m.face_vtx[2 * f + 1]) - origin;
      if (m.face_left[f] != cell) std::swap(a, b);
      std::vector<int> mem{0};
      for (int idx : by) {
        if (static_cast<int>(mem.size()) > m_dir) break;
        if (cross(a, dir[idx]) >= 0.0 && cross(dir[idx], b) >= 0.0) mem.push_back(idx + 1);
      }
      for (int idx : by) {
        if (static_cast<int>(mem.size()) > m_dir) break;
        if (std::find(mem.begin(), mem.end(), idx + 1) == mem.end()) mem.push_back(idx + 1);
      }
      out.push_back(std::move(mem));
    }
  }

  // LSQ rows: member-averaged basis differences (stencil.cpp:129-150)
  void lsq_rows(int cell, const std::vector<Entry>& members, const std::vector<double>& means, int ncols,
                std::vector<double>& A) const {
    const int rows = static_cast<int>(members.size()) - 1;
    A.assign(static_cast<size_t>(rows) * ncols, 0.0);
    std::vector<Vec2> poly;
    std::vector<QPoint> qp;
    double psi[64];
    for (int r = 0; r < rows; ++r) {
      member_poly(cell, members[r + 1], poly);
      const double area = polygon_signed_area(poly);
      polygon_rule(poly, order, qp);
      double* row = &A[static_cast<size_t>(r) * ncols];
      for (const QPoint& q : qp) {
        fam.eval_all(q.p, psi);
        for (int k = 0; k < ncols; ++k) row[k] += q.w * (psi[k] - means[k]);
      }
      for (int k = 0; k < ncols; ++k) row[k] /= area;
    }
  }
};

}  // namespace

bool qr_pinv(const std::vector<double>& A, int rows, int cols, std::vector<double>& pinv) {
  return lsq_pinv(A, rows, cols, pinv);
}

ucfvb_stencils* build_stencils(const ucfvb_mesh_view& m, int order, int si_exponent, int n_threads) {
  if (order < 1) throw ApiError(UCFVB_INVALID, "build_stencils: order must be >= 1");
  if (order > 8) throw ApiError(UCFVB_INVALID, "build_stencils: order must be <= 8");
  auto S = std::make_unique<ucfvb_stencils>();
  const Family fam(order);
  const int n = m.n_cells;
  const int K = fam.K;
  const int nq = (order + 2) / 2;
  S->order = order;
  S->K = K;
  S->nq = nq;
  S->si = si_exponent;
  S->n = n;
  if (m.n_faces > 0 && m.n_qp != nq)
    throw ApiError(UCFVB_INVALID, "solver: mesh was built with " + std::to_string(m.n_qp) +
                                      " face quadrature points but order " + std::to_string(order) + " needs " +
                                      std::to_string(nq));
  const int M_target = 2 * K;
  const int m_dir = 4;
  Builder B{m, fam, order, K, nq, si_exponent};

  // per-cell results, concatenated afterwards in cell order
  struct CellOut {
    std::vector<int32_t> central;  // 3 per entry
    std::vector<double> pinv, pinv_lin, oi, phi;
    std::vector<std::vector<int>> dir;
    std::vector<std::vector<double>> pinv_dir;
    std::vector<int32_t> slots;
  };
  S->central_ptr.assign(1, 0);
  S->pinv_off.assign(1, 0);
  S->pinv_lin_off.assign(1, 0);
  S->dir_ptr.assign(1, 0);
  S->dir_member_ptr.assign(1, 0);
  S->pinv_dir_off.assign(1, 0);
  S->qp_ptr.assign(1, 0);
  S->phi_off.assign(1, 0);
  // cells are built in blocks (parallel inside a block) and appended in cell
  // order, so peak memory is the final arrays plus one block of scratch
  const int64_t block = std::max<int64_t>(4096, 1 << 16);
  std::vector<CellOut> outs;
  for (int64_t b0 = 0; b0 < n; b0 += block) {
  const int64_t b1 = std::min<int64_t>(n, b0 + block);
  outs.assign(static_cast<size_t>(b1 - b0), CellOut{});

  parallel_for(b1 - b0, n_threads, [&](int64_t a0, int64_t a1) {
    a0 += b0;
    a1 += b0;
    std::vector<Entry> central;
    std::vector<double> A, A1, pinv, pl, pd;
    std::vector<Vec2> ref_poly;
    std::vector<QPoint> qp;
    std::vector<std::vector<int>> dirs;
    double d[64], psi[64];
    for (int c = static_cast<int>(a0); c < static_cast<int>(a1); ++c) {
      CellOut& o = outs[c - b0];
      B.member_poly(c, {c, 0, 0}, ref_poly);
      // basis means over the reference cell (build_basis, basis.cpp:125-137)
      const double rarea = polygon_signed_area(ref_poly);
      if (!(rarea > 0.0)) throw ApiError(UCFVB_INVALID, "build_basis: cell polygon must be CCW with positive area");
      polygon_rule(ref_poly, 2 * order, qp);
      std::vector<double> means(K);
      for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (const QPoint& q : qp) s += q.w * fam.horner(k, q.p);
        means[k] = s / rarea;
      }
      // central stencil with rank-deficiency retries (stencil.cpp:206-230)
      int M = M_target;
      for (int attempt = 0;; ++attempt) {
        B.central_stencil(c, M, central);
        B.lsq_rows(c, central, means, K, A);
        bool ok = lsq_pinv(A, M, K, pinv);
        if (ok) {
          A1.assign(static_cast<size_t>(M) * 2, 0.0);
          for (int r = 0; r < M; ++r) {
            A1[r * 2 + 0] = A[static_cast<size_t>(r) * K + 0];
            A1[r * 2 + 1] = A[static_cast<size_t>(r) * K + 1];
          }
          ok = lsq_pinv(A1, M, 2, pl);
        }
        if (ok) break;
        if (attempt >= 2)
          throw ApiError(UCFVB_INVALID, "reconstruction stencil for cell " + std::to_string(c) + " is rank-deficient");
        M += std::max(4, M / 2);
      }
      const int Mf = static_cast<int>(central.size()) - 1;
      for (const Entry& e : central) {
        o.central.push_back(e.cell);
        o.central.push_back(e.px);
        o.central.push_back(e.py);
      }
      o.pinv = pinv;
      o.pinv_lin = pl;
      // directional stencils, grown past m_dir when a sector system is singular (:232-258)
      B.directional(c, central, m_dir, dirs);
      for (auto& mem : dirs) {
        int take = static_cast<int>(mem.size());
        for (;; ++take) {
          std::vector<Entry> sub;
          for (int i = 0; i < std::min(take, static_cast<int>(mem.size())); ++i) sub.push_back(central[mem[i]]);
          const int rows = static_cast<int>(sub.size()) - 1;
          B.lsq_rows(c, sub, means, 2, A);
          if (lsq_pinv(A, rows, 2, pd)) {
            o.pinv_dir.push_back(pd);
            mem.resize(sub.size());
            break;
          }
          if (take >= Mf + 1)
            throw ApiError(UCFVB_INVALID, "reconstruction stencil for cell " + std::to_string(c) + " is rank-deficient");
          for (int cand = 1; cand <= Mf; ++cand)
            if (std::find(mem.begin(), mem.end(), cand) == mem.end()) {
              mem.push_back(cand);
              break;
            }
        }
      }
      o.dir = dirs;
      // oscillation-indicator matrix (stencil.cpp:168-190)
      o.oi.assign(static_cast<size_t>(K) * K, 0.0);
      polygon_rule(ref_poly, 2 * (order > 0 ? order : 1), qp);
      const double hc = m.cell_h[c];
      for (size_t b = 0; b < fam.beta.size(); ++b) {
        const int bt = fam.beta[b][0] + fam.beta[b][1];
        const double hp = si_exponent == 0 ? std::pow(std::abs(hc), bt - 1) : std::pow(std::abs(hc), 2 * bt - 2);
        for (const QPoint& q : qp) {
          fam.eval_all_derivative(static_cast<int>(b), q.p, d);
          const double w = q.w * hp;
          for (int k = 0; k < K; ++k) {
            const double wk = w * d[k];
            for (int l = 0; l < K; ++l) o.oi[static_cast<size_t>(k) * K + l] += wk * d[l];
          }
        }
      }
      // phi at the cell's own face quadrature points + value slots (:262-281)
      const Vec2 ct = B.centroid(c);
      for (int i = m.cell_face_ptr[c]; i < m.cell_face_ptr[c + 1]; ++i) {
        const int f = m.cell_faces[i];
        const int side = m.face_left[f] == c ? 0 : 1;
        for (int q = 0; q < nq; ++q) {
          const Vec2 p{m.face_qp[2 * (f * nq + q)], m.face_qp[2 * (f * nq + q) + 1]};
          const Vec2 xi = (p - ct) / hc;
          fam.eval_all(xi, psi);
          for (int k = 0; k < K; ++k) o.phi.push_back(psi[k] - means[k]);
          o.slots.push_back((f * nq + q) * 2 + side);
        }
      }
    }
  });

  for (auto& o : outs) {
    S->central.insert(S->central.end(), o.central.begin(), o.central.end());
    S->central_ptr.push_back(static_cast<int64_t>(S->central.size() / 3));
    S->pinv.insert(S->pinv.end(), o.pinv.begin(), o.pinv.end());
    S->pinv_off.push_back(static_cast<int64_t>(S->pinv.size()));
    S->pinv_lin.insert(S->pinv_lin.end(), o.pinv_lin.begin(), o.pinv_lin.end());
    S->pinv_lin_off.push_back(static_cast<int64_t>(S->pinv_lin.size()));
    for (size_t s = 0; s < o.dir.size(); ++s) {
      S->dir_members.insert(S->dir_members.end(), o.dir[s].begin(), o.dir[s].end());
      S->dir_member_ptr.push_back(static_cast<int64_t>(S->dir_members.size()));
      S->pinv_dir.insert(S->pinv_dir.end(), o.pinv_dir[s].begin(), o.pinv_dir[s].end());
      S->pinv_dir_off.push_back(static_cast<int64_t>(S->pinv_dir.size()));
    }
    S->dir_ptr.push_back(static_cast<int64_t>(S->dir_member_ptr.size() - 1));
    S->oi.insert(S->oi.end(), o.oi.begin(), o.oi.end());
    S->phi.insert(S->phi.end(), o.phi.begin(), o.phi.end());
    S->phi_off.push_back(static_cast<int64_t>(S->phi.size()));
    S->qp_slot.insert(S->qp_slot.end(), o.slots.begin(), o.slots.end());
    S->qp_ptr.push_back(static_cast<int64_t>(S->qp_slot.size()));
    o = CellOut{};
  }
  }  // blocks
  return S.release();
}

ucfvb_stencil_view stencils_view(const ucfvb_stencils* S) {
  ucfvb_stencil_view v{};
  v.order = S->order;
  v.K = S->K;
  v.n_qp = S->nq;
  v.si_exponent = S->si;
  v.n_cells = S->n;
  v.n_dir_stencils = static_cast<int32_t>(S->dir_member_ptr.size() - 1);
  v.central_ptr = S->central_ptr.data();
  v.central = S->central.data();
  v.pinv_off = S->pinv_off.data();
  v.pinv = S->pinv.data();
  v.pinv_lin_off = S->pinv_lin_off.data();
  v.pinv_lin = S->pinv_lin.data();
  v.dir_ptr = S->dir_ptr.data();
  v.dir_member_ptr = S->dir_member_ptr.data();
  v.dir_members = S->dir_members.data();
  v.pinv_dir_off = S->pinv_dir_off.data();
  v.pinv_dir = S->pinv_dir.data();
  v.oi = S->oi.data();
  v.qp_ptr = S->qp_ptr.data();
  v.phi_off = S->phi_off.data();
  v.phi = S->phi.data();
  v.qp_slot = S->qp_slot.data();
  return v;
}

void stencils_free(ucfvb_stencils* s) { delete s; }

// ---- initial conditions (cases.cpp:14-76 and BASELINE.json configs 1-3) ----
namespace {

void prim_to_cons(double rho, double u, double v, double p, double g, double* s) {
  s[0] = rho;
  s[1] = rho * u;
  s[2] = rho * v;
  s[3] = p / (g - 1.0) + 0.5 * rho * (u * u + v * v);
}

// ic_vortex (cases.cpp:14-27)
void ic_vortex(double x, double y, double g, double* s) {
  const double eps = 5.0;
  const double dx = x - 5.0, dy = y - 5.0;
  const double r2 = dx * dx + dy * dy;
  const double du = eps / (2.0 * M_PI) * std::exp(0.5 * (1.0 - r2)) * (-dy);
  const double dv = eps / (2.0 * M_PI) * std::exp(0.5 * (1.0 - r2)) * dx;
  const double dT = -(g - 1.0) * eps * eps / (8.0 * g * M_PI * M_PI) * std::exp(1.0 - r2);
  const double T = 1.0 + dT;
  const double rho = std::pow(T, 1.0 / (g - 1.0));
  const double pr = std::pow(T, g / (g - 1.0));
  prim_to_cons(rho, 1.0 + du, 1.0 + dv, pr, g, s);
}

}  // namespace

void project_initial(const ucfvb_mesh_view& m, int ic, const double* prm, int n_prm, uint64_t seed, int degree,
                     double g, int n_threads, double* u_out) {
  const int n = m.n_cells;
  double qs[4][4];
  if (ic == 0) {
  } else if (ic == 1) {
    if (n_prm < 7) throw ApiError(UCFVB_INVALID, "shock-sine IC needs 7 parameters");
  } else if (ic == 2) {
    if (n_prm < 3) throw ApiError(UCFVB_INVALID, "quadrant IC needs 3 parameters");
    for (int q = 0; q < 4; ++q) {
      const double rho = 0.1 + 1.4 * uniform01(seed, 1, 4 * q + 0);
      const double uu = -1.0 + 2.0 * uniform01(seed, 1, 4 * q + 1);
      const double vv = -1.0 + 2.0 * uniform01(seed, 1, 4 * q + 2);
      const double pp = 0.1 + 1.4 * uniform01(seed, 1, 4 * q + 3);
      prim_to_cons(rho, uu, vv, pp, g, qs[q]);
    }
  } else {
    throw ApiError(UCFVB_INVALID, "unknown initial condition " + std::to_string(ic));
  }
  const double sc = (ic == 0 && n_prm > 0) ? prm[0] : 1.0;
  parallel_for(n, n_threads, [&](int64_t a0, int64_t a1) {
    std::vector<Vec2> poly;
    std::vector<QPoint> qp;
    for (int c = static_cast<int>(a0); c < static_cast<int>(a1); ++c) {
      poly.clear();
      for (int i = m.cell_vtx_ptr[c]; i < m.cell_vtx_ptr[c + 1]; ++i)
        poly.push_back({m.vertices[2 * m.cell_vtx[i]], m.vertices[2 * m.cell_vtx[i] + 1]});
      polygon_rule(poly, degree, qp);
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (const QPoint& q : qp) {
        double s[4];
        if (ic == 0) {
          ic_vortex(sc * q.p.x, sc * q.p.y, g, s);
        } else if (ic == 1) {
          if (q.p.x < prm[0])
            prim_to_cons(prm[1], prm[2], prm[3], prm[4], g, s);
          else
            prim_to_cons(1.0 + prm[5] * std::sin(prm[6] * q.p.x), 0.0, 0.0, 1.0, g, s);
        } else {
          const int qi = (q.p.x >= prm[0] ? 1 : 0) + (q.p.y >= prm[1] ? 2 : 0);
          for (int v = 0; v < 4; ++v) s[v] = qs[qi][v];
        }
        for (int v = 0; v < 4; ++v) acc[v] += q.w * s[v];
      }
      for (int v = 0; v < 4; ++v) u_out[4 * static_cast<int64_t>(c) + v] = acc[v] / m.cell_area[c];
      if (ic == 2)
        for (int v = 0; v < 4; ++v)
          u_out[4 * static_cast<int64_t>(c) + v] *=
              1.0 + prm[2] * (2.0 * uniform01(seed, 2, 4 * static_cast<uint64_t>(c) + v) - 1.0);
    }
  });
}

}  // namespace ucfvb
