// ORACLE TEST INFRASTRUCTURE -- not product code. Only tests/, the smoke check
// and bench.py's CPU-baseline / reference legs load this library.
//
// Harness around the UNMODIFIED reference sources (/root/reference/proj/src/*.cpp,
// compiled by oracle/Makefile into oracle/_ref/libucfv_ref.so). It adds only
// what BASELINE.json needs and the reference lacks:
//   * jittered structured triangle meshes built through the reference's own
//     assemble_mesh + pair_periodic (mesh.cpp:32-97, 368-446),
//   * the three BASELINE initial conditions projected with the reference's
//     project_initial (cases.cpp:62-76),
//   * an SSP-RK3 (Shu-Osher) driver over the public Solver::compute_residual,
//   * flat C views of the reference's Mesh / StencilSet (include/ucfvb.h) so
//     the GPU path can consume byte-identical operator data,
//   * read access to per-stage intermediates (labels_, val_left_/val_right_,
//     dofs_, bounds_; private at solver.hpp:84-99).
// every standard header the reference headers pull in comes first, so the
// access-specifier override below touches only ucfv's own declarations
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

// intermediates of the stage pass are private members of ucfv::Solver
#define private public
#include "ucfv/solver.hpp"
#undef private
#include "ucfv/cases.hpp"
#include "ucfv/mesh.hpp"
#include "ucfv/quadrature.hpp"
#include "ucfv/run.hpp"
#include "ucfv/stencil.hpp"

#include "ucfvb.h"

using namespace ucfv;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const NonPhysicalError*>(&e)) return UCFVB_NONPHYSICAL;
  if (dynamic_cast<const std::invalid_argument*>(&e) || dynamic_cast<const MeshError*>(&e))
    return UCFVB_INVALID;
  // run_simulation-style wrapping keeps the NonPhysicalError text
  if (std::string(e.what()).find("non-physical") != std::string::npos) return UCFVB_NONPHYSICAL;
  return UCFVB_INVALID;
}

// splitmix64-based counter RNG shared (by definition, not by code) with the
// product's setup; U in [0,1) with 53 random bits.
double uniform01(uint64_t seed, uint64_t stream, uint64_t idx) {
  uint64_t z = seed + stream * 0xD1B54A32D192ED03ULL + (idx + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

// same rule as the file-static tag_rect_patches (mesh.cpp:119-135)
void tag_rect(Mesh& mesh, const Rect& dom) {
  mesh.patch_names = {"left", "right", "bottom", "top"};
  const double tol = 1e-9 * std::max(dom.width(), dom.height());
  for (Face& f : mesh.faces) {
    if (!f.is_boundary()) continue;
    if (std::abs(f.midpoint.x - dom.x0) < tol)
      f.patch = 0;
    else if (std::abs(f.midpoint.x - dom.x1) < tol)
      f.patch = 1;
    else if (std::abs(f.midpoint.y - dom.y0) < tol)
      f.patch = 2;
    else if (std::abs(f.midpoint.y - dom.y1) < tol)
      f.patch = 3;
  }
}

struct MeshHolder {
  Mesh mesh;
  // flat view storage
  std::vector<double> vertices, centroid, area, h, normal, length, midpoint, qp, qw;
  std::vector<int32_t> cvp, cv, cfp, cf, fvtx, fl, fr, patch, partner, shift, pqp;
  std::vector<const char*> pnames;
  ucfvb_mesh_view view{};

  void flatten() {
    const int nc = mesh.n_cells(), nf = mesh.n_faces();
    const int nq = nf ? static_cast<int>(mesh.faces[0].quad_points.size()) : 0;
    vertices.clear();
    for (const Vec2& v : mesh.vertices) {
      vertices.push_back(v.x);
      vertices.push_back(v.y);
    }
    cvp = {0};
    cfp = {0};
    cv.clear();
    cf.clear();
    centroid.clear();
    area.clear();
    h.clear();
    for (const Cell& c : mesh.cells) {
      for (int v : c.vertex_ids) cv.push_back(v);
      for (int f : c.face_ids) cf.push_back(f);
      cvp.push_back(static_cast<int32_t>(cv.size()));
      cfp.push_back(static_cast<int32_t>(cf.size()));
      centroid.push_back(c.centroid.x);
      centroid.push_back(c.centroid.y);
      area.push_back(c.area);
      h.push_back(c.h_c);
    }
    fvtx.clear(); fl.clear(); fr.clear(); normal.clear(); length.clear(); midpoint.clear();
    qp.clear(); qw.clear(); patch.clear(); partner.clear(); shift.clear(); pqp.clear();
    for (const Face& f : mesh.faces) {
      fvtx.push_back(f.vertex_ids[0]);
      fvtx.push_back(f.vertex_ids[1]);
      fl.push_back(f.left_cell);
      fr.push_back(f.right_cell);
      normal.push_back(f.normal.x);
      normal.push_back(f.normal.y);
      length.push_back(f.length);
      midpoint.push_back(f.midpoint.x);
      midpoint.push_back(f.midpoint.y);
      for (int q = 0; q < nq; ++q) {
        qp.push_back(f.quad_points[q].x);
        qp.push_back(f.quad_points[q].y);
        qw.push_back(f.quad_weights[q]);
        pqp.push_back(f.is_periodic() ? f.partner_qp[q] : -1);
      }
      patch.push_back(f.patch);
      partner.push_back(f.periodic_partner);
      shift.push_back(f.shift_ix);
      shift.push_back(f.shift_iy);
    }
    pnames.clear();
    for (const auto& s : mesh.patch_names) pnames.push_back(s.c_str());
    view = ucfvb_mesh_view{};
    view.n_vertices = static_cast<int32_t>(mesh.vertices.size());
    view.n_cells = nc;
    view.n_faces = nf;
    view.n_qp = nq;
    view.n_patches = static_cast<int32_t>(mesh.patch_names.size());
    view.period_x = mesh.period_x;
    view.period_y = mesh.period_y;
    view.vertices = vertices.data();
    view.cell_vtx_ptr = cvp.data();
    view.cell_vtx = cv.data();
    view.cell_face_ptr = cfp.data();
    view.cell_faces = cf.data();
    view.cell_centroid = centroid.data();
    view.cell_area = area.data();
    view.cell_h = h.data();
    view.face_vtx = fvtx.data();
    view.face_left = fl.data();
    view.face_right = fr.data();
    view.face_normal = normal.data();
    view.face_length = length.data();
    view.face_midpoint = midpoint.data();
    view.face_qp = qp.data();
    view.face_qw = qw.data();
    view.face_patch = patch.data();
    view.face_partner = partner.data();
    view.face_shift = shift.data();
    view.face_partner_qp = pqp.data();
    view.patch_names = pnames.data();
  }
};

struct StencilFlat {
  std::vector<int64_t> central_ptr, pinv_off, pinv_lin_off, dir_ptr, dir_member_ptr, pinv_dir_off,
      qp_ptr, phi_off;
  std::vector<int32_t> central, dir_members, qp_slot;
  std::vector<double> pinv, pinv_lin, pinv_dir, oi, phi;
  ucfvb_stencil_view view{};

  void flatten(const StencilSet& s) {
    const int n = static_cast<int>(s.cells.size());
    const int K = s.K;
    central_ptr = {0}; pinv_off = {0}; pinv_lin_off = {0}; dir_ptr = {0}; dir_member_ptr = {0};
    pinv_dir_off = {0}; qp_ptr = {0}; phi_off = {0};
    central.clear(); dir_members.clear(); qp_slot.clear();
    pinv.clear(); pinv_lin.clear(); pinv_dir.clear(); oi.clear(); phi.clear();
    for (int c = 0; c < n; ++c) {
      const CellStencil& cs = s.cells[c];
      for (const auto& e : cs.central) {
        central.push_back(e.cell);
        central.push_back(e.px);
        central.push_back(e.py);
      }
      central_ptr.push_back(static_cast<int64_t>(central.size() / 3));
      pinv.insert(pinv.end(), cs.pinv.begin(), cs.pinv.end());
      pinv_off.push_back(static_cast<int64_t>(pinv.size()));
      pinv_lin.insert(pinv_lin.end(), cs.pinv_linear.begin(), cs.pinv_linear.end());
      pinv_lin_off.push_back(static_cast<int64_t>(pinv_lin.size()));
      for (std::size_t d = 0; d < cs.directional.size(); ++d) {
        for (int m : cs.directional[d]) dir_members.push_back(m);
        dir_member_ptr.push_back(static_cast<int64_t>(dir_members.size()));
        pinv_dir.insert(pinv_dir.end(), cs.pinv_dir[d].begin(), cs.pinv_dir[d].end());
        pinv_dir_off.push_back(static_cast<int64_t>(pinv_dir.size()));
      }
      dir_ptr.push_back(static_cast<int64_t>(dir_member_ptr.size() - 1));
      if (static_cast<int>(cs.oi.size()) != K * K) throw std::logic_error("oi size");
      oi.insert(oi.end(), cs.oi.begin(), cs.oi.end());
      for (int sl : s.cell_qp_slot[c]) qp_slot.push_back(sl);
      qp_ptr.push_back(static_cast<int64_t>(qp_slot.size()));
      phi.insert(phi.end(), s.cell_phi[c].begin(), s.cell_phi[c].end());
      phi_off.push_back(static_cast<int64_t>(phi.size()));
    }
    view = ucfvb_stencil_view{};
    view.order = s.order;
    view.K = K;
    view.n_qp = s.n_qp;
    view.si_exponent = (s.si_exponent == SiExponent::Paper) ? 0 : 1;
    view.n_cells = n;
    view.n_dir_stencils = static_cast<int32_t>(dir_member_ptr.size() - 1);
    view.central_ptr = central_ptr.data();
    view.central = central.data();
    view.pinv_off = pinv_off.data();
    view.pinv = pinv.data();
    view.pinv_lin_off = pinv_lin_off.data();
    view.pinv_lin = pinv_lin.data();
    view.dir_ptr = dir_ptr.data();
    view.dir_member_ptr = dir_member_ptr.data();
    view.dir_members = dir_members.data();
    view.pinv_dir_off = pinv_dir_off.data();
    view.pinv_dir = pinv_dir.data();
    view.oi = oi.data();
    view.qp_ptr = qp_ptr.data();
    view.phi_off = phi_off.data();
    view.phi = phi.data();
    view.qp_slot = qp_slot.data();
  }
};

struct SolverHolder {
  std::shared_ptr<MeshHolder> mesh;  // Solver borrows the mesh (solver.hpp:84)
  std::unique_ptr<Solver> solver;
  StencilFlat flat;
  bool flat_ready = false;
  StateField scratch_a, scratch_b, scratch_r;
};

SolverOptions to_options(const ucfvb_options* o) {
  SolverOptions s;
  s.order = o->order;
  s.mode = static_cast<SchemeMode>(o->mode);
  s.limiter = static_cast<LimiterKind>(o->limiter);
  s.riemann = static_cast<RiemannKind>(o->riemann);
  s.margins.alpha_m = o->margins.alpha_m;
  s.margins.beta_m = o->margins.beta_m;
  s.margins.alpha_w = o->margins.alpha_w;
  s.margins.beta_w = o->margins.beta_w;
  s.margins.kappa = o->margins.kappa;
  s.margins.deact_n = o->margins.deact_n;
  s.lambda1p = o->lambda1p;
  s.weno_eps = o->weno_eps;
  s.weno_b = o->weno_b;
  s.cfl = o->cfl;
  s.venkat_kappa = o->venkat_kappa;
  s.si_exponent = (o->si_exponent == 0) ? SiExponent::Paper : SiExponent::Legacy;
  s.detect_every_stage = o->detect_every_stage != 0;
  s.gamma = o->gamma;
  return s;
}

// out = wa*ua + wb*ub + (wr*dt)*r  -- the reference's combine2 (time_integrator.cpp:31-38)
void combine2(StateField& out, double wa, const StateField& ua, double wb, const StateField& ub,
              double wr, const StateField& r, double dt) {
  const std::size_t n = ua.size();
  out.resize(n);
  const double wrdt = wr * dt;
  for (std::size_t i = 0; i < n; ++i)
    for (int v = 0; v < kNumVars; ++v) out[i][v] = wa * ua[i][v] + wb * ub[i][v] + wrdt * r[i][v];
}

// SSP-RK3 (Shu-Osher) step over the public RhsFn; stage times t, t+dt, t+dt/2.
void rk3_step(SolverHolder& h, double dt, double t) {
  Solver& s = *h.solver;
  s.stage_is_first_ = true;  // what Solver::advance does (solver.cpp:382)
  StateField& u = s.state();
  s.compute_residual(u, t, h.scratch_r);
  combine2(h.scratch_a, 1.0, u, 0.0, u, 1.0, h.scratch_r, dt);
  s.compute_residual(h.scratch_a, t + dt, h.scratch_r);
  combine2(h.scratch_b, 0.75, u, 0.25, h.scratch_a, 0.25, h.scratch_r, dt);
  s.compute_residual(h.scratch_b, t + 0.5 * dt, h.scratch_r);
  combine2(u, 1.0 / 3.0, u, 2.0 / 3.0, h.scratch_b, 2.0 / 3.0, h.scratch_r, dt);
}

State ic_shock_sine(const Vec2& p, const double* prm, double gamma) {
  if (p.x < prm[0]) return prim_to_cons({prm[1], prm[2], prm[3], prm[4]}, gamma);
  return prim_to_cons({1.0 + prm[5] * std::sin(prm[6] * p.x), 0.0, 0.0, 1.0}, gamma);
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

double ref_uniform01(uint64_t seed, uint64_t stream, uint64_t idx) {
  return uniform01(seed, stream, idx);
}

// jittered generate_structured_tri (mesh.cpp:137-157) -> assemble_mesh -> tags -> pair_periodic
int ref_mesh_structured_tri(int nx, int ny, double x0, double y0, double x1, double y1,
                            int diagonal, double jitter, uint64_t seed, int periodic_axis,
                            double tol, int nqp, void** out) {
  try {
    const Rect dom{x0, y0, x1, y1};
    std::vector<Vec2> verts;
    verts.reserve(static_cast<std::size_t>(nx + 1) * (ny + 1));
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i)
        verts.push_back({dom.x0 + dom.width() * i / nx, dom.y0 + dom.height() * j / ny});
    if (jitter != 0.0) {
      const double hx = dom.width() / nx, hy = dom.height() / ny;
      for (int j = 1; j < ny; ++j)
        for (int i = 1; i < nx; ++i) {
          const uint64_t v = static_cast<uint64_t>(j) * (nx + 1) + i;
          verts[v].x += jitter * hx * (2.0 * uniform01(seed, 0, 2 * v) - 1.0);
          verts[v].y += jitter * hy * (2.0 * uniform01(seed, 0, 2 * v + 1) - 1.0);
        }
    }
    auto vid = [&](int i, int j) { return j * (nx + 1) + i; };
    std::vector<std::vector<int>> cells;
    cells.reserve(2 * static_cast<std::size_t>(nx) * ny);
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int v00 = vid(i, j), v10 = vid(i + 1, j), v11 = vid(i + 1, j + 1), v01 = vid(i, j + 1);
        const bool flip = (diagonal == 1) && ((i + j) % 2 == 1);
        if (!flip) {
          cells.push_back({v00, v10, v11});
          cells.push_back({v00, v11, v01});
        } else {
          cells.push_back({v00, v10, v01});
          cells.push_back({v10, v11, v01});
        }
      }
    auto holder = std::make_shared<MeshHolder>();
    holder->mesh = assemble_mesh(std::move(verts), std::move(cells), nqp);
    tag_rect(holder->mesh, dom);
    if (periodic_axis == 1) holder->mesh = pair_periodic(std::move(holder->mesh), Axis::X, tol);
    if (periodic_axis == 2) holder->mesh = pair_periodic(std::move(holder->mesh), Axis::Y, tol);
    if (periodic_axis == 3) holder->mesh = pair_periodic(std::move(holder->mesh), Axis::Both, tol);
    holder->flatten();
    *out = new std::shared_ptr<MeshHolder>(holder);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// the reference generators as-is (for checking the jitter-free path)
int ref_mesh_generate_tri(int nx, int ny, double x0, double y0, double x1, double y1, int diagonal,
                          int periodic_axis, double tol, int nqp, void** out) {
  try {
    auto holder = std::make_shared<MeshHolder>();
    holder->mesh = generate_structured_tri(nx, ny, {x0, y0, x1, y1},
                                           diagonal ? DiagonalRule::Alternating : DiagonalRule::Uniform, nqp);
    if (periodic_axis == 1) holder->mesh = pair_periodic(std::move(holder->mesh), Axis::X, tol);
    if (periodic_axis == 2) holder->mesh = pair_periodic(std::move(holder->mesh), Axis::Y, tol);
    if (periodic_axis == 3) holder->mesh = pair_periodic(std::move(holder->mesh), Axis::Both, tol);
    holder->flatten();
    *out = new std::shared_ptr<MeshHolder>(holder);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_mesh_generate_quad(int nx, int ny, double x0, double y0, double x1, double y1,
                           int periodic_axis, double tol, int nqp, void** out) {
  try {
    auto holder = std::make_shared<MeshHolder>();
    holder->mesh = generate_structured_quad(nx, ny, {x0, y0, x1, y1}, nqp);
    if (periodic_axis == 1) holder->mesh = pair_periodic(std::move(holder->mesh), Axis::X, tol);
    if (periodic_axis == 2) holder->mesh = pair_periodic(std::move(holder->mesh), Axis::Y, tol);
    if (periodic_axis == 3) holder->mesh = pair_periodic(std::move(holder->mesh), Axis::Both, tol);
    holder->flatten();
    *out = new std::shared_ptr<MeshHolder>(holder);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_mesh_view(void* m, ucfvb_mesh_view* out) {
  *out = (*static_cast<std::shared_ptr<MeshHolder>*>(m))->view;
  return 0;
}

void ref_mesh_free(void* m) { delete static_cast<std::shared_ptr<MeshHolder>*>(m); }

// cell averages of the built-in ICs through the reference's project_initial
int ref_project_initial(void* m, int ic, const double* prm, int n_prm, uint64_t seed, int degree,
                        double gamma, double* u_out) {
  try {
    const Mesh& mesh = (*static_cast<std::shared_ptr<MeshHolder>*>(m))->mesh;
    StateField u;
    if (ic == 0) {
      const double sc = n_prm > 0 ? prm[0] : 1.0;
      u = project_initial(mesh, [&](const Vec2& p) { return ic_vortex({sc * p.x, sc * p.y}, gamma); },
                          degree);
    } else if (ic == 1) {
      if (n_prm < 7) throw std::invalid_argument("shock-sine IC needs 7 parameters");
      u = project_initial(mesh, [&](const Vec2& p) { return ic_shock_sine(p, prm, gamma); }, degree);
    } else if (ic == 2) {
      if (n_prm < 3) throw std::invalid_argument("quadrant IC needs 3 parameters");
      State qs[4];
      for (int q = 0; q < 4; ++q) {
        const double rho = 0.1 + 1.4 * uniform01(seed, 1, 4 * q + 0);
        const double uu = -1.0 + 2.0 * uniform01(seed, 1, 4 * q + 1);
        const double vv = -1.0 + 2.0 * uniform01(seed, 1, 4 * q + 2);
        const double pp = 0.1 + 1.4 * uniform01(seed, 1, 4 * q + 3);
        qs[q] = prim_to_cons({rho, uu, vv, pp}, gamma);
      }
      const double xs = prm[0], ys = prm[1], noise = prm[2];
      u = project_initial(mesh, [&](const Vec2& p) {
            const int q = (p.x >= xs ? 1 : 0) + (p.y >= ys ? 2 : 0);
            return qs[q];
          }, degree);
      for (int c = 0; c < mesh.n_cells(); ++c)
        for (int v = 0; v < kNumVars; ++v)
          u[c][v] *= 1.0 + noise * (2.0 * uniform01(seed, 2, 4 * static_cast<uint64_t>(c) + v) - 1.0);
    } else {
      throw std::invalid_argument("unknown initial condition " + std::to_string(ic));
    }
    std::memcpy(u_out, u.data(), u.size() * sizeof(State));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Solver(mesh, opt, bcs) with the reference's BC factories
int ref_solver_create(void* m, const ucfvb_options* o, const ucfvb_bc* bcs, int n_bcs, void** out) {
  try {
    auto h = std::make_unique<SolverHolder>();
    h->mesh = *static_cast<std::shared_ptr<MeshHolder>*>(m);
    std::map<std::string, BoundaryFn> fns;
    for (int i = 0; i < n_bcs; ++i) {
      const ucfvb_bc& b = bcs[i];
      if (b.kind == UCFVB_BC_OUTFLOW) fns[b.patch] = bc_outflow();
      else if (b.kind == UCFVB_BC_WALL) fns[b.patch] = bc_wall();
      else if (b.kind == UCFVB_BC_FIXED)
        fns[b.patch] = bc_fixed(State{b.state[0], b.state[1], b.state[2], b.state[3]});
    }
    h->solver = std::make_unique<Solver>(h->mesh->mesh, to_options(o), fns);
    *out = h.release();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_solver_free(void* s) { delete static_cast<SolverHolder*>(s); }

int ref_stencil_view(void* s, ucfvb_stencil_view* out) {
  auto* h = static_cast<SolverHolder*>(s);
  if (!h->flat_ready) {
    h->flat.flatten(h->solver->stencils());
    h->flat_ready = true;
  }
  *out = h->flat.view;
  return 0;
}

int ref_set_state(void* s, const double* u) {
  auto* h = static_cast<SolverHolder*>(s);
  StateField& st = h->solver->state();
  std::memcpy(st.data(), u, st.size() * sizeof(State));
  return 0;
}

int ref_get_state(void* s, double* u) {
  auto* h = static_cast<SolverHolder*>(s);
  const StateField& st = h->solver->state();
  std::memcpy(u, st.data(), st.size() * sizeof(State));
  return 0;
}

int ref_max_stable_dt(void* s, double* dt) {
  try {
    *dt = static_cast<SolverHolder*>(s)->solver->max_stable_dt();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Solver::compute_residual on a host field; stage_first < 0 leaves the flag alone
int ref_compute_residual(void* s, const double* u, double t, int stage_first, double* out) {
  try {
    auto* h = static_cast<SolverHolder*>(s);
    Solver& sv = *h->solver;
    if (stage_first >= 0) sv.stage_is_first_ = stage_first != 0;
    StateField uin(sv.mesh().n_cells());
    std::memcpy(uin.data(), u, uin.size() * sizeof(State));
    StateField r;
    sv.compute_residual(uin, t, r);
    std::memcpy(out, r.data(), r.size() * sizeof(State));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// one step: rk 0 = Solver::advance (SSPRK(5,4)); rk 1 = SSP-RK3 harness
int ref_advance(void* s, double dt, double t, int rk) {
  try {
    auto* h = static_cast<SolverHolder*>(s);
    if (rk == UCFVB_RK54)
      h->solver->advance(dt, t);
    else
      rk3_step(*h, dt, t);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// run_simulation's loop (run.cpp:97-132) for n_steps with t_end; census
// [n_steps][4] (nullable); returns wall seconds of the stepping loop.
int ref_run_steps(void* s, int n_steps, int rk, double t0, double t_end, double* t_out,
                  int64_t* census, double* wall_s) {
  try {
    auto* h = static_cast<SolverHolder*>(s);
    double t = t0;
    const auto w0 = std::chrono::steady_clock::now();
    for (int k = 0; k < n_steps; ++k) {
      const double dt = std::min(h->solver->max_stable_dt(), t_end - t);
      if (rk == UCFVB_RK54)
        h->solver->advance(dt, t);
      else
        rk3_step(*h, dt, t);
      t += dt;
      if (census) {
        int64_t* row = census + 4 * k;
        row[0] = row[1] = row[2] = row[3] = 0;
        for (Scheme sc : h->solver->step_labels()) ++row[static_cast<int>(sc)];
      }
    }
    if (wall_s)
      *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    if (t_out) *t_out = t;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// run_steps with each step's dt (run.cpp:99-112)
int ref_run_steps_log(void* s, int n_steps, int rk, double t0, double t_end, double* t_out, int64_t* census,
                      double* dts) {
  try {
    auto* h = static_cast<SolverHolder*>(s);
    double t = t0;
    for (int k = 0; k < n_steps; ++k) {
      const double dt = std::min(h->solver->max_stable_dt(), t_end - t);
      if (rk == UCFVB_RK54)
        h->solver->advance(dt, t);
      else
        rk3_step(*h, dt, t);
      t += dt;
      if (dts) dts[k] = dt;
      if (census) {
        int64_t* row = census + 4 * k;
        row[0] = row[1] = row[2] = row[3] = 0;
        for (Scheme sc : h->solver->step_labels()) ++row[static_cast<int>(sc)];
      }
    }
    if (t_out) *t_out = t;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// the reference's own output writers (run.cpp:160-213)
int ref_write_field_snapshot(void* m, const double* state, const uint8_t* labels, double gamma, const char* path) {
  try {
    const Mesh& mesh = (*static_cast<std::shared_ptr<MeshHolder>*>(m))->mesh;
    StateField u(mesh.n_cells());
    std::vector<Scheme> lab(mesh.n_cells());
    for (int c = 0; c < mesh.n_cells(); ++c) {
      for (int v = 0; v < 4; ++v) u[c][v] = state[4 * c + v];
      lab[c] = static_cast<Scheme>(labels[c]);
    }
    write_field_snapshot(mesh, u, lab, gamma, path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_write_census_csv(const ucfvb_census_row* rows, int n_rows, int n_cells, const char* path) {
  try {
    std::vector<CensusRow> r(n_rows);
    for (int i = 0; i < n_rows; ++i) {
      r[i].step = rows[i].step;
      r[i].t = rows[i].t;
      r[i].dt = rows[i].dt;
      for (int k = 0; k < 4; ++k) r[i].counts[k] = rows[i].counts[k];
    }
    write_census_csv(r, n_cells, path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_write_timing_csv(const ucfvb_timing_row* rows, int n_rows, const char* path) {
  try {
    std::vector<TimingRow> r(n_rows);
    for (int i = 0; i < n_rows; ++i) {
      r[i].step = rows[i].step;
      r[i].wall = rows[i].wall;
      r[i].phases.reconstruct = rows[i].reconstruct;
      r[i].phases.detect = rows[i].detect;
      r[i].phases.weights = rows[i].weights;
      r[i].phases.flux = rows[i].flux;
    }
    write_timing_csv(r, path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// taps -----------------------------------------------------------------------
int ref_get_labels(void* s, uint8_t* out, int which) {
  auto* h = static_cast<SolverHolder*>(s);
  const auto& lab = which ? h->solver->step_labels_ : h->solver->labels_;
  for (std::size_t i = 0; i < lab.size(); ++i) out[i] = static_cast<uint8_t>(lab[i]);
  return 0;
}

int ref_get_face_values(void* s, double* left, double* right) {
  auto* h = static_cast<SolverHolder*>(s);
  const auto& L = h->solver->val_left_;
  const auto& R = h->solver->val_right_;
  std::memcpy(left, L.data(), L.size() * sizeof(State));
  std::memcpy(right, R.data(), R.size() * sizeof(State));
  return 0;
}

int ref_get_dofs(void* s, double* out) {
  auto* h = static_cast<SolverHolder*>(s);
  const auto& d = h->solver->dofs_;
  std::memcpy(out, d.data(), d.size() * sizeof(double));
  return 0;
}

int ref_get_bounds(void* s, double* out) {
  auto* h = static_cast<SolverHolder*>(s);
  const auto& b = h->solver->bounds_;
  std::memcpy(out, b.data(), b.size() * sizeof(b[0]));
  return 0;
}

int ref_get_phase_times(void* s, double* out) {
  auto* h = static_cast<SolverHolder*>(s);
  const PhaseTimes& p = h->solver->phase_times();
  out[0] = p.reconstruct;
  out[1] = p.detect;
  out[2] = p.weights;
  out[3] = p.flux;
  return 0;
}

int ref_n_cells(void* s) { return static_cast<SolverHolder*>(s)->solver->mesh().n_cells(); }
int ref_n_faces(void* s) { return static_cast<SolverHolder*>(s)->solver->mesh().n_faces(); }
int ref_K(void* s) { return static_cast<SolverHolder*>(s)->solver->stencils().K; }
int ref_n_qp(void* s) { return static_cast<SolverHolder*>(s)->solver->n_qp(); }

// ---- reference point functions, for known-answer tests --------------------
int ref_compute_margins(const ucfvb_margins* m, double du, double* dm, double* dw) {
  NadMargins nm{m->alpha_m, m->beta_m, m->alpha_w, m->beta_w, m->kappa, m->deact_n};
  const Margins r = compute_margins(nm, du);
  *dm = r.delta_m;
  *dw = r.delta_w;
  return 0;
}

int ref_classify_violation(double v, double dm, double dw) {
  return static_cast<int>(classify_violation(v, Margins{dm, dw}));
}

int ref_deactivate_smooth(double du, double h, double kappa, double n) {
  return deactivate_smooth(du, h, kappa, n) ? 1 : 0;
}

double ref_limiter_bj(double u0, double lo, double hi, const double* q, int nq) {
  return limiter_barth_jespersen(u0, lo, hi, std::span<const double>(q, nq));
}

double ref_limiter_venkat(double u0, double lo, double hi, const double* q, int nq, double eps2) {
  return limiter_venkatakrishnan(u0, lo, hi, std::span<const double>(q, nq), eps2);
}

int ref_flux(const double* ul, const double* ur, double nx, double ny, double gamma, int kind,
             double* out) {
  try {
    const State L{ul[0], ul[1], ul[2], ul[3]}, R{ur[0], ur[1], ur[2], ur[3]};
    const State f = kind == 0 ? hllc_flux(L, R, {nx, ny}, gamma) : hll_flux(L, R, {nx, ny}, gamma);
    for (int v = 0; v < 4; ++v) out[v] = f[v];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

double ref_pow(double x, double y) { return std::pow(x, y); }

}  // extern "C"
