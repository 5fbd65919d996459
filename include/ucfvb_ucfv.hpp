// Reference-side binding: ucfv::GpuSolver, a drop-in for ucfv::Solver
// (/root/reference/proj/include/ucfv/solver.hpp:52-100) over the C ABI of
// ucfvb.h. Header-only; include it from code that already includes the
// reference headers and link libucfvb.so.
//
//   ucfv::Solver    s(mesh, opt, bcs);                 // reference, CPU
//   ucfv::GpuSolver g(mesh, opt, {{"left", UCFVB_BC_OUTFLOW}});  // B200
//   g.state() = project_initial(...);                  // same calls from here on
//   double dt = g.max_stable_dt(); g.advance(dt, t);   // SSPRK(5,4) like Solver::advance
//
// Differences a caller sees: boundary conditions are given as device BC kinds
// (outflow / wall / fixed state -- the reference's bc_outflow/bc_wall/bc_fixed)
// because an arbitrary std::function cannot run on the GPU; errors are the
// reference's exception types rebuilt from the ABI status codes.
#ifndef UCFVB_UCFV_HPP
#define UCFVB_UCFV_HPP

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "ucfv/solver.hpp"
#include "ucfvb.h"

namespace ucfv {

struct GpuBc {
  std::string patch;
  int kind;  // UCFVB_BC_OUTFLOW / UCFVB_BC_WALL / UCFVB_BC_FIXED
  State state{};
};

class GpuSolver {
 public:
  GpuSolver(const Mesh& mesh, SolverOptions opt, const std::vector<GpuBc>& bcs, int device = 0)
      : mesh_(mesh), opt_(opt), stencils_(build_stencils(mesh, opt.order, opt.si_exponent)) {
    flatten_mesh();
    flatten_stencils();
    ucfvb_options o;
    ucfvb_options_default(&o);
    o.order = opt.order;
    o.mode = static_cast<int32_t>(opt.mode);
    o.limiter = static_cast<int32_t>(opt.limiter);
    o.riemann = static_cast<int32_t>(opt.riemann);
    o.margins = {opt.margins.alpha_m, opt.margins.beta_m, opt.margins.alpha_w,
                 opt.margins.beta_w,  opt.margins.kappa,  opt.margins.deact_n};
    o.lambda1p = opt.lambda1p;
    o.weno_eps = opt.weno_eps;
    o.weno_b = opt.weno_b;
    o.cfl = opt.cfl;
    o.venkat_kappa = opt.venkat_kappa;
    o.si_exponent = opt.si_exponent == SiExponent::Paper ? UCFVB_SI_PAPER : UCFVB_SI_LEGACY;
    o.detect_every_stage = opt.detect_every_stage ? 1 : 0;
    o.gamma = opt.gamma;
    std::vector<ucfvb_bc> cb;
    for (const GpuBc& b : bcs) {
      ucfvb_bc x{};
      x.patch = b.patch.c_str();
      x.kind = b.kind;
      for (int v = 0; v < 4; ++v) x.state[v] = b.state[v];
      cb.push_back(x);
    }
    check(ucfvb_create(&mv_, &sv_, &o, cb.data(), static_cast<int32_t>(cb.size()), device, &h_), nullptr);
    state_.assign(mesh.n_cells(), State{});
    step_labels_.assign(mesh.n_cells(), Scheme::Linear);
    host_dirty_ = true;
  }
  ~GpuSolver() { ucfvb_destroy(h_); }
  GpuSolver(const GpuSolver&) = delete;
  GpuSolver& operator=(const GpuSolver&) = delete;

  // Solver::state(): a host mirror, pushed before the next device call
  StateField& state() {
    pull();
    host_dirty_ = true;
    return state_;
  }

  double max_stable_dt() {
    push();
    double dt = 0.0;
    check(ucfvb_max_stable_dt(h_, &dt), h_);
    return dt;
  }

  void advance(double dt, double t) { advance(dt, t, UCFVB_RK54); }
  void advance(double dt, double t, int rk) {
    push();
    check(ucfvb_advance(h_, dt, t, rk), h_);
    device_newer_ = true;
  }

  void compute_residual(const StateField& u, double t, StateField& out) {
    out.resize(u.size());
    check(ucfvb_compute_residual(h_, reinterpret_cast<const double*>(u.data()), t,
                                 reinterpret_cast<double*>(out.data())),
          h_);
  }

  const std::vector<Scheme>& step_labels() {
    std::vector<uint8_t> l(state_.size());
    check(ucfvb_get_step_labels(h_, l.data()), h_);
    for (size_t i = 0; i < l.size(); ++i) step_labels_[i] = static_cast<Scheme>(l[i]);
    return step_labels_;
  }

  PhaseTimes& phase_times() {
    double p[4];
    check(ucfvb_get_phase_times(h_, p), h_);
    times_ = PhaseTimes{p[0], p[1], p[2], p[3]};
    return times_;
  }
  const Mesh& mesh() const { return mesh_; }
  const StencilSet& stencils() const { return stencils_; }
  const SolverOptions& options() const { return opt_; }
  int n_qp() const { return stencils_.n_qp; }

 private:
  static void check(int32_t rc, const ucfvb_solver* h) {
    if (rc == UCFVB_OK) return;
    const std::string msg = ucfvb_last_error(h);
    if (rc == UCFVB_NONPHYSICAL) throw NonPhysicalError(msg);
    if (rc == UCFVB_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
  void push() {
    if (!host_dirty_) return;
    check(ucfvb_set_state(h_, reinterpret_cast<const double*>(state_.data())), h_);
    host_dirty_ = false;
  }
  void pull() {
    if (!device_newer_) return;
    check(ucfvb_get_state(h_, reinterpret_cast<double*>(state_.data())), h_);
    device_newer_ = false;
  }

  void flatten_mesh() {
    const Mesh& m = mesh_;
    const int nq = m.n_faces() ? static_cast<int>(m.faces[0].quad_points.size()) : 0;
    for (const Vec2& v : m.vertices) {
      vtx_.push_back(v.x);
      vtx_.push_back(v.y);
    }
    cvp_ = {0};
    cfp_ = {0};
    for (const Cell& c : m.cells) {
      cv_.insert(cv_.end(), c.vertex_ids.begin(), c.vertex_ids.end());
      cf_.insert(cf_.end(), c.face_ids.begin(), c.face_ids.end());
      cvp_.push_back(static_cast<int32_t>(cv_.size()));
      cfp_.push_back(static_cast<int32_t>(cf_.size()));
      ctr_.push_back(c.centroid.x);
      ctr_.push_back(c.centroid.y);
      area_.push_back(c.area);
      hc_.push_back(c.h_c);
    }
    for (const Face& f : m.faces) {
      fv_.push_back(f.vertex_ids[0]);
      fv_.push_back(f.vertex_ids[1]);
      fl_.push_back(f.left_cell);
      fr_.push_back(f.right_cell);
      fn_.push_back(f.normal.x);
      fn_.push_back(f.normal.y);
      flen_.push_back(f.length);
      fmid_.push_back(f.midpoint.x);
      fmid_.push_back(f.midpoint.y);
      for (int q = 0; q < nq; ++q) {
        fqp_.push_back(f.quad_points[q].x);
        fqp_.push_back(f.quad_points[q].y);
        fqw_.push_back(f.quad_weights[q]);
        fpq_.push_back(f.is_periodic() ? f.partner_qp[q] : -1);
      }
      fpatch_.push_back(f.patch);
      fpart_.push_back(f.periodic_partner);
      fshift_.push_back(f.shift_ix);
      fshift_.push_back(f.shift_iy);
    }
    for (const std::string& s : m.patch_names) pnames_.push_back(s.c_str());
    mv_ = ucfvb_mesh_view{};
    mv_.n_vertices = static_cast<int32_t>(m.vertices.size());
    mv_.n_cells = m.n_cells();
    mv_.n_faces = m.n_faces();
    mv_.n_qp = nq;
    mv_.n_patches = static_cast<int32_t>(pnames_.size());
    mv_.period_x = m.period_x;
    mv_.period_y = m.period_y;
    mv_.vertices = vtx_.data();
    mv_.cell_vtx_ptr = cvp_.data();
    mv_.cell_vtx = cv_.data();
    mv_.cell_face_ptr = cfp_.data();
    mv_.cell_faces = cf_.data();
    mv_.cell_centroid = ctr_.data();
    mv_.cell_area = area_.data();
    mv_.cell_h = hc_.data();
    mv_.face_vtx = fv_.data();
    mv_.face_left = fl_.data();
    mv_.face_right = fr_.data();
    mv_.face_normal = fn_.data();
    mv_.face_length = flen_.data();
    mv_.face_midpoint = fmid_.data();
    mv_.face_qp = fqp_.data();
    mv_.face_qw = fqw_.data();
    mv_.face_patch = fpatch_.data();
    mv_.face_partner = fpart_.data();
    mv_.face_shift = fshift_.data();
    mv_.face_partner_qp = fpq_.data();
    mv_.patch_names = pnames_.data();
  }

  void flatten_stencils() {
    const StencilSet& s = stencils_;
    const int n = static_cast<int>(s.cells.size()), K = s.K;
    cptr_ = {0};
    poff_ = {0};
    ploff_ = {0};
    dptr_ = {0};
    dmptr_ = {0};
    pdoff_ = {0};
    qptr_ = {0};
    phoff_ = {0};
    for (int c = 0; c < n; ++c) {
      const CellStencil& cs = s.cells[c];
      for (const StencilEntry& e : cs.central) {
        cen_.push_back(e.cell);
        cen_.push_back(e.px);
        cen_.push_back(e.py);
      }
      cptr_.push_back(static_cast<int64_t>(cen_.size() / 3));
      pinv_.insert(pinv_.end(), cs.pinv.begin(), cs.pinv.end());
      poff_.push_back(static_cast<int64_t>(pinv_.size()));
      plin_.insert(plin_.end(), cs.pinv_linear.begin(), cs.pinv_linear.end());
      ploff_.push_back(static_cast<int64_t>(plin_.size()));
      for (size_t d = 0; d < cs.directional.size(); ++d) {
        dmem_.insert(dmem_.end(), cs.directional[d].begin(), cs.directional[d].end());
        dmptr_.push_back(static_cast<int64_t>(dmem_.size()));
        pdir_.insert(pdir_.end(), cs.pinv_dir[d].begin(), cs.pinv_dir[d].end());
        pdoff_.push_back(static_cast<int64_t>(pdir_.size()));
      }
      dptr_.push_back(static_cast<int64_t>(dmptr_.size() - 1));
      oi_.insert(oi_.end(), cs.oi.begin(), cs.oi.end());
      slot_.insert(slot_.end(), s.cell_qp_slot[c].begin(), s.cell_qp_slot[c].end());
      qptr_.push_back(static_cast<int64_t>(slot_.size()));
      phi_.insert(phi_.end(), s.cell_phi[c].begin(), s.cell_phi[c].end());
      phoff_.push_back(static_cast<int64_t>(phi_.size()));
    }
    sv_ = ucfvb_stencil_view{};
    sv_.order = s.order;
    sv_.K = K;
    sv_.n_qp = s.n_qp;
    sv_.si_exponent = s.si_exponent == SiExponent::Paper ? UCFVB_SI_PAPER : UCFVB_SI_LEGACY;
    sv_.n_cells = n;
    sv_.n_dir_stencils = static_cast<int32_t>(dmptr_.size() - 1);
    sv_.central_ptr = cptr_.data();
    sv_.central = cen_.data();
    sv_.pinv_off = poff_.data();
    sv_.pinv = pinv_.data();
    sv_.pinv_lin_off = ploff_.data();
    sv_.pinv_lin = plin_.data();
    sv_.dir_ptr = dptr_.data();
    sv_.dir_member_ptr = dmptr_.data();
    sv_.dir_members = dmem_.data();
    sv_.pinv_dir_off = pdoff_.data();
    sv_.pinv_dir = pdir_.data();
    sv_.oi = oi_.data();
    sv_.qp_ptr = qptr_.data();
    sv_.phi_off = phoff_.data();
    sv_.phi = phi_.data();
    sv_.qp_slot = slot_.data();
  }

  const Mesh& mesh_;
  SolverOptions opt_;
  StencilSet stencils_;
  ucfvb_solver* h_ = nullptr;
  StateField state_;
  std::vector<Scheme> step_labels_;
  PhaseTimes times_;
  bool host_dirty_ = false, device_newer_ = false;
  // flat views (the device copies everything at create; kept for the handle's lifetime anyway)
  std::vector<double> vtx_, ctr_, area_, hc_, fn_, flen_, fmid_, fqp_, fqw_;
  std::vector<int32_t> cvp_, cv_, cfp_, cf_, fv_, fl_, fr_, fpatch_, fpart_, fshift_, fpq_;
  std::vector<const char*> pnames_;
  std::vector<int64_t> cptr_, poff_, ploff_, dptr_, dmptr_, pdoff_, qptr_, phoff_;
  std::vector<int32_t> cen_, dmem_, slot_;
  std::vector<double> pinv_, plin_, pdir_, oi_, phi_;
  ucfvb_mesh_view mv_{};
  ucfvb_stencil_view sv_{};
};

}  // namespace ucfv

#endif
