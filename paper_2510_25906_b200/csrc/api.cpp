// extern "C" entry points of include/ucfvb.h. Each wrapper converts C++
// exceptions into the ABI's status codes and keeps the message for
// ucfvb_last_error (the reference throws NonPhysicalError / invalid_argument /
// MeshError; see ucfvb.h).
#include <cstring>
#include <exception>
#include <new>
#include <string>
#include <vector>

#include "decompose.hpp"
#include "layout.hpp"
#include "setup.hpp"
#include "solver.hpp"
#include "ucfvb.h"

struct ucfvb_solver {
  ucfvb::GpuSolver* s = nullptr;
  const ucfvb_subdomain* sub = nullptr;  // borrowed (ucfvb_create_sub); must outlive the solver
  std::string err;
};

namespace ucfvb {
void nccl_unique_id(uint8_t id[128]);
void write_field_snapshot(const ucfvb_mesh_view& m, const double* state, const uint8_t* labels, double gamma,
                          const char* path);
void write_census_csv(const ucfvb_census_row* rows, int n_rows, int64_t n_cells, const char* path);
void write_timing_csv(const ucfvb_timing_row* rows, int n_rows, const char* path);
}

namespace {

thread_local std::string g_err;

template <typename F>
int32_t guard(ucfvb_solver* h, F&& f) {
  try {
    f();
    return UCFVB_OK;
  } catch (const ucfvb::ApiError& e) {
    g_err = e.what();
    if (h) h->err = g_err;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    if (h) h->err = g_err;
    return UCFVB_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    if (h) h->err = g_err;
    return UCFVB_INVALID;
  }
}

}  // namespace

extern "C" {

int32_t ucfvb_abi_version(void) { return UCFVB_ABI_VERSION; }

const char* ucfvb_last_error(const ucfvb_solver* h) { return h ? h->err.c_str() : g_err.c_str(); }

void ucfvb_options_default(ucfvb_options* o) {
  std::memset(o, 0, sizeof *o);
  o->order = 3;
  o->mode = UCFVB_HYBRID;
  o->limiter = UCFVB_BARTH_JESPERSEN;
  o->riemann = UCFVB_HLLC;
  o->margins = ucfvb_margins{1e-4, 0.5, 0.0, 0.0, 5.0, 2.0};
  o->lambda1p = 1e3;
  o->weno_eps = 1e-3;
  o->weno_b = 4.0;
  o->cfl = 0.6;
  o->venkat_kappa = 5.0;
  o->si_exponent = UCFVB_SI_PAPER;
  o->detect_every_stage = 1;
  o->gamma = 1.4;
  o->keep_taps = 0;
  o->use_graphs = 1;
}

int32_t ucfvb_mesh_structured_tri(int32_t nx, int32_t ny, double x0, double y0, double x1, double y1,
                                  int32_t diagonal, double jitter, uint64_t seed, int32_t periodic_axis,
                                  double tol, int32_t n_qp, ucfvb_mesh** out) {
  return guard(nullptr, [&] {
    *out = ucfvb::mesh_structured(nx, ny, x0, y0, x1, y1, /*quads=*/false, diagonal, jitter, seed,
                                  periodic_axis, tol, n_qp);
  });
}

int32_t ucfvb_mesh_structured_quad(int32_t nx, int32_t ny, double x0, double y0, double x1, double y1,
                                   int32_t periodic_axis, double tol, int32_t n_qp, ucfvb_mesh** out) {
  return guard(nullptr, [&] {
    *out = ucfvb::mesh_structured(nx, ny, x0, y0, x1, y1, /*quads=*/true, 0, 0.0, 0, periodic_axis, tol, n_qp);
  });
}

int32_t ucfvb_mesh_get_view(const ucfvb_mesh* m, ucfvb_mesh_view* out) {
  return guard(nullptr, [&] { *out = ucfvb::mesh_view(m); });
}

void ucfvb_mesh_free(ucfvb_mesh* m) { ucfvb::mesh_free(m); }

int32_t ucfvb_build_stencils(const ucfvb_mesh_view* mesh, int32_t order, int32_t si_exponent, int32_t n_threads,
                             ucfvb_stencils** out) {
  return guard(nullptr, [&] { *out = ucfvb::build_stencils(*mesh, order, si_exponent, n_threads); });
}

int32_t ucfvb_stencils_get_view(const ucfvb_stencils* s, ucfvb_stencil_view* out) {
  return guard(nullptr, [&] { *out = ucfvb::stencils_view(s); });
}

void ucfvb_stencils_free(ucfvb_stencils* s) { ucfvb::stencils_free(s); }

int32_t ucfvb_project_initial(const ucfvb_mesh_view* mesh, int32_t ic, const double* params, int32_t n_params,
                              uint64_t seed, int32_t degree, double gamma, int32_t n_threads, double* u_out) {
  return guard(nullptr, [&] {
    ucfvb::project_initial(*mesh, ic, params, n_params, seed, degree, gamma, n_threads, u_out);
  });
}

int32_t ucfvb_create(const ucfvb_mesh_view* mesh, const ucfvb_stencil_view* stencils, const ucfvb_options* opt,
                     const ucfvb_bc* bcs, int32_t n_bcs, int32_t device, ucfvb_solver** out) {
  *out = nullptr;
  return guard(nullptr, [&] {
    auto* h = new ucfvb_solver;
    try {
      h->s = new ucfvb::GpuSolver(*mesh, *stencils, *opt, bcs, n_bcs, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void ucfvb_destroy(ucfvb_solver* h) {
  if (!h) return;
  delete h->s;
  delete h;
}

int32_t ucfvb_set_state(ucfvb_solver* h, const double* u) {
  return guard(h, [&] { h->s->set_state(u); });
}
int32_t ucfvb_get_state(ucfvb_solver* h, double* u) {
  return guard(h, [&] { h->s->get_state(u); });
}
int32_t ucfvb_max_stable_dt(ucfvb_solver* h, double* dt) {
  return guard(h, [&] { *dt = h->s->max_stable_dt(); });
}
int32_t ucfvb_advance(ucfvb_solver* h, double dt, double t, int32_t rk) {
  return guard(h, [&] { h->s->advance(dt, t, rk); });
}
int32_t ucfvb_compute_residual(ucfvb_solver* h, const double* u, double t, double* out) {
  return guard(h, [&] { h->s->compute_residual(u, t, out); });
}
int32_t ucfvb_run_steps(ucfvb_solver* h, int32_t n_steps, int32_t rk, double t0, double t_end, double* t_out,
                        int64_t* census_out) {
  return guard(h, [&] {
    const double t = h->s->run_steps(n_steps, rk, t0, t_end, census_out);
    if (t_out) *t_out = t;
  });
}
int32_t ucfvb_advance_host(ucfvb_solver* h, const double* u_in, double* u_out, int32_t n_steps, int32_t rk,
                           double t0, double* t_out) {
  return guard(h, [&] {
    const double t = h->s->advance_host(u_in, u_out, n_steps, rk, t0);
    if (t_out) *t_out = t;
  });
}
int32_t ucfvb_advance_host_batch(ucfvb_solver* h, int32_t n_batch, const double* const* u_in, double* const* u_out,
                                 int32_t n_steps, int32_t rk, double t0, double* t_out) {
  return guard(h, [&] {
    if (!u_in || !u_out) throw ucfvb::ApiError(UCFVB_INVALID, "advance_host_batch: null pointer table");
    h->s->advance_host_batch(n_batch, u_in, u_out, n_steps, rk, t0, t_out);
  });
}
int32_t ucfvb_run_steps_log(ucfvb_solver* h, int32_t n_steps, int32_t rk, double t0, double t_end, double* t_out,
                            int64_t* census_out, double* dt_out) {
  return guard(h, [&] {
    const double t = h->s->run_steps(n_steps, rk, t0, t_end, census_out, dt_out);
    if (t_out) *t_out = t;
  });
}
int32_t ucfvb_run_until(ucfvb_solver* h, int32_t max_steps, int32_t rk, double t0, double t_end, double* t_out,
                        int32_t* n_steps_out, int64_t* census_out, double* dt_out) {
  return guard(h, [&] {
    int n = 0;
    const double t = h->s->run_until(max_steps, rk, t0, t_end, census_out, dt_out, &n);
    if (t_out) *t_out = t;
    if (n_steps_out) *n_steps_out = n;
  });
}
int32_t ucfvb_write_field_snapshot(const ucfvb_mesh_view* mesh, const double* state, const uint8_t* labels,
                                   double gamma, const char* path) {
  return guard(nullptr, [&] {
    if (!mesh) throw ucfvb::ApiError(UCFVB_INVALID, "write_field_snapshot: null mesh");
    ucfvb::write_field_snapshot(*mesh, state, labels, gamma, path);
  });
}
int32_t ucfvb_write_census_csv(const ucfvb_census_row* rows, int32_t n_rows, int64_t n_cells, const char* path) {
  return guard(nullptr, [&] { ucfvb::write_census_csv(rows, n_rows, n_cells, path); });
}
int32_t ucfvb_write_timing_csv(const ucfvb_timing_row* rows, int32_t n_rows, const char* path) {
  return guard(nullptr, [&] { ucfvb::write_timing_csv(rows, n_rows, path); });
}
int32_t ucfvb_get_step_labels(ucfvb_solver* h, uint8_t* labels) {
  return guard(h, [&] { h->s->get_labels(labels, true); });
}
int32_t ucfvb_get_labels(ucfvb_solver* h, uint8_t* labels) {
  return guard(h, [&] { h->s->get_labels(labels, false); });
}
int32_t ucfvb_get_census(ucfvb_solver* h, int64_t counts[4]) {
  return guard(h, [&] { h->s->get_census(counts); });
}
int32_t ucfvb_set_list_policy(ucfvb_solver* h, int32_t policy) {
  return guard(h, [&] { h->s->set_list_policy(policy); });
}
int32_t ucfvb_get_list_stats(ucfvb_solver* h, int64_t stats[5]) {
  return guard(h, [&] { h->s->get_list_stats(stats); });
}
int32_t ucfvb_get_nad_ties(ucfvb_solver* h, int64_t* ties) {
  return guard(h, [&] { *ties = h->s->nad_ties(); });
}
int32_t ucfvb_get_face_values(ucfvb_solver* h, double* left, double* right) {
  return guard(h, [&] { h->s->get_face_values(left, right); });
}
int32_t ucfvb_get_dofs(ucfvb_solver* h, double* dofs) {
  return guard(h, [&] { h->s->get_dofs(dofs); });
}
int32_t ucfvb_set_phase_timing(ucfvb_solver* h, int32_t enabled) {
  return guard(h, [&] { h->s->set_phase_timing(enabled != 0); });
}
int32_t ucfvb_get_phase_times(ucfvb_solver* h, double times[4]) {
  return guard(h, [&] { h->s->get_phase_times(times); });
}
int32_t ucfvb_n_cells(const ucfvb_solver* h) { return h->s->n_cells(); }
int32_t ucfvb_n_faces(const ucfvb_solver* h) { return h->s->n_faces(); }
int32_t ucfvb_n_qp(const ucfvb_solver* h) { return h->s->n_qp(); }
int32_t ucfvb_state_device_ptr(ucfvb_solver* h, double** dptr) {
  return guard(h, [&] { *dptr = h->s->state_device_ptr(); });
}
int32_t ucfvb_stream(ucfvb_solver* h, void** stream) {
  return guard(h, [&] { *stream = h->s->stream(); });
}
int64_t ucfvb_launch_count(const ucfvb_solver* h) { return h->s->launch_count(); }


int32_t ucfvb_partition_rcb(const ucfvb_mesh_view* mesh, int32_t n_parts, int32_t* part) {
  return guard(nullptr, [&] { ucfvb::partition_rcb(*mesh, n_parts, part); });
}

int32_t ucfvb_subdomain_build(const ucfvb_mesh_view* mesh, const ucfvb_stencil_view* stencils, const int32_t* part,
                              int32_t n_parts, int32_t rank, ucfvb_subdomain** out) {
  return guard(nullptr, [&] { *out = ucfvb::build_subdomain(*mesh, *stencils, part, n_parts, rank); });
}

int32_t ucfvb_subdomain_views(const ucfvb_subdomain* s, ucfvb_mesh_view* mesh, ucfvb_stencil_view* stencils) {
  if (mesh) *mesh = s->mv;
  if (stencils) *stencils = s->sv;
  return UCFVB_OK;
}

int32_t ucfvb_subdomain_info(const ucfvb_subdomain* s, int32_t* n_owned, int32_t* n_local, int32_t* n_peers) {
  if (n_owned) *n_owned = s->n_owned;
  if (n_local) *n_local = s->n_local;
  if (n_peers) *n_peers = static_cast<int32_t>(s->peers.size());
  return UCFVB_OK;
}

int32_t ucfvb_subdomain_interior(const ucfvb_subdomain* s, int32_t* n_interior) {
  *n_interior = s->n_interior;
  return UCFVB_OK;
}

int32_t ucfvb_subdomain_global_ids(const ucfvb_subdomain* s, int32_t* gid) {
  std::memcpy(gid, s->gid.data(), s->gid.size() * sizeof(int32_t));
  return UCFVB_OK;
}

int32_t ucfvb_subdomain_peer(const ucfvb_subdomain* s, int32_t i, int32_t* rank, int32_t* n_send, int32_t* n_recv,
                             int32_t* recv_begin) {
  if (i < 0 || i >= static_cast<int32_t>(s->peers.size())) return UCFVB_INVALID;
  const auto& p = s->peers[i];
  if (rank) *rank = p.rank;
  if (n_send) *n_send = static_cast<int32_t>(p.send.size());
  if (n_recv) *n_recv = p.n_recv;
  if (recv_begin) *recv_begin = p.recv_begin;
  return UCFVB_OK;
}

int32_t ucfvb_subdomain_send_list(const ucfvb_subdomain* s, int32_t i, int32_t* local_ids) {
  if (i < 0 || i >= static_cast<int32_t>(s->peers.size())) return UCFVB_INVALID;
  std::memcpy(local_ids, s->peers[i].send.data(), s->peers[i].send.size() * sizeof(int32_t));
  return UCFVB_OK;
}

void ucfvb_subdomain_free(ucfvb_subdomain* s) { delete s; }

int32_t ucfvb_create_sub(const ucfvb_subdomain* sub, const ucfvb_options* opt, const ucfvb_bc* bcs, int32_t n_bcs,
                         int32_t device, ucfvb_solver** out) {
  *out = nullptr;
  return guard(nullptr, [&] {
    auto* h = new ucfvb_solver;
    try {
      h->s = new ucfvb::GpuSolver(sub->mv, sub->sv, *opt, bcs, n_bcs, device, sub->n_owned);
      h->sub = sub;
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int32_t ucfvb_nccl_unique_id(uint8_t id[128]) {
  return guard(nullptr, [&] { ucfvb::nccl_unique_id(id); });
}

int32_t ucfvb_attach_nccl(ucfvb_solver* h, const uint8_t id[128], int32_t rank, int32_t world) {
  return guard(h, [&] { h->s->attach_nccl(id, rank, world, h->sub); });
}

struct ucfvb_group {
  ucfvb::GpuGroup* g = nullptr;
};

int32_t ucfvb_group_create(ucfvb_solver* const* parts, int32_t n, ucfvb_group** out) {
  *out = nullptr;
  return guard(nullptr, [&] {
    std::vector<ucfvb::GpuSolver*> s(n > 0 ? n : 0);
    std::vector<const ucfvb_subdomain*> sub(s.size());
    for (int32_t i = 0; i < n; ++i) {
      s[i] = parts[i]->s;
      sub[i] = parts[i]->sub;
    }
    auto* h = new ucfvb_group;
    try {
      h->g = new ucfvb::GpuGroup(s.data(), sub.data(), n);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int32_t ucfvb_group_run_steps(ucfvb_group* g, int32_t n_steps, int32_t rk, double t0, double* t_out) {
  return guard(nullptr, [&] {
    const double t = g->g->run_steps(n_steps, rk, t0);
    if (t_out) *t_out = t;
  });
}

int64_t ucfvb_group_launch_count(const ucfvb_group* g) { return g->g->launch_count(); }

void ucfvb_group_free(ucfvb_group* g) {
  if (!g) return;
  delete g->g;
  delete g;
}

}  // extern "C"
