// extern "C" entry points of include/ucfvb3.h (3D stage pass). Exceptions
// become status codes exactly as in api.cpp.
#include <exception>
#include <new>
#include <string>

#include "decompose3.hpp"
#include "layout.hpp"
#include "setup3d.hpp"
#include "solver3d.hpp"
#include "ucfvb3.h"

struct ucfvb3_solver {
  ucfvb::GpuSolver3* s = nullptr;
  std::string err;
};

namespace {

thread_local std::string g_err3;

template <typename F>
int32_t guard3(ucfvb3_solver* h, F&& f) {
  try {
    f();
    return UCFVB_OK;
  } catch (const ucfvb::ApiError& e) {
    g_err3 = e.what();
    if (h) h->err = g_err3;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err3 = "out of memory";
    if (h) h->err = g_err3;
    return UCFVB_CUDA;
  } catch (const std::exception& e) {
    g_err3 = e.what();
    if (h) h->err = g_err3;
    return UCFVB_INVALID;
  }
}

#define NEED(h)                                                   \
  if (!(h) || !(h)->s) {                                          \
    g_err3 = "null solver handle";                                \
    return UCFVB_INVALID;                                         \
  }

}  // namespace

extern "C" {

const char* ucfvb3_last_error(const ucfvb3_solver* h) { return h ? h->err.c_str() : g_err3.c_str(); }

int32_t ucfvb3_mesh_periodic_box(int32_t nx, int32_t ny, int32_t nz, double lx, double ly, double lz, int32_t kind,
                                 double jitter, uint64_t seed, int32_t order, int32_t n_threads, ucfvb3_mesh** out) {
  return guard3(nullptr, [&] {
    if (!out) throw ucfvb::ApiError(UCFVB_INVALID, "null output pointer");
    *out = ucfvb::mesh3_periodic_box(nx, ny, nz, lx, ly, lz, kind, jitter, seed, order, n_threads);
  });
}
int32_t ucfvb3_mesh_get_view(const ucfvb3_mesh* m, ucfvb3_mesh_view* out) {
  return guard3(nullptr, [&] {
    if (!m || !out) throw ucfvb::ApiError(UCFVB_INVALID, "null pointer");
    *out = ucfvb::mesh3_view(m);
  });
}
void ucfvb3_mesh_free(ucfvb3_mesh* m) { ucfvb::mesh3_free(m); }

int32_t ucfvb3_build_stencils(const ucfvb3_mesh_view* mesh, int32_t order, int32_t si_exponent,
                              int32_t lattice_classes, int32_t n_threads, ucfvb3_stencils** out) {
  return guard3(nullptr, [&] {
    if (!mesh || !out) throw ucfvb::ApiError(UCFVB_INVALID, "null pointer");
    *out = ucfvb::build_stencils3(*mesh, order, si_exponent, lattice_classes, n_threads);
  });
}
int32_t ucfvb3_stencils_get_view(const ucfvb3_stencils* s, ucfvb3_stencil_view* out) {
  return guard3(nullptr, [&] {
    if (!s || !out) throw ucfvb::ApiError(UCFVB_INVALID, "null pointer");
    *out = ucfvb::stencils3_view(s);
  });
}
void ucfvb3_stencils_free(ucfvb3_stencils* s) { ucfvb::stencils3_free(s); }

int32_t ucfvb3_project_initial(const ucfvb3_mesh_view* mesh, int32_t ic, const double* params, int32_t n_params,
                               uint64_t seed, int32_t degree, double gamma, int32_t n_threads, double* u_out) {
  return guard3(nullptr, [&] {
    if (!mesh || !u_out) throw ucfvb::ApiError(UCFVB_INVALID, "null pointer");
    ucfvb::project_initial3(*mesh, ic, params, n_params, seed, degree, gamma, n_threads, u_out);
  });
}

int32_t ucfvb3_create(const ucfvb3_mesh_view* mesh, const ucfvb3_stencil_view* st, const ucfvb_options* opt,
                      int32_t device, ucfvb3_solver** out) {
  return guard3(nullptr, [&] {
    if (!mesh || !st || !opt || !out) throw ucfvb::ApiError(UCFVB_INVALID, "null pointer");
    auto* h = new ucfvb3_solver;
    try {
      h->s = new ucfvb::GpuSolver3(*mesh, *st, *opt, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
void ucfvb3_destroy(ucfvb3_solver* h) {
  if (!h) return;
  delete h->s;
  delete h;
}
int32_t ucfvb3_set_state(ucfvb3_solver* h, const double* u) {
  NEED(h);
  return guard3(h, [&] { h->s->set_state(u); });
}
int32_t ucfvb3_get_state(ucfvb3_solver* h, double* u) {
  NEED(h);
  return guard3(h, [&] { h->s->get_state(u); });
}
int32_t ucfvb3_max_stable_dt(ucfvb3_solver* h, double* dt) {
  NEED(h);
  return guard3(h, [&] { *dt = h->s->max_stable_dt(); });
}
int32_t ucfvb3_advance(ucfvb3_solver* h, double dt, double t, int32_t rk) {
  NEED(h);
  return guard3(h, [&] { h->s->advance(dt, t, rk); });
}
int32_t ucfvb3_run_steps(ucfvb3_solver* h, int32_t n_steps, double t0, int32_t rk, double* t_out) {
  NEED(h);
  return guard3(h, [&] {
    const double t = h->s->run_steps(n_steps, t0, rk);
    if (t_out) *t_out = t;
  });
}
int32_t ucfvb3_advance_host(ucfvb3_solver* h, const double* u_in, double* u_out, int32_t n_steps, int32_t rk,
                            double t0, double* t_out) {
  NEED(h);
  return guard3(h, [&] {
    const double t = h->s->advance_host(u_in, u_out, n_steps, rk, t0);
    if (t_out) *t_out = t;
  });
}
int32_t ucfvb3_advance_host_batch(ucfvb3_solver* h, int32_t n_batch, const double* const* u_in,
                                  double* const* u_out, int32_t n_steps, int32_t rk, double t0, double* t_out) {
  NEED(h);
  return guard3(h, [&] {
    if (!u_in || !u_out) throw ucfvb::ApiError(UCFVB_INVALID, "advance_host_batch: null pointer table");
    h->s->advance_host_batch(n_batch, u_in, u_out, n_steps, rk, t0, t_out);
  });
}
int32_t ucfvb3_compute_residual(ucfvb3_solver* h, const double* u, double t, double* out) {
  NEED(h);
  return guard3(h, [&] { h->s->compute_residual(u, t, out); });
}
int32_t ucfvb3_get_labels(ucfvb3_solver* h, int32_t which, uint8_t* out) {
  NEED(h);
  return guard3(h, [&] { h->s->get_labels(which, out); });
}
int32_t ucfvb3_get_face_values(ucfvb3_solver* h, double* out) {
  NEED(h);
  return guard3(h, [&] { h->s->get_face_values(out); });
}
int32_t ucfvb3_get_census(ucfvb3_solver* h, int64_t out[4]) {
  NEED(h);
  return guard3(h, [&] { h->s->census(out); });
}
int32_t ucfvb3_get_nad_ties(ucfvb3_solver* h, int64_t* out) {
  NEED(h);
  return guard3(h, [&] { *out = h->s->nad_ties(); });
}
int32_t ucfvb3_create_sub(const ucfvb3_subdomain* sub, const ucfvb_options* opt, int32_t device,
                          ucfvb3_solver** out) {
  return guard3(nullptr, [&] {
    if (!sub || !opt || !out) throw ucfvb::ApiError(UCFVB_INVALID, "null pointer");
    auto* h = new ucfvb3_solver;
    try {
      h->s = new ucfvb::GpuSolver3(sub->mv, sub->sv, *opt, device, sub);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
int32_t ucfvb3_attach_nccl(ucfvb3_solver* h, const uint8_t unique_id[128], int32_t rank, int32_t world) {
  NEED(h);
  return guard3(h, [&] { h->s->attach_nccl(unique_id, rank, world); });
}
int32_t ucfvb3_set_phase_timing(ucfvb3_solver* h, int32_t on) {
  NEED(h);
  return guard3(h, [&] { h->s->set_phase_timing(on != 0); });
}
int32_t ucfvb3_get_phase_times(ucfvb3_solver* h, double out[5]) {
  NEED(h);
  return guard3(h, [&] { h->s->phase_times(out); });
}
int64_t ucfvb3_launch_count(const ucfvb3_solver* h) { return (h && h->s) ? h->s->launches() : 0; }
void* ucfvb3_stream(const ucfvb3_solver* h) { return (h && h->s) ? h->s->stream() : nullptr; }

}  // extern "C"
