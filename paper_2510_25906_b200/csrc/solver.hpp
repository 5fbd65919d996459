// GpuSolver: C++ host side of the B200 stage pass, mirroring the public API of
// ucfv::Solver (/root/reference/proj/include/ucfv/solver.hpp:52-100).
#pragma once

#include <cstdint>
#include <memory>

#include "ucfvb.h"

namespace ucfvb {

class GpuSolver {
 public:
  // Solver(mesh, opt, bcs) (solver.cpp:36-74); throws ApiError
  // n_owned < 0: every cell is owned (single domain); otherwise the first
  // n_owned cells of a subdomain (ucfvb_subdomain_build) are owned
  GpuSolver(const ucfvb_mesh_view& mesh, const ucfvb_stencil_view& stencils, const ucfvb_options& opt,
            const ucfvb_bc* bcs, int n_bcs, int device, int n_owned = -1);
  ~GpuSolver();
  GpuSolver(const GpuSolver&) = delete;
  GpuSolver& operator=(const GpuSolver&) = delete;

  void set_state(const double* u);                                   // state() = u
  void get_state(double* u);                                         // u = state()
  double max_stable_dt();                                            // solver.cpp:103-111
  void advance(double dt, double t, int rk);                         // solver.cpp:381-387
  void compute_residual(const double* u, double t, double* out);     // solver.cpp:316-379
  double run_steps(int n_steps, int rk, double t0, double t_end, int64_t* census, double* dt_out = nullptr);
  // host state in -> n_steps graph-replayed steps -> host state out, with one
  // synchronisation (the host-buffer form of state() + advance loop)
  double advance_host(const double* u_in, double* u_out, int n_steps, int rk, double t0);
  // n_batch independent states through advance_host, pipelined: uploads and
  // downloads overlap the stepping of the neighbouring entries
  void advance_host_batch(int n_batch, const double* const* u_in, double* const* u_out, int n_steps, int rk,
                          double t0, double* t_out);
  // run_simulation's loop condition (run.cpp:96): steps while t < t_end - 1e-14 t_end, at most max_steps
  double run_until(int max_steps, int rk, double t0, double t_end, int64_t* census, double* dt_out, int* n_done);  // run.cpp:97-132

  void get_labels(uint8_t* out, bool step);
  void get_census(int64_t counts[4]);
  int64_t nad_ties();
  void get_face_values(double* left, double* right);
  void get_dofs(double* dofs);
  // troubled-cell class lists: 0 chunk lists (default), 1 per-cell lists
  void set_list_policy(int policy);
  // last synchronised stage: CWENOZ cells, MUSCL cells, CWENOZ chunks, MUSCL chunks, per-cell lists in use
  void get_list_stats(int64_t out[5]);
  void set_phase_timing(bool on);
  void get_phase_times(double t[4]);

  int n_cells() const;
  int n_faces() const;
  int n_qp() const;
  int K() const;
  int64_t launch_count() const;
  void* stream() const;
  double* state_device_ptr();
  // NCCL communicator + the subdomain's exchange plan (halo exchange after every stage)
  void attach_nccl(const uint8_t id[128], int rank, int world, const ucfvb_subdomain* sub);

  struct Impl;

 private:
  friend class GpuGroup;
  double run_impl(int n_steps, int rk, double t0, double t_end, bool until, int64_t* census, double* dt_out,
                  int* n_done);
  std::unique_ptr<Impl> p_;
};

// In-process loopback group: the subdomain solvers of one partition (part i
// = rank i) on ONE device, stepped together with the multi-GPU schedule of a
// rank -- sent cells first, the halo exchange forked onto each part's exchange
// stream while its interior is updated -- and device-to-device copies (one
// cudaMemcpyAsync per peer block) as the transport, the dt min and the error
// word reduced by kernels across the group; one CUDA graph captures a step of
// all parts. It tests the exchange schedule and plans on a single GPU.
class GpuGroup {
 public:
  GpuGroup(GpuSolver* const* parts, const ucfvb_subdomain* const* subs, int n);
  ~GpuGroup();
  GpuGroup(const GpuGroup&) = delete;
  GpuGroup& operator=(const GpuGroup&) = delete;
  double run_steps(int n_steps, int rk, double t0);
  int64_t launch_count() const;

 private:
  struct Impl;
  std::unique_ptr<Impl> p_;
};

}  // namespace ucfvb
