// 3D device solver (BASELINE configs 4-5): the stage pass of solver.cu for
// five conserved variables on periodic hexahedral / tetrahedral meshes.
#pragma once

#include <cstdint>

#include "ucfvb.h"
#include "ucfvb3.h"

namespace ucfvb {

class GpuSolver3 {
 public:
  GpuSolver3(const ucfvb3_mesh_view& m, const ucfvb3_stencil_view& s, const ucfvb_options& o, int device,
             const ucfvb3_subdomain* sub = nullptr);
  void attach_nccl(const uint8_t id[128], int rank, int world);
  ~GpuSolver3();
  GpuSolver3(const GpuSolver3&) = delete;
  GpuSolver3& operator=(const GpuSolver3&) = delete;

  void set_state(const double* u);
  void get_state(double* u);
  double max_stable_dt();
  void advance(double dt, double t, int rk);
  double run_steps(int n_steps, double t0, int rk);
  double advance_host(const double* u_in, double* u_out, int n_steps, int rk, double t0);
  void advance_host_batch(int n_batch, const double* const* u_in, double* const* u_out, int n_steps, int rk,
                          double t0, double* t_out);
  void compute_residual(const double* u, double t, double* out);
  void get_labels(int which, uint8_t* out);
  void get_face_values(double* out);
  void census(int64_t out[4]);
  int64_t nad_ties();
  void set_phase_timing(bool on);
  void phase_times(double out[5]);
  int64_t launches() const;
  void* stream() const;

  struct Impl;

 private:
  Impl* p_;
};

}  // namespace ucfvb
