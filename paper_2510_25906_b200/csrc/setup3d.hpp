// 3D host setup (mesh, operators, initial conditions); see setup3d.cpp.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "ucfvb3.h"

namespace ucfvb {

// Legendre-product basis P_i(x) P_j(y) P_k(z), 1 <= i+j+k <= r, ordered by
// total degree then descending i, j (basis.cpp:34-68 with a third factor)
struct Family3 {
  int r = 1, K = 0;
  std::vector<std::vector<std::vector<double>>> leg;  // [n][derivative][coefficient]
  std::vector<std::array<int, 3>> deg, beta;
  explicit Family3(int order);
  void tables(const double* xi, int dmax, double* P) const;
  void eval_all(const double* xi, double* out) const;
  void eval_deriv(int b, const double* xi, double* out) const;
};

ucfvb3_mesh* mesh3_periodic_box(int nx, int ny, int nz, double lx, double ly, double lz, int kind, double jitter,
                                uint64_t seed, int order, int n_threads);
ucfvb3_mesh_view mesh3_view(const ucfvb3_mesh* m);
void mesh3_free(ucfvb3_mesh* m);
ucfvb3_stencils* build_stencils3(const ucfvb3_mesh_view& m, int order, int si, int classes, int n_threads);
ucfvb3_stencil_view stencils3_view(const ucfvb3_stencils* s);
void stencils3_free(ucfvb3_stencils* s);
void project_initial3(const ucfvb3_mesh_view& m, int ic, const double* prm, int n_prm, uint64_t seed, int degree,
                      double g, int n_threads, double* u_out);

}  // namespace ucfvb
