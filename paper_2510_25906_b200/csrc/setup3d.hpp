// 3D host setup (mesh, operators, initial conditions); see setup3d.cpp.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "ucfvb3.h"

namespace ucfvb {

// cell numbering of the lattice meshes: cube-major (c = cube * nt + type), or
// for tetrahedra on n^3 % 32 == 0 lattices type-major within blocks of 32
// cubes (c = ((cube / 32) * 6 + type) * 32 + cube % 32)
struct CellOrder {
  int nt, blocked;
  int64_t cell(int64_t cube, int t) const {
    return blocked ? (((cube >> 5) * nt + t) << 5) + (cube & 31) : cube * nt + t;
  }
  int64_t cube(int64_t c) const { return blocked ? (((c >> 5) / nt) << 5) + (c & 31) : c / nt; }
  int type(int64_t c) const { return static_cast<int>(blocked ? (c >> 5) % nt : c % nt); }
};

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
