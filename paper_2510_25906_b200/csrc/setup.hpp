// Host setup on either side of the stage pass: mesh
// generation + periodic pairing, the per-cell operator precompute
// (build_stencils) and initial-condition projection. Multithreaded C++;
// arithmetic follows the reference so operator data can be compared bitwise.
#pragma once

#include <cstdint>
#include <vector>

#include "ucfvb.h"

namespace ucfvb {

ucfvb_mesh* mesh_structured(int nx, int ny, double x0, double y0, double x1, double y1, bool quads, int diagonal,
                            double jitter, uint64_t seed, int periodic_axis, double tol, int n_qp);
ucfvb_mesh_view mesh_view(const ucfvb_mesh* m);
void mesh_free(ucfvb_mesh* m);

ucfvb_stencils* build_stencils(const ucfvb_mesh_view& m, int order, int si_exponent, int n_threads);
ucfvb_stencil_view stencils_view(const ucfvb_stencils* s);
void stencils_free(ucfvb_stencils* s);

// column-pivoting Householder QR least-squares pseudo-inverse (the
// ColPivHouseholderQR restatement in setup_stencil.cpp); false when rank < cols
bool qr_pinv(const std::vector<double>& A, int rows, int cols, std::vector<double>& pinv);

void project_initial(const ucfvb_mesh_view& m, int ic, const double* params, int n_params, uint64_t seed,
                     int degree, double gamma, int n_threads, double* u_out);

}  // namespace ucfvb
