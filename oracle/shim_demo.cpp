// ORACLE TEST INFRASTRUCTURE: the reference-side binding (include/ucfvb_ucfv.hpp)
// exercised exactly as a reference user would: the same Mesh, SolverOptions
// and initial state driven through ucfv::Solver (the unmodified reference,
// CPU) and ucfv::GpuSolver (B200 C ABI), then compared.
//   usage: shim_demo [n] [steps]     prints one JSON line; exit 0 on parity
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "ucfv/cases.hpp"
#include "ucfv/mesh.hpp"
#include "ucfv/solver.hpp"
#include "ucfvb_ucfv.hpp"

using namespace ucfv;

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 24;
  const int steps = argc > 2 ? std::atoi(argv[2]) : 3;
  // the reference's own vortex case mesh (cases.cpp:92-104) at resolution n
  Mesh mesh = pair_periodic(generate_structured_tri(n, n, {0.0, 0.0, 10.0, 10.0}, DiagonalRule::Uniform, 2),
                            Axis::Both, 1e-8);
  SolverOptions opt;
  opt.order = 2;
  opt.lambda1p = 1e4;
  opt.weno_b = 1.0;  // tau^1: exact on both sides, so the whole path is bit-faithful
  Solver cpu(mesh, opt, {});
  GpuSolver gpu(mesh, opt, {});
  const StateField u0 = project_initial(mesh, [](const Vec2& p) { return ic_vortex(p, 1.4); }, 4);
  cpu.state() = u0;
  gpu.state() = u0;
  double t = 0.0, max_abs = 0.0;
  long label_mismatch = 0;
  for (int s = 0; s < steps; ++s) {
    const double dc = cpu.max_stable_dt(), dg = gpu.max_stable_dt();
    if (dc != dg) {
      std::printf("{\"ok\": false, \"why\": \"dt differs\"}\n");
      return 1;
    }
    cpu.advance(dc, t);
    gpu.advance(dc, t);
    t += dc;
    const auto& lc = cpu.step_labels();
    const auto& lg = gpu.step_labels();
    for (size_t i = 0; i < lc.size(); ++i) label_mismatch += lc[i] != lg[i];
  }
  const StateField& uc = cpu.state();
  const StateField& ug = gpu.state();
  for (size_t i = 0; i < uc.size(); ++i)
    for (int v = 0; v < 4; ++v) max_abs = std::fmax(max_abs, std::fabs(uc[i][v] - ug[i][v]));
  const bool ok = max_abs == 0.0 && label_mismatch == 0;
  std::printf("{\"ok\": %s, \"cells\": %d, \"steps\": %d, \"max_abs_diff\": %.3e, \"label_mismatch\": %ld}\n",
              ok ? "true" : "false", mesh.n_cells(), steps, max_abs, label_mismatch);
  return ok ? 0 : 1;
}
