"""Profiling driver for the 3D configs: build, warm up, then run RK3 steps
without CUDA graphs (one launch per kernel, events between kernel groups)
so ncu sees every kernel; prints the per-group times of the last steps."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2510_25906_b200 import _abi as A  # noqa: E402
from paper_2510_25906_b200.solver3d import Solver3  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
c = bench.CONFIGS3[a.config]
mesh, st, u0, setup = bench.build_case3(a.config, n=a.n)
o = A.options_from_dict(order=c["order"], mode=c["mode"], cfl=0.5)
s = Solver3(mesh, o, st)
s.state = u0
s.set_phase_timing(True)
s.run_steps(a.warmup)
p0 = s.phase_times().copy()
s.run_steps(a.steps)
ph = (s.phase_times() - p0) / (3 * a.steps)
print(f"config {a.config}: {mesh.n_cells} cells, setup {setup:.1f}s; us/stage central {1e6*ph[0]:.0f} spread "
      f"{1e6*ph[1]:.0f} weights {1e6*ph[2]:.0f} flux {1e6*ph[3]:.0f} gather {1e6*ph[4]:.0f}; census {s.census()}")
