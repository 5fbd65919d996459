"""Quick timing: graph-replayed RK3 steps (us/stage) + per-phase event times."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2510_25906_b200 import _abi as A  # noqa: E402
from paper_2510_25906_b200.solver import Solver, make_bcs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="2")
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--tag", default="")
a = ap.parse_args()
import torch  # noqa: E402

c = bench.CONFIGS[a.config]
mesh, st, u0, _ = bench.build_case(a.config)
o = A.options_from_dict(order=c["order"], mode="hybrid", **c["opts"])
s = Solver(mesh, o, make_bcs(c["bcs"]), stencils=st)
s.state = u0
s.run_steps(5, A.RK3)
stream = torch.cuda.ExternalStream(s.stream())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(stream)
s.run_steps(a.steps, A.RK3)
e1.record(stream)
e1.synchronize()
ms = e0.elapsed_time(e1)
n = s.n_cells
s.set_phase_timing(True)
p0 = s.phase_times().copy()
s.run_steps(10, A.RK3)
ph = (s.phase_times() - p0) / 30 * 1e6
print(f"{a.tag} config{a.config}: {1e3 * ms / (3 * a.steps):.1f} us/stage  {n * 3 * a.steps / ms / 1e6:.3f} G/s  "
      f"phases(us) central {ph[0]:.1f} detect {ph[1]:.1f} weights {ph[2]:.1f} flux {ph[3]:.1f}  {s.list_stats()}")
