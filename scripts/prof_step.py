"""Profiling driver: build a BASELINE config, warm up, then run a few RK3
steps without CUDA graphs (one launch per kernel) for ncu."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2510_25906_b200 import _abi as A  # noqa: E402
from paper_2510_25906_b200.solver import Solver, make_bcs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="2")
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--graphs", type=int, default=0)
a = ap.parse_args()
c = bench.CONFIGS[a.config]
mesh, st, u0, _ = bench.build_case(a.config)
o = A.options_from_dict(order=c["order"], mode="hybrid", use_graphs=a.graphs, **c["opts"])
s = Solver(mesh, o, make_bcs(c["bcs"]), stencils=st)
s.state = u0
s.run_steps(a.warmup, A.RK3)
s.run_steps(a.steps, A.RK3)
print("launches in last call:", s.launch_count())
