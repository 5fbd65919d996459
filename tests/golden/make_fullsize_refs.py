"""Full-size, full-length reference runs of BASELINE configs 2 and 3.

Runs the compiled reference (oracle/_ref: the unmodified /root/reference
sources) through the harness's SSP-RK3 driver over Solver::compute_residual
(reference loop: src/run.cpp:97-132 over src/solver.cpp:316-379) for the
configured step count, and commits a compact record the GPU test checks
against (tests/test_gpu_fullsize.py):

  * per step: the census of step labels (run.cpp:110-116) and dt (bit pattern)
  * the final time t
  * SHA-256 of the initial and of the final state bytes (n x 4 fp64, AoS)
  * per-variable L1 norm of the final state, sum |U_v|, summed in cell order
  * per-variable block sums of U and |U| over 1024 contiguous cell blocks
  * the full final state of a seeded sample of 65,536 cells (L1 of the
    difference on the sample, relative, is the 1e-8 check)

    python tests/golden/make_fullsize_refs.py 2      # ~5 min, 262,144 cells, 200 steps
    python tests/golden/make_fullsize_refs.py 3      # ~1.5 h, 8,388,608 cells, 50 steps, ~47 GB RAM

Needs /root/reference (the build container); the outputs travel to the GPU box.
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref as R  # noqa: E402
from paper_2510_25906_b200 import _abi as A  # noqa: E402
from paper_2510_25906_b200.solver import make_bcs  # noqa: E402
from tests.cases import case  # noqa: E402
from tests.fullsize_digest import sample_cells, sha256, summarise  # noqa: E402

STEPS = {"config2": 200, "config3": 50}


def main(name):
    mk, order, ic, prm, opts, bcs = case(name)
    nq = (order + 2) // 2
    per = {"both": 3, "y": 2, "x": 1, "none": 0}[mk["periodic"]]
    t0 = time.perf_counter()
    rm = R.RefMesh.structured_tri(mk["nx"], mk["ny"], mk["rect"], jitter=mk["jitter"], seed=1, periodic=per,
                                  n_qp=nq)
    o = A.options_from_dict(order=order, **opts)
    rs = R.RefSolver(rm, o, make_bcs(bcs))
    u0 = rm.project_initial(ic, prm, seed=1, degree=max(2 * order, 2))
    rs.set_state(u0)
    setup = time.perf_counter() - t0
    print(f"{name}: {rs.n_cells} cells, setup {setup:.1f}s", flush=True)
    n_steps = STEPS[name]
    t, cens, dts, walls = 0.0, [], [], []
    for s in range(n_steps):
        w0 = time.perf_counter()
        t, c, d = rs.run_log(1, A.RK3, t)
        walls.append(time.perf_counter() - w0)
        cens.append(c[0])
        dts.append(d[0])
        if s % 5 == 0 or s == n_steps - 1:
            print(f"  step {s + 1}/{n_steps} t={t:.6e} census={c[0].tolist()} {walls[-1]:.1f}s", flush=True)
    u = rs.get_state()
    idx = sample_cells(u.shape[0])
    dg = summarise(u)
    out = ROOT / "tests" / "golden" / f"fullsize_{name}.npz"
    np.savez_compressed(out, census=np.array(cens, dtype=np.int64), dt=np.array(dts, dtype=np.float64),
                        t=np.float64(t), sample_idx=idx, sample_state=u[idx], l1=dg["l1"],
                        block_sum=dg["block_sum"], block_abs=dg["block_abs"])
    meta = {"name": name, "cells": int(u.shape[0]), "steps": n_steps, "order": order, "t_final": t,
            "u0_sha256": sha256(u0),
            "final_sha256": dg["sha256"], "setup_s": round(setup, 1),
            "step_wall_s": round(float(np.sum(walls)), 1),
            "rate_cell_stage_per_s": float(u.shape[0] * 3 * n_steps / np.sum(walls)),
            "generator": "tests/golden/make_fullsize_refs.py over oracle/_ref (unmodified reference sources), "
                         "1 thread, SSP-RK3 harness driver over Solver::compute_residual"}
    (ROOT / "tests" / "golden" / f"fullsize_{name}.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:] or ["2"]:
        main(f"config{a}" if not a.startswith("config") else a)
