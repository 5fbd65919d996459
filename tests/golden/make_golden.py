"""Generate tests/golden/*.npz from the compiled reference (oracle/_ref).

Each fixture holds the reference's OWN flat mesh and StencilSet bytes, the
solver options/BCs, an input state and the reference's outputs:
  one compute_residual stage from u0 (stage_is_first): residual, labels,
  face values (val_left_/val_right_), dofs, bounds;
  two SSP-RK3 steps (harness driver over compute_residual): state, step labels,
  per-step census and dt;
  one SSPRK(5,4) step (Solver::advance): state.
Run in the build container (needs /root/reference):  python tests/golden/make_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref as R  # noqa: E402
from paper_2510_25906_b200 import _abi as A  # noqa: E402
from paper_2510_25906_b200.solver import make_bcs  # noqa: E402

SHOCK = [-4.0, 3.857143, 2.629369, 0.0, 10.33333, 0.2, 5.0]
CASES = {
    "vortex_p2": dict(mesh=("tri", 8, 8, (0, 0, 1, 1), 0.1, 3), order=2, ic=(0, [10.0]),
                      opts=dict(mode=A.HYBRID, lambda1p=1e4, cfl=0.5), bcs={}),
    "quadrants_p3": dict(mesh=("tri", 8, 8, (0, 0, 1, 1), 0.1, 3), order=3, ic=(2, [0.5, 0.5, 0.01]),
                         opts=dict(mode=A.HYBRID, cfl=0.5), bcs={}),
    "shock_p2_outflow": dict(mesh=("tri", 16, 4, (-5, 0, 5, 1), 0.1, 2), order=2, ic=(1, SHOCK),
                             opts=dict(mode=A.HYBRID, cfl=0.5), bcs={"left": "outflow", "right": "outflow"}),
    "quadrants_p2_venkat_hll_frozen": dict(mesh=("tri", 8, 8, (0, 0, 1, 1), 0.1, 3), order=2,
                                           ic=(2, [0.5, 0.5, 0.01]),
                                           opts=dict(mode=A.HYBRID, limiter=A.VENKATAKRISHNAN, riemann=A.HLL,
                                                     detect_every_stage=0, cfl=0.5), bcs={}),
    "quads_p2_linear": dict(mesh=("quad", 6, 6, (0, 0, 1, 1), 0.0, 3), order=2, ic=(0, [10.0]),
                            opts=dict(mode=A.LINEAR, cfl=0.5), bcs={}),
    "walls_p2_hybrid": dict(mesh=("tri", 12, 6, (0, 0, 2, 1), 0.1, 0), order=2, ic=(2, [1.0, 0.5, 0.01]),
                            opts=dict(mode=A.HYBRID, cfl=0.5),
                            bcs={"left": ("fixed", (1.0, 0.5, 0.0, 2.6)), "right": "outflow", "bottom": "wall",
                                 "top": "wall"}),
    "quadrants_p1_cwenoz": dict(mesh=("tri", 8, 8, (0, 0, 1, 1), 0.1, 3), order=1, ic=(2, [0.5, 0.5, 0.01]),
                                opts=dict(mode=A.CWENOZ, cfl=0.5), bcs={}),
    "vortex_p1_cwenoz": dict(mesh=("tri", 8, 8, (0, 0, 1, 1), 0.1, 3), order=1, ic=(0, [10.0]),
                             opts=dict(mode=A.CWENOZ, lambda1p=1e4, cfl=0.5), bcs={}),
    "quadrants_p2_muscl": dict(mesh=("tri", 8, 8, (0, 0, 1, 1), 0.1, 3), order=2, ic=(2, [0.5, 0.5, 0.01]),
                               opts=dict(mode=A.MUSCL, cfl=0.5), bcs={}),
}
OPT_FIELDS = ["order", "mode", "limiter", "riemann", "lambda1p", "weno_eps", "weno_b", "cfl", "venkat_kappa",
              "si_exponent", "detect_every_stage", "gamma"]


def build(name, c):
    kind, nx, ny, rect, jit, per = c["mesh"]
    nq = (c["order"] + 2) // 2
    if kind == "tri":
        m = R.RefMesh.structured_tri(nx, ny, rect, jitter=jit, seed=11, periodic=per, n_qp=nq)
    else:
        m = R.RefMesh.generate_quad(nx, ny, rect, periodic=per, n_qp=nq)
    o = A.options_from_dict(order=c["order"], **c["opts"])
    bcs = make_bcs(c["bcs"])
    return m, o, bcs


def make(name, c):
    m, o, bcs = build(name, c)
    s = R.RefSolver(m, o, bcs)
    ic, prm = c["ic"]
    u0 = m.project_initial(ic, prm, seed=5, degree=max(2 * c["order"], 2))
    out = {}
    for k, v in m.numpy().items():
        out["mesh_" + k] = v
    for k, v in s.stencils_numpy().items():
        out["st_" + k] = v
    out["options"] = np.array([float(getattr(o, f)) for f in OPT_FIELDS])
    out["margins"] = np.array([o.margins.alpha_m, o.margins.beta_m, o.margins.alpha_w, o.margins.beta_w,
                               o.margins.kappa, o.margins.deact_n])
    out["bcs"] = np.array(json.dumps(c["bcs"]))
    out["u0"] = u0
    try:
        out["stage_residual"] = s.compute_residual(u0, 0.0, 1)
    except R.RefError as e:  # the reference throws (NonPhysicalError with the failing face)
        out["error_code"] = np.array(e.code)
        out["error_message"] = np.array(str(e))
        np.savez_compressed(Path(__file__).parent / f"{name}.npz", **out)
        print(name, "cells", len(u0), "reference throws:", e)
        return
    out["stage_labels"] = s.labels()
    L, Rv = s.face_values()
    out["stage_left"], out["stage_right"] = L, Rv
    out["stage_dofs"] = s.dofs()
    out["stage_bounds"] = s.bounds()
    s2 = R.RefSolver(m, o, bcs)
    s2.set_state(u0)
    dts, cens, t = [], [], 0.0
    for _ in range(2):
        dt = s2.max_stable_dt()
        s2.advance(dt, t, A.RK3)
        t += dt
        dts.append(dt)
        cens.append(np.bincount(s2.labels(step=True), minlength=4))
    out["rk3_dt"] = np.array(dts)
    out["rk3_state"] = s2.get_state()
    out["rk3_step_labels"] = s2.labels(step=True)
    out["rk3_census"] = np.array(cens)
    s3 = R.RefSolver(m, o, bcs)
    s3.set_state(u0)
    dt = s3.max_stable_dt()
    s3.advance(dt, 0.0, A.RK54)
    out["rk54_dt"] = np.array([dt])
    out["rk54_state"] = s3.get_state()
    np.savez_compressed(Path(__file__).parent / f"{name}.npz", **out)
    print(name, "cells", len(u0), "labels", np.bincount(out["stage_labels"], minlength=4))


if __name__ == "__main__":
    for n, c in CASES.items():
        make(n, c)
