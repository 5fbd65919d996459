"""Pins the oracle restatement (oracle/ucfv_port.c) to the reference.

1. Against tests/golden/*.npz: the compiled reference's own outputs on its own
   mesh/stencil bytes (always runs; no /root/reference needed).
2. Against the live compiled reference (oracle/_ref) on more configurations
   (skipped when oracle/_ref was not built).
Everything is compared bit-for-bit (np.array_equal).
"""
import numpy as np
import pytest

from oracle import port as P
from oracle import ref as R
from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.solver import make_bcs
from tests.golden_io import Fixture, names


@pytest.mark.parametrize("name", names())
def test_port_matches_golden(name):
    fx = Fixture(name)
    p = P.PortSolver(fx.mesh_view, fx.stencil_view, fx.options, fx.bcs, keep=(fx,))
    if fx.error:
        with pytest.raises(P.PortError) as ei:
            p.compute_residual(fx.u0, 0.0, 1)
        assert ei.value.code == int(fx["error_code"])
        face = str(fx["error_message"]).split(" at face ")[1].split()[0]
        assert f"at face {face} " in str(ei.value)
        return
    r = p.compute_residual(fx.u0, 0.0, 1)
    np.testing.assert_array_equal(r, fx["stage_residual"])
    np.testing.assert_array_equal(p.labels(), fx["stage_labels"])
    L, Rr = p.face_values()
    w = fx.written_right()
    np.testing.assert_array_equal(L, fx["stage_left"])
    np.testing.assert_array_equal(Rr[w], fx["stage_right"][w])
    np.testing.assert_array_equal(p.dofs(), fx["stage_dofs"])
    if fx.options.mode == A.HYBRID:
        np.testing.assert_array_equal(p.bounds(), fx["stage_bounds"])
    # two SSP-RK3 steps
    p2 = P.PortSolver(fx.mesh_view, fx.stencil_view, fx.options, fx.bcs, keep=(fx,))
    p2.state = fx.u0.copy()
    t = 0.0
    for k in range(2):
        dt = p2.max_stable_dt()
        assert dt == fx["rk3_dt"][k]
        p2.advance(dt, t, A.RK3)
        t += dt
        np.testing.assert_array_equal(np.bincount(p2.labels(step=True), minlength=4), fx["rk3_census"][k])
    np.testing.assert_array_equal(p2.state, fx["rk3_state"])
    np.testing.assert_array_equal(p2.labels(step=True), fx["rk3_step_labels"])
    # one SSPRK(5,4) step (Solver::advance)
    p3 = P.PortSolver(fx.mesh_view, fx.stencil_view, fx.options, fx.bcs, keep=(fx,))
    p3.state = fx.u0.copy()
    dt = p3.max_stable_dt()
    assert dt == fx["rk54_dt"][0]
    p3.advance(dt, 0.0, A.RK54)
    np.testing.assert_array_equal(p3.state, fx["rk54_state"])


LIVE = [
    # nx, ny, rect, jitter, periodic axis, order, ic, params, options, bcs
    (24, 24, (0, 0, 1, 1), 0.1, 3, 2, 0, [10.0], dict(mode="hybrid", lambda1p=1e4), {}),
    (24, 24, (0, 0, 1, 1), 0.1, 3, 3, 2, [0.5, 0.5, 0.01], dict(mode="hybrid"), {}),
    (20, 20, (0, 0, 1, 1), 0.1, 3, 4, 0, [10.0], dict(mode="hybrid", lambda1p=1e4), {}),
    (48, 8, (-5, 0, 5, 1), 0.1, 2, 2, 1, [-4.0, 3.857143, 2.629369, 0.0, 10.33333, 0.2, 5.0], dict(mode="hybrid"),
     {"left": "outflow", "right": "outflow"}),
    (24, 24, (0, 0, 1, 1), 0.1, 3, 2, 2, [0.5, 0.5, 0.01],
     dict(mode="hybrid", limiter=A.VENKATAKRISHNAN, si_exponent=A.SI_LEGACY, weno_b=3.0), {}),
    (24, 24, (0, 0, 1, 1), 0.1, 3, 3, 0, [10.0], dict(mode="cwenoz"), {}),
]


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("case", LIVE, ids=[f"live{i}" for i in range(len(LIVE))])
def test_port_matches_live_reference(case):
    nx, ny, rect, jit, per, order, ic, prm, opts, bcs = case
    nq = (order + 2) // 2
    m = R.RefMesh.structured_tri(nx, ny, rect, jitter=jit, seed=2, periodic=per, n_qp=nq)
    o = A.options_from_dict(order=order, cfl=0.5, **opts)
    bcl = make_bcs(bcs)
    s = R.RefSolver(m, o, bcl)
    p = P.PortSolver(m.view(), s.stencil_view(), o, bcl, keep=(m, s))
    u0 = m.project_initial(ic, prm, seed=9, degree=max(2 * order, 2))
    np.testing.assert_array_equal(p.compute_residual(u0, 0.0, 1), s.compute_residual(u0, 0.0, 1))
    np.testing.assert_array_equal(p.labels(), s.labels())
    s.set_state(u0)
    p.state = u0.copy()
    t = 0.0
    for _ in range(3):
        dt = s.max_stable_dt()
        assert dt == p.max_stable_dt()
        s.advance(dt, t, A.RK3)
        p.advance(dt, t, A.RK3)
        t += dt
    np.testing.assert_array_equal(p.state, s.get_state())
