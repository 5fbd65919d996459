"""run_simulation's loop on the device (ucfvb_run_until / run_steps_log) and
the run outputs, against the unmodified reference.

weno_b = 1 makes the whole step bit-exact (tau^b is then exact on both
sides), so dt, t, census and state are compared with equality; the files the
device run writes are compared byte-for-byte with the reference writers fed
the reference run's own rows and state."""
import numpy as np
import pytest

from oracle import ref as R
from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200 import run as RUN
from paper_2510_25906_b200.mesh import Mesh, Stencils
from paper_2510_25906_b200.solver import Solver, ViewHolder, make_bcs
from tests.cases import SHOCK_SINE, VORTEX

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not shipped")]


def pair(kind, weno_b=1.0):
    if kind == "vortex":
        mk = dict(nx=24, ny=24, rect=(0.0, 0.0, 1.0, 1.0), jitter=0.1)
        per, ic, prm, bcs, opts = 3, 0, VORTEX, {}, dict(lambda1p=1e4, cfl=0.5)
    else:
        mk = dict(nx=64, ny=8, rect=(-5.0, 0.0, 5.0, 1.0), jitter=0.1)
        per, ic, prm, bcs, opts = 2, 1, SHOCK_SINE, {"left": "outflow", "right": "outflow"}, dict(lambda1p=1e3,
                                                                                              cfl=0.5)
    o = A.options_from_dict(order=2, weno_b=weno_b, **opts)
    rm = R.RefMesh.structured_tri(mk["nx"], mk["ny"], mk["rect"], jitter=mk["jitter"], seed=1, periodic=per, n_qp=2)
    rs = R.RefSolver(rm, o, make_bcs(bcs))
    u0 = rm.project_initial(ic, prm, seed=1, degree=4)
    rs.set_state(u0)
    mesh = Mesh.structured_tri(mk["nx"], mk["ny"], mk["rect"], jitter=mk["jitter"], seed=1,
                               periodic={3: "both", 2: "y"}[per], n_qp=2)
    g = Solver(mesh, o, make_bcs(bcs), stencils=Stencils(mesh, 2))
    g.state = u0
    return rm, rs, g, u0


@pytest.mark.parametrize("rk", [A.RK3, A.RK54])
def test_run_log_dt_and_census_exact(rk):
    _, rs, g, _ = pair("shock")
    t_r, cen_r, dt_r = rs.run_log(4, rk)
    t_g, cen_g, dt_g = g.run_log(4, rk)
    assert t_g == t_r
    np.testing.assert_array_equal(dt_g, dt_r)
    np.testing.assert_array_equal(cen_g, cen_r)
    np.testing.assert_array_equal(g.state, rs.get_state())


@pytest.mark.parametrize("kind,rk", [("vortex", A.RK3), ("shock", A.RK3), ("vortex", A.RK54)])
def test_run_until_matches_reference_loop(kind, rk):
    _, rs, g, _ = pair(kind)
    dt0 = g.max_stable_dt()
    t_end = 3.7 * dt0  # a short last step: dt = t_end - t (run.cpp:100)
    t_r, cen_r, dt_r = rs.run_until(t_end, rk)
    t_g, n, cen_g, dt_g = g.run_until(t_end, rk, max_steps=50)
    assert n == len(dt_r) >= 4
    assert t_g == t_r
    np.testing.assert_array_equal(dt_g, dt_r)
    np.testing.assert_array_equal(cen_g, cen_r)
    np.testing.assert_array_equal(g.state, rs.get_state())
    # the loop has ended: a further call takes no step and leaves everything alone
    u = g.state
    t2, n2, _, _ = g.run_until(t_end, rk, t0=t_g, max_steps=50)
    assert n2 == 0 and t2 == t_g
    np.testing.assert_array_equal(g.state, u)


def test_run_until_resumes_across_max_steps():
    _, _, g1, u0 = pair("shock")
    t_end = 6.5 * g1.max_stable_dt()
    t_a, n_a, cen_a, dt_a = g1.run_until(t_end, max_steps=100)
    _, _, g2, _ = pair("shock")
    t, parts_c, parts_d, total = 0.0, [], [], 0
    while True:
        t, n, c, d = g2.run_until(t_end, t0=t, max_steps=2)
        parts_c.append(c)
        parts_d.append(d)
        total += n
        if n < 2:
            break
    assert total == n_a and t == t_a
    np.testing.assert_array_equal(np.concatenate(parts_d), dt_a)
    np.testing.assert_array_equal(np.concatenate(parts_c), cen_a)
    np.testing.assert_array_equal(g2.state, g1.state)


def test_run_until_already_at_end():
    _, _, g, u0 = pair("vortex")
    t, n, cen, dts = g.run_until(0.0, max_steps=5)
    assert n == 0 and t == 0.0 and len(dts) == 0
    np.testing.assert_array_equal(g.state, u0)


def test_run_simulation_files_match_reference_writers(tmp_path):
    rm, rs, g, _ = pair("shock")
    t_end = 5.5 * g.max_stable_dt()
    res = RUN.run_simulation(g, ViewHolder(rm.view(), keep=rm), t_end, out_dir=str(tmp_path / "ours"),
                             output_every=2)
    t_r, cen_r, dt_r = rs.run_until(t_end)
    assert res.steps == len(dt_r) and res.t == t_r
    ref_dir = tmp_path / "ref"
    ref_dir.mkdir()
    rows, t = [], 0.0
    for k in range(len(dt_r)):
        t += dt_r[k]
        rows.append((k + 1, t, dt_r[k], cen_r[k].tolist()))
    R.write_census_csv(rows, rm.n_cells, ref_dir / "census.csv")
    R.write_field_snapshot(rm, rs.get_state(), rs.labels(step=True), 1.4, ref_dir / "final.vtk")
    ours = tmp_path / "ours"
    assert (ours / "census.csv").read_bytes() == (ref_dir / "census.csv").read_bytes()
    assert (ours / f"fields_{res.steps}.vtk").read_bytes() == (ref_dir / "final.vtk").read_bytes()
    for s in range(2, res.steps, 2):  # output_every snapshots exist
        assert (ours / f"fields_{s}.vtk").stat().st_size > 0


def test_run_simulation_phase_timing_rows(tmp_path):
    rm, _, g, _ = pair("vortex")
    t_end = 2.5 * g.max_stable_dt()
    res = RUN.run_simulation(g, ViewHolder(rm.view(), keep=rm), t_end, out_dir=str(tmp_path), phase_timing=True)
    lines = (tmp_path / "timing.csv").read_text().splitlines()
    assert lines[0] == "step,wall,reconstruct,detect,weights,flux"
    assert res.steps >= 3 and len(lines) == 1 + res.steps
    vals = np.array([[float(x) for x in ln.split(",")] for ln in lines[1:]])
    assert np.all(vals[:, 2:] > 0.0) and np.all(np.diff(vals[:, 1]) > 0.0)


def test_advance_host_matches_run_steps():
    """ucfvb_advance_host (host state in/out, one synchronisation) is the same
    computation as set_state + run_steps + get_state."""
    import numpy as np
    from paper_2510_25906_b200 import _abi as A
    from paper_2510_25906_b200.mesh import Mesh, Stencils
    from paper_2510_25906_b200.solver import Solver

    mesh = Mesh.structured_tri(24, 24, (0.0, 0.0, 1.0, 1.0), jitter=0.1, seed=1, periodic="both", n_qp=2)
    st = Stencils(mesh, 2)
    o = A.options_from_dict(order=2, mode="hybrid", lambda1p=1e3, cfl=0.5)
    u0 = mesh.project_initial(2, [0.5, 0.5, 0.01], seed=3, degree=4)
    a = Solver(mesh, o, stencils=st)
    out, t = a.advance_host(u0, 3)
    b = Solver(mesh, o, stencils=st)
    b.state = u0
    t2, _ = b.run_steps(3, A.RK3)
    assert t == t2
    np.testing.assert_array_equal(out, b.state)
    bad = u0.copy()
    bad[5, 0] = -1.0
    import pytest
    with pytest.raises(A.NonPhysicalError):
        a.advance_host(bad, 1)


def test_advance_host_batch_matches_serial():
    """ucfvb_advance_host_batch (pipelined uploads / downloads over independent states)
    gives every entry the bits of its own ucfvb_advance_host call; a failing entry is named."""
    import numpy as np
    import pytest
    from paper_2510_25906_b200 import _abi as A
    from paper_2510_25906_b200.mesh import Mesh, Stencils
    from paper_2510_25906_b200.solver import Solver

    mesh = Mesh.structured_tri(24, 24, (0.0, 0.0, 1.0, 1.0), jitter=0.1, seed=1, periodic="both", n_qp=2)
    st = Stencils(mesh, 2)
    o = A.options_from_dict(order=2, mode="hybrid", lambda1p=1e3, cfl=0.5)
    ins = [mesh.project_initial(2, [0.5, 0.5, 0.01], seed=3 + i, degree=4) * (1.0 + 0.05 * i) for i in range(5)]
    a = Solver(mesh, o, stencils=st)
    for n_steps in (1, 2):
        outs, ts = a.advance_host_batch(ins, n_steps)
        for u, out, t in zip(ins, outs, ts):
            ref, t_ref = a.advance_host(u, n_steps)
            assert t == t_ref
            np.testing.assert_array_equal(out, ref)
    bad = [u.copy() for u in ins]
    bad[3][5, 0] = -1.0
    with pytest.raises(A.NonPhysicalError, match="batch entry 3"):
        a.advance_host_batch(bad, 1)
    # the solver is usable after the failure; one- and two-entry batches (no pipelining yet)
    outs, _ = a.advance_host_batch(ins[:2], 1)
    np.testing.assert_array_equal(outs[1], a.advance_host(ins[1], 1)[0])
    outs, ts = a.advance_host_batch(ins[4:5], 3)
    ref, t_ref = a.advance_host(ins[4], 3)
    assert ts[0] == t_ref
    np.testing.assert_array_equal(outs[0], ref)
