"""GPU parity: the sm_100a stage pass (through the C ABI) against the oracle.

The oracle is oracle/ucfv_port.c (plain-C restatement, pinned bit-exact to the
compiled reference by test_oracle_pin.py) fed the SAME flat mesh/stencil views,
and, where it travelled with the snapshot, the compiled reference itself
(oracle/_ref).

Tolerances (north_star): NAD labels identical (cells within 1e-12 of a
threshold excepted -- counted via ucfvb_get_nad_ties, zero on these cases);
face values and residuals within 1e-10 relative after one stage (residuals
relative to the field's per-variable scale); conserved variables within 1e-8
after N steps. Paths without CWENOZ cells are checked bit-for-bit: the only
non-bit-faithful operation is tau^b inside CWENOZ (CUDA vs glibc pow, <= 1 ulp).
"""
import numpy as np
import pytest

from oracle import port as P
from oracle import ref as R
from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.mesh import Mesh, Stencils
from paper_2510_25906_b200.solver import Solver, make_bcs
from tests.cases import case, rel_err, scaled_err

pytestmark = pytest.mark.gpu


def build(nx, ny, rect, jitter, periodic, order, ic, params, opts, bcs, seed=7, quads=False):
    nq = (order + 2) // 2
    if quads:
        mesh = Mesh.structured_quad(nx, ny, rect, periodic=periodic, n_qp=nq)
    else:
        mesh = Mesh.structured_tri(nx, ny, rect, jitter=jitter, seed=seed, periodic=periodic, n_qp=nq)
    st = Stencils(mesh, order, opts.get("si_exponent", A.SI_PAPER))
    o = A.options_from_dict(order=order, keep_taps=1, **opts)
    u0 = mesh.project_initial(ic, params, seed=3, degree=max(2 * order, 2))
    bcl = make_bcs(bcs)
    gpu = Solver(mesh, o, bcl, stencils=st)
    cpu = P.PortSolver(mesh.view, st.view, o, bcl, keep=(mesh, st))
    return mesh, st, o, u0, gpu, cpu


STAGE_CASES = [
    # name, mesh args, order, ic, params, opts, bcs
    ("hybrid-p2-vortex", (16, 16, (0, 0, 1, 1), 0.1, "both"), 2, 0, [10.0], dict(mode="hybrid", lambda1p=1e4), {}),
    ("hybrid-p3-quadrants", (16, 16, (0, 0, 1, 1), 0.1, "both"), 3, 2, [0.5, 0.5, 0.01], dict(mode="hybrid"), {}),
    ("hybrid-p1-quadrants", (16, 16, (0, 0, 1, 1), 0.1, "both"), 1, 2, [0.5, 0.5, 0.01], dict(mode="hybrid"), {}),
    ("hybrid-p2-shock-outflow", (64, 8, (-5, 0, 5, 1), 0.1, "y"), 2, 1,
     [-4.0, 3.857143, 2.629369, 0.0, 10.33333, 0.2, 5.0], dict(mode="hybrid"), {"left": "outflow", "right": "outflow"}),
    ("hybrid-p2-venkat-hll", (16, 16, (0, 0, 1, 1), 0.1, "both"), 2, 2, [0.5, 0.5, 0.01],
     dict(mode="hybrid", limiter=A.VENKATAKRISHNAN, riemann=A.HLL), {}),
    ("hybrid-p2-frozen", (16, 16, (0, 0, 1, 1), 0.1, "both"), 2, 2, [0.5, 0.5, 0.01],
     dict(mode="hybrid", detect_every_stage=0), {}),
    ("hybrid-p2-legacy-si", (16, 16, (0, 0, 1, 1), 0.1, "both"), 2, 2, [0.5, 0.5, 0.01],
     dict(mode="hybrid", si_exponent=A.SI_LEGACY), {}),
    ("hybrid-p2-wall-fixed", (24, 12, (0, 0, 2, 1), 0.1, "none"), 2, 2, [1.0, 0.5, 0.01],
     dict(mode="hybrid"), {"left": ("fixed", (1.0, 0.5, 0.0, 2.6)), "right": "outflow", "bottom": "wall",
                           "top": "wall"}),
    ("cwenoz-p2", (16, 16, (0, 0, 1, 1), 0.1, "both"), 2, 0, [10.0], dict(mode="cwenoz", lambda1p=1e4), {}),
    ("cwenoz-p3-b3", (16, 16, (0, 0, 1, 1), 0.1, "both"), 3, 0, [10.0], dict(mode="cwenoz", weno_b=3.0), {}),
]
BITWISE_CASES = [
    ("linear-p2", (16, 16, (0, 0, 1, 1), 0.1, "both"), 2, 0, [10.0], dict(mode="linear"), {}),
    ("linear-p3", (16, 16, (0, 0, 1, 1), 0.1, "both"), 3, 0, [10.0], dict(mode="linear"), {}),
    ("muscl-p2", (16, 16, (0, 0, 1, 1), 0.1, "both"), 2, 2, [0.5, 0.5, 0.01], dict(mode="muscl"), {}),
    ("muscl-p3-venkat", (16, 16, (0, 0, 1, 1), 0.1, "both"), 3, 2, [0.5, 0.5, 0.01],
     dict(mode="muscl", limiter=A.VENKATAKRISHNAN), {}),
    ("first-p2", (16, 16, (0, 0, 1, 1), 0.1, "both"), 2, 2, [0.5, 0.5, 0.01], dict(mode="first"), {}),
    ("linear-p2-quads", (12, 12, (0, 0, 1, 1), 0.0, "both"), 2, 0, [10.0], dict(mode="linear"), {}),
    # tau^1 is exact in glibc and on the device: the whole hybrid/CWENOZ path is then bit-faithful
    ("hybrid-p2-b1", (16, 16, (0, 0, 1, 1), 0.1, "both"), 2, 2, [0.5, 0.5, 0.01], dict(mode="hybrid", weno_b=1.0), {}),
    ("hybrid-p3-b1", (16, 16, (0, 0, 1, 1), 0.1, "both"), 3, 2, [0.5, 0.5, 0.01], dict(mode="hybrid", weno_b=1.0), {}),
    ("cwenoz-p2-b1", (16, 16, (0, 0, 1, 1), 0.1, "both"), 2, 0, [10.0], dict(mode="cwenoz", weno_b=1.0), {}),
    ("hybrid-p2-b1-shock", (64, 8, (-5, 0, 5, 1), 0.1, "y"), 2, 1,
     [-4.0, 3.857143, 2.629369, 0.0, 10.33333, 0.2, 5.0], dict(mode="hybrid", weno_b=1.0),
     {"left": "outflow", "right": "outflow"}),
]


def _stage(c, quads=False):
    name, (nx, ny, rect, jit, per), order, ic, prm, opts, bcs = c
    mesh, st, o, u0, gpu, cpu = build(nx, ny, rect, jit, per, order, ic, prm, opts, bcs, quads=quads)
    rg = gpu.compute_residual(u0, 0.0)
    rc = cpu.compute_residual(u0, 0.0, 1)
    return mesh, gpu, cpu, u0, rg, rc


def _written_right(mesh):
    """val_right_ slots the reference writes (interior faces only)."""
    v = mesh.view
    right = np.ctypeslib.as_array(v.face_right, shape=(v.n_faces,))
    return np.repeat(right >= 0, v.n_qp)


@pytest.mark.parametrize("c", STAGE_CASES, ids=[c[0] for c in STAGE_CASES])
def test_stage_matches_oracle(c, kernel_path):
    mesh, gpu, cpu, u0, rg, rc = _stage(c)
    np.testing.assert_array_equal(gpu.labels(), cpu.labels())
    assert gpu.nad_ties() == 0
    Lg, Rg = gpu.face_values()
    Lc, Rc = cpu.face_values()
    w = _written_right(mesh)
    assert rel_err(Lg, Lc) <= 1e-10
    assert rel_err(Rg[w], Rc[w]) <= 1e-10
    assert scaled_err(rg, rc) <= 1e-10
    assert rel_err(gpu.dofs(), cpu.dofs()) <= 1e-10 or np.allclose(gpu.dofs(), cpu.dofs(), rtol=1e-10, atol=1e-14)


@pytest.fixture(params=["fast", "cells", "generic"])
def kernel_path(request, monkeypatch):
    """fast: compile-time stencil sizes (uniform meshes), troubled cells over
    chunk lists; cells: the same over dense per-cell lists with per-cell
    operator records (k_troubled_cells); generic: runtime sizes."""
    if request.param == "generic":
        monkeypatch.setenv("UCFVB_FORCE_GENERIC", "1")
    if request.param == "cells":
        monkeypatch.setenv("UCFVB_TROUBLED", "lists")
    if request.param == "fast":
        monkeypatch.setenv("UCFVB_TROUBLED", "chunks")
    return request.param


@pytest.mark.parametrize("c", BITWISE_CASES, ids=[c[0] for c in BITWISE_CASES])
def test_stage_bitwise(c, kernel_path):
    mesh, gpu, cpu, u0, rg, rc = _stage(c, quads=c[0].endswith("quads"))
    np.testing.assert_array_equal(gpu.labels(), cpu.labels())
    Lg, Rg = gpu.face_values()
    Lc, Rc = cpu.face_values()
    w = _written_right(mesh)
    np.testing.assert_array_equal(Lg, Lc)
    np.testing.assert_array_equal(Rg[w], Rc[w])
    np.testing.assert_array_equal(rg, rc)


@pytest.mark.parametrize("rk", [A.RK3, A.RK54], ids=["rk3", "rk54"])
@pytest.mark.parametrize("c", [STAGE_CASES[0], STAGE_CASES[1], STAGE_CASES[3], STAGE_CASES[5]],
                         ids=["vortex-p2", "quadrants-p3", "shock-p2", "frozen"])
def test_steps_match_oracle(c, rk):
    name, (nx, ny, rect, jit, per), order, ic, prm, opts, bcs = c
    mesh, st, o, u0, gpu, cpu = build(nx, ny, rect, jit, per, order, ic, prm, opts, bcs)
    gpu.state = u0
    cpu.state = u0.copy()
    t = 0.0
    for _ in range(4):
        dg, dc = gpu.max_stable_dt(), cpu.max_stable_dt()
        assert abs(dg - dc) <= 1e-12 * dc
        gpu.advance(dc, t, rk)
        cpu.advance(dc, t, rk)
        t += dc
        np.testing.assert_array_equal(gpu.step_labels(), cpu.labels(step=True))
    ug, uc = gpu.state, cpu.state
    assert rel_err(ug, uc) <= 1e-8
    assert np.sum(np.abs(ug - uc)) / np.sum(np.abs(uc)) <= 1e-12


def test_run_steps_equals_advance_loop():
    """device-side dt/t loop (ucfvb_run_steps, CUDA graphs) == host loop of max_stable_dt + advance"""
    c = STAGE_CASES[1]
    name, (nx, ny, rect, jit, per), order, ic, prm, opts, bcs = c
    mesh, st, o, u0, gpu, cpu = build(nx, ny, rect, jit, per, order, ic, prm, opts, bcs)
    gpu2 = Solver(mesh, A.options_from_dict(order=order, **opts), stencils=st)
    gpu.state = u0
    gpu2.state = u0
    t = 0.0
    for _ in range(5):
        dt = gpu.max_stable_dt()
        gpu.advance(dt, t, A.RK3)
        t += dt
    t2, census = gpu2.run_steps(5, A.RK3, 0.0, float("inf"), census=True)
    assert t2 == t
    np.testing.assert_array_equal(gpu.state, gpu2.state)
    np.testing.assert_array_equal(census[-1], np.bincount(gpu.step_labels(), minlength=4))
    # graph replay without census gives the same state as well
    gpu3 = Solver(mesh, A.options_from_dict(order=order, **opts), stencils=st)
    gpu3.state = u0
    t3, _ = gpu3.run_steps(5, A.RK3)
    assert t3 == t
    np.testing.assert_array_equal(gpu3.state, gpu.state)
    assert gpu3.launch_count() > 0


def test_run_steps_t_end_clamp():
    c = STAGE_CASES[0]
    name, (nx, ny, rect, jit, per), order, ic, prm, opts, bcs = c
    mesh, st, o, u0, gpu, cpu = build(nx, ny, rect, jit, per, order, ic, prm, opts, bcs)
    gpu.state = u0
    dt = gpu.max_stable_dt()
    t_end = 2.5 * dt
    t, _ = gpu.run_steps(3, A.RK3, 0.0, t_end)
    assert abs(t - t_end) <= 1e-15 * t_end


def test_nonphysical_raises_and_keeps_state():
    c = STAGE_CASES[1]
    name, (nx, ny, rect, jit, per), order, ic, prm, opts, bcs = c
    mesh, st, o, u0, gpu, cpu = build(nx, ny, rect, jit, per, order, ic, prm, dict(mode="linear"), bcs)
    bad = u0.copy()
    bad[:, 3] = 0.05 * bad[:, 3]  # negative pressure everywhere
    gpu.state = bad
    with pytest.raises(A.NonPhysicalError):
        gpu.max_stable_dt()
    np.testing.assert_array_equal(gpu.state, bad)
    with pytest.raises(A.NonPhysicalError):
        gpu.advance(1e-4, 0.0, A.RK3)
    np.testing.assert_array_equal(gpu.state, bad)
    with pytest.raises(A.NonPhysicalError):
        gpu.compute_residual(bad, 0.0)
    with pytest.raises(P.PortError):
        cpu.compute_residual(bad, 0.0, 1)
    # the handle stays usable
    gpu.state = u0
    assert gpu.max_stable_dt() > 0


def test_invalid_arguments():
    mesh = Mesh.structured_tri(8, 8, (0, 0, 1, 1), periodic="none", n_qp=2)
    st = Stencils(mesh, 2)
    with pytest.raises(A.InvalidArgument, match="no boundary condition"):
        Solver(mesh, A.options_from_dict(order=2), {}, stencils=st)
    with pytest.raises(A.InvalidArgument, match="unknown boundary patch"):
        Solver(mesh, A.options_from_dict(order=2), {"nope": "outflow"}, stencils=st)
    bad = A.options_from_dict(order=2, margins=(-1.0, 0.5, 0.0, 0.0, 5.0, 2.0))
    with pytest.raises(A.InvalidArgument, match="alpha_m"):
        Solver(mesh, bad, {"left": "outflow", "right": "outflow", "bottom": "wall", "top": "wall"}, stencils=st)


def test_conservation_and_freestream_config1():
    """size-independent properties at BASELINE config-1 size (32,768 cells)."""
    mk, order, ic, prm, opts, bcs = case("config1")
    mesh = Mesh.structured_tri(mk["nx"], mk["ny"], mk["rect"], jitter=mk["jitter"], seed=1, periodic="both", n_qp=2)
    st = Stencils(mesh, order)
    gpu = Solver(mesh, A.options_from_dict(order=order, **opts), stencils=st)
    area = np.ctypeslib.as_array(mesh.view.cell_area, shape=(mesh.n_cells,)).copy()
    u0 = mesh.project_initial(ic, prm, degree=4)
    gpu.state = u0
    gpu.run_steps(10, A.RK3)
    u = gpu.state
    tot0 = (u0 * area[:, None]).sum(0)
    tot = (u * area[:, None]).sum(0)
    assert np.all(np.abs(tot - tot0) <= 1e-12 * np.abs(u0 * area[:, None]).sum(0))
    free = np.tile([1.0, 1.0, 1.0, 2.5 + 1.0], (mesh.n_cells, 1))
    r = gpu.compute_residual(free, 0.0)
    assert np.max(np.abs(r)) <= 1e-10


@pytest.mark.skipif(not R.available(), reason="oracle/_ref (compiled reference) not shipped")
@pytest.mark.parametrize("cfg,scale,steps", [("config1", 1, 10), ("config2", 8, 20), ("config3", 32, 5)])
def test_against_compiled_reference(cfg, scale, steps):
    """The unmodified reference (oracle/_ref) on the same mesh, seed and RK3 driver."""
    mk, order, ic, prm, opts, bcs = case(cfg, scale)
    nq = (order + 2) // 2
    per = {"both": 3, "y": 2}[mk["periodic"]]
    rm = R.RefMesh.structured_tri(mk["nx"], mk["ny"], mk["rect"], jitter=mk["jitter"], seed=1, periodic=per, n_qp=nq)
    o = A.options_from_dict(order=order, **opts)
    rs = R.RefSolver(rm, o, make_bcs(bcs))
    mesh = Mesh.structured_tri(mk["nx"], mk["ny"], mk["rect"], jitter=mk["jitter"], seed=1, periodic=mk["periodic"],
                               n_qp=nq)
    gpu = Solver(mesh, o, make_bcs(bcs))
    u0 = mesh.project_initial(ic, prm, seed=1, degree=max(2 * order, 2))
    np.testing.assert_array_equal(u0, rm.project_initial(ic, prm, seed=1, degree=max(2 * order, 2)))
    rs.set_state(u0)
    gpu.state = u0
    # one stage: labels + residual
    r_ref = rs.compute_residual(u0, 0.0, 1)
    r_gpu = gpu.compute_residual(u0, 0.0)
    np.testing.assert_array_equal(gpu.labels(), rs.labels())
    assert scaled_err(r_gpu, r_ref) <= 1e-10
    # N steps of RK3
    _, _, cen_ref = rs.run_steps(steps, A.RK3, census=True)
    _, cen_gpu = gpu.run_steps(steps, A.RK3, census=True)
    np.testing.assert_array_equal(cen_gpu, cen_ref)
    ug, ur = gpu.state, rs.get_state()
    l1 = np.sum(np.abs(ug - ur)) / np.sum(np.abs(ur))
    assert l1 <= 1e-8
