"""GPU parity of the 3D stage pass (sm_100a, through include/ucfvb3.h)
against the 3D oracle restatement (oracle/ucfv3_port.c) on identical views.

Bar (north_star): NAD labels identical (threshold ties counted, zero here);
face values / residuals within 1e-10 relative after one stage; conserved
variables within 1e-8 after the configured steps. Everything except the
CWENOZ tau^b (correctly rounded x^4 on the device vs glibc pow) is
bit-identical, so runs without CWENOZ cells are compared bit-for-bit.
"""
import numpy as np
import pytest

from oracle.port3 import Port3Solver
from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.solver3d import (HEX, IC_BLAST, IC_RANDOM_PHASE, IC_TGV, TET, Mesh3, Solver3,
                                            Stencils3)

pytestmark = pytest.mark.gpu

PARAMS = {IC_TGV: [0.1], IC_BLAST: [3.0, 3.2, 3.1, 1.6, 1.0, 8.0, 0.3, 0.5], IC_RANDOM_PHASE: [0.8, 2.0, 4]}


def build(kind, order, jitter, ic, n=5, classes=False, **opts):
    m = Mesh3(n, kind=kind, jitter=jitter, order=order, seed=7)
    st = Stencils3(m, order, lattice_classes=classes)
    o = A.options_from_dict(order=order, cfl=0.5, **opts)
    u0 = m.project_initial(ic, PARAMS[ic], seed=3)
    return m, st, o, u0, Solver3(m, o, st), Port3Solver(m, st, o)


def rel(a, b):
    scale = np.abs(b).max(axis=tuple(range(b.ndim - 1)), keepdims=True) + 1e-300
    return float(np.abs(a - b).max() / scale.min()) if a.size else 0.0


CASES = [
    (HEX, 2, 0.05, IC_BLAST, "hybrid", {}),
    (HEX, 2, 0.05, IC_TGV, "hybrid", {}),
    (TET, 3, 0.0, IC_BLAST, "hybrid", {}),
    (TET, 2, 0.05, IC_RANDOM_PHASE, "hybrid", {}),
    (HEX, 3, 0.0, IC_BLAST, "hybrid", {"limiter": A.VENKATAKRISHNAN}),
    (HEX, 1, 0.1, IC_BLAST, "hybrid", {"riemann": A.HLL}),
    (TET, 1, 0.05, IC_BLAST, "hybrid", {}),
    (HEX, 2, 0.05, IC_RANDOM_PHASE, "cwenoz", {}),
    (TET, 3, 0.0, IC_BLAST, "muscl", {}),
    (HEX, 2, 0.0, IC_BLAST, "linear", {}),
    (HEX, 2, 0.0, IC_TGV, "linear", {}),
    (TET, 2, 0.0, IC_BLAST, "first", {}),
    (HEX, 2, 0.05, IC_BLAST, "hybrid", {"weno_b": 1.0}),
    (TET, 2, 0.05, IC_BLAST, "hybrid", {"detect_every_stage": 0, "weno_b": 1.0}),
]


@pytest.mark.parametrize("kind,order,jitter,ic,mode,extra", CASES)
def test_stage_parity(kind, order, jitter, ic, mode, extra):
    m, st, o, u0, gpu, cpu = build(kind, order, jitter, ic, mode=mode, **extra)
    try:
        rg = gpu.compute_residual(u0)
    except A.NonPhysicalError as e:
        # unlimited modes can produce non-physical face states: the oracle must fail at the same face
        face = str(e).split("face ")[1]
        with pytest.raises(Exception, match=f"face {face}$"):
            cpu.compute_residual(u0)
        return
    rc = cpu.compute_residual(u0)
    lg, lc = gpu.labels(), cpu.labels()
    assert np.array_equal(lg, lc), f"labels differ at {np.nonzero(lg != lc)[0][:10]}"
    fg, fc = gpu.face_values(), cpu.face_values()
    exact = mode in ("linear", "muscl", "first") or extra.get("weno_b") == 1.0 or not np.any(lc == A.SCHEME_CWENOZ)
    if exact:
        assert np.array_equal(fg, fc)
        assert np.array_equal(rg, rc)
    else:
        assert rel(fg, fc) <= 1e-10
        assert rel(rg, rc) <= 1e-10
    assert gpu.nad_ties() == 0


@pytest.mark.parametrize("kind,order,jitter,ic,mode,extra", CASES[:8] + CASES[-1:])
def test_rk3_steps(kind, order, jitter, ic, mode, extra):
    m, st, o, u0, gpu, cpu = build(kind, order, jitter, ic, mode=mode, **extra)
    gpu.state = u0
    cpu.state = u0.copy()
    for _ in range(3):
        dg, dc = gpu.max_stable_dt(), cpu.max_stable_dt()
        assert dg == dc
        gpu.advance(dg, 0.0, A.RK3)
        cpu.advance(dc, 0.0, A.RK3)
        assert np.array_equal(gpu.step_labels(), cpu.labels(step=True))
    assert rel(gpu.state, cpu.state) <= 1e-8
    census = np.bincount(cpu.labels(step=True), minlength=4)
    assert gpu.census() == census.tolist()


def test_rk54_step():
    m, st, o, u0, gpu, cpu = build(TET, 2, 0.05, IC_BLAST, mode="hybrid", weno_b=1.0)
    gpu.state = u0
    cpu.state = u0.copy()
    dt = cpu.max_stable_dt()
    gpu.advance(dt, 0.0, A.RK54)
    cpu.advance(dt, 0.0, A.RK54)
    assert np.array_equal(gpu.state, cpu.state)


def test_run_steps_matches_advance():
    m, st, o, u0, gpu, cpu = build(HEX, 2, 0.05, IC_BLAST, mode="hybrid")
    gpu.state = u0
    t = gpu.run_steps(4, 0.0)
    a = gpu.state
    g2 = Solver3(m, o, st)
    g2.state = u0
    tt = 0.0
    for _ in range(4):
        dt = g2.max_stable_dt()
        g2.advance(dt, tt)
        tt += dt
    assert np.array_equal(a, g2.state)
    assert t == pytest.approx(tt, rel=1e-14)
    assert gpu.launch_count() > 0


def test_lattice_classes_match_port():
    m, st, o, u0, gpu, cpu = build(TET, 3, 0.0, IC_RANDOM_PHASE, n=8, classes=True, mode="hybrid", weno_b=1.0)
    assert m.view.cell_order == 1  # type-blocked numbering: the staged kernels run
    assert st.n_ops == 6
    gpu.state = u0
    cpu.state = u0.copy()
    for _ in range(2):
        dt = cpu.max_stable_dt()
        gpu.advance(dt)
        cpu.advance(dt)
    assert np.array_equal(gpu.state, cpu.state)


def test_forced_cwenoz_blast_fails_at_same_face():
    """Forced CWENOZ has no fallback (solver.cpp:343-368): the blast drives a
    face state non-physical; device and oracle name the same (first) face."""
    m, st, o, u0, gpu, cpu = build(HEX, 2, 0.05, IC_BLAST, mode="cwenoz")
    with pytest.raises(A.NonPhysicalError) as eg:
        gpu.compute_residual(u0)
    with pytest.raises(Exception) as ec:
        cpu.compute_residual(u0)
    face = str(eg.value).split("face ")[1]
    assert f"face {face}" in str(ec.value)


@pytest.mark.parametrize("rk", [A.RK3, A.RK54], ids=["rk3", "rk54"])
def test_failure_keeps_failing_step_input3(rk):
    """A non-physical failure inside a graph-replayed run leaves U at the
    failing step's input (the reference throws before touching state_): the
    step's result reaches U only through a commit gated on the error word,
    and every later kernel of the run exits."""
    m, st, o, u0, gpu, cpu = build(HEX, 2, 0.05, IC_BLAST, mode="cwenoz")
    gpu.state = u0
    with pytest.raises(A.NonPhysicalError, match="face"):
        gpu.run_steps(4, rk=rk)
    np.testing.assert_array_equal(gpu.state, u0)
    bad = u0.copy()
    bad[11, 0] = -1.0
    gpu.state = bad
    with pytest.raises(A.NonPhysicalError, match="cell 11"):
        gpu.run_steps(3, rk=rk)
    np.testing.assert_array_equal(gpu.state, bad)


def test_nonphysical_reports_face():
    m, st, o, u0, gpu, cpu = build(HEX, 2, 0.0, IC_BLAST, mode="first")
    u = u0.copy()
    u[17, 0] = -1.0
    with pytest.raises(A.NonPhysicalError):
        gpu.compute_residual(u)
    with pytest.raises(Exception):
        cpu.compute_residual(u)
    gpu.state = u
    with pytest.raises(A.NonPhysicalError, match="cell 17"):
        gpu.max_stable_dt()


@pytest.mark.parametrize("kind,order,n,classes", [(HEX, 2, 24, False), (TET, 3, 12, True)])
def test_larger_mesh_parity_and_conservation(kind, order, n, classes):
    """Mid-size meshes (13.8 k hexahedra / 10.4 k tetrahedra): 3 RK3 steps vs
    the oracle, conservation of every variable to 1e-13 of its scale."""
    m = Mesh3(n, kind=kind, jitter=0.05 if not classes else 0.0, order=order, seed=4)
    st = Stencils3(m, order, lattice_classes=classes)
    o = A.options_from_dict(order=order, cfl=0.5, mode="hybrid")
    ic = IC_TGV if kind == HEX else IC_RANDOM_PHASE
    u0 = m.project_initial(ic, {IC_TGV: [0.1], IC_RANDOM_PHASE: [0.6, 4.0, 6]}[ic], seed=3,
                           degree=4 if ic == IC_TGV else 1)
    gpu, cpu = Solver3(m, o, st), Port3Solver(m, st, o)
    gpu.state = u0
    cpu.state = u0.copy()
    for _ in range(3):
        dt = cpu.max_stable_dt()
        gpu.advance(dt)
        cpu.advance(dt)
        assert np.array_equal(gpu.step_labels(), cpu.labels(step=True))
    assert rel(gpu.state, cpu.state) <= 1e-8
    tot0 = (u0 * m.volume[:, None]).sum(0)
    tot = (gpu.state * m.volume[:, None]).sum(0)
    assert np.all(np.abs(tot - tot0) <= 1e-13 * np.abs(u0).max() * m.volume.sum())


class GpuRank3:
    def __init__(self, sub, opts):
        self.g = Solver3.on_subdomain(sub, opts)
        self.sub = sub
        self.last_census = np.zeros(4, dtype=np.int64)

    def max_stable_dt(self, u):
        self.g.state = u
        return self.g.max_stable_dt()

    def residual(self, u, t, first):
        return self.g.compute_residual(u, t)

    def record_census(self):
        self.last_census = np.bincount(self.g.labels()[: self.sub.n_owned], minlength=4)


@pytest.mark.parametrize("name", ["hex-p2-blast", "tet-p2-classes"])
@pytest.mark.parametrize("n_parts", [2, 4])
def test_gpu_subdomains_match_single_domain3(name, n_parts):
    from paper_2510_25906_b200.solver3d import Subdomain3, partition_rcb3
    from tests.decomp_driver import local_exchange, run_rk3
    from tests.test_decompose3 import setup3

    c, m, st, o, u0 = setup3(name)
    single = Solver3(m, o, st)
    single.state = u0
    t_ref, cen_ref = 0.0, []
    for _ in range(2):
        dt = single.max_stable_dt()
        single.advance(dt, t_ref)
        t_ref += dt
        cen_ref.append(single.census())
    part = partition_rcb3(m, n_parts)
    subs = [Subdomain3(m, st, part, n_parts, r) for r in range(n_parts)]
    ranks = [GpuRank3(s, o) for s in subs]
    states = [s.local_state(u0) for s in subs]
    t, census = run_rk3(ranks, subs, states, 2, local_exchange, min)
    assert t == t_ref
    out = np.zeros_like(u0)
    for s, u in zip(subs, states):
        out[s.gid[: s.n_owned]] = u[: s.n_owned]
    np.testing.assert_array_equal(out, single.state)
    for a, b in zip(census, cen_ref):
        np.testing.assert_array_equal(a, b)


def test_nccl_single_rank_path3():
    from paper_2510_25906_b200.solver import nccl_unique_id
    from paper_2510_25906_b200.solver3d import Subdomain3, partition_rcb3
    from tests.test_decompose3 import setup3

    c, m, st, o, u0 = setup3("hex-p2-blast")
    sub = Subdomain3(m, st, partition_rcb3(m, 1), 1, 0)
    g = Solver3.on_subdomain(sub, o)
    g.attach_nccl(nccl_unique_id(), 0, 1)
    g.state = sub.local_state(u0)
    plain = Solver3(m, o, st)
    plain.state = u0
    t1 = g.run_steps(3)
    t2 = plain.run_steps(3)
    assert t1 == t2
    np.testing.assert_array_equal(g.state[np.argsort(sub.gid)], plain.state)
    assert g.census() == plain.census()


@pytest.mark.parametrize("cfg,n,steps", [("4", 16, 100), ("4c", 12, 100), ("5", 8, 50)])
def test_configured_step_count_reduced_mesh(cfg, n, steps):
    """BASELINE configs 4/4c/5 on reduced meshes for their full step counts:
    the L1 norm of every conserved variable within 1e-8 (relative) of the
    3D oracle's, step labels identical at every step."""
    import bench
    c = bench.CONFIGS3[cfg]
    m, st, u0, _ = bench.build_case3(cfg, n=n)
    o = A.options_from_dict(order=c["order"], mode=c["mode"], cfl=0.5)
    gpu, cpu = Solver3(m, o, st), Port3Solver(m, st, o)
    gpu.state = u0
    cpu.state = u0.copy()
    for _ in range(steps):
        dt = cpu.max_stable_dt()
        assert gpu.max_stable_dt() == pytest.approx(dt, rel=1e-12)
        gpu.advance(dt)
        cpu.advance(dt)
        assert np.array_equal(gpu.step_labels(), cpu.labels(step=True))
    l1g = (np.abs(gpu.state) * m.volume[:, None]).sum(0)
    l1c = (np.abs(cpu.state) * m.volume[:, None]).sum(0)
    assert np.all(np.abs(l1g - l1c) <= 1e-8 * np.abs(l1c).max())


def test_advance_host_matches_run_steps3():
    m, st, o, u0, gpu, cpu = build(TET, 2, 0.05, IC_BLAST, mode="hybrid")
    out, t = gpu.advance_host(u0, 3)
    g2 = Solver3(m, o, st)
    g2.state = u0
    t2 = g2.run_steps(3)
    assert t == t2
    np.testing.assert_array_equal(out, g2.state)
    bad = u0.copy()
    bad[3, 0] = -1.0
    with pytest.raises(A.NonPhysicalError):
        gpu.advance_host(bad, 1)


def test_advance_host_batch_matches_serial3():
    """ucfvb3_advance_host_batch (pipelined uploads / downloads over independent states): every
    entry has the bits of its own ucfvb3_advance_host call; a failing entry is named and leaves
    the others untouched."""
    m, st, o, u0, gpu, cpu = build(TET, 2, 0.05, IC_BLAST, mode="hybrid")
    ins = [u0 * (1.0 + 0.03 * i) for i in range(5)]
    for n_steps in (1, 2):
        outs, ts = gpu.advance_host_batch(ins, n_steps)
        for u, out, t in zip(ins, outs, ts):
            ref, t_ref = gpu.advance_host(u, n_steps)
            assert t == t_ref
            np.testing.assert_array_equal(out, ref)
    bad = [u.copy() for u in ins]
    bad[2][3, 0] = -1.0
    with pytest.raises(A.NonPhysicalError, match="batch entry 2"):
        gpu.advance_host_batch(bad, 1)
    outs, _ = gpu.advance_host_batch(ins[:2], 1)
    np.testing.assert_array_equal(outs[1], gpu.advance_host(ins[1], 1)[0])


@pytest.mark.parametrize("order", [2, 3])
def test_staged_tensor_core_path_with_troubled_cells(order):
    """Type-blocked lattice-class mesh (8^3 cubes x 6 tets: staged rows, DMMA
    central / CWENOZ / OI.p1) with a blast, so the CWENOZ and MUSCL kernels have
    real work: labels, face values and states bit-identical to the oracle
    (weno_b = 1 keeps tau^b exact)."""
    m, st, o, u0, gpu, cpu = build(TET, order, 0.0, IC_BLAST, n=8, classes=True, mode="hybrid", weno_b=1.0)
    assert m.view.cell_order == 1 and st.n_ops == 6
    rg, rc = gpu.compute_residual(u0), cpu.compute_residual(u0)
    lab = cpu.labels()
    counts = np.bincount(lab, minlength=4)
    assert counts[1] > 50 and counts[2] > 50, counts  # CWENOZ and MUSCL cells present
    assert np.array_equal(gpu.labels(), lab)
    assert np.array_equal(gpu.face_values(), cpu.face_values())
    assert np.array_equal(rg, rc)
    gpu.state = u0
    cpu.state = u0.copy()
    for _ in range(2):
        dt = cpu.max_stable_dt()
        gpu.advance(dt)
        cpu.advance(dt)
        assert np.array_equal(gpu.step_labels(), cpu.labels(step=True))
    assert np.array_equal(gpu.state, cpu.state)
