"""BASELINE.json configurations at full size on the GPU.

* Config 2 (262,144 cells): against the compiled reference (oracle/_ref) on the
  same mesh/seed -- one stage (labels identical, residual within 1e-10) and
  two SSP-RK3 steps (census identical, L1 within 1e-8).
* Configs 2 and 3 for their configured step counts (200 / 50) against the
  committed record of the reference's own full-length run.
* Config 3 (8,388,608 cells, p=3): size-independent properties -- discrete
  conservation on the fully periodic domain, run-to-run bit-determinism, and
  (at quarter scale) a 4-subdomain decomposition reproducing the single-domain
  state bit-for-bit.
"""
import numpy as np
import pytest

from oracle import ref as R
from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.decompose import Subdomain, partition_rcb
from paper_2510_25906_b200.mesh import Mesh, Stencils
from paper_2510_25906_b200.solver import Solver, make_bcs
from tests.cases import case, scaled_err
from tests.decomp_driver import local_exchange, run_rk3

pytestmark = pytest.mark.gpu


def product_case(name, scale=1):
    mk, order, ic, prm, opts, bcs = case(name, scale)
    nq = (order + 2) // 2
    mesh = Mesh.structured_tri(mk["nx"], mk["ny"], mk["rect"], jitter=mk["jitter"], seed=1, periodic=mk["periodic"],
                               n_qp=nq)
    st = Stencils(mesh, order)
    u0 = mesh.project_initial(ic, prm, seed=1, degree=max(2 * order, 2))
    return mk, order, ic, prm, opts, bcs, mesh, st, u0


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not shipped")
def test_config2_full_size_against_reference():
    mk, order, ic, prm, opts, bcs, mesh, st, u0 = product_case("config2")
    o = A.options_from_dict(order=order, **opts)
    rm = R.RefMesh.structured_tri(mk["nx"], mk["ny"], mk["rect"], jitter=mk["jitter"], seed=1, periodic=2, n_qp=2)
    rs = R.RefSolver(rm, o, make_bcs(bcs))
    g = Solver(mesh, o, make_bcs(bcs), stencils=st)
    r_ref = rs.compute_residual(u0, 0.0, 1)
    r_gpu = g.compute_residual(u0, 0.0)
    np.testing.assert_array_equal(g.labels(), rs.labels())
    assert g.nad_ties() == 0
    assert scaled_err(r_gpu, r_ref) <= 1e-10
    rs.set_state(u0)
    g.state = u0
    _, _, cen_ref = rs.run_steps(2, A.RK3, census=True)
    _, cen_gpu = g.run_steps(2, A.RK3, census=True)
    np.testing.assert_array_equal(cen_gpu, cen_ref)
    ug, ur = g.state, rs.get_state()
    assert np.sum(np.abs(ug - ur)) / np.sum(np.abs(ur)) <= 1e-8


@pytest.mark.parametrize("name", ["config2", "config3"])
def test_full_length_against_reference_run(name):
    """The configured step count at full size against the committed record of
    the compiled reference's own run (tests/golden/make_fullsize_refs.py;
    reference loop run.cpp:97-132 over solver.cpp:316-379): identical input
    state, the census of step labels identical on EVERY step, dt equal every
    step, and the final conserved variables within L1 1e-8 (relative, per
    variable, on the stored 65,536-cell sample; per-variable L1 norms and
    1024 block sums likewise)."""
    import json
    from pathlib import Path

    from tests.fullsize_digest import sha256, summarise

    gold = Path(__file__).resolve().parent / "golden"
    if not (gold / f"fullsize_{name}.npz").exists():
        pytest.skip(f"no committed reference run for {name}")
    meta = json.loads((gold / f"fullsize_{name}.json").read_text())
    ref = np.load(gold / f"fullsize_{name}.npz")
    mk, order, ic, prm, opts, bcs, mesh, st, u0 = product_case(name)
    assert mesh.n_cells == meta["cells"]
    assert sha256(u0) == meta["u0_sha256"]  # the product setup reproduces the reference's initial state
    o = A.options_from_dict(order=order, **opts)
    g = Solver(mesh, o, make_bcs(bcs), stencils=st)
    del st
    g.state = u0
    n = meta["steps"]
    t, cen, dts = g.run_log(n, A.RK3)
    ties = g.nad_ties()
    np.testing.assert_array_equal(cen, ref["census"])
    # dt is a min over cells of the state: bit-equal while the states are; the
    # tau^b ulp differences of CWENOZ cells may move it in the last bits
    assert np.max(np.abs(dts - ref["dt"]) / ref["dt"]) <= 1e-12
    assert abs(t - float(ref["t"])) <= 1e-12 * float(ref["t"])
    u = g.state
    idx = ref["sample_idx"]
    us, ur = u[idx], ref["sample_state"]
    l1 = np.abs(us - ur).sum(0) / np.abs(ur).sum(0)
    assert np.all(l1 <= 1e-8), l1
    dg = summarise(u)
    assert np.all(np.abs(dg["l1"] - ref["l1"]) <= 1e-8 * ref["l1"])
    assert np.all(np.abs(dg["block_sum"] - ref["block_sum"]) <= 1e-8 * ref["block_abs"])
    print(f"{name}: {n} steps, census identical, max dt rel diff "
          f"{np.max(np.abs(dts - ref['dt']) / ref['dt']):.2e}, sample L1 rel {l1.max():.2e}, "
          f"final state bit-identical: {dg['sha256'] == meta['final_sha256']}, NAD ties {ties}")


def test_config3_full_size_conservation_and_determinism():
    mk, order, ic, prm, opts, bcs, mesh, st, u0 = product_case("config3")
    assert mesh.n_cells == 8_388_608
    o = A.options_from_dict(order=order, **opts)
    g = Solver(mesh, o, stencils=st)
    area = np.ctypeslib.as_array(mesh.view.cell_area, shape=(mesh.n_cells,)).copy()
    g.state = u0
    t1, cen = g.run_steps(2, A.RK3, census=True)
    u1 = g.state
    # discrete conservation on the periodic domain (telescoping face fluxes)
    tot0 = (u0 * area[:, None]).sum(0)
    tot1 = (u1 * area[:, None]).sum(0)
    scale = np.abs(u0 * area[:, None]).sum(0)
    assert np.all(np.abs(tot1 - tot0) <= 1e-12 * scale)
    assert cen.sum(1).tolist() == [mesh.n_cells] * 2
    # bit-determinism: the same run again
    g.state = u0
    t2, cen2 = g.run_steps(2, A.RK3, census=True)
    assert t2 == t1
    np.testing.assert_array_equal(cen2, cen)
    np.testing.assert_array_equal(g.state, u1)


def test_config3_quarter_scale_decomposition_bit_exact():
    mk, order, ic, prm, opts, bcs, mesh, st, u0 = product_case("config3", scale=4)
    o = A.options_from_dict(order=order, **opts)
    single = Solver(mesh, o, stencils=st)
    single.state = u0
    t_ref = 0.0
    for _ in range(2):
        dt = single.max_stable_dt()
        single.advance(dt, t_ref, A.RK3)
        t_ref += dt
    ref = single.state
    del single
    n = 4
    part = partition_rcb(mesh, n)
    subs = [Subdomain(mesh, st, part, n, r) for r in range(n)]

    class Rank:
        def __init__(self, sub):
            self.g = Solver.on_subdomain(sub, o)
            self.sub = sub
            self.last_census = np.zeros(4, dtype=np.int64)

        def max_stable_dt(self, u):
            self.g.state = u
            return self.g.max_stable_dt()

        def residual(self, u, t, first):
            return self.g.compute_residual(u, t)

        def record_census(self):
            self.last_census = np.bincount(self.g.labels()[: self.sub.n_owned], minlength=4)

    ranks = [Rank(s) for s in subs]
    states = [s.local_state(u0) for s in subs]
    t, _ = run_rk3(ranks, subs, states, 2, local_exchange, min)
    assert t == t_ref
    out = np.zeros_like(u0)
    for s, u in zip(subs, states):
        out[s.gid[: s.n_owned]] = u[: s.n_owned]
    np.testing.assert_array_equal(out, ref)


@pytest.mark.parametrize("name,scale", [("config2", 1), ("config3", 4)])
def test_class_list_policies_bit_identical(name, scale):
    """Chunk lists and per-cell lists give the same state and the same list
    statistics; the statistics agree with the last stage's labels (a listed
    cell whose reconstruction fell back to first order is labelled 3)."""
    mk, order, ic, prm, opts, bcs, mesh, st, u0 = product_case(name, scale)
    o = A.options_from_dict(order=order, **opts)
    g = Solver(mesh, o, make_bcs(bcs), stencils=st)
    out = {}
    for pol in ("lists", "chunks"):
        g.set_list_policy(pol)
        g.state = u0
        g.run_steps(2, A.RK3)
        out[pol] = (g.state, g.list_stats(), g.labels())
    np.testing.assert_array_equal(out["lists"][0], out["chunks"][0])
    np.testing.assert_array_equal(out["lists"][2], out["chunks"][2])
    sl, sc, lab = out["lists"][1], out["chunks"][1], out["chunks"][2]
    assert sl.pop("lists") == "per-cell" and sc.pop("lists") == "chunks"
    assert sl == sc
    pad = lambda m: np.pad(m, (0, -len(m) % 32)).reshape(-1, 32)
    n1, n2, n3 = (int((lab == k).sum()) for k in (1, 2, 3))
    assert n1 <= sc["cwenoz_cells"] and n2 <= sc["muscl_cells"]
    assert sc["cwenoz_cells"] + sc["muscl_cells"] <= n1 + n2 + n3
    assert int(pad(lab == 1).any(1).sum()) <= sc["cwenoz_chunks"] <= int(pad(lab >= 1).any(1).sum())
    assert int(pad(lab == 2).any(1).sum()) <= sc["muscl_chunks"] <= int(pad(lab >= 1).any(1).sum())
    assert 32 * sc["cwenoz_chunks"] >= sc["cwenoz_cells"] and 32 * sc["muscl_chunks"] >= sc["muscl_cells"]


@pytest.mark.parametrize("policy", ["chunks", "lists"])
def test_wide_spread_ragged_mesh_against_oracle(policy):
    """A jittered p = 2 mesh of 727 x 727 x 2 = 1,057,058 triangles: above the size where
    k_spread runs eight cells per thread, and not a multiple of its 1,024-cell block (nor of the
    32-cell chunk), with all three NAD classes present (shock into a sine wave, periodic in y,
    transmissive in x). One stage and one SSP-RK3 step against the oracle port: labels identical,
    residual within 1e-10, with chunk lists and with per-cell lists."""
    from oracle.port import PortSolver
    from tests.cases import SHOCK_SINE

    mesh = Mesh.structured_tri(727, 727, (-5.0, 0.0, 5.0, 1.0), jitter=0.1, seed=5, periodic="y", n_qp=2)
    assert mesh.n_cells == 1_057_058 and mesh.n_cells % 1024 != 0 and mesh.n_cells % 32 != 0
    st = Stencils(mesh, 2)
    bcs = make_bcs({"left": "outflow", "right": "outflow"})
    o = A.options_from_dict(order=2, mode="hybrid", lambda1p=1e3, cfl=0.5)
    u0 = mesh.project_initial(1, SHOCK_SINE, seed=1, degree=4)
    g = Solver(mesh, o, bcs, stencils=st)
    g.set_list_policy(policy)
    cpu = PortSolver(mesh.view, st.view, o, bcs, keep=(mesh, st))
    r_gpu = g.compute_residual(u0, 0.0)
    r_cpu = cpu.compute_residual(u0, 0.0, 1)
    lab = g.labels()
    np.testing.assert_array_equal(lab, cpu.labels())
    census = np.bincount(lab, minlength=4)
    assert census[0] > 0 and census[1] > 0 and census[2] > 0, census
    assert scaled_err(r_gpu, r_cpu) <= 1e-10
    g.state = u0
    cpu.state = u0.copy()
    dt = g.max_stable_dt()
    assert dt == cpu.max_stable_dt()
    g.advance(dt, 0.0, A.RK3)
    cpu.advance(dt, 0.0, A.RK3)
    np.testing.assert_array_equal(g.step_labels(), cpu.labels(step=True))
    assert scaled_err(g.state, cpu.state) <= 1e-10
