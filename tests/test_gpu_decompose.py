"""Subdomain solvers on the GPU (ucfvb_create_sub): N subdomains driven stage
by stage with a host halo refresh reproduce the single-domain GPU run
bit-for-bit on owned cells; the in-graph exchange schedule (sent cells first,
the halo exchange forked onto an exchange stream while the interior is
updated) over the loopback transport likewise; the NCCL path (dt/census/error
all-reduces inside the captured step) runs with a 1-rank communicator."""
import numpy as np
import pytest

from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.decompose import Subdomain, partition_rcb
from paper_2510_25906_b200.solver import Group, Solver, make_bcs, nccl_unique_id
from tests.decomp_driver import local_exchange, run_rk3
from tests.test_decompose import CASES, setup

pytestmark = pytest.mark.gpu


class GpuRank:
    def __init__(self, sub, opts, bcs):
        self.g = Solver.on_subdomain(sub, opts, make_bcs(bcs))
        self.sub = sub
        self.last_census = np.zeros(4, dtype=np.int64)

    def max_stable_dt(self, u):
        self.g.state = u
        return self.g.max_stable_dt()

    def residual(self, u, t, first):
        return self.g.compute_residual(u, t)

    def record_census(self):
        self.last_census = np.bincount(self.g.labels()[: self.sub.n_owned], minlength=4)


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("n", [2, 4])
def test_gpu_subdomains_match_single_domain(name, n):
    c, mesh, st, o, u0 = setup(name)
    steps = 3
    single = Solver(mesh, o, make_bcs(c["bcs"]), stencils=st)
    single.state = u0
    t_ref = 0.0
    cen_ref = []
    for _ in range(steps):
        dt = single.max_stable_dt()
        single.advance(dt, t_ref, A.RK3)
        t_ref += dt
        cen_ref.append(single.census())
    ref = single.state
    part = partition_rcb(mesh, n)
    subs = [Subdomain(mesh, st, part, n, r) for r in range(n)]
    ranks = [GpuRank(s, o, c["bcs"]) for s in subs]
    states = [s.local_state(u0) for s in subs]
    t, census = run_rk3(ranks, subs, states, steps, local_exchange, min)
    assert t == t_ref
    out = np.zeros_like(u0)
    for s, u in zip(subs, states):
        out[s.gid[: s.n_owned]] = u[: s.n_owned]
    np.testing.assert_array_equal(out, ref)
    for a, b in zip(census, cen_ref):
        np.testing.assert_array_equal(a, b)


def test_nccl_single_rank_path_matches_plain_solver():
    c, mesh, st, o, u0 = setup("shock-p2")
    part = partition_rcb(mesh, 1)
    sub = Subdomain(mesh, st, part, 1, 0)
    g = Solver.on_subdomain(sub, o, make_bcs(c["bcs"]))
    g.attach_nccl(nccl_unique_id(), 0, 1)
    g.state = sub.local_state(u0)
    plain = Solver(mesh, o, make_bcs(c["bcs"]), stencils=st)
    plain.state = u0
    assert g.max_stable_dt() == plain.max_stable_dt()
    t1, cen1 = g.run_steps(4, A.RK3, census=True)
    t2, cen2 = plain.run_steps(4, A.RK3, census=True)
    assert t1 == t2
    np.testing.assert_array_equal(cen1, cen2)
    np.testing.assert_array_equal(g.state[np.argsort(sub.gid)], plain.state)
    t3, _ = g.run_steps(3, A.RK3)  # graph-replayed steps with the in-graph all-reduce
    t4, _ = plain.run_steps(3, A.RK3)
    np.testing.assert_array_equal(g.state[np.argsort(sub.gid)], plain.state)


@pytest.mark.parametrize("rk", [A.RK3, A.RK54], ids=["rk3", "rk54"])
@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("n", [2, 3])
def test_loopback_group_schedule_matches_single_domain(name, n, rk):
    """The multi-GPU step schedule on one device: n subdomain solvers in one
    captured graph, each stage's sent cells updated first, the pack + one
    cudaMemcpyAsync per peer block on the forked exchange stream while the
    interior is updated, dt and error word reduced across the parts. Owned
    states and times are bit-identical to the single domain."""
    c, mesh, st, o, u0 = setup(name)
    steps = 4
    single = Solver(mesh, o, make_bcs(c["bcs"]), stencils=st)
    single.state = u0
    t_ref, _ = single.run_steps(steps, rk)
    ref = single.state
    part = partition_rcb(mesh, n)
    subs = [Subdomain(mesh, st, part, n, r) for r in range(n)]
    assert all(0 <= s.n_interior < s.n_owned for s in subs)
    parts = [Solver.on_subdomain(s, o, make_bcs(c["bcs"])) for s in subs]
    for p, s in zip(parts, subs):
        p.state = s.local_state(u0)
    g = Group(parts)
    t = g.run_steps(2, rk)
    t = g.run_steps(steps - 2, rk, t0=t)  # second call replays the other graph parity too
    assert t == t_ref
    out = np.zeros_like(u0)
    for p, s in zip(parts, subs):
        out[s.gid[: s.n_owned]] = p.state[: s.n_owned]
    np.testing.assert_array_equal(out, ref)


def test_loopback_group_failure_rolls_back_every_part():
    """A non-physical state on one part: every part returns to the failing
    step's input (the error word is reduced across the group each step)."""
    c, mesh, st, o, u0 = setup("shock-p2")
    part = partition_rcb(mesh, 2)
    subs = [Subdomain(mesh, st, part, 2, r) for r in range(2)]
    parts = [Solver.on_subdomain(s, o, make_bcs(c["bcs"])) for s in subs]
    bad = u0.copy()
    bad[subs[1].gid[0], 0] = -1.0  # an owned cell of part 1
    for p, s in zip(parts, subs):
        p.state = s.local_state(bad)
    before = [p.state for p in parts]
    g = Group(parts)
    with pytest.raises(A.NonPhysicalError):
        g.run_steps(3)
    for p, b in zip(parts, before):
        np.testing.assert_array_equal(p.state, b)
