"""Subdomain solvers on the GPU (ucfvb_create_sub): N subdomains driven stage
by stage with a host halo refresh reproduce the single-domain GPU run
bit-for-bit on owned cells; the NCCL path (dt/census/error all-reduces inside
the captured step) runs with a 1-rank communicator."""
import numpy as np
import pytest

from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.decompose import Subdomain, partition_rcb
from paper_2510_25906_b200.solver import Solver, make_bcs, nccl_unique_id
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
