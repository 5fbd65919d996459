"""3D domain decomposition (csrc/decompose3.cpp) checked with the 3D oracle:
N subdomains advanced with a halo refresh after every RK stage reproduce the
single-domain run bit-for-bit on owned cells (in one process), for per-cell
and lattice-class operators."""
import numpy as np
import pytest

from oracle.port3 import Port3Solver
from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.solver3d import (HEX, IC_BLAST, IC_RANDOM_PHASE, TET, Mesh3, Stencils3, Subdomain3,
                                            _StencilFacade, partition_rcb3)
from tests.decomp_driver import local_exchange, run_rk3

CASES3 = {
    "hex-p2-blast": dict(kind=HEX, n=6, jitter=0.05, order=2, classes=False, ic=(IC_BLAST, [3.0, 3.2, 3.1, 1.6, 1.0, 8.0, 0.3, 0.5])),
    "tet-p2-classes": dict(kind=TET, n=6, jitter=0.0, order=2, classes=True, ic=(IC_RANDOM_PHASE, [0.8, 2.0, 4])),
}


def setup3(name):
    c = CASES3[name]
    m = Mesh3(c["n"], kind=c["kind"], jitter=c["jitter"], order=c["order"], seed=3)
    st = Stencils3(m, c["order"], lattice_classes=c["classes"])
    o = A.options_from_dict(order=c["order"], mode="hybrid", cfl=0.5)
    u0 = m.project_initial(*c["ic"], seed=2)
    return c, m, st, o, u0


class Port3Rank:
    def __init__(self, sub, opts):
        self.p = Port3Solver(sub, _StencilFacade(sub.stencil_view), opts)
        self.sub = sub
        self.last_census = np.zeros(4, dtype=np.int64)

    def max_stable_dt(self, u):
        self.p.state = u
        return self.p.max_stable_dt()

    def residual(self, u, t, first):
        return self.p.compute_residual(u, t)

    def record_census(self):
        self.last_census = np.bincount(self.p.labels()[: self.sub.n_owned], minlength=4)


def single3(m, st, o, u0, steps):
    p = Port3Solver(m, st, o)
    p.state = u0.copy()
    t, census = 0.0, []
    for _ in range(steps):
        dt = p.max_stable_dt()
        p.advance(dt, t, A.RK3)
        t += dt
        census.append(np.bincount(p.labels(step=True), minlength=4))
    return p.state, t, census


@pytest.mark.parametrize("name", sorted(CASES3))
@pytest.mark.parametrize("n_parts", [2, 3])
def test_subdomains_match_single_domain(name, n_parts):
    c, m, st, o, u0 = setup3(name)
    steps = 2
    ref, t_ref, cen_ref = single3(m, st, o, u0, steps)
    part = partition_rcb3(m, n_parts)
    assert np.bincount(part).min() > 0
    subs = [Subdomain3(m, st, part, n_parts, r) for r in range(n_parts)]
    ranks = [Port3Rank(s, o) for s in subs]
    states = [s.local_state(u0) for s in subs]
    t, census = run_rk3(ranks, subs, states, steps, local_exchange, min)
    assert t == t_ref
    out = np.zeros_like(u0)
    for s, u in zip(subs, states):
        out[s.gid[: s.n_owned]] = u[: s.n_owned]
    np.testing.assert_array_equal(out, ref)
    for a, b in zip(census, cen_ref):
        np.testing.assert_array_equal(a, b)


def test_partition_is_balanced_and_complete():
    m = Mesh3(8, kind=TET, order=2)
    for n_parts in (2, 4, 8):
        part = partition_rcb3(m, n_parts)
        cnt = np.bincount(part, minlength=n_parts)
        assert cnt.sum() == m.n_cells and cnt.max() - cnt.min() <= 1


def test_exchange_plan_is_consistent3():
    c, m, st, o, u0 = setup3("tet-p2-classes")
    n = 4
    part = partition_rcb3(m, n)
    subs = [Subdomain3(m, st, part, n, r) for r in range(n)]
    for s in subs:
        assert np.array_equal(np.sort(s.gid[: s.n_owned]), np.flatnonzero(part == s.rank))
        assert np.all(part[s.gid[s.n_owned:]] != s.rank)
        for p in s.peers:
            q = subs[p.rank]
            back = next(pp for pp in q.peers if pp.rank == s.rank)
            assert len(back.send) == p.n_recv
            np.testing.assert_array_equal(q.gid[back.send], s.gid[p.recv_begin:p.recv_begin + p.n_recv])


def _gloo_worker3(rank, world, port, name, steps, result):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, m, st, o, u0 = setup3(name)
        part = partition_rcb3(m, world)
        sub = Subdomain3(m, st, part, world, rank)
        me = Port3Rank(sub, o)

        def exchange(subs, new):
            (s,), (u,) = subs, new
            reqs, bufs = [], []
            for p in s.peers:
                if len(p.send):
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(u[p.send])), p.rank))
                if p.n_recv:
                    b = torch.empty((p.n_recv, 5), dtype=torch.float64)
                    bufs.append((p, b))
                    reqs.append(dist.irecv(b, p.rank))
            for r in reqs:
                r.wait()
            for p, b in bufs:
                u[p.recv_begin:p.recv_begin + p.n_recv] = b.numpy()

        def dt_min(vals):
            t = torch.tensor([min(vals)], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            return float(t.item())

        states = [sub.local_state(u0)]
        t, census = run_rk3([me], [sub], states, steps, exchange, dt_min)
        cen = torch.from_numpy(np.array(census, dtype=np.int64))
        dist.all_reduce(cen)
        full = torch.zeros((m.n_cells, 5), dtype=torch.float64)
        full[torch.from_numpy(sub.gid[: sub.n_owned].astype(np.int64))] = torch.from_numpy(
            np.ascontiguousarray(states[0][: sub.n_owned]))
        dist.all_reduce(full)  # owned blocks are disjoint: the sum assembles the global state
        if rank == 0:
            result.put((full.numpy(), t, cen.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_gloo_ranks_match_single_domain3():
    import socket

    import torch.multiprocessing as mp

    steps = 2
    name = "tet-p2-classes"
    c, m, st, o, u0 = setup3(name)
    ref, t_ref, cen_ref = single3(m, st, o, u0, steps)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker3, args=(r, 2, port, name, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, t, cen = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == t_ref
    np.testing.assert_array_equal(out, ref)
    np.testing.assert_array_equal(cen, np.array(cen_ref))
