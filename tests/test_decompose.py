"""Domain decomposition (csrc/decompose.cpp) checked with the oracle port:
N subdomains advanced with a halo refresh after every RK stage reproduce the
single-domain run bit-for-bit (owned cells), in one process and across two
gloo ranks (torch.distributed, world_size 2)."""
import os
import socket

import numpy as np
import pytest

from oracle import port as P
from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.decompose import Subdomain, partition_rcb
from paper_2510_25906_b200.mesh import Mesh, Stencils
from paper_2510_25906_b200.solver import make_bcs
from tests.decomp_driver import local_exchange, run_rk3

SHOCK = [-4.0, 3.857143, 2.629369, 0.0, 10.33333, 0.2, 5.0]
CASES = {
    "quadrants-p2": dict(nx=24, ny=24, rect=(0, 0, 1, 1), periodic="both", order=2, ic=(2, [0.5, 0.5, 0.01]),
                         opts=dict(mode="hybrid", cfl=0.5), bcs={}),
    "vortex-p3": dict(nx=20, ny=20, rect=(0, 0, 1, 1), periodic="both", order=3, ic=(0, [10.0]),
                      opts=dict(mode="hybrid", lambda1p=1e4, cfl=0.5), bcs={}),
    "shock-p2": dict(nx=64, ny=8, rect=(-5, 0, 5, 1), periodic="y", order=2, ic=(1, SHOCK),
                     opts=dict(mode="hybrid", cfl=0.5), bcs={"left": "outflow", "right": "outflow"}),
}


class PortRank:
    def __init__(self, sub, opts, bcs):
        bcl = make_bcs({**bcs, "__halo__": "outflow"})
        self.p = P.PortSolver(sub.mesh_view, sub.stencil_view, opts, bcl, keep=(sub,))
        self.sub = sub
        self.last_census = np.zeros(4, dtype=np.int64)

    def max_stable_dt(self, u):
        self.p.state = u
        return self.p.max_stable_dt()

    def residual(self, u, t, first):
        return self.p.compute_residual(u, t, first)

    def record_census(self):
        self.last_census = np.bincount(self.p.labels()[: self.sub.n_owned], minlength=4)


def setup(name, seed=3):
    c = CASES[name]
    nq = (c["order"] + 2) // 2
    mesh = Mesh.structured_tri(c["nx"], c["ny"], c["rect"], jitter=0.1, seed=seed, periodic=c["periodic"], n_qp=nq)
    st = Stencils(mesh, c["order"])
    o = A.options_from_dict(order=c["order"], **c["opts"])
    u0 = mesh.project_initial(*c["ic"], seed=1, degree=max(2 * c["order"], 2))
    return c, mesh, st, o, u0


def single_domain(c, mesh, st, o, u0, steps):
    p = P.PortSolver(mesh.view, st.view, o, make_bcs(c["bcs"]), keep=(mesh, st))
    p.state = u0.copy()
    t, census = 0.0, []
    for _ in range(steps):
        dt = p.max_stable_dt()
        p.advance(dt, t, A.RK3)
        t += dt
        census.append(np.bincount(p.labels(step=True), minlength=4))
    return p.state, t, census


def test_partition_balanced():
    mesh = Mesh.structured_tri(30, 17, (0, 0, 3, 1), jitter=0.1, seed=1, periodic="both", n_qp=2)
    for n in (1, 2, 3, 4, 7, 8):
        part = partition_rcb(mesh, n)
        counts = np.bincount(part, minlength=n)
        assert counts.min() >= 1 and counts.max() - counts.min() <= 1


def test_exchange_plan_is_consistent():
    c, mesh, st, o, u0 = setup("shock-p2")
    n = 4
    part = partition_rcb(mesh, n)
    subs = [Subdomain(mesh, st, part, n, r) for r in range(n)]
    for s in subs:
        assert np.array_equal(np.sort(s.gid[: s.n_owned]), np.flatnonzero(part == s.rank))
        assert np.all(part[s.gid[s.n_owned:]] != s.rank)
        for p in s.peers:
            q = subs[p.rank]
            back = next(pp for pp in q.peers if pp.rank == s.rank)
            # what q sends to s is exactly s's receive block, in order
            assert len(back.send) == p.n_recv
            np.testing.assert_array_equal(q.gid[back.send], s.gid[p.recv_begin:p.recv_begin + p.n_recv])


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("n", [2, 3, 5])
def test_decomposed_port_matches_single_domain(name, n):
    c, mesh, st, o, u0 = setup(name)
    steps = 3
    ref, t_ref, cen_ref = single_domain(c, mesh, st, o, u0, steps)
    part = partition_rcb(mesh, n)
    subs = [Subdomain(mesh, st, part, n, r) for r in range(n)]
    ranks = [PortRank(s, o, c["bcs"]) for s in subs]
    states = [s.local_state(u0) for s in subs]
    t, census = run_rk3(ranks, subs, states, steps, local_exchange, min)
    assert t == t_ref
    out = np.zeros_like(u0)
    for s, u in zip(subs, states):
        out[s.gid[: s.n_owned]] = u[: s.n_owned]
    np.testing.assert_array_equal(out, ref)
    for a, b in zip(census, cen_ref):
        np.testing.assert_array_equal(a, b)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, name, steps, result):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, mesh, st, o, u0 = setup(name)
        part = partition_rcb(mesh, world)
        sub = Subdomain(mesh, st, part, world, rank)
        me = PortRank(sub, o, c["bcs"])

        def exchange(subs, new):
            (s,), (u,) = subs, new
            reqs = []
            bufs = []
            for p in s.peers:
                if len(p.send):
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(u[p.send])), p.rank))
                if p.n_recv:
                    b = torch.empty((p.n_recv, 4), dtype=torch.float64)
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
        owned = torch.from_numpy(np.ascontiguousarray(states[0][: sub.n_owned]))
        gids = torch.from_numpy(sub.gid[: sub.n_owned].astype(np.int64))
        cen = torch.from_numpy(np.array(census, dtype=np.int64))
        dist.all_reduce(cen)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([sub.n_owned]))
        mx = int(max(x.item() for x in sizes))
        pad_u = torch.zeros((mx, 4), dtype=torch.float64)
        pad_u[: sub.n_owned] = owned
        pad_g = torch.full((mx,), -1, dtype=torch.int64)
        pad_g[: sub.n_owned] = gids
        all_u = [torch.zeros_like(pad_u) for _ in range(world)]
        all_g = [torch.zeros_like(pad_g) for _ in range(world)]
        dist.all_gather(all_u, pad_u)
        dist.all_gather(all_g, pad_g)
        if rank == 0:
            out = np.zeros_like(u0)
            for uu, gg in zip(all_u, all_g):
                m = gg.numpy() >= 0
                out[gg.numpy()[m]] = uu.numpy()[m]
            result.put((out, t, cen.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["quadrants-p2", "shock-p2"])
def test_two_gloo_ranks_match_single_domain(name):
    import torch.multiprocessing as mp

    steps = 2
    c, mesh, st, o, u0 = setup(name)
    ref, t_ref, cen_ref = single_domain(c, mesh, st, o, u0, steps)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, name, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    out, t, cen = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == t_ref
    np.testing.assert_array_equal(out, ref)
    np.testing.assert_array_equal(cen, np.array(cen_ref))
