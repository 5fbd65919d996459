"""Decomposed-run drivers used by the tests: every subdomain advances with
compute_residual + the reference's combine2, and halo cells are refreshed from
their owners after every stage (the exchange the NCCL path performs on the
device). `exchange` is pluggable: in-process copies or torch.distributed."""
from __future__ import annotations

import numpy as np

from paper_2510_25906_b200 import _abi as A

RK3 = [  # (wa, wb, wr, stage-time fraction) of combine2 per stage; ub = previous stage
    (1.0, 0.0, 1.0, 0.0),
    (0.75, 0.25, 0.25, 1.0),
    (1.0 / 3.0, 2.0 / 3.0, 2.0 / 3.0, 0.5),
]


def combine2(wa, ua, wb, ub, wr, r, dt):
    return wa * ua + wb * ub + (wr * dt) * r  # time_integrator.cpp:31-38 operation order


def local_exchange(subs, states):
    """in-process halo refresh: every rank's halo block from its owners"""
    by_rank = {s.rank: s for s in subs}
    for s in subs:
        for p in s.peers:
            if p.n_recv:
                q = by_rank[p.rank]
                sq = next(pp for pp in q.peers if pp.rank == s.rank)
                states[s.rank][p.recv_begin:p.recv_begin + p.n_recv] = states[q.rank][sq.send]


def run_rk3(solvers, subs, states, steps, exchange, dt_min):
    """solvers[i] has compute_residual(u, t, stage_first) -> residual and max_stable_dt(u)."""
    t = 0.0
    census = []
    for _ in range(steps):
        dt = dt_min([sv.max_stable_dt(u) for sv, u in zip(solvers, states)])
        u0 = [u.copy() for u in states]
        prev = [u.copy() for u in states]
        for k, (wa, wb, wr, tf) in enumerate(RK3):
            new = []
            for sv, s, u_n, u_s in zip(solvers, subs, u0, prev):
                r = sv.residual(u_s, t + tf * dt, 1 if k == 0 else 0)
                out = u_s.copy()
                o = s.n_owned
                out[:o] = combine2(wa, u_n[:o], wb, u_s[:o], wr, r[:o], dt)
                if k == 0:
                    sv.record_census()
                new.append(out)
            exchange(subs, new)
            prev = new
        states[:] = prev
        census.append(sum(sv.last_census for sv in solvers))
        t += dt
    return t, census
