"""Halo sizes and redundant-compute fractions of the 2D domain decomposition
(DESIGN.md §8): for a BASELINE config split into N RCB subdomains, per rank
the owned cells, the classification halo (layers 1-2: reconstructed again,
redundantly), the U-only halo, the cells sent every stage and the interior
the exchange overlaps with.

    python scripts/halo_stats.py --config 3 --parts 2 4 8 > profiles/r02_halo_config3.json
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2510_25906_b200.decompose import Subdomain, partition_rcb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="3")
ap.add_argument("--parts", type=int, nargs="+", default=[2, 4, 8])
a = ap.parse_args()
t0 = time.perf_counter()
mesh, st, u0, _ = bench.build_case(a.config, n_threads=os.cpu_count() or 1)
n = mesh.n_cells
out = {"config": a.config, "cells": n, "setup_s": round(time.perf_counter() - t0, 1), "parts": {}}
for N in a.parts:
    part = partition_rcb(mesh, N)
    rows = []
    for r in range(N):
        s = Subdomain(mesh, st, part, N, r)
        halo = s.n_local - s.n_owned
        # classification halo: local halo cells carrying real stencils (layers 1-2)
        sv = st.view  # global view; local inert stencils are self-members only
        sent = sum(len(p.send) for p in s.peers)
        recv = sum(p.n_recv for p in s.peers)
        rows.append({"rank": r, "owned": s.n_owned, "halo": halo, "interior": s.n_interior,
                     "sent_cells": s.n_owned - s.n_interior, "send_entries": sent, "recv_entries": recv,
                     "peers": len(s.peers), "bytes_per_stage_out": 32 * sent, "bytes_per_stage_in": 32 * recv})
        del s
    own = np.array([x["owned"] for x in rows])
    halo = np.array([x["halo"] for x in rows])
    out["parts"][N] = {
        "ranks": rows,
        "max_owned": int(own.max()), "imbalance": round(float(own.max() / own.mean()), 4),
        "halo_over_owned_max": round(float((halo / own).max()), 4),
        "redundant_local_cells_frac": round(float(halo.sum() / own.sum()), 4),
        "interior_frac_min": round(float(min(x["interior"] / x["owned"] for x in rows)), 4),
        "exchange_MB_per_stage_max": round(max(x["bytes_per_stage_in"] for x in rows) / 1e6, 3),
    }
    print(N, json.dumps({k: v for k, v in out["parts"][N].items() if k != "ranks"}), file=sys.stderr)
print(json.dumps(out, indent=1))
