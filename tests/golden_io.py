"""Load tests/golden/*.npz fixtures (made by tests/golden/make_golden.py from
the compiled reference) back into flat views, options and BCs."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.solver import make_bcs

GOLDEN = Path(__file__).resolve().parent / "golden"
OPT_FIELDS = ["order", "mode", "limiter", "riemann", "lambda1p", "weno_eps", "weno_b", "cfl", "venkat_kappa",
              "si_exponent", "detect_every_stage", "gamma"]
INT_FIELDS = {"order", "mode", "limiter", "riemann", "si_exponent", "detect_every_stage"}


def names():
    # fullsize_*.npz are digests of full-length reference runs (tests/golden/make_fullsize_refs.py), not stage fixtures
    return sorted(p.stem for p in GOLDEN.glob("*.npz") if not p.stem.startswith("fullsize_"))


class Fixture:
    def __init__(self, name):
        self.name = name
        self.d = dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
        self.mesh_np = {k[5:]: v for k, v in self.d.items() if k.startswith("mesh_")}
        self.st_np = {k[3:]: v for k, v in self.d.items() if k.startswith("st_")}
        self.mesh_view, self._mk = A.mesh_view_from_numpy(self.mesh_np)
        self.stencil_view, self._sk = A.stencil_view_from_numpy(self.st_np)
        o = A.default_options()
        for f, v in zip(OPT_FIELDS, self.d["options"]):
            setattr(o, f, int(v) if f in INT_FIELDS else float(v))
        o.margins = A.Margins(*[float(x) for x in self.d["margins"]])
        self.options = o
        self.bcs_spec = json.loads(str(self.d["bcs"]))
        self.bcs = make_bcs(self.bcs_spec)
        self.u0 = self.d["u0"]
        self.error = "error_code" in self.d

    def __getitem__(self, k):
        return self.d[k]

    @property
    def view(self):  # so a Fixture can stand in for a Mesh
        return self.mesh_view

    def written_right(self):
        right = self.mesh_np["face_right"]
        return np.repeat(right >= 0, int(self.mesh_np["n_qp"]))


class StencilHolder:
    def __init__(self, view, keep):
        self.view = view
        self.keep = keep
