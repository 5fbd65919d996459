"""Test-side case builders (BASELINE.json configs, down-scaled variants)."""
from __future__ import annotations

import numpy as np

from paper_2510_25906_b200 import _abi as A

# BASELINE.json config 2 shock-into-sine parameters: x_shock, rho, u, v, p (left), amplitude, wavenumber
SHOCK_SINE = [-4.0, 3.857143, 2.629369, 0.0, 10.33333, 0.2, 5.0]
QUADRANTS = [0.5, 0.5, 0.01]  # split x, split y, 1% multiplicative cell noise
VORTEX = [10.0]  # ic_vortex(10x, 10y): the reference vortex scaled into the unit square


def case(name, scale=1):
    """(mesh kwargs, order, ic, params, option overrides, bc mapping) of a named case.

    scale divides the BASELINE resolution (for CPU-oracle-sized parity runs)."""
    if name == "config1":
        n = 128 // scale
        return dict(nx=n, ny=n, rect=(0.0, 0.0, 1.0, 1.0), jitter=0.1, periodic="both"), 2, 0, VORTEX, \
            dict(lambda1p=1e4, cfl=0.5), {}
    if name == "config2":
        return dict(nx=2048 // scale, ny=64 // scale, rect=(-5.0, 0.0, 5.0, 1.0), jitter=0.1, periodic="y"), 2, 1, \
            SHOCK_SINE, dict(lambda1p=1e3, cfl=0.5), {"left": "outflow", "right": "outflow"}
    if name == "config3":
        n = 2048 // scale
        return dict(nx=n, ny=n, rect=(0.0, 0.0, 1.0, 1.0), jitter=0.0, periodic="both"), 3, 2, QUADRANTS, \
            dict(lambda1p=1e3, cfl=0.5), {}
    raise KeyError(name)


def rel_err(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.abs(a - b) / den)) if a.size else 0.0


def scaled_err(a, b):
    """max |a-b| / max(|b|, per-variable scale) -- relative error robust to near-zero entries."""
    a = np.asarray(a).reshape(-1, 4)
    b = np.asarray(b).reshape(-1, 4)
    scale = np.maximum(np.max(np.abs(b), axis=0), 1e-300)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-6 * scale))) if a.size else 0.0
