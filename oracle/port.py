"""ORACLE TEST INFRASTRUCTURE -- not product code.

ctypes wrapper over oracle/_build/libucfv_port.so, the plain-C restatement of
the reference stage pass (oracle/ucfv_port.c). It consumes the same flat views
(include/ucfvb.h) as the GPU path, so GPU-vs-port comparisons are on identical
inputs; the port itself is pinned to the compiled reference (oracle/_ref) and
to tests/golden/ by tests/test_oracle_pin.py.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2510_25906_b200 import _abi as A

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "_build" / "libucfv_port.so"
_lib = None


def available() -> bool:
    return PORT_LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not PORT_LIB.exists():
            raise RuntimeError(f"{PORT_LIB} not built (make -C oracle port)")
        L = C.CDLL(str(PORT_LIB))
        H = C.c_void_p
        dp = C.POINTER(C.c_double)
        sig = {
            "port_last_error": (C.c_char_p, []),
            "port_create": (C.c_int, [C.POINTER(A.MeshView), C.POINTER(A.StencilView), C.POINTER(A.Options),
                                      C.POINTER(A.BC), C.c_int, C.POINTER(H)]),
            "port_free": (None, [H]),
            "port_compute_residual": (C.c_int, [H, dp, C.c_double, C.c_int, dp]),
            "port_max_stable_dt": (C.c_int, [H, dp, dp]),
            "port_advance": (C.c_int, [H, dp, C.c_double, C.c_double, C.c_int]),
            "port_get_labels": (None, [H, C.POINTER(C.c_uint8), C.c_int]),
            "port_get_face_values": (None, [H, dp, dp]),
            "port_get_dofs": (None, [H, dp]),
            "port_get_bounds": (None, [H, dp]),
            "port_compute_margins": (None, [C.POINTER(A.Margins), C.c_double, dp, dp]),
            "port_classify_violation": (C.c_int, [C.c_double, C.c_double, C.c_double]),
            "port_deactivate_smooth": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double]),
            "port_limiter_bj": (C.c_double, [C.c_double, C.c_double, C.c_double, dp, C.c_int]),
            "port_limiter_venkat": (C.c_double, [C.c_double, C.c_double, C.c_double, dp, C.c_int, C.c_double]),
            "port_flux": (C.c_int, [dp, dp, C.c_double, C.c_double, C.c_double, C.c_int, dp]),
            "port_cwenoz_blend": (C.c_int, [dp, C.c_int, dp, dp, C.c_int, C.c_double, C.c_double, C.c_double, dp]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


class PortError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class PortSolver:
    """Restated ucfv::Solver over flat views. Keeps the views (and whatever
    owns their buffers) alive; the state is held here as a numpy array."""

    def __init__(self, mesh_view, stencil_view, options, bcs=(), keep=()):
        self._keep = (mesh_view, stencil_view, options, keep)
        self.n_cells = mesh_view.n_cells
        self.n_faces = mesh_view.n_faces
        self.n_qp = stencil_view.n_qp
        self.K = stencil_view.K
        arr = (A.BC * max(1, len(bcs)))(*bcs)
        self._bcs = arr
        h = C.c_void_p()
        rc = lib().port_create(C.byref(mesh_view), C.byref(stencil_view), C.byref(options), arr, len(bcs),
                               C.byref(h))
        if rc:
            raise PortError(rc, lib().port_last_error().decode())
        self.h = h
        self.state = np.zeros((self.n_cells, 4))

    def _ck(self, rc):
        if rc:
            raise PortError(rc, lib().port_last_error().decode())

    def compute_residual(self, u, t=0.0, stage_first=1):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros((self.n_cells, 4))
        self._ck(lib().port_compute_residual(self.h, _dp(u), t, stage_first, _dp(out)))
        return out

    def max_stable_dt(self):
        d = C.c_double()
        self._ck(lib().port_max_stable_dt(self.h, _dp(self.state), C.byref(d)))
        return d.value

    def advance(self, dt, t, rk=A.RK3):
        u = np.ascontiguousarray(self.state.copy())
        self._ck(lib().port_advance(self.h, _dp(u), dt, t, rk))
        self.state = u

    def run_steps(self, n_steps, rk=A.RK3, t0=0.0, t_end=float("inf")):
        t = t0
        for _ in range(n_steps):
            dt = min(self.max_stable_dt(), t_end - t)
            self.advance(dt, t, rk)
            t += dt
        return t

    def labels(self, step=False):
        out = np.zeros(self.n_cells, dtype=np.uint8)
        lib().port_get_labels(self.h, out.ctypes.data_as(C.POINTER(C.c_uint8)), 1 if step else 0)
        return out

    def face_values(self):
        L = np.zeros((self.n_faces * self.n_qp, 4))
        R = np.zeros_like(L)
        lib().port_get_face_values(self.h, _dp(L), _dp(R))
        return L, R

    def dofs(self):
        d = np.zeros((self.n_cells, self.K, 4))
        lib().port_get_dofs(self.h, _dp(d))
        return d

    def bounds(self):
        b = np.zeros((self.n_cells, 4))
        lib().port_get_bounds(self.h, _dp(b))
        return b

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.port_free(self.h)
            self.h = None
