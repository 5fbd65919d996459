"""ORACLE TEST INFRASTRUCTURE -- not product code.

ctypes wrapper over oracle/_build/libucfv3_port.so, the plain-C 3D
restatement of the reference stage pass (oracle/ucfv3_port.c). It consumes
the same views (include/ucfvb3.h) as the GPU path. The reference is 2D only,
so the 3D restatement is parity-unpinned; its 2D sibling
oracle/ucfv_port.c is pinned to the compiled reference.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.solver3d import MeshView3, StencilView3, NV

HERE = Path(__file__).resolve().parent
PORT3_LIB = HERE / "_build" / "libucfv3_port.so"
_lib = None
_dp = C.POINTER(C.c_double)


def lib():
    global _lib
    if _lib is None:
        if not PORT3_LIB.exists():
            raise RuntimeError(f"{PORT3_LIB} not built (make -C oracle port)")
        L = C.CDLL(str(PORT3_LIB))
        H = C.c_void_p
        sig = {
            "port3_last_error": (C.c_char_p, []),
            "port3_create": (C.c_int, [C.POINTER(MeshView3), C.POINTER(StencilView3), C.POINTER(A.Options),
                                       C.POINTER(H)]),
            "port3_free": (None, [H]),
            "port3_compute_residual": (C.c_int, [H, _dp, C.c_double, _dp]),
            "port3_max_stable_dt": (C.c_int, [H, _dp, _dp]),
            "port3_advance": (C.c_int, [H, _dp, C.c_double, C.c_double, C.c_int]),
            "port3_get_labels": (None, [H, C.POINTER(C.c_uint8), C.c_int]),
            "port3_get_face_values": (None, [H, _dp]),
            "port3_get_dofs": (None, [H, _dp]),
            "port3_bad_face": (C.c_int64, [H]),
            "port3_flux": (C.c_int, [_dp, _dp, _dp, C.c_double, C.c_int, _dp]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


class Port3Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Port3Solver:
    """3D restated ucfv::Solver over the same views as solver3d.Solver3."""

    def __init__(self, mesh, stencils, opt):
        self.mesh, self.stencils, self.opt = mesh, stencils, opt  # keep views alive
        self.n = mesh.n_cells
        h = C.c_void_p()
        rc = lib().port3_create(C.byref(mesh.view), C.byref(stencils.view), C.byref(opt), C.byref(h))
        self._check(rc)
        self._h = h
        self.state = np.zeros((self.n, NV))

    def _check(self, rc):
        if rc:
            raise Port3Error(rc, lib().port3_last_error().decode())

    def __del__(self):
        if getattr(self, "_h", None):
            lib().port3_free(self._h)
            self._h = None

    def max_stable_dt(self):
        d = C.c_double()
        self._check(lib().port3_max_stable_dt(self._h, self.state.ctypes.data_as(_dp), C.byref(d)))
        return d.value

    def advance(self, dt, t=0.0, rk=A.RK3):
        self.state = np.ascontiguousarray(self.state)
        self._check(lib().port3_advance(self._h, self.state.ctypes.data_as(_dp), dt, t, rk))

    def compute_residual(self, u, t=0.0):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros((self.n, NV))
        self._check(lib().port3_compute_residual(self._h, u.ctypes.data_as(_dp), t, out.ctypes.data_as(_dp)))
        return out

    def labels(self, step=False):
        out = np.zeros(self.n, np.uint8)
        lib().port3_get_labels(self._h, out.ctypes.data_as(C.POINTER(C.c_uint8)), int(step))
        return out

    def face_values(self):
        out = np.zeros((self.mesh.n_faces, self.mesh.nq, 2, NV))
        lib().port3_get_face_values(self._h, out.ctypes.data_as(_dp))
        return out


def flux(ul, ur, n, gamma=1.4, kind=A.HLLC):
    ul, ur, n = (np.ascontiguousarray(x, dtype=np.float64) for x in (ul, ur, n))
    out = np.zeros(NV)
    rc = lib().port3_flux(ul.ctypes.data_as(_dp), ur.ctypes.data_as(_dp), n.ctypes.data_as(_dp), gamma, kind,
                          out.ctypes.data_as(_dp))
    return out if rc == 0 else None
