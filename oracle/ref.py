"""ORACLE TEST INFRASTRUCTURE -- not product code.

ctypes wrapper over oracle/_ref/libucfv_ref.so: the UNMODIFIED reference
sources (/root/reference/proj/src) plus oracle/ref_harness.cpp. Used only by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2510_25906_b200 import _abi as A

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libucfv_ref.so"

_lib = None


def available() -> bool:
    return REF_LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not REF_LIB.exists():
            raise RuntimeError(f"{REF_LIB} not built (make -C oracle ref)")
        L = C.CDLL(str(REF_LIB))
        H = C.c_void_p
        dp = C.POINTER(C.c_double)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_uniform01": (C.c_double, [C.c_uint64, C.c_uint64, C.c_uint64]),
            "ref_mesh_structured_tri": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                                  C.c_double, C.c_int, C.c_double, C.c_uint64, C.c_int,
                                                  C.c_double, C.c_int, C.POINTER(H)]),
            "ref_mesh_generate_tri": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                                C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                                                C.POINTER(H)]),
            "ref_mesh_generate_quad": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                                 C.c_double, C.c_int, C.c_double, C.c_int, C.POINTER(H)]),
            "ref_mesh_view": (C.c_int, [H, C.POINTER(A.MeshView)]),
            "ref_mesh_free": (None, [H]),
            "ref_project_initial": (C.c_int, [H, C.c_int, dp, C.c_int, C.c_uint64, C.c_int, C.c_double, dp]),
            "ref_solver_create": (C.c_int, [H, C.POINTER(A.Options), C.POINTER(A.BC), C.c_int, C.POINTER(H)]),
            "ref_solver_free": (None, [H]),
            "ref_stencil_view": (C.c_int, [H, C.POINTER(A.StencilView)]),
            "ref_set_state": (C.c_int, [H, dp]),
            "ref_get_state": (C.c_int, [H, dp]),
            "ref_max_stable_dt": (C.c_int, [H, dp]),
            "ref_compute_residual": (C.c_int, [H, dp, C.c_double, C.c_int, dp]),
            "ref_advance": (C.c_int, [H, C.c_double, C.c_double, C.c_int]),
            "ref_run_steps": (C.c_int, [H, C.c_int, C.c_int, C.c_double, C.c_double, dp,
                                        C.POINTER(C.c_int64), dp]),
            "ref_run_steps_log": (C.c_int, [H, C.c_int, C.c_int, C.c_double, C.c_double, dp,
                                            C.POINTER(C.c_int64), dp]),
            "ref_write_field_snapshot": (C.c_int, [H, dp, C.POINTER(C.c_uint8), C.c_double, C.c_char_p]),
            "ref_write_census_csv": (C.c_int, [C.POINTER(A.CensusRow), C.c_int, C.c_int, C.c_char_p]),
            "ref_write_timing_csv": (C.c_int, [C.POINTER(A.TimingRow), C.c_int, C.c_char_p]),
            "ref_get_labels": (C.c_int, [H, C.POINTER(C.c_uint8), C.c_int]),
            "ref_get_face_values": (C.c_int, [H, dp, dp]),
            "ref_get_dofs": (C.c_int, [H, dp]),
            "ref_get_bounds": (C.c_int, [H, dp]),
            "ref_get_phase_times": (C.c_int, [H, dp]),
            "ref_n_cells": (C.c_int, [H]),
            "ref_n_faces": (C.c_int, [H]),
            "ref_K": (C.c_int, [H]),
            "ref_n_qp": (C.c_int, [H]),
            "ref_compute_margins": (C.c_int, [C.POINTER(A.Margins), C.c_double, dp, dp]),
            "ref_classify_violation": (C.c_int, [C.c_double, C.c_double, C.c_double]),
            "ref_deactivate_smooth": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double]),
            "ref_limiter_bj": (C.c_double, [C.c_double, C.c_double, C.c_double, dp, C.c_int]),
            "ref_limiter_venkat": (C.c_double, [C.c_double, C.c_double, C.c_double, dp, C.c_int, C.c_double]),
            "ref_flux": (C.c_int, [dp, dp, C.c_double, C.c_double, C.c_double, C.c_int, dp]),
            "ref_pow": (C.c_double, [C.c_double, C.c_double]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ck(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class RefMesh:
    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    @classmethod
    def structured_tri(cls, nx, ny, rect=(0.0, 0.0, 1.0, 1.0), diagonal=0, jitter=0.0, seed=0,
                       periodic=3, tol=1e-8, n_qp=2):
        h = C.c_void_p()
        _ck(lib().ref_mesh_structured_tri(nx, ny, *rect, diagonal, jitter, seed, periodic, tol, n_qp,
                                          C.byref(h)))
        return cls(h.value)

    @classmethod
    def generate_tri(cls, nx, ny, rect, diagonal=0, periodic=3, tol=1e-8, n_qp=2):
        h = C.c_void_p()
        _ck(lib().ref_mesh_generate_tri(nx, ny, *rect, diagonal, periodic, tol, n_qp, C.byref(h)))
        return cls(h.value)

    @classmethod
    def generate_quad(cls, nx, ny, rect, periodic=3, tol=1e-8, n_qp=2):
        h = C.c_void_p()
        _ck(lib().ref_mesh_generate_quad(nx, ny, *rect, periodic, tol, n_qp, C.byref(h)))
        return cls(h.value)

    def view(self) -> A.MeshView:
        v = A.MeshView()
        _ck(lib().ref_mesh_view(self.h, C.byref(v)))
        return v

    def numpy(self) -> dict:
        return A.mesh_view_to_numpy(self.view())

    @property
    def n_cells(self):
        return self.view().n_cells

    def project_initial(self, ic, params, seed=0, degree=4, gamma=1.4):
        p = np.ascontiguousarray(params, dtype=np.float64)
        u = np.zeros((self.n_cells, 4))
        _ck(lib().ref_project_initial(self.h, ic, _dp(p), len(p), seed, degree, gamma, _dp(u)))
        return u

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_mesh_free(self.h)
            self.h = None


class RefSolver:
    """The reference ucfv::Solver, driven through the harness."""

    def __init__(self, mesh: RefMesh, options: A.Options, bcs=()):
        self.mesh = mesh
        arr = (A.BC * max(1, len(bcs)))(*bcs)
        h = C.c_void_p()
        _ck(lib().ref_solver_create(mesh.h, C.byref(options), arr, len(bcs), C.byref(h)))
        self.h = h
        self.n_cells = lib().ref_n_cells(h)
        self.n_faces = lib().ref_n_faces(h)
        self.K = lib().ref_K(h)
        self.n_qp = lib().ref_n_qp(h)

    def stencil_view(self) -> A.StencilView:
        v = A.StencilView()
        _ck(lib().ref_stencil_view(self.h, C.byref(v)))
        return v

    def stencils_numpy(self) -> dict:
        return A.stencil_view_to_numpy(self.stencil_view())

    def set_state(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        _ck(lib().ref_set_state(self.h, _dp(u)))

    def get_state(self):
        u = np.zeros((self.n_cells, 4))
        _ck(lib().ref_get_state(self.h, _dp(u)))
        return u

    def max_stable_dt(self):
        d = C.c_double()
        _ck(lib().ref_max_stable_dt(self.h, C.byref(d)))
        return d.value

    def compute_residual(self, u, t=0.0, stage_first=1):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros((self.n_cells, 4))
        _ck(lib().ref_compute_residual(self.h, _dp(u), t, stage_first, _dp(out)))
        return out

    def advance(self, dt, t, rk=A.RK3):
        _ck(lib().ref_advance(self.h, dt, t, rk))

    def run_steps(self, n_steps, rk=A.RK3, t0=0.0, t_end=float("inf"), census=False):
        t = C.c_double()
        w = C.c_double()
        cen = np.zeros((n_steps, 4), dtype=np.int64)
        _ck(lib().ref_run_steps(self.h, n_steps, rk, t0, t_end, C.byref(t),
                                cen.ctypes.data_as(C.POINTER(C.c_int64)) if census else None,
                                C.byref(w)))
        return t.value, w.value, (cen if census else None)

    def run_log(self, n_steps, rk=A.RK3, t0=0.0, t_end=float("inf")):
        """(t, census[n,4], dt[n]) of n reference steps."""
        t = C.c_double()
        cen = np.zeros((n_steps, 4), dtype=np.int64)
        dts = np.zeros(n_steps)
        _ck(lib().ref_run_steps_log(self.h, n_steps, rk, t0, t_end, C.byref(t),
                                    cen.ctypes.data_as(C.POINTER(C.c_int64)), dts.ctypes.data_as(C.POINTER(C.c_double))))
        return t.value, cen, dts

    def run_until(self, t_end, rk=A.RK3, t0=0.0):
        """run_simulation's loop (run.cpp:96): step while t < t_end - 1e-14 t_end."""
        t, cens, dts = t0, [], []
        while t < t_end - 1e-14 * t_end:
            t, c, d = self.run_log(1, rk, t, t_end)
            cens.append(c[0])
            dts.append(d[0])
        return t, np.array(cens, dtype=np.int64).reshape(-1, 4), np.array(dts)

    def labels(self, step=False):
        out = np.zeros(self.n_cells, dtype=np.uint8)
        _ck(lib().ref_get_labels(self.h, out.ctypes.data_as(C.POINTER(C.c_uint8)), 1 if step else 0))
        return out

    def face_values(self):
        L = np.zeros((self.n_faces * self.n_qp, 4))
        R = np.zeros_like(L)
        _ck(lib().ref_get_face_values(self.h, _dp(L), _dp(R)))
        return L, R

    def dofs(self):
        d = np.zeros((self.n_cells, self.K, 4))
        _ck(lib().ref_get_dofs(self.h, _dp(d)))
        return d

    def bounds(self):
        b = np.zeros((self.n_cells, 4))
        _ck(lib().ref_get_bounds(self.h, _dp(b)))
        return b

    def phase_times(self):
        p = np.zeros(4)
        _ck(lib().ref_get_phase_times(self.h, _dp(p)))
        return p

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_solver_free(self.h)
            self.h = None


def write_field_snapshot(mesh: "RefMesh", state, labels, gamma, path):
    u = np.ascontiguousarray(state, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint8)
    _ck(lib().ref_write_field_snapshot(mesh.h, u.ctypes.data_as(C.POINTER(C.c_double)),
                                       lab.ctypes.data_as(C.POINTER(C.c_uint8)), gamma, str(path).encode()))


def write_census_csv(rows, n_cells, path):
    arr = (A.CensusRow * max(1, len(rows)))()
    for i, (step, t, dt, counts) in enumerate(rows):
        arr[i].step, arr[i].t, arr[i].dt = step, t, dt
        for k in range(4):
            arr[i].counts[k] = int(counts[k])
    _ck(lib().ref_write_census_csv(arr, len(rows), n_cells, str(path).encode()))


def write_timing_csv(rows, path):
    arr = (A.TimingRow * max(1, len(rows)))()
    for i, r in enumerate(rows):
        arr[i].step = r[0]
        arr[i].wall, arr[i].reconstruct, arr[i].detect, arr[i].weights, arr[i].flux = r[1:6]
    _ck(lib().ref_write_timing_csv(arr, len(rows), str(path).encode()))
