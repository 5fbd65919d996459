"""Python face of the B200 stage pass: mirrors ucfv::Solver
(/root/reference/proj/include/ucfv/solver.hpp:52-100) over the C ABI.

    solver = Solver(mesh, options, bcs)       # Solver(mesh, opt, bcs)
    solver.state = u0                          # state() = ...
    dt = solver.max_stable_dt()
    solver.advance(dt, t)                      # one step (RK54 like the reference, or RK3)
    r = solver.compute_residual(u, t)
    solver.step_labels()

Every call runs on the GPU through libucfvb.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A
from .mesh import Mesh, Stencils


def _dp(a):
    return a.ctypes.data_as(A.c_dp)


def make_options(**kw) -> A.Options:
    """SolverOptions with keyword overrides (mode may be a name: 'hybrid', 'cwenoz', ...)."""
    return A.options_from_dict(**kw)


def make_bcs(mapping) -> list:
    """{'left': 'outflow', 'right': ('fixed', state), 'top': 'wall'} -> [BC]."""
    out = []
    for patch, spec in (mapping or {}).items():
        if isinstance(spec, str):
            kind, state = spec, (0.0, 0.0, 0.0, 0.0)
        else:
            kind, state = spec[0], spec[1]
        k = {"outflow": A.BC_OUTFLOW, "wall": A.BC_WALL, "fixed": A.BC_FIXED}[kind]
        out.append(A.BC(patch.encode(), k, (C.c_double * 4)(*state)))
    return out


class Solver:
    """Device-resident drop-in for ucfv::Solver.

    mesh: a `Mesh` (or any object with `.view` -> MeshView); stencils: a
    `Stencils` built for options.order, or None to build them here; bcs: a
    list of A.BC or a {patch: kind} mapping.
    """

    def __init__(self, mesh, options: A.Options | None = None, bcs=None, stencils=None, device: int = 0,
                 keep=(), subdomain=None):
        self._lib = A.load_library()
        self.options = options if options is not None else A.default_options()
        if subdomain is None and stencils is None:
            stencils = Stencils(mesh, self.options.order, self.options.si_exponent)
        self.mesh = mesh
        self.stencils = stencils
        self.subdomain = subdomain
        self._keep = keep
        if isinstance(bcs, dict):
            bcs = make_bcs(bcs)
        bcs = list(bcs or [])
        self._bcs = (A.BC * max(1, len(bcs)))(*bcs)
        h = C.c_void_p()
        if subdomain is not None:
            rc = self._lib.ucfvb_create_sub(subdomain.handle, C.byref(self.options), self._bcs, len(bcs), int(device),
                                            C.byref(h))
            stencils = type("SV", (), {"view": subdomain.stencil_view})()
        else:
            rc = self._lib.ucfvb_create(C.byref(mesh.view), C.byref(stencils.view), C.byref(self.options),
                                        self._bcs, len(bcs), int(device), C.byref(h))
        if rc != A.OK:
            raise A.error_for(rc, self._lib.ucfvb_last_error(None).decode())
        self._h = h
        self.n_cells = self._lib.ucfvb_n_cells(h)
        self.n_faces = self._lib.ucfvb_n_faces(h)
        self.n_qp = self._lib.ucfvb_n_qp(h)
        self.K = stencils.view.K

    @classmethod
    def on_subdomain(cls, subdomain, options=None, bcs=None, device: int = 0):
        """Solver over a Subdomain (decompose.py): owned cells + halo; RK updates,
        dt and census cover owned cells; attach_nccl adds the per-stage halo exchange."""
        return cls(subdomain, options, bcs, device=device, subdomain=subdomain)

    def attach_nccl(self, unique_id: bytes, rank: int, world: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self._ck(self._lib.ucfvb_attach_nccl(self._h, buf, int(rank), int(world)))

    # -- errors ------------------------------------------------------------
    def _ck(self, rc):
        if rc != A.OK:
            raise A.error_for(rc, self._lib.ucfvb_last_error(self._h).decode())

    # -- Solver API ----------------------------------------------------------
    @property
    def state(self) -> np.ndarray:
        u = np.zeros((self.n_cells, 4))
        self._ck(self._lib.ucfvb_get_state(self._h, _dp(u)))
        return u

    @state.setter
    def state(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        if u.shape != (self.n_cells, 4):
            raise ValueError(f"state must be ({self.n_cells}, 4)")
        self._ck(self._lib.ucfvb_set_state(self._h, _dp(u)))

    def set_state(self, u):
        self.state = u

    def get_state(self):
        return self.state

    def max_stable_dt(self) -> float:
        d = C.c_double()
        self._ck(self._lib.ucfvb_max_stable_dt(self._h, C.byref(d)))
        return d.value

    def advance(self, dt: float, t: float, rk: int = A.RK54):
        """One step in place; rk=RK54 is Solver::advance, RK3 the BASELINE integrator."""
        self._ck(self._lib.ucfvb_advance(self._h, float(dt), float(t), int(rk)))

    def compute_residual(self, u, t: float = 0.0) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros((self.n_cells, 4))
        self._ck(self._lib.ucfvb_compute_residual(self._h, _dp(u), float(t), _dp(out)))
        return out

    def run_steps(self, n_steps: int, rk: int = A.RK3, t0: float = 0.0, t_end: float = float("inf"),
                  census: bool = False):
        """run_simulation's stepping loop on the device; returns (t, census[n_steps,4] or None)."""
        t = C.c_double()
        cen = np.zeros((n_steps, 4), dtype=np.int64) if census else None
        self._ck(self._lib.ucfvb_run_steps(self._h, int(n_steps), int(rk), float(t0), float(t_end), C.byref(t),
                                           cen.ctypes.data_as(A.c_i64p) if census else None))
        return t.value, cen

    def advance_host(self, u_in, n_steps: int = 1, rk: int = A.RK3, t0: float = 0.0, u_out=None):
        """host state in -> n_steps steps (device dt) -> host state out, one synchronisation"""
        u_in = np.ascontiguousarray(u_in, dtype=np.float64).reshape(self.n_cells, 4)
        out = np.empty_like(u_in) if u_out is None else u_out
        t = C.c_double()
        self._ck(self._lib.ucfvb_advance_host(self._h, _dp(u_in), _dp(out), n_steps, rk, t0, C.byref(t)))
        return out, t.value

    def advance_host_batch(self, u_in, n_steps: int = 1, rk: int = A.RK3, t0: float = 0.0, u_out=None):
        """advance_host over independent states (an ensemble), pipelined: the PCIe copies of
        neighbouring entries overlap the stepping. u_in / u_out: sequences of [n_cells][4] arrays
        (pinned for true overlap). Returns (outs, t[n_batch])."""
        ins = [np.ascontiguousarray(u, dtype=np.float64).reshape(self.n_cells, 4) for u in u_in]
        outs = [np.empty_like(u) for u in ins] if u_out is None else list(u_out)
        nb = len(ins)
        tab_in = (A.c_dp * nb)(*[_dp(u) for u in ins])
        tab_out = (A.c_dp * nb)(*[_dp(u) for u in outs])
        t = np.zeros(nb)
        self._ck(self._lib.ucfvb_advance_host_batch(self._h, nb, tab_in, tab_out, int(n_steps), int(rk), float(t0),
                                                    _dp(t)))
        return outs, t

    def run_log(self, n_steps: int, rk: int = A.RK3, t0: float = 0.0, t_end: float = float("inf")):
        """run_steps that also returns each step's dt: (t, census[n,4], dt[n])."""
        t = C.c_double()
        cen = np.zeros((n_steps, 4), dtype=np.int64)
        dts = np.zeros(n_steps)
        self._ck(self._lib.ucfvb_run_steps_log(self._h, int(n_steps), int(rk), float(t0), float(t_end), C.byref(t),
                                               cen.ctypes.data_as(A.c_i64p), _dp(dts)))
        return t.value, cen, dts

    def run_until(self, t_end: float, rk: int = A.RK3, t0: float = 0.0, max_steps: int = 1 << 20,
                  census: bool = True):
        """run_simulation's loop (run.cpp:96-132): step while t < t_end - 1e-14 t_end (at most
        max_steps). Returns (t, n_steps, census[n,4] or None, dt[n])."""
        t = C.c_double()
        n = C.c_int32()
        cen = np.zeros((max_steps, 4), dtype=np.int64) if census else None
        dts = np.zeros(max_steps)
        self._ck(self._lib.ucfvb_run_until(self._h, int(max_steps), int(rk), float(t0), float(t_end), C.byref(t),
                                           C.byref(n), cen.ctypes.data_as(A.c_i64p) if census else None, _dp(dts)))
        k = n.value
        return t.value, k, (cen[:k] if census else None), dts[:k]

    def step_labels(self) -> np.ndarray:
        out = np.zeros(self.n_cells, dtype=np.uint8)
        self._ck(self._lib.ucfvb_get_step_labels(self._h, out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out

    def labels(self) -> np.ndarray:
        out = np.zeros(self.n_cells, dtype=np.uint8)
        self._ck(self._lib.ucfvb_get_labels(self._h, out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out

    def census(self) -> np.ndarray:
        c = np.zeros(4, dtype=np.int64)
        self._ck(self._lib.ucfvb_get_census(self._h, c.ctypes.data_as(A.c_i64p)))
        return c

    def nad_ties(self) -> int:
        t = C.c_int64()
        self._ck(self._lib.ucfvb_get_nad_ties(self._h, C.byref(t)))
        return t.value

    LIST_POLICIES = {"chunks": 0, "lists": 1, "auto": 2}

    def set_list_policy(self, policy: str):
        """Troubled-cell class lists: "chunks", "lists" (per cell) or "auto" (default: by chunk fill)."""
        self._ck(self._lib.ucfvb_set_list_policy(self._h, self.LIST_POLICIES[policy]))

    def list_stats(self) -> dict:
        """Class-list sizes of the last synchronised stage and the lists in use."""
        s = np.zeros(5, dtype=np.int64)
        self._ck(self._lib.ucfvb_get_list_stats(self._h, s.ctypes.data_as(A.c_i64p)))
        return {"cwenoz_cells": int(s[0]), "muscl_cells": int(s[1]), "cwenoz_chunks": int(s[2]),
                "muscl_chunks": int(s[3]), "lists": "per-cell" if s[4] else "chunks"}

    def face_values(self):
        L = np.zeros((self.n_faces * self.n_qp, 4))
        R = np.zeros_like(L)
        self._ck(self._lib.ucfvb_get_face_values(self._h, _dp(L), _dp(R)))
        return L, R

    def dofs(self) -> np.ndarray:
        d = np.zeros((self.n_cells, self.K, 4))
        self._ck(self._lib.ucfvb_get_dofs(self._h, _dp(d)))
        return d

    def set_phase_timing(self, on: bool = True):
        self._ck(self._lib.ucfvb_set_phase_timing(self._h, 1 if on else 0))

    def phase_times(self) -> np.ndarray:
        p = np.zeros(4)
        self._ck(self._lib.ucfvb_get_phase_times(self._h, _dp(p)))
        return p

    def launch_count(self) -> int:
        return int(self._lib.ucfvb_launch_count(self._h))

    def state_device_ptr(self) -> int:
        p = A.c_dp()
        self._ck(self._lib.ucfvb_state_device_ptr(self._h, C.byref(p)))
        return C.cast(p, C.c_void_p).value or 0

    def stream(self) -> int:
        s = C.c_void_p()
        self._ck(self._lib.ucfvb_stream(self._h, C.byref(s)))
        return s.value or 0

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ucfvb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Group:
    """In-process loopback group (ucfvb_group_*): the subdomain solvers of one
    n-part partition on one device, stepped together with a rank's multi-GPU
    schedule and device-to-device copies as the halo transport."""

    def __init__(self, parts):
        self._lib = A.load_library()
        self.parts = list(parts)  # keep the solvers alive
        arr = (C.c_void_p * len(self.parts))(*[p._h.value if hasattr(p._h, "value") else p._h for p in self.parts])
        h = C.c_void_p()
        rc = self._lib.ucfvb_group_create(arr, len(self.parts), C.byref(h))
        if rc != A.OK:
            raise A.error_for(rc, self._lib.ucfvb_last_error(None).decode())
        self._h = h

    def run_steps(self, n_steps: int, rk: int = A.RK3, t0: float = 0.0) -> float:
        t = C.c_double()
        rc = self._lib.ucfvb_group_run_steps(self._h, int(n_steps), int(rk), float(t0), C.byref(t))
        if rc != A.OK:
            raise A.error_for(rc, self._lib.ucfvb_last_error(None).decode())
        return t.value

    def launch_count(self) -> int:
        return int(self._lib.ucfvb_group_launch_count(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and A._LIB is not None:
            A._LIB.ucfvb_group_free(self._h)
            self._h = None


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the native library (rank 0 creates, all ranks attach)."""
    lib = A.load_library()
    buf = (C.c_uint8 * 128)()
    rc = lib.ucfvb_nccl_unique_id(buf)
    if rc != A.OK:
        raise A.error_for(rc, lib.ucfvb_last_error(None).decode())
    return bytes(buf)


class ViewHolder:
    """Wraps a raw (MeshView or StencilView) + keep-alive objects so Solver can take views from elsewhere."""

    def __init__(self, view, keep=None):
        self.view = view
        self.keep = keep
