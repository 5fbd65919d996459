"""Python mirror of the 3D C ABI (include/ucfvb3.h): periodic hexahedral /
tetrahedral meshes, the 3D operator precompute and the device solver for
BASELINE configs 4-5.

The class names follow the reference interface they generalise
(`ucfv::Solver`, include/ucfv/solver.hpp:52-100: state, max_stable_dt,
advance, compute_residual, step_labels). Every compute call goes through
libucfvb.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A

NV = 5
HEX, TET = 0, 1
IC_TGV, IC_RANDOM_PHASE, IC_UNIFORM, IC_BLAST = 0, 1, 2, 3

P = C.POINTER
_i32p, _i8p, _dp = P(C.c_int32), P(C.c_int8), P(C.c_double)


class MeshView3(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("kind", "nx", "ny", "nz", "n_types", "n_cells", "n_faces", "nf", "nq",
                                         "nvc", "cell_order")] + [
        ("period", C.c_double * 3),
        ("cell_vtx", _dp), ("cell_centroid", _dp), ("cell_volume", _dp), ("cell_h", _dp),
        ("cell_faces", _i32p), ("cell_nbr", _i32p), ("cell_nbr_shift", _i32p), ("cell_side", _i8p),
        ("face_left", _i32p), ("face_right", _i32p), ("face_qp", _dp), ("face_normal", _dp), ("face_wa", _dp),
        ("face_vtx", _dp),
    ]


class StencilView3(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("order", "K", "M", "MD", "nf", "nq", "Q", "n_cells", "n_ops",
                                         "si_exponent")] + [
        ("central", _i32p), ("op_index", _i32p), ("pinv", _dp), ("pinv_lin", _dp), ("dir_members", _i32p),
        ("pinv_dir", _dp), ("oi", _dp), ("phi", _dp), ("qp_slot", _i32p),
    ]


_DECLARED = False


def lib():
    global _DECLARED
    L = A.load_library()
    if not _DECLARED:
        H = C.c_void_p
        sig = {
            "ucfvb3_last_error": (C.c_char_p, [H]),
            "ucfvb3_mesh_periodic_box": (C.c_int32, [C.c_int32] * 3 + [C.c_double] * 3 +
                                         [C.c_int32, C.c_double, C.c_uint64, C.c_int32, C.c_int32, P(H)]),
            "ucfvb3_mesh_get_view": (C.c_int32, [H, P(MeshView3)]),
            "ucfvb3_mesh_free": (None, [H]),
            "ucfvb3_build_stencils": (C.c_int32, [P(MeshView3), C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(H)]),
            "ucfvb3_stencils_get_view": (C.c_int32, [H, P(StencilView3)]),
            "ucfvb3_stencils_free": (None, [H]),
            "ucfvb3_project_initial": (C.c_int32, [P(MeshView3), C.c_int32, _dp, C.c_int32, C.c_uint64, C.c_int32,
                                                   C.c_double, C.c_int32, _dp]),
            "ucfvb3_create": (C.c_int32, [P(MeshView3), P(StencilView3), P(A.Options), C.c_int32, P(H)]),
            "ucfvb3_destroy": (None, [H]),
            "ucfvb3_set_state": (C.c_int32, [H, _dp]),
            "ucfvb3_get_state": (C.c_int32, [H, _dp]),
            "ucfvb3_max_stable_dt": (C.c_int32, [H, _dp]),
            "ucfvb3_advance": (C.c_int32, [H, C.c_double, C.c_double, C.c_int32]),
            "ucfvb3_run_steps": (C.c_int32, [H, C.c_int32, C.c_double, C.c_int32, _dp]),
            "ucfvb3_compute_residual": (C.c_int32, [H, _dp, C.c_double, _dp]),
            "ucfvb3_advance_host": (C.c_int32, [H, _dp, _dp, C.c_int32, C.c_int32, C.c_double, _dp]),
            "ucfvb3_advance_host_batch": (C.c_int32, [H, C.c_int32, C.POINTER(_dp), C.POINTER(_dp), C.c_int32,
                                                  C.c_int32, C.c_double, _dp]),
            "ucfvb3_get_labels": (C.c_int32, [H, C.c_int32, P(C.c_uint8)]),
            "ucfvb3_get_face_values": (C.c_int32, [H, _dp]),
            "ucfvb3_get_census": (C.c_int32, [H, P(C.c_int64)]),
            "ucfvb3_get_nad_ties": (C.c_int32, [H, P(C.c_int64)]),
            "ucfvb3_launch_count": (C.c_int64, [H]),
            "ucfvb3_partition_rcb": (C.c_int32, [P(MeshView3), C.c_int32, _i32p]),
            "ucfvb3_subdomain_build": (C.c_int32, [P(MeshView3), P(StencilView3), _i32p, C.c_int32, C.c_int32,
                                                   P(H)]),
            "ucfvb3_subdomain_views": (C.c_int32, [H, P(MeshView3), P(StencilView3)]),
            "ucfvb3_subdomain_info": (C.c_int32, [H, _i32p, _i32p, _i32p]),
            "ucfvb3_subdomain_global_ids": (C.c_int32, [H, _i32p]),
            "ucfvb3_subdomain_peer": (C.c_int32, [H, C.c_int32, _i32p, _i32p, _i32p, _i32p]),
            "ucfvb3_subdomain_send_list": (C.c_int32, [H, C.c_int32, _i32p]),
            "ucfvb3_subdomain_free": (None, [H]),
            "ucfvb3_decomp_last_error": (C.c_char_p, []),
            "ucfvb3_create_sub": (C.c_int32, [H, P(A.Options), C.c_int32, P(H)]),
            "ucfvb3_attach_nccl": (C.c_int32, [H, P(C.c_uint8), C.c_int32, C.c_int32]),
            "ucfvb3_set_phase_timing": (C.c_int32, [H, C.c_int32]),
            "ucfvb3_get_phase_times": (C.c_int32, [H, _dp]),
            "ucfvb3_stream": (C.c_void_p, [H]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _DECLARED = True
    return L


def _ck(rc, h=None):
    if rc != A.OK:
        msg = lib().ucfvb3_last_error(h)
        raise A.error_for(rc, msg.decode() if msg else f"status {rc}")


def _np(ptr, n, dtype):
    return np.ctypeslib.as_array(ptr, shape=(n,)).view(dtype) if n else np.zeros(0, dtype)


class Mesh3:
    """Periodic box of nx*ny*nz cubes (hexahedra, or 6 Freudenthal tetrahedra
    each) with seeded vertex jitter; face rules for polynomial `order`."""

    def __init__(self, n, length=2 * np.pi, kind=HEX, jitter=0.0, seed=1, order=2, n_threads=0):
        nx, ny, nz = (n, n, n) if np.isscalar(n) else n
        lx, ly, lz = (length,) * 3 if np.isscalar(length) else length
        h = C.c_void_p()
        _ck(lib().ucfvb3_mesh_periodic_box(nx, ny, nz, lx, ly, lz, kind, jitter, seed, order, n_threads,
                                           C.byref(h)))
        self._h = h
        self.view = MeshView3()
        _ck(lib().ucfvb3_mesh_get_view(h, C.byref(self.view)))
        v = self.view
        self.n_cells, self.n_faces, self.nf, self.nq = v.n_cells, v.n_faces, v.nf, v.nq
        self.kind = kind

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ucfvb3_mesh_free(self._h)
            self._h = None

    # numpy views (borrowed from the C++ mesh)
    @property
    def volume(self):
        return np.ctypeslib.as_array(self.view.cell_volume, shape=(self.n_cells,))

    @property
    def h(self):
        return np.ctypeslib.as_array(self.view.cell_h, shape=(self.n_cells,))

    @property
    def centroid(self):
        return np.ctypeslib.as_array(self.view.cell_centroid, shape=(self.n_cells, 3))

    def cube_and_type(self):
        """lattice cube and type of every cell (ucfvb3_mesh_view.cell_order)"""
        c = np.arange(self.n_cells, dtype=np.int64)
        nt = self.view.n_types
        if self.view.cell_order:
            return ((c >> 5) // nt) * 32 + (c & 31), (c >> 5) % nt
        return c // nt, c % nt

    def arr(self, name, shape, dtype=None):
        a = np.ctypeslib.as_array(getattr(self.view, name), shape=shape)
        return a if dtype is None else a.view(dtype)

    def project_initial(self, ic, params, seed=1, degree=4, gamma=1.4, n_threads=0):
        p = np.ascontiguousarray(params, dtype=np.float64)
        out = np.zeros((self.n_cells, NV))
        _ck(lib().ucfvb3_project_initial(C.byref(self.view), ic, p.ctypes.data_as(_dp), len(p), seed, degree,
                                         gamma, n_threads, out.ctypes.data_as(_dp)))
        return out


class Stencils3:
    def __init__(self, mesh: Mesh3, order, si_exponent=A.SI_PAPER, lattice_classes=False, n_threads=0):
        h = C.c_void_p()
        _ck(lib().ucfvb3_build_stencils(C.byref(mesh.view), order, si_exponent, int(lattice_classes), n_threads,
                                        C.byref(h)))
        self._h = h
        self.mesh = mesh
        self.view = StencilView3()
        _ck(lib().ucfvb3_stencils_get_view(h, C.byref(self.view)))
        v = self.view
        self.K, self.M, self.MD, self.Q, self.n_ops = v.K, v.M, v.MD, v.Q, v.n_ops

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ucfvb3_stencils_free(self._h)
            self._h = None

    def arr(self, name, shape):
        return np.ctypeslib.as_array(getattr(self.view, name), shape=shape)


def _ckd(rc):
    if rc != A.OK:
        raise A.error_for(rc, lib().ucfvb3_decomp_last_error().decode())


def partition_rcb3(mesh: Mesh3, n_parts: int) -> np.ndarray:
    """recursive coordinate bisection of the cell centroids into n_parts parts"""
    part = np.zeros(mesh.n_cells, dtype=np.int32)
    _ckd(lib().ucfvb3_partition_rcb(C.byref(mesh.view), int(n_parts), part.ctypes.data_as(_i32p)))
    return part


class Peer3:
    def __init__(self, rank, send, recv_begin, n_recv):
        self.rank, self.send, self.recv_begin, self.n_recv = rank, send, recv_begin, n_recv


class Subdomain3:
    """Rank `rank`'s owned cells + stencil-depth halo (csrc/decompose3.cpp) as
    a local mesh/stencil pair; local order [owned | halo grouped by owner].
    Keeps the global mesh and stencils alive (lattice-class rows are borrowed)."""

    def __init__(self, mesh: Mesh3, stencils: Stencils3, part, n_parts: int, rank: int):
        self._keep = (mesh, stencils)
        part = np.ascontiguousarray(part, dtype=np.int32)
        h = C.c_void_p()
        _ckd(lib().ucfvb3_subdomain_build(C.byref(mesh.view), C.byref(stencils.view), part.ctypes.data_as(_i32p),
                                          int(n_parts), int(rank), C.byref(h)))
        self._h = h
        self.rank, self.n_parts = rank, n_parts
        self.mesh_view, self.stencil_view = MeshView3(), StencilView3()
        _ckd(lib().ucfvb3_subdomain_views(h, C.byref(self.mesh_view), C.byref(self.stencil_view)))
        no, nl, npr = C.c_int32(), C.c_int32(), C.c_int32()
        _ckd(lib().ucfvb3_subdomain_info(h, C.byref(no), C.byref(nl), C.byref(npr)))
        self.n_owned, self.n_local = no.value, nl.value
        self.gid = np.zeros(self.n_local, dtype=np.int32)
        _ckd(lib().ucfvb3_subdomain_global_ids(h, self.gid.ctypes.data_as(_i32p)))
        self.peers = []
        for i in range(npr.value):
            r, ns, nr, rb = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
            _ckd(lib().ucfvb3_subdomain_peer(h, i, C.byref(r), C.byref(ns), C.byref(nr), C.byref(rb)))
            send = np.zeros(ns.value, dtype=np.int32)
            if ns.value:
                _ckd(lib().ucfvb3_subdomain_send_list(h, i, send.ctypes.data_as(_i32p)))
            self.peers.append(Peer3(r.value, send, rb.value, nr.value))
        # a Mesh3-like facade for the port and the solver
        self.view = self.mesh_view
        self.n_cells, self.n_faces = self.n_local, self.mesh_view.n_faces
        self.nf, self.nq = self.mesh_view.nf, self.mesh_view.nq

    def local_state(self, u_global):
        return np.ascontiguousarray(u_global[self.gid])

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ucfvb3_subdomain_free(self._h)
            self._h = None


class _StencilFacade:
    def __init__(self, view):
        self.view = view


class Solver3:
    """ucfv::Solver API (solver.hpp:52-100) for the 3D stage pass on one GPU."""

    def __init__(self, mesh: Mesh3, opt: A.Options, stencils: Stencils3, device=0):
        h = C.c_void_p()
        self.mesh, self.stencils = mesh, stencils
        self.n = mesh.n_cells
        _ck(lib().ucfvb3_create(C.byref(mesh.view), C.byref(stencils.view), C.byref(opt), device, C.byref(h)))
        self._h = h

    @classmethod
    def on_subdomain(cls, sub: "Subdomain3", opt: A.Options, device=0):
        """Solver over a Subdomain3: census and errors cover owned cells;
        attach_nccl adds the per-stage halo exchange and the dt all-reduce."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        self.mesh, self.stencils, self.sub = sub, _StencilFacade(sub.stencil_view), sub
        self.n = sub.n_local
        _ck(lib().ucfvb3_create_sub(sub._h, C.byref(opt), device, C.byref(h)))
        self._h = h
        return self

    def attach_nccl(self, unique_id: bytes, rank: int, world: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _ck(lib().ucfvb3_attach_nccl(self._h, buf, rank, world), self._h)

    def close(self):
        if getattr(self, "_h", None):
            lib().ucfvb3_destroy(self._h)
            self._h = None

    __del__ = close

    @property
    def state(self):
        out = np.zeros((self.n, NV))
        _ck(lib().ucfvb3_get_state(self._h, out.ctypes.data_as(_dp)), self._h)
        return out

    @state.setter
    def state(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64).reshape(self.n, NV)
        _ck(lib().ucfvb3_set_state(self._h, u.ctypes.data_as(_dp)), self._h)

    def max_stable_dt(self):
        d = C.c_double()
        _ck(lib().ucfvb3_max_stable_dt(self._h, C.byref(d)), self._h)
        return d.value

    def advance(self, dt, t=0.0, rk=A.RK3):
        _ck(lib().ucfvb3_advance(self._h, dt, t, rk), self._h)

    def run_steps(self, n_steps, t0=0.0, rk=A.RK3):
        t = C.c_double()
        _ck(lib().ucfvb3_run_steps(self._h, n_steps, t0, rk, C.byref(t)), self._h)
        return t.value

    def advance_host(self, u_in, n_steps=1, rk=A.RK3, t0=0.0, u_out=None):
        """host state in -> n_steps steps (device dt) -> host state out, one synchronisation"""
        u_in = np.ascontiguousarray(u_in, dtype=np.float64).reshape(self.n, NV)
        out = np.empty_like(u_in) if u_out is None else u_out
        t = C.c_double()
        _ck(lib().ucfvb3_advance_host(self._h, u_in.ctypes.data_as(_dp), out.ctypes.data_as(_dp), n_steps, rk, t0,
                                      C.byref(t)), self._h)
        return out, t.value

    def advance_host_batch(self, u_in, n_steps=1, rk=A.RK3, t0=0.0, u_out=None):
        """advance_host over independent states, pipelined (uploads / downloads overlap the stepping).
        Returns (outs, t[n_batch])."""
        ins = [np.ascontiguousarray(u, dtype=np.float64).reshape(self.n, NV) for u in u_in]
        outs = [np.empty_like(u) for u in ins] if u_out is None else list(u_out)
        nb = len(ins)
        tab_in = (_dp * nb)(*[u.ctypes.data_as(_dp) for u in ins])
        tab_out = (_dp * nb)(*[u.ctypes.data_as(_dp) for u in outs])
        t = np.zeros(nb)
        _ck(lib().ucfvb3_advance_host_batch(self._h, nb, tab_in, tab_out, n_steps, rk, t0, t.ctypes.data_as(_dp)),
            self._h)
        return outs, t

    def compute_residual(self, u, t=0.0):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros((self.n, NV))
        _ck(lib().ucfvb3_compute_residual(self._h, u.ctypes.data_as(_dp), t, out.ctypes.data_as(_dp)), self._h)
        return out

    def labels(self, step=False):
        out = np.zeros(self.n, np.uint8)
        _ck(lib().ucfvb3_get_labels(self._h, int(step), out.ctypes.data_as(P(C.c_uint8))), self._h)
        return out

    def step_labels(self):
        return self.labels(step=True)

    def face_values(self):
        out = np.zeros((self.mesh.n_faces, self.mesh.nq, 2, NV))
        _ck(lib().ucfvb3_get_face_values(self._h, out.ctypes.data_as(_dp)), self._h)
        return out

    def census(self):
        out = (C.c_int64 * 4)()
        _ck(lib().ucfvb3_get_census(self._h, out), self._h)
        return list(out)

    def nad_ties(self):
        t = C.c_int64()
        _ck(lib().ucfvb3_get_nad_ties(self._h, C.byref(t)), self._h)
        return t.value

    def set_phase_timing(self, on):
        _ck(lib().ucfvb3_set_phase_timing(self._h, int(on)), self._h)

    def phase_times(self):
        out = np.zeros(5)
        _ck(lib().ucfvb3_get_phase_times(self._h, out.ctypes.data_as(_dp)), self._h)
        return out

    def launch_count(self):
        return lib().ucfvb3_launch_count(self._h)

    def stream(self):
        return lib().ucfvb3_stream(self._h)
