"""Domain decomposition for the multi-GPU stage pass, over the
native partitioner / subdomain builder (csrc/decompose.cpp)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A


def _lib():
    return A.load_library()


def _ck(rc):
    if rc != A.OK:
        raise A.error_for(rc, _lib().ucfvb_last_error(None).decode())


def partition_rcb(mesh, n_parts: int) -> np.ndarray:
    """Recursive coordinate bisection of cell centroids into n_parts balanced parts."""
    part = np.zeros(mesh.view.n_cells, dtype=np.int32)
    _ck(_lib().ucfvb_partition_rcb(C.byref(mesh.view), int(n_parts), part.ctypes.data_as(A.c_i32p)))
    return part


class Peer:
    def __init__(self, rank, send, recv_begin, n_recv):
        self.rank, self.send, self.recv_begin, self.n_recv = rank, send, recv_begin, n_recv


class Subdomain:
    """Rank `rank`'s owned cells + stencil-depth halo as a local mesh/stencil pair.

    Local cells are [owned interior | owned sent cells | halo grouped by owner];
    `gid` maps local -> global.
    Keep the global mesh alive (the local view borrows its vertex array)."""

    def __init__(self, mesh, stencils, part: np.ndarray, n_parts: int, rank: int):
        self._keep = (mesh, stencils, part)
        part = np.ascontiguousarray(part, dtype=np.int32)
        self._part = part
        h = C.c_void_p()
        _ck(_lib().ucfvb_subdomain_build(C.byref(mesh.view), C.byref(stencils.view), part.ctypes.data_as(A.c_i32p),
                                         int(n_parts), int(rank), C.byref(h)))
        self._h = h
        self.rank, self.n_parts = rank, n_parts
        self.mesh_view, self.stencil_view = A.MeshView(), A.StencilView()
        _ck(_lib().ucfvb_subdomain_views(h, C.byref(self.mesh_view), C.byref(self.stencil_view)))
        no, nl, npr = C.c_int32(), C.c_int32(), C.c_int32()
        _ck(_lib().ucfvb_subdomain_info(h, C.byref(no), C.byref(nl), C.byref(npr)))
        self.n_owned, self.n_local = no.value, nl.value
        ni = C.c_int32()
        _ck(_lib().ucfvb_subdomain_interior(h, C.byref(ni)))
        self.n_interior = ni.value  # owned cells [0, n_interior) are never sent
        self.gid = np.zeros(self.n_local, dtype=np.int32)
        _ck(_lib().ucfvb_subdomain_global_ids(h, self.gid.ctypes.data_as(A.c_i32p)))
        self.peers = []
        for i in range(npr.value):
            r, ns, nr, rb = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
            _ck(_lib().ucfvb_subdomain_peer(h, i, C.byref(r), C.byref(ns), C.byref(nr), C.byref(rb)))
            send = np.zeros(ns.value, dtype=np.int32)
            if ns.value:
                _ck(_lib().ucfvb_subdomain_send_list(h, i, send.ctypes.data_as(A.c_i32p)))
            self.peers.append(Peer(r.value, send, rb.value, nr.value))

    @property
    def view(self):  # the local mesh view (so a Subdomain stands in for a Mesh)
        return self.mesh_view

    @property
    def handle(self):
        return self._h

    def local_state(self, u_global: np.ndarray) -> np.ndarray:
        return np.ascontiguousarray(u_global[self.gid])

    def __del__(self):
        if getattr(self, "_h", None) and A._LIB is not None:
            A._LIB.ucfvb_subdomain_free(self._h)
            self._h = None
