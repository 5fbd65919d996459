"""Host setup wrappers: meshes, operator precompute and initial conditions.

These are the callers on either side of the stage pass,
implemented natively in csrc/setup_*.cpp and reached through the C ABI.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A

AXIS = {"none": 0, "x": 1, "y": 2, "both": 3}


def _lib():
    return A.load_library()


def _ck(rc):
    if rc != A.OK:
        raise A.error_for(rc, _lib().ucfvb_last_error(None).decode())


class Mesh:
    """Flattened ucfv::Mesh (reference include/ucfv/mesh.hpp:47-75) owned by the native library."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        self._view = A.MeshView()
        _ck(_lib().ucfvb_mesh_get_view(self._h, C.byref(self._view)))

    @classmethod
    def structured_tri(cls, nx, ny, rect=(0.0, 0.0, 1.0, 1.0), diagonal="uniform", jitter=0.0, seed=0,
                       periodic="both", tol=1e-8, n_qp=2):
        """generate_structured_tri (mesh.cpp:137-157) + seeded interior jitter + pair_periodic."""
        h = C.c_void_p()
        _ck(_lib().ucfvb_mesh_structured_tri(nx, ny, *map(float, rect), 1 if diagonal == "alternating" else 0,
                                             float(jitter), int(seed), AXIS[periodic], float(tol), int(n_qp),
                                             C.byref(h)))
        return cls(h.value)

    @classmethod
    def structured_quad(cls, nx, ny, rect=(0.0, 0.0, 1.0, 1.0), periodic="both", tol=1e-8, n_qp=2):
        h = C.c_void_p()
        _ck(_lib().ucfvb_mesh_structured_quad(nx, ny, *map(float, rect), AXIS[periodic], float(tol), int(n_qp),
                                              C.byref(h)))
        return cls(h.value)

    @property
    def view(self) -> A.MeshView:
        return self._view

    @property
    def n_cells(self) -> int:
        return self._view.n_cells

    @property
    def n_faces(self) -> int:
        return self._view.n_faces

    def numpy(self) -> dict:
        return A.mesh_view_to_numpy(self._view)

    def project_initial(self, ic, params, seed=0, degree=4, gamma=1.4, n_threads=0):
        """Cell averages of a built-in IC (cases.cpp:62-76); see ucfvb.h for the ic codes."""
        p = np.ascontiguousarray(params, dtype=np.float64)
        u = np.zeros((self.n_cells, 4))
        _ck(_lib().ucfvb_project_initial(C.byref(self._view), int(ic), p.ctypes.data_as(A.c_dp), len(p),
                                         int(seed), int(degree), float(gamma), int(n_threads),
                                         u.ctypes.data_as(A.c_dp)))
        return u

    def __del__(self):
        if getattr(self, "_h", None) and A._LIB is not None:
            A._LIB.ucfvb_mesh_free(self._h)
            self._h = None


class Stencils:
    """Flattened ucfv::StencilSet built by the native precompute (stencil.cpp:192-284)."""

    def __init__(self, mesh: Mesh, order: int, si_exponent: int = A.SI_PAPER, n_threads: int = 0):
        self.mesh = mesh  # the views borrow the mesh
        h = C.c_void_p()
        _ck(_lib().ucfvb_build_stencils(C.byref(mesh.view), int(order), int(si_exponent), int(n_threads),
                                        C.byref(h)))
        self._h = h
        self._view = A.StencilView()
        _ck(_lib().ucfvb_stencils_get_view(self._h, C.byref(self._view)))

    @property
    def view(self) -> A.StencilView:
        return self._view

    def numpy(self) -> dict:
        return A.stencil_view_to_numpy(self._view)

    def __del__(self):
        if getattr(self, "_h", None) and A._LIB is not None:
            A._LIB.ucfvb_stencils_free(self._h)
            self._h = None
