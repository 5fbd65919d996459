"""ctypes mirror of include/ucfvb.h (the C ABI of the B200 stage pass).

Only struct layouts, enums and the library loader live here. The loader
fails loudly when the compiled extension is missing: there is no CPU
fallback for the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["UCFVB_LIB"]) if os.environ.get("UCFVB_LIB") else PKG_DIR / "lib" / "libucfvb.so"  # UCFVB_LIB: A/B builds

# enums (ucfvb.h)
OK, NONPHYSICAL, INVALID, CUDA_ERR, UNSUPPORTED = 0, 1, 2, 3, 4
LINEAR, MUSCL, CWENOZ, HYBRID, FIRST = 0, 1, 2, 3, 4
BARTH_JESPERSEN, VENKATAKRISHNAN = 0, 1
HLLC, HLL = 0, 1
SI_PAPER, SI_LEGACY = 0, 1
RK54, RK3 = 0, 1
SCHEME_LINEAR, SCHEME_CWENOZ, SCHEME_MUSCL, SCHEME_FIRST = 0, 1, 2, 3
BC_NONE, BC_OUTFLOW, BC_WALL, BC_FIXED = 0, 1, 2, 3

MODE_NAMES = {"linear": LINEAR, "muscl": MUSCL, "cwenoz": CWENOZ, "hybrid": HYBRID, "first": FIRST}

P = C.POINTER
c_i32p = P(C.c_int32)
c_i64p = P(C.c_int64)
c_dp = P(C.c_double)


class Margins(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("alpha_m", "beta_m", "alpha_w", "beta_w", "kappa", "deact_n")]


class Options(C.Structure):
    _fields_ = [
        ("order", C.c_int32),
        ("mode", C.c_int32),
        ("limiter", C.c_int32),
        ("riemann", C.c_int32),
        ("margins", Margins),
        ("lambda1p", C.c_double),
        ("weno_eps", C.c_double),
        ("weno_b", C.c_double),
        ("cfl", C.c_double),
        ("venkat_kappa", C.c_double),
        ("si_exponent", C.c_int32),
        ("detect_every_stage", C.c_int32),
        ("gamma", C.c_double),
        ("keep_taps", C.c_int32),
        ("use_graphs", C.c_int32),
    ]


def default_options() -> Options:
    """SolverOptions{} defaults (reference solver.hpp:29-43, detector.hpp:24-31)."""
    o = Options()
    o.order = 3
    o.mode = HYBRID
    o.limiter = BARTH_JESPERSEN
    o.riemann = HLLC
    o.margins = Margins(1e-4, 0.5, 0.0, 0.0, 5.0, 2.0)
    o.lambda1p = 1e3
    o.weno_eps = 1e-3
    o.weno_b = 4.0
    o.cfl = 0.6
    o.venkat_kappa = 5.0
    o.si_exponent = SI_PAPER
    o.detect_every_stage = 1
    o.gamma = 1.4
    o.keep_taps = 0
    o.use_graphs = 1
    return o


class BC(C.Structure):
    _fields_ = [("patch", C.c_char_p), ("kind", C.c_int32), ("state", C.c_double * 4)]


class MeshView(C.Structure):
    _fields_ = [
        ("n_vertices", C.c_int32), ("n_cells", C.c_int32), ("n_faces", C.c_int32),
        ("n_qp", C.c_int32), ("n_patches", C.c_int32),
        ("period_x", C.c_double), ("period_y", C.c_double),
        ("vertices", c_dp),
        ("cell_vtx_ptr", c_i32p), ("cell_vtx", c_i32p),
        ("cell_face_ptr", c_i32p), ("cell_faces", c_i32p),
        ("cell_centroid", c_dp), ("cell_area", c_dp), ("cell_h", c_dp),
        ("face_vtx", c_i32p), ("face_left", c_i32p), ("face_right", c_i32p),
        ("face_normal", c_dp), ("face_length", c_dp), ("face_midpoint", c_dp),
        ("face_qp", c_dp), ("face_qw", c_dp),
        ("face_patch", c_i32p), ("face_partner", c_i32p), ("face_shift", c_i32p),
        ("face_partner_qp", c_i32p),
        ("patch_names", P(C.c_char_p)),
    ]


class CensusRow(C.Structure):
    """ucfvb_census_row = CensusRow (run.hpp:15-19)."""
    _fields_ = [("step", C.c_int32), ("t", C.c_double), ("dt", C.c_double), ("counts", C.c_int64 * 4)]


class TimingRow(C.Structure):
    """ucfvb_timing_row = TimingRow (run.hpp:21-25), per-step phase deltas in seconds."""
    _fields_ = [("step", C.c_int32), ("wall", C.c_double), ("reconstruct", C.c_double), ("detect", C.c_double),
                ("weights", C.c_double), ("flux", C.c_double)]


class StencilView(C.Structure):
    _fields_ = [
        ("order", C.c_int32), ("K", C.c_int32), ("n_qp", C.c_int32), ("si_exponent", C.c_int32),
        ("n_cells", C.c_int32), ("n_dir_stencils", C.c_int32),
        ("central_ptr", c_i64p), ("central", c_i32p),
        ("pinv_off", c_i64p), ("pinv", c_dp),
        ("pinv_lin_off", c_i64p), ("pinv_lin", c_dp),
        ("dir_ptr", c_i64p), ("dir_member_ptr", c_i64p), ("dir_members", c_i32p),
        ("pinv_dir_off", c_i64p), ("pinv_dir", c_dp),
        ("oi", c_dp),
        ("qp_ptr", c_i64p), ("phi_off", c_i64p), ("phi", c_dp), ("qp_slot", c_i32p),
    ]


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(int(n),)).astype(dtype, copy=True)


def mesh_view_to_numpy(v: MeshView) -> dict:
    """Copy a mesh view into a dict of numpy arrays (for tests and fixtures)."""
    nc, nf, nq, nv = v.n_cells, v.n_faces, v.n_qp, v.n_vertices
    cvp = _arr(v.cell_vtx_ptr, nc + 1, np.int32)
    cfp = _arr(v.cell_face_ptr, nc + 1, np.int32)
    return {
        "n_qp": np.int32(nq),
        "period": np.array([v.period_x, v.period_y]),
        "vertices": _arr(v.vertices, 2 * nv, np.float64).reshape(nv, 2),
        "cell_vtx_ptr": cvp,
        "cell_vtx": _arr(v.cell_vtx, cvp[-1], np.int32),
        "cell_face_ptr": cfp,
        "cell_faces": _arr(v.cell_faces, cfp[-1], np.int32),
        "cell_centroid": _arr(v.cell_centroid, 2 * nc, np.float64).reshape(nc, 2),
        "cell_area": _arr(v.cell_area, nc, np.float64),
        "cell_h": _arr(v.cell_h, nc, np.float64),
        "face_vtx": _arr(v.face_vtx, 2 * nf, np.int32).reshape(nf, 2),
        "face_left": _arr(v.face_left, nf, np.int32),
        "face_right": _arr(v.face_right, nf, np.int32),
        "face_normal": _arr(v.face_normal, 2 * nf, np.float64).reshape(nf, 2),
        "face_length": _arr(v.face_length, nf, np.float64),
        "face_midpoint": _arr(v.face_midpoint, 2 * nf, np.float64).reshape(nf, 2),
        "face_qp": _arr(v.face_qp, 2 * nf * nq, np.float64).reshape(nf, nq, 2),
        "face_qw": _arr(v.face_qw, nf * nq, np.float64).reshape(nf, nq),
        "face_patch": _arr(v.face_patch, nf, np.int32),
        "face_partner": _arr(v.face_partner, nf, np.int32),
        "face_shift": _arr(v.face_shift, 2 * nf, np.int32).reshape(nf, 2),
        "face_partner_qp": _arr(v.face_partner_qp, nf * nq, np.int32).reshape(nf, nq),
        "patch_names": np.array([v.patch_names[i].decode() for i in range(v.n_patches)]),
    }


def stencil_view_to_numpy(v: StencilView) -> dict:
    nc, nd, K = v.n_cells, v.n_dir_stencils, v.K
    cp = _arr(v.central_ptr, nc + 1, np.int64)
    po = _arr(v.pinv_off, nc + 1, np.int64)
    plo = _arr(v.pinv_lin_off, nc + 1, np.int64)
    dp = _arr(v.dir_ptr, nc + 1, np.int64)
    dmp = _arr(v.dir_member_ptr, nd + 1, np.int64)
    pdo = _arr(v.pinv_dir_off, nd + 1, np.int64)
    qpp = _arr(v.qp_ptr, nc + 1, np.int64)
    pho = _arr(v.phi_off, nc + 1, np.int64)
    return {
        "meta": np.array([v.order, K, v.n_qp, v.si_exponent, nc, nd], dtype=np.int64),
        "central_ptr": cp,
        "central": _arr(v.central, 3 * cp[-1], np.int32).reshape(-1, 3),
        "pinv_off": po,
        "pinv": _arr(v.pinv, po[-1], np.float64),
        "pinv_lin_off": plo,
        "pinv_lin": _arr(v.pinv_lin, plo[-1], np.float64),
        "dir_ptr": dp,
        "dir_member_ptr": dmp,
        "dir_members": _arr(v.dir_members, dmp[-1], np.int32),
        "pinv_dir_off": pdo,
        "pinv_dir": _arr(v.pinv_dir, pdo[-1], np.float64),
        "oi": _arr(v.oi, nc * K * K, np.float64),
        "qp_ptr": qpp,
        "phi_off": pho,
        "phi": _arr(v.phi, pho[-1], np.float64),
        "qp_slot": _arr(v.qp_slot, qpp[-1], np.int32),
    }


class _Keep:
    """Holds numpy buffers alive behind a view built from a dict."""

    def __init__(self):
        self.bufs = []

    def ptr(self, a, ctype):
        a = np.ascontiguousarray(a)
        self.bufs.append(a)
        return a.ctypes.data_as(P(ctype))


def mesh_view_from_numpy(d: dict):
    k = _Keep()
    v = MeshView()
    v.n_vertices = d["vertices"].shape[0]
    v.n_cells = d["cell_area"].shape[0]
    v.n_faces = d["face_left"].shape[0]
    v.n_qp = int(d["n_qp"])
    names = [str(s).encode() for s in d["patch_names"]]
    v.n_patches = len(names)
    v.period_x, v.period_y = float(d["period"][0]), float(d["period"][1])
    for name, ct, dt in [
        ("vertices", C.c_double, np.float64), ("cell_vtx_ptr", C.c_int32, np.int32),
        ("cell_vtx", C.c_int32, np.int32), ("cell_face_ptr", C.c_int32, np.int32),
        ("cell_faces", C.c_int32, np.int32), ("cell_centroid", C.c_double, np.float64),
        ("cell_area", C.c_double, np.float64), ("cell_h", C.c_double, np.float64),
        ("face_vtx", C.c_int32, np.int32), ("face_left", C.c_int32, np.int32),
        ("face_right", C.c_int32, np.int32), ("face_normal", C.c_double, np.float64),
        ("face_length", C.c_double, np.float64), ("face_midpoint", C.c_double, np.float64),
        ("face_qp", C.c_double, np.float64), ("face_qw", C.c_double, np.float64),
        ("face_patch", C.c_int32, np.int32), ("face_partner", C.c_int32, np.int32),
        ("face_shift", C.c_int32, np.int32), ("face_partner_qp", C.c_int32, np.int32),
    ]:
        setattr(v, name, k.ptr(np.asarray(d[name], dtype=dt), ct))
    arr = (C.c_char_p * max(1, len(names)))(*names)
    k.bufs.append(arr)
    v.patch_names = C.cast(arr, P(C.c_char_p))
    return v, k


def stencil_view_from_numpy(d: dict):
    k = _Keep()
    v = StencilView()
    m = d["meta"]
    v.order, v.K, v.n_qp, v.si_exponent, v.n_cells, v.n_dir_stencils = (int(x) for x in m)
    for name, ct, dt in [
        ("central_ptr", C.c_int64, np.int64), ("central", C.c_int32, np.int32),
        ("pinv_off", C.c_int64, np.int64), ("pinv", C.c_double, np.float64),
        ("pinv_lin_off", C.c_int64, np.int64), ("pinv_lin", C.c_double, np.float64),
        ("dir_ptr", C.c_int64, np.int64), ("dir_member_ptr", C.c_int64, np.int64),
        ("dir_members", C.c_int32, np.int32), ("pinv_dir_off", C.c_int64, np.int64),
        ("pinv_dir", C.c_double, np.float64), ("oi", C.c_double, np.float64),
        ("qp_ptr", C.c_int64, np.int64), ("phi_off", C.c_int64, np.int64),
        ("phi", C.c_double, np.float64), ("qp_slot", C.c_int32, np.int32),
    ]:
        setattr(v, name, k.ptr(np.asarray(d[name], dtype=dt).ravel(), ct))
    return v, k


def options_from_dict(**kw) -> Options:
    o = default_options()
    for key, val in kw.items():
        if key == "mode" and isinstance(val, str):
            val = MODE_NAMES[val]
        if key == "margins" and not isinstance(val, Margins):
            val = Margins(*val)
        setattr(o, key, val)
    return o


_LIB = None


def load_library(path: str | os.PathLike | None = None):
    """Load libucfvb.so (built by __graft_entry__.build()). Raises if absent."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"B200 extension {p} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback for the stage pass)")
    lib = C.CDLL(str(p))
    _declare(lib)
    if path is None:
        _LIB = lib
    return lib


def _declare(lib):
    H = C.c_void_p
    sig = {
        "ucfvb_abi_version": (C.c_int32, []),
        "ucfvb_last_error": (C.c_char_p, [H]),
        "ucfvb_options_default": (None, [P(Options)]),
        "ucfvb_mesh_structured_tri": (C.c_int32, [C.c_int32, C.c_int32, C.c_double, C.c_double,
                                                  C.c_double, C.c_double, C.c_int32, C.c_double,
                                                  C.c_uint64, C.c_int32, C.c_double, C.c_int32,
                                                  P(H)]),
        "ucfvb_mesh_structured_quad": (C.c_int32, [C.c_int32, C.c_int32, C.c_double, C.c_double,
                                                   C.c_double, C.c_double, C.c_int32, C.c_double,
                                                   C.c_int32, P(H)]),
        "ucfvb_mesh_get_view": (C.c_int32, [H, P(MeshView)]),
        "ucfvb_mesh_free": (None, [H]),
        "ucfvb_build_stencils": (C.c_int32, [P(MeshView), C.c_int32, C.c_int32, C.c_int32, P(H)]),
        "ucfvb_stencils_get_view": (C.c_int32, [H, P(StencilView)]),
        "ucfvb_stencils_free": (None, [H]),
        "ucfvb_project_initial": (C.c_int32, [P(MeshView), C.c_int32, c_dp, C.c_int32, C.c_uint64,
                                              C.c_int32, C.c_double, C.c_int32, c_dp]),
        "ucfvb_create": (C.c_int32, [P(MeshView), P(StencilView), P(Options), P(BC), C.c_int32,
                                     C.c_int32, P(H)]),
        "ucfvb_destroy": (None, [H]),
        "ucfvb_set_state": (C.c_int32, [H, c_dp]),
        "ucfvb_get_state": (C.c_int32, [H, c_dp]),
        "ucfvb_max_stable_dt": (C.c_int32, [H, c_dp]),
        "ucfvb_advance": (C.c_int32, [H, C.c_double, C.c_double, C.c_int32]),
        "ucfvb_compute_residual": (C.c_int32, [H, c_dp, C.c_double, c_dp]),
        "ucfvb_run_steps": (C.c_int32, [H, C.c_int32, C.c_int32, C.c_double, C.c_double, c_dp, c_i64p]),
        "ucfvb_advance_host": (C.c_int32, [H, c_dp, c_dp, C.c_int32, C.c_int32, C.c_double, c_dp]),
        "ucfvb_advance_host_batch": (C.c_int32, [H, C.c_int32, P(c_dp), P(c_dp), C.c_int32, C.c_int32,
                                                 C.c_double, c_dp]),
        "ucfvb_run_steps_log": (C.c_int32, [H, C.c_int32, C.c_int32, C.c_double, C.c_double, c_dp, c_i64p,
                                            c_dp]),
        "ucfvb_run_until": (C.c_int32, [H, C.c_int32, C.c_int32, C.c_double, C.c_double, c_dp, c_i32p, c_i64p,
                                        c_dp]),
        "ucfvb_write_field_snapshot": (C.c_int32, [P(MeshView), c_dp, P(C.c_uint8), C.c_double, C.c_char_p]),
        "ucfvb_write_census_csv": (C.c_int32, [P(CensusRow), C.c_int32, C.c_int64, C.c_char_p]),
        "ucfvb_write_timing_csv": (C.c_int32, [P(TimingRow), C.c_int32, C.c_char_p]),
        "ucfvb_get_step_labels": (C.c_int32, [H, P(C.c_uint8)]),
        "ucfvb_get_labels": (C.c_int32, [H, P(C.c_uint8)]),
        "ucfvb_get_census": (C.c_int32, [H, c_i64p]),
        "ucfvb_get_nad_ties": (C.c_int32, [H, c_i64p]),
        "ucfvb_set_list_policy": (C.c_int32, [H, C.c_int32]),
        "ucfvb_get_list_stats": (C.c_int32, [H, c_i64p]),
        "ucfvb_get_face_values": (C.c_int32, [H, c_dp, c_dp]),
        "ucfvb_get_dofs": (C.c_int32, [H, c_dp]),
        "ucfvb_set_phase_timing": (C.c_int32, [H, C.c_int32]),
        "ucfvb_get_phase_times": (C.c_int32, [H, c_dp]),
        "ucfvb_n_cells": (C.c_int32, [H]),
        "ucfvb_n_faces": (C.c_int32, [H]),
        "ucfvb_n_qp": (C.c_int32, [H]),
        "ucfvb_state_device_ptr": (C.c_int32, [H, P(c_dp)]),
        "ucfvb_stream": (C.c_int32, [H, P(C.c_void_p)]),
        "ucfvb_launch_count": (C.c_int64, [H]),
        "ucfvb_partition_rcb": (C.c_int32, [P(MeshView), C.c_int32, c_i32p]),
        "ucfvb_subdomain_build": (C.c_int32, [P(MeshView), P(StencilView), c_i32p, C.c_int32, C.c_int32, P(H)]),
        "ucfvb_subdomain_views": (C.c_int32, [H, P(MeshView), P(StencilView)]),
        "ucfvb_subdomain_info": (C.c_int32, [H, c_i32p, c_i32p, c_i32p]),
        "ucfvb_subdomain_global_ids": (C.c_int32, [H, c_i32p]),
        "ucfvb_subdomain_peer": (C.c_int32, [H, C.c_int32, c_i32p, c_i32p, c_i32p, c_i32p]),
        "ucfvb_subdomain_send_list": (C.c_int32, [H, C.c_int32, c_i32p]),
        "ucfvb_subdomain_free": (None, [H]),
        "ucfvb_create_sub": (C.c_int32, [H, P(Options), P(BC), C.c_int32, C.c_int32, P(H)]),
        "ucfvb_nccl_unique_id": (C.c_int32, [P(C.c_uint8)]),
        "ucfvb_attach_nccl": (C.c_int32, [H, P(C.c_uint8), C.c_int32, C.c_int32]),
        "ucfvb_subdomain_interior": (C.c_int32, [H, c_i32p]),
        "ucfvb_group_create": (C.c_int32, [P(H), C.c_int32, P(H)]),
        "ucfvb_group_run_steps": (C.c_int32, [H, C.c_int32, C.c_int32, C.c_double, c_dp]),
        "ucfvb_group_launch_count": (C.c_int64, [H]),
        "ucfvb_group_free": (None, [H]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args


# every exported symbol of include/ucfvb.h, for the ABI test
ABI_SYMBOLS = [
    "ucfvb_abi_version", "ucfvb_last_error", "ucfvb_options_default",
    "ucfvb_mesh_structured_tri", "ucfvb_mesh_structured_quad", "ucfvb_mesh_get_view",
    "ucfvb_mesh_free", "ucfvb_build_stencils", "ucfvb_stencils_get_view", "ucfvb_stencils_free",
    "ucfvb_project_initial", "ucfvb_create", "ucfvb_destroy", "ucfvb_set_state",
    "ucfvb_get_state", "ucfvb_max_stable_dt", "ucfvb_advance", "ucfvb_compute_residual",
    "ucfvb_run_steps", "ucfvb_run_steps_log", "ucfvb_run_until", "ucfvb_advance_host", "ucfvb_advance_host_batch", "ucfvb_write_field_snapshot", "ucfvb_write_census_csv",
    "ucfvb_write_timing_csv", "ucfvb_get_step_labels", "ucfvb_get_labels", "ucfvb_get_census",
    "ucfvb_get_nad_ties", "ucfvb_set_list_policy", "ucfvb_get_list_stats", "ucfvb_get_face_values", "ucfvb_get_dofs", "ucfvb_set_phase_timing",
    "ucfvb_get_phase_times", "ucfvb_n_cells", "ucfvb_n_faces", "ucfvb_n_qp",
    "ucfvb_state_device_ptr", "ucfvb_stream", "ucfvb_launch_count",
    "ucfvb_partition_rcb", "ucfvb_subdomain_build", "ucfvb_subdomain_views", "ucfvb_subdomain_info",
    "ucfvb_subdomain_global_ids", "ucfvb_subdomain_peer", "ucfvb_subdomain_send_list", "ucfvb_subdomain_free",
    "ucfvb_create_sub", "ucfvb_nccl_unique_id", "ucfvb_attach_nccl", "ucfvb_subdomain_interior",
    "ucfvb_group_create", "ucfvb_group_run_steps", "ucfvb_group_launch_count", "ucfvb_group_free",
]


class UcfvbError(RuntimeError):
    """Base error of the C ABI (status code in .code)."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class NonPhysicalError(UcfvbError):
    """The reference's NonPhysicalError (euler.hpp:18-20)."""


class InvalidArgument(UcfvbError, ValueError):
    """std::invalid_argument / MeshError of the reference."""


class CudaError(UcfvbError):
    pass


class Unsupported(UcfvbError):
    pass


def error_for(code, msg) -> UcfvbError:
    cls = {NONPHYSICAL: NonPhysicalError, INVALID: InvalidArgument, CUDA_ERR: CudaError,
           UNSUPPORTED: Unsupported}.get(code, UcfvbError)
    return cls(code, msg)
