"""Known-answer tests of the hot-path point functions (SPEC.md worked
examples) on the oracle restatement and, when built, the compiled reference."""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import port as P
from oracle import ref as R
from paper_2510_25906_b200 import _abi as A

IMPLS = ["port"] + (["ref"] if R.available() else [])


def fns(impl):
    L = P.lib() if impl == "port" else R.lib()
    pre = "port_" if impl == "port" else "ref_"

    def margins(m, du):
        dm, dw = C.c_double(), C.c_double()
        getattr(L, pre + "compute_margins")(C.byref(m), du, C.byref(dm), C.byref(dw))
        return dm.value, dw.value

    def bj(u0, lo, hi, q):
        a = np.ascontiguousarray(q, dtype=np.float64)
        return getattr(L, pre + "limiter_bj")(u0, lo, hi, a.ctypes.data_as(A.c_dp), len(a))

    def venkat(u0, lo, hi, q, eps2):
        a = np.ascontiguousarray(q, dtype=np.float64)
        return getattr(L, pre + "limiter_venkat")(u0, lo, hi, a.ctypes.data_as(A.c_dp), len(a), eps2)

    def flux(ul, ur, n, kind=0, g=1.4):
        ul = np.ascontiguousarray(ul, dtype=np.float64)
        ur = np.ascontiguousarray(ur, dtype=np.float64)
        out = np.zeros(4)
        rc = getattr(L, pre + "flux")(ul.ctypes.data_as(A.c_dp), ur.ctypes.data_as(A.c_dp), n[0], n[1], g, kind,
                                      out.ctypes.data_as(A.c_dp))
        return rc, out

    return dict(margins=margins, classify=getattr(L, pre + "classify_violation"),
                deact=getattr(L, pre + "deactivate_smooth"), bj=bj, venkat=venkat, flux=flux)


def cons(rho, u, v, p, g=1.4):
    return [rho, rho * u, rho * v, p / (g - 1) + 0.5 * rho * (u * u + v * v)]


@pytest.mark.parametrize("impl", IMPLS)
def test_margins(impl):
    f = fns(impl)
    assert f["margins"](A.Margins(1e-4, 0.5, 0, 0, 5, 2), 1.0) == (0.5, 0.0)
    assert f["margins"](A.Margins(0, 0, 0, -0.5, 5, 2), 1.0) == (0.0, -0.5)
    assert f["margins"](A.Margins(1e-4, 0.5, 0, 0, 5, 2), 0.0) == (1e-4, 0.0)


@pytest.mark.parametrize("impl", IMPLS)
def test_band_rule(impl):  # bounds (0,1), delta_m=0.5, delta_w=0
    f = fns(impl)
    assert f["classify"](1.2 - 1.0, 0.5, 0.0) == A.SCHEME_CWENOZ
    assert f["classify"](1.7 - 1.0, 0.5, 0.0) == A.SCHEME_MUSCL
    assert f["classify"](-0.1, 0.5, 0.0) == A.SCHEME_LINEAR


@pytest.mark.parametrize("impl", IMPLS)
def test_deactivation(impl):
    f = fns(impl)
    assert f["deact"](0.0, 0.01, 5.0, 2.0) == 1
    assert f["deact"](0.001, 0.01, 5.0, 2.0) == 1
    assert f["deact"](0.1, 0.01, 5.0, 2.0) == 0
    assert f["deact"](0.0, 0.01, 0.0, 2.0) == 0  # kappa = 0 disables deactivation


@pytest.mark.parametrize("impl", IMPLS)
def test_limiters(impl):  # SPEC.md:296 (theta = 0.5) and uniform field
    f = fns(impl)
    assert f["bj"](1.0, 0.5, 1.5, [1.2, 2.0, 0.9]) == 0.5
    assert f["bj"](1.0, 1.0, 1.0, [1.0, 1.0]) == 1.0
    assert f["venkat"](1.0, 1.0, 1.0, [1.0, 1.0], 1e-3) == 1.0
    th = [f["venkat"](1.0, 0.5, 1.5, [2.0, 0.3], e) for e in (1e-6, 1e-3, 1e-1)]
    assert th == sorted(th)  # nondecreasing in eps2 (kappa_v)
    assert th[0] <= f["bj"](1.0, 0.5, 1.5, [2.0, 0.3]) + 1e-6


@pytest.mark.parametrize("impl", IMPLS)
@pytest.mark.parametrize("kind", [A.HLLC, A.HLL])
def test_flux_consistency_and_upwinding(impl, kind):
    f = fns(impl)
    rc, F = f["flux"](cons(1, 0, 0, 1), cons(1, 0, 0, 1), (1.0, 0.0), kind)
    assert rc == 0 and np.allclose(F, [0, 1, 0, 0], atol=1e-15)
    # supersonic right-moving: flux = physical flux of the left state
    UL, UR = cons(1.0, 3.0, 0.5, 1.0), cons(0.5, 2.5, 0.0, 0.4)
    rc, F = f["flux"](UL, UR, (1.0, 0.0), kind)
    rho, u, v, p = 1.0, 3.0, 0.5, 1.0
    E = UL[3]
    assert np.allclose(F, [rho * u, rho * u * u + p, rho * u * v, (E + p) * u], rtol=1e-14)
    # rotational equivariance
    phi = 0.7
    rot = np.array([[math.cos(phi), -math.sin(phi)], [math.sin(phi), math.cos(phi)]])
    n = rot @ np.array([1.0, 0.0])
    UL2, UR2 = np.array(UL), np.array(UR)
    UL2[1:3], UR2[1:3] = rot @ UL2[1:3], rot @ UR2[1:3]
    rc, F2 = f["flux"](UL2, UR2, n, kind)
    assert np.allclose(F2[[0, 3]], F[[0, 3]], rtol=1e-12) and np.allclose(F2[1:3], rot @ F[1:3], rtol=1e-12)
    # non-physical input
    rc, _ = f["flux"](cons(1, 0, 0, 1), [1.0, 0.0, 0.0, -1.0], (1.0, 0.0), kind)
    assert rc == A.NONPHYSICAL


def test_cwenoz_lambda():  # lambda1' = 1e4 -> lambda1 = 0.9999, lambda_s = 1e-4/3
    # constant field: SI = 0, tau = 0, weights = linear weights, blended dofs = 0
    K = 5
    oi = np.eye(K).ravel()
    out = np.zeros(K)
    central = np.zeros(K)
    dirs = np.zeros((3, 2))
    rc = P.lib().port_cwenoz_blend(oi.ctypes.data_as(A.c_dp), K, central.ctypes.data_as(A.c_dp),
                                   dirs.ctypes.data_as(A.c_dp), 3, 1e4, 1e-3, 4.0, out.ctypes.data_as(A.c_dp))
    assert rc == 0 and np.all(out == 0.0)
    # smooth field: directional dofs equal the central linear part -> blend returns the central dofs
    central = np.array([0.3, -0.2, 1e-3, 2e-3, -1e-3])
    dirs = np.tile(central[:2], (3, 1))
    oi = np.diag([1.0, 1.0, 0.1, 0.1, 0.1]).ravel()
    rc = P.lib().port_cwenoz_blend(oi.ctypes.data_as(A.c_dp), K, central.ctypes.data_as(A.c_dp),
                                   dirs.ctypes.data_as(A.c_dp), 3, 1e4, 1e-3, 4.0, out.ctypes.data_as(A.c_dp))
    assert np.allclose(out, central, rtol=1e-6)
    rc = P.lib().port_cwenoz_blend(oi.ctypes.data_as(A.c_dp), K, central.ctypes.data_as(A.c_dp),
                                   dirs.ctypes.data_as(A.c_dp), 3, 1.0, 1e-3, 4.0, out.ctypes.data_as(A.c_dp))
    assert rc == A.INVALID  # lambda1' <= 1 throws invalid_argument (reconstruct.cpp:102-103)


def test_dt_example():  # still gas on h_c = 0.1, CFL 1 -> 0.1/sqrt(1.4)
    from paper_2510_25906_b200.mesh import Mesh, Stencils
    m = Mesh.structured_quad(10, 10, (0.0, 0.0, 1.0, 1.0), periodic="both", n_qp=2)
    st = Stencils(m, 2)
    p = P.PortSolver(m.view, st.view, A.options_from_dict(order=2, cfl=1.0), keep=(m, st))
    p.state = np.tile(cons(1, 0, 0, 1), (m.n_cells, 1))
    assert abs(p.max_stable_dt() - 0.1 / math.sqrt(1.4)) < 1e-15
