"""3D host setup and 3D oracle (BASELINE configs 4-5), CPU.

The reference is 2D only, so there is no reference output to pin the 3D
restatement against ("parity unpinned"). These tests pin it
by properties instead: closed cells, exact volumes, polynomial exactness of
the least-squares reconstruction, discrete conservation, flux consistency
and symmetry, and the invariance of a uniform state.
"""
import numpy as np
import pytest

from oracle.port3 import Port3Solver, flux
from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.solver3d import (HEX, IC_BLAST, IC_RANDOM_PHASE, IC_TGV, IC_UNIFORM, TET, Mesh3,
                                            Stencils3)

L = 2 * np.pi
CASES = [(HEX, 1, 0.1), (HEX, 2, 0.05), (HEX, 3, 0.0), (TET, 1, 0.05), (TET, 2, 0.0), (TET, 3, 0.0)]


@pytest.mark.parametrize("kind,order,jitter", CASES)
def test_mesh_geometry(kind, order, jitter):
    m = Mesh3(5, kind=kind, jitter=jitter, order=order, seed=11)
    n, nf, nq = m.n_cells, m.nf, m.nq
    assert n == 125 * (1 if kind == HEX else 6)
    assert m.n_faces * 2 == n * nf
    assert abs(m.volume.sum() / L**3 - 1) < 1e-13
    assert np.all(m.volume > 0)
    np.testing.assert_allclose(m.h, np.cbrt(m.volume), rtol=1e-15)
    fn = m.arr("face_normal", (m.n_faces, nq, 3))
    fw = m.arr("face_wa", (m.n_faces, nq))
    np.testing.assert_allclose(np.linalg.norm(fn, axis=-1), 1.0, rtol=1e-14)
    cf, cs = m.arr("cell_faces", (n, nf)), m.arr("cell_side", (n, nf))
    an = (fn * fw[..., None]).sum(1)
    closure = (an[cf] * np.where(cs == 0, 1.0, -1.0)[..., None]).sum(1)
    assert np.abs(closure).max() < 1e-13  # every cell is closed (divergence theorem)
    # neighbour relation is symmetric and consistent with the faces
    nb = m.arr("cell_nbr", (n, nf))
    fl, fr = m.arr("face_left", (m.n_faces,)), m.arr("face_right", (m.n_faces,))
    own = np.where(cs == 0, fl[cf], fr[cf])
    oth = np.where(cs == 0, fr[cf], fl[cf])
    assert np.array_equal(own, np.repeat(np.arange(n)[:, None], nf, 1))
    assert np.array_equal(oth, nb)
    # outward normals: face points lie away from the left cell's centroid
    c = m.centroid
    fq = m.arr("face_qp", (m.n_faces, nq, 3))
    assert np.all(((fq - c[fl][:, None, :]) * fn).sum(-1) > 0)


def _linear_field(m, a, b):
    """cell averages of a linear field = its value at the centroid"""
    return a[None, :] + m.centroid @ b.T


@pytest.mark.parametrize("kind,order,jitter,classes", [(HEX, 1, 0.1, False), (HEX, 2, 0.05, False),
                                                       (TET, 2, 0.05, False), (TET, 3, 0.0, True),
                                                       (HEX, 2, 0.0, True)])
def test_linear_exactness(kind, order, jitter, classes):
    """The central LSQ reconstruction reproduces a linear field exactly at every
    face point of cells whose stencil does not wrap around the periodic box."""
    n_c = 8
    m = Mesh3(n_c, kind=kind, jitter=jitter, order=order, seed=5)
    st = Stencils3(m, order, lattice_classes=classes)
    a = np.array([2.0, 0.3, -0.2, 0.1, 50.0])
    b = np.array([[0.05, 0.02, -0.03], [0.01, 0.0, 0.02], [0.0, -0.01, 0.01], [0.02, 0.01, 0.0], [0.3, -0.2, 0.1]])
    u = _linear_field(m, a, b)
    o = A.options_from_dict(order=order, mode="linear")
    P = Port3Solver(m, st, o)
    P.compute_residual(u)
    fv = P.face_values()
    nq, nf = m.nq, m.nf
    cube, _ = m.cube_and_type()
    ijk = np.stack([cube % n_c, (cube // n_c) % n_c, cube // (n_c * n_c)], 1)
    inner = np.all((ijk >= 3) & (ijk <= 4), axis=1)
    fq = m.arr("face_qp", (m.n_faces, nq, 3))
    fl, fr = m.arr("face_left", (m.n_faces,)), m.arr("face_right", (m.n_faces,))
    ok = inner[fl] & inner[fr]
    assert ok.sum() > 10
    exact = a[None, None, :] + fq[ok] @ b.T
    np.testing.assert_allclose(fv[ok, :, 0, :], exact, rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(fv[ok, :, 1, :], exact, rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("kind,order,jitter,mode,ic", [
    (HEX, 2, 0.05, "hybrid", IC_TGV), (TET, 2, 0.0, "hybrid", IC_BLAST), (HEX, 1, 0.1, "muscl", IC_BLAST),
    (TET, 3, 0.0, "cwenoz", IC_RANDOM_PHASE), (HEX, 2, 0.0, "first", IC_BLAST)])
def test_conservation(kind, order, jitter, mode, ic):
    m = Mesh3(5, kind=kind, jitter=jitter, order=order, seed=2)
    st = Stencils3(m, order)
    params = {IC_TGV: [0.1], IC_BLAST: [3.0, 3.2, 3.1, 1.5, 1.0, 5.0, 0.5, 1.0], IC_RANDOM_PHASE: [0.3, 2.0, 4]}[ic]
    u0 = m.project_initial(ic, params, seed=4)
    P = Port3Solver(m, st, A.options_from_dict(order=order, mode=mode, cfl=0.5))
    P.state = u0.copy()
    tot0 = (u0 * m.volume[:, None]).sum(0)
    for _ in range(3):
        P.advance(P.max_stable_dt(), rk=A.RK3)
    tot = (P.state * m.volume[:, None]).sum(0)
    scale = np.abs(u0).max() * m.volume.sum()
    assert np.all(np.abs(tot - tot0) <= 1e-13 * scale)
    assert np.all(np.isfinite(P.state))


def test_uniform_state_is_steady():
    m = Mesh3(4, kind=TET, jitter=0.05, order=2, seed=9)
    st = Stencils3(m, 2)
    u0 = m.project_initial(IC_UNIFORM, [1.2, 0.3, -0.4, 0.5, 2.0])
    P = Port3Solver(m, st, A.options_from_dict(order=2, mode="hybrid"))
    r = P.compute_residual(u0)
    assert np.abs(r).max() < 1e-12 * np.abs(u0).max()
    assert np.all(P.labels() == A.SCHEME_LINEAR)


def test_flux_consistency_and_symmetry():
    rng = np.random.default_rng(1)
    g = 1.4
    for kind in (A.HLLC, A.HLL):
        for _ in range(50):
            def state():
                rho, p = rng.uniform(0.2, 2.0), rng.uniform(0.2, 3.0)
                vel = rng.uniform(-2, 2, 3)
                return np.array([rho, *(rho * vel), p / (g - 1) + 0.5 * rho * vel @ vel])
            n = rng.normal(size=3)
            n /= np.linalg.norm(n)
            ul, ur = state(), state()
            # consistency F(U, U, n) = F_phys(U) . n
            f = flux(ul, ul, n, g, kind)
            rho, vel = ul[0], ul[1:4] / ul[0]
            p = (g - 1) * (ul[4] - 0.5 * rho * vel @ vel)
            un = vel @ n
            phys = np.array([rho * un, *(rho * vel * un + p * n), (ul[4] + p) * un])
            np.testing.assert_allclose(f, phys, rtol=1e-12, atol=1e-12)
            # conservation across the face: F(L, R, n) = -F(R, L, -n)
            np.testing.assert_allclose(flux(ul, ur, n, g, kind), -flux(ur, ul, -n, g, kind), rtol=1e-11,
                                       atol=1e-11)
    # non-physical states report failure
    assert flux(np.array([-1.0, 0, 0, 0, 1.0]), np.array([1.0, 0, 0, 0, 2.5]), np.array([1.0, 0, 0]), g) is None


def test_random_phase_ic():
    m = Mesh3(8, kind=TET, order=3)
    u = m.project_initial(IC_RANDOM_PHASE, [0.6, 4.0, 6], seed=5)
    assert np.allclose(u[:, 0], 1.0)
    vel = u[:, 1:4] / u[:, :1]
    rms = np.sqrt((m.volume * (vel**2).sum(1)).sum() / m.volume.sum())
    assert abs(rms - 0.6) < 1e-12
    # solenoidal modes: the mean divergence through the faces is small against |u|/h
    u2 = m.project_initial(IC_RANDOM_PHASE, [0.6, 4.0, 6], seed=6)
    assert not np.allclose(u, u2)


def test_lattice_classes_need_unjittered_mesh():
    m = Mesh3(4, kind=TET, jitter=0.05, order=2)
    with pytest.raises(A.InvalidArgument):
        Stencils3(m, 2, lattice_classes=True)
    m0 = Mesh3(4, kind=TET, jitter=0.0, order=2)
    s = Stencils3(m0, 2, lattice_classes=True)
    assert s.n_ops == 6
    with pytest.raises(A.InvalidArgument):
        Mesh3(2, kind=HEX)


def test_blocked_cell_order():
    """4^3 = 64 cubes of tetrahedra: type-major numbering in blocks of 32 cubes
    (every 32-cell chunk one type); 5^3 keeps the cube-major numbering."""
    m = Mesh3(4, kind=TET, order=2)
    assert m.view.cell_order == 1
    cube, typ = m.cube_and_type()
    assert np.array_equal(np.sort(cube * 6 + typ), np.arange(m.n_cells))
    assert np.all(typ.reshape(-1, 32) == typ.reshape(-1, 32)[:, :1])
    st = Stencils3(m, 2, lattice_classes=True)
    assert np.array_equal(st.arr("op_index", (m.n_cells,)), typ)
    assert Mesh3(5, kind=TET, order=2).view.cell_order == 0


def test_solver3_argument_validation_without_gpu():
    """ucfvb3_create validates its arguments before touching the device (the
    reference's constructor / cwenoz_blend_scalar exceptions): lambda1' <= 1,
    bad margins, an unknown mode, and a stencil set of another mesh."""
    from paper_2510_25906_b200.solver3d import Solver3
    m = Mesh3(4, kind=HEX, order=2)
    st = Stencils3(m, 2)
    for kw in (dict(lambda1p=1.0), dict(margins=(-1.0, 0.5, 0.0, 0.0, 5.0, 2.0)), dict(mode=7),
               dict(margins=(1e-4, 0.5, 1e-3, 0.6, 5.0, 2.0))):
        o = A.options_from_dict(order=2, **kw)
        with pytest.raises(A.InvalidArgument):
            Solver3(m, o, st)
    other = Mesh3(5, kind=HEX, order=2)
    with pytest.raises(A.InvalidArgument):
        Solver3(other, A.options_from_dict(order=2), st)


def test_mesh3_and_stencils3_argument_errors():
    with pytest.raises(A.InvalidArgument):
        Mesh3(4, kind=7)
    with pytest.raises(A.InvalidArgument):
        Mesh3(4, kind=HEX, order=0)
    with pytest.raises(A.InvalidArgument):
        Mesh3(4, kind=HEX, jitter=0.3)
    m = Mesh3(4, kind=HEX, order=2)
    with pytest.raises(A.InvalidArgument):
        Stencils3(m, 1)  # the mesh face rule was built for order 2 (2x2 points; order 1 needs 1)
    with pytest.raises(A.InvalidArgument):
        m.project_initial(99, [1.0])


def test_3d_riemann_flux_reduces_to_the_pinned_2d_flux():
    """With w = 0 and an in-plane normal the 3D HLLC/HLL (Cartesian form) is
    the reference's 2D flux (euler.cpp:40-89, rotated frame) -- checked against
    the 2D port, which is pinned bit-exactly to the compiled reference."""
    import ctypes as C

    from oracle import port as P2
    rng = np.random.default_rng(3)
    g = 1.4
    dp = C.POINTER(C.c_double)
    for kind in (A.HLLC, A.HLL):
        for _ in range(200):
            def state2():
                rho, p = rng.uniform(0.2, 2.0), rng.uniform(0.2, 3.0)
                u, v = rng.uniform(-2, 2, 2)
                return np.array([rho, rho * u, rho * v, p / (g - 1) + 0.5 * rho * (u * u + v * v)])
            ul2, ur2 = state2(), state2()
            th = rng.uniform(0, 2 * np.pi)
            nx, ny = np.cos(th), np.sin(th)
            f2 = np.zeros(4)
            rc = P2.lib().port_flux(ul2.ctypes.data_as(dp), ur2.ctypes.data_as(dp), nx, ny, g, kind,
                                    f2.ctypes.data_as(dp))
            assert rc == 0
            up = lambda s: np.array([s[0], s[1], s[2], 0.0, s[3]])
            f3 = flux(up(ul2), up(ur2), np.array([nx, ny, 0.0]), g, kind)
            np.testing.assert_allclose(f3[[0, 1, 2, 4]], f2, rtol=1e-12, atol=1e-12 * np.abs(f2).max())
            assert abs(f3[3]) <= 1e-14 * np.abs(f2).max()
