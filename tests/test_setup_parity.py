"""The product's native host setup (csrc/setup_*.cpp: mesh generation, periodic
pairing, operator precompute, IC projection) reproduces the reference's setup
bit-for-bit: against the golden fixtures (the reference's own mesh and
StencilSet bytes) and, where oracle/_ref exists, against the live reference."""
import numpy as np
import pytest

from oracle import ref as R
from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.mesh import Mesh, Stencils
from tests.golden.make_golden import CASES
from tests.golden_io import Fixture

AXIS = {0: "none", 1: "x", 2: "y", 3: "both"}


def product_mesh(c):
    kind, nx, ny, rect, jit, per = c["mesh"]
    nq = (c["order"] + 2) // 2
    if kind == "tri":
        return Mesh.structured_tri(nx, ny, rect, jitter=jit, seed=11, periodic=AXIS[per], n_qp=nq)
    return Mesh.structured_quad(nx, ny, rect, periodic=AXIS[per], n_qp=nq)


def assert_dicts_equal(a, b):
    assert set(a) == set(b)
    for k in a:
        if a[k].dtype.kind == "U":
            assert list(a[k]) == list(b[k]), k
        else:
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)


@pytest.mark.parametrize("name", sorted(CASES))
def test_setup_matches_golden(name):
    c = CASES[name]
    fx = Fixture(name)
    m = product_mesh(c)
    assert_dicts_equal(m.numpy(), fx.mesh_np)
    st = Stencils(m, c["order"], int(fx.options.si_exponent))
    assert_dicts_equal(st.numpy(), fx.st_np)
    ic, prm = c["ic"]
    np.testing.assert_array_equal(m.project_initial(ic, prm, seed=5, degree=max(2 * c["order"], 2)), fx.u0)


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("nx,ny,rect,jit,per,order,si", [
    (40, 40, (0, 0, 1, 1), 0.1, 3, 2, 0),
    (64, 16, (-5, 0, 5, 1), 0.1, 2, 2, 0),
    (32, 32, (0, 0, 1, 1), 0.0, 3, 3, 1),
    (24, 24, (0, 0, 10, 10), 0.1, 1, 4, 0),
])
def test_setup_matches_live_reference(nx, ny, rect, jit, per, order, si):
    nq = (order + 2) // 2
    rm = R.RefMesh.structured_tri(nx, ny, rect, jitter=jit, seed=4, periodic=per, n_qp=nq)
    pm = Mesh.structured_tri(nx, ny, rect, jitter=jit, seed=4, periodic=AXIS[per], n_qp=nq)
    assert_dicts_equal(pm.numpy(), rm.numpy())
    bcs = [] if per == 3 else [A.BC(p.encode(), A.BC_OUTFLOW) for p in ("left", "right", "bottom", "top")]
    rs = R.RefSolver(rm, A.options_from_dict(order=order, si_exponent=si), bcs)
    assert_dicts_equal(Stencils(pm, order, si).numpy(), rs.stencils_numpy())


def test_generate_tri_without_jitter_matches_reference_generator():
    if not R.available():
        pytest.skip("oracle/_ref not built")
    a = R.RefMesh.generate_tri(10, 7, (0.0, 0.0, 2.0, 1.0), diagonal=1, periodic=3, n_qp=2)
    b = Mesh.structured_tri(10, 7, (0.0, 0.0, 2.0, 1.0), diagonal="alternating", periodic="both", n_qp=2)
    assert_dicts_equal(b.numpy(), a.numpy())


def test_setup_errors():
    with pytest.raises(A.InvalidArgument):
        Mesh.structured_tri(0, 4)
    with pytest.raises(A.InvalidArgument, match="zero-size"):
        Mesh.structured_tri(4, 4, (0.0, 0.0, 0.0, 1.0))
    m = Mesh.structured_tri(4, 4, n_qp=2)
    with pytest.raises(A.InvalidArgument, match="quadrature points"):
        Stencils(m, 3 + 1)  # order 4 needs 3 points per face
    with pytest.raises(A.InvalidArgument, match="mesh too small"):
        Stencils(Mesh.structured_tri(2, 2, periodic="none", n_qp=3), 5)
