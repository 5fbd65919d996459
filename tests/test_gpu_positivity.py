"""The fallback positivity check (solver.cpp:229-264, is_physical euler.hpp:34-36)
in isolation, against the unmodified reference.

The NAD margins are set so that the relaxed DMP can never demote a cell
(delta_m huge) -- every FirstOrder label then comes from a face point with
rho <= 0 or p <= 0 -- on a state with near-vacuum cells next to fast flow, so
that many candidate face points are non-physical. Two regimes:
* all cells Linear (delta_w huge too): the central kernel's butterfly-
  transposed check (group_nonphysical) decides every demotion;
* delta_w = 0 and no deactivation: every cell with an overshoot is CWENOZ,
  the troubled kernel's shared-memory-spread check decides.
Labels must be identical and at least a few cells must be demoted."""
import numpy as np
import pytest

from oracle import ref as R
from paper_2510_25906_b200 import _abi as A
from paper_2510_25906_b200.mesh import Mesh, Stencils
from paper_2510_25906_b200.solver import Solver
from tests.cases import scaled_err

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not shipped")]


def vacuum_state(n, seed):
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.5, 1.5, n)
    u = rng.normal(0.0, 2.0, n)
    v = rng.normal(0.0, 2.0, n)
    p = rng.uniform(0.5, 1.5, n)
    low = rng.random(n) < 0.15
    rho[low] = 1e-3
    p[low] = 1e-6
    E = p / 0.4 + 0.5 * rho * (u * u + v * v)
    return np.stack([rho, rho * u, rho * v, E], axis=1)


@pytest.mark.parametrize("regime", ["linear", "cwenoz"])
@pytest.mark.parametrize("order", [2, 3])
def test_positivity_demotions_match_reference(regime, order):
    nx = 24
    nq = (order + 2) // 2
    big = 1e300
    if regime == "linear":
        margins = (big, 1.0, big, 0.5, 5.0, 2.0)  # delta_w = delta_m = 1e300: never CWENOZ/MUSCL
    else:
        margins = (big, 0.0, 0.0, 0.0, 0.0, 2.0)  # delta_w = 0, kappa = 0: no deactivation
    o = A.options_from_dict(order=order, margins=margins, lambda1p=1e3, weno_b=1.0)
    mesh = Mesh.structured_tri(nx, nx, (0.0, 0.0, 1.0, 1.0), jitter=0.1, seed=5, periodic="both", n_qp=nq)
    g = Solver(mesh, o, stencils=Stencils(mesh, order))
    rm = R.RefMesh.structured_tri(nx, nx, (0.0, 0.0, 1.0, 1.0), jitter=0.1, seed=5, periodic=3, n_qp=nq)
    rs = R.RefSolver(rm, o, [])
    u = vacuum_state(mesh.n_cells, 11 + order)
    try:
        r_ref = rs.compute_residual(u, 0.0, 1)
        ref_err = None
    except R.RefError as e:  # NonPhysicalError in the fluxes: both must agree on that too
        ref_err = e
    if ref_err is None:
        r_gpu = g.compute_residual(u, 0.0)
        assert scaled_err(r_gpu, r_ref) <= 1e-10
    else:
        with pytest.raises(A.UcfvbError):
            g.compute_residual(u, 0.0)
    lab_g, lab_r = g.labels(), rs.labels()
    np.testing.assert_array_equal(lab_g, lab_r)
    counts = np.bincount(lab_r, minlength=4)
    assert counts[3] >= 5, counts
    if regime == "linear":
        assert counts[1] == counts[2] == 0
    else:
        assert counts[1] > 0 and counts[2] == 0
