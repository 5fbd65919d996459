"""Run outputs: the native writers in libucfvb.so produce
byte-identical files to the reference's own write_field_snapshot /
write_census_csv / write_timing_csv (run.cpp:160-213), called through
oracle/_ref on the same inputs. Host-only: no GPU needed."""
import numpy as np
import pytest

from oracle import ref as R
from paper_2510_25906_b200 import run as RUN
from paper_2510_25906_b200.solver import ViewHolder

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def _state(n, rng, extreme=False):
    u = np.empty((n, 4))
    u[:, 0] = rng.uniform(0.1, 3.0, n)
    u[:, 1:3] = rng.normal(0.0, 1.0, (n, 2))
    u[:, 3] = rng.uniform(2.0, 10.0, n)
    if extreme:  # formatting corner cases: tiny / huge / negative zero / non-physical
        u[0] = (1e-300, -0.0, 5e-324, 1e300)
        u[1] = (-1.0, 2.0, 3.0, -4.0)
        u[2] = (0.0, 1.0, 1.0, 1.0)  # divides by zero: inf / nan in pressure and velocity
        u[3] = (1.0 / 3.0, 2.0 / 3.0, np.pi, np.e)
    return u


@pytest.mark.parametrize("kind", ["tri", "quad", "tri_large"])
def test_field_snapshot_bytes(tmp_path, kind):
    rng = np.random.default_rng(7)
    if kind == "quad":
        m = R.RefMesh.generate_quad(7, 5, (0.0, 0.0, 1.0, 1.0))
    elif kind == "tri":
        m = R.RefMesh.structured_tri(9, 6, jitter=0.1, seed=3, periodic=2)
    else:  # > one 32,768-row formatting range
        m = R.RefMesh.structured_tri(160, 120, jitter=0.1, seed=3, periodic=3)
    n = m.n_cells
    u = _state(n, rng, extreme=True)
    lab = rng.integers(0, 4, n).astype(np.uint8)
    a, b = tmp_path / "ref.vtk", tmp_path / "ours.vtk"
    with np.errstate(all="ignore"):
        R.write_field_snapshot(m, u, lab, 1.4, a)
    RUN.write_field_snapshot(ViewHolder(m.view(), keep=m), u, lab, 1.4, b)
    assert a.read_bytes() == b.read_bytes()


def test_census_and_timing_csv_bytes(tmp_path):
    rng = np.random.default_rng(11)
    rows, trows, t = [], [], 0.0
    for s in range(1, 38):
        dt = float(rng.uniform(1e-4, 1e-2))
        t += dt
        counts = rng.integers(0, 10**6, 4)
        rows.append((s, t, dt, counts.tolist()))
        trows.append((s, float(rng.uniform(0, 100)), *rng.uniform(0, 1, 4).tolist()))
    for n_cells in (262_144, 8_388_608, 3):
        a, b = tmp_path / f"ref_{n_cells}.csv", tmp_path / f"ours_{n_cells}.csv"
        R.write_census_csv(rows, n_cells, a)
        RUN.write_census_csv(rows, n_cells, b)
        assert a.read_bytes() == b.read_bytes()
    a, b = tmp_path / "ref_t.csv", tmp_path / "ours_t.csv"
    R.write_timing_csv(trows, a)
    RUN.write_timing_csv(trows, b)
    assert a.read_bytes() == b.read_bytes()
    # empty runs: header only, like the reference
    R.write_census_csv([], 5, a)
    RUN.write_census_csv([], 5, b)
    assert a.read_bytes() == b.read_bytes()


def test_writer_errors(tmp_path):
    from paper_2510_25906_b200 import _abi as A
    with pytest.raises(A.UcfvbError):
        RUN.write_census_csv([], 5, tmp_path / "no_such_dir" / "x.csv")
