"""The reference-side C++ binding (include/ucfvb_ucfv.hpp): ucfv::GpuSolver
used exactly like ucfv::Solver on the reference's own vortex case, against the
unmodified reference in the same process (oracle/_build/shim_demo)."""
import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
DEMO = Path(__file__).resolve().parents[1] / "oracle" / "_build" / "shim_demo"


@pytest.mark.skipif(not DEMO.exists(), reason="shim_demo not built (needs the reference sources at build time)")
@pytest.mark.parametrize("n,steps", [(16, 3), (32, 2)])
def test_gpu_solver_drop_in_matches_reference_solver(n, steps):
    r = subprocess.run([str(DEMO), str(n), str(steps)], capture_output=True, text=True, timeout=300)
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0 and line["ok"], line
    assert line["max_abs_diff"] == 0.0 and line["label_mismatch"] == 0
