"""The driver's bench contract for the reference arm (runs on CPU): one JSON
line with the documented keys, the BASELINE metric and the impl tag; the 3D
configurations' reference arm (the 3D oracle restatement) likewise."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True, env=env,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_json_line():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    d = _run(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "3"], {"UCFVB_REF_BUDGET_S": "1"})
    import bench
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    # the same static config dict the B200 arm prints (the driver compares them)
    assert d["config"] == bench.workload_config("1")
    for k in ("value", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "dtype", "data",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["warmup"] == 3  # untimed warm-up steps actually run (timing rule: W >= 3)


def test_reference_arm_3d_json_line():
    d = _run(["--impl", "reference", "--config", "5", "--steps", "1", "--warmup", "3"], {"UCFVB_CPU_S": "0.5"})
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["warmup"] == 3
    import bench
    assert d["config"] == bench.workload_config3("5")


def test_default_config_is_the_largest_2d_mesh():
    import bench
    assert bench.workload_config("3")["cells"] == 8_388_608
    c, sample = bench.cpu_sample_case("3")
    assert 2 * c["nx"] * c["ny"] == 524_288 and "tile of config 3" in sample


def test_traffic_is_keyed_by_config(tmp_path, monkeypatch):
    import bench
    (tmp_path / "profiles").mkdir()
    (tmp_path / "profiles" / "traffic.json").write_text(json.dumps({"config3": {"cells": 8388608, "cwenoz+muscl": 5.0}}))
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    assert bench.traffic_for("3", 8388608, "cwenoz+muscl") == 5.0
    assert bench.traffic_for("3", 1000, "cwenoz+muscl") is None
    assert bench.traffic_for("2", 262144, "cwenoz+muscl") is None
