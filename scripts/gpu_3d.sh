set -x
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_3d.py -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu3d.log
cat gpurun_out/pytest_gpu3d.log
