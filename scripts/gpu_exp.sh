cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_run.py -q -x 2>&1 | tail -30
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
