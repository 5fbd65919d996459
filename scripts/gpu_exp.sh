cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_positivity.py -q -x 2>&1 | tail -2
for cfg in 3 2; do timeout 600 python scripts/time_steps.py --config $cfg --steps 50 --tag "oi-global-p3" 2>&1 | tail -1; done
