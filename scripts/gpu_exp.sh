cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in 2 1 3; do timeout 600 python scripts/time_steps.py --config $cfg --steps 100 --tag "nad-minmax" 2>&1 | tail -1; done
