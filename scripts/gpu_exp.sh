cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for l2 in 0 1; do
  UCFVB_L2_PERSIST=$l2 timeout 600 python scripts/time_steps.py --config 2 --steps 200 --tag "l2persist=$l2" 2>&1 | tail -1
  UCFVB_L2_PERSIST=$l2 timeout 600 python scripts/time_steps.py --config 1 --steps 200 --tag "l2persist=$l2" 2>&1 | tail -1
done
