cd "$GRAFT_REPO_ROOT"
for cs in 1 2 3; do for ts in 1 2 3; do
  UCFVB_TMA_STAGES_CENTRAL=$cs UCFVB_TMA_STAGES_TROUBLED=$ts timeout 120 python scripts/time_steps.py --tag "central=$cs troubled=$ts" 2>&1 | tail -1
done; done
