# tests of the latest changes (3D candidate stores, raw-MUSCL dofs), L2-persistence A/B on config 3, config 5 timing
cd "$GRAFT_REPO_ROOT"
timeout 1200 python -m pytest tests/test_gpu_3d.py tests/test_gpu_parity.py tests/test_gpu_golden.py -q -x 2>&1 | tail -3
export UCFVB_TROUBLED=lists
for p in 1 0; do
  UCFVB_L2_PERSIST=$p timeout 900 python scripts/time_steps.py --config 3 --steps 10 --tag "l2persist=$p" 2>&1 | tail -1 | cut -c1-170
done
UCFVB_L2_PERSIST=0 timeout 900 python scripts/time_steps.py --config 2 --steps 100 --tag "l2persist=0" 2>&1 | tail -1 | cut -c1-170
timeout 900 python scripts/prof3d.py --config 5 2>&1 | tail -2
