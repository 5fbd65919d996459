# round 2: per-cell troubled kernel -- GPU tests, then chunk vs per-cell timing on configs 3, 2, 1
cd "$GRAFT_REPO_ROOT"
timeout 2400 python -m pytest tests -m gpu -q -x -s 2>&1 | grep -E "passed|failed|Error|error|config[23]:|assert" | tail -30 > gpurun_out/r02_cells_pytest.log
cat gpurun_out/r02_cells_pytest.log
for mode in chunks lists; do
  UCFVB_TROUBLED=$mode timeout 900 python scripts/time_steps.py --config 3 --steps 20 --tag $mode 2>&1 | tail -1
  UCFVB_TROUBLED=$mode timeout 600 python scripts/time_steps.py --config 2 --steps 100 --tag $mode 2>&1 | tail -1
  UCFVB_TROUBLED=$mode timeout 600 python scripts/time_steps.py --config 1 --steps 200 --tag $mode 2>&1 | tail -1
done | tee gpurun_out/r02_cells_time.log
