cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "class_list" 2>&1 | tail -3
for mode in chunks lists; do
  UCFVB_TROUBLED=$mode timeout 1500 python scripts/time_steps.py --config 3 --steps 20 --tag $mode 2>&1 | tail -1
  UCFVB_TROUBLED=$mode timeout 600 python scripts/time_steps.py --config 1 --steps 200 --tag $mode 2>&1 | tail -1
  UCFVB_TROUBLED=$mode timeout 600 python scripts/time_steps.py --config 2 --steps 100 --tag $mode 2>&1 | tail -1
done
