cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py::test_config3_full_size_conservation_and_determinism 2>&1 | tail -1
for pdl in 0 1; do
  UCFVB_PDL=$pdl timeout 600 python scripts/time_steps.py --config 2 --steps 200 --tag "pdl=$pdl" 2>&1 | tail -1
  UCFVB_PDL=$pdl timeout 600 python scripts/time_steps.py --config 1 --steps 200 --tag "pdl=$pdl" 2>&1 | tail -1
done
