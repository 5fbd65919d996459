cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -q -x 2>&1 | tail -2
for cfg in 2 3; do timeout 600 python scripts/time_steps.py --config $cfg --steps 100 --tag "pair-b(102r)" 2>&1 | tail -1; done
cp scratch/kp_a.cuh paper_2510_25906_b200/csrc/kernels_pair.cuh && make -C paper_2510_25906_b200 -j8 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -q -x 2>&1 | tail -2
for cfg in 2 3; do timeout 600 python scripts/time_steps.py --config $cfg --steps 100 --tag "pair-a(96r,spill)" 2>&1 | tail -1; done
