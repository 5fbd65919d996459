set -x
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_3d.py -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu3d.log
cat gpurun_out/pytest_gpu3d.log
for cfg in ${CFGS:-4 4c 5}; do timeout 600 python scripts/prof3d.py --config $cfg --n ${N:-96} > gpurun_out/prof3d_$cfg.log 2>&1; cat gpurun_out/prof3d_$cfg.log; done
