# full GPU test suite + smoke + the config-3 launch list (lists policy, second call) + 3D A/B
cd "$GRAFT_REPO_ROOT"
timeout 3000 python -m pytest tests -m gpu -q -x -s 2>&1 | grep -E "passed|failed|Error|config[23]:|^E " | tail -30 > gpurun_out/r02_tests.log
cat gpurun_out/r02_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/r02_launches3.csv python scripts/prof_step.py --config 3 --warmup 2 --steps 2 > gpurun_out/r02_ncu_launch3.log 2>&1
tail -1 gpurun_out/r02_ncu_launch3.log
LIBS="base b3d cw3m3" bash scripts/gpu_ab_3d.sh
