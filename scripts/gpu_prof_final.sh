# Final round-1 evidence for the current build: the step's launch list
# (scripts/prof_step.py, un-graphed), the bench command's launch list, and one
# `ncu --set full` capture of the four main kernels.
cd "$GRAFT_REPO_ROOT"
PROF_NAME=prof_r1z bash scripts/gpu_prof.sh
timeout 300 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
echo bench_ncu_rc=$?
