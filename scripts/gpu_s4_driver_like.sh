# what the driver runs at round end: GPU suite, smoke, the reference arm, the default bench line
cd "$GRAFT_REPO_ROOT"
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4_ref_arm.json 2> gpurun_out/s4_ref_arm.err; echo ref=$?; tail -1 gpurun_out/s4_ref_arm.json | cut -c1-400
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4_driver_bench.json 2> gpurun_out/s4_driver_bench.err; echo bench=$?; tail -1 gpurun_out/s4_driver_bench.json | cut -c1-300
