cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/${TESTS:-test_gpu_run.py} -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py --steps 200 --warmup 5 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value']/1e9, 'e2e', d['e2e']['value']/1e9, 'frac', d['roofline']['frac'], d['roofline']['phase_us'])"
