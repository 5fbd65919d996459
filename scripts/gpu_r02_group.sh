# round 2: multi-GPU schedule on one device (loopback group), decomposition + 3D error tests, parity
cd "$GRAFT_REPO_ROOT"
timeout 1800 python -m pytest tests/test_gpu_decompose.py tests/test_gpu_3d.py tests/test_gpu_parity.py tests/test_gpu_run.py -q -x 2>&1 | tail -25 > gpurun_out/r02_group_pytest.log
cat gpurun_out/r02_group_pytest.log
