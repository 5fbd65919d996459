# session-4 final evidence of the committed tree: full GPU suite, smoke, bench lines of every config,
# the default bench's launch list, ncu --set full of config 3's kernels and of the 3D kernels
cd "$GRAFT_REPO_ROOT"
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/s4_bench_3.json 2> gpurun_out/s4_bench_3.err; echo bench3=$?
for cfg in 1 2; do
  timeout 900 python bench.py --config $cfg --steps 50 --warmup 5 > gpurun_out/s4_bench_$cfg.json 2> gpurun_out/s4_bench_$cfg.err; echo bench$cfg=$?
done
for cfg in 4 4c 5; do
  timeout 1500 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/s4_bench_$cfg.json 2> gpurun_out/s4_bench_$cfg.err; echo bench$cfg=$?
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/s4_launches_config3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s4_ncu_launch3.log 2>&1
tail -1 gpurun_out/s4_ncu_launch3.log | cut -c1-200
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_troubled_cells|k_central_tma|k_face_flux|k_gather|k_spread" -s 12 -c 6 -o gpurun_out/s4_full3 python scripts/prof_step.py --config 3 --warmup 1 --steps 1 > gpurun_out/s4_ncu_full3.log 2>&1
tail -2 gpurun_out/s4_ncu_full3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_central|k3_cwenoz|k3_muscl|k3_face_flux|k3_spread" -s 5 -c 5 -o gpurun_out/s4_final3d_5 python scripts/prof3d.py --config 5 --n 64 --warmup 0 --steps 1 > gpurun_out/s4_final3d_5.log 2>&1; tail -2 gpurun_out/s4_final3d_5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_central|k3_face_flux" -s 2 -c 2 -o gpurun_out/s4_final3d_4 python scripts/prof3d.py --config 4 --n 96 --warmup 0 --steps 1 > gpurun_out/s4_final3d_4.log 2>&1; tail -2 gpurun_out/s4_final3d_4.log
