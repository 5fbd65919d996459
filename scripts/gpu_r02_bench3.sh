# round 2: register A/B of the per-cell kernel, the default bench (config 3), ncu launch list + full capture
cd "$GRAFT_REPO_ROOT"
for v in base t8m20 t8m12; do
  UCFVB_LIB=scratch/ab/$v.so timeout 900 python scripts/time_steps.py --config 3 --steps 10 --tag $v 2>&1 | tail -1 | cut -c1-130
done
for v in base t8m20 t8m12; do
  UCFVB_LIB=scratch/ab/$v.so timeout 900 python scripts/time_steps.py --config 2 --steps 100 --tag $v 2>&1 | tail -1 | cut -c1-130
done
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench3.log 2>&1; tail -1 gpurun_out/r02_bench3.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_launches3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_launch3.log 2>&1
tail -1 gpurun_out/r02_ncu_launch3.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_troubled_cells|k_central_tma|k_face_flux|k_gather|k_spread" -s 10 -c 5 -o gpurun_out/r02_full3 python scripts/prof_step.py --config 3 --warmup 1 --steps 1 > gpurun_out/r02_ncu_full3.log 2>&1
tail -2 gpurun_out/r02_ncu_full3.log
