# Round-2a evidence on one B200: GPU tests, bench line, launch list, ncu --set full of the TMA SpMV and the sweep.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_r2a.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu_r2a.log
timeout 900 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo bench_rc=$?
tail -3 gpurun_out/bench_r2a.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_r2a.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kmeans > gpurun_out/ncu_ll.log 2>&1; echo ncu_ll_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lz_update_p|k_spmv_tma" -s 250 -c 2 -o /tmp/prof_r2a \
  python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
ncu -i /tmp/prof_r2a.ncu-rep --page details --csv > gpurun_out/prof_r2a_details.csv 2>&1
ncu -i /tmp/prof_r2a.ncu-rep --page raw --csv > gpurun_out/prof_r2a_raw.csv 2>&1
cp /tmp/prof_r2a.ncu-rep gpurun_out/ 2>/dev/null
ls -la gpurun_out/
