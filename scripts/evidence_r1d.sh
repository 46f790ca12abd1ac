# Round-1d evidence on one B200: bench line, ncu launch list of the bench command, ncu --set full of the two
# hot kernels (summaries extracted on the box; the .ncu-rep itself is not kept: gpurun_out/ is size-capped).
python bench.py > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err; echo bench_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_r1d.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kmeans > gpurun_out/ncu_ll.log 2>&1; echo ncu_ll_rc=$?
python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/probe_r1d.json 2>&1; echo probe_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_lz_update|k_spmm" -s 250 -c 2 -o /tmp/prof_r1d \
  python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
ncu -i /tmp/prof_r1d.ncu-rep --page details --csv > gpurun_out/prof_r1d_details.csv 2>&1
ncu -i /tmp/prof_r1d.ncu-rep --page raw --csv > gpurun_out/prof_r1d_raw.csv 2>&1
ls -la gpurun_out/
