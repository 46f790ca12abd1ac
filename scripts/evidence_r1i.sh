# Round-1i ncu evidence on one B200 (after each command exited 0 without ncu): launch list of the bench command,
# ncu --set full of the sweep + SpMV at J ~ 125 and of one Ritz GEMM; reports reduced to CSV on the box.
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kmeans > gpurun_out/bench_plain_r1i.json 2>&1; echo plain_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_r1i.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kmeans > gpurun_out/ncu_ll.log 2>&1; echo ncu_ll_rc=$?
python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/probe_r1i.json 2>&1; echo probe_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_lz_update_p|k_spmm" -s 250 -c 2 -o /tmp/prof_r1i \
  python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
ncu --set full --clock-control none -k regex:"k_ritz_dmma2" -c 1 -o /tmp/prof_r1i_ritz \
  python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/ncu_ritz.log 2>&1; echo ncu_ritz_rc=$?
for r in prof_r1i prof_r1i_ritz; do
  ncu -i /tmp/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>&1
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>&1
done
ls -la gpurun_out/
