# Round-2 final ncu evidence (after the bench command exited 0 without ncu): launch list of one bench solve,
# ncu --set full of the TMA SpMV and of the pair sweep at J ~ 126 (exact kernel-name match) and of one Ritz GEMM
set -x
python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kmeans > gpurun_out/bench_plain_r2k.json 2>&1; echo plain_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_r2k.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kmeans > gpurun_out/ncu_ll_r2k.log 2>&1; echo ll_rc=$?
timeout 900 ncu -f --set full --clock-control none --import-source on -k k_lz_pair -s 62 -c 1 -o /tmp/r2k_pair \
  python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/ncu_r2k_pair.log 2>&1; echo pair_rc=$?
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_spmv_tma" -s 100 -c 1 -o /tmp/r2k_spmv \
  python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/ncu_r2k_spmv.log 2>&1; echo spmv_rc=$?
timeout 900 ncu -f --set full --clock-control none -k regex:"k_ritz_dmma2" -c 1 -o /tmp/r2k_ritz \
  python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/ncu_r2k_ritz.log 2>&1; echo ritz_rc=$?
for r in r2k_pair r2k_spmv r2k_ritz; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>&1
done
ncu -i /tmp/r2k_pair.ncu-rep --page source --csv > gpurun_out/r2k_pair_source.csv 2>&1
ls -la gpurun_out/ | grep r2k
