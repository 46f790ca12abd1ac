# Round-2p evidence on the final code: full GPU suite + smoke, the default bench line and the reference arm,
# then (after the bench exited 0 without ncu) the launch list of one bench solve and ncu --set full of the
# pair sweep at J = 125 (MAXQ 16), the TMA SpMV, the Ritz GEMM (p = 80) and the three-term kernel
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r2p.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_gpu_r2p.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2p.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke_r2p.log
timeout 1200 python bench.py > gpurun_out/bench_r2p.json 2> gpurun_out/bench_r2p.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r2p.json 2> gpurun_out/bench_ref_r2p.err; echo ref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_r2p.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kmeans > gpurun_out/ncu_ll_r2p.log 2>&1; echo ll_rc=$?
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_lz_pair<" -s 62 -c 1 -o /tmp/r2p_pair \
  python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/ncu_r2p_pair.log 2>&1; echo pair_rc=$?
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"k_spmv_tma" -s 100 -c 1 -o /tmp/r2p_spmv \
  python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/ncu_r2p_spmv.log 2>&1; echo spmv_rc=$?
timeout 900 ncu -f --set full --clock-control none -k regex:"k_ritz_dmma2" -c 1 -o /tmp/r2p_ritz \
  python scripts/probe_cfg4.py --restarts 2 --applies 4 > gpurun_out/ncu_r2p_ritz.log 2>&1; echo ritz_rc=$?
timeout 900 ncu -f --set full --clock-control none -k regex:"k_lz_three" -s 20 -c 1 -o /tmp/r2p_three \
  python scripts/probe_cfg4.py --restarts 1 --applies 4 > gpurun_out/ncu_r2p_three.log 2>&1; echo three_rc=$?
for r in r2p_pair r2p_spmv r2p_ritz r2p_three; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>&1
done
ls -la gpurun_out/ | grep r2p
