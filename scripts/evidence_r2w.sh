# Round-2w: final evidence on HEAD (4-stage Ritz ring, bench with roofline.gather_ceiling): full GPU suite + smoke,
# the default bench line and the reference arm, then (after the plain runs exited 0) the launch list of one bench
# solve and one ncu --set full capture of the Ritz GEMM and the SpMV
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r2w.log 2>&1; echo pytest_rc=$?
tail -n 4 gpurun_out/pytest_gpu_r2w.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2w.log 2>&1; echo smoke_rc=$?
tail -n 2 gpurun_out/smoke_r2w.log
timeout 1200 python bench.py > gpurun_out/bench_r2w.json 2> gpurun_out/bench_r2w.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r2w.json 2> gpurun_out/bench_ref_r2w.err; echo ref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_r2w.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kmeans > gpurun_out/ncu_ll_r2w.log 2>&1; echo ll_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ritz_dmma2 -c 1 \
  -o gpurun_out/r2w_ritz python scripts/probe_cfg4.py --restarts 2 --applies 2 > gpurun_out/ncu_r2w_ritz.log 2>&1; echo ncu_ritz_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tma -s 20 -c 1 \
  -o gpurun_out/r2w_spmv python scripts/probe_cfg4.py --restarts 1 --applies 2 > gpurun_out/ncu_r2w_spmv.log 2>&1; echo ncu_spmv_rc=$?
ls -la gpurun_out/ | grep r2w
