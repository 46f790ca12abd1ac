# Round-2t (HEAD after NVTX) evidence on the final code: full GPU suite + smoke, the default bench line and the reference arm, then
# (after the bench exited 0 without ncu) the launch list of one bench solve
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r2t.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_gpu_r2t.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2t.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke_r2t.log
timeout 1200 python bench.py > gpurun_out/bench_r2t.json 2> gpurun_out/bench_r2t.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r2t.json 2> gpurun_out/bench_ref_r2t.err; echo ref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_r2t.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kmeans > gpurun_out/ncu_ll_r2t.log 2>&1; echo ll_rc=$?
ls -la gpurun_out/ | grep r2t
