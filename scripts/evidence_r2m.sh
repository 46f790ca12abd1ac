# Round-2m: full GPU suite + smoke + the default bench line on the final code
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r2m.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_gpu_r2m.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2m.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/smoke_r2m.log
timeout 1200 python bench.py > gpurun_out/bench_r2m.json 2> gpurun_out/bench_r2m.err; echo bench_rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r2m.json 2> gpurun_out/bench_ref_r2m.err; echo ref_rc=$?
tail -1 gpurun_out/bench_ref_r2m.json
