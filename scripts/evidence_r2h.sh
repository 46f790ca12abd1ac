# Round-2h: full GPU suite with the paired solver as default (cfg-4 full-size test needs its golden) + bench
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not config4_full_size" > gpurun_out/pytest_gpu_r2h.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu_r2h.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r2h.json 2> gpurun_out/bench_r2h.err; echo bench_rc=$?
