# Round-2c: GPU test suite (cfg-4 full-size test deselected until its golden lands) + bench with the 2048-entry tiles
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not config4_full_size" > gpurun_out/pytest_gpu_r2c.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu_r2c.log
timeout 900 python bench.py > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err; echo bench_rc=$?
