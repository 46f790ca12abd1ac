# Round-2y: the config-5 fixed-budget bench line at N = 1 on HEAD (the E(P) anchor of SURVEY 8(d) metric 2: the same
# thick-restart budget is what `torchrun ... bench.py --gpus N --config 5 --max-restarts 3` runs row-partitioned)
set -x
timeout 1500 python bench.py --config 5 --max-restarts 3 --steps 1 --warmup 3 --no-cpu-baseline --no-kmeans --no-e2e \
  > gpurun_out/bench_r2y_cfg5.json 2> gpurun_out/bench_r2y_cfg5.err; echo bench5_rc=$?
tail -n 3 gpurun_out/bench_r2y_cfg5.err
cut -c1-1500 gpurun_out/bench_r2y_cfg5.json
