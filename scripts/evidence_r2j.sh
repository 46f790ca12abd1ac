# Round-2j: full GPU suite (incl. the config-4 full-size test with its Tier S golden), config-5 virtual parts
# (8 vs 1, basis 100: per-part kernel costs for the multi-GPU model), the full bench line
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_r2j.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu_r2j.log
timeout 900 python scripts/probe_cfg5_parts.py --parts 8 > gpurun_out/cfg5_vp8.json 2> gpurun_out/cfg5_vp8.err; echo vp8_rc=$?
timeout 900 python scripts/probe_cfg5_parts.py --parts 1 > gpurun_out/cfg5_vp1.json 2> gpurun_out/cfg5_vp1.err; echo vp1_rc=$?
timeout 1200 python bench.py > gpurun_out/bench_r2j.json 2> gpurun_out/bench_r2j.err; echo bench_rc=$?
