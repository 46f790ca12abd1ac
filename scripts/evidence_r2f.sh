# Round-2f: dense-F (rank-deficient) GPU tests, §8(f) N3 cost sweep, config-4 tight-residual attempt,
# oracle timing on the box's host, config-5 virtual_parts=8 per-part costs
set -x
timeout 900 python -m pytest tests/test_gpu_dense_f.py -q -p no:cacheprovider > gpurun_out/pytest_dense_r2f.log 2>&1; echo dense_rc=$?
tail -3 gpurun_out/pytest_dense_r2f.log
timeout 1500 python scripts/exp1_cost.py --out gpurun_out/exp1_cost.json > gpurun_out/exp1_cost.log 2>&1; echo exp1_rc=$?
tail -3 gpurun_out/exp1_cost.log
timeout 1200 python scripts/cfg4_tight.py --out gpurun_out/cfg4_tight.json > gpurun_out/cfg4_tight.log 2>&1; echo tight_rc=$?
tail -2 gpurun_out/cfg4_tight.log
timeout 900 python scripts/probe_cfg4.py --config 5 --vparts 8 --restarts 1 --applies 4 > gpurun_out/cfg5_vparts8.json 2> gpurun_out/cfg5_vparts8.err; echo vp8_rc=$?
timeout 900 python scripts/probe_cfg4.py --config 5 --restarts 1 --applies 4 > gpurun_out/cfg5_vparts1.json 2> gpurun_out/cfg5_vparts1.err; echo vp1_rc=$?
timeout 1200 python tests/tools/oracle_timing.py --tier-d 1 --tier-s 1,2,3 --out gpurun_out/oracle_timing.json > gpurun_out/oracle_timing.log 2>&1; echo ot_rc=$?
