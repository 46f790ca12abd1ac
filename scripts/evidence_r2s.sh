# Round-2s: per-part costs of the row-partitioned solver on the final kernels (DESIGN §9 model): config 4 and
# config 5 with virtual_parts 8 against one part (one GPU runs the P parts serially)
set -x
timeout 600 python scripts/probe_cfg4.py --restarts 3 --applies 4 --vparts 8 > gpurun_out/r2s_cfg4_vp8.json 2> gpurun_out/r2s_cfg4_vp8.err; echo c4v8=$?
timeout 600 python scripts/probe_cfg4.py --restarts 3 --applies 4 > gpurun_out/r2s_cfg4_vp1.json 2> gpurun_out/r2s_cfg4_vp1.err; echo c4v1=$?
timeout 900 python scripts/probe_cfg5_parts.py --parts 8 > gpurun_out/r2s_cfg5_vp8.json 2> gpurun_out/r2s_cfg5_vp8.err; echo c5v8=$?
timeout 900 python scripts/probe_cfg5_parts.py --parts 1 > gpurun_out/r2s_cfg5_vp1.json 2> gpurun_out/r2s_cfg5_vp1.err; echo c5v1=$?
