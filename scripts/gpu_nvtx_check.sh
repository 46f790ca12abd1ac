# NVTX ranges: list the kernels ncu sees inside sfairsc.restart_sync (the prefetch sweep,
# normalisation, SpMV and the Ritz GEMM of a restart) and inside sfairsc.true_residuals
timeout 600 ncu --nvtx --nvtx-include "sfairsc.restart_sync/" --metrics gpu__time_duration.sum -c 12 --csv \
  python scripts/probe_cfg4.py --restarts 2 --applies 4 > gpurun_out/nvtx_restart.csv 2> gpurun_out/nvtx_restart.err; echo nvtx_rc=$?
grep -o '"[^"]*k_[a-z_0-9]*[^"]*"' gpurun_out/nvtx_restart.csv | sort | uniq -c | head -20
