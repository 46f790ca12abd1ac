# Round-2u: A/C of the 4-stage Ritz GEMM ring (C) against HEAD (A): full config-4
# solves alternating, per-kernel profiled solves, then the GPU suite's solve subset on C and an ncu capture of
# C's Ritz GEMM and three-term pass (after the plain runs exited 0)
set -x
SPEC="170,80;170,80" VARIANTS="A C" KPROF=1 bash scripts/gpu_ab_solve.sh > gpurun_out/ab_r2u.log 2>&1; echo ab_rc=$?
cat gpurun_out/ab_r2u.log
cp ab_libs/C.so paper_2210_16435_b200/lib/libsfairsc.so
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_r2u.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu_r2u.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_ritz_dmma2|k_lz_three' -c 2 \
  -o gpurun_out/r2u_ritz python scripts/probe_cfg4.py --restarts 2 --applies 2 > gpurun_out/ncu_r2u.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_r2u.log
