# Round-2v: C (HEAD: 4-stage Ritz ring) vs D (persistent Ritz GEMM, one k-tile stream across output tiles):
# full config-4 solves alternating + per-kernel profiled solves; GPU suite on D; bench line on D; then (after the
# plain runs exited 0) ncu --set full of D's Ritz GEMM
set -x
SPEC="170,80;170,80" VARIANTS="C D" KPROF=1 bash scripts/gpu_ab_solve.sh > gpurun_out/ab_r2v.log 2>&1; echo ab_rc=$?
cat gpurun_out/ab_r2v.log
cp ab_libs/D.so paper_2210_16435_b200/lib/libsfairsc.so
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu_r2v.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu_r2v.log
timeout 1200 python bench.py > gpurun_out/bench_r2v.json 2> gpurun_out/bench_r2v.err; echo bench_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ritz_dmma2 -c 1 \
  -o gpurun_out/r2v_ritz python scripts/probe_cfg4.py --restarts 2 --applies 2 > gpurun_out/ncu_r2v.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/ncu_r2v.log
