# Round-2d: GPU tests after the kernel pruning + compute-sanitizer memcheck / racecheck / synccheck
set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "not config4_full_size" > gpurun_out/pytest_gpu_r2d.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu_r2d.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --leak-check full --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/sanitize_memcheck_r2d.log 2>&1; echo memcheck_rc=$?
timeout 1200 $CS --tool synccheck --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/sanitize_synccheck_r2d.log 2>&1; echo synccheck_rc=$?
timeout 1800 $CS --tool racecheck --racecheck-report analysis --print-limit 50 python scripts/sanitize_cases.py cfg1_default cfg1_cgs2 cfg1_block2 colblk_unit dense_F virtual_parts > gpurun_out/sanitize_racecheck_r2d.log 2>&1; echo racecheck_rc=$?
tail -4 gpurun_out/sanitize_*_r2d.log
