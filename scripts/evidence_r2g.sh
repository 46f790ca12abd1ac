# Round-2g: paired-step solver (reorth 3) first check: small parity tests, then the config 2/4 A/B
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "eigs or config1 or config2 or planted or cliques" > gpurun_out/pytest_pair_r2g.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_pair_r2g.log
timeout 600 python scripts/pair_ab.py 2 4 > gpurun_out/pair_ab.log 2>&1; echo ab_rc=$?
cat gpurun_out/pair_ab.log | tail -12
