#!/bin/bash
# A/B of ab_libs/A.so vs ab_libs/B.so on the config-4 probe (scripts/ab_probe.sh), then the solver parity
# tests with B in place.  Exploration only.
R=${R:-6} bash scripts/ab_probe.sh > gpurun_out/ab.log 2>&1
cp ab_libs/B.so paper_2210_16435_b200/lib/libsfairsc.so
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_dist.py} -m gpu -q -x -p no:cacheprovider > gpurun_out/ab_pytest.log 2>&1
echo pytest rc $? >> gpurun_out/ab.log
tail -n 3 gpurun_out/ab_pytest.log >> gpurun_out/ab.log
