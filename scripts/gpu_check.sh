#!/bin/bash
# solver parity subset + config-4 bench on the in-tree library (exploration; the full suite is pytest -m gpu)
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_fullsize.py} -m gpu -q -x -p no:cacheprovider > gpurun_out/check_pytest.log 2>&1
echo pytest rc $?; tail -n 3 gpurun_out/check_pytest.log
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py --steps ${STEPS:-3} --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
  python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k:d[k] for k in ('value','ms_per_step','clocks')}); r=d['roofline']; print(r['frac'], {k:(round(v['us_per_launch'],1),v['launches']) for k,v in r['per_kernel'].items()})"
fi
