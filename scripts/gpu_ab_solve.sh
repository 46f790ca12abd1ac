#!/bin/bash
# A/B(/C...) of library builds ab_libs/<V>.so: full config-4 solves (profiling off), alternating; then one
# profiled probe per variant.  Exploration only.
L=paper_2210_16435_b200/lib/libsfairsc.so
for r in 1 2 3; do for v in ${VARIANTS:-A B}; do
  cp ab_libs/$v.so $L
  echo -n "$v$r "; timeout 300 python scripts/basis_scan.py "${SPEC:-170,80}" 2>/dev/null | tail -1
done; done
if [ -n "$PROBE" ]; then for v in ${VARIANTS:-A B}; do
  cp ab_libs/$v.so $L
  timeout 300 python scripts/probe_cfg4.py --restarts 3 --applies 4 > gpurun_out/probe_$v.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/probe_$v.json')); e=d['eigs']
print('$v', {k:(round(x['us'],1), x['launches']) for k,x in e.items()})"
done; fi
if [ -n "$KPROF" ]; then for r in 1 2; do for v in ${VARIANTS:-A B}; do
  cp ab_libs/$v.so $L
  echo -n "prof $v$r "; timeout 300 python scripts/ab_profile.py 2>/dev/null | tail -1
done; done; fi
