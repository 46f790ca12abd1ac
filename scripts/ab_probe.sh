#!/bin/bash
# A/B of two library builds (ab_libs/A.so, ab_libs/B.so) on the config-4 probe, alternating twice.
# Exploration only; prints per-kernel mean times.
L=paper_2210_16435_b200/lib/libsfairsc.so
for r in 1 2; do for v in A B; do
  cp ab_libs/$v.so $L
  timeout 300 python scripts/probe_cfg4.py --restarts ${R:-3} --applies 4 "$@" > gpurun_out/ab_$v$r.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/ab_$v$r.json')); e=d['eigs']
print('$v$r', d['stats']['applies'], round(sum(x['us']*x['launches'] for x in e.values())/1e3,1), {k:(round(x['us'],1), x['launches']) for k,x in e.items()})"
done; done
