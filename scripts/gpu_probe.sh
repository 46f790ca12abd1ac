#!/bin/bash
# config-4 probe (a few restart cycles, per-kernel events) run N times on the in-tree library, then a short
# bench.  Exploration only.
for r in $(seq 1 ${NRUN:-3}); do
  timeout 300 python scripts/probe_cfg4.py --restarts ${R:-6} --applies 4 > gpurun_out/probe_$r.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/probe_$r.json')); e=d['eigs']
print('run$r', d['stats']['applies'], round(sum(x['us']*x['launches'] for x in e.values())/1e3,1), {k:(round(x['us'],1), x['launches']) for k,x in e.items()})"
done
if [ -n "$BENCH" ]; then timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.json; fi
