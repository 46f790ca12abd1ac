#!/bin/bash
# A/B of reorthogonalisation sweep kernels on the config-4 probe
run() {
  env $2 timeout 300 python scripts/probe_cfg4.py --restarts 2 > gpurun_out/probe_$1.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/probe_$1.json')); e=d['eigs']
print('$1', {k:(round(v['us'],1), round(v['GBps'])) for k,v in e.items() if k in ('dots','upd_dots','upd_norm','spmv','ritz','normalize')}, round(d['wall_s'],3))
"
}
run tma2d "SFAIRSC_SWEEP=2"
run tma2d_m2reg "SFAIRSC_SWEEP=2 SFAIRSC_TMA_MODE2=0"
run reg "SFAIRSC_SWEEP=0"
