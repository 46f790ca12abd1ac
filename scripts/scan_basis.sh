# basis size / kept Ritz vectors scan at config 4 (full solves, profiling on): time, applies, restarts
for mk in "170 80" "192 80" "192 95" "192 110" "180 90" "170 95"; do
  set -- $mk
  python scripts/probe_cfg4.py --restarts 100000 --applies 4 --m $1 --keep $2 > gpurun_out/scan.json 2>&1
  python3 -c "
import json;s=open('gpurun_out/scan.json').read();d=json.loads(s[s.index('{'):]);st=d['stats']
print(json.dumps({'m':$1,'keep':$2,'wall_s':round(d['wall_s'],3),'applies':st['applies'],'restarts':st['restarts'],'resid':st['max_resid_rel'],'us':{k:round(v['us'],1) for k,v in d['eigs'].items() if k in ('spmv','upd_dots','ritz')}}))"
done
