"""Probe: time sfairsc_embed_kmeans on a BASELINE config after the eigensolve,
with launch counts and (optionally) a per-kernel breakdown via torch.profiler's
CUPTI trace.  Usage: probe_kmeans.py [config] [--trace]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_16435_b200 import lib  # noqa: E402
from synth import baseline_config  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 4
trace = "--trace" in sys.argv
dev = torch.device("cuda:0")
g, cfg = baseline_config(c)
k = cfg["k_eig"]
t = lambda a: torch.from_numpy(a).to(dev)
rp, ci, vv, gr = t(g.row_ptr), t(g.col), t(g.val), t(g.groups.astype(np.int32))
ctx = lib.sfairsc_build_operator(rp, ci, vv, gr, k, cfg["normalized"], h=g.h)
ev, _, st = lib.sfairsc_eigs(ctx, k, cfg["tol"], want_evecs=False)
lab = torch.empty(g.n, dtype=torch.int32, device=dev)
res = {"config": c, "n": g.n, "k": k, "t_eigs_s": st["t_eigs_s"]}
for rep in range(2):
    l0 = lib.launch_count()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, wcss = lib.sfairsc_embed_kmeans(ctx, 1, lab)
    torch.cuda.synchronize()
    res[f"kmeans_s_{rep}"] = time.perf_counter() - t0
    res[f"launches_{rep}"] = lib.launch_count() - l0
    res["wcss"] = wcss
if g.clusters is not None and (g.clusters >= 0).all():
    from oracle.metrics import error_rate  # test infrastructure: scoring only
    res["error_rate"] = float(error_rate(g.clusters, lab.cpu().numpy(), k))
if trace:
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        lib.sfairsc_embed_kmeans(ctx, 1, lab)
        torch.cuda.synchronize()
    agg = {}
    for e in prof.events():
        if e.device_type.name == "CUDA":
            a = agg.setdefault(e.name[:60], [0, 0.0])
            a[0] += 1
            a[1] += e.device_time_total / 1e3 if hasattr(e, "device_time_total") else e.cuda_time_total / 1e3
    res["trace_ms"] = {k2: [v[0], round(v[1], 3)] for k2, v in sorted(agg.items(), key=lambda x: -x[1][1])[:12]}
print(json.dumps(res, indent=1), flush=True)
json.dump(res, open(os.path.join(os.environ.get("OUT", "gpurun_out"), f"kmeans_cfg{c}.json"), "w"), indent=1)
