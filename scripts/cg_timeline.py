"""GPU timeline of one batched deflated CG solve (CUPTI via torch.profiler):
every kernel's start/end on the device, the idle gaps between them and the
kernel that precedes each large gap.
usage: python scripts/cg_timeline.py [config] [nalpha] [out.json]"""
import json
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2407_06834_b200 as nld  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
na = int(sys.argv[2]) if len(sys.argv) > 2 else 16
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/cg_timeline.json"
feats, wins, f_img = synth.make_problem(cfg)
op = nld.AnovaOperator(torch.from_numpy(feats).cuda(), wins, synth.SIGMA,
                       n_expansion=32, cutoff=4, oversampling=2.0)
eta = op.degree_device()
alphas = synth.alpha_sweep(float(eta.mean()), na)
f = torch.from_numpy(np.ascontiguousarray(f_img[:, 0])).cuda()
nld.deflated_solve_batched(op, f, 1.0, alphas, prec="jacobi", tol=synth.CG_TOL, maxit=200)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    res = nld.deflated_solve_batched(op, f, 1.0, alphas, prec="jacobi", tol=synth.CG_TOL,
                                     maxit=200)
    torch.cuda.synchronize()
evs = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        evs.append((e.time_range.start, e.time_range.end, e.name))
evs.sort()
t0, t1 = evs[0][0], max(e[1] for e in evs)
busy = 0.0
gaps = []
cur_end = evs[0][0]
prev = None
for s, e, n in evs:
    if s > cur_end:
        gaps.append((s - cur_end, prev, n))
    if e > cur_end:
        busy += e - max(s, cur_end)
        cur_end = e
    prev = n
gaps.sort(reverse=True)
tot_gap = sum(g[0] for g in gaps)
kern = {}
for s, e, n in evs:
    k = kern.setdefault(n[:60], [0, 0.0])
    k[0] += 1
    k[1] += (e - s) / 1e3
summary = {
    "span_ms": (t1 - t0) / 1e3, "busy_ms": busy / 1e3, "idle_ms": tot_gap / 1e3,
    "n_gaps": len(gaps),
    "iterations": [r.iterations for r in res],
    "top_gaps_us": [[round(g[0], 1), g[1][:50], g[2][:50]] for g in gaps[:40]],
    "gaps_by_prev": {},
    "kernels_ms": {k: [v[0], round(v[1], 3)] for k, v in sorted(kern.items(), key=lambda x: -x[1][1])},
}
by = {}
for g, p, n in gaps:
    key = f"{p[:40]} -> {n[:40]}"
    b = by.setdefault(key, [0, 0.0])
    b[0] += 1
    b[1] += g / 1e3
summary["gaps_by_prev"] = {k: [v[0], round(v[1], 3)] for k, v in
                           sorted(by.items(), key=lambda x: -x[1][1])[:25]}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: summary[k] for k in ("span_ms", "busy_ms", "idle_ms", "n_gaps")}))
