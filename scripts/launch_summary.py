"""Summarise an `ncu --metrics gpu__time_duration.sum` launch list (CSV)."""
import csv
import json
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
seq = []
for r in rows[1:]:
    name = r[ik].split("(")[0].replace("nld::", "").replace("<unnamed>::", "")
    name = name.replace("mma::", "").replace("oz::", "").replace("void ", "")
    ns = float(r[iv]) * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r[iu], 1)
    seq.append((name, ns / 1e6))
# one steady-state matvec step.  Sliced path: every product starts with the
# per-rhs max kernel (k_vmax) -> the launches from the second-to-last k_vmax
# up to the last one.  fp64 DMMA path: after the second-to-last epilogue up
# to the last one.
starts = [i for i, (n, _) in enumerate(seq) if "k_vmax" in n]
ends = [i for i, (n, _) in enumerate(seq) if n.startswith("k_epilogue")]
if len(starts) >= 2:
    step = seq[starts[-2]:starts[-1]]
elif len(ends) >= 2:
    step = seq[ends[-2] + 1:ends[-1] + 1]
else:
    step = []
agg = OrderedDict()
cnt = OrderedDict()
for n, ms in step:
    n = n.split("<")[0]
    agg[n] = agg.get(n, 0.0) + ms
    cnt[n] = cnt.get(n, 0) + 1
tot = sum(agg.values())
out = {"launches_total": len(seq), "step_launches": len(step),
       "step_ms_serialized": tot,
       "step_share": {k: {"ms": v, "share": v / tot} for k, v in agg.items()},
       "step_launch_counts": cnt}
print(json.dumps(out, indent=1))
