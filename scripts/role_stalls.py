"""Attribute ncu warp-stall samples of a warp-specialised kernel to roles by
SASS address ranges (helper lines such as mbar_wait are inlined, so their
samples belong to the role whose code surrounds them).
usage: python scripts/role_stalls.py SRC_cuda_sass.csv FILE ROLE:LO-HI ..."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
target = sys.argv[2]
roles = []
for spec in sys.argv[3:]:
    name, rng = spec.split(":")
    lo, hi = map(int, rng.split("-"))
    roles.append((name, lo, hi))
cur_file = None
line = None
ins = []   # (addr, file, line, samples, reasons)
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if len(r) < 8 or r[0] == "Function Name" or not r[2].startswith("0x"):
        if len(r) >= 2 and r[0]:
            try:
                line = int(r[0])
            except ValueError:
                pass
        continue
    if r[0]:
        line = int(r[0])
    try:
        s = float(r[4])
    except ValueError:
        continue
    reasons = {hdr[i][6:]: float(r[i]) for i in range(len(hdr))
               if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i] and r[i]}
    ins.append((int(r[2], 16), cur_file, line, s, reasons, r[3].strip()))
ins.sort()
owner = None
agg = {}
tot = sum(x[3] for x in ins)
for addr, f, ln, s, rs, sass in ins:
    if f == target:
        for name, lo, hi in roles:
            if lo <= ln <= hi:
                owner = name
    key = owner or "prologue"
    a = agg.setdefault(key, {"samples": 0.0})
    a["samples"] += s
    for k, v in rs.items():
        a[k] = a.get(k, 0.0) + v
for k, a in sorted(agg.items(), key=lambda x: -x[1]["samples"]):
    top = sorted(((v, r) for r, v in a.items() if r != "samples"), reverse=True)[:6]
    print(f"{k:12s} {a['samples'] / tot * 100:5.1f}%  " +
          " ".join(f"{r}:{v / tot * 100:.1f}" for v, r in top))
