"""Rank SASS lines of an ncu source-page CSV (--print-source sass) by stall
samples and by excessive shared-memory wavefronts.
usage: python scripts/sass_hot.py SRC.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
ix = {h: i for i, h in enumerate(hdr)}
S = ix["Warp Stall Sampling (All Samples)"]
X = ix["L1 Wavefronts Shared Excessive"]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[S]) for r in data)
print("total samples", tot)


def top_reasons(r):
    v = sorted(((float(r[ix[c]]), c[6:]) for c in stall_cols), reverse=True)[:3]
    return " ".join(f"{c}:{x:.0f}" for x, c in v if x > 0)


for r in sorted(data, key=lambda r: -float(r[S]))[:n]:
    print(f"{float(r[S]) / tot * 100:5.1f}% {r[0][-5:]} {r[1].strip()[:60]:60s} {top_reasons(r)}")
print("--- excessive shared wavefronts")
for r in sorted(data, key=lambda r: -float(r[X] or 0))[:12]:
    if float(r[X] or 0) > 0:
        print(f"{float(r[X]):12.0f} {r[0][-5:]} {r[1].strip()[:70]}")
