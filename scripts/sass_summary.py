"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
by SASS opcode: stall samples, executed instructions, excess smem wavefronts.
usage: ncu -i rep --page source --csv --print-source cuda,sass > src.csv;
       python scripts/sass_summary.py src.csv [function-substring]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
agg = defaultdict(lambda: [0, 0, 0, 0])
fn = ""
hdr = None
seen = set()
for row in csv.reader(open(path)):
    if not row:
        continue
    if row[0] == "Function Name":
        fn = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 8 or want not in fn or row[2] in ("-", "", "Address"):
        continue
    if (fn, row[2]) in seen:
        continue
    seen.add((fn, row[2]))
    op = row[3].strip().split()[0] if row[3].strip() else "?"
    if op.startswith("@"):
        op = row[3].strip().split()[1]
    op = op.split(".")[0]
    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    a = agg[op]
    a[0] += num(row[4])
    a[1] += num(row[7])
    a[2] += num(row[18])
    a[3] += num(row[hdr.index("stall_wait")])
tot = sum(v[0] for v in agg.values())
print(f"{'op':10s} {'samples':>9s} {'%':>6s} {'executed':>12s} {'smem_excess':>12s} {'wait':>8s}")
for op, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{op:10s} {v[0]:9d} {100*v[0]/max(tot,1):6.1f} {v[1]:12d} {v[2]:12d} {v[3]:8d}")
