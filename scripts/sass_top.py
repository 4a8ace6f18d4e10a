"""Top SASS instructions of one function in an ncu source-page CSV, with
their leading stall reasons.  usage: sass_top.py src.csv func [min_samples]"""
import csv
import sys

path, want = sys.argv[1], sys.argv[2]
thr = int(sys.argv[3]) if len(sys.argv) > 3 else 1500
hdr = None
fn = ""
seen = set()


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


rows = []
for row in csv.reader(open(path)):
    if not row:
        continue
    if row[0] == "Function Name":
        fn = row[1]
        continue
    if row[0] == "Line No":
        hdr = row
        cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if hdr is None or len(row) < 8 or want not in fn or row[2] in ("-", ""):
        continue
    if row[2] in seen:
        continue
    seen.add(row[2])
    s = num(row[4])
    if s >= thr:
        st = {c[6:]: num(row[hdr.index(c)]) for c in cols}
        top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        rows.append((row[2][-5:], row[3].strip()[:58], s, num(row[7]), top))
for r in rows:
    print(r[0], r[1].ljust(58), r[2], r[3], r[4])
