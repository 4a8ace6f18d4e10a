"""Per CUDA source line stall samples from an ncu `--page source --print-source
cuda,sass --csv` export (all files of the kernel)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
agg = collections.Counter(); text = {}
fname = None; hdr = None; cur = None
for r in rows:
    if r and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 5: continue
    if r[0]:
        cur = (fname, r[0]); text[cur] = r[1]
    try: s = float(r[4])
    except ValueError: continue
    if cur: agg[cur] += s
tot = sum(agg.values()); print("total", tot)
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{v/tot*100:5.1f}% {k[0]}:{k[1]}  {text[k].strip()[:100]}")
