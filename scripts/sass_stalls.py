"""Per-SASS-line stall reasons of an ncu source export (--page source --print-source sass --csv).
usage: sass_stalls.py file.csv [min_samples] [addr_lo addr_hi]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 300
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 62
st = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
def f(r, k):
    try: return float(r[ix[k]])
    except (ValueError, IndexError): return 0.0
tot = {s: 0.0 for s in st}
for r in rows[2:]:
    a = int(r[ix['Address']], 16) & 0xfffff
    if not (lo <= a < hi): continue
    for s in st: tot[s] += f(r, s)
    n = f(r, 'Warp Stall Sampling (All Samples)')
    if n >= mn:
        top = sorted(((f(r, s), s[6:]) for s in st), reverse=True)[:3]
        print(f"{a:05x} {int(n):6d} {int(f(r,'Instructions Executed')):9d}  " + " ".join(f"{k}:{int(v)}" for v, k in top) + "  | " + r[ix['Source']].strip()[:70])
print("totals:", {k[6:]: int(v) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v > 0})
