"""Stall-reason totals of an ncu SASS export (--page source --print-source sass
--csv) per address range: usage sass_ranges.py FILE.csv LO-HI [LO-HI ...]
(hex suffixes of the Address column, e.g. 75000-77800); no range = a histogram
of samples per 0x400 bytes of code to find the roles."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
def f(r, k):
    try: return float(r[ix[k]])
    except (ValueError, IndexError): return 0.0
body = [r for r in rows[2:] if len(r) > 5 and r[0].startswith("0x")]
base = int(body[0][0], 16)
if len(sys.argv) == 2:
    h = collections.Counter(); n = collections.Counter()
    for r in body:
        b = (int(r[0], 16) - base) // 0x400
        h[b] += f(r, "Warp Stall Sampling (All Samples)"); n[b] += f(r, "Instructions Executed")
    for b in sorted(h): print(f"+{b*0x400:06x} samples {int(h[b]):7d} inst {int(n[b]):12d}")
    sys.exit()
for spec in sys.argv[2:]:
    lo, hi = [int(x, 16) for x in spec.split("-")]
    tot = collections.Counter(); s = 0; inst = 0
    for r in body:
        a = int(r[0], 16) - base
        if lo <= a < hi:
            s += f(r, "Warp Stall Sampling (All Samples)"); inst += f(r, "Instructions Executed")
            for k in reasons: tot[k] += f(r, k)
    print(spec, "samples", int(s), "warp-inst", int(inst))
    for k, v in tot.most_common(8): print(f"   {k:28s} {v/max(s,1)*100:5.1f}%")
