"""Top SASS lines of an ncu source export (--page source --print-source sass --csv)
by excessive shared wavefronts and by stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = rows[2:]
def f(r, k):
    try: return float(r[ix[k]])
    except (ValueError, KeyError, IndexError): return 0.0
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in body)
print("total samples", tot)
print("--- excessive shared wavefronts")
for r in sorted(body, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:12]:
    print(int(f(r, "L1 Wavefronts Shared Excessive")), int(f(r, "L1 Wavefronts Shared")), r[ix["Address"]][-5:], r[ix["Source"]].strip()[:90])
print("--- stall samples")
for r in sorted(body, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(int(f(r, "Warp Stall Sampling (All Samples)")), r[ix["Address"]][-5:], r[ix["Source"]].strip()[:100])
