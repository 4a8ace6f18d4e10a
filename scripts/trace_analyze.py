"""Summarise an NLD_OZ_TRACE wait log (site warp start end per line) of CTA 0."""
import collections
import sys

rows = [tuple(int(x) for x in l.split()) for l in open(sys.argv[1])]
roles = dict(a.split("=") for a in sys.argv[2:]) if len(sys.argv) > 2 else {}
t0 = min(r[2] for r in rows)
t1 = max(r[3] for r in rows)
span = t1 - t0
print(f"events {len(rows)}, span {span} cycles")
per = collections.defaultdict(lambda: [0, 0])
for site, warp, a, b in rows:
    k = (warp, site)
    per[k][0] += 1
    per[k][1] += b - a
for (warp, site), (n, tot) in sorted(per.items()):
    print(f"warp {warp:2d} site {site:2d}: n {n:6d}  wait {tot:10d} ({tot / span * 100:5.1f}%)  avg {tot / max(n, 1):8.0f}")
# the issuer's per-tile period (site 1 = y_full wait per tile)
iss = [r for r in rows if r[0] == 1]
if len(iss) > 4:
    ends = sorted(r[3] for r in iss)
    d = [b - a for a, b in zip(ends, ends[1:])]
    d.sort()
    print("issuer tile period: median", d[len(d) // 2], "p10", d[len(d) // 10], "p90", d[9 * len(d) // 10])
# epilogue warp 0 per-tile period (site 21 marker)
ep = sorted(r[3] for r in rows if r[0] == 21 and r[1] == 0)
if len(ep) > 4:
    d = sorted(b - a for a, b in zip(ep, ep[1:]))
    print("epilogue warp0 tile period: median", d[len(d) // 2], "p10", d[len(d) // 10], "p90", d[9 * len(d) // 10])
# a slice of the timeline in the middle
mid = t0 + span // 2
win = sorted((r for r in rows if mid <= r[2] < mid + 20000), key=lambda r: r[2])
for site, warp, a, b in win[:120]:
    print(f"{a - mid:7d} {b - mid:7d} w{warp:2d} s{site:2d} {'wait ' + str(b - a) if b > a else ''}")
