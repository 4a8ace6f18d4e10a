"""Drive probe_pattern.cu: cycles per 32-node tile of each UMMA issue pattern."""
import ctypes
import os

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe_pattern.so"))
names = {0: "gather pattern (SS, shifted D)", 1: "12 x N=32 disjoint", 2: "12 x N=192 same D",
         3: "gather pattern, A in TMEM", 4: "12 x N=256 same D", 5: "4 x N=256",
         6: "gather pattern, p outer", 7: "spread pattern (per chunk)", 8: "spread pattern, 2 chunks chained (per 2 chunks)"}
for v in ():
    c = ctypes.c_double()
    rc = lib.pattern_rate(v, 20000, 148, ctypes.byref(c))
    print(f"variant {v} {names[v]:34s} rc={rc} {c.value:8.1f} cycles/tile", flush=True)
for w in ():
    c = ctypes.c_double()
    rc = lib.tld_rate(w, 20000, 148, ctypes.byref(c))
    print(f"tcgen05.ld 32x32b.x8, {w:2d} warps/SM rc={rc} {c.value:8.1f} B/cycle/SM", flush=True)
for mma in (0, 1):
    for blocks in (1, 148):
        c = ctypes.c_double()
        rc = lib.commit_rt(2000, mma, blocks, ctypes.byref(c))
        print(f"commit round trip (mma={mma}, blocks={blocks}) rc={rc} {c.value:8.1f} cycles", flush=True)
