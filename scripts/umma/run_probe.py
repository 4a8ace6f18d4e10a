"""Drive scripts/umma/probe_umma.cu: layout check + i8 UMMA throughput.
usage: run_probe.py check M N K variant swap | rate M N K blocks"""
import ctypes
import os
import sys

import numpy as np

lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "probe_umma.so"))
P = ctypes.c_void_p
rng = np.random.default_rng(0)
mode = sys.argv[1]
if mode == "check":
    M, N, K, variant, swap = map(int, sys.argv[2:7])
    A = rng.integers(-128, 128, size=(M, K), dtype=np.int8)
    B = rng.integers(-128, 128, size=(N, K), dtype=np.int8)
    ref = A.astype(np.int64) @ B.astype(np.int64).T
    D = np.zeros((M, N), dtype=np.int32)
    rc = lib.umma_check(A.ctypes.data_as(P), B.ctypes.data_as(P), M, N, K,
                        D.ctypes.data_as(P), variant, swap)
    ok = np.array_equal(D.astype(np.int64), ref)
    print(f"check M={M} N={N} K={K} variant={variant} swap={swap} rc={rc} ok={ok}"
          f" maxdiff={np.abs(D - ref).max()}", flush=True)
    if not ok and rc == 0:
        # which entries match?  print a small corner for layout forensics
        print("D[:4,:8]", D[:4, :8].tolist())
        print("ref[:4,:8]", ref[:4, :8].tolist())
elif mode == "rate":
    M, N, K, blocks, nacc = map(int, sys.argv[2:7])
    t = ctypes.c_double()
    rc = lib.umma_rate(M, N, K, 4000, blocks, ctypes.byref(t), nacc)
    per = 2 * M * N * K / (t.value * 1e12 / blocks / 1.965e9) if t.value else 0
    print(f"rate M={M} N={N} K={K} blocks={blocks} nacc={nacc} rc={rc} {t.value:.1f} TOPS "
          f"~{per:.0f} clk per instr", flush=True)

if mode == "slice":
    n = 4096
    x = rng.uniform(-2**46 + 1, 2**46 - 1, n) / 3.0
    y = rng.uniform(-1, 1, n)
    out = np.zeros(n // 4 * 6, dtype=np.uint32)
    rc = lib.slice_check(x.ctypes.data_as(P), y.ctypes.data_as(P), n, out.ctypes.data_as(P))
    d = out.view(np.int8).reshape(n // 4, 6, 4)   # [group][p][element]
    bad = 0
    for g in range(n // 4):
        for e in range(4):
            val = sum(int(d[g, p, e]) * 256 ** (5 - p) for p in range(6))
            ref = x[4 * g + e] * y[4 * g + e]
            if abs(val - ref) > 1.0:
                bad += 1
                if bad < 5:
                    print("bad", g, e, val, ref, d[g, :, e].tolist())
    print("slice rc", rc, "bad", bad, "of", n)

if mode == "tmemA":
    for N in (64, 256):
        A = rng.integers(-128, 128, size=(128, 32), dtype=np.int8)
        B = rng.integers(-128, 128, size=(N, 32), dtype=np.int8)
        ref = A.astype(np.int64) @ B.astype(np.int64).T
        D = np.zeros((128, N), dtype=np.int32)
        rc = lib.umma_check_tmemA(A.ctypes.data_as(P), B.ctypes.data_as(P), N, D.ctypes.data_as(P))
        print("tmemA N", N, "rc", rc, "ok", np.array_equal(D.astype(np.int64), ref),
              "maxdiff", np.abs(D - ref).max())
