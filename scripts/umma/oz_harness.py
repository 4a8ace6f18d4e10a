"""Sliced spread kernel vs fp64 on one synthetic subproblem."""
import ctypes
import os
import sys

import numpy as np

lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), os.environ.get("OZH", "oz_harness.so")))
P = ctypes.c_void_p
nsub = int(sys.argv[1])
mag = float(sys.argv[2])
for K in [int(k) for k in sys.argv[3:]] or [32, 64, 509]:
    rng = np.random.default_rng(K)
    rows = rng.uniform(-1.0, 1.0, size=(K, 24)) * 2.0 ** rng.integers(-10, 10, size=(K, 24)) * mag
    v = rng.standard_normal((K, 16))
    blk = np.zeros((512 * nsub, 16))
    ex = np.zeros(24 * nsub, dtype=np.int16)
    rc = lib.oz_spread_one(rows.ctypes.data_as(P), v.ctypes.data_as(P), K, blk.ctypes.data_as(P),
                           ex.ctypes.data_as(P), nsub)
    A, B, C = rows[:, :8], rows[:, 8:16], rows[:, 16:]
    ref = np.zeros((512 * nsub, 16))
    for i in range(nsub):
        lo = i * (K // nsub)
        hi = K if i == nsub - 1 else lo + K // nsub
        ref[512 * i:512 * (i + 1)] = np.einsum("jr,ja,jb,jc->abcr", v[lo:hi], A[lo:hi], B[lo:hi],
                                               C[lo:hi]).reshape(512, 16)
    err = np.linalg.norm(blk - ref) / np.linalg.norm(ref)
    print(f"nsub={nsub} mag={mag} K={K} rc={rc} rel={err:.3e} ex={ex[:24].tolist()}")
    if err > 1e-8:
        for (a, bc, r) in [(0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0), (0, 8, 0)]:
            print("  ", a, bc, r, blk[a * 64 + bc, r], ref[a * 64 + bc, r])

if os.path.exists("/tmp/oz_sub0.bin") and nsub == 1 and mag == 0:
    raw = np.fromfile("/tmp/oz_sub0.bin", dtype=np.uint8)
    K = int(raw[:4].view(np.int32)[0])
    rows = raw[4:4 + K * 24 * 8].view(np.float64).reshape(K, 24).copy()
    v = raw[4 + K * 24 * 8:].view(np.float64).reshape(K, 16).copy()
    blk = np.zeros((512, 16))
    ex = np.zeros(24, dtype=np.int16)
    rc = lib.oz_spread_one(rows.ctypes.data_as(P), v.ctypes.data_as(P), K, blk.ctypes.data_as(P),
                           ex.ctypes.data_as(P), 1)
    A, B, C = rows[:, :8], rows[:, 8:16], rows[:, 16:]
    ref = np.einsum("jr,ja,jb,jc->abcr", v, A, B, C).reshape(512, 16)
    print("real sub0 K", K, "rel", np.linalg.norm(blk - ref) / np.linalg.norm(ref), ex.tolist())
