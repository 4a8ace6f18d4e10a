"""fp64 throughput probes: DFMA loop vs DMMA (mma.sync m8n8k4 f64)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2407_06834_b200 import _lib  # noqa: E402

st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for name in ("nld_probe_fp64", "nld_probe_dmma"):
    for blocks in (0, 148 * 2, 148 * 16):
        tf, ms = ctypes.c_double(), ctypes.c_double()
        _lib.check(getattr(_lib.lib, name)(1 << 15, blocks, ctypes.byref(tf),
                                           ctypes.byref(ms), st))
        print(f"{name} blocks={blocks} {tf.value:.2f} TFLOP/s ({ms.value:.1f} ms)")
# mixed: DMMA warps + DFMA warps in the same CTAs
for im, ifm in ((1 << 14, 0), (0, 1 << 17), (1 << 14, 1 << 17), (1 << 14, 1 << 16)):
    tf, ms = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.lib.nld_probe_mixed(im, ifm, ctypes.byref(tf), ctypes.byref(ms), st))
    print(f"mixed mma_iters={im} fma_iters={ifm}: {tf.value:.2f} TFLOP/s ({ms.value:.1f} ms)")
