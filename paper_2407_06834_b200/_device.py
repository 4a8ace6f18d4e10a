"""Host <-> device plumbing for the drop-in (PyTorch as the allocator only).

Inputs may be numpy arrays (the reference's convention: results come back as
numpy, with the host<->device copies inside the call) or torch CUDA tensors
(device-resident: results stay on the device).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch


def is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


def pick_device(*candidates) -> torch.device:
    for c in candidates:
        if isinstance(c, torch.Tensor) and c.is_cuda:
            return c.device
        if isinstance(c, (str, torch.device)):
            return torch.device(c)
        if isinstance(c, int):
            return torch.device("cuda", c)
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2407_06834_b200 needs a CUDA device (B200); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, device: torch.device, dtype=torch.float64) -> torch.Tensor:
    """Contiguous device tensor holding x (numpy copies via pinned memory)."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=dtype)
        return t.contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    host = torch.from_numpy(arr)
    if arr.size >= (1 << 16):
        host = host.pin_memory()
    return host.to(device, non_blocking=True)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").numpy()


def like_input(t: torch.Tensor, template):
    """Return t as the same kind (numpy / torch) as the template input."""
    if isinstance(template, torch.Tensor):
        return t
    return to_host(t)


def stream_of(device: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())
