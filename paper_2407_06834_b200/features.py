"""Feature and window preparation on the device (reference features.py).

Same API as ``nldenoise.features``: ``extract_patches`` (zero padding, raster
patch order), ``center_column``, ``mutual_information_scores`` (16 x 16 plug-in
MI with the patch centre), ``split_windows`` (descending score, ties by index,
consecutive triples) and ``feature_windows``.  The patch extraction and the
joint histograms run in CUDA kernels (integer counts, exact); the final sort
of <= 49 scores into windows is host logic, as in the reference.
``baseline_features`` builds BASELINE's reflect-padded, 0.4 (v - 0.5) mapped
features on the device (identical to ``synth.patch_features``).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _device as dv
from ._lib import check, lib
from .errors import WindowSizeError

MI_BINS = 16          # features.py:16
WINDOW_DIMS = 3       # features.py:17


def _image_planar(image):
    """Channel-planar device image [C][h][w] and the input kind."""
    pix = getattr(image, "pixels", image)
    if dv.is_torch(pix):
        t = pix.to(torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(pix, np.float64)))
    if t.dim() == 2:
        t = t.unsqueeze(0)
    elif t.dim() == 3:
        t = t.permute(2, 0, 1)            # (h, w, C) -> (C, h, w)
    else:
        raise ValueError("expected a 2-d image")
    dev = dv.pick_device(pix)
    return t.to(dev).contiguous(), pix


def _patches(image, patch_size, mode, a, b):
    if patch_size < 1 or patch_size % 2 == 0:
        raise ValueError("patch size must be odd and positive")
    img, src = _image_planar(image)
    c, h, w = img.shape
    out = torch.empty((h * w, c * patch_size * patch_size), dtype=torch.float64,
                      device=img.device)
    check(lib.nld_extract_patches(dv.ptr(img), h, w, c, patch_size, mode, float(a),
                                  float(b), dv.ptr(out), dv.stream_of(img.device)))
    return out if dv.is_torch(src) else out.cpu().numpy()


def extract_patches(image, patch_size: int):
    """Feature matrix (n_pixels, patch_size**2), zero padding (features.py:20-36)."""
    pix = getattr(image, "pixels", image)
    if len(tuple(pix.shape) if hasattr(pix, "shape") else np.shape(pix)) != 2:
        raise ValueError("expected a 2-d image")
    return _patches(image, patch_size, 0, 1.0, 0.0)


def baseline_features(image, patch_size: int):
    """BASELINE features: reflect padding, 0.4 (v - 0.5), channel-major."""
    return _patches(image, patch_size, 1, 0.4, 0.5)


def center_column(patch_size: int) -> int:
    """Raster-order index of the patch centre (features.py:39-41)."""
    return (patch_size * patch_size) // 2


def mutual_information_scores(features, center=None) -> np.ndarray:
    """Plug-in mutual information (nats) of each column with the centre."""
    f = features if dv.is_torch(features) else np.asarray(features, np.float64)
    n, d = tuple(f.shape)
    if center is None:
        center = (d - 1) // 2
    if not 0 <= center < d:
        raise ValueError("center column out of range")
    dev = dv.pick_device(f)
    ft = dv.to_device(f, dev)
    scores = np.empty(d)
    check(lib.nld_mi_scores(dv.ptr(ft), n, d, int(center),
                            scores.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                            dv.stream_of(dev)))
    return scores


def split_windows(scores) -> list[np.ndarray]:
    """Descending score, ties by ascending index, consecutive triples (:81-89)."""
    s = np.asarray(scores, dtype=np.float64)
    order = np.lexsort((np.arange(s.size), -s))
    return [order[i:i + WINDOW_DIMS] for i in range(0, s.size, WINDOW_DIMS)]


def feature_windows(image, patch_size: int):
    """Patches, MI ranking, window split (features.py:92-104)."""
    feats = extract_patches(image, patch_size)
    scores = mutual_information_scores(feats, center_column(patch_size))
    windows = split_windows(scores)
    for w in windows:
        if w.size > WINDOW_DIMS:
            raise WindowSizeError("window wider than the 3-d transform limit")
    return feats, windows
