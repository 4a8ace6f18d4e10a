"""Seeded synthetic inputs for the BASELINE.json configurations.

BASELINE.json describes the workloads only in words; this module pins one
concrete reading of them so the GPU path, the CPU oracle and the bench all see
bit-identical features:

* image: linear-gradient background, 6 axis-aligned rectangles and 4 discs
  painted with U[0,1] intensities, plus 3 low-frequency sinusoids of
  amplitude 0.05; iid N(0, 0.1^2) noise; clipped to [0, 1].
* features: k x k patches per pixel with *reflect* padding, patch entries in
  row-major order (channel-major for RGB), mapped by 0.4 (v - 0.5) into
  [-0.2, 0.2].
* windows: consecutive triples of feature indices, the remainder as a last
  short window (3x3 -> 3 windows of 3; 5x5 -> 8 x 3 + 1 x 1; RGB 3x3 ->
  9 windows of 3, one per channel-row).

The reference builds its features differently (zero padding, MIS ranking,
``features.py:20-104``); BASELINE fixes the features itself, and the operator
under test (``kernel.py:28``) takes features and windows as given, so this
generator sits outside the hot path.  It is NOT the oracle.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SIGMA = 0.1          # kernel length (BASELINE: exp(-||x-y||^2 / 0.1^2))
N_EXPANSION = 32     # NFFT bandwidth per dimension
OVERSAMPLING = 2.0   # grid 64 per dimension
CUTOFF = 4           # Kaiser-Bessel window cutoff m
CG_TOL = 1e-6
ALPHA_SCALE = 10.0   # alpha = 10 / mean(eta)


@dataclass(frozen=True)
class Config:
    name: str
    side: int
    channels: int
    patch: int
    seed: int
    n_alpha: int = 1

    @property
    def n(self) -> int:
        return self.side * self.side


CONFIGS = {
    "c0": Config("c0", 64, 1, 3, 0),
    "c1": Config("c1", 256, 1, 3, 1),
    "c2": Config("c2", 1024, 1, 5, 2),
    "c3": Config("c3", 512, 3, 3, 3),
    "c4": Config("c4", 4096, 1, 3, 4, n_alpha=16),
}


def synthetic_channel(side: int, rng: np.random.Generator) -> np.ndarray:
    """One clean [0,1]-ish channel: gradient + rectangles + discs + sinusoids."""
    yy, xx = np.mgrid[0:side, 0:side].astype(np.float64) / max(side - 1, 1)
    theta = rng.uniform(0.0, 2.0 * np.pi)
    lo, hi = np.sort(rng.uniform(0.0, 1.0, size=2))
    proj = np.cos(theta) * xx + np.sin(theta) * yy
    proj = (proj - proj.min()) / max(proj.max() - proj.min(), 1e-12)
    img = lo + (hi - lo) * proj
    for _ in range(6):
        r0, r1 = np.sort(rng.integers(0, side, size=2))
        c0, c1 = np.sort(rng.integers(0, side, size=2))
        img[r0:r1 + 1, c0:c1 + 1] = rng.uniform(0.0, 1.0)
    for _ in range(4):
        cy, cx = rng.uniform(0.0, 1.0, size=2)
        rad = rng.uniform(0.05, 0.2)
        mask = (yy - cy) ** 2 + (xx - cx) ** 2 < rad * rad
        img[mask] = rng.uniform(0.0, 1.0)
    for _ in range(3):
        fy, fx = rng.uniform(0.5, 3.0, size=2)
        phase = rng.uniform(0.0, 2.0 * np.pi)
        img += 0.05 * np.sin(2.0 * np.pi * (fy * yy + fx * xx) + phase)
    return img


def noisy_image(cfg: Config) -> np.ndarray:
    """(side, side) or (side, side, channels) noisy image in [0, 1]."""
    rng = np.random.default_rng(cfg.seed)
    chans = []
    for _ in range(cfg.channels):
        clean = synthetic_channel(cfg.side, rng)
        noisy = clean + 0.1 * rng.standard_normal(clean.shape)
        chans.append(np.clip(noisy, 0.0, 1.0))
    if cfg.channels == 1:
        return chans[0]
    return np.stack(chans, axis=-1)


def patch_features(img: np.ndarray, k: int) -> np.ndarray:
    """(N, k*k*C) reflect-padded patch features mapped into [-0.2, 0.2]."""
    if img.ndim == 2:
        img = img[:, :, None]
    h, w, c = img.shape
    r = k // 2
    pad = np.pad(img, ((r, r), (r, r), (0, 0)), mode="reflect")
    feats = np.empty((h * w, c * k * k), dtype=np.float64)
    col = 0
    for ch in range(c):
        for dy in range(k):
            for dx in range(k):
                feats[:, col] = pad[dy:dy + h, dx:dx + w, ch].ravel()
                col += 1
    return 0.4 * (feats - 0.5)


def row_windows(n_features: int, size: int = 3) -> list[np.ndarray]:
    """Consecutive feature triples, the remainder as a final short window."""
    return [np.arange(s, min(s + size, n_features))
            for s in range(0, n_features, size)]


def make_problem(name: str):
    """(features (N,D) fp64, windows, f (N,) fp64 raster order)."""
    cfg = CONFIGS[name]
    img = noisy_image(cfg)
    feats = patch_features(img, cfg.patch)
    wins = row_windows(feats.shape[1])
    f = img.reshape(cfg.n, -1)
    return feats, wins, np.ascontiguousarray(f)


def random_vector(n: int, seed: int = 1234, nrhs: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((nrhs, n)) if nrhs > 1 else rng.standard_normal(n)
    return v


def alpha_sweep(mean_eta: float, count: int) -> np.ndarray:
    """config 4: count alphas log-spaced over [1, 100] / mean(eta)."""
    return np.logspace(0.0, 2.0, count) / mean_eta
