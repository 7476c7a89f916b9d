"""Seeded synthetic workloads of BASELINE.json's configurations -- host-side input generation.

The paper's corpora (Fruit, City, CIFAR-10, ...) are not available here and are not
reproduced; seeded planted-dictionary images with the configurations' shapes stand in
for them.  This module only generates inputs (numpy, float64); it is used by bench.py,
the tests and the scripts, and never by the compute path.

Generator:
  * ground-truth filters (M, K0) from default_rng(seed) ~ N(0, 1), unit L2 columns;
  * image i draws from default_rng([seed, start + i]): codes N(0,1) * [U(0,1) < density]
    on the unpadded H0 x W0 grid, circular convolution with the filters (the reference's
    transforms.py:137-141 convention: filter taps at the grid origin), plus noise * N(0,1);
  * each image standardised to zero mean / unit variance (BASELINE addition), then
    zero-padded bottom/right to the FFT grid (BASELINE addition, cfg 1 and 3).
"""

from __future__ import annotations

import numpy as np

# BASELINE.json configs 0-3; rho_code = rho_dict = 1 (BASELINE "rho = 1").
CONFIGS = {
    0: dict(n=10, dims0=(100, 100), grid=(100, 100), K0=20, K=100, beta=1.0, B=1, passes=1, dtype="float64"),
    1: dict(n=50_000, dims0=(32, 32), grid=(42, 42), K0=20, K=100, beta=1.0, B=50, passes=1, dtype="float32"),
    2: dict(n=1_000, dims0=(100, 100), grid=(100, 100), K0=20, K=100, beta=1.0, B=10, passes=2, dtype="float32"),
    3: dict(n=2_000, dims0=(256, 256), grid=(266, 266), K0=64, K=256, beta=0.5, B=32, passes=1, dtype="float32"),
}


def _pair(d) -> tuple[int, int]:
    d = tuple(int(v) for v in d)
    return d if len(d) == 2 else (1, d[0])


def synth_images(n: int, dims0, grid, K0: int, filter_dims=(11, 11), seed: int = 0,
                 density: float = 0.01, noise: float = 0.01, start: int = 0) -> np.ndarray:
    """(n, Hg, Wg) float64 planted-dictionary images (module docstring); `start` offsets the
    per-image streams so a long stream can be generated in chunks."""
    H0, W0 = _pair(dims0)
    Hg, Wg = _pair(grid)
    M0, M1 = _pair(filter_dims)
    taps = np.random.default_rng(seed).normal(size=(M0 * M1, K0))
    taps = taps / np.linalg.norm(taps, axis=0)
    planes = np.zeros((K0, H0, W0))
    planes[:, :M0, :M1] = taps.T.reshape(K0, M0, M1)
    spec = np.fft.fft2(planes)                                  # (K0, H0, W0) filter spectra
    out = np.zeros((n, Hg, Wg))
    for j in range(n):
        rng = np.random.default_rng([seed, start + j])
        codes = rng.normal(size=(K0, H0, W0)) * (rng.random(size=(K0, H0, W0)) < density)
        img = np.fft.ifft2((spec * np.fft.fft2(codes)).sum(axis=0)).real
        img = img + noise * rng.normal(size=(H0, W0))
        out[j, :H0, :W0] = (img - img.mean()) / img.std()
    return out
