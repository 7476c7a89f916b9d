"""Image preparation on the device (reference preprocessing.py:1-100).

Same names, defaults and error behaviour as the reference (`PreprocessSpec`, `load_image`,
`grayscale`, `local_contrast_normalize`, `edge_taper`, `preprocess`); the arithmetic runs in
ONE fused CUDA kernel (csrc/preprocess.cu: grayscale -> LCN -> taper, scipy "reflect"
borders, float64).  `preprocess_batch` is the streaming form that feeds the trainer: a stack
of raw images (u8 / f32 / f64, gray or RGB) in, a device tensor (N, H, W) out, with the
per-image taper seeds `spec.seed + index` the reference CLI uses for a corpus (cli.py:116).

Numpy in -> numpy out (drop-in); torch tensors stay on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatchError

_LUMA = np.array([0.299, 0.587, 0.114])  # preprocessing.py:13
LCN, TAPER = 1, 2


@dataclass(frozen=True)
class PreprocessSpec:
    """Parameters of the fixed preprocessing chain (preprocessing.py:16-25)."""

    lcn_window: int = 9
    lcn_sigma: float = 3.0
    lcn_epsilon: float = 1e-4
    taper_size: int = 11
    taper_sigma_range: tuple[float, float] = (1.0, 3.0)
    seed: int = 0


def load_image(path) -> np.ndarray:
    """Read an image file as float64, (H, W) grayscale or (H, W, 3) RGB (preprocessing.py:28-33)."""
    from PIL import Image

    with Image.open(path) as img:
        if img.mode not in ("L", "RGB"):
            img = img.convert("RGB")
        return np.asarray(img, dtype=np.float64)


def gaussian_kernel(size: int, sigma: float) -> np.ndarray:
    """Normalised sampled Gaussian centred at (size-1)/2 (preprocessing.py:46-50); host copy of
    the weights the kernel builds in shared memory, for callers that want to inspect them."""
    xs = np.arange(size) - (size - 1) / 2.0
    kern = np.exp(-0.5 * (xs / sigma) ** 2)
    return kern / kern.sum()


def taper_sigmas(seed0: int, n: int, sigma_range=(1.0, 3.0)) -> np.ndarray:
    """default_rng(seed0 + i).uniform(*sigma_range) for i < n, via the library's host-side
    SeedSequence + PCG64 (bit-identical to numpy; the stream the kernel draws on the device)."""
    out = np.empty(n, dtype=np.float64)
    _lib.call("ocsc_taper_sigmas", int(seed0), int(n), float(sigma_range[0]), float(sigma_range[1]),
              out.ctypes.data if n else None)
    return out


def taper_sigma(spec: PreprocessSpec, seed: int | None = None) -> float:
    """The seeded random taper width of `preprocess` (preprocessing.py:98-99)."""
    return float(taper_sigmas(spec.seed if seed is None else seed, 1, spec.taper_sigma_range)[0])


_DT = {torch.uint8: _lib.U8, torch.float32: _lib.F32, torch.float64: _lib.F64}


def _run(images, flags: int, spec: PreprocessSpec = PreprocessSpec(), sigmas=None, seed0: int = 0,
         out_dtype=torch.float64, batched: bool = False, to_host: bool | None = None):
    numpy_in = not isinstance(images, torch.Tensor)
    t = torch.from_numpy(np.ascontiguousarray(images)) if numpy_in else images
    if t.dtype not in _DT:
        t = t.to(torch.float64)
    if not batched:
        t = t.unsqueeze(0)
    if t.dim() == 3:
        channels = 1
    elif t.dim() == 4 and t.shape[3] == 3:
        channels = 3
    else:
        raise ShapeMismatchError(f"expected (H, W) or (H, W, 3), got {tuple(t.shape[1:])}")
    if seed0 < 0:
        raise ValueError("seeds must be non-negative")
    dev = _lib.device()
    t = t.to(dev).contiguous()
    n, h, w = t.shape[:3]
    out = torch.empty((n, h, w), dtype=out_dtype, device=dev)
    sg = None if sigmas is None else torch.as_tensor(np.asarray(sigmas, dtype=np.float64)).to(dev)
    lo, hi = spec.taper_sigma_range
    _lib.call("ocsc_preprocess", _DT[t.dtype], _lib.code(out_dtype), n, h, w, channels, _lib.ptr(t), flags,
              spec.lcn_window, float(spec.lcn_sigma), float(spec.lcn_epsilon), spec.taper_size, _lib.ptr(sg),
              int(seed0), float(lo), float(hi), _lib.ptr(out), _lib.stream())
    if not batched:
        out = out[0]
    return out.cpu().numpy() if (numpy_in if to_host is None else to_host) else out


def grayscale(image):
    """Luminance-weighted channel mix; grayscale input passes through (preprocessing.py:36-43)."""
    if isinstance(image, torch.Tensor):
        shape = tuple(image.shape)
    else:
        image = np.asarray(image, dtype=np.float64)
        shape = image.shape
    if len(shape) == 2:
        return image
    if len(shape) == 3 and shape[2] == 3:
        return _run(image, 0)
    raise ShapeMismatchError(f"expected (H, W) or (H, W, 3), got {shape}")


def local_contrast_normalize(image, window: int = 9, sigma: float = 3.0, epsilon: float = 1e-4):
    """(x - local mean) / max(local std, epsilon), Gaussian window (preprocessing.py:58-71)."""
    _check_2d(image)
    return _run(image, LCN, PreprocessSpec(lcn_window=window, lcn_sigma=sigma, lcn_epsilon=epsilon))


def edge_taper(image, size: int = 11, sigma: float = 2.0):
    """Blend the border band toward the Gaussian blur, linear ramp of width `size` (:74-89)."""
    _check_2d(image)
    return _run(image, TAPER, PreprocessSpec(taper_size=size), sigmas=[sigma])


def preprocess(image, spec: PreprocessSpec = PreprocessSpec()):
    """Grayscale, then LCN, then the seeded random-sigma edge taper (preprocessing.py:92-100)."""
    return _run(image, LCN | TAPER, spec, seed0=spec.seed)


def preprocess_batch(images, spec: PreprocessSpec = PreprocessSpec(), seeds=None,
                     out_dtype: torch.dtype = torch.float64) -> torch.Tensor:
    """(N, H, W[, 3]) raw images -> device (N, H, W) preprocessed, one kernel launch.

    Image i's taper sigma is default_rng(seeds[i]).uniform(*spec.taper_sigma_range), default
    seeds[i] = spec.seed + i (the reference corpus loader, cli.py:116) -- drawn on the device.
    Output float64 (reference) or float32 (feeds the float32 trainer without another pass).
    """
    n = images.shape[0]
    sigmas = None
    if seeds is not None:
        seeds = list(seeds)
        if len(seeds) != n:
            raise ShapeMismatchError(f"{len(seeds)} seeds for {n} images")
        sigmas = np.array([taper_sigmas(s, 1, spec.taper_sigma_range)[0] for s in seeds])
    return _run(images, LCN | TAPER, spec, sigmas=sigmas, seed0=spec.seed, out_dtype=out_dtype, batched=True,
                to_host=False)


def _check_2d(image):
    shape = tuple(image.shape) if isinstance(image, torch.Tensor) else np.shape(image)
    if len(shape) != 2:
        raise ShapeMismatchError(f"expected a (H, W) image, got {shape}")
