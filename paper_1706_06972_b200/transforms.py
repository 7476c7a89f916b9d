"""Geometry and frequency-domain plumbing of the drop-in API (reference transforms.py).

Conventions are the reference's (transforms.py:1-8): a sample crosses the API
as a flat (P,) vector (row-major H x W), columns are (P, K) with K fastest,
the forward DFT is unnormalised and the inverse carries 1/P, filters occupy
the top-left M0 x M1 block of the grid.  Every transform runs on the GPU
through libocsc_b200.so (cuFFT + the library's kernels); numpy arrays in,
numpy arrays out.  Inside the trainer the hot path never uses these
full-spectrum helpers -- it keeps half spectra resident on the device.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import prod

import numpy as np
import torch

from . import _lib
from .errors import NumericalConsistencyError, ShapeMismatchError

RESIDUE_TOL = 1e-8  # transforms.py:21


@dataclass(frozen=True)
class SignalShape:
    """Grid extents `dims` and filter extents `filter_dims` (1-D or 2-D); transforms.py:24-61."""

    dims: tuple[int, ...]
    filter_dims: tuple[int, ...]

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        fdims = tuple(int(d) for d in self.filter_dims)
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "filter_dims", fdims)
        if len(dims) not in (1, 2):
            raise ShapeMismatchError(f"signals must be 1-D or 2-D, got dims={dims}")
        if len(fdims) != len(dims):
            raise ShapeMismatchError(f"filter rank {len(fdims)} does not match signal rank {len(dims)}")
        if min(dims + fdims) <= 0:
            raise ShapeMismatchError("all extents must be positive")
        for f, d in zip(fdims, dims):
            if f > d:
                raise ShapeMismatchError(f"filter extents {fdims} exceed signal extents {dims}")

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def size(self) -> int:
        return prod(self.dims)

    @property
    def filter_size(self) -> int:
        return prod(self.filter_dims)

    # device-side geometry: a 1-D signal is the H = 1 grid
    @property
    def grid(self) -> tuple[int, int]:
        return (1, self.dims[0]) if self.ndim == 1 else self.dims

    @property
    def support(self) -> tuple[int, int]:
        return (1, self.filter_dims[0]) if self.ndim == 1 else self.filter_dims

    @property
    def half_size(self) -> int:
        H, W = self.grid
        return H * (W // 2 + 1)


# ----------------------------------------------------------------- helpers --

def _dev(a, dtype=torch.float64) -> torch.Tensor:
    dev = _lib.device()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(dev)


def _np(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def _signal(a, shape: SignalShape, name="signal") -> np.ndarray:
    arr = np.asarray(a, dtype=np.float64)
    if arr.size != shape.size:
        raise ShapeMismatchError(f"{name} has {arr.size} entries, expected {shape.size} for dims {shape.dims}")
    return arr.reshape(-1)


def _cols(a, shape: SignalShape, dtype, what="columns") -> np.ndarray:
    arr = np.asarray(a, dtype=dtype)
    if arr.ndim != 2 or arr.shape[0] != shape.size:
        raise ShapeMismatchError(f"expected (P, K) = ({shape.size}, *) {what}, got {arr.shape}")
    return arr


def dft_cols_dev(cols: torch.Tensor, shape: SignalShape, inverse: bool = False) -> torch.Tensor:
    """Unnormalised full DFT of device columns (P, K) (real or complex) -> complex (P, K)."""
    H, W = shape.grid
    K = cols.shape[1]
    out = torch.empty((shape.size, K), dtype=torch.complex128, device=cols.device)
    _lib.call("ocsc_dft_cols", _lib.F64, H, W, K, _lib.ptr(cols), int(cols.is_complex()),
              _lib.ptr(out), int(inverse), _lib.stream())
    return out


def inverse_cols_dev(spec: torch.Tensor, shape: SignalShape) -> torch.Tensor:
    """Inverse DFT (1/P) of full-spectrum columns with the residue guard (transforms.py:102-109)."""
    spatial = dft_cols_dev(spec, shape, inverse=True)
    stats = torch.zeros(2, dtype=torch.float64, device=spec.device)
    _lib.call("ocsc_residue_stats", _lib.F64, spec.numel(), _lib.ptr(spatial), _lib.ptr(spec),
              _lib.ptr(stats), _lib.stream())
    P = shape.size
    residue, peak = (float(v) for v in stats.cpu())
    residue /= P
    bound = RESIDUE_TOL * (1.0 + peak)
    if spec.numel() and residue > bound:
        raise NumericalConsistencyError(
            f"imaginary residue {residue:.3e} exceeds bound {bound:.3e}; "
            "input is not the spectrum of a real array")
    out = torch.empty(spec.shape, dtype=torch.float64, device=spec.device)
    _lib.call("ocsc_real_part", _lib.F64, spec.numel(), _lib.ptr(spatial), 1.0 / P, _lib.ptr(out), _lib.stream())
    return out


def half_to_cols_dev(half: torch.Tensor, shape: SignalShape) -> torch.Tensor:
    """(nplanes, H, Wh) half spectra -> (P, nplanes) full columns by Hermitian extension."""
    H, W = shape.grid
    n = half.shape[0]
    out = torch.empty((shape.size, n), dtype=half.dtype, device=half.device)
    _lib.call("ocsc_half_to_cols", _lib.code(half.dtype), H, W, n, _lib.ptr(half), _lib.ptr(out), _lib.stream())
    return out


def cols_to_half_dev(cols: torch.Tensor, shape: SignalShape) -> torch.Tensor:
    H, W = shape.grid
    n = cols.shape[1]
    out = torch.empty((n, H, W // 2 + 1), dtype=cols.dtype, device=cols.device)
    _lib.call("ocsc_cols_to_half", _lib.code(cols.dtype), H, W, n, _lib.ptr(cols), _lib.ptr(out), _lib.stream())
    return out


def hermitian_defect(cols: torch.Tensor, shape: SignalShape) -> tuple[float, float]:
    H, W = shape.grid
    stats = torch.zeros(2, dtype=torch.float64, device=cols.device)
    _lib.call("ocsc_hermitian_defect", _lib.code(cols.dtype), H, W, cols.shape[1], _lib.ptr(cols),
              _lib.ptr(stats), _lib.stream())
    a, b = stats.cpu().tolist()
    return a, b


def rfft2_dev(planes: torch.Tensor, shape: SignalShape, out: torch.Tensor | None = None) -> torch.Tensor:
    """(n, H, W) real -> (n, H, Wh) half spectra (into `out` when given)."""
    H, W = shape.grid
    n = planes.shape[0]
    cdt = torch.complex64 if planes.dtype == torch.float32 else torch.complex128
    if out is None:
        out = torch.empty((n, H, W // 2 + 1), dtype=cdt, device=planes.device)
    _lib.call("ocsc_rfft2", _lib.code(planes.dtype), H, W, n, _lib.ptr(planes), _lib.ptr(out), _lib.stream())
    return out


def irfft2_dev(half: torch.Tensor, shape: SignalShape) -> torch.Tensor:
    """(n, H, Wh) -> (n, H, W) real with 1/P (input is preserved: a scratch copy is transformed)."""
    H, W = shape.grid
    n = half.shape[0]
    rdt = torch.float32 if half.dtype == torch.complex64 else torch.float64
    scratch = half.clone()
    out = torch.empty((n, H, W), dtype=rdt, device=half.device)
    _lib.call("ocsc_irfft2", _lib.code(rdt), H, W, n, _lib.ptr(scratch), _lib.ptr(out), _lib.stream())
    return out


# ------------------------------------------------------------ public API --

def forward_dft(a, shape: SignalShape) -> np.ndarray:
    """Unnormalised DFT of a real (P,) signal -> (P,) complex (transforms.py:82-87)."""
    x = _dev(_signal(a, shape).reshape(shape.size, 1))
    return _np(dft_cols_dev(x, shape)).reshape(shape.size)


def inverse_dft(a_freq, shape: SignalShape) -> np.ndarray:
    """Inverse DFT with 1/P and the residue guard -> (P,) real (transforms.py:90-109)."""
    arr = np.asarray(a_freq, dtype=np.complex128)
    if arr.size != shape.size:
        raise ShapeMismatchError(f"spectrum has {arr.size} entries, expected {shape.size} for dims {shape.dims}")
    spec = _dev(arr.reshape(shape.size, 1), torch.complex128)
    return _np(inverse_cols_dev(spec, shape)).reshape(shape.size)


def forward_dft_cols(cols, shape: SignalShape) -> np.ndarray:
    """(P, K) real -> (P, K) complex (transforms.py:148-158)."""
    arr = _cols(cols, shape, np.float64)
    return _np(dft_cols_dev(_dev(arr), shape))


def inverse_dft_cols(cols_freq, shape: SignalShape) -> np.ndarray:
    """(P, K) complex -> (P, K) real, residue-checked (transforms.py:161-176)."""
    arr = _cols(cols_freq, shape, np.complex128)
    return _np(inverse_cols_dev(_dev(arr, torch.complex128), shape))


def pad_filter(d, shape: SignalShape) -> np.ndarray:
    """(M,) filter -> (P,) zero-padded grid (transforms.py:112-125)."""
    arr = np.asarray(d, dtype=np.float64)
    if arr.size != shape.filter_size:
        raise ShapeMismatchError(f"filter has {arr.size} entries, expected {shape.filter_size}")
    return pad_filter_cols(arr.reshape(-1, 1), shape)[:, 0]


def crop_filter(v, shape: SignalShape) -> np.ndarray:
    """(P,) padded grid -> (M,) leading support (transforms.py:128-134)."""
    arr = _signal(v, shape, name="padded filter")
    return crop_filter_cols(arr.reshape(-1, 1), shape)[:, 0]


def pad_filter_cols(filters, shape: SignalShape) -> np.ndarray:
    """(M, K) -> (P, K) zero-padded (transforms.py:179-196)."""
    arr = np.asarray(filters, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[0] != shape.filter_size:
        raise ShapeMismatchError(f"expected (M, K) = ({shape.filter_size}, *) filters, got {arr.shape}")
    H, W = shape.grid
    M0, M1 = shape.support
    K = arr.shape[1]
    src = _dev(arr).reshape(M0, M1, K)
    out = torch.zeros((H, W, K), dtype=torch.float64, device=src.device)
    out[:M0, :M1, :] = src
    return _np(out.reshape(shape.size, K))


def crop_filter_cols(padded, shape: SignalShape) -> np.ndarray:
    """(P, K) -> (M, K) support copy (transforms.py:199-211)."""
    arr = _cols(padded, shape, np.float64)
    H, W = shape.grid
    M0, M1 = shape.support
    K = arr.shape[1]
    src = _dev(arr).reshape(H, W, K)
    return _np(src[:M0, :M1, :].reshape(M0 * M1, K))


def circular_convolve(d, z, shape: SignalShape) -> np.ndarray:
    """Circular convolution of an (M,) filter with a (P,) signal (transforms.py:137-141):
    both spectra, their product and the inverse stay on the device."""
    pd = _dev(pad_filter(d, shape).reshape(shape.size, 1))
    zs = _dev(_signal(z, shape).reshape(shape.size, 1))
    prod = dft_cols_dev(pd, shape) * dft_cols_dev(zs, shape)
    return _np(inverse_cols_dev(prod, shape)).reshape(shape.size)
