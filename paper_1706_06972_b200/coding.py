"""Sparse coding against a fixed dictionary -- drop-in for the reference coding.py.

The per-sample ADMM (coding.py:67-119) runs on the device through
`ocsc_code_admm`, batched over samples: one cuFFT R2C/C2R pair per iteration
for all (sample, filter) planes, a fused per-frequency residual kernel and a
fused shrink/dual/norm kernel; each sample stops at exactly the reference's
iteration.  `infer_code` keeps the reference signature and return type;
`infer_codes` is the batched device entry the trainer uses.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DivergenceError, NumericalConsistencyError, ShapeMismatchError
from .transforms import (
    RESIDUE_TOL,
    SignalShape,
    _dev,
    _np,
    cols_to_half_dev,
    half_to_cols_dev,
    hermitian_defect,
    irfft2_dev,
    rfft2_dev,
)


@dataclass(frozen=True)
class CodingConfig:
    """Per-sample solver settings (coding.py:25-32)."""

    beta: float = 1.0
    rho: float = 1.0
    max_iters: int = 300
    rel_tol: float = 1e-3


@dataclass
class CodeState:
    """ADMM output (coding.py:35-42): last frequency iterate, sparse code, scaled dual."""

    z_freq: np.ndarray
    code: np.ndarray
    dual: np.ndarray
    iterations: int = 0


def soft_threshold(x, t: float) -> np.ndarray:
    """sign(x) * max(|x| - t, 0), elementwise (coding.py:45-48)."""
    arr = np.asarray(x, dtype=np.float64)
    src = _dev(arr.reshape(-1))
    out = torch.empty_like(src)
    _lib.call("ocsc_soft_threshold", _lib.F64, src.numel(), _lib.ptr(src), float(t), _lib.ptr(out), _lib.stream())
    return _np(out).reshape(arr.shape)


def solve_code_rows(dict_freq, x_freq, target, rho: float) -> np.ndarray:
    """Closed-form per-frequency code solve, all rows (coding.py:51-64)."""
    d = np.asarray(dict_freq, dtype=np.complex128)
    t = np.asarray(target, dtype=np.complex128)
    x = np.asarray(x_freq, dtype=np.complex128).reshape(-1)
    if d.ndim != 2 or t.shape != d.shape or x.shape[0] != d.shape[0]:
        raise ShapeMismatchError(f"rows must be (P, K) with (P,) samples, got {d.shape}, {x.shape}, {t.shape}")
    dd, xd, td = _dev(d, torch.complex128), _dev(x, torch.complex128), _dev(t, torch.complex128)
    out = torch.empty_like(dd)
    _lib.call("ocsc_solve_code_rows", _lib.F64, d.shape[0], d.shape[1], _lib.ptr(dd), _lib.ptr(xd), _lib.ptr(td),
              float(rho), _lib.ptr(out), _lib.stream())
    return _np(out)


# --------------------------------------------------------- device batch API --

class CodeBuffers:
    """Reusable device buffers for batched coding of up to B samples of one geometry."""

    def __init__(self, shape: SignalShape, K: int, B: int, dtype: torch.dtype, want_z: bool = False):
        self.shape, self.K, self.B, self.dtype, self.want_z = shape, K, B, dtype, want_z
        H, W = shape.grid
        dev = _lib.device()
        cdt = torch.complex64 if dtype == torch.float32 else torch.complex128
        self.u = torch.zeros((B, K, H, W), dtype=dtype, device=dev)
        self.t = torch.zeros((B, K, H, W), dtype=dtype, device=dev)
        self.zh = torch.empty((B, K, H, W // 2 + 1), dtype=cdt, device=dev) if want_z else None
        lib = _lib.load()
        nbytes = lib.ocsc_code_workspace_bytes(_lib.code(dtype), H, W, K, B, int(want_z))
        if lib.ocsc_code_stream_supported(_lib.code(dtype), H, W):
            nbytes = max(nbytes, lib.ocsc_code_stream_workspace_bytes(_lib.code(dtype), H, W, K, B))
        self.work = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
        self.iters = torch.zeros(B, dtype=torch.int32, device=dev)
        self.status = torch.zeros(B, dtype=torch.int32, device=dev)


def code_den(Wh: torch.Tensor, rho: float) -> torch.Tensor:
    """den[p] = rho + sum_k |Wh_k[p]|^2 for a (K, H, Wh) half-spectrum dictionary."""
    K = Wh.shape[0]
    nf = Wh[0].numel()
    rdt = torch.float32 if Wh.dtype == torch.complex64 else torch.float64
    den = torch.empty(nf, dtype=rdt, device=Wh.device)
    _lib.call("ocsc_code_den", _lib.code(rdt), K, nf, _lib.ptr(Wh), float(rho), _lib.ptr(den), _lib.stream())
    return den


def stream_supported(shape: SignalShape, dtype: torch.dtype) -> bool:
    """True when the streaming FFT kernels (csrc/code_stream.cu) cover this grid and dtype."""
    H, W = shape.grid
    return bool(_lib.load().ocsc_code_stream_supported(_lib.code(dtype), H, W))


def infer_codes_stream(xh: torch.Tensor, Wh: torch.Tensor, den: torch.Tensor, shape: SignalShape,
                       config: CodingConfig, buf: CodeBuffers, B: int, poll: int = 16) -> None:
    """Cold-start batched ADMM through the streaming row/column FFT kernels; codes in buf.u."""
    H, W = shape.grid
    _lib.call("ocsc_code_stream", _lib.code(buf.dtype), H, W, buf.K, B, _lib.ptr(xh), _lib.ptr(Wh), _lib.ptr(den),
              float(config.beta), float(config.rho), int(config.max_iters), float(config.rel_tol),
              _lib.ptr(buf.u), _lib.ptr(buf.work), _lib.ptr(buf.iters), _lib.ptr(buf.status), int(poll),
              _lib.stream())


def infer_codes(xh: torch.Tensor, Wh: torch.Tensor, den: torch.Tensor, shape: SignalShape,
                config: CodingConfig, buf: CodeBuffers, B: int, warm: bool = False,
                max_iters: int | None = None, poll: int = 16) -> None:
    """Batched device ADMM on the first B slots of `buf` (u, t zeroed unless warm)."""
    H, W = shape.grid
    if not warm:
        buf.u[:B].zero_()
        buf.t[:B].zero_()
    _lib.call("ocsc_code_admm", _lib.code(buf.dtype), H, W, buf.K, B, _lib.ptr(xh), _lib.ptr(Wh), _lib.ptr(den),
              float(config.beta), float(config.rho), int(config.max_iters if max_iters is None else max_iters),
              float(config.rel_tol), _lib.ptr(buf.u), _lib.ptr(buf.t), _lib.ptr(buf.zh), _lib.ptr(buf.work),
              _lib.ptr(buf.iters), _lib.ptr(buf.status), int(poll), _lib.stream())


def code_objectives(xh: torch.Tensor, Wh: torch.Tensor, u: torch.Tensor, shape: SignalShape, beta: float,
                    B: int, uh: torch.Tensor, want_resid: bool = False):
    """Per-sample objective (coding.py:129-134) of codes u[:B]; fills uh = rfft2(u)."""
    H, W = shape.grid
    K = u.shape[1]
    obj = torch.empty(B, dtype=torch.float64, device=u.device)
    resid = torch.empty(B, dtype=torch.float64, device=u.device) if want_resid else None
    _lib.call("ocsc_code_objective", _lib.code(u.dtype), H, W, K, B, _lib.ptr(xh), _lib.ptr(Wh), _lib.ptr(u),
              float(beta), _lib.ptr(uh), _lib.ptr(obj), _lib.ptr(resid), _lib.stream())
    return obj, resid


# ------------------------------------------------------------- public API --

def _dict_half(dict_freq, shape: SignalShape) -> torch.Tensor:
    """Validate a reference (P, K) dictionary spectrum and return it as (K, H, Wh) on device.

    The reference codes against full complex spectra and would reject (via the
    residue guard, transforms.py:102-109) any iterate that is not the spectrum of
    a real array; a dictionary spectrum that is not Hermitian produces exactly
    such iterates, so it is rejected up front with the same exception.
    """
    d = np.asarray(dict_freq, dtype=np.complex128)
    if d.ndim != 2 or d.shape[0] != shape.size:
        raise ShapeMismatchError(f"dictionary spectrum must be ({shape.size}, K), got {d.shape}")
    dd = _dev(d, torch.complex128)
    defect, peak = hermitian_defect(dd, shape)
    if defect > RESIDUE_TOL * (1.0 + peak):
        raise NumericalConsistencyError(
            f"dictionary spectrum is not Hermitian (defect {defect:.3e}); it is not the spectrum of real filters")
    return cols_to_half_dev(dd, shape)


def infer_code(x, dict_freq, shape: SignalShape, config: CodingConfig = CodingConfig(),
               warm: CodeState | None = None, monitor=None) -> CodeState:
    """ADMM sparse coding of one signal (coding.py:67-119), on the device.

    monitor(iteration, code) is called after each iteration when given (the
    loop then advances one device iteration per call).
    """
    Wh = _dict_half(dict_freq, shape)
    K = Wh.shape[0]
    P = shape.size
    x = np.asarray(x, dtype=np.float64)
    if x.size != P:
        raise ShapeMismatchError(f"signal has {x.size} entries, expected {P} for dims {shape.dims}")
    H, W = shape.grid
    xh = rfft2_dev(_dev(x).reshape(1, H, W), shape)
    den = code_den(Wh, config.rho)
    buf = CodeBuffers(shape, K, 1, torch.float64, want_z=True)
    if warm is not None:
        if warm.code.shape != (P, K):
            raise ShapeMismatchError("warm start does not match (P, K)")
        u0 = np.asarray(warm.code, dtype=np.float64)
        g0 = np.asarray(warm.dual, dtype=np.float64)
        buf.u[0] = _dev(u0.T.reshape(K, H, W))
        buf.t[0] = _dev((u0 - g0).T.reshape(K, H, W))
    buf.zh.zero_()
    iterations = 0
    if monitor is None:
        infer_codes(xh, Wh, den, shape, config, buf, 1, warm=True)
        iterations, status = (int(v) for v in torch.stack([buf.iters[0], buf.status[0]]).cpu())
        if status == 2:
            raise DivergenceError(f"code solver diverged at iteration {iterations}")
    else:
        for it in range(1, config.max_iters + 1):
            infer_codes(xh, Wh, den, shape, config, buf, 1, warm=True, max_iters=1, poll=0)
            status = int(buf.status[0].cpu())
            iterations = it
            if status == 2:
                raise DivergenceError(f"code solver diverged at iteration {it}")
            monitor(it, _np(buf.u[0].reshape(K, P).T))
            if status == 1:
                break
    code = buf.u[0].reshape(K, P).T
    dual = (buf.u[0] - buf.t[0]).reshape(K, P).T
    z_freq = half_to_cols_dev(buf.zh[0], shape)
    return CodeState(z_freq=_np(z_freq), code=_np(code), dual=_np(dual), iterations=iterations)


def reconstruct(dict_freq, code, shape: SignalShape) -> np.ndarray:
    """sum_k d_k (*) code_k as a flat (P,) signal (coding.py:122-126)."""
    Wh = _dict_half(dict_freq, shape)
    K = Wh.shape[0]
    c = np.asarray(code, dtype=np.float64)
    if c.shape != (shape.size, K):
        raise ShapeMismatchError(f"code must be ({shape.size}, {K}), got {c.shape}")
    H, W = shape.grid
    uh = rfft2_dev(_dev(c.T.reshape(K, H, W).copy()), shape)
    out = torch.empty((1, H, W // 2 + 1), dtype=torch.complex128, device=uh.device)
    _lib.call("ocsc_synthesize", _lib.F64, K, shape.half_size, 1, _lib.ptr(Wh), _lib.ptr(uh), _lib.ptr(out),
              _lib.stream())
    return _np(irfft2_dev(out, shape)).reshape(shape.size)


def coding_objective(x, dict_freq, code, shape: SignalShape, beta: float) -> float:
    """0.5 ||x - reconstruction||^2 + beta ||code||_1 (coding.py:129-134)."""
    Wh = _dict_half(dict_freq, shape)
    K = Wh.shape[0]
    c = np.asarray(code, dtype=np.float64)
    if c.shape != (shape.size, K):
        raise ShapeMismatchError(f"code must be ({shape.size}, {K}), got {c.shape}")
    H, W = shape.grid
    xh = rfft2_dev(_dev(np.asarray(x, dtype=np.float64).reshape(1, H, W)), shape)
    u = _dev(c.T.reshape(1, K, H, W).copy())
    uh = torch.empty((1, K, H, W // 2 + 1), dtype=torch.complex128, device=u.device)
    obj, _ = code_objectives(xh, Wh, u, shape, beta, 1, uh)
    return float(obj.cpu()[0])
