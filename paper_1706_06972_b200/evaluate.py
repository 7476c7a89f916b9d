"""Held-out objective and PSNR (reference evaluate.py:32-76), batched on the device.

SURVEY.md 8(f) row f1: the same code-ADMM kernels as training, no history.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .coding import CodeBuffers, CodingConfig, code_den, code_objectives, infer_codes
from .errors import DivergenceError, ShapeMismatchError
from .transforms import SignalShape, rfft2_dev

PSNR_PEAK_SQ = 255.0 ** 2  # evaluate.py:18


@dataclass
class EvalResult:
    test_objective: float
    psnr: float
    per_image_psnr: list[float] = field(default_factory=list)
    infinite_count: int = 0
    n_images: int = 0


def evaluate_dictionary(filters, samples, shape: SignalShape, coding: CodingConfig = CodingConfig(),
                        dtype: str = "float64", batch: int = 64) -> EvalResult:
    """Code every sample against frozen (M, K) filters; mean objective and PSNR."""
    filters = np.asarray(filters, dtype=np.float64)
    samples = np.atleast_2d(np.asarray(samples, dtype=np.float64))
    if samples.shape[1] != shape.size:
        raise ShapeMismatchError(f"samples must be (N, {shape.size}), got {samples.shape}")
    if filters.ndim != 2 or filters.shape[0] != shape.filter_size:
        # the reference raises here through pad_filter_cols (transforms.py:179-196)
        raise ShapeMismatchError(f"filters must be ({shape.filter_size}, K), got {filters.shape}")
    rdt = torch.float32 if dtype == "float32" else torch.float64
    cdt = torch.complex64 if rdt == torch.float32 else torch.complex128
    dev = _lib.device()
    H, W = shape.grid
    M0, M1 = shape.support
    K = filters.shape[1]
    alpha = torch.as_tensor(filters.T.copy(), dtype=rdt).to(dev)
    Wh = torch.empty((K, H, W // 2 + 1), dtype=cdt, device=dev)
    _lib.call("ocsc_support_rfft", _lib.code(rdt), H, W, M0, M1, K, _lib.ptr(alpha), _lib.ptr(Wh), _lib.stream())
    den = code_den(Wh, coding.rho)
    n = samples.shape[0]
    B = min(batch, n)
    buf = CodeBuffers(shape, K, B, rdt)
    uh = torch.empty((B, K, H, W // 2 + 1), dtype=cdt, device=dev)
    objs, errs = [], []
    for s in range(0, n, B):
        chunk = samples[s:s + B]
        b = chunk.shape[0]
        x = torch.as_tensor(chunk.reshape(b, H, W), dtype=rdt).to(dev)
        xh = rfft2_dev(x, shape)
        infer_codes(xh, Wh, den, shape, coding, buf, b)
        status = buf.status[:b].cpu()
        if bool((status == 2).any()):  # coding.py:105-106, as the reference's infer_code raises
            it = int(buf.iters[:b][status.to(buf.iters.device) == 2].min().cpu())
            raise DivergenceError(f"code solver diverged at iteration {it}")
        obj, resid = code_objectives(xh, Wh, buf.u, shape, coding.beta, b, uh, want_resid=True)
        objs.extend(obj.cpu().tolist())
        errs.extend(resid.cpu().tolist())
    psnrs, infinite = [], 0
    for err in errs:
        if err == 0.0:
            psnrs.append(float("inf"))
            infinite += 1
        else:
            psnrs.append(10.0 * np.log10(PSNR_PEAK_SQ * shape.size / err))
    finite = [p for p in psnrs if np.isfinite(p)]
    if infinite:
        warnings.warn(f"{infinite} perfect reconstruction(s) excluded from the PSNR mean", stacklevel=2)
    return EvalResult(test_objective=float(np.mean(objs)), psnr=float(np.mean(finite)) if finite else float("inf"),
                      per_image_psnr=psnrs, infinite_count=infinite, n_images=n)
