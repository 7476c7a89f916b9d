"""Constant-size history and the ADMM dictionary update -- drop-in for dictionary.py.

State layout (device).  The reference keeps cross = (1/t) sum conj(x) z and the
exact inverse ((1/t) sum z z^H + rho P I)^-1 per frequency, refreshed by an
O(K^3) solve per sample (dictionary.py:73-114).  This build keeps the
un-normalised sums

    S_p = sum z_p z_p^H   (packed lower Hermitian, K(K+1)/2 per frequency)
    c_p = sum conj(x_p) z_p

which a rank-B kernel updates per mini-batch, and rebuilds the regularised
inverse (per-frequency in-place Gauss-Jordan on the HPD matrix, in registers /
shared memory) only when a dictionary update needs it.
The reference's `cross` and `inv_gram` are derived views (c/t and
t (S + t rho P I)^-1), bit-for-bit the same quantities up to rounding.

The API-level HistoryState covers all P frequencies, so arbitrary complex
inputs behave exactly as in the reference; the trainer's device state keeps
only the half spectrum of real signals (see training.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DivergenceError, ShapeMismatchError, UninitializedHistoryError
from .transforms import (
    SignalShape,
    _dev,
    _np,
    dft_cols_dev,
    inverse_cols_dev,
    pad_filter_cols,
)


def _npk(K: int) -> int:
    return K * (K + 1) // 2


class HistoryState:
    """Running frequency-domain summary of all samples seen (dictionary.py:30-54)."""

    # largest K the in-register / shared-memory Gauss-Jordan inverse handles, per history dtype
    GJ_MAX_K = {torch.complex128: 118, torch.complex64: 167}

    def __init__(self, shape: SignalShape, n_filters: int, rho: float, nfreq: int | None = None,
                 dtype: torch.dtype = torch.complex128, inv_dtype: torch.dtype | None = None,
                 solver: str = "auto"):
        self.shape = shape
        self.rho = float(rho)
        self.count = 0
        self.K = int(n_filters)
        self.nfreq = shape.size if nfreq is None else nfreq
        dev = _lib.device()
        self.S = torch.zeros((self.nfreq, _npk(self.K)), dtype=dtype, device=dev)
        self.c = torch.zeros((self.nfreq, self.K), dtype=dtype, device=dev)
        self.inv_dtype = dtype if inv_dtype is None else inv_dtype
        if solver == "auto":
            solver = "gj" if self.K <= self.GJ_MAX_K[dtype] else "chol"
        if solver not in ("gj", "chol"):
            raise ValueError(f"history solver must be 'gj', 'chol' or 'auto', got {solver!r}")
        self.solver = solver      # "gj": explicit packed inverse; "chol": blocked Cholesky factor
        self._inv = None          # packed (S + t rho P I)^-1, valid for count == _inv_count
        self._inv_count = -1
        self._info = torch.zeros(1, dtype=torch.int32, device=dev)

    # -- reference attributes ------------------------------------------------
    @property
    def n_filters(self) -> int:
        return self.K

    @property
    def nbytes(self) -> int:
        """Device bytes of the history (constant in the sample count)."""
        return self.S.numel() * self.S.element_size() + self.c.numel() * self.c.element_size()

    @property
    def ridge(self) -> float:
        return self.rho * self.shape.size

    @property
    def cross(self) -> np.ndarray:
        """(P, K) averaged cross term (1/t) sum conj(x) z."""
        if self.count == 0:
            return np.zeros((self.nfreq, self.K), dtype=np.complex128)
        return _np(self.c / self.count).astype(np.complex128)

    @property
    def inv_gram(self) -> np.ndarray:
        """(P, K, K) exact inverse of (averaged Gram + rho P I)."""
        if self.count == 0:
            return np.zeros((self.nfreq, self.K, self.K), dtype=np.complex128)
        return _np(self._inv_gram_dev()).astype(np.complex128)

    def _inv_gram_dev(self) -> torch.Tensor:
        """t (S + t rho P I)^-1 on the device, full (nfreq, K, K) layout."""
        if self.solver == "gj":
            inv = self.inverse()
            full = torch.empty((self.nfreq, self.K, self.K), dtype=inv.dtype, device=inv.device)
            _lib.call("ocsc_packed_to_full", _lib.code(inv.dtype), self.K, self.nfreq, _lib.ptr(inv),
                      float(self.count), _lib.ptr(full), _lib.stream())
            return full
        # Cholesky path: column j of A^-1 is the row solve of the unit vector e_j with c = 0
        # (conj(d) = L^-H L^-1 (0 + 1 * conj(e_j))), one launch per column
        L = self.factor()
        dt = self.S.dtype
        K, nf = self.K, self.nfreq
        zero_c = torch.zeros((nf, K), dtype=dt, device=self.S.device)
        unit = torch.zeros((nf, K), dtype=dt, device=self.S.device)
        zero_t = torch.zeros_like(unit)
        col = torch.empty_like(unit)
        full = torch.empty((nf, K, K), dtype=dt, device=self.S.device)
        for j in range(K):
            unit.zero_()
            unit[:, j] = 1.0
            _lib.call("ocsc_dict_rowsolve_chol", _lib.code(dt), _lib.code(dt), K, nf, _lib.ptr(L), _lib.ptr(zero_c),
                      1.0, _lib.ptr(unit), _lib.ptr(zero_t), 1, K, _lib.ptr(col), _lib.stream())
            full[:, :, j] = col.conj() * self.count
        return full

    def _gram_dev(self) -> torch.Tensor:
        full = torch.empty((self.nfreq, self.K, self.K), dtype=self.S.dtype, device=self.S.device)
        scale = 1.0 / self.count if self.count else 0.0
        _lib.call("ocsc_packed_to_full", _lib.code(self.S.dtype), self.K, self.nfreq, _lib.ptr(self.S), scale,
                  _lib.ptr(full), _lib.stream())
        return full

    def gram(self) -> np.ndarray:
        """(P, K, K) averaged Gram (1/t) sum z z^H (reconstruct_gram's value, exact)."""
        return _np(self._gram_dev()).astype(np.complex128)

    # -- device operations ---------------------------------------------------
    def accumulate(self, z: torch.Tensor, zs: tuple[int, int, int], x: torch.Tensor, xs: tuple[int, int],
                   B: int) -> None:
        """Rank-B update from strided device spectra; count += B."""
        _lib.call("ocsc_history_accumulate", _lib.code(z.dtype), _lib.code(self.S.dtype), self.K, self.nfreq, B,
                  _lib.ptr(z), zs[0], zs[1], zs[2], _lib.ptr(x), xs[0], xs[1], _lib.ptr(self.S), _lib.ptr(self.c),
                  _lib.stream())
        self.count += B

    def factor(self, check: bool = True) -> torch.Tensor:
        """Full-layout Cholesky factor L of S + t rho P I (large-K path, cached); (nfreq, Kp, Kp)
        with Kp = K rounded up to a multiple of 32 (decoupled ridge * I padding)."""
        if self._inv is None:
            nbytes = _lib.load().ocsc_history_factor_bytes(_lib.code(self.S.dtype), self.K, self.nfreq)
            Kp = -(-self.K // 32) * 32
            self._inv = torch.empty((self.nfreq, Kp, Kp), dtype=self.S.dtype, device=self.S.device)
            assert self._inv.numel() * self._inv.element_size() == nbytes
        if self._inv_count != self.count:
            _lib.call("ocsc_history_factor", _lib.code(self.S.dtype), self.K, self.nfreq, _lib.ptr(self.S),
                      self.count * self.ridge, _lib.ptr(self._inv), _lib.ptr(self._info), _lib.stream())
            self._inv_count = self.count
            if check and int(self._info.cpu()[0]) != 0:
                raise DivergenceError("history Gram matrix lost positive definiteness")
        return self._inv

    def rowsolve(self, vh: torch.Tensor, th: torch.Tensor, sk: int, sp: int, out: torch.Tensor,
                 check: bool = True) -> torch.Tensor:
        """conj(D_p) = (S + t rho P I)^-1 (c_p + t rho P conj(V_p - Theta_p)) into `out` (row solve)."""
        ridge = self.count * self.ridge
        if self.solver == "chol":
            L = self.factor(check)
            _lib.call("ocsc_dict_rowsolve_chol", _lib.code(vh.dtype), _lib.code(self.S.dtype), self.K, self.nfreq,
                      _lib.ptr(L), _lib.ptr(self.c), ridge, _lib.ptr(vh), _lib.ptr(th), sk, sp, _lib.ptr(out),
                      _lib.stream())
        else:
            inv = self.inverse(check)
            _lib.call("ocsc_dict_rowsolve", _lib.code(vh.dtype), _lib.code(self.S.dtype), _lib.code(inv.dtype),
                      self.K, self.nfreq, _lib.ptr(inv), _lib.ptr(self.c), ridge, _lib.ptr(vh), _lib.ptr(th), sk, sp,
                      _lib.ptr(out), _lib.stream())
        return out

    def inverse(self, check: bool = True) -> torch.Tensor:
        """Packed (S + t rho P I)^-1 for the current count (cached)."""
        if self.solver != "gj":
            raise ValueError(f"explicit inverse not available on the blocked Cholesky path (K={self.K})")
        if self._inv is None:
            self._inv = torch.empty(self.S.shape, dtype=self.inv_dtype, device=self.S.device)
        if self._inv_count != self.count:
            _lib.call("ocsc_history_invert", _lib.code(self.S.dtype), _lib.code(self.inv_dtype), self.K, self.nfreq,
                      _lib.ptr(self.S), self.count * self.ridge, 1.0, _lib.ptr(self._inv), _lib.ptr(self._info),
                      _lib.stream())
            self._inv_count = self.count
            if check and int(self._info.cpu()[0]) != 0:
                raise DivergenceError("history Gram matrix lost positive definiteness")
        return self._inv


def empty_history(shape: SignalShape, n_filters: int, rho: float = 10.0) -> HistoryState:
    """History before any sample (dictionary.py:57-66)."""
    return HistoryState(shape, n_filters, rho)


def _nonfinite(t: torch.Tensor) -> bool:
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    reals = torch.view_as_real(t) if t.is_complex() else t
    _lib.call("ocsc_nonfinite", _lib.code(reals.dtype), reals.numel(), _lib.ptr(reals), _lib.ptr(flag), _lib.stream())
    return bool(int(flag.cpu()[0]))


def update_history(h: HistoryState, z_freq, x_freq) -> HistoryState:
    """Fold one (code spectrum, sample spectrum) pair into h, in place (dictionary.py:73-114)."""
    z = np.asarray(z_freq, dtype=np.complex128)
    x = np.asarray(x_freq, dtype=np.complex128).ravel()
    P, K = h.nfreq, h.K
    if z.shape != (P, K):
        raise ShapeMismatchError(f"code spectrum must be ({P}, {K}), got {z.shape}")
    if x.shape != (P,):
        raise ShapeMismatchError(f"sample spectrum must be ({P},), got {x.shape}")
    zd, xd = _dev(z, torch.complex128), _dev(x, torch.complex128)
    if _nonfinite(zd) or _nonfinite(xd):
        raise DivergenceError("non-finite spectrum rejected before history update")
    h.accumulate(zd, (0, 1, K), xd, (0, 1), 1)
    return h


def batch_history(z_freqs, x_freqs, shape: SignalShape, rho: float = 10.0) -> HistoryState:
    """History of a whole corpus at once with uniform weights (dictionary.py:117-131)."""
    z = np.asarray(z_freqs, dtype=np.complex128)
    x = np.asarray(x_freqs, dtype=np.complex128)
    if z.ndim != 3 or x.ndim != 2 or z.shape[:2] != (x.shape[0], shape.size):
        raise ShapeMismatchError("expected (N, P, K) code and (N, P) sample spectra")
    n, P, K = z.shape
    h = HistoryState(shape, K, rho)
    h.accumulate(_dev(z, torch.complex128), (P * K, 1, K), _dev(x, torch.complex128), (P, 1), n)
    return h


def _rowsolve_dev(h: HistoryState, vh: torch.Tensor, th: torch.Tensor, sk: int, sp: int) -> torch.Tensor:
    return h.rowsolve(vh, th, sk, sp, torch.empty_like(vh))


def solve_dict_rows(h: HistoryState, v_freq, dual_freq) -> np.ndarray:
    """Row minimiser (conj(cross) + rho P (v - dual)) . inv_gram (dictionary.py:134-142)."""
    if h.count == 0:
        raise UninitializedHistoryError("row solve requested at t=0")
    v = _dev(np.asarray(v_freq, dtype=np.complex128), torch.complex128)
    d = _dev(np.asarray(dual_freq, dtype=np.complex128), torch.complex128)
    if v.shape != (h.nfreq, h.K) or d.shape != v.shape:
        raise ShapeMismatchError(f"expected ({h.nfreq}, {h.K}) spectra")
    return _np(_rowsolve_dev(h, v, d, 1, h.K))


def _project_dev(freq_cols: torch.Tensor, shape: SignalShape) -> torch.Tensor:
    spatial = inverse_cols_dev(freq_cols, shape)
    H, W = shape.grid
    M0, M1 = shape.support
    out = torch.empty_like(spatial)
    _lib.call("ocsc_crop_normalize_cols", _lib.F64, H, W, M0, M1, spatial.shape[1], _lib.ptr(spatial),
              _lib.ptr(out), _lib.stream())
    return out


def project_filter_cols(freq_cols, shape: SignalShape) -> np.ndarray:
    """Crop to support and scale into the unit ball; spectra in, padded spatial out (dictionary.py:145-154)."""
    arr = np.asarray(freq_cols, dtype=np.complex128)
    if arr.ndim != 2 or arr.shape[0] != shape.size:
        raise ShapeMismatchError(f"expected (P, K) = ({shape.size}, *) columns, got {arr.shape}")
    return _np(_project_dev(_dev(arr, torch.complex128), shape))


@dataclass
class DictState:
    """Dictionary ADMM iterate (dictionary.py:157-163): spectrum, feasible padded copy, dual."""

    freq: np.ndarray
    v: np.ndarray
    dual: np.ndarray


def dict_state_from_filters(filters, shape: SignalShape) -> DictState:
    """Start the iterate from (M, K) spatial filters (dictionary.py:166-173)."""
    padded = pad_filter_cols(filters, shape)
    freq = _np(dft_cols_dev(_dev(padded), shape))
    return DictState(freq=freq, v=padded, dual=np.zeros(padded.shape, dtype=np.complex128))


def update_dictionary(d_prev: DictState, h: HistoryState, iters: int, tol: float | None = None,
                      monitor=None) -> DictState:
    """Inner dictionary ADMM given the history (dictionary.py:176-215), on the device."""
    if h.count == 0:
        raise UninitializedHistoryError("dictionary update requested at t=0")
    if iters == 0:
        return d_prev
    shape = h.shape
    K = h.K
    v = _dev(np.asarray(d_prev.v, dtype=np.float64))
    vh = dft_cols_dev(v, shape)
    th = torch.zeros_like(vh)
    d = _dev(np.asarray(d_prev.freq, dtype=np.complex128), torch.complex128)
    for tau in range(1, iters + 1):
        d = _rowsolve_dev(h, vh, th, 1, K)
        v = _project_dev(d + th, shape)
        vh = dft_cols_dev(v, shape)
        th = th + d - vh
        if monitor is not None:
            monitor(tau, _np(d), _np(v))
        if tol is not None:
            gaps = torch.linalg.vector_norm(d - vh, dim=0)
            scales = torch.clamp(torch.linalg.vector_norm(d, dim=0), min=1e-12)
            if float((gaps / scales).max()) < tol:
                break
    return DictState(freq=_np(d), v=_np(v), dual=_np(th))


def reconstruct_gram(h: HistoryState) -> np.ndarray:
    """Averaged Gram matrices (dictionary.py:218-227); exact here since the sums are stored."""
    return h.gram()


def quadratic_objective(d_freq, gram, cross, size: int) -> float:
    """(1/2P) sum_p d G d^H - (1/P) sum_p Re(d . cross) (dictionary.py:230-240)."""
    dev = _lib.device()
    d = torch.as_tensor(np.asarray(d_freq, dtype=np.complex128), device=dev)
    g = torch.as_tensor(np.asarray(gram, dtype=np.complex128), device=dev)
    c = torch.as_tensor(np.asarray(cross, dtype=np.complex128), device=dev)
    quad = torch.einsum("pj,pjk,pk->", d, g, d.conj()).real
    lin = torch.einsum("pk,pk->", d, c).real
    return float((0.5 * quad - lin) / size)


def dict_objective(d_freq, h: HistoryState) -> float:
    """History data term at a dictionary spectrum (dictionary.py:243-247)."""
    if h.count == 0:
        raise UninitializedHistoryError("objective undefined at t=0")
    return quadratic_objective(d_freq, h.gram(), h.cross, h.shape.size)
