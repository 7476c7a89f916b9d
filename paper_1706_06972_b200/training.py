"""Online training driver -- drop-in for the reference training.py, device-resident.

`OnlineTrainer` keeps every piece of learner state on the GPU in the half
spectrum of the real-signal FFT (H x Wh frequencies):

    Wh (K, H, Wh)        working dictionary spectrum F(V) the codes are solved against
    den (H*Wh)           rho_code + sum_k |Wh_k|^2, the rank-one solve denominator
    Dh, Th (K, H, Wh)    dictionary ADMM spectrum and dual
    alpha (K, M)         feasible filters crop(V) (unit ball, support M0 x M1)
    S, c                 history sums, packed per frequency (dictionary.py docstring)

`partial_fit(X)` is one mini-batch of the composed reference semantics
(SURVEY.md 8(c)); with B = 1 it is exactly `OnlineTrainer.step`
(training.py:128-155): code every sample against Wh (cold start), objective,
fold F(U) into the history, J rounds of dictionary ADMM, Wh <- F(V).
"""

from __future__ import annotations

import ctypes
import hashlib
import time
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _lib
from .coding import (CodeBuffers, CodeState, CodingConfig, code_den, code_objectives, infer_codes,
                     infer_codes_stream, stream_supported)
from .dictionary import DictState, HistoryState
from .errors import DivergenceError, ShapeMismatchError
from .transforms import SignalShape, _np, half_to_cols_dev, rfft2_dev

_REAL = {"float32": torch.float32, "float64": torch.float64}
_CPLX = {torch.float32: torch.complex64, torch.float64: torch.complex128}


@dataclass(frozen=True)
class TrainConfig:
    """Training knobs (training.py:39-64) plus the B200 build's mini-batch/precision fields."""

    n_filters: int = 100
    beta: float = 1.0
    rho_code: float = 1.0
    rho_dict: float = 10.0
    inner_iters: int = 10
    max_passes: int = 10
    stop_tol: float = 1e-3
    seed: int = 0
    code_max_iters: int = 300
    code_rel_tol: float = 1e-3
    batch_dict_iters: int = 200
    batch_dict_tol: float = 1e-4
    fista_iters: int = 100
    mode: str = "online"
    # --- B200 build ---
    batch_size: int = 1            # samples per partial_fit mini-batch
    dtype: str = "float64"         # code/dictionary arithmetic: float64 (parity) or float32
    history_dtype: str = "float64" # history sums and Cholesky
    poll: int = 16                 # code-ADMM convergence poll interval (iterations)
    fused: bool = True             # on-chip cluster kernel when the grid has one (else cuFFT path)
    stream: bool = True            # streaming FFT kernels for larger grids that have them (else cuFFT)
    history_solver: str = "auto"   # "gj" explicit inverse (K <= 118/167) | "chol" blocked Cholesky | "auto"
    overlap: bool = True           # fused plan with a tail: invert the history of the main part on a
                                   # side stream while the tail is coded, then a Woodbury refresh

    def coding(self) -> CodingConfig:
        return CodingConfig(beta=self.beta, rho=self.rho_code, max_iters=self.code_max_iters,
                            rel_tol=self.code_rel_tol)


@dataclass
class PassRecord:
    """One training-log row per pass (training.py:67-77)."""

    index: int
    time_s: float
    train_obj: float
    test_obj: float | None
    psnr: float | None
    history_bytes: int
    snapshot_id: str


@dataclass
class TrainReport:
    """Run output (training.py:80-88) plus the per-sample objective trace."""

    config: TrainConfig
    shape: SignalShape
    records: list[PassRecord] = field(default_factory=list)
    filters: np.ndarray | None = None
    stopped_early: bool = False
    objectives: list[float] = field(default_factory=list)
    codes: list[np.ndarray] | None = None


@dataclass
class BatchResult:
    """What one partial_fit returns: per-sample objectives and iteration counts (host)."""

    objectives: np.ndarray
    iterations: np.ndarray
    codes: torch.Tensor | None = None   # device (B, K, H, W) view, valid until the next call


def init_dictionary(shape: SignalShape, n_filters: int, seed: int) -> np.ndarray:
    """Seeded Gaussian (M, K) filters with unit columns (training.py:91-95).

    Drawn on the host with numpy's generator so the start point is bit-identical
    to the reference's for the same seed.
    """
    f = np.random.default_rng(seed).normal(size=(shape.filter_size, n_filters))
    return f / np.linalg.norm(f, axis=0)


def _snapshot_id(filters: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(filters).tobytes()).hexdigest()[:12]


class _HalfHistory(HistoryState):
    """Trainer history over the half spectrum; `cross`/`inv_gram` materialise the full one."""

    def _full_index(self):
        H, W = self.shape.grid
        Wh = W // 2 + 1
        u, v = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
        stored = v < Wh
        uu = np.where(stored, u, (H - u) % H)
        vv = np.where(stored, v, W - v)
        return (uu * Wh + vv).ravel(), ~stored.ravel()

    def _extend(self, half: torch.Tensor) -> torch.Tensor:
        idx, conj = self._full_index()
        full = half[torch.as_tensor(idx, device=half.device)]
        mask = torch.as_tensor(conj, device=half.device).reshape((-1,) + (1,) * (full.dim() - 1))
        return torch.where(mask, full.conj(), full)

    @property
    def cross(self) -> np.ndarray:
        if self.count == 0:
            return np.zeros((self.shape.size, self.K), dtype=np.complex128)
        return _np(self._extend(self.c / self.count)).astype(np.complex128)

    def gram(self) -> np.ndarray:
        """Averaged Gram over all P frequencies (the half spectrum's mirror is its conjugate)."""
        return _np(self._extend(self._gram_dev())).astype(np.complex128)

    @property
    def inv_gram(self) -> np.ndarray:
        if self.count == 0:
            return np.zeros((self.shape.size, self.K, self.K), dtype=np.complex128)
        return _np(self._extend(self._inv_gram_dev())).astype(np.complex128)


class OnlineTrainer:
    """Streaming trainer (training.py:102-169); `step` = one sample, `partial_fit` = one mini-batch."""

    def __init__(self, shape: SignalShape, config: TrainConfig):
        self.shape = shape
        self.config = config
        self.coding_config = config.coding()
        if config.dtype not in _REAL or config.history_dtype not in _REAL:
            raise ValueError("dtype/history_dtype must be 'float32' or 'float64'")
        self.dtype = _REAL[config.dtype]
        self.cdtype = _CPLX[self.dtype]
        hist_cdtype = _CPLX[_REAL[config.history_dtype]]
        if self.dtype == torch.float64 and hist_cdtype == torch.complex64:
            raise ValueError("history_dtype must be at least as wide as dtype")
        self.dev = _lib.device()
        H, W = shape.grid
        self.H, self.W = H, W
        self.M0, self.M1 = shape.support
        self.K = K = config.n_filters
        self.nf = shape.half_size
        filters = init_dictionary(shape, K, config.seed)
        self.initial_filters = filters
        self.alpha = torch.as_tensor(filters.T.copy(), dtype=self.dtype).to(self.dev)        # (K, M)
        self.Wh = torch.empty((K, H, W // 2 + 1), dtype=self.cdtype, device=self.dev)
        self._support_rfft(self.alpha, self.Wh)
        self.Dh = self.Wh.clone()
        self.Th = torch.zeros_like(self.Wh)
        self.den = code_den(self.Wh, self.coding_config.rho)
        self.history = self._make_history(hist_cdtype)
        self.rng = np.random.default_rng(config.seed)
        self._prev_code = None
        self._prev_alpha = self.alpha.clone()
        self._metrics = torch.zeros(4, dtype=torch.float64, device=self.dev)
        self.code_change = np.inf
        self.dict_change = np.inf
        self.last_objective = np.nan
        self._buf = None
        self._uh = None
        self._x = None
        self._obj = None
        self._fused_ok = {}
        # the reference's per-sample `step` path (B = 1, want_z): buffers, cuFFT plans and the
        # code ADMM's iteration graph (ocsc_code_admm captures it on the second use of an argument
        # set) made here, so the first steps do not pay one-time setup
        if config.batch_size == 1:
            buf = self._buffers(1, want_z=True)
            _lib.call("ocsc_fft_prepare", _lib.code(self.dtype), self.H, self.W, self.K)
            _lib.call("ocsc_fft_prepare", _lib.code(self.dtype), self.H, self.W, 1)
            self._xh[:1].zero_()  # a zero sample converges at iteration 1; the run is scratch only
            infer_codes(self._xh[:1], self.Wh, self.den, shape, self.coding_config, buf, 1,
                        max_iters=max(2 * config.poll, 1), poll=config.poll)
        self._side = None          # side stream + scratch of the overlapped history inverse
        self._tl = None            # dev aid: list collecting (label, timing event) of the overlap
        self.last_path = None      # device path of the last partial_fit (see partial_fit)

    # ---------------------------------------------------------- internals --
    def _make_history(self, hist_cdtype: torch.dtype) -> HistoryState:
        # the inverse the J row solves re-read is stored at the arithmetic precision
        return _HalfHistory(self.shape, self.K, self.config.rho_dict, nfreq=self.nf, dtype=hist_cdtype,
                            inv_dtype=self.cdtype, solver=self.config.history_solver)

    def _support_rfft(self, alpha: torch.Tensor, out: torch.Tensor) -> None:
        _lib.call("ocsc_support_rfft", _lib.code(self.dtype), self.H, self.W, self.M0, self.M1, self.K,
                  _lib.ptr(alpha), _lib.ptr(out), _lib.stream())

    def _buffers(self, B: int, want_z: bool) -> CodeBuffers:
        if self._buf is None or self._buf.B < B or (want_z and not self._buf.want_z):
            self._buf = CodeBuffers(self.shape, self.K, B, self.dtype, want_z=want_z)
            self._uh = torch.empty((B, self.K, self.H, self.W // 2 + 1), dtype=self.cdtype, device=self.dev)
            self._x = torch.empty((B, self.H, self.W), dtype=self.dtype, device=self.dev)
            self._xh = torch.empty((B, self.H, self.W // 2 + 1), dtype=self.cdtype, device=self.dev)
            self._obj = torch.empty(B, dtype=torch.float64, device=self.dev)
        return self._buf

    def use_fused(self, B: int) -> bool:
        """True when the on-chip cluster kernel covers this grid/dtype (ocsc_code_fused_cluster)."""
        if not self.config.fused:
            return False
        key = (B,)
        if key not in self._fused_ok:
            self._fused_ok[key] = _lib.load().ocsc_code_fused_cluster(_lib.code(self.dtype), self.H, self.W,
                                                                      self.K, B) > 0
        return self._fused_ok[key]

    def _split_plan(self, B: int) -> int:
        """b_main when the fused plan codes B samples on two cluster shapes (main waves + a tail
        of <= 16 samples) and the history inverse can overlap the tail; 0 otherwise."""
        key = ("split", B)
        if key not in self._fused_ok:
            info = (ctypes.c_int32 * 8)()
            lib = _lib.load()
            lib.ocsc_code_fused_info(_lib.code(self.dtype), self.H, self.W, self.K, B, info)
            b1 = int(info[5])
            h = self.history
            ok = (self.config.overlap and 0 < b1 < B and B - b1 <= 16 and info[6] > 0
                  and type(self)._fold is OnlineTrainer._fold and h.solver == "gj"
                  and h.S.dtype == torch.complex128
                  and lib.ocsc_history_woodbury_smem(self.K, B - b1) <= 227 * 1024)
            self._fused_ok[key] = b1 if ok else 0
        return self._fused_ok[key]

    def _code_fused(self, xh, buf, uh, obj, b0: int, b1: int) -> None:
        """ocsc_code_fused on samples [b0, b1) of the mini-batch (pointer offsets; own plan)."""
        n = b1 - b0
        if n <= 0:
            return
        cc = self.coding_config
        P, nf = self.H * self.W, self.nf
        es, ce = buf.u.element_size(), uh.element_size()
        _lib.call("ocsc_code_fused", _lib.code(self.dtype), self.H, self.W, self.K, n,
                  xh.data_ptr() + b0 * nf * xh.element_size(), _lib.ptr(self.Wh), _lib.ptr(self.den), cc.beta,
                  cc.rho, cc.max_iters, cc.rel_tol, buf.u.data_ptr() + b0 * self.K * P * es, None,
                  uh.data_ptr() + b0 * self.K * nf * ce, obj.data_ptr() + b0 * obj.element_size(), None,
                  buf.iters.data_ptr() + b0 * 4, buf.status.data_ptr() + b0 * 4, _lib.stream())

    def _mark(self, label: str) -> None:
        if self._tl is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self._tl.append((label, ev))

    def _side_state(self) -> dict:
        h = self.history
        if self._side is None or self._side["S"].shape != h.S.shape:
            self._side = {"stream": torch.cuda.Stream(device=self.dev),
                          "hi": torch.cuda.Stream(device=self.dev, priority=-8),
                          "S": torch.empty_like(h.S), "c": torch.empty_like(h.c), "inv": torch.empty_like(h.S),
                          "info": torch.zeros(2, dtype=torch.int32, device=self.dev)}
        return self._side

    def _prefold_side(self, uh, xh, b1: int, B: int, ready: torch.cuda.Event) -> torch.cuda.Event:
        """Side stream, after `ready`: S' = S + (samples [0, b1)), c' likewise, and the f64 inverse
        of S' + t_final rho P I; the history itself is untouched (a divergence found after the
        tail leaves it as it was)."""
        h, nf, K = self.history, self.nf, self.K
        sd = self._side_state()
        with torch.cuda.stream(sd["stream"]):
            sd["stream"].wait_event(ready)
            self._mark("side start")
            sd["S"].copy_(h.S)
            sd["c"].copy_(h.c)
            _lib.call("ocsc_history_accumulate", _lib.code(uh.dtype), _lib.code(h.S.dtype), K, nf, b1, _lib.ptr(uh),
                      K * nf, nf, 1, _lib.ptr(xh), nf, 1, _lib.ptr(sd["S"]), _lib.ptr(sd["c"]), _lib.stream())
            _lib.call("ocsc_history_invert", _lib.code(h.S.dtype), _lib.code(h.S.dtype), K, nf, _lib.ptr(sd["S"]),
                      (h.count + B) * h.ridge, 1.0, _lib.ptr(sd["inv"]), _lib.ptr(sd["info"]), _lib.stream())
            self._mark("side end")
            done = torch.cuda.Event()
            done.record()
        return done

    def _fold_overlapped(self, uh, xh, b1: int, B: int, side_done: torch.cuda.Event) -> None:
        """Main stream: fold the tail samples into S', Woodbury-refresh the inverse, adopt S'/c'."""
        h, nf, K, sd = self.history, self.nf, self.K, self._side
        torch.cuda.current_stream().wait_event(side_done)
        self._mark("fold start")
        nb = B - b1
        ce = uh.element_size()
        if h._inv is None:
            h._inv = torch.empty(h.S.shape, dtype=h.inv_dtype, device=h.S.device)
        # one pass: Woodbury refresh of the inverse with the tail samples + their fold into S', c'
        _lib.call("ocsc_history_woodbury", _lib.code(uh.dtype), _lib.code(h.inv_dtype), K, nf, nb, _lib.ptr(sd["inv"]),
                  uh.data_ptr() + b1 * K * nf * ce, K * nf, nf, 1, _lib.ptr(h._inv), _lib.ptr(sd["info"][1:]),
                  xh.data_ptr() + b1 * nf * xh.element_size(), nf, 1, _lib.ptr(sd["S"]), _lib.ptr(sd["c"]),
                  _lib.stream())
        h.S, sd["S"] = sd["S"], h.S
        h.c, sd["c"] = sd["c"], h.c
        h.count += B
        h._inv_count = h.count  # (the hot path's row solves run with check=False, as before)
        self._mark("fold end")
        # (the rest of the step: J row-solve + projection rounds, den)

    def _invert_beside_plan(self, B: int) -> int:
        """CTAs for the history inverse beside the plane-resident stream kernel (0: no overlap).

        The plane kernel occupies one CTA per SM for a fixed set of (sample, filter group) CTAs;
        the remaining SMs run a persistent Gauss-Jordan of S + t_final rho P I during coding, a
        full grid finishes it, and a Woodbury refresh folds the batch in."""
        key = ("beside", B)
        if key not in self._fused_ok:
            lib = _lib.load()
            h = self.history
            ctas = lib.ocsc_code_stream_plane_ctas(_lib.code(self.dtype), self.H, self.W, self.K, B)
            sms = torch.cuda.get_device_properties(self.dev).multi_processor_count
            ok = (self.config.overlap and ctas > 0 and sms - ctas >= 4 and B <= 16 and 32 < self.K <= 100
                  and type(self)._fold is OnlineTrainer._fold and h.solver == "gj"
                  and h.S.dtype == torch.complex128
                  and lib.ocsc_history_woodbury_smem(self.K, B) <= 227 * 1024)
            self._fused_ok[key] = sms - ctas if ok else 0
        return self._fused_ok[key]

    def _invert_beside_coding(self, B: int, ctas: int):
        """Side stream: zero the claim counter, launch `ctas` persistent inverse CTAs on S."""
        h = self.history
        sd = self._side_state()
        if "ctr" not in sd:
            sd["ctr"] = torch.zeros(1, dtype=torch.int32, device=self.dev)
        ready = torch.cuda.Event()
        ready.record()
        with torch.cuda.stream(sd["stream"]):
            sd["stream"].wait_event(ready)
            sd["ctr"].zero_()
            sd["info"].zero_()
            zeroed = torch.cuda.Event()  # both the claim counter and info are zero past this event
            zeroed.record()
            _lib.call("ocsc_history_invert_claim", _lib.code(h.S.dtype), _lib.code(h.S.dtype), self.K, self.nf,
                      _lib.ptr(h.S), (h.count + B) * h.ridge, 1.0, _lib.ptr(sd["inv"]), _lib.ptr(sd["info"]),
                      _lib.ptr(sd["ctr"]), int(ctas), _lib.stream())
            self._mark("side inverse end")
            done = torch.cuda.Event()
            done.record()
        return zeroed, done

    def _finish_inverse(self, B: int, zeroed: torch.cuda.Event) -> None:
        """Main stream, after coding: a full grid claims the frequencies the side CTAs have not."""
        h, sd = self.history, self._side
        torch.cuda.current_stream().wait_event(zeroed)
        _lib.call("ocsc_history_invert_claim", _lib.code(h.S.dtype), _lib.code(h.S.dtype), self.K, self.nf,
                  _lib.ptr(h.S), (h.count + B) * h.ridge, 1.0, _lib.ptr(sd["inv"]), _lib.ptr(sd["info"]),
                  _lib.ptr(sd["ctr"]), int(min(self.nf, 4 * 148)), _lib.stream())

    def _fold_woodbury(self, uh, xh, B: int, side_done: torch.cuda.Event) -> None:
        """Main stream: Woodbury refresh of the inverse with the whole batch + its fold into S, c."""
        h, nf, K, sd = self.history, self.nf, self.K, self._side
        torch.cuda.current_stream().wait_event(side_done)
        if h._inv is None:
            h._inv = torch.empty(h.S.shape, dtype=h.inv_dtype, device=h.S.device)
        _lib.call("ocsc_history_woodbury", _lib.code(uh.dtype), _lib.code(h.inv_dtype), K, nf, B, _lib.ptr(sd["inv"]),
                  _lib.ptr(uh), K * nf, nf, 1, _lib.ptr(h._inv), _lib.ptr(sd["info"][1:]), _lib.ptr(xh), nf, 1,
                  _lib.ptr(h.S), _lib.ptr(h.c), _lib.stream())
        h.count += B
        h._inv_count = h.count

    def _load(self, X) -> tuple[torch.Tensor, int]:
        P = self.shape.size
        if isinstance(X, torch.Tensor):
            if X.numel() % P or X.numel() == 0:
                raise ShapeMismatchError(f"sample has {X.numel()} entries, expected a multiple of {P}")
            B = X.numel() // P
            return X.reshape(B, self.H, self.W), B
        arr = np.asarray(X, dtype=np.float64)
        if arr.size % P or arr.size == 0:
            raise ShapeMismatchError(f"sample has {arr.size} entries, expected {P}")
        B = arr.size // P
        return torch.from_numpy(np.ascontiguousarray(arr.reshape(B, self.H, self.W))), B

    def _dictionary_update(self) -> None:
        """J rounds of DictOCSC (dictionary.py:176-215) on device state; Wh <- F(V)."""
        J = self.config.inner_iters
        if J == 0:
            return
        h = self.history
        dt = _lib.code(self.dtype)
        s = _lib.stream()
        self.Th.zero_()
        for _ in range(J):
            h.rowsolve(self.Wh, self.Th, self.nf, 1, self.Dh, check=False)
            _lib.call("ocsc_dict_project", dt, self.H, self.W, self.M0, self.M1, self.K, _lib.ptr(self.Dh),
                      _lib.ptr(self.Th), _lib.ptr(self.Wh), _lib.ptr(self.alpha), s)
        _lib.call("ocsc_code_den", dt, self.K, self.nf, _lib.ptr(self.Wh), self.coding_config.rho,
                  _lib.ptr(self.den), s)

    # -------------------------------------------------------------- API --
    _collective = False  # True when partial_fit must agree with other ranks after coding

    def _agree(self, B: int, diverged_at: int) -> int:
        """First divergence iteration over all participants (-1: none); one process here."""
        return diverged_at

    def _fold(self, uh: torch.Tensor, xh: torch.Tensor, B: int) -> None:
        """History += this mini-batch (overridden by the distributed trainer)."""
        nf = self.nf
        self.history.accumulate(uh, (self.K * nf, nf, 1), xh, (nf, 1), B)

    def _track_changes(self, last: torch.Tensor) -> None:
        """Device partial sums of code_change / dict_change (training.py:146-154)."""
        self._metrics.zero_()
        if self._prev_code is not None:
            _lib.call("ocsc_norms2", _lib.code(self.dtype), last.numel(), _lib.ptr(last),
                      _lib.ptr(self._prev_code), _lib.ptr(self._metrics), _lib.stream())
            self._prev_code.copy_(last)
        else:
            self._prev_code = last.clone()
        _lib.call("ocsc_norms2", _lib.code(self.dtype), self.alpha.numel(), _lib.ptr(self.alpha),
                  _lib.ptr(self._prev_alpha), _lib.ptr(self._metrics[2:]), _lib.stream())
        self._prev_alpha.copy_(self.alpha)

    def partial_fit(self, X, want_z: bool = False, check: bool = True) -> BatchResult:
        """One mini-batch of B samples (rows of X, each P entries) through the hot path.

        check=True syncs once after coding to raise DivergenceError before the
        history is touched (the reference's order, coding.py:105-106); the
        per-sample objectives/iterations come back to the host at the end.
        """
        xs, B = self._load(X)
        buf = self._buffers(B, want_z)
        x = self._x[:B]
        x.copy_(xs, non_blocking=True)
        # persistent spectrum buffer: the cuFFT path's CUDA graphs are keyed on stable pointers
        xh = rfft2_dev(x, self.shape, out=self._xh[:B])
        uh = self._uh[:B]
        nvtx = torch.cuda.nvtx
        nvtx.range_push("ocsc.code")  # NVTX phase ranges (tracing); no-ops without a profiler
        fused = self.use_fused(B) and not want_z
        stream = not fused and not want_z and self.config.stream and stream_supported(self.shape, self.dtype)
        split = self._split_plan(B) if fused else 0
        # which device path codes this batch (tests assert it): fused cluster kernel (+ the tail
        # split with the overlapped inverse), streaming FFT kernels (+ the inverse beside them), cuFFT
        self.last_path = ("fused+split" if split else "fused") if fused else (
            ("stream+beside" if self._invert_beside_plan(B) else "stream") if stream else "cufft")
        if fused:
            obj = self._obj[:B]
            if split:
                # main waves on the trainer's stream; the tail on a high-priority stream so its
                # clusters are placed before the side stream's history kernels fill the free SMs
                self._mark("main start")
                self._code_fused(xh, buf, uh, obj, 0, split)
                main_done = torch.cuda.Event()
                main_done.record()
                self._mark("main end")
                sd = self._side_state()
                with torch.cuda.stream(sd["hi"]):
                    sd["hi"].wait_event(main_done)
                    self._mark("tail start")
                    self._code_fused(xh, buf, uh, obj, split, B)
                    tail_done = torch.cuda.Event()
                    tail_done.record()
                    self._mark("tail end")
                side_done = self._prefold_side(uh, xh, split, B, main_done)
                torch.cuda.current_stream().wait_event(tail_done)
            else:
                self._mark("code start")
                self._code_fused(xh, buf, uh, obj, 0, B)
                self._mark("code end")
        elif stream:
            pre = self._invert_beside_plan(B)
            if pre:  # the history inverse of S (+ this batch's ridge) runs on the SMs coding leaves idle
                inv_zeroed, side_done = self._invert_beside_coding(B, pre)
            self._mark("code start")
            infer_codes_stream(xh, self.Wh, self.den, self.shape, self.coding_config, buf, B, poll=self.config.poll)
            self._mark("code end")
        else:
            self._mark("code start")
            infer_codes(xh, self.Wh, self.den, self.shape, self.coding_config, buf, B, poll=self.config.poll)
            self._mark("code end")
        pre = self._invert_beside_plan(B) if stream else 0
        if pre:  # finish the inverse on the full grid (the side CTAs keep claiming frequencies)
            self._mark("coded")
            self._finish_inverse(B, inv_zeroed)
            self._mark("inverse finished")
        nvtx.range_pop()
        if check or self._collective:
            it = -1
            if B:
                status = buf.status[:B].cpu()
                if bool((status == 2).any()):
                    it = int(buf.iters[:B][status.to(buf.iters.device) == 2].min().cpu())
            it = self._agree(B, it)  # (sharded trainer: every rank learns every rank's outcome)
            if it >= 0:
                if pre:
                    side_done.synchronize()
                raise DivergenceError(f"code solver diverged at iteration {it}")
        nvtx.range_push("ocsc.fold")
        if not fused:
            obj, _ = code_objectives(xh, self.Wh, buf.u, self.shape, self.config.beta, B, uh)
        if split:
            self._fold_overlapped(uh, xh, split, B, side_done)
        elif pre:
            self._fold_woodbury(uh, xh, B, side_done)
            self._mark("woodbury")
        else:
            self._fold(uh, xh, B)
        nvtx.range_pop()
        nvtx.range_push("ocsc.dictionary")
        self._dictionary_update()
        nvtx.range_pop()
        self._mark("dict end")
        track = self.config.stop_tol > 0
        if track:
            self._track_changes(buf.u[B - 1])
        parts = [obj, buf.iters[:B].double(), self._metrics]
        overlapped = bool(split or pre)
        if overlapped:  # the overlapped inverse's positive-definiteness flags ride on the one sync
            parts.append(self._side["info"].double())
        host = torch.cat(parts).cpu().numpy()
        objectives, iterations = host[:B], host[B:2 * B].astype(np.int64)
        if overlapped and check and bool(np.any(host[2 * B + 4:] != 0)):
            raise DivergenceError("history Gram matrix lost positive definiteness")
        if track:
            self._set_changes(host[2 * B:2 * B + 4], B)
        self.last_objective = float(objectives[-1])
        return BatchResult(objectives=objectives, iterations=iterations, codes=buf.u[:B])

    def _set_changes(self, m: np.ndarray, B: int) -> None:
        if self.history.count > B:
            self.code_change = float(np.sqrt(m[0]) / max(np.sqrt(m[1]), 1e-12))
        self.dict_change = float(np.sqrt(m[2]) / max(np.sqrt(m[3]), 1e-12))

    def step(self, x) -> CodeState:
        """Code one sample, absorb it, refresh the dictionary (training.py:128-155)."""
        arr = np.asarray(x, dtype=np.float64).ravel() if not isinstance(x, torch.Tensor) else x
        n = arr.numel() if isinstance(arr, torch.Tensor) else arr.size
        if n != self.shape.size:
            raise ShapeMismatchError(f"sample has {n} entries, expected {self.shape.size}")
        res = self.partial_fit(arr, want_z=True)
        buf = self._buf
        K, P = self.K, self.shape.size
        u = buf.u[0].reshape(K, P)
        dual = (buf.u[0] - buf.t[0]).reshape(K, P)
        z_freq = half_to_cols_dev(buf.zh[0], self.shape)
        return CodeState(z_freq=_np(z_freq).astype(np.complex128), code=_np(u.T).astype(np.float64),
                         dual=_np(dual.T).astype(np.float64), iterations=int(res.iterations[0]))

    def converged(self) -> bool:
        tol = self.config.stop_tol
        return self.code_change < tol and self.dict_change < tol

    def coding_filters(self) -> np.ndarray:
        """Feasible filters coding uses, (M, K) (training.py:161-163)."""
        return _np(self.alpha.T).astype(np.float64)

    def final_filters(self) -> np.ndarray:
        """crop(F^-1(D)), (M, K) (training.py:165-169)."""
        out = torch.empty_like(self.alpha)
        _lib.call("ocsc_crop_irfft", _lib.code(self.dtype), self.H, self.W, self.M0, self.M1, self.K,
                  _lib.ptr(self.Dh), _lib.ptr(out), _lib.stream())
        return _np(out.T).astype(np.float64)

    # reference attribute views (host copies, full spectra)
    @property
    def working_freq(self) -> np.ndarray:
        return _np(half_to_cols_dev(self.Wh, self.shape)).astype(np.complex128)

    @property
    def dict_state(self) -> DictState:
        H, W = self.shape.grid
        v = torch.zeros((self.K, H, W), dtype=self.dtype, device=self.dev)
        v[:, :self.M0, :self.M1] = self.alpha.reshape(self.K, self.M0, self.M1)
        return DictState(freq=_np(half_to_cols_dev(self.Dh, self.shape)).astype(np.complex128),
                         v=_np(v.reshape(self.K, -1).T).astype(np.float64),
                         dual=_np(half_to_cols_dev(self.Th, self.shape)).astype(np.complex128))


def _evaluate_pass(filters, test_samples, shape, coding, config):
    if test_samples is None:
        return None
    from .evaluate import evaluate_dictionary
    return evaluate_dictionary(filters, test_samples, shape, coding, dtype=config.dtype)


def train_online(samples, shape: SignalShape, config: TrainConfig, test_samples=None,
                 return_codes: bool = False) -> TrainReport:
    """Shuffled passes of mini-batches until both change metrics settle (training.py:178-223)."""
    samples = np.atleast_2d(np.asarray(samples, dtype=np.float64))
    trainer = OnlineTrainer(shape, config)
    report = TrainReport(config=config, shape=shape, codes=[] if return_codes else None)
    if samples.size == 0:
        report.filters = trainer.coding_filters()
        return report
    if samples.shape[1] != shape.size:
        raise ShapeMismatchError(f"samples must be (N, {shape.size}), got {samples.shape}")
    B = max(1, int(config.batch_size))
    train_seconds = 0.0
    for pass_idx in range(1, config.max_passes + 1):
        order = trainer.rng.permutation(samples.shape[0])
        objectives = []
        tic = time.perf_counter()
        stopped = False
        for start in range(0, len(order), B):
            res = trainer.partial_fit(samples[order[start:start + B]])
            objectives.extend(res.objectives.tolist())
            if return_codes:
                report.codes.append(_np(res.codes.reshape(res.codes.shape[0], trainer.K, -1)).transpose(0, 2, 1))
            if trainer.converged():
                stopped = True
                break
        train_seconds += time.perf_counter() - tic
        filters = trainer.final_filters()
        result = _evaluate_pass(trainer.coding_filters(), test_samples, shape, config.coding(), config)
        report.objectives.extend(objectives)
        report.records.append(PassRecord(
            index=pass_idx, time_s=train_seconds, train_obj=float(np.mean(objectives)),
            test_obj=None if result is None else result.test_objective,
            psnr=None if result is None else result.psnr,
            history_bytes=trainer.history.nbytes, snapshot_id=_snapshot_id(filters)))
        if stopped:
            report.stopped_early = True
            break
    report.filters = trainer.final_filters()
    return report


def fit(samples, shape: SignalShape, config: TrainConfig, test_samples=None, return_codes: bool = False
        ) -> TrainReport:
    """North-star name for `train_online`: filters, objective trace and (optionally) codes."""
    return train_online(samples, shape, config, test_samples, return_codes=return_codes)


def _dictionary_to_tolerance(tr: OnlineTrainer, iters: int, tol: float | None) -> None:
    """update_dictionary(d_prev, h, iters, tol) (dictionary.py:176-215) on trainer device state."""
    h = tr.history
    dt = _lib.code(tr.dtype)
    s = _lib.stream()
    gaps = torch.empty(2 * tr.K, dtype=torch.float64, device=tr.dev)
    tr.Th.zero_()
    for _ in range(iters):
        h.rowsolve(tr.Wh, tr.Th, tr.nf, 1, tr.Dh, check=False)
        _lib.call("ocsc_dict_project", dt, tr.H, tr.W, tr.M0, tr.M1, tr.K, _lib.ptr(tr.Dh), _lib.ptr(tr.Th),
                  _lib.ptr(tr.Wh), _lib.ptr(tr.alpha), s)
        if tol is not None:
            _lib.call("ocsc_dict_gaps", dt, tr.H, tr.W, tr.K, _lib.ptr(tr.Dh), _lib.ptr(tr.Wh), _lib.ptr(gaps), s)
            g = gaps.cpu().numpy().reshape(tr.K, 2)
            if (np.sqrt(g[:, 0]) / np.maximum(np.sqrt(g[:, 1]), 1e-12)).max() < tol:
                break
    _lib.call("ocsc_code_den", dt, tr.K, tr.nf, _lib.ptr(tr.Wh), tr.coding_config.rho, _lib.ptr(tr.den), s)


def train_batch(samples, shape: SignalShape, config: TrainConfig, test_samples=None) -> TrainReport:
    """Batch alternation (training.py:234-305), device-resident.

    Every outer iteration codes the whole corpus at once (warm-started from the previous
    codes, cuFFT code-ADMM path), rebuilds the history from all codes (rank-N accumulation,
    uniform weights: batch_history, dictionary.py:117-131), and runs the dictionary ADMM to
    `batch_dict_tol` (at most `batch_dict_iters` rounds).
    """
    samples = np.atleast_2d(np.asarray(samples, dtype=np.float64))
    filters0 = init_dictionary(shape, config.n_filters, config.seed)
    report = TrainReport(config=config, shape=shape)
    if samples.size == 0:
        report.filters = filters0
        return report
    if samples.shape[1] != shape.size:
        raise ShapeMismatchError(f"samples must be (N, {shape.size}), got {samples.shape}")
    n = samples.shape[0]
    tr = OnlineTrainer(shape, replace(config, batch_size=n, fused=False))
    coding = config.coding()
    buf = tr._buffers(n, False)
    x = tr._x[:n]
    x.copy_(torch.from_numpy(samples.reshape(n, tr.H, tr.W)))
    xh = rfft2_dev(x, shape)
    uh = tr._uh[:n]
    prev_u = None
    prev_filters = tr.alpha.clone()
    hist_cdtype = tr.history.S.dtype
    norms = torch.zeros(2, dtype=torch.float64, device=tr.dev)
    train_seconds = 0.0
    final = tr.final_filters()
    for outer in range(1, config.max_passes + 1):
        tic = time.perf_counter()
        infer_codes(xh, tr.Wh, tr.den, shape, coding, buf, n, warm=outer > 1, poll=config.poll)
        status = buf.status[:n].cpu()
        if bool((status == 2).any()):
            it = int(buf.iters[:n][status.to(buf.iters.device) == 2].min().cpu())
            raise DivergenceError(f"code solver diverged at iteration {it}")
        code_change = 0.0
        if prev_u is not None:
            # per-sample ||u - u_prev||^2 and ||u||^2 into one (n, 2) buffer: one host sync per
            # outer iteration instead of one per sample
            per = torch.zeros((n, 2), dtype=torch.float64, device=tr.dev)
            for b in range(n):
                _lib.call("ocsc_norms2", _lib.code(tr.dtype), buf.u[b].numel(), _lib.ptr(buf.u[b]),
                          _lib.ptr(prev_u[b]), _lib.ptr(per[b]), _lib.stream())
            p2 = per.cpu().numpy()
            changes = np.sqrt(p2[:, 0]) / np.maximum(np.sqrt(p2[:, 1]), 1e-12)
            code_change = float(np.mean(changes))
            prev_u.copy_(buf.u[:n])
        else:
            prev_u = buf.u[:n].clone()
        _lib.call("ocsc_rfft2", _lib.code(tr.dtype), tr.H, tr.W, n * tr.K, _lib.ptr(buf.u), _lib.ptr(uh),
                  _lib.stream())
        tr.history = _HalfHistory(shape, tr.K, config.rho_dict, nfreq=tr.nf, dtype=hist_cdtype,
                                  inv_dtype=tr.cdtype, solver=config.history_solver)
        tr.history.accumulate(uh, (tr.K * tr.nf, tr.nf, 1), xh, (tr.nf, 1), n)
        _dictionary_to_tolerance(tr, config.batch_dict_iters, config.batch_dict_tol)
        train_seconds += time.perf_counter() - tic
        norms.zero_()
        _lib.call("ocsc_norms2", _lib.code(tr.dtype), tr.alpha.numel(), _lib.ptr(tr.alpha), _lib.ptr(prev_filters),
                  _lib.ptr(norms), _lib.stream())
        a2, b2 = norms.cpu().tolist()
        dict_change = np.sqrt(a2) / max(np.sqrt(b2), 1e-12)
        prev_filters.copy_(tr.alpha)
        # objectives of the current codes against the refreshed dictionary (training.py:280-283)
        obj, _ = code_objectives(xh, tr.Wh, buf.u, shape, config.beta, n, torch.empty_like(uh))
        result = _evaluate_pass(tr.coding_filters(), test_samples, shape, coding, config)
        final = tr.final_filters()
        report.records.append(PassRecord(
            index=outer, time_s=train_seconds, train_obj=float(obj.cpu().mean()),
            test_obj=None if result is None else result.test_objective,
            psnr=None if result is None else result.psnr,
            history_bytes=tr.history.nbytes, snapshot_id=_snapshot_id(final)))
        if outer > 1 and code_change < config.stop_tol and dict_change < config.stop_tol:
            report.stopped_early = True
            break
    report.filters = final
    return report


def train(mode: str, samples, shape, config, test_samples=None) -> TrainReport:
    """Mode dispatch (training.py:374-383): online (the hot path) and batch (row f2)."""
    if mode == "online":
        return train_online(samples, shape, replace(config, mode=mode), test_samples)
    if mode == "batch":
        return train_batch(samples, shape, replace(config, mode=mode), test_samples)
    if mode == "fista-dict":
        raise NotImplementedError("training mode 'fista-dict' is a baseline outside the B200 hot path "
                                  "(SURVEY.md 2.1 row 7)")
    raise ValueError(f"unknown training mode: {mode!r}")
