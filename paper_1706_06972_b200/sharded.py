"""Frequency-sharded multi-GPU online training (both axes).

One process per GPU.  Two independent axes are split:

* **samples** -- a global mini-batch of G*B samples, rank r codes rows r*B .. r*B+B-1 against
  the replicated working spectrum (as in parallel.DistributedTrainer);
* **frequencies** -- rank r owns rows [u0_r, u1_r) of the (H, W/2+1) half spectrum: its slice
  of the history (S, c), of the Gauss-Jordan inverse / Cholesky factor, and of the dictionary
  ADMM state (D, V, Theta).  History memory and the O(K^3) per-frequency work drop by G.

Per mini-batch there is one bulk exchange and J small all-reduces:

* **A (codes -> frequency owners)**: ``exchange="all_to_all"`` (default) sends each rank the
  code/sample spectra of its frequency rows for every sample of the global batch (all_to_all,
  (G-1)/G * B * (K+1) * nfreq * 2s bytes per rank); the owner folds them in rank order, so its
  slice is bit-identical to a single GPU's.  ``exchange="reduce_scatter"`` is the north_star's
  alternative: every rank accumulates the increment of ALL frequencies from its own samples and
  the increments are summed across ranks (equal in value, (K+1)G/(2B) times the bytes).
* **B (projection, once per dictionary round)**: each rank's share of crop(irfft2(D + Theta))
  over its rows -- K x M float64 partial supports -- is all-reduced (48 KB at K=100, M=121);
  normalisation and the pruned forward DFT back onto the rank's rows are local
  (ocsc_crop_irfft_rows / ocsc_normalize_support / ocsc_support_rfft_rows).
* **C (working spectrum)**: every rank rebuilds the full F(V) for coding from the all-reduced
  support with K pruned forward DFTs -- no collective.

`Comm` abstracts the collectives: `DistComm` (torch.distributed: NCCL on GPUs, gloo in the CPU
tests) and `LocalComm` (world 1).  `ShardedTrainer` with `LocalComm` is the unsharded trainer
computed through the sharded code path, which the single-GPU parity tests exploit.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .dictionary import HistoryState
from .training import OnlineTrainer, TrainConfig, _HalfHistory
from .transforms import SignalShape


def row_slices(H: int, world: int) -> list[tuple[int, int]]:
    """Contiguous near-equal split of the H spectrum rows (first H % world ranks get one more)."""
    if world < 1:
        raise ValueError("world size must be positive")
    base, extra = divmod(H, world)
    out, u = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((u, u + n))
        u += n
    return out


class Comm:
    world = 1
    rank = 0

    def all_to_all(self, send: torch.Tensor, send_splits: list[int], recv_splits: list[int]) -> torch.Tensor:
        raise NotImplementedError

    def all_reduce_(self, t: torch.Tensor) -> torch.Tensor:
        raise NotImplementedError

    def broadcast_(self, t: torch.Tensor, src: int) -> torch.Tensor:
        raise NotImplementedError


class LocalComm(Comm):
    """World of one: every collective is the identity."""

    def all_to_all(self, send, send_splits, recv_splits):
        return send

    def all_reduce_(self, t):
        return t

    def broadcast_(self, t, src):
        return t


class DistComm(Comm):
    """torch.distributed process group: NCCL on GPUs (device tensors, NVLink); a gloo group
    (the multi-process tests) stages device tensors through host memory."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.host = dist.get_backend(group) == "gloo"

    def _run(self, fn, *tensors):
        if not self.host or all(not t.is_cuda for t in tensors):
            fn(*tensors)
            return tensors
        staged = [t.cpu() for t in tensors]
        fn(*staged)
        for t, h in zip(tensors, staged):
            t.copy_(h)
        return tensors

    def all_to_all(self, send, send_splits, recv_splits):
        out = torch.empty(sum(recv_splits), dtype=send.dtype, device=send.device)
        self._run(lambda o, i: dist.all_to_all_single(o, i, output_split_sizes=list(recv_splits),
                                                      input_split_sizes=list(send_splits), group=self.group),
                  out, send.contiguous())
        return out

    def all_reduce_(self, t):
        self._run(lambda x: dist.all_reduce(x, group=self.group), t)
        return t

    def broadcast_(self, t, src):
        g = dist.get_global_rank(self.group, src) if self.group is not None else src
        self._run(lambda x: dist.broadcast(x, src=g, group=self.group), t)
        return t


def exchange_codes(uh: torch.Tensor, xh: torch.Tensor, rows: list[tuple[int, int]], comm: Comm):
    """Exchange A (all_to_all): this rank's (B, K, H, Wh) code spectra and (B, H, Wh) sample
    spectra -> every sample of the global batch restricted to this rank's rows, in rank order:
    ((G*B, K, nfl), (G*B, nfl)) with nfl = (u1 - u0) * Wh.  Pure tensor plumbing (CPU or GPU)."""
    B, K, H, Wh = uh.shape
    G, me = comm.world, comm.rank
    parts, splits = [], []
    for (u0, u1) in rows:
        parts.append(uh[:, :, u0:u1].reshape(-1))
        parts.append(xh[:, u0:u1].reshape(-1))
        splits.append(B * (K + 1) * (u1 - u0) * Wh)
    send = torch.cat(parts) if parts else uh.new_empty(0)
    nfl = (rows[me][1] - rows[me][0]) * Wh
    recv = comm.all_to_all(send, splits, [B * (K + 1) * nfl] * G)
    blocks = recv.view(G, B * (K + 1) * nfl)
    z = blocks[:, :B * K * nfl].reshape(G * B, K, nfl)
    x = blocks[:, B * K * nfl:].reshape(G * B, nfl)
    return z.contiguous(), x.contiguous()


class ShardedTrainer(OnlineTrainer):
    """OnlineTrainer with samples AND frequencies sharded over `comm` (see module docstring).

    `partial_fit` takes this rank's B samples of the global mini-batch.  History, factor and
    dictionary-ADMM state exist only for this rank's spectrum rows; `alpha` (the feasible
    filters) and the working spectrum used for coding are replicated.
    """

    def __init__(self, shape: SignalShape, config: TrainConfig, comm: Comm | None = None,
                 exchange: str = "all_to_all"):
        if exchange not in ("all_to_all", "reduce_scatter"):
            raise ValueError(f"unknown exchange {exchange!r}")
        self.comm = comm if comm is not None else LocalComm()
        self.exchange = exchange
        H, W = shape.grid
        self.all_rows = row_slices(H, self.comm.world)
        self.rows = self.all_rows[self.comm.rank]
        self.Whalf = W // 2 + 1
        self.nfl = (self.rows[1] - self.rows[0]) * self.Whalf
        super().__init__(shape, config)
        K, M = self.K, self.M0 * self.M1
        self.Dh_s = torch.zeros((K, self.nfl), dtype=self.cdtype, device=self.dev)
        self.Th_s = torch.zeros_like(self.Dh_s)
        self.Vh_s = torch.zeros_like(self.Dh_s)
        self.apart = torch.zeros((K, M), dtype=torch.float64, device=self.dev)
        self.Dh = None  # the full-plane D exists only as slices

    def _make_history(self, hist_cdtype: torch.dtype) -> HistoryState:
        return _HalfHistory(self.shape, self.K, self.config.rho_dict, nfreq=self.nfl, dtype=hist_cdtype,
                            inv_dtype=self.cdtype, solver=self.config.history_solver)

    # -------------------------------------------------------------- exchange A --
    def _fold(self, uh: torch.Tensor, xh: torch.Tensor, B: int) -> None:
        G = self.comm.world
        uh4 = uh.reshape(B, self.K, self.H, self.Whalf)
        xh3 = xh.reshape(B, self.H, self.Whalf)
        if self.exchange == "all_to_all" or G == 1:
            z, x = exchange_codes(uh4, xh3, self.all_rows, self.comm)
            self.history.accumulate(z, (self.K * self.nfl, self.nfl, 1), x, (self.nfl, 1), G * B)
            return
        # reduce_scatter: increment of every frequency from the local samples, summed over ranks
        full = _HalfHistory(self.shape, self.K, self.config.rho_dict, nfreq=self.nf, dtype=self.history.S.dtype,
                            inv_dtype=self.cdtype, solver="gj" if self.K <= 118 else "chol")
        full.accumulate(uh, (self.K * self.nf, self.nf, 1), xh, (self.nf, 1), B)
        self.comm.all_reduce_(full.S)
        self.comm.all_reduce_(full.c)
        f0, f1 = self.rows[0] * self.Whalf, self.rows[1] * self.Whalf
        self.history.S += full.S[f0:f1]
        self.history.c += full.c[f0:f1]
        self.history.count += G * B

    # ---------------------------------------------------------- exchange B, C --
    def _project_round(self) -> None:
        dt = _lib.code(self.dtype)
        s = _lib.stream()
        u0, u1 = self.rows
        _lib.call("ocsc_crop_irfft_rows", dt, self.H, self.W, self.M0, self.M1, self.K, u0, u1,
                  _lib.ptr(self.Dh_s), _lib.ptr(self.Th_s), _lib.ptr(self.apart), s)
        self.comm.all_reduce_(self.apart)
        _lib.call("ocsc_normalize_support", dt, self.M0 * self.M1, self.K, _lib.ptr(self.apart),
                  _lib.ptr(self.alpha), s)
        _lib.call("ocsc_support_rfft_rows", dt, self.H, self.W, self.M0, self.M1, self.K, u0, u1,
                  _lib.ptr(self.alpha), _lib.ptr(self.Vh_s), _lib.ptr(self.Dh_s), _lib.ptr(self.Th_s), s)

    def _dictionary_update(self) -> None:
        """J rounds of DictOCSC on this rank's rows; one K x M all-reduce per round."""
        J = self.config.inner_iters
        if J == 0:
            return
        u0, u1 = self.rows
        self.Vh_s.copy_(self.Wh[:, u0:u1].reshape(self.K, self.nfl))
        self.Th_s.zero_()
        for _ in range(J):
            self.history.rowsolve(self.Vh_s, self.Th_s, self.nfl, 1, self.Dh_s, check=False)
            self._project_round()
        self._support_rfft(self.alpha, self.Wh)  # exchange C: local, from the replicated support
        _lib.call("ocsc_code_den", _lib.code(self.dtype), self.K, self.nf, _lib.ptr(self.Wh),
                  self.coding_config.rho, _lib.ptr(self.den), _lib.stream())

    def _set_changes(self, m: np.ndarray, B: int) -> None:
        # the reference compares the LAST sample of the batch: it lives on the last rank
        G = self.comm.world
        t = torch.as_tensor(m, dtype=torch.float64, device=self.dev)
        self.comm.broadcast_(t, G - 1)
        super()._set_changes(t.cpu().numpy(), B * G)

    def final_filters(self) -> np.ndarray:
        """crop(F^-1(D)) (training.py:165-169), assembled from the rank slices by all-reduce."""
        u0, u1 = self.rows
        _lib.call("ocsc_crop_irfft_rows", _lib.code(self.dtype), self.H, self.W, self.M0, self.M1, self.K, u0, u1,
                  _lib.ptr(self.Dh_s), None, _lib.ptr(self.apart), _lib.stream())
        self.comm.all_reduce_(self.apart)
        return self.apart.to(self.dtype).double().T.cpu().numpy()

    def dict_state(self):
        raise NotImplementedError("the sharded trainer holds D only as frequency slices; use final_filters()")
