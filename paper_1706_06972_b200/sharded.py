"""Frequency-sharded multi-GPU online training (both axes).

One process per GPU.  Two independent axes are split:

* **samples** -- a global mini-batch of B samples is split into contiguous, possibly ragged
  shards in rank order (`sample_shards`: the first B % G ranks get one more; ranks may hold
  none when B < G); rank r codes its shard against the replicated working spectrum;
* **frequencies** -- rank r owns rows [u0_r, u1_r) of the (H, W/2+1) half spectrum
  (`row_slices`): its slice of the history (S, c), of the Gauss-Jordan inverse / Cholesky
  factor, and of the dictionary ADMM state (D, V, Theta).  History memory and the O(K^3)
  per-frequency work drop by G.

The global mini-batch keeps the reference's semantics (reference
training.py:128-155 per sample): whatever G is, the dictionary is updated once per B samples.

Per mini-batch there is one small agreement, one bulk exchange and J small all-reduces:

* **agreement** (after coding): an all-gather of (shard size, first divergence iteration) per
  rank.  Every rank learns the global batch size and raises the same DivergenceError when any
  rank diverged (coding.py:105-106), instead of one rank raising while the others block in
  the exchange.
* **A (codes -> frequency owners)**: ``exchange="all_to_all"`` (default) sends each rank the
  code/sample spectra of its frequency rows for every sample of the global batch (ragged
  all_to_all, (G-1)/G * B * (K+1) * nfreq * 2s bytes per rank); the owner folds them in global
  sample order, so its slice is bit-identical to a single GPU's.  ``exchange="reduce_scatter"``
  is the north_star's alternative: every rank accumulates the increment of ALL frequencies from
  its own samples into a persistent rank-chunked buffer and one NCCL reduce-scatter
  (``reduce_scatter_tensor`` over the row slices, padded to the largest slice) leaves each rank
  the summed increment of its rows ((K+1)G/(2B) times the all_to_all bytes).
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

import json

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .dictionary import DictState, HistoryState
from .errors import ShapeMismatchError
from .training import BatchResult, OnlineTrainer, TrainConfig, _HalfHistory
from .transforms import SignalShape, half_to_cols_dev


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


def sample_shards(n_global: int, world: int) -> list[slice]:
    """Rows of a global mini-batch owned by each rank: contiguous, rank order, sizes differing by
    at most one (the first n % world ranks get one more; B < world leaves trailing ranks empty)."""
    return [slice(u0, u1) for u0, u1 in row_slices(n_global, world)]


class Comm:
    world = 1
    rank = 0

    def all_to_all(self, send: torch.Tensor, send_splits: list[int], recv_splits: list[int]) -> torch.Tensor:
        raise NotImplementedError

    def all_reduce_(self, t: torch.Tensor) -> torch.Tensor:
        raise NotImplementedError

    def reduce_scatter(self, out: torch.Tensor, inp: torch.Tensor) -> torch.Tensor:
        """out = chunk `rank` of the element-wise sum over ranks of inp (world equal chunks)."""
        raise NotImplementedError

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor) -> torch.Tensor:
        """out = concatenation over ranks (rank order) of inp (equal shapes)."""
        raise NotImplementedError

    def broadcast_(self, t: torch.Tensor, src: int) -> torch.Tensor:
        raise NotImplementedError

    def gather_ints(self, vals: list[int]) -> np.ndarray:
        """(world, len(vals)) int64 table of every rank's vals (a tiny all-gather)."""
        raise NotImplementedError


class LocalComm(Comm):
    """World of one: every collective is the identity."""

    def all_to_all(self, send, send_splits, recv_splits):
        return send

    def all_reduce_(self, t):
        return t

    def reduce_scatter(self, out, inp):
        out.copy_(inp.reshape(out.shape))
        return out

    def all_gather(self, out, inp):
        out.copy_(inp.reshape(out.shape))
        return out

    def broadcast_(self, t, src):
        return t

    def gather_ints(self, vals):
        return np.asarray([vals], dtype=np.int64)


def _real(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t) if t.is_complex() else t


class DistComm(Comm):
    """torch.distributed process group: NCCL on GPUs (device tensors over NVLink / NVSwitch);
    a gloo group (the multi-process CPU tests) stages device tensors through host memory and
    emulates reduce-scatter by all-reduce + slice (gloo has no reduce_scatter)."""

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
                  _real(out), _real(send.contiguous()))
        return out

    def all_reduce_(self, t):
        self._run(lambda x: dist.all_reduce(x, group=self.group), _real(t))
        return t

    def reduce_scatter(self, out, inp):
        if self.host:
            full = inp.clone()
            self.all_reduce_(full)
            out.copy_(full.reshape((self.world,) + tuple(out.shape))[self.rank])
            return out
        dist.reduce_scatter_tensor(_real(out).view(-1), _real(inp.contiguous()).reshape(-1), group=self.group)
        return out

    def all_gather(self, out, inp):
        self._run(lambda o, i: dist.all_gather_into_tensor(o, i, group=self.group), _real(out).view(-1),
                  _real(inp.contiguous()).reshape(-1))
        return out

    def broadcast_(self, t, src):
        g = dist.get_global_rank(self.group, src) if self.group is not None else src
        self._run(lambda x: dist.broadcast(x, src=g, group=self.group), _real(t))
        return t

    def gather_ints(self, vals):
        dev = "cpu" if self.host else torch.device("cuda", torch.cuda.current_device())
        mine = torch.as_tensor(vals, dtype=torch.int64, device=dev)
        out = torch.empty((self.world, len(vals)), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(out.view(-1), mine, group=self.group)
        return out.cpu().numpy()


def exchange_codes(uh: torch.Tensor, xh: torch.Tensor, rows: list[tuple[int, int]], comm: Comm,
                   counts: list[int] | None = None):
    """Exchange A (all_to_all): this rank's (b, K, H, Wh) code spectra and (b, H, Wh) sample
    spectra -> every sample of the global batch restricted to this rank's rows, in rank order
    (= global sample order): ((B, K, nfl), (B, nfl)) with B = sum(counts), nfl = (u1 - u0) * Wh.
    `counts` are the per-rank shard sizes (ragged; default: all equal to b).  Pure tensor
    plumbing (CPU or GPU)."""
    b, K, H, Wh = uh.shape
    G, me = comm.world, comm.rank
    counts = [b] * G if counts is None else [int(c) for c in counts]
    if counts[me] != b:
        raise ShapeMismatchError(f"rank {me} holds {b} samples, the agreed shard size is {counts[me]}")
    parts, splits = [], []
    for (u0, u1) in rows:
        parts.append(uh[:, :, u0:u1].reshape(-1))
        parts.append(xh[:, u0:u1].reshape(-1))
        splits.append(b * (K + 1) * (u1 - u0) * Wh)
    send = torch.cat(parts) if parts else uh.new_empty(0)
    nfl = (rows[me][1] - rows[me][0]) * Wh
    recv = comm.all_to_all(send, splits, [c * (K + 1) * nfl for c in counts])
    zs, xs, o = [], [], 0
    for c in counts:
        zs.append(recv[o:o + c * K * nfl].view(c, K, nfl))
        xs.append(recv[o + c * K * nfl:o + c * (K + 1) * nfl].view(c, nfl))
        o += c * (K + 1) * nfl
    return torch.cat(zs).contiguous(), torch.cat(xs).contiguous()


class ShardedTrainer(OnlineTrainer):
    """OnlineTrainer with samples AND frequencies sharded over `comm` (see module docstring).

    `partial_fit` takes this rank's shard of the global mini-batch (`sample_shards`; an empty
    shard is allowed).  History, factor and dictionary-ADMM state exist only for this rank's
    spectrum rows; `alpha` (the feasible filters) and the working spectrum used for coding are
    replicated.
    """

    _collective = True

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
        self.nfl_max = max(u1 - u0 for u0, u1 in self.all_rows) * self.Whalf
        super().__init__(shape, config)
        K, M = self.K, self.M0 * self.M1
        self.Dh_s = torch.zeros((K, self.nfl), dtype=self.cdtype, device=self.dev)
        self.Th_s = torch.zeros_like(self.Dh_s)
        self.Vh_s = torch.zeros_like(self.Dh_s)
        self.apart = torch.zeros((K, M), dtype=torch.float64, device=self.dev)
        self.Dh = None  # the full-plane D exists only as slices
        self._counts = [0] * self.comm.world
        self._rs = None  # persistent reduce-scatter scratch (exchange="reduce_scatter")

    def _make_history(self, hist_cdtype: torch.dtype) -> HistoryState:
        return _HalfHistory(self.shape, self.K, self.config.rho_dict, nfreq=self.nfl, dtype=hist_cdtype,
                            inv_dtype=self.cdtype, solver=self.config.history_solver)

    # ------------------------------------------------------------- agreement --
    def _agree(self, B: int, diverged_at: int) -> int:
        table = self.comm.gather_ints([B, diverged_at])
        self._counts = [int(v) for v in table[:, 0]]
        bad = table[:, 1][table[:, 1] >= 0]
        return int(bad.min()) if bad.size else -1

    def _load(self, X):
        if isinstance(X, torch.Tensor) and X.numel() == 0 or not isinstance(X, torch.Tensor) and np.size(X) == 0:
            return None, 0
        return super()._load(X)

    def partial_fit(self, X, want_z: bool = False, check: bool = True) -> BatchResult:
        """One global mini-batch; X is this rank's shard (possibly empty)."""
        xs, b = self._load(X)
        if b:
            return super().partial_fit(xs, want_z=want_z, check=check)
        # empty shard (global B < world): take part in every collective of the step
        from .errors import DivergenceError

        it = self._agree(0, -1)
        if it >= 0:
            raise DivergenceError(f"code solver diverged at iteration {it}")
        H, Wh = self.H, self.Whalf
        self._fold(torch.empty((0, self.K, H, Wh), dtype=self.cdtype, device=self.dev),
                   torch.empty((0, H, Wh), dtype=self.cdtype, device=self.dev), 0)
        self._dictionary_update()
        if self.config.stop_tol > 0:
            self._set_changes(np.zeros(4), 0)
        self.last_path = "empty shard"
        return BatchResult(objectives=np.zeros(0), iterations=np.zeros(0, dtype=np.int64), codes=None)

    # -------------------------------------------------------------- exchange A --
    def _fold(self, uh: torch.Tensor, xh: torch.Tensor, B: int) -> None:
        G = self.comm.world
        counts = self._counts if G > 1 else [B]
        B_glob = int(sum(counts))
        uh4 = uh.reshape(B, self.K, self.H, self.Whalf)
        xh3 = xh.reshape(B, self.H, self.Whalf)
        if self.exchange == "all_to_all" or G == 1:
            z, x = exchange_codes(uh4, xh3, self.all_rows, self.comm, counts)
            self.history.accumulate(z, (self.K * self.nfl, self.nfl, 1), x, (self.nfl, 1), B_glob)
            return
        # reduce_scatter: this rank's increment of EVERY rank's rows (chunk q = rank q's slice,
        # padded to the largest slice), one reduce-scatter of the chunks
        npk = self.K * (self.K + 1) // 2
        hdt = self.history.S.dtype
        if self._rs is None:
            self._rs = {"S": torch.empty((G, self.nfl_max, npk), dtype=hdt, device=self.dev),
                        "c": torch.empty((G, self.nfl_max, self.K), dtype=hdt, device=self.dev),
                        "S_out": torch.empty((self.nfl_max, npk), dtype=hdt, device=self.dev),
                        "c_out": torch.empty((self.nfl_max, self.K), dtype=hdt, device=self.dev)}
        rs = self._rs
        rs["S"].zero_()
        rs["c"].zero_()
        nf, Wh = self.nf, self.Whalf
        for q, (u0, u1) in enumerate(self.all_rows):
            n = (u1 - u0) * Wh
            if n == 0 or B == 0:
                continue
            f0 = u0 * Wh
            _lib.call("ocsc_history_accumulate", _lib.code(uh.dtype), _lib.code(hdt), self.K, n, B,
                      uh.data_ptr() + f0 * uh.element_size(), self.K * nf, nf, 1,
                      xh.data_ptr() + f0 * xh.element_size(), nf, 1,
                      _lib.ptr(rs["S"][q]), _lib.ptr(rs["c"][q]), _lib.stream())
        self.comm.reduce_scatter(rs["S_out"], rs["S"])
        self.comm.reduce_scatter(rs["c_out"], rs["c"])
        self.history.S += rs["S_out"][:self.nfl]
        self.history.c += rs["c_out"][:self.nfl]
        self.history.count += B_glob

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
        # the reference compares the LAST sample of the global batch: it lives on the last rank
        # with a non-empty shard
        counts = self._counts if self.comm.world > 1 else [B]
        src = max((r for r, c in enumerate(counts) if c > 0), default=self.comm.world - 1)
        t = torch.as_tensor(np.asarray(m, dtype=np.float64), device=self.dev)
        self.comm.broadcast_(t, src)
        super()._set_changes(t.cpu().numpy(), int(sum(counts)))

    # -------------------------------------------------------- whole-state views --
    def _gather_rows(self, part: torch.Tensor) -> torch.Tensor:
        """(K, nfl) slices of every rank -> the full (K, H, Wh) half spectrum (all-gather of the
        slices padded to the largest one)."""
        G, K = self.comm.world, self.K
        pad = torch.zeros((K, self.nfl_max), dtype=part.dtype, device=part.device)
        pad[:, :self.nfl] = part
        out = torch.empty((G, K, self.nfl_max), dtype=part.dtype, device=part.device)
        self.comm.all_gather(out, pad)
        full = torch.empty((K, self.H, self.Whalf), dtype=part.dtype, device=part.device)
        for q, (u0, u1) in enumerate(self.all_rows):
            full[:, u0:u1] = out[q, :, :(u1 - u0) * self.Whalf].reshape(K, u1 - u0, self.Whalf)
        return full

    def final_filters(self) -> np.ndarray:
        """crop(F^-1(D)) (training.py:165-169), assembled from the rank slices by all-reduce."""
        u0, u1 = self.rows
        _lib.call("ocsc_crop_irfft_rows", _lib.code(self.dtype), self.H, self.W, self.M0, self.M1, self.K, u0, u1,
                  _lib.ptr(self.Dh_s), None, _lib.ptr(self.apart), _lib.stream())
        self.comm.all_reduce_(self.apart)
        return self.apart.to(self.dtype).double().T.cpu().numpy()

    @property
    def dict_state(self) -> DictState:
        """The dictionary ADMM iterate over all frequencies (collective: every rank must call it)."""
        H, W = self.shape.grid
        D = self._gather_rows(self.Dh_s)
        T = self._gather_rows(self.Th_s)
        v = torch.zeros((self.K, H, W), dtype=self.dtype, device=self.dev)
        v[:, :self.M0, :self.M1] = self.alpha.reshape(self.K, self.M0, self.M1)
        return DictState(freq=half_to_cols_dev(D, self.shape).cpu().numpy().astype(np.complex128),
                         v=v.reshape(self.K, -1).T.cpu().numpy().astype(np.float64),
                         dual=half_to_cols_dev(T, self.shape).cpu().numpy().astype(np.complex128))

    # ---------------------------------------------------------------- checkpoint --
    def save_checkpoint(self, path) -> str:
        """This rank's state -> `<path>.rank<r>of<G>.npz` (replicated + this rank's frequency rows)."""
        h = self.history
        arrays = {name: getattr(self, name).detach().cpu().numpy()
                  for name in ("Wh", "den", "alpha", "_prev_alpha", "Dh_s", "Th_s", "Vh_s")}
        arrays["hist_S"] = h.S.detach().cpu().numpy()
        arrays["hist_c"] = h.c.detach().cpu().numpy()
        if self._prev_code is not None:
            arrays["prev_code"] = self._prev_code.detach().cpu().numpy()
        meta = {"config": self.config.__dict__, "dims": self.shape.dims, "filter_dims": self.shape.filter_dims,
                "count": h.count, "code_change": self.code_change, "dict_change": self.dict_change,
                "last_objective": self.last_objective, "rng": self.rng.bit_generator.state,
                "world": self.comm.world, "rank": self.comm.rank, "rows": list(self.rows),
                "exchange": self.exchange}
        out = f"{path}.rank{self.comm.rank}of{self.comm.world}.npz"
        np.savez(out, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8), **arrays)
        return out

    @classmethod
    def load_checkpoint(cls, path, comm: Comm | None = None) -> "ShardedTrainer":
        """Rebuild this rank's trainer from `save_checkpoint(path)` (same world size)."""
        comm = comm if comm is not None else LocalComm()
        z = np.load(f"{path}.rank{comm.rank}of{comm.world}.npz", allow_pickle=False)
        meta = json.loads(bytes(z["meta"]).decode())
        if meta["world"] != comm.world or meta["rank"] != comm.rank:
            raise ShapeMismatchError("checkpoint was written by a different world / rank")
        shape = SignalShape(tuple(meta["dims"]), tuple(meta["filter_dims"]))
        tr = cls(shape, TrainConfig(**meta["config"]), comm, exchange=meta["exchange"])
        for name in ("Wh", "den", "alpha", "_prev_alpha", "Dh_s", "Th_s", "Vh_s"):
            getattr(tr, name).copy_(torch.from_numpy(z[name]))
        h = tr.history
        h.S.copy_(torch.from_numpy(z["hist_S"]))
        h.c.copy_(torch.from_numpy(z["hist_c"]))
        h.count = int(meta["count"])
        h._inv_count = -1
        if "prev_code" in z.files:
            tr._prev_code = torch.from_numpy(z["prev_code"]).to(tr.dev)
        tr.code_change = float(meta["code_change"])
        tr.dict_change = float(meta["dict_change"])
        tr.last_objective = float(meta["last_objective"])
        tr.rng.bit_generator.state = meta["rng"]
        return tr
