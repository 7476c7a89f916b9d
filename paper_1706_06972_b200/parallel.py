"""Multi-GPU online training: one process per GPU, samples sharded, dictionary replicated.

SURVEY.md 8(e).  A global mini-batch of G*B samples is split by rank (rank r
owns rows r*B .. r*B+B-1).  Each rank codes its B samples against the shared
working spectrum (no communication: codes are independent per sample).  The
fold needs every sample's code spectrum, so the per-rank spectra F(U) and
F(x) (B*(K+1)*nfreq complex) are all-gathered over NCCL in rank order and
every rank folds the full global batch -- byte-for-byte the same history as a
single GPU fed the G*B batch in the same order -- and runs the (cheap,
O(J*K^2*nfreq)) dictionary ADMM redundantly, so the next working spectrum is
identical everywhere without a second collective.

The all-gather of codes moves (G-1)/G * G*B*K*nfreq*2s bytes per rank per
mini-batch, (K+1)G/(2B) times less than the reduce-scatter of the history
increment the north_star sketches, so it is the
default exchange.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .training import OnlineTrainer, TrainConfig
from .transforms import SignalShape


def shard_rows(n_global: int, rank: int, world: int) -> slice:
    """Rows of a global mini-batch owned by `rank` (equal contiguous shards, rank order)."""
    if n_global % world:
        raise ValueError(f"global mini-batch {n_global} is not divisible by world size {world}")
    b = n_global // world
    return slice(rank * b, (rank + 1) * b)


def gather_rank_ordered(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather equal-shaped per-rank tensors, concatenated along dim 0 in rank order."""
    world = dist.get_world_size(group)
    if world == 1:
        return local
    out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out


class DistributedTrainer(OnlineTrainer):
    """OnlineTrainer over a process group: `partial_fit` takes this rank's shard of the mini-batch."""

    def __init__(self, shape: SignalShape, config: TrainConfig, group=None):
        super().__init__(shape, config)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def _fold(self, uh: torch.Tensor, xh: torch.Tensor, B: int) -> None:
        if self.world == 1:
            return super()._fold(uh, xh, B)
        uh_all = gather_rank_ordered(uh, self.group)
        xh_all = gather_rank_ordered(xh, self.group)
        super()._fold(uh_all, xh_all, B * self.world)

    def _set_changes(self, m: np.ndarray, B: int) -> None:
        # the reference compares the LAST sample of the batch: it lives on the last rank
        t = torch.as_tensor(m, dtype=torch.float64, device=self.dev)
        dist.broadcast(t, src=dist.get_global_rank(self.group, self.world - 1) if self.group else self.world - 1,
                       group=self.group)
        super()._set_changes(t.cpu().numpy(), B * self.world)

    def gather_objectives(self, local: np.ndarray) -> np.ndarray:
        """Objective trace of the whole global mini-batch (rank order) on every rank."""
        t = torch.as_tensor(np.asarray(local, dtype=np.float64), device=self.dev)
        return gather_rank_ordered(t, self.group).cpu().numpy()
