"""Mini-batch of source-encoded gradients sharded over GPUs.

Realization r of a mini-batch of B goes to rank r mod W (PAPER.md
§4.5 :307-309): each rank computes its B/W complete TR gradients into the engine's
device accumulator (no intra-gradient communication), then ONE collective averages the
accumulators over ranks (average_estimates). On GPUs the collective is
the engine's NCCL all-reduce over NVLink (ustfwi_gpu_allreduce_mean); the same driver runs
with a torch.distributed reducer (gloo on CPU) for the multi-process tests.
"""
from __future__ import annotations

from typing import Callable, List, Protocol

import numpy as np


def shard(batch: int, world: int, rank: int) -> List[int]:
    """Realization indices of `rank`: r = rank, rank + W, ... < batch."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return list(range(rank, batch, world))


class Engine(Protocol):
    def set_sources(self, s) -> None: ...
    def upload_observed(self, obs) -> None: ...
    def run_gradient(self, thickness: int, accumulate: bool = False) -> None: ...
    def download_gradient(self, scale_div: float = 1.0): ...


class Reducer(Protocol):
    def allreduce_mean(self, engine, batch: int) -> None: ...


class NcclReducer:
    """Sum the device accumulators over ranks with the engine's NCCL communicator, / B."""

    def allreduce_mean(self, engine, batch: int) -> None:
        engine.allreduce_mean(batch)


class TorchReducer:
    """torch.distributed all-reduce of the downloaded accumulator (gloo on CPU tests)."""

    def __init__(self, group=None):
        self.group = group
        self.result = None

    def allreduce_mean(self, engine, batch: int) -> None:
        import torch
        import torch.distributed as dist
        loss, grad = engine.download_gradient(1.0)
        t = torch.from_numpy(np.concatenate([grad.ravel(), [loss]]).astype(np.float64))
        dist.all_reduce(t, group=self.group)
        v = t.numpy() / batch
        self.result = (float(v[-1]), v[:-1].reshape(grad.shape))


def run_minibatch(engine, encoded_source: Callable[[int], object], observed: Callable[[int], np.ndarray],
                  thickness: int, batch: int, world: int, rank: int, reducer) -> int:
    """Compute this rank's share of the mini-batch into the accumulator and average over
    ranks. Returns the number of gradients computed locally. A rank with no realization
    contributes zeros (accumulator cleared by a zero-accumulate convention below)."""
    mine = shard(batch, world, rank)
    for k, r in enumerate(mine):
        engine.set_sources(encoded_source(r))
        engine.upload_observed(observed(r))
        engine.run_gradient(thickness, accumulate=k > 0)
    if not mine:
        raise ValueError("batch smaller than world size: a rank would idle")
    reducer.allreduce_mean(engine, batch)
    return len(mine)
