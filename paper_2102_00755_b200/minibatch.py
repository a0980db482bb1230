"""Mini-batch of source-encoded gradients sharded over GPUs.

Realization r of a mini-batch of B goes to rank r mod W (PAPER.md
§4.5 :307-309), into slot r // W of that rank's engine: each rank computes its
ceil(B/W) complete TR gradients with no intra-gradient communication, then ONE collective
forms the mean (average_estimates). The mean is worker-count independent
(SURVEY §5.8(a)): every rank's slots are all-gathered and the B gradients
are summed in realization order in fp64, then scaled by 1/B once — the same arithmetic for
W = 1 and W = 8, so the results are bit-identical. On GPUs the collective is the engine's
NCCL all-gather over NVLink plus the ordered-sum kernel (ustfwi_gpu_batch_mean); the same
driver runs with a torch.distributed reducer (gloo on CPU) for the multi-process tests.
A rank with no realization (B < W) keeps empty slots and still joins the collective.
"""
from __future__ import annotations

from typing import Callable, List, Protocol

import numpy as np


def shard(batch: int, world: int, rank: int) -> List[int]:
    """Realization indices of `rank`: r = rank, rank + W, ... < batch."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if batch < 1:
        raise ValueError("batch must be >= 1")
    return list(range(rank, batch, world))


def slots_per_rank(batch: int, world: int) -> int:
    return -(-batch // world)


def ordered_mean(gathered: np.ndarray, losses: np.ndarray, batch: int, world: int):
    """The reduction of ustfwi_gpu_batch_mean on the host: gathered [W, slots, ...] fp32,
    losses [W, slots]; realization r at (r % W, r // W); fp64 sum in realization order,
    one multiplication by 1/B, the gradient rounded to fp32."""
    inv_b = 1.0 / batch
    acc = np.zeros(gathered.shape[2:], dtype=np.float64)
    loss = 0.0
    for r in range(batch):
        acc += gathered[r % world, r // world].astype(np.float64)
        loss += float(losses[r % world, r // world])
    return loss * inv_b, (acc * inv_b).astype(np.float32).astype(np.float64)


class Engine(Protocol):
    def set_sources(self, s) -> None: ...
    def upload_observed(self, obs) -> None: ...
    def batch_reserve(self, slots: int) -> None: ...
    def run_gradient_slot(self, thickness: int, slot: int) -> None: ...


class NcclReducer:
    """The engine's NCCL all-gather + ordered fp64 mean (ustfwi_gpu_batch_mean)."""

    def batch_mean(self, engine, batch: int, world: int) -> None:
        engine.batch_mean(batch)


class TorchReducer:
    """torch.distributed all-gather of the engine's slots (gloo on CPU tests), then the same
    ordered mean on the host."""

    def __init__(self, group=None):
        self.group = group
        self.result = None

    def batch_mean(self, engine, batch: int, world: int) -> None:
        import torch
        import torch.distributed as dist
        losses, grads = engine.slot_gradients()
        g = torch.from_numpy(np.ascontiguousarray(grads, dtype=np.float32))
        l = torch.from_numpy(np.ascontiguousarray(losses, dtype=np.float64))
        gg = [torch.empty_like(g) for _ in range(world)]
        ll = [torch.empty_like(l) for _ in range(world)]
        dist.all_gather(gg, g, group=self.group)
        dist.all_gather(ll, l, group=self.group)
        self.result = ordered_mean(np.stack([t.numpy() for t in gg]), np.stack([t.numpy() for t in ll]),
                                   batch, world)


def run_minibatch(engine, encoded_source: Callable[[int], object], observed: Callable[[int], np.ndarray],
                  thickness: int, batch: int, world: int, rank: int, reducer) -> int:
    """Compute this rank's share of the mini-batch into its slots and form the mean over
    ranks. Returns the number of gradients computed locally (0 on an idle rank)."""
    mine = shard(batch, world, rank)
    engine.batch_reserve(slots_per_rank(batch, world))
    for r in mine:
        engine.set_sources(encoded_source(r))
        engine.upload_observed(observed(r))
        engine.run_gradient_slot(thickness, r // world)
    reducer.batch_mean(engine, batch, world)
    return len(mine)
