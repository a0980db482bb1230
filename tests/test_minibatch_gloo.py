"""Multi-process (gloo, world_size 2) test of the mini-batch sharding + deterministic mean (CPU).

The device engine is replaced by a stand-in whose "gradient" of realization r is a fixed
fp32 array; the sharding, slot assignment, all-gather and the realization-ordered fp64 mean
of paper_2102_00755_b200.minibatch are the host logic bench.py runs at N > 1 GPUs (there the
all-gather is NCCL's and the ordered sum is ustfwi_gpu_batch_mean's kernel, the same
arithmetic as minibatch.ordered_mean). The W-rank mean must be BIT-identical to the 1-rank
mean, including batches smaller than the world and ragged batches."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_00755_b200.minibatch import TorchReducer, ordered_mean, run_minibatch, shard, slots_per_rank

SHAPE = (6, 5, 4)


def fake_grad(r):
    rng = np.random.default_rng(1000 + r)
    return rng.standard_normal(SHAPE).astype(np.float32), float(rng.random())


class FakeEngine:
    def __init__(self):
        self.slots = None
        self.losses = None
        self.cur = None

    def set_sources(self, r):
        self.cur = r

    def upload_observed(self, obs):
        pass

    def batch_reserve(self, slots):
        self.slots = np.zeros((slots,) + SHAPE, np.float32)
        self.losses = np.zeros(slots)

    def run_gradient_slot(self, thickness, slot):
        g, l = fake_grad(self.cur)
        self.slots[slot] = g
        self.losses[slot] = l

    def slot_gradients(self):
        return self.losses, self.slots


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batch, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = FakeEngine()
    red = TorchReducer()
    n = run_minibatch(eng, lambda r: r, lambda r: None, 8, batch, world, rank, red)
    loss, grad = red.result
    out[rank] = (n, loss, grad.tobytes())
    dist.destroy_process_group()


def single_rank_mean(batch):
    eng = FakeEngine()
    eng.batch_reserve(batch)
    for r in range(batch):
        eng.set_sources(r)
        eng.run_gradient_slot(8, r)
    return ordered_mean(eng.slots[None], eng.losses[None], batch, 1)


def test_shard_assignment():
    assert shard(8, 2, 0) == [0, 2, 4, 6] and shard(8, 2, 1) == [1, 3, 5, 7]
    assert sorted(sum((shard(7, 3, r) for r in range(3)), [])) == list(range(7))
    assert shard(1, 2, 1) == [] and slots_per_rank(1, 2) == 1 and slots_per_rank(7, 3) == 3
    with pytest.raises(ValueError):
        shard(4, 2, 2)
    with pytest.raises(ValueError):
        shard(0, 2, 0)


@pytest.mark.parametrize("batch", [1, 3, 8])
def test_two_rank_mean_is_bit_identical_to_single_rank(batch):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), batch, out), nprocs=world, join=True)
    want_l, want_g = single_rank_mean(batch)
    # and the plain mean within fp32 rounding
    ref = np.mean([fake_grad(r)[0].astype(np.float64) for r in range(batch)], axis=0)
    np.testing.assert_allclose(want_g, ref, rtol=1e-6, atol=1e-7)
    for rank in range(world):
        n, loss, grad = out[rank]
        assert n == len(shard(batch, world, rank))
        assert grad == want_g.tobytes()          # bit-identical across world sizes
        assert loss == want_l
