"""Multi-process (gloo, world_size 2) test of the mini-batch sharding + mean (CPU).

The device engine is replaced by a deterministic stand-in whose "gradient" of realization
r is a fixed array; the sharding, accumulate-then-reduce order and the 1/B scaling of
paper_2102_00755_b200.minibatch are the code paths bench.py runs at N > 1 GPUs."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_00755_b200.minibatch import TorchReducer, run_minibatch, shard

SHAPE = (6, 5, 4)


def fake_grad(r):
    rng = np.random.default_rng(1000 + r)
    return rng.standard_normal(SHAPE), float(rng.random())


class FakeEngine:
    def __init__(self):
        self.acc = np.zeros(SHAPE)
        self.loss = 0.0
        self.cur = None

    def set_sources(self, r):
        self.cur = r

    def upload_observed(self, obs):
        pass

    def run_gradient(self, thickness, accumulate=False):
        g, l = fake_grad(self.cur)
        self.acc = (self.acc if accumulate else 0.0) + g
        self.loss = (self.loss if accumulate else 0.0) + l

    def download_gradient(self, scale_div=1.0):
        return self.loss / scale_div, self.acc / scale_div


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
    out[rank] = (n, loss, grad.tolist())
    dist.destroy_process_group()


def test_shard_assignment():
    assert shard(8, 2, 0) == [0, 2, 4, 6] and shard(8, 2, 1) == [1, 3, 5, 7]
    assert sorted(sum((shard(7, 3, r) for r in range(3)), [])) == list(range(7))
    with pytest.raises(ValueError):
        shard(4, 2, 2)


@pytest.mark.parametrize("batch", [2, 8])
def test_two_rank_mean_equals_single_rank_mean(batch):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), batch, out), nprocs=world, join=True)
    want_g = np.mean([fake_grad(r)[0] for r in range(batch)], axis=0)
    want_l = np.mean([fake_grad(r)[1] for r in range(batch)])
    for rank in range(world):
        n, loss, grad = out[rank]
        assert n == len(shard(batch, world, rank))
        np.testing.assert_allclose(np.array(grad), want_g, rtol=1e-12, atol=1e-12)
        assert abs(loss - want_l) < 1e-12
