"""Deterministic mini-batch mean through the engine (C ABI): slots, NCCL all-gather and the
realization-ordered fp64 sum (ustfwi_gpu_batch_mean).

Single GPU: the mean over local slots (no communicator) and through a 1-rank NCCL
communicator must both be bit-identical to the host restatement of the same ordered sum
(minibatch.ordered_mean) of the per-realization gradients. With >= 2 visible devices a
2-rank run of the real engine over NCCL must be bit-identical to the 1-rank mean."""
import os
import socket

import numpy as np
import pytest

from paper_2102_00755_b200 import scenario
from paper_2102_00755_b200.engine import GpuEngine, nccl_unique_id
from paper_2102_00755_b200.minibatch import NcclReducer, ordered_mean, run_minibatch

pytestmark = pytest.mark.gpu
BATCH = 3


def _singles(eng, sc, obs, batch):
    out = []
    for r in range(batch):
        eng.set_sources(sc.encoded(r))
        eng.upload_observed(obs)
        eng.run_gradient(8)
        out.append(eng.download_gradient())
    return out


def _host_mean(singles, batch):
    g = np.stack([s[1].astype(np.float32) for s in singles])[None]
    l = np.array([s[0] for s in singles])[None]
    return ordered_mean(g, l, batch, 1)


def test_batch_mean_local_and_nccl_single_rank_bit_identical():
    sc = scenario.config_a(nt=40)
    obs = np.zeros((len(sc.sensors.positions), sc.grid.nt))
    with GpuEngine(sc.grid) as eng:
        eng.set_medium(sc.model)
        eng.set_sensors(sc.sensors)
        n = run_minibatch(eng, lambda r: sc.encoded(r), lambda r: obs, 8, batch=BATCH, world=1, rank=0,
                          reducer=NcclReducer())
        assert n == BATCH
        loss_local, grad_local = eng.download_gradient()
        eng.comm_init(nccl_unique_id(), 1, 0)
        run_minibatch(eng, lambda r: sc.encoded(r), lambda r: obs, 8, batch=BATCH, world=1, rank=0,
                      reducer=NcclReducer())
        loss_nccl, grad_nccl = eng.download_gradient()
        singles = _singles(eng, sc, obs, BATCH)
    want_l, want_g = _host_mean(singles, BATCH)
    assert grad_local.tobytes() == want_g.tobytes()
    assert grad_nccl.tobytes() == want_g.tobytes()
    assert loss_local == loss_nccl
    assert abs(loss_local - want_l) <= 1e-15 * abs(want_l)


def _rank(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    torch.cuda.set_device(rank)
    sc = scenario.config_a(nt=40)
    obs = np.zeros((len(sc.sensors.positions), sc.grid.nt))
    with GpuEngine(sc.grid, device=rank) as eng:
        eng.set_medium(sc.model)
        eng.set_sensors(sc.sensors)
        eng.comm_init(uid[0], world, rank)
        run_minibatch(eng, lambda r: sc.encoded(r), lambda r: obs, 8, BATCH, world, rank, NcclReducer())
        loss, grad = eng.download_gradient()
    out[rank] = (loss, grad.tobytes())
    dist.destroy_process_group()


def test_two_rank_engine_mean_matches_single_rank():
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 visible GPUs")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.Manager().dict()
    mp.spawn(_rank, args=(2, port, out), nprocs=2, join=True)
    sc = scenario.config_a(nt=40)
    obs = np.zeros((len(sc.sensors.positions), sc.grid.nt))
    with GpuEngine(sc.grid) as eng:
        eng.set_medium(sc.model)
        eng.set_sensors(sc.sensors)
        run_minibatch(eng, lambda r: sc.encoded(r), lambda r: obs, 8, BATCH, 1, 0, NcclReducer())
        loss1, grad1 = eng.download_gradient()
    for rank in range(2):
        assert out[rank][1] == grad1.tobytes()
        assert out[rank][0] == loss1
