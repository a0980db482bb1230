"""Mini-batch mean through the engine's NCCL communicator (C ABI), single rank.

NCCL refuses two ranks on one device, so on a 1-GPU box the collective path is checked
with nranks = 1: after comm_init the all-reduce is the identity sum and the mean divides
by the batch size. The multi-rank sharding/averaging logic is covered by the gloo tests
(tests/test_minibatch_gloo.py); bench.py runs the real N-rank path under torchrun."""
import numpy as np
import pytest

from paper_2102_00755_b200 import scenario
from paper_2102_00755_b200.engine import GpuEngine, nccl_unique_id
from paper_2102_00755_b200.minibatch import NcclReducer, run_minibatch

pytestmark = pytest.mark.gpu


def test_nccl_single_rank_mean_and_minibatch_driver():
    sc = scenario.config_a(nt=40)
    obs = np.zeros((len(sc.sensors.positions), sc.grid.nt))
    with GpuEngine(sc.grid) as eng:
        eng.set_medium(sc.model)
        eng.set_sensors(sc.sensors)
        eng.comm_init(nccl_unique_id(), 1, 0)
        # two realizations accumulated on the device, then the NCCL mean over 1 rank / batch 2
        n = run_minibatch(eng, lambda r: sc.encoded(r), lambda r: obs, 8, batch=2, world=1, rank=0,
                          reducer=NcclReducer())
        assert n == 2
        loss, grad = eng.download_gradient()
        # reference: the same two gradients one by one
        singles = []
        for r in range(2):
            eng.set_sources(sc.encoded(r))
            eng.upload_observed(obs)
            eng.run_gradient(8)
            singles.append(eng.download_gradient())
    want_g = (singles[0][1] + singles[1][1]) / 2
    want_l = (singles[0][0] + singles[1][0]) / 2
    assert np.linalg.norm(grad - want_g) <= 1e-6 * np.linalg.norm(want_g)
    assert abs(loss - want_l) <= 1e-12 * abs(want_l)
