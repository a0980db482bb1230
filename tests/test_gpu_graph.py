"""CUDA-graph replay of the TR gradient (engine.cu gradient_tr): the first call with a
configuration runs eagerly, the second captures the ~9 launches per simulation step into one
graph, later calls replay it. All three must be bit-identical, count the same launches, and
re-binding (set_sources / set_medium) must invalidate the graph."""
import numpy as np
import pytest

from paper_2102_00755_b200 import scenario
from paper_2102_00755_b200.engine import GpuEngine, SourceSet

pytestmark = pytest.mark.gpu


def test_graph_replay_is_bit_identical_to_eager():
    sc = scenario.config_a(nt=96)
    obs = np.zeros((len(sc.sensors.positions), sc.grid.nt))
    with GpuEngine(sc.grid) as eng:
        eng.set_medium(sc.model)
        eng.set_sources(sc.encoded(0))
        eng.set_sensors(sc.sensors)
        eng.upload_observed(obs)
        res, counts = [], []
        for _ in range(4):          # eager, capture + launch, replay, replay
            l0 = eng.launch_count()
            eng.run_gradient(8)
            counts.append(eng.launch_count() - l0)
            res.append(eng.download_gradient())
        for loss, grad in res[1:]:
            assert loss == res[0][0] and grad.tobytes() == res[0][1].tobytes()
        assert len(set(counts)) == 1 and counts[0] > 9 * 96
        # a new source set invalidates the graph: the result follows the new sources (half the
        # amplitude: a quarter of the gradient; note g(w) = g(-w) for a sign flip)
        eng.set_sources(SourceSet(sc.sources.positions, [0.5 * np.asarray(x) for x in sc.sources.signals]))
        eng.upload_observed(obs)
        eng.run_gradient(8)
        l1, g1 = eng.download_gradient()
        eng.run_gradient(8)
        l2, g2 = eng.download_gradient()
    assert g1.tobytes() == g2.tobytes() and l1 == l2
    assert np.linalg.norm(g1 - 0.25 * res[0][1]) <= 1e-5 * np.linalg.norm(g1)


def test_new_c0_values_reuse_the_graph_correctly():
    """An optimizer iterate: set_medium with new c0 values but the same structure (uniform
    rho0, no absorption, same gamma) keeps the captured graph (the c0^2 field is updated in
    place); the result must equal a fresh engine's for the new medium, bit for bit. A new
    uniform rho0 value (baked into the launches as a scalar) must invalidate it."""
    from paper_2102_00755_b200.engine import Medium
    sc = scenario.config_a(nt=96)
    obs = np.zeros((len(sc.sensors.positions), sc.grid.nt))
    m = sc.model
    c0b = np.asarray(m.c0) * (1.0 + 0.01 * np.sin(np.arange(np.asarray(m.c0).size)).reshape(np.shape(m.c0)))
    c0b = np.clip(c0b, m.c0_min, m.c0_max)
    mb = Medium(c0=c0b, rho0=m.rho0, gamma=m.gamma, c0_min=m.c0_min, c0_max=m.c0_max)
    mr = Medium(c0=c0b, rho0=np.asarray(m.rho0) * 1.05, gamma=m.gamma, c0_min=m.c0_min, c0_max=m.c0_max)

    def fresh(medium):
        with GpuEngine(sc.grid) as e:
            e.set_medium(medium)
            e.set_sources(sc.encoded(0))
            e.set_sensors(sc.sensors)
            return e.gradient_tr(obs, 8)

    want_b, want_r = fresh(mb), fresh(mr)
    with GpuEngine(sc.grid) as eng:
        eng.set_medium(m)
        eng.set_sources(sc.encoded(0))
        eng.set_sensors(sc.sensors)
        for _ in range(3):          # eager, capture, replay
            eng.gradient_tr(obs, 8)
        eng.set_medium(mb)
        eng.set_sensors(sc.sensors)  # the same array: no rebinding
        got_b = [eng.gradient_tr(obs, 8) for _ in range(2)]
        eng.set_medium(mr)
        got_r = [eng.gradient_tr(obs, 8) for _ in range(3)]
    for loss, grad in got_b:
        assert loss == want_b[0] and grad.tobytes() == want_b[1].tobytes()
    for loss, grad in got_r:
        assert loss == want_r[0] and grad.tobytes() == want_r[1].tobytes()
    assert want_b[1].tobytes() != want_r[1].tobytes()


def test_pair_loop_runs_on_two_sm_partitions():
    """The adjoint / replay streams of the TR pair loop live in two green contexts with
    disjoint SM sets (engine.cu green_partition): 48 % of the SMs (a multiple of 8) for the
    adjoint, the rest for the replay."""
    import os
    import torch
    if "USTFWI_GREEN" in os.environ:
        pytest.skip("partition overridden by USTFWI_GREEN")
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    sc = scenario.config_a(nt=24)
    with GpuEngine(sc.grid) as eng:
        a, r = eng.partition()
    assert a > 0 and r > 0 and a + r == n_sm and a % 8 == 0
    assert a == -(-(n_sm * 48 + 99) // 100 // 8) * 8 or a == (n_sm * 48 + 99) // 100
