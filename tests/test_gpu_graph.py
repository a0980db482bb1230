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
