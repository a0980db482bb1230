"""Edge cases of the device path against the fp64 numpy oracle (small grids).

Mirrors the cases the reference code handles (SourceSet::sample past the end,
medium.hpp:80-84; shell_indices errors :168-178; several sources at one position, injected
in order, simulate.hpp:82-85) plus boundary positions and the empty sensor set."""
import numpy as np
import pytest

from oracle import ustfwi_oracle as orc
from paper_2102_00755_b200 import capi
from paper_2102_00755_b200.engine import GpuEngine, Medium, SensorArray, SourceSet, make_homogeneous_medium

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def small():
    g = capi.make_grid([12, 12, 12], 1e-3, 1800.0, 1.5e-5)
    sh = g.shape
    f = lambda x, y, z: (x * sh[1] + y) * sh[2] + z
    pulse = capi.synth_source_pulse(g, 0.8, 1350.0)
    eng = GpuEngine(g)
    yield g, f, pulse, eng
    eng.close()


def oracle_forward(g, m, src, sens):
    w = None if src.weights is None else list(src.weights)
    d = None if src.delays is None else list(src.delays)
    return orc.simulate_forward(orc.Grid.of(g), m.c0, m.rho0, list(src.positions), [np.asarray(s) for s in src.signals],
                                list(sens.positions), weights=w, delays=d)[0]


def test_duplicate_positions_and_grid_corners(small):
    g, f, pulse, eng = small
    n = g.points
    m = make_homogeneous_medium(g)
    src = SourceSet([f(10, 12, 14), f(10, 12, 14), 0, n - 1], [pulse, -0.4 * pulse, 0.3 * pulse, 0.2 * pulse])
    sens = SensorArray([f(20, 20, 20), 0, n - 1, f(10, 12, 14), f(20, 20, 20)])  # repeated sensor too
    eng.set_medium(m)
    eng.set_sources(src)
    eng.set_sensors(sens)
    data, _ = eng.forward(0)
    want = oracle_forward(g, m, src, sens)
    assert rel(data, want) < 1e-4
    assert np.array_equal(data[0], data[4])


def test_signals_past_the_end_and_large_delays(small):
    g, f, pulse, eng = small
    m = make_homogeneous_medium(g)
    long_sig = np.concatenate([pulse, pulse[::-1], np.ones(3 * g.nt)])  # longer than nt
    src = SourceSet([f(14, 14, 14), f(18, 16, 20)], [long_sig, pulse], weights=np.array([1.0, -1.0]),
                    delays=np.array([3, g.nt + 5]))  # second source never fires
    sens = SensorArray([f(22, 22, 22)])
    eng.set_medium(m)
    eng.set_sources(src)
    eng.set_sensors(sens)
    data, _ = eng.forward(0)
    want = oracle_forward(g, m, src, sens)
    assert rel(data, want) < 1e-4
    only_first = SourceSet([f(14, 14, 14)], [long_sig], weights=np.array([1.0]), delays=np.array([3]))
    eng.set_sources(only_first)
    d1, _ = eng.forward(0)
    assert np.array_equal(d1, data)


def test_shell_thickness_exceeding_gamma_is_rejected(small):
    g, f, pulse, eng = small
    m = make_homogeneous_medium(g)
    m.gamma = capi.ball_mask(g.shape, [16, 16, 16], 2.5)
    eng.set_medium(m)
    eng.set_sources(SourceSet([f(5, 5, 5)], [pulse]))
    eng.set_sensors(SensorArray([f(25, 25, 25)]))
    with pytest.raises(ValueError, match="shell thickness exceeds"):
        eng.forward(8)
    with pytest.raises(ValueError, match="must be >= 1"):
        capi.shell_indices(m.gamma, 0)


def test_no_sensors_gives_zero_loss_and_gradient(small):
    g, f, pulse, eng = small
    m = make_homogeneous_medium(g)
    m.gamma = capi.ball_mask(g.shape, [16, 16, 16], 6.0)
    eng.set_medium(m)
    eng.set_sources(SourceSet([f(5, 5, 5)], [pulse]))
    eng.set_sensors(SensorArray([]))
    loss, grad = eng.gradient_tr(np.zeros((0, g.nt)), 2)
    assert loss == 0.0 and np.all(grad == 0.0)


def test_heterogeneous_c0_gradient_matches_oracle(small):
    g, f, pulse, eng = small
    rng = np.random.default_rng(2)
    c0 = 1500.0 + 40.0 * rng.random(g.shape)
    gamma = capi.ball_mask(g.shape, [16, 16, 16], 7.0)
    m = Medium(c0=c0, rho0=np.full(g.shape, 1000.0), gamma=gamma)
    src = SourceSet([f(4, 16, 16), f(27, 9, 20)], [pulse, 0.5 * pulse])
    sens = SensorArray([f(27, 27, 16), f(16, 4, 5), f(6, 26, 26)])
    obs = np.zeros((3, g.nt))
    eng.set_medium(m)
    eng.set_sources(src)
    eng.set_sensors(sens)
    loss, grad = eng.gradient_tr(obs, 3)
    shell = capi.shell_indices(gamma, 3)
    wl, wg = orc.gradient_tr(orc.Grid.of(g), c0, m.rho0, gamma, list(src.positions),
                             [np.asarray(s) for s in src.signals], list(sens.positions), obs, 3, shell)
    assert abs(loss - wl) <= 1e-4 * wl
    assert rel(grad, wg) < 1e-3


def test_shell_follows_gamma_changes(small):
    # the engine keeps the boundary shell while gamma is unchanged and rebuilds it otherwise
    g, f, pulse, eng = small
    m = make_homogeneous_medium(g)
    eng.set_sources(SourceSet([f(5, 5, 5)], [pulse]))
    eng.set_sensors(SensorArray([f(25, 25, 25)]))
    sizes = []
    for r in (6.0, 6.0, 8.0):
        m.gamma = capi.ball_mask(g.shape, [16, 16, 16], r)
        eng.set_medium(m)
        _, trace = eng.forward(2)
        sizes.append(trace.shape[1])
        assert trace.shape[1] == len(capi.shell_indices(m.gamma, 2))
    assert sizes[0] == sizes[1] < sizes[2]


def test_two_engines_in_two_threads_match_sequential():
    # distinct engines may run concurrently (engine.hpp:14-16): no hidden
    # shared state in the library (map caches are per thread, attributes per device)
    import threading

    from paper_2102_00755_b200 import scenario
    sc = scenario.config_a(nt=60)
    obs = np.zeros((len(sc.sensors.positions), sc.grid.nt))

    def run(idx, out):
        with GpuEngine(sc.grid) as eng:
            eng.set_medium(sc.model)
            eng.set_sources(sc.encoded(idx))
            eng.set_sensors(sc.sensors)
            out[idx] = eng.gradient_tr(obs, 8)

    seq, par = {}, {}
    for k in (0, 1):
        run(k, seq)
    th = [threading.Thread(target=run, args=(k, par)) for k in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for k in (0, 1):
        assert seq[k][0] == par[k][0] and np.array_equal(seq[k][1], par[k][1])
