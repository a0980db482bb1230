"""GPU parity and property tests of the device engine, called through the C ABI.

Parity bars (BASELINE.json north_star): rel l2 <= 1e-4 on recorded traces, <= 1e-3 on the
gradient volume (fp32 device vs fp64 reference). Oracle = the reference itself
(oracle/_ref, via golden fixtures from tests/golden/make_golden.py).
Property tests mirror test_solver.cpp (zero sources :50-58, linearity :82-119, delay
exactness :121-141, CFL :352-358) and SPEC.md adjoint_gradients invariants.
"""
import numpy as np
import pytest

from paper_2102_00755_b200 import capi, scenario
from paper_2102_00755_b200.engine import (GpuEngine, Medium, NumericalError, SensorArray, SourceSet,
                                          average_estimates, draw_realization, encode, gradient_time_reversal,
                                          make_homogeneous_medium, simulate_forward)

pytestmark = pytest.mark.gpu

TRACE_TOL = 1e-4
GRAD_TOL = 1e-3


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.fixture(scope="module")
def deriv_golden(golden):
    return golden("derivative_3d")


def test_derivative_matches_reference(deriv_golden):
    z = deriv_golden
    g = capi.grid_from(list(z["dims"]), float(z["dx"]), float(z["dt"]), 4, [0, 0, 0], float(z["c_ref"]))
    with GpuEngine(g) as eng:
        for axis in range(3):
            for st in ("none", "plus", "minus"):
                d = eng.derivative(z["f"], axis, st)
                assert rel(d, z[f"d{axis}_{st}"]) < 1e-5, (axis, st)


def test_derivative_padded_grid(deriv_golden):
    z = deriv_golden
    d = z["g2"]
    g = capi.grid_from(list(d[:3]), 1e-3, float(z["g2_dt"]), int(d[6]), list(d[3:6]), 1800.0)
    with GpuEngine(g) as eng:
        for axis in range(3):
            assert rel(eng.derivative(z["f2"], axis, "plus"), z[f"g2_d{axis}_plus"]) < 1e-5


def test_derivative_adjointness_3d():
    # test_grid.cpp:106-121 on a 3-D grid: <d+ u, v> = -<u, d- v>
    g = capi.grid_from([24, 18, 20], 1e-3, 0.3e-3 / 1500.0, 4, [0, 0, 0], 1500.0)
    rng = np.random.default_rng(11)
    u, v = rng.standard_normal(g.shape), rng.standard_normal(g.shape)
    with GpuEngine(g) as eng:
        for axis in range(3):
            lhs = np.sum(eng.derivative(u, axis, "plus") * v)
            rhs = np.sum(u * eng.derivative(v, axis, "minus"))
            assert abs(lhs + rhs) < 1e-5 * np.linalg.norm(u) * np.linalg.norm(v)


def test_forward_2d_matches_reference(golden):
    z = golden("forward_2d")
    g = capi.make_grid([64, 64], 1e-3, 1800.0, 5e-5)
    m = make_homogeneous_medium(g)
    pulse = z["pulse"]
    src = SourceSet(positions=list(z["pos"]), signals=[pulse, -0.7 * pulse])
    res = simulate_forward(m, src, SensorArray(list(z["sens"])), g)
    assert rel(res.data, z["data"]) < TRACE_TOL


@pytest.fixture(scope="module")
def config_a_short(golden):
    z = golden("config_a_short")
    sc = scenario.config_a(nt=int(z["nt"]))
    eng = GpuEngine(sc.grid)
    yield sc, z, eng
    eng.close()


def test_config_a_short_traces_and_shell(config_a_short):
    sc, z, eng = config_a_short
    eng.set_medium(sc.model)
    eng.set_sources(sc.sources)
    eng.set_sensors(sc.sensors)
    data, trace = eng.forward(8)
    assert rel(data, z["data_model"]) < TRACE_TOL
    s0, s1 = z["trace_stride"]
    assert rel(trace[::s0, ::s1], z["trace_sub"]) < TRACE_TOL
    assert abs(trace.sum() - z["trace_checksum"][0]) <= 1e-4 * z["trace_checksum"][1]


def test_config_a_short_gradient(config_a_short):
    sc, z, eng = config_a_short
    eng.set_medium(sc.model)
    eng.set_sources(sc.sources)
    eng.set_sensors(sc.sensors)
    loss, grad = eng.gradient_tr(z["observed"], 8)
    assert abs(loss - float(z["loss"])) <= 1e-4 * abs(float(z["loss"]))
    flat = grad.ravel()
    assert rel(flat[z["gamma_idx"]], z["grad_gamma"]) < GRAD_TOL
    outside = np.ones(flat.size, bool)
    outside[z["gamma_idx"]] = False
    assert np.all(flat[outside] == 0.0)


def test_config_a_full_gradient(golden):
    z = golden("config_a")
    sc = scenario.config_a()
    with GpuEngine(sc.grid) as eng:
        eng.set_medium(sc.truth)
        eng.set_sources(sc.sources)
        eng.set_sensors(sc.sensors)
        obs_gpu, _ = eng.forward(0)
        assert rel(obs_gpu, z["observed"]) < TRACE_TOL
        eng.set_medium(sc.model)
        data, trace = eng.forward(8)
        assert rel(data, z["data_model"]) < TRACE_TOL
        loss, grad = eng.gradient_tr(z["observed"], 8)
        assert abs(loss - float(z["loss"])) <= 1e-3 * abs(float(z["loss"]))
        assert rel(grad.ravel()[z["gamma_idx"]], z["grad_gamma"]) < GRAD_TOL


def test_zero_sources_give_zero_data():
    g = capi.make_grid([44, 44, 44], 1e-3, 1800.0, 2e-5)
    m = make_homogeneous_medium(g)
    res = simulate_forward(m, SourceSet([], []), SensorArray([(32 * 64 + 32) * 64 + 32]), g)
    assert np.all(res.data == 0.0)


def _small_setup(nt_duration=3e-5):
    g = capi.make_grid([28, 28, 28], 1e-3, 1800.0, nt_duration)
    m = make_homogeneous_medium(g)
    pulse = capi.synth_source_pulse(g, 0.8, 1500.0)
    sh = g.shape
    f = lambda x, y, z: (x * sh[1] + y) * sh[2] + z
    return g, m, pulse, f


def test_linearity_and_scaling():
    g, m, pulse, f = _small_setup()
    sens = SensorArray([f(30, 30, 30), f(20, 26, 22)])
    with GpuEngine(g) as eng:
        r1 = simulate_forward(m, SourceSet([f(18, 20, 24)], [pulse]), sens, g, engine=eng).data
        r2 = simulate_forward(m, SourceSet([f(24, 18, 20)], [-0.7 * pulse]), sens, g, engine=eng).data
        rb = simulate_forward(m, SourceSet([f(18, 20, 24), f(24, 18, 20)], [pulse, -0.7 * pulse]), sens, g,
                              engine=eng).data
        assert rel(rb, r1 + r2) < 1e-5
        rs = simulate_forward(m, SourceSet([f(18, 20, 24)], [3.25 * pulse]), sens, g, engine=eng).data
        assert rel(rs, 3.25 * r1) < 1e-5


def test_delay_is_exact():
    g, m, pulse, f = _small_setup()
    sens = SensorArray([f(30, 30, 30)])
    delay = 17
    with GpuEngine(g) as eng:
        r0 = simulate_forward(m, SourceSet([f(20, 20, 20)], [pulse]), sens, g, engine=eng).data
        rd = simulate_forward(m, SourceSet([f(20, 20, 20)], [np.concatenate([np.zeros(delay), pulse])]), sens, g,
                              engine=eng).data
        # same arithmetic shifted in time: bit-identical on the device
        assert np.all(rd[:, :delay] == 0.0)
        assert np.array_equal(rd[:, delay:], r0[:, :-delay])
        # the encoded form (weights/delays) is the same computation
        re = simulate_forward(m, SourceSet([f(20, 20, 20)], [pulse], weights=np.array([1.0]),
                                           delays=np.array([delay])), sens, g, engine=eng).data
        assert np.array_equal(re, rd)


def test_encoded_forward_is_weighted_sum_of_delayed_singles():
    g, m, pulse, f = _small_setup()
    sens = SensorArray([f(30, 30, 30), f(14, 30, 16)])
    pos = [f(18, 20, 24), f(24, 18, 20), f(16, 28, 18)]
    r = draw_realization(3, 10 * g.dt, g.dt, 20210201, 0, 4)
    base = SourceSet(pos, [pulse] * 3)
    with GpuEngine(g) as eng:
        singles = [simulate_forward(m, SourceSet([p], [pulse]), sens, g, engine=eng).data for p in pos]
        enc, f_hat, nt_ext = encode(base, singles, r, g.nt)
        got = simulate_forward(m, enc, sens, g, engine=eng).data
    assert rel(got, f_hat[:, :g.nt]) < 1e-5


def test_zero_residual_gives_zero_gradient_and_determinism():
    sc = scenario.config_a(nt=80)
    with GpuEngine(sc.grid) as eng:
        eng.set_medium(sc.model)
        eng.set_sources(sc.sources)
        eng.set_sensors(sc.sensors)
        obs, _ = eng.forward(0)
        loss, grad = eng.gradient_tr(obs, 8)
        assert loss == 0.0 and np.all(grad == 0.0)
        obs2 = np.zeros_like(obs)
        l1, g1 = eng.gradient_tr(obs2, 8)
        l2, g2 = eng.gradient_tr(obs2, 8)
        assert l1 == l2 and np.array_equal(g1, g2) and np.abs(g1).max() > 0


def test_minibatch_accumulate_equals_average():
    sc = scenario.config_a(nt=80)
    obs = np.zeros((len(sc.sensors.positions), sc.grid.nt))
    with GpuEngine(sc.grid) as eng:
        eng.set_medium(sc.model)
        eng.set_sensors(sc.sensors)
        eng.upload_observed(obs)
        res = []
        for r in range(3):
            eng.set_sources(sc.encoded(r))
            res.append(gradient_time_reversal(sc.model, sc.encoded(r), sc.sensors, obs, sc.grid, 8, engine=eng))
        mean = average_estimates(res)
        eng.upload_observed(obs)
        for r in range(3):
            eng.set_sources(sc.encoded(r))
            eng.run_gradient(8, accumulate=r > 0)
        loss, grad = eng.download_gradient(3.0)
    assert rel(grad, mean.grad) < 1e-6
    assert abs(loss - mean.loss) <= 1e-12 * abs(mean.loss)


def test_error_mapping():
    g = capi.make_grid([28, 28, 28], 1e-3, 1500.0, 1e-5)
    with GpuEngine(g) as eng:
        m = make_homogeneous_medium(g, 1500.0)
        m.c0 = np.full(g.shape, 1700.0)          # c_max > c_ref at cfl 0.3 ... still stable
        eng.set_medium(m)
        bad = make_homogeneous_medium(g, 1500.0)
        bad.c0 = np.full(g.shape, 1900.0)        # outside [c0_min, c0_max]
        with pytest.raises(ValueError):
            eng.set_medium(bad)
        lossy = make_homogeneous_medium(g, 1500.0, alpha0=0.5, y=3.0)  # y outside (1,3), medium.hpp:52
        with pytest.raises(ValueError, match="power-law exponent"):
            eng.set_medium(lossy)
        lossy.alpha0 = np.full(g.shape, -0.5)
        lossy.y = 1.5
        with pytest.raises(ValueError, match="alpha0 must be non-negative"):
            eng.set_medium(lossy)
    g.dt = 1e-3 / 1500.0  # cfl = 1 > 2/pi (test_solver.cpp:352-358)
    with GpuEngine(g) as eng:
        with pytest.raises(NumericalError):
            eng.set_medium(make_homogeneous_medium(g, 1500.0))


def test_divergence_is_reported():
    g, m, pulse, f = _small_setup(1.5e-5)
    bad = pulse.copy()
    bad[3] = np.nan
    with GpuEngine(g) as eng:
        with pytest.raises(NumericalError, match="diverged at step 64"):
            simulate_forward(m, SourceSet([f(20, 20, 20)], [bad]), SensorArray([f(30, 30, 30)]), g, engine=eng)


def test_heterogeneous_density_staggering():
    # dt/rho0~ via the device fourier_shift must match the oracle forward traces
    from oracle import ustfwi_oracle as orc
    g = capi.make_grid([12, 12, 12], 1e-3, 1800.0, 1.2e-5)
    rng = np.random.default_rng(5)
    rho0 = 1000.0 + 80.0 * rng.random(g.shape)
    c0 = 1500.0 + 50.0 * rng.random(g.shape)
    sh = g.shape
    src = [(16 * sh[1] + 14) * sh[2] + 15]
    sens = [(8 * sh[1] + 20) * sh[2] + 22, (22 * sh[1] + 10) * sh[2] + 12]
    pulse = capi.synth_source_pulse(g, 0.8, 1350.0)
    want, _ = orc.simulate_forward(orc.Grid.of(g), c0, rho0, src, [pulse], sens)
    res = simulate_forward(Medium(c0=c0, rho0=rho0), SourceSet(src, [pulse]), SensorArray(sens), g)
    assert rel(res.data, want) < TRACE_TOL


@pytest.mark.parametrize("dims", [
    (4, 6, 8), (10, 14, 18), (16, 96, 10), (12, 12, 96), (48, 12, 10), (6, 480, 6), (480, 4, 4),
    (4, 4, 512), (14, 6, 14), (22, 4, 4), (4, 26, 6), (8, 8, 144), (144, 6, 8), (64, 64), (96, 96), (12, 256),
    (256,), (90,),
])
def test_derivative_fft_sizes(dims):
    """Every radix path of the device FFT (16/8/4/2/5/3/7 and the generic odd stage) on all
    three pass kinds, 1-D/2-D/3-D, against the fp64 numpy restatement."""
    from oracle import ustfwi_oracle as orc
    g = capi.grid_from(list(dims), 1e-3, 0.3e-3 / 1800.0, 4, [0] * len(dims), 1800.0)
    f = np.random.default_rng(sum(dims)).standard_normal(dims)
    og = orc.Grid.of(g)
    oe = orc.SpectralEngine(og)
    with GpuEngine(g) as eng:
        for axis in range(len(dims)):
            for st in ("none", "plus", "minus"):
                assert rel(eng.derivative(f, axis, st), oe.derivative(f, axis, st)) < 2e-5, (axis, st)


@pytest.mark.parametrize("nt", [2, 3, 4, 5, 8])
def test_short_durations_gradient_matches_reference(nt):
    """The pair loop's edges (engine.cu gradient_core: the 4-slot replay ring, the replay
    leading the adjoint by up to two steps, the first and last correlations) at nt = 2..8
    against the reference itself (oracle/_ref): source and receiver inside Gamma, 2 voxels
    apart, random observed data, so the forward and adjoint fields overlap from the first step."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    g = capi.make_grid([24, 24, 24], 1e-3, 1540.0, 1e-5)
    g.nt = nt
    sh = g.shape
    c = [d // 2 for d in sh]
    f = lambda x, y, z: (x * sh[1] + y) * sh[2] + z
    rng = np.random.default_rng(nt)
    c0 = 1500.0 + 20.0 * rng.random(sh)
    gamma = capi.ball_mask(sh, c, 7.0)
    m = Medium(c0=c0, rho0=np.full(sh, 1000.0), gamma=gamma, c0_min=1350.0, c0_max=1800.0)
    src, sens = [f(*c)], [f(c[0], c[1], c[2] + 2), f(c[0] + 1, c[1] - 1, c[2])]
    sig = [np.sin(np.arange(nt) * 0.7) + 0.3]
    obs = 1e-3 * rng.standard_normal((len(sens), nt))
    with GpuEngine(g) as eng:
        eng.set_medium(m)
        eng.set_sources(SourceSet(src, sig))
        eng.set_sensors(SensorArray(sens))
        for _ in range(3):  # eager, graph capture, replay
            loss, grad = eng.gradient_tr(obs, 2)
    loss_r, grad_r = ref.gradient_time_reversal(g, m, src, sig, sens, obs, 2)
    assert abs(loss - loss_r) <= TRACE_TOL * abs(loss_r)
    if not np.any(grad_r):  # nt = 2: no correlation step in the reference either
        assert not np.any(grad)
        return
    assert rel(grad, grad_r) <= GRAD_TOL
    assert np.all(grad[~np.asarray(gamma, bool)] == 0)
