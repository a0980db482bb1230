"""The config-C/D kernel set (480-point TMA pencils, paired-residue z rows for nz = 256,
the pressure kernel) against the fp64 oracle on a small grid that selects the same
kernels, and size-independent properties on the full config-D grid (480x480x256)."""
import numpy as np
import pytest

from oracle import ustfwi_oracle as orc
from paper_2102_00755_b200 import capi, scenario
from paper_2102_00755_b200.engine import GpuEngine, Medium, SensorArray, SourceSet

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_nz256_step_kernels_against_oracle():
    # nz = 256 selects zvel2 / zrho2 / zp2 <M = 128>; x, y of 32 the register pencils
    dims = [32, 32, 256]
    dt = 0.3e-3 / 1800.0
    g = capi.grid_from(dims, 1e-3, dt, 70, [4, 4, 10], 1800.0)
    sh = g.shape
    f = lambda x, y, z: (x * sh[1] + y) * sh[2] + z
    rng = np.random.default_rng(11)
    c0 = 1480.0 + 60.0 * rng.random(sh)
    gamma = capi.ball_mask(sh, [16, 16, 128], 9.0)
    m = Medium(c0=c0, rho0=np.full(sh, 1000.0), gamma=gamma)
    pulse = capi.synth_source_pulse(g, 0.8, 1350.0)
    src = SourceSet([f(16, 16, 40), f(8, 24, 200)], [pulse, -0.6 * pulse])
    sens = SensorArray([f(16, 16, 52), f(12, 22, 190), f(20, 10, 46)])  # within reach in 70 steps
    with GpuEngine(g) as eng:
        eng.set_medium(m)
        eng.set_sources(src)
        eng.set_sensors(sens)
        data, _ = eng.forward(0)
        obs = np.zeros_like(data)
        loss, grad = eng.gradient_tr(obs, 3)
    og = orc.Grid.of(g)
    want = orc.simulate_forward(og, c0, m.rho0, list(src.positions), [np.asarray(s) for s in src.signals],
                                list(sens.positions))[0]
    assert rel(data, want) < 1e-4
    shell = capi.shell_indices(gamma, 3)
    wl, wg = orc.gradient_tr(og, c0, m.rho0, gamma, list(src.positions), [np.asarray(s) for s in src.signals],
                             list(sens.positions), obs, 3, shell)
    assert abs(loss - wl) <= 1e-4 * wl
    assert rel(grad, wg) < 1e-3


@pytest.fixture(scope="module")
def config_d_short():
    sc = scenario.config_d(nt=24)
    with GpuEngine(sc.grid) as eng:
        eng.set_medium(sc.model)
        # receivers plus sensors on 16 emitters (the bowl receivers are out of reach in 24 steps)
        eng.set_sensors(SensorArray(list(sc.sensors.positions) + list(sc.sources.positions[:16])))
        yield sc, eng


def test_config_d_scaling_is_exact(config_d_short):
    # every operation is linear and a power-of-two scale is exact in fp32: data(2 s) == 2 data(s)
    sc, eng = config_d_short
    enc = sc.encoded(0)
    eng.set_sources(enc)
    d1, t1 = eng.forward(sc.thickness)
    eng.set_sources(SourceSet(enc.positions, [2.0 * np.asarray(s) for s in enc.signals], weights=enc.weights,
                              delays=enc.delays))
    d2, t2 = eng.forward(sc.thickness)
    assert np.abs(d1).max() > 0 and np.array_equal(d2, 2.0 * d1) and np.array_equal(t2, 2.0 * t1)


def test_config_d_delay_shift_is_exact(config_d_short):
    # time invariance of the device stepper at full size: a source delayed by k steps gives
    # the same traces shifted by k, bit for bit (test_solver.cpp:121-141 analogue)
    sc, eng = config_d_short
    enc = sc.encoded(0)
    k = 5
    eng.set_sources(SourceSet(enc.positions, enc.signals, weights=enc.weights, delays=np.asarray(enc.delays)))
    d0, _ = eng.forward(0)
    eng.set_sources(SourceSet(enc.positions, enc.signals, weights=enc.weights, delays=np.asarray(enc.delays) + k))
    dk, _ = eng.forward(0)
    assert np.abs(d0).max() > 0
    assert np.all(dk[:, :k] == 0.0) and np.array_equal(dk[:, k:], d0[:, :-k])
