"""Absorbing media on the device against the reference itself.

Fixture tests/golden/config_a_absorb.npz comes from oracle/_ref (the unmodified reference
headers, make_golden.py): config A at nt = 96 with alpha0 = 3 dB/(MHz^y cm) in gamma and
0.5 outside. Covered: the absorbing update_pressure with the dispersion term (y = 1.5) and
without it (y = 2, engine.hpp:191), and the TR c0 gradient with the absorption terms of
GradientAccumulator (gradient.hpp:63-74,183-203) and the flipped replay sign (:429-431)."""
import copy

import numpy as np
import pytest

from paper_2102_00755_b200 import scenario
from paper_2102_00755_b200.engine import GpuEngine

pytestmark = pytest.mark.gpu

TRACE_TOL = 1e-4
GRAD_TOL = 1e-3


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def absorbing(m, y):
    a = copy.copy(m)
    gam = np.asarray(m.gamma, bool)
    a.alpha0 = np.where(gam, 3.0, 0.5)
    a.y = y
    return a


@pytest.fixture(scope="module")
def setup(golden):
    z = golden("config_a_absorb")
    sc = scenario.config_a(nt=int(z["nt"]))
    eng = GpuEngine(sc.grid)
    eng.set_sources(sc.sources)
    eng.set_sensors(sc.sensors)
    yield sc, z, eng
    eng.close()


def test_absorbing_forward_with_dispersion(setup):
    sc, z, eng = setup
    eng.set_medium(absorbing(sc.model, 1.5))
    data, trace = eng.forward(8)
    assert rel(data, z["data_y15"]) < TRACE_TOL
    # the absorption is visible at this tolerance (3 % of the lossless traces)
    assert rel(data, z["data_lossless"]) > 100 * TRACE_TOL
    assert abs(trace.sum() - z["trace_checksum"][0]) <= 1e-4 * z["trace_checksum"][1]


def test_absorbing_forward_without_dispersion(setup):
    sc, z, eng = setup
    eng.set_medium(absorbing(sc.model, 2.0))
    data, _ = eng.forward(0)
    assert rel(data, z["data_y20"]) < TRACE_TOL


def test_absorbing_tr_gradient(setup):
    sc, z, eng = setup
    eng.set_medium(absorbing(sc.model, 1.5))
    observed = np.zeros((len(sc.sensors.positions), int(z["nt"])))
    loss, grad = eng.gradient_tr(observed, 8)
    assert abs(loss - float(z["loss"])) <= 1e-4 * abs(float(z["loss"]))
    assert rel(grad.ravel()[z["gamma_idx"]], z["grad_gamma"]) < GRAD_TOL


def test_absorbing_tr_gradient_dispersion_disabled(setup):
    # GradientOptions::dispersion_enabled = false: adjoint and replay drop the dispersion
    # term, the forward simulation keeps it (gradient.hpp:381-384,424-426)
    sc, z, eng = setup
    eng.set_medium(absorbing(sc.model, 1.5))
    observed = np.zeros((len(sc.sensors.positions), int(z["nt"])))
    loss, grad = eng.gradient_tr(observed, 8, dispersion_enabled=False)
    assert abs(loss - float(z["loss_nodisp"])) <= 1e-4 * abs(float(z["loss_nodisp"]))
    g = grad.ravel()[z["gamma_idx"]]
    assert rel(g, z["grad_gamma_nodisp"]) < GRAD_TOL
    # the switch matters at this tolerance
    assert rel(z["grad_gamma_nodisp"], z["grad_gamma"]) > 10 * GRAD_TOL


def test_lossless_after_absorbing_medium(setup, golden):
    # switching back to alpha0 = None releases the absorbing path
    sc, z, eng = setup
    eng.set_medium(sc.model)
    data, _ = eng.forward(0)
    assert rel(data, z["data_lossless"]) < TRACE_TOL


@pytest.mark.parametrize("param,key,lossless", [("alpha0", "grad_alpha0", False), ("y", "grad_y", False),
                                                ("alpha0", "grad_alpha0_lossless", True)])
def test_alpha0_and_y_gradients(setup, param, key, lossless):
    # GradientParam alpha0 / y (gradient.hpp:76-116): no c0 ddot term, |k|^y and |k|^(y+1)
    # (times log|k|^2 for y) fields of the replay pressures; the alpha0 weights do not depend
    # on alpha0, so the lossless model has a non-zero alpha0 gradient too
    sc, z, eng = setup
    eng.set_medium(sc.model if lossless else absorbing(sc.model, 1.5))
    observed = np.zeros((len(sc.sensors.positions), int(z["nt"])))
    loss, grad = eng.gradient_tr(observed, 8, param=param)
    if not lossless:
        assert abs(loss - float(z["loss_" + param])) <= 1e-4 * abs(float(z["loss_" + param]))
    assert rel(grad.ravel()[z["gamma_idx"]], z[key]) < GRAD_TOL


def test_rho0_gradient_is_computed(setup):
    # GradientParam::rho0 (gradient.hpp:117-128,213-239); parity against the reference is in
    # tests/test_gpu_encoding.py::test_rho0_gradient_matches_reference
    sc, z, eng = setup
    eng.set_medium(sc.model)
    loss, grad = eng.gradient_tr(np.zeros((len(sc.sensors.positions), int(z["nt"]))), 8, param="rho0")
    assert loss > 0 and np.isfinite(grad).all() and np.abs(grad).max() > 0
