"""Gradient invariants of the device TR gradient against the reference's own values
(SPEC.md adjoint_gradients; fixture tests/golden/config_a_fd.npz from oracle/_ref, made by
tests/golden/make_golden.py --fd-only):

* the directional derivative <G, delta> of the TR gradient (shell = all of gamma) and the
  central finite difference of the loss along delta, each equal to the reference's value.
  The reference's own pair disagrees by ~27 % at config A (its adjoint-state gradient is not
  the discrete gradient of its loss: SPEC.md:224's 1e-3 FD bar does not hold for it), so the
  test pins both numbers to the reference instead of to each other;
* the time-reversal error decreases as the boundary shell thickens, with the
  errors of thickness 1/2/4/8 against the full-thickness replay equal to the reference's."""
import numpy as np
import pytest

from paper_2102_00755_b200 import scenario
from paper_2102_00755_b200.engine import GpuEngine, Medium

pytestmark = pytest.mark.gpu


def fd_direction(shape, gamma):  # = tests/golden/make_golden.py fd_direction
    c = [n // 2 for n in shape]
    ix, iy, iz = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    r2 = (ix - c[0] - 2) ** 2 + (iy - c[1] + 1) ** 2 + (iz - c[2]) ** 2
    return np.exp(-r2 / (2 * 3.0 ** 2)) * np.asarray(gamma, dtype=np.float64)


def _with_c0(m, c0):
    return Medium(c0=c0, rho0=m.rho0, gamma=m.gamma, c0_min=m.c0_min, c0_max=m.c0_max)


def _loss(eng, m, obs):
    eng.set_medium(m)
    data, _ = eng.forward(0)
    r = data.astype(np.float64) - obs
    return 0.5 * float(np.sum(r * r))


@pytest.fixture(scope="module")
def fd_case(golden):
    z = golden("config_a_fd")
    sc = scenario.config_a()
    eng = GpuEngine(sc.grid)
    eng.set_sources(sc.sources)
    eng.set_sensors(sc.sensors)
    eng.set_medium(sc.truth)
    obs, _ = eng.forward(0)
    eng.set_medium(sc.model)
    yield sc, z, eng, obs
    eng.close()


def test_directional_derivative_and_finite_difference_match_reference(fd_case):
    sc, z, eng, obs = fd_case
    delta = fd_direction(sc.grid.shape, sc.model.gamma)
    eng.set_medium(sc.model)
    loss, grad = eng.gradient_tr(obs, 12)
    dJ = float(np.sum(grad.astype(np.float64) * delta))
    eps = float(z["eps"])
    c0 = np.asarray(sc.model.c0, dtype=np.float64)
    fd = (_loss(eng, _with_c0(sc.model, c0 + eps * delta), obs) -
          _loss(eng, _with_c0(sc.model, c0 - eps * delta), obs)) / (2 * eps)
    assert abs(loss - float(z["loss"])) <= 1e-3 * abs(float(z["loss"]))
    assert abs(dJ - float(z["dJ"])) <= 1e-3 * abs(float(z["dJ"])), (dJ, float(z["dJ"]))
    assert abs(fd - float(z["fd"])) <= 1e-3 * abs(float(z["fd"])), (fd, float(z["fd"]))


def test_tr_error_decreases_with_shell_thickness(fd_case):
    sc, z, eng, obs = fd_case
    eng.set_medium(sc.model)
    _, g_full = eng.gradient_tr(obs, 12)
    errs = []
    for t in z["thickness"]:
        _, g = eng.gradient_tr(obs, int(t))
        errs.append(float(np.linalg.norm(g - g_full) / np.linalg.norm(g_full)))
    assert all(a >= b for a, b in zip(errs, errs[1:])), errs
    ref_errs = np.asarray(z["tr_err_vs_12"])
    # errors are differences of nearly equal gradients: compare at 1e-3 of the full gradient
    assert np.all(np.abs(np.asarray(errs) - ref_errs) <= 1e-3 + 1e-2 * ref_errs), (errs, ref_errs.tolist())
