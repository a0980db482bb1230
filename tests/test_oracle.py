"""CPU tests pinning the oracles.

1. The reference's own 35 Catch2 unit tests (test_grid.cpp, test_filter.cpp,
   test_solver.cpp) pass against oracle/_ref (reference + FFTW-API shim).
2. The product's host setup equals the reference's (pulse, shell, PML).
3. The numpy restatement (oracle/ustfwi_oracle.py) reproduces the reference's golden
   fixtures: derivatives, 2-D forward traces, config-A gradient/loss.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import ref
from oracle import ustfwi_oracle as orc
from paper_2102_00755_b200 import capi, scenario

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (make -C oracle)")


@needs_ref
def test_reference_unit_tests_pass_under_shims():
    exe = os.path.join(ROOT, "oracle", "_ref", "unit_tests")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "35 passed, 0 failed" in r.stdout


@needs_ref
def test_host_setup_matches_reference():
    rng = np.random.default_rng(3)
    for interior, dx in (([44, 44, 44], 1e-3), ([64, 64], 1e-3), ([108, 108, 108], 1e-3), ([48], 2e-3)):
        g = capi.make_grid(interior, dx, 1800.0, 1e-4)
        r = ref.make_grid(interior, dx, 1800.0, 1e-4)
        assert g.nt == r.nt and g.dt == r.dt and list(g.dims) == list(r.dims)
        assert np.array_equal(capi.synth_source_pulse(g, 0.8, 1350.0).size, ref.synth_source_pulse(g, 0.8, 1350.0).size)
        np.testing.assert_allclose(capi.synth_source_pulse(g, 0.8, 1350.0), ref.synth_source_pulse(g, 0.8, 1350.0),
                                   rtol=0, atol=1e-12)
        cr, cs = capi.make_pml(g)
        rr, rs = ref.make_pml(g)
        for a in range(len(cr)):
            assert np.array_equal(cr[a], rr[a]) and np.array_equal(cs[a], rs[a])
    for _ in range(5):
        mask = (rng.random((20, 18, 16)) > 0.2).astype(np.uint8)
        mask = capi.ball_mask(mask.shape, [10, 9, 8], 7.5) | mask * 0
        for t in (1, 2, 3):
            assert np.array_equal(capi.shell_indices(mask, t), ref.shell_indices(mask, t))
    m2 = (rng.random((30, 30)) > 0.3).astype(np.uint8)
    assert np.array_equal(capi.shell_indices(m2, 1), ref.shell_indices(m2, 1))


def test_numpy_oracle_derivatives_match_reference_golden(golden):
    z = golden("derivative_3d")
    g = orc.Grid(z["dims"], float(z["dx"]), float(z["dt"]), 4, [0, 0, 0], float(z["c_ref"]))
    eng = orc.SpectralEngine(g)
    for axis in range(3):
        for st in ("none", "plus", "minus"):
            np.testing.assert_allclose(eng.derivative(z["f"], axis, st), z[f"d{axis}_{st}"], rtol=0, atol=1e-9)
    d = z["g2"]
    g2 = orc.Grid(d[:3], 1e-3, float(z["g2_dt"]), int(d[6]), d[3:6], 1800.0)
    eng2 = orc.SpectralEngine(g2)
    for axis in range(3):
        np.testing.assert_allclose(eng2.derivative(z["f2"], axis, "plus"), z[f"g2_d{axis}_plus"], rtol=0, atol=1e-9)


def test_numpy_oracle_forward_2d_matches_reference_golden(golden):
    z = golden("forward_2d")
    gg = capi.make_grid([64, 64], 1e-3, 1800.0, 5e-5)
    g = orc.Grid.of(gg)
    shape = g.dims
    pulse = z["pulse"]
    data, _ = orc.simulate_forward(g, np.full(shape, 1500.0), np.full(shape, 1000.0), list(z["pos"]),
                                   [pulse, -0.7 * pulse], list(z["sens"]))
    ref_data = z["data"]
    assert np.abs(ref_data).max() > 0
    np.testing.assert_allclose(data, ref_data, rtol=0, atol=1e-12 * np.abs(ref_data).max())


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.slow
def test_numpy_oracle_gradient_matches_reference_golden(golden):
    z = golden("config_a_short")
    sc = scenario.config_a(nt=int(z["nt"]))
    g = orc.Grid.of(sc.grid)
    shell = capi.shell_indices(sc.model.gamma, 8)
    loss, grad = orc.gradient_tr(g, sc.model.c0, sc.model.rho0, sc.model.gamma, list(sc.sources.positions),
                                 [np.asarray(s) for s in sc.sources.signals], list(sc.sensors.positions),
                                 z["observed"], 8, shell)
    assert abs(loss - float(z["loss"])) <= 1e-10 * abs(float(z["loss"]))
    gg = grad.ravel()[z["gamma_idx"]]
    assert _rel(gg, z["grad_gamma"]) < 1e-10
