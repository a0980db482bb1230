"""Scenario kit (SPEC.md scenario_kit :517-581): noise model, transducer placement, phantom
invariants; host-side input generation (no device)."""
import numpy as np

from paper_2102_00755_b200 import scenario


def test_add_noise_examples():
    # RMS 1, SNR 5 -> sigma = 10^-0.25
    f = np.ones((64, 4096))
    noisy = scenario.add_noise(f, 5.0, seed=3)
    sigma = float(np.std(noisy - f))
    assert abs(sigma - 10 ** -0.25) < 3 * 10 ** -0.25 / np.sqrt(f.size) * 3
    assert abs(float(np.mean(noisy - f))) < 3 * 10 ** -0.25 / np.sqrt(f.size)
    assert np.array_equal(scenario.add_noise(f, np.inf, 1), f)
    assert np.array_equal(scenario.add_noise(np.zeros((3, 5)), 10.0, 1), np.zeros((3, 5)))
    assert np.array_equal(scenario.add_noise(f, 5.0, seed=3), noisy)  # deterministic per seed


def test_golden_section_placement():
    shape = (80, 80, 60)
    center = (40.0, 40.0, 8.0)
    R = 30.0
    emit, recv = scenario.golden_section_placement(2048, R, center, shape)
    pts = emit + recv
    assert len(set(emit) & set(recv)) == 0 and len(set(pts)) == len(pts)
    xyz = np.array([np.unravel_index(p, shape) for p in pts], dtype=np.float64)
    d = np.linalg.norm(xyz - np.array(center), axis=1)
    assert np.all(np.abs(d - R) <= np.sqrt(3) / 2 + 1e-9)  # grid snapping: radius +- half a diagonal
    assert abs(len(emit) - len(recv)) <= len(pts) * 0.05


def test_breast_phantom_invariants():
    sc = scenario.config_b(nt=4)
    c0 = np.asarray(sc.truth.c0)
    assert set(np.unique(c0)) <= {1470.0, 1500.0, 1515.0, 1584.0, 1650.0}
    gam = np.asarray(sc.truth.gamma).astype(bool)
    assert np.all(gam[c0 != 1500.0])                       # gamma covers all tissue
    pos = list(sc.sources.positions) + list(sc.sensors.positions)
    assert not np.any(gam.ravel()[pos])                    # and no transducer
    sc2 = scenario.config_b(nt=4)
    assert np.array_equal(np.asarray(sc2.truth.c0), c0)   # deterministic per seed
