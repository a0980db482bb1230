"""SLBFGS on the device: the HBM-resident two-loop recursion against the
numpy oracle (oracle/slbfgs_oracle.py, itself pinned by the SPEC examples in
tests/test_oracle_slbfgs.py), the optimizer loop of Algorithm 2, the SGD baselines, and one
end-to-end run driving the TR gradient engine."""
import numpy as np
import pytest

from oracle import slbfgs_oracle as so
from paper_2102_00755_b200 import scenario
from paper_2102_00755_b200.engine import GpuEngine
from paper_2102_00755_b200.optim import DeviceLbfgs, sgd_momentum_run, sgd_run, slbfgs_run

pytestmark = pytest.mark.gpu


def test_two_loop_matches_oracle_with_ring_wraparound():
    rng = np.random.default_rng(3)
    n, m = 10_000, 8
    d = 1.0 + rng.random(n)  # diagonal SPD curvature
    P = so.Pairs(m)
    with DeviceLbfgs(n, m) as H:
        g = rng.standard_normal(n)
        assert np.array_equal(H.apply(g), g)  # empty history: H0 = I
        for k in range(11):  # wraps the ring of 8
            s = rng.standard_normal(n)
            y = d * s + 0.01 * rng.standard_normal(n)
            assert H.push(s, y) == P.push(s, y)
        # a non-curvature pair is rejected and leaves the state unchanged
        s = rng.standard_normal(n)
        assert not H.push(s, -s) and not P.push(s, -s)
        cnt, gam = H.pairs()
        assert cnt == m and abs(gam - P.gamma) <= 1e-14 * abs(P.gamma)
        out = H.apply(g)
        want = so.two_loop(g, P)
        assert np.linalg.norm(out - want) <= 1e-12 * np.linalg.norm(want)
        # determinism of the device reductions
        assert np.array_equal(H.apply(g), out)
        H.reset()
        assert np.array_equal(H.apply(g), g)


def test_two_loop_dense_bfgs_and_secant():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((5, 5))
    A = A @ A.T + 5 * np.eye(5)
    P = so.Pairs(64)
    with DeviceLbfgs(5, 64) as H:
        for _ in range(3):
            s = rng.standard_normal(5)
            assert H.push(s, A @ s) and P.push(s, A @ s)
        g = rng.standard_normal(5)
        assert np.linalg.norm(H.apply(g) - so.dense_bfgs(P) @ g) <= 1e-10 * np.linalg.norm(g)
    with DeviceLbfgs(1, 64) as H:
        a = 3.7
        H.push(np.array([-1.5]), np.array([-1.5 * a]))
        assert abs(H.apply(np.array([1.3]))[0] - 1.3 / a) < 1e-15


def _quadratic(seed=1, n=100):
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((n, n))
    A = Q @ Q.T / n + np.eye(n)
    b = rng.standard_normal(n)
    return A, b, np.linalg.solve(A, b)


def test_slbfgs_deterministic_quadratic_matches_oracle():
    A, b, ustar = _quadratic()

    def est(u, th, k):
        return 0.5 * u @ A @ u - b @ u, A @ u - b

    res = slbfgs_run(est, np.zeros(100), 50, nu=0.5)
    assert res.n_evl <= 50 and np.linalg.norm(res.u - ustar) < 1e-8
    u_o, e_o, _ = so.slbfgs(est, np.zeros(100), 50, nu=0.5)
    assert np.allclose(res.energy, e_o, rtol=1e-9, atol=1e-14)
    assert np.linalg.norm(res.u - u_o) < 1e-10


def test_slbfgs_bounds_and_seed_pairing():
    target = np.array([2.0, -3.0, 0.25])
    seeds = []

    def est(u, th, k):
        seeds.append(k)
        return 0.5 * np.sum((u - target) ** 2), u - target

    res = slbfgs_run(est, np.zeros(3), 20, nu=1.0, bounds=(-1.0, 1.0))
    assert np.allclose(res.u, [1.0, -1.0, 0.25], atol=1e-12)
    # both estimator calls of an iteration use the same realization index
    assert seeds[0::2] == seeds[1::2] == list(range(1, len(seeds) // 2 + 1))


def test_iterate_averaging_weights():
    # constant gradient c, nu = 1: u_i = u0 - i c; energy rises at i = 2 -> averaging from i = 3
    c = np.array([1.0, -2.0])

    def est(u, th, k):
        return float(k), c.copy()

    res = sgd_run(est, np.zeros(2), 5, nu=1.0)
    u = {i: -i * c for i in range(1, 6)}
    want = (27 * u[3] + 64 * u[4] + 125 * u[5]) / (27 + 64 + 125)
    assert res.averaging_from == 3 and np.allclose(res.u, want, rtol=1e-15)


def test_momentum_zero_is_plain_sgd():
    A, b, _ = _quadratic(2, 20)

    def est(u, th, k):
        return 0.5 * u @ A @ u - b @ u, A @ u - b

    r0 = sgd_run(est, np.zeros(20), 30, nu=0.2)
    r1 = sgd_momentum_run(est, np.zeros(20), 30, nu=0.2, beta=0.0)
    assert np.array_equal(r0.u, r1.u) and r0.energy == r1.energy


def test_slbfgs_drives_the_tr_gradient_engine():
    # c0 inside gamma as the unknown, observed data from the truth medium (config A)
    sc = scenario.config_a()
    gam = np.asarray(sc.model.gamma, bool).ravel()
    with GpuEngine(sc.grid) as eng:
        eng.set_sources(sc.sources)
        eng.set_sensors(sc.sensors)
        eng.set_medium(sc.truth)
        observed, _ = eng.forward(0)
        base = np.asarray(sc.model.c0, dtype=np.float64).ravel().copy()

        def est(u, th, k):
            # the wave model is only defined inside the medium bounds: evaluate on the box
            m = sc.model
            c0 = base.copy()
            c0[gam] = np.clip(u, 1400.0, 1600.0)
            m.c0 = c0.reshape(sc.grid.shape)
            eng.set_medium(m)
            loss, grad = eng.gradient_tr(observed, 8)
            return loss, grad.ravel()[gam]

        u0 = base[gam].copy()
        F0, G0 = est(u0, 0.0, 0)
        nu = 2.0 / np.abs(G0).max()  # first step moves c0 by <= 2 m/s
        res = slbfgs_run(est, u0, 4, nu=nu, bounds=(1400.0, 1600.0))
    assert res.n_evl == 4 and all(np.isfinite(res.energy))
    # the first trial step along -G (H0 = I) decreases the data misfit: J_1 = min(F_u, F_z) < F_u
    assert res.energy[0] < F0
    assert res.log[0]["pair_accepted"]


def test_slbfgs_device_resident_vectors_match_host():
    # the same Algorithm 2 run with torch CUDA fp64 iterates (push / apply on device pointers,
    # no transfers) and with numpy host iterates
    import torch
    A, b, ustar = _quadratic(3, 200)
    At, bt = torch.tensor(A, device="cuda"), torch.tensor(b, device="cuda")

    def est_h(u, th, k):
        return 0.5 * u @ A @ u - b @ u, A @ u - b

    def est_d(u, th, k):
        return float(0.5 * u @ (At @ u) - bt @ u), At @ u - bt

    rh = slbfgs_run(est_h, np.zeros(200), 40, nu=0.5)
    rd = slbfgs_run(est_d, torch.zeros(200, dtype=torch.float64, device="cuda"), 40, nu=0.5)
    assert torch.is_tensor(rd.u) and rd.u.is_cuda
    assert np.allclose(rh.energy, rd.energy, rtol=1e-9, atol=1e-13)
    assert np.linalg.norm(rd.u.cpu().numpy() - rh.u) <= 1e-9 * np.linalg.norm(rh.u)
