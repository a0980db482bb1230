"""The SLBFGS oracle against the SPEC's own examples — pins the CPU
restatement used by the GPU optimizer tests."""
import numpy as np

from oracle import slbfgs_oracle as so


def test_empty_buffers_give_identity():
    g = np.arange(5.0)
    assert np.array_equal(so.two_loop(g, so.Pairs(64)), g)


def test_one_dimensional_quadratic_secant():
    # J = a u^2 / 2, one stored pair -> direction g / a exactly
    a = 3.7
    P = so.Pairs(64)
    u0, u1 = np.array([2.0]), np.array([0.5])
    assert P.push(u1 - u0, a * u1 - a * u0)
    g = np.array([1.3])
    assert abs(so.two_loop(g, P)[0] - g[0] / a) < 1e-15


def test_two_loop_matches_dense_bfgs_on_spd():
    # random SPD 5x5 with 3 pairs, 1e-10
    rng = np.random.default_rng(0)
    A = rng.standard_normal((5, 5))
    A = A @ A.T + 5 * np.eye(5)
    P = so.Pairs(64)
    for _ in range(3):
        s = rng.standard_normal(5)
        assert P.push(s, A @ s)
    g = rng.standard_normal(5)
    assert np.linalg.norm(so.two_loop(g, P) - so.dense_bfgs(P) @ g) <= 1e-10 * np.linalg.norm(g)


def test_non_curvature_pair_is_rejected():
    P = so.Pairs(4)
    assert not P.push(np.array([1.0, 0.0]), np.array([-1.0, 0.0]))
    assert len(P.S) == 0


def test_deterministic_quadratic_converges():
    # 100-dim convex quadratic, theta = 0: |u - u*| < 1e-8 within 50 evaluations
    rng = np.random.default_rng(1)
    Q = rng.standard_normal((100, 100))
    A = Q @ Q.T / 100 + np.eye(100)
    b = rng.standard_normal(100)
    ustar = np.linalg.solve(A, b)

    def est(u, th, n):
        return 0.5 * u @ A @ u - b @ u, A @ u - b

    u, energy, evl = so.slbfgs(est, np.zeros(100), 50, nu=0.5)
    assert evl <= 50 and np.linalg.norm(u - ustar) < 1e-8


def test_bounds_clip_onto_active_face():
    # minimizer outside the box -> the projected point
    target = np.array([2.0, -3.0, 0.25])

    def est(u, th, n):
        return 0.5 * np.sum((u - target) ** 2), u - target

    u, _, _ = so.slbfgs(est, np.zeros(3), 20, nu=1.0, bounds=(-1.0, 1.0))
    assert np.allclose(u, [1.0, -1.0, 0.25], atol=1e-12)
