"""Host-side optimizer logic (no device): the SPEC.md optimizer examples for line_search and
the SGD / SGD-with-inertia baselines."""
import numpy as np

from paper_2102_00755_b200.optim import line_search, sgd_momentum_run, sgd_run


def quad(a=2.0, b=1.0):
    def f(u):
        u = np.asarray(u, dtype=np.float64)
        return 0.5 * a * float(u @ u) - b * float(u.sum()), a * u - b
    return f


def test_line_search_exact_step_accepts_immediately():
    # quadratic with nu0 at the exact minimiser step -> accepted at once, 1 evaluation
    a, b = 2.0, 1.0
    f = quad(a, b)
    u = np.array([3.0, -1.0])
    F0, G0 = f(u)
    z = -G0
    nu_star = 1.0 / a
    F, G, nu, evals, ok = line_search(f, u, z, nu_star, F0, G0)
    assert ok and evals == 1 and nu == nu_star


def test_line_search_large_step_backtracks_near_the_line_minimum():
    a = 2.0
    f = quad(a, 0.0)
    u = np.array([1.0, 2.0, -0.5])
    F0, G0 = f(u)
    z = -G0
    nu_star = 1.0 / a
    F, G, nu, evals, ok = line_search(f, u, z, 100.0 * nu_star, F0, G0)
    assert ok and nu_star / 2 <= nu <= 2 * nu_star and F < F0


def test_line_search_flags_non_descent():
    f = quad()
    u = np.array([1.0, 1.0])
    F0, G0 = f(u)
    F, G, nu, evals, ok = line_search(f, u, G0, 0.1, F0, G0)
    assert not ok


def test_sgd_converges_monotonically_below_2_over_L():
    rng = np.random.default_rng(3)
    Q = rng.standard_normal((10, 10))
    A = Q @ Q.T + np.eye(10)
    b = rng.standard_normal(10)
    L = np.linalg.eigvalsh(A).max()

    def est(u, th, k):
        return 0.5 * u @ A @ u - b @ u, A @ u - b

    res = sgd_run(est, np.zeros(10), 60, nu=1.0 / L)
    e = np.array(res.energy)
    assert np.all(np.diff(e) <= 1e-12) and res.averaging_from is None


def test_inertia_reaches_tolerance_in_fewer_iterations():
    rng = np.random.default_rng(4)
    Q = rng.standard_normal((20, 20))
    A = Q @ Q.T / 20 + 0.05 * np.eye(20)
    b = rng.standard_normal(20)
    ustar = np.linalg.solve(A, b)
    L = np.linalg.eigvalsh(A).max()

    def est(u, th, k):
        return 0.5 * u @ A @ u - b @ u, A @ u - b

    def iters_to(tol, beta):
        u = np.zeros(20)
        v = np.zeros(20)
        for i in range(1, 5000):
            g = A @ u - b
            v = beta * v - (1.0 / L) * g
            u = u + v
            if np.linalg.norm(u - ustar) < tol:
                return i
        return 5000

    assert iters_to(1e-6, 0.5) < iters_to(1e-6, 0.0)
    # and the library's momentum run equals this recursion
    r = sgd_momentum_run(est, np.zeros(20), 30, nu=1.0 / L, beta=0.5)
    u = np.zeros(20)
    v = np.zeros(20)
    for _ in range(30):
        v = 0.5 * v - (1.0 / L) * (A @ u - b)
        u = u + v
    # averaging is off while the energy decreases monotonically
    assert r.averaging_from is None and np.allclose(r.u, u, rtol=1e-12, atol=1e-15)
