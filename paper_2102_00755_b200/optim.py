"""Stochastic L-BFGS (Algorithm 2, Appendix D) and the SGD baselines (§4.4), the
direct caller of the encoded-gradient estimator (SPEC.md optimizer
module).

The curvature history (S, Y rings of m_h = 64 fp64 vectors, rho_i, H0 = gamma I) lives on
the device behind the C ABI (`ustfwi_lbfgs_*`, csrc/lbfgs.cu); the two-loop recursion runs
there. The iterate bookkeeping (projection, averaging, energy history) runs on whatever the
caller's vectors are: numpy arrays (host) or torch CUDA fp64 tensors, in which case every
vector of Algorithm 2 stays in HBM (push / apply pass device pointers, no transfers).

Estimator contract (Algorithm 2 inputs): ``estimator(u, theta, n) -> (F, G)`` where the same
``(theta, n)`` selects the same stochastic approximation (seed pairing).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Tuple

import numpy as np

from .capi import check, lib, ptr

Estimator = Callable[[np.ndarray, float, int], Tuple[float, np.ndarray]]


def _is_cuda(x) -> bool:
    return type(x).__module__.split(".")[0] == "torch" and bool(getattr(x, "is_cuda", False))


class _Np:
    """Vector ops of Algorithm 2 on numpy (host)."""
    @staticmethod
    def vec(x, shape):
        return np.asarray(x, dtype=np.float64).reshape(shape)

    copy = staticmethod(lambda x: np.array(x, dtype=np.float64, copy=True))
    zeros_like = staticmethod(np.zeros_like)
    norm = staticmethod(lambda x: float(np.linalg.norm(x)))
    dot = staticmethod(lambda a, b: float(np.dot(a.ravel(), b.ravel())))
    clip = staticmethod(lambda u, lo, hi: np.maximum(np.minimum(u, hi), lo))


class _Torch:
    """The same ops on torch CUDA fp64 tensors (device-resident iterates)."""
    @staticmethod
    def vec(x, shape):
        return x.to(dtype=__import__("torch").float64).reshape(shape)

    copy = staticmethod(lambda x: x.detach().clone().to(dtype=__import__("torch").float64))
    zeros_like = staticmethod(lambda x: __import__("torch").zeros_like(x))
    norm = staticmethod(lambda x: float(__import__("torch").linalg.vector_norm(x)))
    dot = staticmethod(lambda a, b: float(__import__("torch").dot(a.reshape(-1), b.reshape(-1))))
    clip = staticmethod(lambda u, lo, hi: __import__("torch").clamp(u, lo, hi))


def _ops(x):
    return _Torch if _is_cuda(x) else _Np


class DeviceLbfgs:
    """LbfgsState (SPEC.md optimizer) with the buffers in HBM."""

    def __init__(self, n: int, history: int = 64, device: int = 0, reject_tol: float = 1e-10):
        L = lib()
        L.ustfwi_lbfgs_create.argtypes = [C.c_int, C.c_size_t, C.c_int, C.POINTER(C.c_void_p)]
        L.ustfwi_lbfgs_destroy.argtypes = [C.c_void_p]
        L.ustfwi_lbfgs_reset.argtypes = [C.c_void_p]
        L.ustfwi_lbfgs_push.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.POINTER(C.c_int)]
        L.ustfwi_lbfgs_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ustfwi_lbfgs_pairs.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double)]
        self.n = int(n)
        self.history = int(history)
        self.reject_tol = float(reject_tol)
        h = C.c_void_p()
        check(L.ustfwi_lbfgs_create(int(device), self.n, self.history, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().ustfwi_lbfgs_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def reset(self):
        check(lib().ustfwi_lbfgs_reset(self._h))

    def push(self, s: np.ndarray, y: np.ndarray) -> bool:
        """updateBuffer(s, S), updateBuffer(y, Y); False when the curvature pair is rejected.
        Host arrays or torch CUDA tensors (device pointers, no transfer)."""
        if _is_cuda(s):
            import torch
            s = s.detach().to(torch.float64).contiguous().reshape(-1)
            y = y.detach().to(torch.float64).contiguous().reshape(-1)
            if s.numel() != self.n or y.numel() != self.n:
                raise ValueError("pair length does not match the state")
            torch.cuda.current_stream(s.device).synchronize()
            ok = C.c_int(0)
            check(lib().ustfwi_lbfgs_push(self._h, C.c_void_p(s.data_ptr()), C.c_void_p(y.data_ptr()),
                                          self.reject_tol, C.byref(ok)))
            return bool(ok.value)
        s = np.ascontiguousarray(s, dtype=np.float64).ravel()
        y = np.ascontiguousarray(y, dtype=np.float64).ravel()
        if s.size != self.n or y.size != self.n:
            raise ValueError("pair length does not match the state")
        ok = C.c_int(0)
        check(lib().ustfwi_lbfgs_push(self._h, ptr(s, C.c_double), ptr(y, C.c_double), self.reject_tol,
                                      C.byref(ok)))
        return bool(ok.value)

    def apply(self, g: np.ndarray) -> np.ndarray:
        """H_k g by the two-loop recursion (Algorithm 2 twoLoopRecursion); a torch CUDA tensor
        in gives a torch CUDA tensor out (device pointers, no transfer)."""
        if _is_cuda(g):
            import torch
            gd = g.detach().to(torch.float64).contiguous().reshape(-1)
            if gd.numel() != self.n:
                raise ValueError("vector length does not match the state")
            out = torch.empty_like(gd)
            torch.cuda.current_stream(gd.device).synchronize()
            check(lib().ustfwi_lbfgs_apply(self._h, C.c_void_p(gd.data_ptr()), C.c_void_p(out.data_ptr())))
            return out
        g = np.ascontiguousarray(g, dtype=np.float64).ravel()
        if g.size != self.n:
            raise ValueError("vector length does not match the state")
        out = np.empty_like(g)
        check(lib().ustfwi_lbfgs_apply(self._h, ptr(g, C.c_double), ptr(out, C.c_double)))
        return out

    def pairs(self) -> Tuple[int, float]:
        cnt = C.c_int(0)
        gam = C.c_double(0.0)
        check(lib().ustfwi_lbfgs_pairs(self._h, C.byref(cnt), C.byref(gam)))
        return cnt.value, gam.value


@dataclass
class OptResult:
    u: np.ndarray                    # \\hat u (weighted average once active, else last iterate)
    energy: List[float]              # J_i
    n_evl: int
    iterations: int
    averaging_from: Optional[int]    # iteration at which averaging became active
    log: List[dict] = field(default_factory=list)


def _project(u, bounds):
    if bounds is None:
        return u
    lo, hi = bounds
    return _ops(u).clip(u, lo, hi)


def line_search(f: Callable[[np.ndarray], Tuple[float, np.ndarray]], u: np.ndarray, z: np.ndarray, nu0: float,
                F0: float, G0: np.ndarray, c1: float = 1e-4, max_trials: int = 8):
    """Backtracking Armijo search (SPEC.md optimizer line_search): halving from nu0, at most
    8 trials. Returns (F, G, nu, evals, ok)."""
    slope = _ops(z).dot(G0, z)
    if not slope < 0.0:
        F, G = f(u + nu0 * z)
        return F, G, nu0, 1, False
    nu = nu0
    for t in range(1, max_trials + 1):
        F, G = f(u + nu * z)
        if F <= F0 + c1 * nu * slope:
            return F, G, nu, t, True
        if t < max_trials:
            nu *= 0.5
    return F, G, nu, max_trials, False


def slbfgs_run(estimator: Estimator, u0: np.ndarray, n_evl: int, nu: float = 1.0, history: int = 64,
               bounds=None, theta: Callable[[int], float] = lambda i: 0.0,
               weight: Callable[[int], float] = lambda i: float(i) ** 3, do_linesearch: bool = False,
               device: int = 0, reject_tol: float = 1e-10, h0: float = 1.0) -> OptResult:
    """Algorithm 2: per iteration two estimator calls with the same
    (theta(i), i), pair (nu z, G_z - G_u), second update z <- z - H_k G_z, projection,
    J_i = min(F_u, F_z), i^3 averaging from the first energy increase.

    H_0 (an Algorithm 2 input): h0 * I while the buffer is empty, then the standard
    gamma = <s,y>/<y,y> scaling of the newest pair. The step size nu multiplies
    both updates, so with gradients not in parameter units keep nu = 1 and put the scale of
    the first step into h0."""
    X = _ops(u0)
    u = X.copy(u0)
    shape = tuple(u.shape)
    u_bar = X.zeros_like(u)
    w_bar = 0.0
    J_prev = math.inf
    energy: List[float] = []
    log: List[dict] = []
    average = False
    avg_from = None
    u_hat = X.copy(u)
    evl = 0
    i = 0
    n = int(np.prod(shape)) if shape else 1
    with DeviceLbfgs(n, history, device, reject_tol) as H:
        def apply_h(g):
            r = H.apply(g).reshape(shape)
            return h0 * r if H.pairs()[0] == 0 else r

        while evl < n_evl:
            i += 1
            th = theta(i)
            F_u, G_u = estimator(u, th, i)
            evl += 1
            G_u = X.vec(G_u, shape)
            z = -apply_h(G_u)
            step = nu
            if do_linesearch:
                F_z, G_z, step, m_evl, _ = line_search(lambda v: estimator(v, th, i), u, z, nu, F_u, G_u)
            else:
                F_z, G_z = estimator(u + nu * z, th, i)
                m_evl = 1
            evl += m_evl
            G_z = X.vec(G_z, shape)
            accepted = H.push(step * z, G_z - G_u)
            z = z - apply_h(G_z)
            u = _project(u + step * z, bounds)
            J = min(F_u, F_z)
            energy.append(J)
            if average:
                w = weight(i)
                u_bar += w * u
                w_bar += w
                u_hat = u_bar / w_bar
            else:
                if J > J_prev:
                    average = True
                    avg_from = i + 1
                u_hat = X.copy(u)
            J_prev = J
            log.append({"iter": i, "n_evl": evl, "J": J, "step_norm": X.norm(step * z),
                        "grad_norm": X.norm(G_u), "averaging_active": average,
                        "pair_accepted": accepted})
    return OptResult(u_hat, energy, evl, i, avg_from, log)


def sgd_run(estimator: Estimator, u0: np.ndarray, n_evl: int, nu: float, beta: float = 0.0, bounds=None,
            theta: Callable[[int], float] = lambda i: 0.0,
            weight: Callable[[int], float] = lambda i: float(i) ** 3) -> OptResult:
    """Plain SGD (beta = 0) and SGD with momentum v <- beta v - nu g, u <- clip(u + v)
    (§4.4 baselines, beta = 0.5 there; SPEC.md sgd_run / sgd_momentum_run), with the
    same averaging rule as SLBFGS."""
    u = np.array(u0, dtype=np.float64, copy=True)
    v = np.zeros_like(u)
    u_bar = np.zeros_like(u)
    w_bar = 0.0
    J_prev = math.inf
    energy: List[float] = []
    average = False
    avg_from = None
    u_hat = u.copy()
    for i in range(1, n_evl + 1):
        F, G = estimator(u, theta(i), i)
        v = beta * v - nu * np.asarray(G, dtype=np.float64).reshape(u.shape)
        u = _project(u + v, bounds)
        energy.append(F)
        if average:
            w = weight(i)
            u_bar += w * u
            w_bar += w
            u_hat = u_bar / w_bar
        else:
            if F > J_prev:
                average = True
                avg_from = i + 1
            u_hat = u.copy()
        J_prev = F
    return OptResult(u_hat, energy, n_evl, n_evl, avg_from)


def sgd_momentum_run(estimator: Estimator, u0: np.ndarray, n_evl: int, nu: float, beta: float = 0.5, **kw):
    return sgd_run(estimator, u0, n_evl, nu, beta=beta, **kw)
