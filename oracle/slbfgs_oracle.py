"""CPU oracle for the SLBFGS optimizer (TEST INFRASTRUCTURE ONLY: imported by tests/, never by
the product path).

There is no reference code for the optimizer (spec only), so this is a
plain numpy restatement of the published algorithm, pinned by the SPEC's own examples
(tests/test_oracle_slbfgs.py):
  two_loop       standard L-BFGS two-loop product H_k g (Algorithm 2
                 "twoLoopRecursion"), H0 = gamma I with gamma = <s,y>/<y,y> of
                 the newest pair, identity when empty
  dense_bfgs     the dense-matrix oracle of SPEC.md:371: H <- (I - rho s y^T) H (I - rho y s^T)
                 + rho s s^T applied to H0 over the stored pairs
  slbfgs         Algorithm 2 with the SPEC curvature rejection
                 <s,y> > 1e-10 |s||y| and i^3 averaging from the first energy
                 increase
"""
from __future__ import annotations

import math
from typing import Callable, List, Tuple

import numpy as np


class Pairs:
    def __init__(self, m: int, reject_tol: float = 1e-10):
        self.m = m
        self.tol = reject_tol
        self.S: List[np.ndarray] = []
        self.Y: List[np.ndarray] = []
        self.gamma = 1.0

    def push(self, s, y) -> bool:
        s = np.asarray(s, dtype=np.float64).ravel()
        y = np.asarray(y, dtype=np.float64).ravel()
        sy = float(s @ y)
        if not (np.isfinite(sy) and sy > self.tol * np.linalg.norm(s) * np.linalg.norm(y) and y @ y > 0):
            return False
        self.S.append(s)
        self.Y.append(y)
        if len(self.S) > self.m:
            self.S.pop(0)
            self.Y.pop(0)
        self.gamma = sy / float(y @ y)
        return True


def two_loop(g, P: Pairs) -> np.ndarray:
    q = np.asarray(g, dtype=np.float64).ravel().copy()
    alpha = []
    for s, y in zip(reversed(P.S), reversed(P.Y)):
        a = (s @ q) / (y @ s)
        alpha.append(a)
        q -= a * y
    r = P.gamma * q if P.S else q
    for (s, y), a in zip(zip(P.S, P.Y), reversed(alpha)):
        b = (y @ r) / (y @ s)
        r += s * (a - b)
    return r


def dense_bfgs(P: Pairs) -> np.ndarray:
    n = P.S[0].size if P.S else 0
    H = P.gamma * np.eye(n)
    for s, y in zip(P.S, P.Y):
        rho = 1.0 / (y @ s)
        V = np.eye(n) - rho * np.outer(y, s)
        H = V.T @ H @ V + rho * np.outer(s, s)
    return H


def slbfgs(estimator: Callable[[np.ndarray, float, int], Tuple[float, np.ndarray]], u0, n_evl: int, nu: float = 1.0,
           m: int = 64, bounds=None, weight=lambda i: float(i) ** 3):
    u = np.array(u0, dtype=np.float64, copy=True).ravel()
    P = Pairs(m)
    u_bar = np.zeros_like(u)
    w_bar = 0.0
    J_prev = math.inf
    energy = []
    average = False
    u_hat = u.copy()
    evl = i = 0
    while evl < n_evl:
        i += 1
        F_u, G_u = estimator(u, 0.0, i)
        evl += 1
        z = -two_loop(G_u, P)
        F_z, G_z = estimator(u + nu * z, 0.0, i)
        evl += 1
        P.push(nu * z, np.asarray(G_z).ravel() - np.asarray(G_u).ravel())
        z = z - two_loop(G_z, P)
        u = u + nu * z
        if bounds is not None:
            u = np.maximum(np.minimum(u, bounds[1]), bounds[0])
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
            u_hat = u.copy()
        J_prev = J
    return u_hat, energy, evl
