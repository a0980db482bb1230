"""Encoded-gradient estimators as Algorithm 2's estimator (SPEC.md stochastic_estimators
:272-347; §3.2, §4.4).

``EncodedEstimator(u, theta, i)`` draws the realizations (master_seed, iteration i, index k)
for k < batch with maximal delay tau = theta (seed pairing: both calls of an SLBFGS iteration
see the same realizations), encodes the per-source observed data to f^ over
nt + ceil(tau/dt) samples, evaluates each encoded TR gradient on the device
over that extended duration, and returns the mean (F, G) restricted to the unknowns.
``delay_schedule(b)`` is the paper's tau = b (i - 1).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np

from .engine import GpuEngine, Medium, SensorArray, SourceSet, draw_realization, encode


def delay_schedule(b: float) -> Callable[[int], float]:
    """tau(i) = b (i - 1) seconds; b = 0 recovers conventional source encoding."""
    if b < 0:
        raise ValueError("b must be non-negative")
    return lambda i: b * (i - 1)


class EncodedEstimator:
    """estimator(u, theta, i) -> (F, G) of the c0 unknowns inside `mask` (flat boolean),
    one or more encoded TR gradients per call on one engine."""

    def __init__(self, engine: GpuEngine, medium: Medium, sources: SourceSet, data: Sequence[np.ndarray],
                 sensors: SensorArray, thickness: int, mask: np.ndarray, master_seed: int = 20210201,
                 batch: int = 1, c0_bounds: Optional[tuple] = None):
        self.eng = engine
        self.medium = medium
        self.sources = sources
        self.data = [np.asarray(f, np.float64) for f in data]
        self.sensors = sensors
        self.thickness = int(thickness)
        self.mask = np.asarray(mask, bool).ravel()
        self.seed = int(master_seed)
        self.batch = int(batch)
        self.bounds = c0_bounds
        self.nt = int(engine.grid.nt)
        self.dt = float(engine.grid.dt)
        self.base_c0 = np.asarray(medium.c0, np.float64).ravel().copy()
        self.history: List[dict] = []   # per call: iteration, tau, nt_ext, loss

    def medium_of(self, u: np.ndarray) -> Medium:
        c0 = self.base_c0.copy()
        v = np.asarray(u, np.float64).ravel()
        if self.bounds is not None:
            v = np.clip(v, *self.bounds)
        c0[self.mask] = v
        m = self.medium
        return Medium(c0=c0.reshape(m.c0.shape), rho0=m.rho0, alpha0=m.alpha0, y=m.y, gamma=m.gamma,
                      c0_min=m.c0_min, c0_max=m.c0_max)

    def __call__(self, u: np.ndarray, theta: float, i: int):
        eng = self.eng
        eng.set_medium(self.medium_of(u))
        eng.set_sensors(self.sensors)
        F = 0.0
        G = np.zeros(int(self.mask.sum()))
        for k in range(self.batch):
            r = draw_realization(len(self.sources.positions), float(theta), self.dt, self.seed, int(i), k)
            enc, f_hat, nt_ext = encode(self.sources, self.data, r, self.nt)
            if nt_ext != eng.grid.nt:
                eng.set_nt(nt_ext)
            eng.set_sources(enc)
            loss, grad = eng.gradient_tr(f_hat, self.thickness)
            F += loss
            G += grad.ravel()[self.mask]
            self.history.append({"iteration": int(i), "tau": float(theta), "nt_ext": int(nt_ext), "loss": loss})
        return F / self.batch, G / self.batch
