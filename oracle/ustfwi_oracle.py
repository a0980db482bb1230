"""CPU restatement of the reference hot path in numpy (fp64) — TEST INFRASTRUCTURE ONLY.

This is the oracle the GPU engine is checked against. It restates, function by function,
the reference C++ (`/root/reference/proj/include/ustfwi`, paths below relative to it):

  wavenumbers          core/fft.hpp:121-130
  sinc / kappa         grid/grid.hpp:106-109, solver/engine.hpp:35-44
  derivative mults     solver/engine.hpp:46-78 (Nyquist: real part / zero)
  make_pml             grid/grid.hpp:153-178
  Stepper              solver/engine.hpp:184-347 (lossless branch; absorption is out of scope)
  simulate_forward     solver/simulate.hpp:30-105
  adjoint_source       adjoint/gradient.hpp:264-289
  gradient_tr          adjoint/gradient.hpp:333-464 (TR branch, GradientParam::c0)

numpy's pocketfft rfftn/irfftn have FFTW's r2c/c2r semantics (half spectrum on the last
axis, unnormalised forward, 1/N inverse). Pinned against the reference itself through the
golden fixtures in tests/golden (generated from oracle/_ref by tests/golden/make_golden.py)
and against the reference's own known-answer tests (oracle/_ref/unit_tests).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use this module.
"""
from __future__ import annotations

import math

import numpy as np


def wavenumbers(n: int, dx: float) -> np.ndarray:
    """core/fft.hpp:121-130: FFT order, Nyquist bin negative."""
    m = np.arange(n)
    m = np.where(m < n // 2, m, m - n)
    return 2.0 * math.pi / (n * dx) * m


def sinc(x):
    """grid/grid.hpp:106-109."""
    x = np.asarray(x, dtype=np.float64)
    small = np.abs(x) < 1e-8
    safe = np.where(small, 1.0, x)
    return np.where(small, 1.0 - x * x / 6.0, np.sin(safe) / safe)


def pml_profiles(n: int, layer: int, dx: float, dt: float, c_ref: float, alpha: float = 2.0):
    """grid/grid.hpp:153-178 -> (regular, staggered)."""
    def prof(u):
        if layer < 2:
            return np.ones_like(u)
        inner = float(layer - 1)
        ramp = np.where(u < inner, (inner - u) / inner, 0.0)
        ur = (n - 1) - u
        ramp = np.maximum(ramp, np.where(ur < inner, (inner - ur) / inner, 0.0))
        sigma = alpha * (c_ref / dx) * ramp ** 4
        return np.exp(-sigma * dt / 2.0)
    i = np.arange(n, dtype=np.float64)
    return prof(i), prof(i + 0.5)


class Grid:
    def __init__(self, dims, dx, dt, nt, pml_size, c_ref):
        self.dims = tuple(int(d) for d in dims)
        self.dx = [float(dx)] * len(self.dims) if np.isscalar(dx) else [float(v) for v in dx]
        self.dt = float(dt)
        self.nt = int(nt)
        self.pml_size = [int(p) for p in pml_size]
        self.c_ref = float(c_ref)

    @classmethod
    def of(cls, g):
        nd = g.ndim
        return cls([g.dims[a] for a in range(nd)], [g.dx[a] for a in range(nd)], g.dt, g.nt,
                   [g.pml_size[a] for a in range(nd)], g.c_ref)

    @property
    def ndim(self):
        return len(self.dims)


class SpectralEngine:
    """solver/engine.hpp:17-151 (half-spectrum multipliers)."""

    def __init__(self, g: Grid):
        self.g = g
        nd = g.ndim
        k = [wavenumbers(g.dims[a], g.dx[a]) for a in range(nd)]
        half = list(g.dims)
        half[-1] = g.dims[-1] // 2 + 1
        self.half = tuple(half)
        kk = []
        for a in range(nd):
            ka = k[a][: half[a]] if a == nd - 1 else k[a]
            shp = [1] * nd
            shp[a] = half[a]
            kk.append(ka.reshape(shp))
        k2 = sum(x * x for x in kk)
        self.kappa = sinc(0.5 * g.c_ref * g.dt * np.sqrt(k2))
        self.mult = {}
        for a in range(nd):
            n = g.dims[a]
            ka = kk[a]
            idx = np.arange(half[a]).reshape([half[a] if b == a else 1 for b in range(nd)])
            nyq = idx == n // 2
            base = 1j * ka * self.kappa
            h = 0.5 * g.dx[a]
            plus = base * np.exp(1j * ka * h)
            minus = base * np.exp(-1j * ka * h)
            self.mult[(a, "none")] = np.where(nyq, 0.0, base)
            self.mult[(a, "plus")] = np.where(nyq, plus.real, plus)
            self.mult[(a, "minus")] = np.where(nyq, minus.real, minus)

    def fwd(self, f):
        return np.fft.rfftn(f)

    def inv(self, s):
        return np.fft.irfftn(s, s=self.g.dims, axes=list(range(len(self.g.dims))))

    def derivative(self, f, axis, stagger):
        """engine.hpp:118-121."""
        return self.inv(self.fwd(f) * self.mult[(axis, stagger)])


def fourier_shift_half(field, axis, dx):
    """spectral.hpp:94-112 with shift +1/2 cell (the staggered density, engine.hpp:219-231)."""
    n = field.shape[axis]
    ka = wavenumbers(n, dx)
    m = np.exp(1j * ka * 0.5 * dx)
    m[n // 2] = m[n // 2].real
    shp = [1] * field.ndim
    shp[axis] = n
    spec = np.fft.fftn(field.astype(np.complex128))
    return np.fft.ifftn(spec * m.reshape(shp)).real


class Stepper:
    """WaveStepper, lossless branch (engine.hpp:184-347)."""

    def __init__(self, g: Grid, c0, rho0, eng: SpectralEngine):
        self.g, self.eng = g, eng
        nd = g.ndim
        self.c0_sq = c0 * c0
        self.dt_rho0 = g.dt * rho0
        uniform = np.all(rho0 == rho0.flat[0])
        self.dt_over_rho_stag = []
        for a in range(nd):
            sh = rho0 if uniform else fourier_shift_half(rho0, a, g.dx[a])
            self.dt_over_rho_stag.append(g.dt / sh)
        self.pml_reg, self.pml_stag = [], []
        for a in range(nd):
            r, s = pml_profiles(g.dims[a], g.pml_size[a], g.dx[a], g.dt, g.c_ref)
            shp = [1] * nd
            shp[a] = g.dims[a]
            self.pml_reg.append(r.reshape(shp))
            self.pml_stag.append(s.reshape(shp))
        self.v = [np.zeros(g.dims) for _ in range(nd)]
        self.rho = [np.zeros(g.dims) for _ in range(nd)]
        self.p = np.zeros(g.dims)
        self.step_index = 0

    def update_velocity_density(self):
        nd = self.g.ndim
        P = self.eng.fwd(self.p)
        for a in range(nd):
            ga = self.eng.inv(P * self.eng.mult[(a, "plus")])
            pm = self.pml_stag[a]
            self.v[a] = pm * (pm * self.v[a] - self.dt_over_rho_stag[a] * ga)
        for a in range(nd):
            du = self.eng.derivative(self.v[a], a, "minus")
            pm = self.pml_reg[a]
            self.rho[a] = pm * (pm * self.rho[a] - self.dt_rho0 * du)

    def inject_mass_source(self, flat_index, amp):
        """engine.hpp:296-300."""
        scale = 2.0 * self.g.dt / (self.g.ndim * self.g.dx[0] * math.sqrt(self.c0_sq.flat[flat_index]))
        for r in self.rho:
            r.flat[flat_index] += amp * scale

    def enforce_shell(self, shell, values):
        """engine.hpp:304-307."""
        for r in self.rho:
            r.flat[shell] = values

    def refresh_pressure(self):
        """engine.hpp:311-316."""
        s = np.zeros(self.g.dims)
        for r in self.rho:
            s += r
        self.p = self.c0_sq * s

    def update_pressure(self):
        """engine.hpp:318-347 (lossless)."""
        self.refresh_pressure()
        self.step_index += 1
        if (self.step_index & 63) == 0 and not np.isfinite(self.p.flat[0]):
            raise FloatingPointError(f"pressure field diverged at step {self.step_index}")


def _sample(sig, n):
    return sig[n] if 0 <= n < len(sig) else 0.0


def simulate_forward(g: Grid, c0, rho0, positions, signals, sensors, shell=None, weights=None, delays=None):
    """simulate.hpp:76-103 -> (data [ns, nt], trace [nt, n_shell] or None). Encoded sources:
    sample = w_i * s_i(n - d_i)."""
    eng = SpectralEngine(g)
    st = Stepper(g, c0, rho0, eng)
    ns = len(sensors)
    data = np.zeros((ns, g.nt))
    trace = np.zeros((g.nt, len(shell))) if shell is not None else None
    for n in range(g.nt):
        st.update_velocity_density()
        for i, pos in enumerate(positions):
            w = 1.0 if weights is None else weights[i]
            d = 0 if delays is None else int(delays[i])
            amp = w * _sample(signals[i], n - d)
            if amp != 0.0:
                st.inject_mass_source(pos, amp)
        st.update_pressure()
        data[:, n] = st.p.flat[np.asarray(sensors, dtype=np.int64)]
        if trace is not None:
            trace[n] = st.p.flat[shell]
    if not np.all(np.isfinite(data)):
        raise FloatingPointError("sensor data contains non-finite values")
    return data, trace


def adjoint_source(sim, obs, integrate=True):
    """gradient.hpp:264-289 -> (q [nt, ns], loss); Kahan loss in (n, s) order."""
    ns, nt = sim.shape
    r = (sim - obs)[:, ::-1].T.copy()  # q[n][s] = r[s][nt-1-n]
    loss, comp = 0.0, 0.0
    for v in (0.5 * r * r).ravel():
        term = v - comp
        t = loss + term
        comp = (t - loss) - term
        loss = t
    q = np.cumsum(r, axis=0) if integrate else r
    return q, loss


def gradient_tr(g: Grid, c0, rho0, gamma, positions, signals, sensors, observed, thickness, shell,
                weights=None, delays=None):
    """compute_gradient TR branch (gradient.hpp:359-462), c0 parameter -> (loss, grad)."""
    data, trace = simulate_forward(g, c0, rho0, positions, signals, sensors, shell, weights, delays)
    q, loss = adjoint_source(data, observed)
    eng = SpectralEngine(g)
    adj = Stepper(g, c0, rho0, eng)
    rep = Stepper(g, c0, rho0, eng)
    c2 = c0 * c0
    g_scaled = trace / (g.ndim * c2.flat[shell])[None, :]
    w_ddot = 2.0 / c0 ** 3
    grad = np.zeros(g.dims)
    last = g.nt - 1
    inv_dt = 1.0 / g.dt
    rep.enforce_shell(shell, g_scaled[last])
    rep.refresh_pressure()
    window = [rep.p.copy()]
    rep.update_velocity_density()
    rep.enforce_shell(shell, g_scaled[last - 1])
    rep.update_pressure()
    window.insert(0, rep.p.copy())
    sens = np.asarray(sensors, dtype=np.int64)
    for n in range(1, last):
        adj.update_velocity_density()
        for s, pos in enumerate(sens):
            if q[n, s] != 0.0:
                adj.inject_mass_source(pos, q[n, s])
        adj.update_pressure()
        rep.update_velocity_density()
        rep.enforce_shell(shell, g_scaled[last - n - 1])
        rep.update_pressure()
        window.insert(0, rep.p.copy())
        window = window[:3]
        newer, mid, older = window
        grad += w_ddot * ((newer - 2.0 * mid + older) * inv_dt) * adj.p
    grad = np.where(np.asarray(gamma, bool), grad, 0.0)
    return loss, grad
