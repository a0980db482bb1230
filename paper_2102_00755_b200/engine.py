"""Python mirror of the reference hot-path API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/ustfwi):

  Medium / SourceSet / SensorArray         solver/medium.hpp:26-91
  GpuEngine  (device SpectralEngine+steppers) solver/engine.hpp:17-386
  simulate_forward                         solver/simulate.hpp:30-105
  gradient_time_reversal                   adjoint/gradient.hpp:478-488 (-> compute_gradient :333-464)
  evaluate_loss                            adjoint/gradient.hpp:491-505
  encode / encoded_gradient / average_estimates   SPEC.md stochastic_estimators :296-322

Every compute call goes through libustfwi_b200.so; nothing here computes on the CPU
beyond argument marshalling.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import capi
from .capi import NumericalError, UstfwiGrid, check, lib, ptr

__all__ = [
    "Medium", "SourceSet", "SensorArray", "GpuEngine", "make_homogeneous_medium",
    "simulate_forward", "gradient_time_reversal", "evaluate_loss", "EncodingRealization",
    "draw_realization", "encode", "encoded_gradient", "average_estimates", "NumericalError",
]


@dataclass
class Medium:
    """solver/medium.hpp:26-58 (alpha0 in dB/(MHz^y cm); lossless when None)."""
    c0: np.ndarray
    rho0: np.ndarray
    alpha0: Optional[np.ndarray] = None
    y: float = 1.5
    gamma: Optional[np.ndarray] = None
    c0_min: float = 1350.0
    c0_max: float = 1800.0


def make_homogeneous_medium(g: UstfwiGrid, c0=1500.0, rho0=1000.0, alpha0=0.0, y=1.5) -> Medium:
    """make_homogeneous_medium (medium.hpp:60-70)."""
    shape = g.shape
    return Medium(c0=np.full(shape, c0), rho0=np.full(shape, rho0),
                  alpha0=None if alpha0 == 0.0 else np.full(shape, alpha0), y=y,
                  c0_min=min(1350.0, c0), c0_max=max(1800.0, c0))


@dataclass
class SourceSet:
    """solver/medium.hpp:74-85: positions are flat row-major indices; signals read as zero
    past their end. weights/delays (encoded super-source) default to 1 / 0."""
    positions: Sequence[int]
    signals: Sequence[np.ndarray]
    weights: Optional[np.ndarray] = None
    delays: Optional[np.ndarray] = None

    def count(self):
        return len(self.positions)


@dataclass
class SensorArray:
    """solver/medium.hpp:88-91."""
    positions: Sequence[int]

    def count(self):
        return len(self.positions)


class GpuEngine:
    """One device context: the analogue of a SpectralEngine plus its WaveSteppers.
    Not thread-safe; one per worker (engine.hpp:14-16)."""

    def __init__(self, grid: UstfwiGrid, device: int = 0):
        self.grid = grid
        self.device = device
        h = C.c_void_p()
        check(lib().ustfwi_gpu_create(int(device), C.byref(grid), C.byref(h)))
        self._h = h
        self.n_sensors = 0
        self._gamma = None

    # -- lifecycle ---------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().ustfwi_gpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    # -- state ------------------------------------------------------------------------
    def set_medium(self, m: Medium):
        n = self.grid.points
        c0 = np.ascontiguousarray(m.c0, dtype=np.float64).ravel()
        rho0 = np.ascontiguousarray(m.rho0, dtype=np.float64).ravel()
        if c0.size != n or rho0.size != n:
            raise ValueError("medium fields must match the grid")
        a0 = None
        a0p = None
        if m.alpha0 is not None:
            a0 = np.ascontiguousarray(m.alpha0, dtype=np.float64).ravel()
            if a0.size != n:
                raise ValueError("medium fields must match the grid")
            a0p = ptr(a0, C.c_double)
        gp = None
        if m.gamma is not None:
            gm = np.ascontiguousarray(m.gamma, dtype=np.uint8).ravel()
            if gm.size != n:
                raise ValueError("gamma mask must match the grid")
            gp = ptr(gm, C.c_uint8)
            self._gamma = gm.reshape(self.grid.shape)
        else:
            self._gamma = None
        check(lib().ustfwi_gpu_set_medium(self._h, ptr(c0, C.c_double), ptr(rho0, C.c_double), a0p,
                                          C.c_double(m.y), gp, C.c_double(m.c0_min), C.c_double(m.c0_max)))

    def set_sources(self, s: SourceSet):
        n = len(s.positions)
        pos = np.ascontiguousarray(s.positions, dtype=np.uint64)
        lens = [len(x) for x in s.signals]
        off = np.zeros(n + 1, dtype=np.uint64)
        off[1:] = np.cumsum(lens) if n else []
        sig = np.ascontiguousarray(np.concatenate([np.asarray(x, np.float64) for x in s.signals])
                                   if n and sum(lens) else np.zeros(1), dtype=np.float64)
        wp = dp = None
        if s.weights is not None:
            w = np.ascontiguousarray(s.weights, dtype=np.float64)
            wp = ptr(w, C.c_double)
        if s.delays is not None:
            d = np.ascontiguousarray(s.delays, dtype=np.int32)
            dp = ptr(d, C.c_int32)
        check(lib().ustfwi_gpu_set_sources(self._h, C.c_size_t(n), ptr(pos, C.c_size_t), ptr(off, C.c_size_t),
                                           ptr(sig, C.c_double), wp, dp))

    def set_nt(self, nt: int):
        """Simulation length of the following calls (Grid::nt): the encoded duration
        T + tau of a delayed realization. Observed data must be re-uploaded."""
        check(lib().ustfwi_gpu_set_nt(self._h, int(nt)))
        g = capi.UstfwiGrid.from_buffer_copy(self.grid)
        g.nt = int(nt)
        self.grid = g

    def set_sensors(self, s: SensorArray):
        pos = np.ascontiguousarray(s.positions, dtype=np.uint64)
        check(lib().ustfwi_gpu_set_sensors(self._h, C.c_size_t(len(pos)), ptr(pos, C.c_size_t)))
        self.n_sensors = len(pos)

    # -- hot path ---------------------------------------------------------------------
    def forward(self, boundary_thickness: int = 0, want_trace: bool = True):
        """-> (data [n_sensors, nt], trace [nt, n_shell] or None)."""
        nt = self.grid.nt
        data = np.zeros((self.n_sensors, nt))
        nsh = C.c_size_t(0)
        trace = None
        tp = None
        if boundary_thickness > 0 and want_trace:
            if self._gamma is None:
                raise ValueError("boundary recording requires a gamma mask")
            n_shell = len(capi.shell_indices(self._gamma, boundary_thickness))
            trace = np.zeros((nt, n_shell))
            tp = ptr(trace, C.c_double)
        check(lib().ustfwi_gpu_forward(self._h, int(boundary_thickness), ptr(data, C.c_double), tp, C.byref(nsh)))
        return data, trace

    def upload_observed(self, observed: np.ndarray):
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        if obs.shape != (self.n_sensors, self.grid.nt):
            raise ValueError("observed data dimensions do not match the simulation")
        check(lib().ustfwi_gpu_upload_observed(self._h, ptr(obs, C.c_double)))

    def run_gradient(self, thickness: int, accumulate: bool = False):
        check(lib().ustfwi_gpu_run_gradient(self._h, int(thickness), int(bool(accumulate))))

    def download_gradient(self, scale_div: float = 1.0):
        grad = np.empty(self.grid.shape)  # every element is written by the library
        loss = C.c_double(0.0)
        check(lib().ustfwi_gpu_download_gradient(self._h, C.c_double(scale_div), ptr(grad, C.c_double),
                                                 C.byref(loss)))
        return loss.value, grad

    PARAMS = {"c0": 0, "rho0": 1, "alpha0": 2, "y": 3}

    def gradient_tr(self, observed: np.ndarray, thickness: int, dispersion_enabled: bool = True,
                    param: str = "c0"):
        """-> (loss, grad) ; grad zero outside gamma. dispersion_enabled: GradientOptions
        (gradient.hpp:31), the adjoint / replay dispersion term of absorbing media; param:
        GradientParam c0 | rho0 | alpha0 | y (gradient.hpp:9)."""
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        if obs.shape != (self.n_sensors, self.grid.nt):
            raise ValueError("observed data dimensions do not match the simulation")
        if param not in self.PARAMS:
            raise ValueError("unknown gradient parameter")
        check(lib().ustfwi_gpu_set_gradient_options(self._h, int(bool(dispersion_enabled))))
        check(lib().ustfwi_gpu_set_gradient_param(self._h, self.PARAMS[param]))
        grad = np.empty(self.grid.shape)  # every element is written by the library
        loss = C.c_double(0.0)
        check(lib().ustfwi_gpu_gradient_tr(self._h, ptr(obs, C.c_double), int(thickness), ptr(grad, C.c_double),
                                           C.byref(loss)))
        return loss.value, grad

    def evaluate_loss(self, observed: np.ndarray) -> float:
        obs = np.ascontiguousarray(observed, dtype=np.float64)
        loss = C.c_double(0.0)
        check(lib().ustfwi_gpu_evaluate_loss(self._h, ptr(obs, C.c_double), C.byref(loss)))
        return loss.value

    def derivative(self, f: np.ndarray, axis: int, stagger: str = "none") -> np.ndarray:
        fa = np.ascontiguousarray(f, dtype=np.float64)
        out = np.zeros_like(fa)
        check(lib().ustfwi_gpu_derivative(self._h, ptr(fa, C.c_double), int(axis), capi.STAGGER[stagger],
                                          ptr(out, C.c_double)))
        return out

    # -- device-resident plumbing --------------------------------------------------------
    def synchronize(self):
        check(lib().ustfwi_gpu_synchronize(self._h))

    def stream_ptr(self) -> int:
        return int(lib().ustfwi_gpu_stream(self._h) or 0)

    def partition(self):
        """(adjoint SMs, replay SMs) of the TR pair loop's green contexts; (0, 0) = shared SMs."""
        a, r = C.c_int(0), C.c_int(0)
        check(lib().ustfwi_gpu_partition(self._h, C.byref(a), C.byref(r)))
        return a.value, r.value

    def launch_count(self) -> int:
        return int(lib().ustfwi_gpu_launch_count(self._h))

    def shell_size(self) -> int:
        return int(lib().ustfwi_gpu_shell_size(self._h))

    def set_profiling(self, enable: bool):
        check(lib().ustfwi_gpu_set_profiling(self._h, int(bool(enable))))

    def kernel_stats(self):
        """{kind: (total_ms, launches, algorithmic_bytes)} since set_profiling(True)."""
        out = {}
        for k, name in enumerate(capi.KERNEL_KINDS):
            ms = C.c_double(0)
            n = C.c_uint64(0)
            b = C.c_double(0)
            check(lib().ustfwi_gpu_kernel_stats(self._h, k, C.byref(ms), C.byref(n), C.byref(b)))
            out[name] = (ms.value, int(n.value), b.value)
        return out

    def accumulator(self):
        g = C.POINTER(C.c_float)()
        l = C.POINTER(C.c_double)()
        check(lib().ustfwi_gpu_accumulator(self._h, C.byref(g), C.byref(l)))
        return C.cast(g, C.c_void_p).value, C.cast(l, C.c_void_p).value

    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib().ustfwi_gpu_comm_init(self._h, buf, int(nranks), int(rank)))

    def batch_reserve(self, slots: int):
        """Per-realization gradient slots of a mini-batch (ustfwi_gpu_batch_reserve)."""
        check(lib().ustfwi_gpu_batch_reserve(self._h, int(slots)))

    def run_gradient_slot(self, thickness: int, slot: int):
        check(lib().ustfwi_gpu_run_gradient_slot(self._h, int(thickness), int(slot)))

    def batch_mean(self, batch: int):
        """Deterministic mean of the batch over every rank's slots into the accumulator
        (NCCL all-gather + realization-ordered fp64 sum, ustfwi_gpu_batch_mean)."""
        check(lib().ustfwi_gpu_batch_mean(self._h, int(batch)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().ustfwi_nccl_unique_id(buf))
    return buf.raw


# ---- reference-style free functions -------------------------------------------------------

def _engine_for(grid, engine):
    return engine if engine is not None else GpuEngine(grid)


@dataclass
class SimResult:
    """simulate.hpp:21-26 (data sensor-major [n_sensors, nt]; trace step-major [nt, n_shell])."""
    data: np.ndarray
    trace: Optional[np.ndarray] = None
    layer_indices: Optional[np.ndarray] = None


def simulate_forward(medium: Medium, sources: SourceSet, sensors: SensorArray, grid: UstfwiGrid,
                     boundary_thickness: int = 0, engine: Optional[GpuEngine] = None) -> SimResult:
    eng = _engine_for(grid, engine)
    eng.set_medium(medium)
    eng.set_sources(sources)
    eng.set_sensors(sensors)
    data, trace = eng.forward(boundary_thickness)
    layer = None
    if boundary_thickness > 0:
        layer = capi.shell_indices(np.asarray(medium.gamma, np.uint8), boundary_thickness)
    return SimResult(data=data, trace=trace, layer_indices=layer)


@dataclass
class GradientResult:
    """gradient.hpp:34-42."""
    loss: float
    grad: np.ndarray
    param: str = "c0"
    method: str = "time_reversal"
    boundary_thickness: int = 0
    n_simulations: int = 3


def gradient_time_reversal(medium: Medium, source: SourceSet, sensors: SensorArray, observed: np.ndarray,
                           grid: UstfwiGrid, boundary_thickness: int, param: str = "c0",
                           engine: Optional[GpuEngine] = None) -> GradientResult:
    if medium.gamma is None:
        raise ValueError("gradient computation requires a gamma mask")
    if observed.shape[1] != grid.nt:
        raise ValueError("observed data length does not match the grid")
    eng = _engine_for(grid, engine)
    eng.set_medium(medium)
    eng.set_sources(source)
    eng.set_sensors(sensors)
    loss, grad = eng.gradient_tr(observed, boundary_thickness, param=param)
    return GradientResult(loss=loss, grad=grad, param=param, boundary_thickness=boundary_thickness)


def evaluate_loss(medium: Medium, source: SourceSet, sensors: SensorArray, observed: np.ndarray,
                  grid: UstfwiGrid, engine: Optional[GpuEngine] = None) -> float:
    eng = _engine_for(grid, engine)
    eng.set_medium(medium)
    eng.set_sources(source)
    eng.set_sensors(sensors)
    return eng.evaluate_loss(observed)


# ---- source encoding (SPEC.md stochastic_estimators) -------------------------------------

@dataclass
class EncodingRealization:
    """w_i in {-1,+1}, d_i in [0,1], tau >= 0, keyed by the RNG stream;
    delay_steps = round(d_i tau / dt) (delays quantized to whole time steps)."""
    weights: np.ndarray
    delays_unit: np.ndarray
    delay_steps: np.ndarray
    tau: float
    seed: tuple = field(default_factory=tuple)
    dt: float = 0.0

    def extension(self) -> int:
        """ceil(tau / dt): the samples appended to the duration."""
        return extension_steps(self.tau, self.dt)


def extension_steps(tau: float, dt: float) -> int:
    """ceil(tau/dt), robust to tau being an integer multiple of dt up to rounding."""
    if tau <= 0.0:
        return 0
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    return int(np.ceil(tau / dt - 1e-9))


def draw_realization(n_src: int, tau: float, dt: float, master_seed: int, iteration: int,
                     index: int) -> EncodingRealization:
    w, d, u = capi.draw_realization(n_src, tau, dt, master_seed, iteration, index)
    return EncodingRealization(weights=w.astype(np.float64), delays_unit=u, delay_steps=d, tau=tau,
                               seed=(master_seed, iteration, index), dt=dt)


def encode(sources: SourceSet, data: Optional[Sequence[np.ndarray]], r: EncodingRealization, nt: int):
    """s^ = sum w_i s_i(t - d_i tau), f^ = sum w_i f_i(t - d_i tau), both zero
    padded to nt_ext = nt + ceil(tau/dt) samples (the delay is already quantized in
    r.delay_steps, each <= ceil(tau/dt)). Errors: tau < 0; a realization of another size; data
    that is not one [n_sensors, <= nt] array per source on a common sensor array.
    Returns (encoded SourceSet, encoded data [n_sensors, nt_ext] or None, nt_ext)."""
    if r.tau < 0:
        raise ValueError("tau must be non-negative")
    if len(r.weights) != len(sources.positions) or len(r.delay_steps) != len(sources.positions):
        raise ValueError("realization size does not match the sources")
    ext = extension_steps(r.tau, r.dt) if r.tau > 0 else 0
    if len(r.delay_steps) and int(np.max(r.delay_steps)) > ext:
        raise ValueError("delay exceeds ceil(tau/dt)")
    nt_ext = nt + ext
    enc = SourceSet(positions=list(sources.positions), signals=list(sources.signals),
                    weights=np.asarray(r.weights, np.float64), delays=np.asarray(r.delay_steps, np.int32))
    f_hat = None
    if data is not None:
        if len(data) != len(sources.positions):
            raise ValueError("one SensorData per source is required")
        ns = np.asarray(data[0]).shape[0]
        for f in data:
            f = np.asarray(f)
            if f.ndim != 2 or f.shape[0] != ns or f.shape[1] > nt:
                raise ValueError("per-source data must be [n_sensors, <= nt] on a common sensor array")
        f_hat = np.zeros((ns, nt_ext))
        for i, f in enumerate(data):
            d = int(r.delay_steps[i])
            f = np.asarray(f, np.float64)
            f_hat[:, d:d + f.shape[1]] += r.weights[i] * f
    return enc, f_hat, nt_ext


def encoded_gradient(engine: GpuEngine, medium: Medium, encoded: SourceSet, sensors: SensorArray,
                     observed: np.ndarray, thickness: int) -> GradientResult:
    """one TR gradient of the encoded super-source over the duration of
    `observed` (f^, nt_ext = nt + ceil(tau/dt) samples; the engine's nt follows it)."""
    nt_ext = int(np.asarray(observed).shape[1])
    if nt_ext != engine.grid.nt:
        engine.set_nt(nt_ext)
    return gradient_time_reversal(medium, encoded, sensors, observed, engine.grid, thickness, engine=engine)


def average_estimates(results: Sequence[GradientResult]) -> GradientResult:
    """arithmetic mean of gradients and losses (fixed order)."""
    if not results:
        raise ValueError("nothing to average")
    shape = results[0].grad.shape
    g = np.zeros(shape)
    loss = 0.0
    for r in results:
        if r.grad.shape != shape:
            raise ValueError("mismatched dims")
        g += r.grad
        loss += r.loss
    n = len(results)
    return GradientResult(loss=loss / n, grad=g / n, boundary_thickness=results[0].boundary_thickness)
