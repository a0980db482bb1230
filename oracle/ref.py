"""ctypes loader for oracle/_ref/libustfwi_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the UNMODIFIED reference (`/root/reference/proj/include`) compiled with
the in-repo FFTW-API shim by `oracle/Makefile` (see `oracle/ref_driver.cpp` for the
entry points and the reference file:line each one wraps). Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libustfwi_ref.so")


class RefGrid(C.Structure):
    _fields_ = [
        ("ndim", C.c_int),
        ("dims", C.c_int * 3),
        ("dx", C.c_double * 3),
        ("dt", C.c_double),
        ("nt", C.c_int),
        ("pml_size", C.c_int * 3),
        ("c_ref", C.c_double),
    ]


class RefMedium(C.Structure):
    _fields_ = [
        ("c0", C.POINTER(C.c_double)),
        ("rho0", C.POINTER(C.c_double)),
        ("alpha0", C.POINTER(C.c_double)),
        ("y", C.c_double),
        ("gamma", C.POINTER(C.c_uint8)),
        ("c0_min", C.c_double),
        ("c0_max", C.c_double),
    ]


class RefSources(C.Structure):
    _fields_ = [
        ("n", C.c_size_t),
        ("pos", C.POINTER(C.c_size_t)),
        ("sig_off", C.POINTER(C.c_size_t)),
        ("sig", C.POINTER(C.c_double)),
    ]


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle`")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
    return _lib


def _check(code: int):
    if code != 0:
        raise RefError(code, lib().ref_last_error().decode())


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def grid_struct(g) -> RefGrid:
    """Accepts any object with ndim/dims/dx/dt/nt/pml_size/c_ref attributes."""
    s = RefGrid()
    nd = int(getattr(g, "ndim", len(g.dims)))
    s.ndim = nd
    for a in range(nd):
        s.dims[a] = int(g.dims[a])
        s.dx[a] = float(g.dx[a])
        s.pml_size[a] = int(g.pml_size[a])
    s.dt = float(g.dt)
    s.nt = int(g.nt)
    s.c_ref = float(g.c_ref)
    return s


@dataclass
class _Keep:
    arrays: list


def _medium(m, keep: list) -> RefMedium:
    c0 = np.ascontiguousarray(m.c0, dtype=np.float64).ravel()
    rho0 = np.ascontiguousarray(m.rho0, dtype=np.float64).ravel()
    s = RefMedium()
    s.c0 = _p(c0, C.c_double)
    s.rho0 = _p(rho0, C.c_double)
    keep += [c0, rho0]
    if getattr(m, "alpha0", None) is not None:
        a0 = np.ascontiguousarray(m.alpha0, dtype=np.float64).ravel()
        s.alpha0 = _p(a0, C.c_double)
        keep.append(a0)
    s.y = float(getattr(m, "y", 1.5))
    if getattr(m, "gamma", None) is not None:
        gm = np.ascontiguousarray(m.gamma, dtype=np.uint8).ravel()
        s.gamma = _p(gm, C.c_uint8)
        keep.append(gm)
    s.c0_min = float(getattr(m, "c0_min", 1350.0))
    s.c0_max = float(getattr(m, "c0_max", 1800.0))
    return s


def _sources(positions, signals, keep: list) -> RefSources:
    pos = np.ascontiguousarray(positions, dtype=np.uint64)
    lens = [len(s) for s in signals]
    off = np.zeros(len(signals) + 1, dtype=np.uint64)
    off[1:] = np.cumsum(lens)
    sig = np.ascontiguousarray(np.concatenate([np.asarray(s, np.float64) for s in signals])
                               if signals else np.zeros(1), dtype=np.float64)
    keep += [pos, off, sig]
    s = RefSources()
    s.n = len(pos)
    s.pos = _p(pos, C.c_size_t)
    s.sig_off = _p(off, C.c_size_t)
    s.sig = _p(sig, C.c_double)
    return s


def make_grid(interior, dx, c_max, duration, cfl=0.3):
    g = RefGrid()
    arr = (C.c_int * len(interior))(*interior)
    _check(lib().ref_make_grid(len(interior), arr, C.c_double(dx), C.c_double(c_max),
                               C.c_double(duration), C.c_double(cfl), C.byref(g)))
    return g


def choose_pml_size(interior):
    arr = (C.c_int * len(interior))(*interior)
    out = (C.c_int * len(interior))()
    _check(lib().ref_choose_pml_size(len(interior), arr, out))
    return list(out)


def make_pml(g, alpha=2.0):
    s = grid_struct(g)
    dims = [g.dims[a] for a in range(int(getattr(g, "ndim", len(g.dims))))]
    tot = sum(dims)
    reg = np.zeros(tot)
    stag = np.zeros(tot)
    _check(lib().ref_make_pml(C.byref(s), C.c_double(alpha), _p(reg, C.c_double), _p(stag, C.c_double)))
    out_r, out_s, o = [], [], 0
    for n in dims:
        out_r.append(reg[o:o + n].copy())
        out_s.append(stag[o:o + n].copy())
        o += n
    return out_r, out_s


def engine_derivative(g, f, axis, stagger):
    """SpectralEngine::derivative (engine.hpp:118-121); stagger 0 none, 1 plus, 2 minus."""
    s = grid_struct(g)
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros_like(f)
    _check(lib().ref_engine_derivative(C.byref(s), _p(f, C.c_double), axis, stagger, _p(out, C.c_double)))
    return out


def spectral_derivative(g, f, axis, stagger):
    s = grid_struct(g)
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros_like(f)
    _check(lib().ref_spectral_derivative(C.byref(s), _p(f, C.c_double), axis, stagger, _p(out, C.c_double)))
    return out


def fourier_shift(g, f, axis, shift_cells):
    s = grid_struct(g)
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.zeros_like(f)
    _check(lib().ref_fourier_shift(C.byref(s), _p(f, C.c_double), axis, C.c_double(shift_cells),
                                   _p(out, C.c_double)))
    return out


def shell_indices(mask, thickness):
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    dims = (C.c_int * m.ndim)(*m.shape)
    cnt = C.c_size_t(0)
    _check(lib().ref_shell_indices(m.ndim, dims, _p(m, C.c_uint8), thickness, None, C.byref(cnt)))
    out = np.zeros(cnt.value, dtype=np.uint64)
    _check(lib().ref_shell_indices(m.ndim, dims, _p(m, C.c_uint8), thickness, _p(out, C.c_size_t),
                                   C.byref(cnt)))
    return out.astype(np.int64)


def synth_source_pulse(g, frac, c0_min):
    s = grid_struct(g)
    n = C.c_int(0)
    _check(lib().ref_synth_source_pulse(C.byref(s), C.c_double(frac), C.c_double(c0_min), None, C.byref(n)))
    out = np.zeros(n.value)
    _check(lib().ref_synth_source_pulse(C.byref(s), C.c_double(frac), C.c_double(c0_min),
                                        _p(out, C.c_double), C.byref(n)))
    return out


def simulate_forward(g, medium, positions, signals, sensors, boundary_thickness=0, pml_enabled=True):
    """simulate_forward (simulate.hpp:30-105). Returns (data [ns, nt], trace [nt, n_shell] or None)."""
    keep: list = []
    s = grid_struct(g)
    m = _medium(medium, keep)
    src = _sources(positions, signals, keep)
    sens = np.ascontiguousarray(sensors, dtype=np.uint64)
    data = np.zeros((len(sens), g.nt))
    shape = tuple(g.dims[a] for a in range(int(getattr(g, "ndim", len(g.dims)))))
    n_shell = C.c_size_t(0)
    trace_ptr = None
    trace = None
    if boundary_thickness > 0:
        gm = np.asarray(medium.gamma, dtype=np.uint8)
        n_sh = len(shell_indices(gm, boundary_thickness))
        trace = np.zeros((g.nt, n_sh))
        trace_ptr = _p(trace, C.c_double)
    _check(lib().ref_simulate_forward(C.byref(s), C.byref(m), C.byref(src), C.c_size_t(len(sens)),
                                      _p(sens, C.c_size_t), boundary_thickness, int(pml_enabled),
                                      _p(data, C.c_double), trace_ptr, C.byref(n_shell)))
    return data, trace


def gradient_time_reversal(g, medium, positions, signals, sensors, observed, thickness):
    """gradient_time_reversal (gradient.hpp:478-488) -> (loss, grad)."""
    keep: list = []
    s = grid_struct(g)
    m = _medium(medium, keep)
    src = _sources(positions, signals, keep)
    sens = np.ascontiguousarray(sensors, dtype=np.uint64)
    obs = np.ascontiguousarray(observed, dtype=np.float64)
    grad = np.zeros(tuple(g.dims[a] for a in range(int(getattr(g, "ndim", len(g.dims))))))
    loss = C.c_double(0.0)
    _check(lib().ref_gradient_tr(C.byref(s), C.byref(m), C.byref(src), C.c_size_t(len(sens)),
                                 _p(sens, C.c_size_t), _p(obs, C.c_double), thickness,
                                 _p(grad, C.c_double), C.byref(loss)))
    return loss.value, grad


PARAM = {"c0": 0, "rho0": 1, "alpha0": 2, "y": 3}


def gradient_tr_opts(g, medium, positions, signals, sensors, observed, thickness, dispersion_enabled=True,
                     param="c0"):
    """compute_gradient (gradient.hpp:333-464), TR method, GradientParam, with
    GradientOptions::dispersion_enabled."""
    keep: list = []
    s = grid_struct(g)
    m = _medium(medium, keep)
    src = _sources(positions, signals, keep)
    sens = np.ascontiguousarray(sensors, dtype=np.uint64)
    obs = np.ascontiguousarray(observed, dtype=np.float64)
    grad = np.zeros(tuple(g.dims[a] for a in range(int(getattr(g, "ndim", len(g.dims))))))
    loss = C.c_double(0.0)
    _check(lib().ref_gradient_tr_opts(C.byref(s), C.byref(m), C.byref(src), C.c_size_t(len(sens)),
                                      _p(sens, C.c_size_t), _p(obs, C.c_double), thickness,
                                      int(bool(dispersion_enabled)), PARAM[param], _p(grad, C.c_double),
                                      C.byref(loss)))
    return loss.value, grad


def evaluate_loss(g, medium, positions, signals, sensors, observed):
    keep: list = []
    s = grid_struct(g)
    m = _medium(medium, keep)
    src = _sources(positions, signals, keep)
    sens = np.ascontiguousarray(sensors, dtype=np.uint64)
    obs = np.ascontiguousarray(observed, dtype=np.float64)
    loss = C.c_double(0.0)
    _check(lib().ref_evaluate_loss(C.byref(s), C.byref(m), C.byref(src), C.c_size_t(len(sens)),
                                   _p(sens, C.c_size_t), _p(obs, C.c_double), C.byref(loss)))
    return loss.value


def time_steps(g, medium, k_fwd, k_pair):
    """Seconds per forward step and per adjoint+TR pair-step of the reference (CPU)."""
    keep: list = []
    s = grid_struct(g)
    m = _medium(medium, keep)
    a = C.c_double(0)
    b = C.c_double(0)
    _check(lib().ref_time_steps(C.byref(s), C.byref(m), k_fwd, k_pair, C.byref(a), C.byref(b)))
    return a.value, b.value


def fourier_interpolate(f, new_dims, blackman=False):
    """fourier_interpolate (spectral.hpp:166-212)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    nd = len(f.shape)
    dims = (C.c_int * nd)(*f.shape)
    ndims = (C.c_int * nd)(*new_dims)
    out = np.zeros(tuple(new_dims))
    _check(lib().ref_fourier_interpolate(nd, dims, _p(f, C.c_double), ndims, int(bool(blackman)),
                                         _p(out, C.c_double)))
    return out


def lowpass_timeseries(sig, dt, cutoff_hz, transition=0.1, atten_db=60.0):
    """lowpass_filter_timeseries (filter.hpp:88-101)."""
    x = np.ascontiguousarray(sig, dtype=np.float64)
    out = np.zeros_like(x)
    _check(lib().ref_lowpass_timeseries(_p(x, C.c_double), C.c_size_t(x.size), C.c_double(dt), C.c_double(cutoff_hz),
                                        C.c_double(transition), C.c_double(atten_db), _p(out, C.c_double)))
    return out
