"""Multigrid transfer on the device (§3.3 / Appendix C;
SPEC.md:463-470): prolong_model = Blackman-tapered Fourier interpolation of a model to the
finer grid (grid/spectral.hpp:166-212), restrict_data = the traces of a finer level
resampled to the coarser time step, Kaiser low-passed (grid/filter.hpp) and scaled by
eta^(d-1). The transforms run in csrc/resample.cu behind the C ABI."""
from __future__ import annotations

import ctypes as C
from typing import Sequence, Tuple

import numpy as np

from .capi import check, lib, ptr


def _L():
    L = lib()
    L.ustfwi_fourier_interpolate.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.c_void_p, C.POINTER(C.c_int),
                                             C.c_int, C.c_void_p]
    L.ustfwi_lowpass_timeseries.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_void_p, C.c_double, C.c_double,
                                            C.c_double, C.c_double, C.c_void_p]
    L.ustfwi_restrict_traces.argtypes = [C.c_int, C.c_size_t, C.c_size_t, C.c_void_p, C.c_int, C.c_int, C.c_double,
                                         C.c_double, C.c_void_p, C.POINTER(C.c_size_t)]
    return L


def fourier_interpolate(field: np.ndarray, new_dims: Sequence[int], blackman: bool = False, device: int = 0):
    """fourier_interpolate(field, new_dims, window) (spectral.hpp:166-212)."""
    f = np.ascontiguousarray(field, dtype=np.float64)
    nd = f.ndim
    if len(new_dims) != nd:
        raise ValueError("target dimensionality mismatch")
    dims = (C.c_int * nd)(*f.shape)
    ndims = (C.c_int * nd)(*[int(v) for v in new_dims])
    out = np.zeros(tuple(int(v) for v in new_dims))
    check(_L().ustfwi_fourier_interpolate(device, nd, dims, ptr(f, C.c_double), ndims, int(bool(blackman)),
                                          ptr(out, C.c_double)))
    return out


def prolong_model(u_coarse: np.ndarray, fine_dims: Sequence[int], device: int = 0) -> np.ndarray:
    """models upsampled with Blackman-windowed Fourier interpolation."""
    return fourier_interpolate(u_coarse, fine_dims, blackman=True, device=device)


def lowpass_timeseries(series: np.ndarray, dt: float, cutoff_hz: float, transition: float = 0.1,
                       atten_db: float = 60.0, device: int = 0) -> np.ndarray:
    """lowpass_filter_timeseries (filter.hpp:88-101) of every row of `series`."""
    x = np.ascontiguousarray(np.atleast_2d(series), dtype=np.float64)
    out = np.zeros_like(x)
    check(_L().ustfwi_lowpass_timeseries(device, x.shape[0], x.shape[1], ptr(x, C.c_double), dt, cutoff_hz,
                                         transition, atten_db, ptr(out, C.c_double)))
    return out.reshape(np.shape(series))


def restrict_data(data: np.ndarray, eta: int, ndim: int, dt_fine: float, cutoff_hz: float,
                  device: int = 0) -> np.ndarray:
    """restrict_data: traces [n_sensors, nt] -> [n_sensors, ceil(nt/eta)],
    Fourier-resampled to the coarse sampling, Kaiser low-passed at `cutoff_hz` (the coarse
    grid's supported band) and scaled by eta^(ndim-1) (Appendix C)."""
    x = np.ascontiguousarray(np.atleast_2d(data), dtype=np.float64)
    L = _L()
    ntc = C.c_size_t(0)
    check(L.ustfwi_restrict_traces(device, x.shape[0], x.shape[1], ptr(x, C.c_double), int(eta), int(ndim),
                                   dt_fine, cutoff_hz, None, C.byref(ntc)))
    out = np.zeros((x.shape[0], ntc.value))
    check(L.ustfwi_restrict_traces(device, x.shape[0], x.shape[1], ptr(x, C.c_double), int(eta), int(ndim),
                                   dt_fine, cutoff_hz, ptr(out, C.c_double), C.byref(ntc)))
    return out
