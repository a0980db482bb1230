"""ctypes binding of the C ABI in include/ustfwi_capi.h (libustfwi_b200.so, in-tree).

This is the Python-side view of the drop-in boundary (the C++ drop-in headers in
include/ustfwi/ are the other). Status codes are mapped back to the reference's
exception types: USTFWI_ERR_INVALID -> ValueError (std::invalid_argument),
USTFWI_ERR_NUMERICAL -> NumericalError (ustfwi::NumericalError, core/errors.hpp:10-12).
There is no CPU fallback: if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libustfwi_b200.so")

OK, ERR_INVALID, ERR_NUMERICAL, ERR_CUDA, ERR_OOM, ERR_NCCL = 0, 1, 2, 3, 4, 5
STAGGER = {"none": 0, "plus": 1, "minus": 2}
KERNEL_KINDS = ["y_pass", "x_pass", "z_vel", "z_rho", "aux", "yxy_chain"]

# Every symbol include/ustfwi_capi.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "ustfwi_last_error", "ustfwi_version", "ustfwi_grid_validate", "ustfwi_choose_pml_size",
    "ustfwi_make_grid", "ustfwi_make_pml", "ustfwi_shell_indices", "ustfwi_ball_mask",
    "ustfwi_synth_source_pulse", "ustfwi_draw_realization", "ustfwi_gpu_create", "ustfwi_gpu_destroy",
    "ustfwi_gpu_set_medium", "ustfwi_gpu_set_gradient_options", "ustfwi_gpu_set_gradient_param", "ustfwi_gpu_set_sources", "ustfwi_gpu_set_sensors", "ustfwi_gpu_forward",
    "ustfwi_gpu_gradient_tr", "ustfwi_gpu_evaluate_loss", "ustfwi_gpu_derivative",
    "ustfwi_gpu_upload_observed", "ustfwi_gpu_run_gradient", "ustfwi_gpu_download_gradient",
    "ustfwi_gpu_accumulator", "ustfwi_gpu_synchronize", "ustfwi_gpu_stream", "ustfwi_gpu_launch_count",
    "ustfwi_gpu_shell_size", "ustfwi_gpu_set_profiling", "ustfwi_gpu_kernel_stats", "ustfwi_nccl_unique_id", "ustfwi_gpu_comm_init",
    "ustfwi_gpu_batch_reserve", "ustfwi_gpu_run_gradient_slot", "ustfwi_gpu_batch_mean", "ustfwi_gpu_set_nt", "ustfwi_host_fft", "ustfwi_design_kaiser_lowpass", "ustfwi_gpu_half_shift",
    "ustfwi_gpu_stepper_init", "ustfwi_gpu_stepper_reset", "ustfwi_gpu_stepper_update_velocity_density",
    "ustfwi_gpu_stepper_inject", "ustfwi_gpu_stepper_enforce", "ustfwi_gpu_stepper_refresh_pressure",
    "ustfwi_gpu_stepper_update_pressure", "ustfwi_gpu_stepper_read", "ustfwi_gpu_stepper_gather",
    "ustfwi_gpu_stepper_step_index", "ustfwi_gpu_chain_stats", "ustfwi_gpu_partition",
    "ustfwi_lbfgs_create", "ustfwi_lbfgs_destroy", "ustfwi_lbfgs_reset", "ustfwi_lbfgs_push", "ustfwi_lbfgs_apply",
    "ustfwi_lbfgs_pairs", "ustfwi_fourier_interpolate", "ustfwi_lowpass_timeseries", "ustfwi_restrict_traces",
]


class NumericalError(RuntimeError):
    """ustfwi::NumericalError (core/errors.hpp:10-12)."""


class CudaError(RuntimeError):
    pass


class UstfwiGrid(C.Structure):
    """Field-for-field image of ustfwi::Grid (grid/grid.hpp:14-20)."""
    _fields_ = [
        ("ndim", C.c_int),
        ("dims", C.c_int * 3),
        ("dx", C.c_double * 3),
        ("dt", C.c_double),
        ("nt", C.c_int),
        ("pml_size", C.c_int * 3),
        ("c_ref", C.c_double),
    ]

    @property
    def shape(self):
        return tuple(self.dims[a] for a in range(self.ndim))

    @property
    def points(self):
        return int(np.prod(self.shape))

    def __repr__(self):
        return (f"Grid(dims={self.shape}, dx={self.dx[0]:g}, dt={self.dt:g}, nt={self.nt}, "
                f"pml={tuple(self.pml_size[a] for a in range(self.ndim))}, c_ref={self.c_ref:g})")


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2102_00755_b200.build`"
                              " (there is no CPU fallback)")
        if "USTFWI_NCCL_LIB" not in os.environ:
            # the NCCL torch is built against (pip wheel), so that importing torch after the
            # engine loaded NCCL does not bind torch to an older system libnccl
            try:
                import importlib.util
                spec = importlib.util.find_spec("nvidia.nccl")
                if spec and spec.submodule_search_locations:
                    cand = os.path.join(list(spec.submodule_search_locations)[0], "lib", "libnccl.so.2")
                    if os.path.exists(cand):
                        os.environ["USTFWI_NCCL_LIB"] = cand
            except Exception:
                pass
        L = C.CDLL(LIB_PATH)
        L.ustfwi_last_error.restype = C.c_char_p
        L.ustfwi_version.restype = C.c_char_p
        L.ustfwi_gpu_stream.restype = C.c_void_p
        L.ustfwi_gpu_stream.argtypes = [C.c_void_p]
        L.ustfwi_gpu_launch_count.restype = C.c_uint64
        L.ustfwi_gpu_launch_count.argtypes = [C.c_void_p]
        L.ustfwi_gpu_shell_size.restype = C.c_size_t
        L.ustfwi_gpu_shell_size.argtypes = [C.c_void_p]
        L.ustfwi_gpu_destroy.restype = None
        L.ustfwi_gpu_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def check(code: int):
    if code == OK:
        return
    msg = lib().ustfwi_last_error().decode()
    if code == ERR_INVALID:
        raise ValueError(msg)
    if code == ERR_NUMERICAL:
        raise NumericalError(msg)
    if code == ERR_OOM:
        raise MemoryError(msg)
    raise CudaError(f"[{code}] {msg}")


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def dptr(a):
    return ptr(np.ascontiguousarray(a, dtype=np.float64), C.c_double)


# ---- host setup --------------------------------------------------------------------------

def make_grid(interior, dx, c_max, duration, cfl=0.3) -> UstfwiGrid:
    g = UstfwiGrid()
    arr = (C.c_int * len(interior))(*[int(v) for v in interior])
    check(lib().ustfwi_make_grid(len(interior), arr, C.c_double(dx), C.c_double(c_max),
                                 C.c_double(duration), C.c_double(cfl), C.byref(g)))
    return g


def grid_from(dims, dx, dt, nt, pml_size, c_ref) -> UstfwiGrid:
    g = UstfwiGrid()
    g.ndim = len(dims)
    for a in range(len(dims)):
        g.dims[a] = int(dims[a])
        g.dx[a] = float(dx if np.isscalar(dx) else dx[a])
        g.pml_size[a] = int(pml_size[a])
    g.dt = float(dt)
    g.nt = int(nt)
    g.c_ref = float(c_ref)
    return g


def validate_grid(g: UstfwiGrid):
    check(lib().ustfwi_grid_validate(C.byref(g)))


def choose_pml_size(interior):
    arr = (C.c_int * len(interior))(*interior)
    out = (C.c_int * len(interior))()
    check(lib().ustfwi_choose_pml_size(len(interior), arr, out))
    return list(out)


def make_pml(g: UstfwiGrid, alpha=2.0):
    tot = sum(g.shape)
    reg = np.zeros(tot)
    stag = np.zeros(tot)
    check(lib().ustfwi_make_pml(C.byref(g), C.c_double(alpha), ptr(reg, C.c_double), ptr(stag, C.c_double)))
    out_r, out_s, o = [], [], 0
    for n in g.shape:
        out_r.append(reg[o:o + n].copy())
        out_s.append(stag[o:o + n].copy())
        o += n
    return out_r, out_s


def shell_indices(mask: np.ndarray, thickness: int) -> np.ndarray:
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    dims = (C.c_int * m.ndim)(*m.shape)
    cnt = C.c_size_t(0)
    check(lib().ustfwi_shell_indices(m.ndim, dims, ptr(m, C.c_uint8), int(thickness), None, C.byref(cnt)))
    out = np.zeros(cnt.value, dtype=np.uint64)
    check(lib().ustfwi_shell_indices(m.ndim, dims, ptr(m, C.c_uint8), int(thickness), ptr(out, C.c_size_t),
                                     C.byref(cnt)))
    return out.astype(np.int64)


def ball_mask(dims, center, radius_points) -> np.ndarray:
    out = np.zeros(tuple(dims), dtype=np.uint8)
    d = (C.c_int * len(dims))(*dims)
    c = (C.c_double * len(dims))(*[float(v) for v in center])
    check(lib().ustfwi_ball_mask(len(dims), d, c, C.c_double(radius_points), ptr(out, C.c_uint8)))
    return out


def synth_source_pulse(g: UstfwiGrid, frac: float, c0_min: float) -> np.ndarray:
    n = C.c_int(0)
    check(lib().ustfwi_synth_source_pulse(C.byref(g), C.c_double(frac), C.c_double(c0_min), None, C.byref(n)))
    out = np.zeros(n.value)
    check(lib().ustfwi_synth_source_pulse(C.byref(g), C.c_double(frac), C.c_double(c0_min),
                                          ptr(out, C.c_double), C.byref(n)))
    return out


def draw_realization(n_src, tau, dt, master_seed, iteration, index):
    """-> (weights int8 {-1,+1}, delay_steps int32, delays_unit float64 in [0,1))."""
    w = np.zeros(n_src, dtype=np.int8)
    d = np.zeros(n_src, dtype=np.int32)
    u = np.zeros(n_src, dtype=np.float64)
    check(lib().ustfwi_draw_realization(C.c_size_t(n_src), C.c_double(tau), C.c_double(dt),
                                        C.c_uint64(master_seed), C.c_uint64(iteration), C.c_uint64(index),
                                        ptr(w, C.c_int8), ptr(d, C.c_int32), ptr(u, C.c_double)))
    return w, d, u
