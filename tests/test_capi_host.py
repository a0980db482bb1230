"""CPU tests of the C-ABI library: it loads without a GPU, exports every symbol the header
declares, and its host-side setup matches the reference (oracle/_ref) exactly.

Mirrors test_grid.cpp (choose_pml_size :26-48, wavenumbers :50-57, PML :191-214,
validation :183-189) against the product's C ABI."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2102_00755_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "ustfwi_capi.h")).read()
    return sorted(set(re.findall(r"USTFWI_API\s+[\w\s\*]+?\b(ustfwi_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = capi.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(capi.EXPORTS) == syms


def test_gpu_create_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = capi.make_grid([4, 4, 4], 1e-3, 1800.0, 1e-6)
    h = C.c_void_p()
    rc = capi.lib().ustfwi_gpu_create(0, C.byref(g), C.byref(h))
    assert rc == capi.ERR_CUDA
    assert "no CUDA device" in capi.lib().ustfwi_last_error().decode() or "device" in capi.lib().ustfwi_last_error().decode()


def test_choose_pml_size_known_answers():
    assert capi.choose_pml_size([44]) == [10]
    assert capi.choose_pml_size([100]) == [14]
    assert capi.choose_pml_size([108]) == [10]
    assert capi.choose_pml_size([44, 100]) == [10, 14]
    assert capi.choose_pml_size([442, 442, 222]) == [19, 19, 17]  # config D -> 480x480x256


def test_choose_pml_size_brute_force():
    rng = np.random.default_rng(7)
    def lpf(n):
        best, f = 1, 2
        while f * f <= n:
            while n % f == 0:
                best, n = f, n // f
            f += 1
        return n if n > 1 else best
    for interior in rng.integers(4, 601, size=200):
        t = capi.choose_pml_size([int(interior)])[0]
        assert 10 <= t <= 20
        p = lpf(int(interior) + 2 * t)
        for t2 in range(10, 21):
            p2 = lpf(int(interior) + 2 * t2)
            assert p <= p2
            if p2 == p:
                assert t <= t2


def test_grid_validation():
    g = capi.grid_from([16, 16], 1e-3, 1e-7, 16, [0, 0], 1500.0)
    capi.validate_grid(g)
    for bad in ([15, 16], [2, 16]):
        with pytest.raises(ValueError):
            capi.validate_grid(capi.grid_from(bad, 1e-3, 1e-7, 16, [0, 0], 1500.0))
    g.dt = -1.0
    with pytest.raises(ValueError):
        capi.validate_grid(g)


def test_make_grid_configs():
    a = capi.make_grid([44, 44, 44], 1e-3, 1800.0, 2 * 0.044 / 1350.0)
    assert a.shape == (64, 64, 64) and a.nt == 393
    d = capi.make_grid([442, 442, 222], 0.5e-3, 1800.0, 2 * 0.221 / 1350.0)
    assert d.shape == (480, 480, 256)


def test_pml_profiles_range():
    g = capi.grid_from([64, 64], 1e-3, 0.3e-3 / 1500.0, 8, [10, 12], 1500.0)
    reg, stag = capi.make_pml(g)
    for a in range(2):
        p = g.pml_size[a]
        assert np.all(reg[a][p:64 - p] == 1.0)
        assert np.all((reg[a] > 0) & (reg[a] <= 1)) and np.all((stag[a] > 0) & (stag[a] <= 1))
        assert reg[a][0] < 0.9


def test_draw_realization_contract():
    w1, d1, u1 = capi.draw_realization(1000, 2e-6, 1e-7, 20210201, 3, 5)
    w2, d2, u2 = capi.draw_realization(1000, 2e-6, 1e-7, 20210201, 3, 5)
    assert np.array_equal(w1, w2) and np.array_equal(d1, d2) and np.array_equal(u1, u2)
    w3, _, _ = capi.draw_realization(1000, 2e-6, 1e-7, 20210201, 3, 6)
    assert not np.array_equal(w1, w3)
    assert set(np.unique(w1)) <= {-1, 1}
    assert np.all((u1 >= 0) & (u1 < 1))
    assert np.array_equal(d1, np.rint(u1 * 2e-6 / 1e-7).astype(np.int32))
    _, d0, _ = capi.draw_realization(10, 0.0, 1e-7, 1, 0, 0)
    assert np.all(d0 == 0)
    with pytest.raises(ValueError):
        capi.draw_realization(4, -1.0, 1e-7, 1, 0, 0)


def test_rademacher_moments():
    # E[w] = 0, Cov[w] = I over 1e5 draws within 3 sigma
    n_src, draws = 4, 100000
    W = np.stack([capi.draw_realization(n_src, 0.0, 1.0, 20210201, 0, r)[0] for r in range(draws)]).astype(float)
    sig = 3.0 / np.sqrt(draws)
    assert np.all(np.abs(W.mean(0)) < sig)
    cov = W.T @ W / draws
    assert np.all(np.abs(cov - np.eye(n_src)) < sig + 1e-12)
