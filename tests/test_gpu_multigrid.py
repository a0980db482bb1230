"""Multigrid transfer on the device against the reference's own
fourier_interpolate / lowpass_filter_timeseries (fixture from oracle/_ref, make_golden.py)
and the SPEC.md:463-470 / :494 properties of restrict_data."""
import numpy as np
import pytest

from paper_2102_00755_b200 import multigrid

pytestmark = pytest.mark.gpu

TOL = 1e-5  # fp32 device transforms vs the fp64 reference


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("case", ["up", "down", "mixed", "2d"])
@pytest.mark.parametrize("window", ["none", "blackman"])
def test_fourier_interpolate_matches_reference(golden, case, window):
    z = golden("multigrid")
    out = multigrid.fourier_interpolate(z[f"{case}_in"], z[f"{case}_dims"], blackman=(window == "blackman"))
    assert out.shape == tuple(z[f"{case}_dims"])
    assert rel(out, z[f"{case}_{window}"]) < TOL


def test_up_down_round_trip_is_exact():
    # resample_spectrum_axis splits / folds the Nyquist bin so that up-down is the identity
    f = np.random.default_rng(5).standard_normal((8, 6, 10))
    back = multigrid.fourier_interpolate(multigrid.fourier_interpolate(f, (16, 12, 20)), f.shape)
    assert rel(back, f) < 1e-6


def test_fourier_interpolate_errors():
    with pytest.raises(ValueError, match="even and >= 4"):
        multigrid.fourier_interpolate(np.zeros((8, 8)), (6, 5))
    with pytest.raises(ValueError, match="source dims must be even"):
        multigrid.fourier_interpolate(np.zeros((7, 8)), (8, 8))


def test_lowpass_matches_reference(golden):
    z = golden("multigrid")
    assert rel(multigrid.lowpass_timeseries(z["lp_in"], 1e-7, 1e6), z["lp_1MHz"]) < TOL
    assert rel(multigrid.lowpass_timeseries(z["lp_in"], 1e-7, 2e6, 0.2, 40.0), z["lp_2MHz_tr02_a40"]) < TOL
    with pytest.raises(ValueError, match="Nyquist"):
        multigrid.lowpass_timeseries(z["lp_in"], 1e-7, 6e6)


def test_restrict_data_properties():
    rng = np.random.default_rng(9)
    d = rng.standard_normal((5, 301))
    # eta = 1 -> identity, no filtering, scale 1
    assert np.array_equal(multigrid.restrict_data(d, 1, 3, 1e-7, 1e6), d)
    # coarse sample count ceil(nt / eta); 3-D eta = 2 -> amplitude x4, 2-D -> x2
    # on a constant trace away from the zero-padded ends (DC preserved)
    c = np.full((2, 801), 0.75)
    for ndim, scale in [(3, 4.0), (2, 2.0)]:
        r = multigrid.restrict_data(c, 2, ndim, 1e-7, 1e6)
        assert r.shape == (2, 401)
        mid = r[:, 120:-120]  # beyond the 183-tap Kaiser filter's reach into the zero padding
        assert np.allclose(mid, 0.75 * scale, rtol=1e-5)


def test_restrict_data_odd_nt_keeps_arrival_time():
    # with nt % eta != 0 the coarse spacing must stay eta * dt_fine (traces are
    # zero-padded to ceil(nt/eta) * eta before resampling): a band-limited pulse centred at
    # fine sample 250 of a 301-sample trace lands at coarse sample 125 (eta = 2)
    dt = 1e-7
    t = np.arange(301)
    pulse = np.exp(-0.5 * ((t - 250.0) / 6.0) ** 2)[None, :]
    r = multigrid.restrict_data(pulse, 2, 3, dt, 1.5e6)[0]
    k = int(np.argmax(r))
    y0, y1, y2 = r[k - 1], r[k], r[k + 1]
    peak = k + 0.5 * (y0 - y2) / (y0 - 2 * y1 + y2)   # parabolic refinement
    assert abs(peak - 125.0) < 0.05, peak
