"""Propagator properties of the device engine, mirroring the reference's solver tests
(tests/test_solver.cpp): the analytic first-arrival time (:60-80), reciprocity (:143-169)
and PML reflections below 1 % of the incident pulse (:171-196) — the same 2-D setups,
thresholds and measurement rules — plus the reciprocity check on a 3-D grid."""
import numpy as np
import pytest

from paper_2102_00755_b200 import capi
from paper_2102_00755_b200.engine import GpuEngine, SensorArray, SourceSet, make_homogeneous_medium, simulate_forward

pytestmark = pytest.mark.gpu


def onset_index(trace, frac):  # test_solver.cpp:16-22
    a = np.abs(np.asarray(trace))
    idx = np.flatnonzero(a >= frac * a.max())
    return int(idx[0]) if idx.size else -1


def flat(g, x, y, z):
    sh = g.shape
    return (x * sh[1] + y) * sh[2] + z


def flat2(g, x, y):
    return x * g.shape[1] + y


def test_first_arrival_matches_travel_time():
    c, dx = 1500.0, 1e-3
    g = capi.make_grid([128, 128], dx, c, 1.3e-4)
    m = make_homogeneous_medium(g, c)
    mid = g.shape[1] // 2
    p = g.pml_size[0]
    src = SourceSet([flat2(g, p + 15, mid)], [capi.synth_source_pulse(g, 1.0, c)])
    # receiver pair on the same ray, outside the near field: the waveform shape cancels in the
    # differential onset, leaving the travel time over d
    sens = SensorArray([flat2(g, p + 45, mid), flat2(g, p + 105, mid)])
    with GpuEngine(g) as eng:
        data = simulate_forward(m, src, sens, g, engine=eng).data
    n1, n2 = onset_index(data[0], 0.1), onset_index(data[1], 0.1)
    assert n2 > n1
    assert abs((n2 - n1) * g.dt - 60 * dx / c) <= 2.0 * g.dt


def test_reciprocity_2d():
    g = capi.make_grid([96, 96], 1e-3, 1800.0, 6e-5)
    m = make_homogeneous_medium(g)
    pulse = capi.synth_source_pulse(g, 0.8, 1500.0)
    a, b = flat2(g, 30, 42), flat2(g, 75, 58)
    with GpuEngine(g) as eng:
        ab = simulate_forward(m, SourceSet([a], [pulse]), SensorArray([b]), g, engine=eng).data[0]
        ba = simulate_forward(m, SourceSet([b], [pulse]), SensorArray([a]), g, engine=eng).data[0]
    # 1e-6 in fp64 (test_solver.cpp:167); the device computes in fp32
    assert np.linalg.norm(ab - ba) / np.linalg.norm(ba) < 1e-5


def test_reciprocity_3d():
    g = capi.make_grid([44, 44, 44], 1e-3, 1800.0, 6e-5)
    m = make_homogeneous_medium(g)
    pulse = capi.synth_source_pulse(g, 0.8, 1500.0)
    a, b = flat(g, 18, 26, 30), flat(g, 44, 36, 22)
    with GpuEngine(g) as eng:
        ab = simulate_forward(m, SourceSet([a], [pulse]), SensorArray([b]), g, engine=eng).data[0]
        ba = simulate_forward(m, SourceSet([b], [pulse]), SensorArray([a]), g, engine=eng).data[0]
    assert np.abs(ba).max() > 0
    assert np.linalg.norm(ab - ba) / np.linalg.norm(ba) < 1e-5


def test_pml_reflections_below_one_percent():
    c, dx = 1500.0, 1e-3
    g = capi.make_grid([128, 128], dx, c, 2.2e-4)
    m = make_homogeneous_medium(g, c)
    mid = g.shape[0] // 2
    src = SourceSet([flat2(g, mid, mid)], [capi.synth_source_pulse(g, 0.8, c)])
    sens = SensorArray([flat2(g, mid + 30, mid)])
    with GpuEngine(g) as eng:
        tr = simulate_forward(m, src, sens, g, engine=eng).data[0]
    # the direct wave passes the receiver around t_direct; anything after the shortest
    # boundary round trip is reflection (test_solver.cpp:185-194)
    t = np.arange(g.nt) * g.dt
    pml = g.pml_size[0]
    t_direct = 30 * dx / c
    t_reflect = ((mid - pml) + (mid - 30 - pml)) * dx / c
    incident = np.abs(tr[t < t_direct + 4e-5]).max()
    reflected = np.abs(tr[t > t_reflect + 4e-5]).max()
    assert incident > 0
    assert reflected < 0.01 * incident
