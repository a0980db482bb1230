"""Synthetic benchmark scenarios.

Input side only (SPEC.md scenario_kit :517-581, §4.1 :184-193): grids via the
C-ABI make_grid, a 3-D breast phantom (tissue table 1470/1500/1515/1584/1650 m/s,
PAPER.md:184), golden-spiral hemispherical bowl with alternating emitters/receivers
(PAPER.md:192), Rademacher encoding of the emitters. Deterministic per
seed. Nothing here is on the timed path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import capi
from .engine import Medium, SensorArray, SourceSet

MASTER_SEED = 20210201
C0_MIN, C0_MAX = 1350.0, 1800.0
WATER, FAT, GLAND, VESSEL, SKIN = 1500.0, 1470.0, 1515.0, 1584.0, 1650.0


@dataclass
class Scenario:
    name: str
    grid: capi.UstfwiGrid
    model: Medium          # medium the gradient is evaluated at (water initialisation)
    truth: Medium          # medium that generates the observed data
    sources: SourceSet     # emitters with the (un-encoded) base pulse
    sensors: SensorArray
    pulse: np.ndarray
    thickness: int = 8

    @property
    def n_src(self):
        return len(self.sources.positions)

    @property
    def voxel_updates_per_gradient(self):
        # forward nt + replay (nt-1 incl. look-ahead) + adjoint nt-2 = 3nt-3 steps
        return self.grid.points * (3 * self.grid.nt - 3)

    def encoded(self, realization_index: int, tau: float = 0.0, iteration: int = 0,
                master_seed: int = MASTER_SEED) -> SourceSet:
        w, d, _ = capi.draw_realization(self.n_src, tau, self.grid.dt, master_seed, iteration,
                                        realization_index)
        return SourceSet(positions=list(self.sources.positions), signals=list(self.sources.signals),
                         weights=w.astype(np.float64), delays=d)


def flat(shape, x, y, z):
    return (int(x) * shape[1] + int(y)) * shape[2] + int(z)


def golden_section_placement(n: int, radius: float, center, shape, pml=(0, 0, 0), exclude=None):
    """golden_section_placement (§4.1 "distribute 2048 transducer
    locations over the half-sphere by the golden section method"): golden-spiral points on
    the hemisphere z >= center_z, snapped to the grid inside the PML, duplicates and points in
    `exclude` dropped, alternately assigned to emitters / receivers. Returns (emitters,
    receivers) as flat indices."""
    if n < 2:
        raise ValueError("n must be >= 2")
    golden = np.pi * (3.0 - np.sqrt(5.0))
    cx, cy, cz0 = center
    emit, recv, seen = [], [], set()
    ex = None if exclude is None else np.asarray(exclude).ravel()
    for i in range(n):
        cz = (i + 0.5) / n
        st = np.sqrt(max(0.0, 1.0 - cz * cz))
        phi = golden * i
        x = int(round(cx + radius * st * np.cos(phi)))
        y = int(round(cy + radius * st * np.sin(phi)))
        z = int(round(cz0 + radius * cz))
        x = min(max(x, pml[0]), shape[0] - pml[0] - 1)
        y = min(max(y, pml[1]), shape[1] - pml[1] - 1)
        z = min(max(z, pml[2]), shape[2] - pml[2] - 1)
        f = flat(shape, x, y, z)
        if f in seen or (ex is not None and ex[f]):
            continue
        seen.add(f)
        (emit if i % 2 == 0 else recv).append(f)
    return emit, recv


def add_noise(data: np.ndarray, snr_db: float, seed: int) -> np.ndarray:
    """add_noise (Appendix F): i.i.d. zero-mean Gaussian noise with
    sigma = RMS(f) * 10^(-SNR/20), RMS over the whole clean dataset; SNR = inf -> unchanged."""
    f = np.asarray(data, dtype=np.float64)
    if np.isinf(snr_db) and snr_db > 0:
        return f.copy()
    rms = float(np.sqrt(np.mean(f * f))) if f.size else 0.0
    sigma = rms * 10.0 ** (-snr_db / 20.0)
    if sigma == 0.0:
        return f.copy()
    return f + np.random.default_rng(seed).normal(0.0, sigma, size=f.shape)


def per_source_data(engine, sc: "Scenario", medium=None) -> np.ndarray:
    """Clean SensorData per emitter (ScanScenario): one device forward per
    source on `medium` (default: the truth phantom) -> [n_src, n_receivers, nt]."""
    m = sc.truth if medium is None else medium
    engine.set_medium(m)
    engine.set_sensors(sc.sensors)
    out = np.zeros((sc.n_src, len(sc.sensors.positions), sc.grid.nt))
    for k, (p, sig) in enumerate(zip(sc.sources.positions, sc.sources.signals)):
        engine.set_sources(SourceSet([p], [sig]))
        out[k] = engine.forward(0)[0]
    return out


def config_a(nt: Optional[int] = None) -> Scenario:
    """64^3 water, 1 source, 8 sensors, Gaussian bump, ball gamma r=12."""
    interior, dx = [44, 44, 44], 1e-3
    g = capi.make_grid(interior, dx, C0_MAX, 2 * interior[0] * dx / C0_MIN)
    if nt is not None:
        g.nt = int(nt)
    shape = g.shape
    c = [s // 2 for s in shape]
    gamma = capi.ball_mask(shape, c, 12.0)
    ix, iy, iz = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    r2 = (ix - c[0]) ** 2 + (iy - c[1]) ** 2 + (iz - c[2]) ** 2
    c0_true = WATER + 30.0 * np.exp(-r2 / (2 * 4.0 ** 2))
    model = Medium(c0=np.full(shape, WATER), rho0=np.full(shape, 1000.0), gamma=gamma,
                   c0_min=C0_MIN, c0_max=C0_MAX)
    truth = Medium(c0=c0_true, rho0=np.full(shape, 1000.0), gamma=gamma, c0_min=C0_MIN, c0_max=C0_MAX)
    pulse = capi.synth_source_pulse(g, 0.8, C0_MIN)
    src = SourceSet(positions=[flat(shape, 14, c[1], c[2])], signals=[pulse])
    sens = []
    for k in range(8):
        th = np.deg2rad(22.5 + 45.0 * k)
        sens.append(flat(shape, round(c[0] + 18 * np.cos(th)), round(c[1] + 18 * np.sin(th)), c[2]))
    return Scenario("A", g, model, truth, src, SensorArray(sens), pulse, thickness=8)


def _ellipsoid(shape, center, semi, zmin):
    ix, iy, iz = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")
    q = ((ix - center[0]) / semi[0]) ** 2 + ((iy - center[1]) / semi[1]) ** 2 + ((iz - center[2]) / semi[2]) ** 2
    return (q <= 1.0) & (iz >= zmin)


def breast_scenario(name: str, interior, dx: float, n_src: int, nt: Optional[int] = None,
                    seed: int = 1) -> Scenario:
    """Hemi-ellipsoidal breast hanging into a golden-spiral hemispherical bowl."""
    L = max(interior) * dx
    g = capi.make_grid(list(interior), dx, C0_MAX, 2 * L / C0_MIN)
    if nt is not None:
        g.nt = int(nt)
    shape = g.shape
    pml = [g.pml_size[a] for a in range(3)]
    rng = np.random.default_rng(seed)
    cx = pml[0] + interior[0] / 2.0
    cy = pml[1] + interior[1] / 2.0
    zw = pml[2] + 2.0                        # chest wall plane
    R = 0.47 * min(interior[0], interior[1])  # bowl radius (104.5 mm at 0.5 mm)
    R = min(R, interior[2] - 4.0)
    scale = interior[0] / 108.0
    a, h = 0.62 * R, 0.72 * R               # breast semi-axes (lateral, depth)

    breast = _ellipsoid(shape, (cx, cy, zw), (a, a, h), zw)
    inner = _ellipsoid(shape, (cx, cy, zw), (a - 2, a - 2, h - 2), zw)
    c0 = np.full(shape, WATER)
    c0[breast] = SKIN
    c0[inner] = FAT
    ix, iy, iz = np.meshgrid(*[np.arange(n, dtype=np.float64) for n in shape], indexing="ij")
    for _ in range(12):  # fibroglandular blobs
        while True:
            p = np.array([cx + rng.uniform(-a, a), cy + rng.uniform(-a, a), zw + rng.uniform(0, h)])
            if ((p[0] - cx) / (a - 2)) ** 2 + ((p[1] - cy) / (a - 2)) ** 2 + ((p[2] - zw) / (h - 2)) ** 2 < 0.6:
                break
        r = rng.uniform(3.0, 8.0) * scale
        blob = ((ix - p[0]) ** 2 + (iy - p[1]) ** 2 + (iz - p[2]) ** 2 <= r * r) & inner
        c0[blob] = GLAND
    for _ in range(6):  # vessels: thin tubes between two random interior points
        p0 = np.array([cx + rng.uniform(-0.6, 0.6) * a, cy + rng.uniform(-0.6, 0.6) * a, zw + rng.uniform(0.1, 0.7) * h])
        p1 = np.array([cx + rng.uniform(-0.6, 0.6) * a, cy + rng.uniform(-0.6, 0.6) * a, zw + rng.uniform(0.1, 0.7) * h])
        n = int(np.linalg.norm(p1 - p0) * 2) + 2
        rv = max(1.0, 1.0 * scale)
        for t in np.linspace(0, 1, n):
            q = p0 + t * (p1 - p0)
            lo = np.floor(q - rv - 1).astype(int)
            hi = np.ceil(q + rv + 1).astype(int) + 1
            sl = tuple(slice(max(0, lo[d]), min(shape[d], hi[d])) for d in range(3))
            sub = (ix[sl] - q[0]) ** 2 + (iy[sl] - q[1]) ** 2 + (iz[sl] - q[2]) ** 2 <= rv * rv
            sub &= inner[sl]
            c0[sl][sub] = VESSEL
    gamma = _ellipsoid(shape, (cx, cy, zw), (a + 2, a + 2, h + 2), zw - 2).astype(np.uint8)

    # golden-spiral hemisphere, alternating emitter / receiver
    emit, recv = golden_section_placement(2 * n_src, R, (cx, cy, zw), shape, pml, exclude=gamma)
    model = Medium(c0=np.full(shape, WATER), rho0=np.full(shape, 1000.0), gamma=gamma,
                   c0_min=C0_MIN, c0_max=C0_MAX)
    truth = Medium(c0=c0, rho0=np.full(shape, 1000.0), gamma=gamma, c0_min=C0_MIN, c0_max=C0_MAX)
    pulse = capi.synth_source_pulse(g, 0.8, C0_MIN)
    src = SourceSet(positions=emit, signals=[pulse] * len(emit))
    return Scenario(name, g, model, truth, src, SensorArray(recv), pulse, thickness=8)


def config_b(nt=None):
    return breast_scenario("B", [108, 108, 108], 1e-3, 64, nt)


def config_c(nt=None):
    return breast_scenario("C", [236, 236, 236], 1e-3, 256, nt)


def config_d(nt=3912):
    """442x442x222 at 0.5 mm -> 480x480x256, nt = 3912 as in the paper."""
    return breast_scenario("D", [442, 442, 222], 0.5e-3, 1024, nt)


def config_e(level: int, nt=None):
    """Multigrid levels 2 / 1 / 0.5 mm."""
    interiors = {0: ([112, 112, 56], 2e-3, 978), 1: ([222, 222, 112], 1e-3, 1956), 2: ([442, 442, 222], 0.5e-3, 3912)}
    interior, dx, nt_paper = interiors[level]
    return breast_scenario(f"E{level}", interior, dx, 1024 >> (2 * (2 - level)) if level < 2 else 1024,
                           nt if nt is not None else nt_paper)


def encoding_problem(n_src: int, nt: Optional[int] = None):
    """Small 3-D source-encoding problem (24^3 interior -> 64^3, up to 4 emitters, 6 receivers,
    ball gamma r = 8, Gaussian c0 bump): the inputs of the delayed / unbiasedness parity
    fixtures (tests/golden/make_golden_delayed.py) and tests/test_gpu_encoding.py.
    Returns (grid, model, truth, emitter positions, receiver positions, pulse)."""
    interior, dx = [24, 24, 24], 1e-3
    g = capi.make_grid(interior, dx, C0_MAX, 2 * interior[0] * dx / C0_MIN)
    if nt is not None:
        g.nt = int(nt)
    shape = g.shape
    c = [s // 2 for s in shape]
    gamma = capi.ball_mask(shape, c, 8.0)
    ix, iy, iz = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    r2 = (ix - c[0] - 1) ** 2 + (iy - c[1]) ** 2 + (iz - c[2] + 1) ** 2
    truth_c0 = WATER + 25.0 * np.exp(-r2 / (2 * 3.0 ** 2))
    model = Medium(c0=np.full(shape, WATER), rho0=np.full(shape, 1000.0), gamma=gamma,
                   c0_min=C0_MIN, c0_max=C0_MAX)
    truth = Medium(c0=truth_c0, rho0=np.full(shape, 1000.0), gamma=gamma, c0_min=C0_MIN,
                   c0_max=C0_MAX)
    p = g.pml_size[0]
    src_xyz = [(p + 2, c[1], c[2]), (c[0], p + 2, c[2] + 2), (shape[0] - p - 3, c[1] - 3, c[2]),
               (c[0] + 2, shape[1] - p - 3, c[2] - 2)][:n_src]
    srcs = [flat(shape, *q) for q in src_xyz]
    sens = []
    for k in range(6):
        th = np.deg2rad(15.0 + 60.0 * k)
        sens.append(flat(shape, round(c[0] + 10 * np.cos(th)), round(c[1] + 10 * np.sin(th)), c[2] + 3))
    pulse = capi.synth_source_pulse(g, 0.8, C0_MIN)
    return g, model, truth, srcs, sens, pulse


def config_d_gradient_problem():
    """The config-D grid and phantom with 16 emitters on a ring 1 voxel outside Gamma (z = 40)
    and 16 receivers 2 voxels beside them, nt = 28, the config-D pulse advanced to peak near
    sample 12, observed data zero: the forward and adjoint fields overlap inside Gamma from
    about step 8 to 19, so a 28-step TR gradient at the full 480 x 480 x 256 size (the
    480-point pencils, the nz = 256 rows, the 1.16 M-voxel shell record / replay, the
    correlation) is non-trivial while the fp64 reference finishes in about 1.5 h
    (tests/golden/make_golden_large.py Dgrad, tests/test_gpu_large.py).
    Returns (scenario with nt = 28, emitters, receivers, pulse)."""
    nt = 28
    sc = config_d(nt=nt)
    sh = sc.grid.shape
    gam = np.asarray(sc.model.gamma, bool)
    cx = cy = sh[0] // 2
    full = config_d().pulse          # the untruncated pulse of the config-D grid
    k0 = int(np.argmax(np.abs(full))) - 12
    pulse = np.asarray(full[k0:k0 + nt], np.float64)
    z = 40
    r_g = 0
    while gam[cx + r_g + 1, cy, z]:
        r_g += 1

    def ring(gap, dtheta):
        rr = r_g + gap
        pts = []
        for k in range(16):
            th = 2 * np.pi * k / 16 + dtheta
            x, y = int(round(cx + rr * np.cos(th))), int(round(cy + rr * np.sin(th)))
            while gam[x, y, z]:  # rounding landed on Gamma: step outwards
                x, y = int(round(x + np.cos(th))), int(round(y + np.sin(th)))
            pts.append(flat(sh, x, y, z))
        return pts
    return sc, ring(1, 0.0), ring(1, 2.0 / (r_g + 1)), pulse


CONFIGS = {"A": config_a, "B": config_b, "C": config_c, "D": config_d,
           "E0": lambda nt=None: config_e(0, nt), "E1": lambda nt=None: config_e(1, nt)}
