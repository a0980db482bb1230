"""Generate the committed golden fixtures from the REFERENCE itself (oracle/_ref).

oracle/_ref/libustfwi_ref.so is the unmodified reference headers compiled with the
in-repo FFTW-API shim (oracle/Makefile). Run here (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py [--quick]

Fixtures (small, committed):
  derivative_3d.npz   SpectralEngine::derivative on a seeded 16x12x10 field, all axes/staggers
  forward_2d.npz      simulate_forward on the reference's 2-D linearity-test grid
  config_a.npz        config A (64^3, nt=393): observed data (truth medium), model traces,
                      subsampled shell trace, TR gradient on gamma and loss
  config_a_short.npz  config A truncated to nt=96 with f_obs = 0 (fast GPU parity case)
  multigrid.npz       fourier_interpolate (up / down / mixed, with and without the Blackman
                      taper, 3-D and 2-D) and lowpass_filter_timeseries on seeded inputs
  config_a_absorb.npz config A at nt=96 with power-law absorption (alpha0 3 dB/(MHz^y cm) in
                      gamma, 0.5 outside): y = 1.5 traces + TR gradient + loss (f_obs = 0), the
                      same gradient with GradientOptions::dispersion_enabled = false, the alpha0
                      and y gradients (GradientParam), the alpha0 gradient of the lossless model,
                      y = 2 (no dispersion term) traces
  config_a_fd.npz     config A (nt=393): loss, the directional derivative <G, delta> of the
                      TR gradient with the shell = all of gamma (thickness 12), the central finite
                      difference of evaluate_loss along delta (eps 0.5 m/s), and the relative l2
                      distance of the thickness-1/2/4/8 TR gradients to the thickness-12 one
                      (`--fd-only`; ~25 min single-threaded)
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2102_00755_b200 import capi, scenario  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def derivative_fixture():
    g = capi.grid_from([16, 12, 10], 1e-3, 0.3e-3 / 1500.0, 4, [0, 0, 0], 1500.0)
    rng = np.random.default_rng(17)
    f = rng.standard_normal(g.shape)
    out = {"f": f, "dims": np.array(g.shape), "dx": 1e-3, "dt": g.dt, "c_ref": 1500.0}
    for axis in range(3):
        for st, name in enumerate(["none", "plus", "minus"]):
            out[f"d{axis}_{name}"] = ref.engine_derivative(g, f, axis, st)
    # a PML-padded grid as well (kappa with c_ref from make_grid)
    g2 = capi.make_grid([4, 4, 4], 1e-3, 1800.0, 2e-6)
    f2 = rng.standard_normal(g2.shape)
    out["f2"] = f2
    out["g2"] = np.array([*g2.shape, g2.pml_size[0], g2.pml_size[1], g2.pml_size[2], g2.nt])
    out["g2_dt"] = g2.dt
    for axis in range(3):
        out[f"g2_d{axis}_plus"] = ref.engine_derivative(g2, f2, axis, 1)
    np.savez_compressed(os.path.join(OUT, "derivative_3d.npz"), **out)


def forward_2d_fixture():
    # test_solver.cpp:82-119 grid: make_grid({64,64}, 1e-3, 1800, 5e-5)
    g = capi.make_grid([64, 64], 1e-3, 1800.0, 5e-5)
    shape = g.shape
    pulse = capi.synth_source_pulse(g, 0.8, 1500.0)
    c0 = np.full(shape, 1500.0)
    rho0 = np.full(shape, 1000.0)

    class M:
        pass
    m = M()
    m.c0, m.rho0, m.alpha0, m.y, m.gamma, m.c0_min, m.c0_max = c0, rho0, None, 1.5, None, 1350.0, 1800.0
    pos = [24 * shape[1] + 30, 30 * shape[1] + 24]
    sig = [pulse, -0.7 * pulse]
    sens = [40 * shape[1] + 40, 20 * shape[1] + 50, 70 * shape[1] + 70]
    data, _ = ref.simulate_forward(g, m, pos, sig, sens)
    np.savez_compressed(os.path.join(OUT, "forward_2d.npz"), data=data, pos=np.array(pos), sens=np.array(sens),
                        pulse=pulse, nt=g.nt, dims=np.array(shape))


def config_a_fixture(nt, name, trace_stride=(8, 16), observed_zero=False):
    """observed_zero: use f_obs = 0 (residual = the model data) so that a short run still
    has an O(1) residual and a well-conditioned gradient."""
    sc = scenario.config_a(nt=nt)
    g = sc.grid
    t0 = time.time()
    pos, sig = list(sc.sources.positions), [np.asarray(s) for s in sc.sources.signals]
    if observed_zero:
        observed = np.zeros((len(sc.sensors.positions), g.nt))
    else:
        observed, _ = ref.simulate_forward(g, sc.truth, pos, sig, sc.sensors.positions)
    t1 = time.time()
    data_model, trace = ref.simulate_forward(g, sc.model, pos, sig, sc.sensors.positions, boundary_thickness=8)
    t2 = time.time()
    loss, grad = ref.gradient_time_reversal(g, sc.model, pos, sig, sc.sensors.positions, observed, 8)
    t3 = time.time()
    gidx = np.flatnonzero(np.asarray(sc.model.gamma).ravel())
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"), observed=observed, data_model=data_model,
        trace_sub=trace[::trace_stride[0], ::trace_stride[1]], trace_stride=np.array(trace_stride),
        trace_checksum=np.array([trace.sum(), np.abs(trace).sum(), (trace ** 2).sum()]),
        loss=loss, grad_gamma=grad.ravel()[gidx], gamma_idx=gidx, nt=g.nt,
        grad_outside_max=np.abs(np.delete(grad.ravel(), gidx)).max() if grad.size > gidx.size else 0.0,
        seconds=np.array([t1 - t0, t2 - t1, t3 - t2]))
    print(f"{name}: fwd {t1 - t0:.1f}s fwd+trace {t2 - t1:.1f}s gradient {t3 - t2:.1f}s loss {loss:.6e}")


def multigrid_fixture():
    rng = np.random.default_rng(23)
    out = {}
    cases = {"up": ((12, 10, 8), (16, 20, 12)), "down": ((16, 20, 12), (8, 10, 6)), "mixed": ((12, 10, 8), (8, 20, 8)),
             "2d": ((32, 24), (48, 16))}
    for name, (src, dst) in cases.items():
        f = rng.standard_normal(src)
        out[f"{name}_in"] = f
        out[f"{name}_dims"] = np.array(dst)
        out[f"{name}_none"] = ref.fourier_interpolate(f, dst, False)
        out[f"{name}_blackman"] = ref.fourier_interpolate(f, dst, True)
    sig = rng.standard_normal((4, 500))
    out["lp_in"] = sig
    out["lp_1MHz"] = np.stack([ref.lowpass_timeseries(x, 1e-7, 1e6) for x in sig])
    out["lp_2MHz_tr02_a40"] = np.stack([ref.lowpass_timeseries(x, 1e-7, 2e6, 0.2, 40.0) for x in sig])
    np.savez_compressed(os.path.join(OUT, "multigrid.npz"), **out)


def absorbing_medium(m, y):
    import copy
    a = copy.copy(m)
    gam = np.asarray(m.gamma, bool)
    a.alpha0 = np.where(gam, 3.0, 0.5)
    a.y = y
    return a


def config_a_absorb_fixture(nt=96):
    sc = scenario.config_a(nt=nt)
    g = sc.grid
    pos, sig = list(sc.sources.positions), [np.asarray(s) for s in sc.sources.signals]
    m15 = absorbing_medium(sc.model, 1.5)
    m20 = absorbing_medium(sc.model, 2.0)
    observed = np.zeros((len(sc.sensors.positions), g.nt))
    data15, trace = ref.simulate_forward(g, m15, pos, sig, sc.sensors.positions, boundary_thickness=8)
    data20, _ = ref.simulate_forward(g, m20, pos, sig, sc.sensors.positions)
    lossless, _ = ref.simulate_forward(g, sc.model, pos, sig, sc.sensors.positions)
    loss, grad = ref.gradient_time_reversal(g, m15, pos, sig, sc.sensors.positions, observed, 8)
    loss_nd, grad_nd = ref.gradient_tr_opts(g, m15, pos, sig, sc.sensors.positions, observed, 8,
                                            dispersion_enabled=False)
    loss_a0, grad_a0 = ref.gradient_tr_opts(g, m15, pos, sig, sc.sensors.positions, observed, 8, param="alpha0")
    loss_y, grad_y = ref.gradient_tr_opts(g, m15, pos, sig, sc.sensors.positions, observed, 8, param="y")
    _, grad_a0_lossless = ref.gradient_tr_opts(g, sc.model, pos, sig, sc.sensors.positions, observed, 8,
                                               param="alpha0")
    gidx = np.flatnonzero(np.asarray(sc.model.gamma).ravel())
    extra = dict(grad_alpha0=grad_a0.ravel()[gidx], grad_y=grad_y.ravel()[gidx],
                 grad_alpha0_lossless=grad_a0_lossless.ravel()[gidx], loss_alpha0=loss_a0, loss_y=loss_y)
    np.savez_compressed(os.path.join(OUT, "config_a_absorb.npz"), **extra, nt=g.nt, data_y15=data15, data_y20=data20,
                        data_lossless=lossless, trace_checksum=np.array([trace.sum(), np.abs(trace).sum()]),
                        loss=loss, grad_gamma=grad.ravel()[gidx], gamma_idx=gidx,
                        loss_nodisp=loss_nd, grad_gamma_nodisp=grad_nd.ravel()[gidx])
    print(f"config_a_absorb: loss {loss:.6e}, |abs - lossless| / |lossless| = "
          f"{np.linalg.norm(data15 - lossless) / np.linalg.norm(lossless):.3e}")


def fd_direction(shape, gamma):
    """Smooth bump inside gamma, the same formula as tests/test_gpu_gradcheck.py."""
    c = [n // 2 for n in shape]
    ix, iy, iz = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    r2 = (ix - c[0] - 2) ** 2 + (iy - c[1] + 1) ** 2 + (iz - c[2]) ** 2
    return np.exp(-r2 / (2 * 3.0 ** 2)) * np.asarray(gamma, dtype=np.float64)


def config_a_fd_fixture(eps=0.5):
    from paper_2102_00755_b200.engine import Medium
    sc = scenario.config_a()
    g = sc.grid
    pos, sig, sens = list(sc.sources.positions), list(sc.sources.signals), list(sc.sensors.positions)
    delta = fd_direction(g.shape, sc.model.gamma)
    obs, _ = ref.simulate_forward(g, sc.truth, pos, sig, sens)
    loss, g_full = ref.gradient_time_reversal(g, sc.model, pos, sig, sens, obs, 12)
    dJ = float(np.sum(g_full * delta))
    c0 = np.asarray(sc.model.c0, dtype=np.float64)

    def with_c0(cc):
        m = sc.model
        return Medium(c0=cc, rho0=m.rho0, gamma=m.gamma, c0_min=m.c0_min, c0_max=m.c0_max)
    jp = ref.evaluate_loss(g, with_c0(c0 + eps * delta), pos, sig, sens, obs)
    jm = ref.evaluate_loss(g, with_c0(c0 - eps * delta), pos, sig, sens, obs)
    errs = []
    for t in (1, 2, 4, 8):
        _, gt = ref.gradient_time_reversal(g, sc.model, pos, sig, sens, obs, t)
        errs.append(float(np.linalg.norm(gt - g_full) / np.linalg.norm(g_full)))
    np.savez_compressed(os.path.join(OUT, "config_a_fd.npz"), loss=loss, dJ=dJ, fd=(jp - jm) / (2 * eps), eps=eps,
                        thickness=np.array([1, 2, 4, 8]), tr_err_vs_12=np.array(errs))
    print(f"config_a_fd: dJ {dJ:.6e} fd {(jp - jm) / (2 * eps):.6e} tr errors {errs}")


if __name__ == "__main__":
    if "--fd-only" in sys.argv:
        config_a_fd_fixture()
        sys.exit(0)
    if "--multigrid-only" in sys.argv:
        multigrid_fixture()
        sys.exit(0)
    if "--absorb-only" in sys.argv:
        config_a_absorb_fixture()
        sys.exit(0)
    if not ref.available():
        sys.exit("oracle/_ref missing: make -C oracle")
    derivative_fixture()
    forward_2d_fixture()
    config_a_fixture(96, "config_a_short", observed_zero=True)
    multigrid_fixture()
    config_a_absorb_fixture()
    if "--quick" not in sys.argv:
        config_a_fixture(None, "config_a")
