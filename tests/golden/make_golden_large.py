"""Large parity fixtures from the REFERENCE itself (oracle/_ref), pinning the benchmarked inputs.

Run here (where /root/reference exists), one fixture per process (hours of fp64 CPU work):

    make -C oracle
    python tests/golden/make_golden_large.py B       # config B, full nt = 961, 64 Rademacher-encoded emitters
    python tests/golden/make_golden_large.py D       # config D grid + bench phantom + 1024 encoded emitters, nt = 160
    python tests/golden/make_golden_large.py drift   # config A geometry at nt = 3912 (fp32 drift over 3*3912 steps)
    python tests/golden/make_golden_large.py rho0    # config A (nt = 393), heterogeneous rho0: rho0 and c0 gradients
    python tests/golden/make_golden_large.py Dgrad   # config-D grid, 16 + 16 transducers next to Gamma, nt = 28 TR gradient
    python tests/golden/make_golden_large.py E0      # config E level 0 (2 mm, 144x144x96), full nt = 978, observed = 0

Every input is built exactly as bench.py / scenario.py build it (same seeds, same encoding
realization r = 0 of master seed 20210201, tau = 0), so the device run in
tests/test_gpu_large.py sees the same SourceSet the reference saw: an encoded SourceSet
of n emitters with signals w_i * pulse (SPEC.md:296-304 with tau = 0; the reference's
SourceSet::sample, medium.hpp:80-84, sums them per step).

Stored: traces (float64, small), loss, the shell-trace checksums, and the Gamma-restricted
gradient as float32 (the parity bar is 1e-3) plus its fp64 norm / checksum.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2102_00755_b200 import scenario  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def encoded_inputs(sc, r=0):
    enc = sc.encoded(r)
    assert not np.any(enc.delays), "tau = 0 fixtures"
    pos = list(enc.positions)
    sig = [float(w) * np.asarray(s, np.float64) for w, s in zip(enc.weights, enc.signals)]
    return enc, pos, sig


def trace_checksums(trace):
    t = np.asarray(trace, np.float64)
    return np.array([t.sum(), np.abs(t).sum(), (t ** 2).sum()])


def gradient_fixture(sc, name, r=0, observed_zero=False):
    g = sc.grid
    enc, pos, sig = encoded_inputs(sc, r)
    sens = list(sc.sensors.positions)
    t0 = time.time()
    if observed_zero:
        observed = np.zeros((len(sens), g.nt))
    else:
        observed, _ = ref.simulate_forward(g, sc.truth, pos, sig, sens)
    t1 = time.time()
    data_model, trace = ref.simulate_forward(g, sc.model, pos, sig, sens, boundary_thickness=sc.thickness)
    t2 = time.time()
    loss, grad = ref.gradient_time_reversal(g, sc.model, pos, sig, sens, observed, sc.thickness)
    t3 = time.time()
    gidx = np.flatnonzero(np.asarray(sc.model.gamma).ravel())
    gg = grad.ravel()[gidx]
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"), observed=observed, data_model=data_model, nt=g.nt,
        weights=np.asarray(enc.weights), trace_checksum=trace_checksums(trace), loss=loss,
        grad_gamma=gg.astype(np.float32), grad_norm=np.linalg.norm(gg), grad_sum=gg.sum(), gamma_idx=gidx,
        grad_outside_max=np.abs(np.delete(grad.ravel(), gidx)).max(), seconds=np.array([t1 - t0, t2 - t1, t3 - t2]))
    print(f"{name}: obs {t1 - t0:.0f}s fwd+trace {t2 - t1:.0f}s gradient {t3 - t2:.0f}s loss {loss:.6e}", flush=True)


def config_b_fixture():
    gradient_fixture(scenario.config_b(), "config_b")


def config_e0_fixture():
    # the 2 mm multigrid level at its full nt = 978: 144 x 144 x 96 (the 144-point pencils and
    # the nz = 96 z kernels), 64 encoded emitters; observed = 0 (the residual is the model data)
    gradient_fixture(scenario.config_e(0), "config_e0", observed_zero=True)


def drift_fixture():
    # config A geometry run for the config-D step count: fp32 error growth over 3*3912 steps
    gradient_fixture(scenario.config_a(nt=3912), "config_a_nt3912")


def config_d_fixture(nt=160):
    sc = scenario.config_d(nt=nt)
    g = sc.grid
    enc, pos, sig = encoded_inputs(sc)
    sens = list(sc.sensors.positions)
    t0 = time.time()
    data, trace = ref.simulate_forward(g, sc.model, pos, sig, sens, boundary_thickness=sc.thickness)
    t1 = time.time()
    tsum = trace_checksums(trace)
    # a per-step checksum of the shell trace (catches a step-dependent error at any Gamma voxel)
    per_step = np.asarray(trace, np.float64).sum(axis=1)
    per_step_abs = np.abs(np.asarray(trace, np.float64)).sum(axis=1)
    sub = np.asarray(trace, np.float64)[::8, ::97]
    np.savez_compressed(os.path.join(OUT, "config_d_short.npz"), data_model=data, nt=g.nt,
                        weights=np.asarray(enc.weights), trace_checksum=tsum, trace_step_sum=per_step,
                        trace_step_abs=per_step_abs, trace_sub=sub, trace_stride=np.array([8, 97]),
                        n_shell=np.asarray(trace).shape[1], seconds=np.array([t1 - t0]))
    print(f"config_d_short: forward {t1 - t0:.0f}s, |data| {np.linalg.norm(data):.6e}", flush=True)


def config_d_gradient_fixture():
    sc, emit, recv, pulse = scenario.config_d_gradient_problem()
    g = sc.grid
    sig = [pulse * (1.0 if k % 2 == 0 else -1.0) for k in range(len(emit))]  # a fixed +-1 encoding
    observed = np.zeros((len(recv), g.nt))
    t0 = time.time()
    loss, grad = ref.gradient_time_reversal(g, sc.model, emit, sig, recv, observed, sc.thickness)
    t1 = time.time()
    gidx = np.flatnonzero(np.asarray(sc.model.gamma).ravel())
    gg = grad.ravel()[gidx]
    sel = np.flatnonzero(np.abs(gg) > 1e-3 * np.abs(gg).max())
    np.savez_compressed(os.path.join(OUT, "config_d_grad.npz"), nt=g.nt, loss=loss, grad_norm=np.linalg.norm(gg),
                        grad_sum=gg.sum(), grad_abs_sum=np.abs(gg).sum(), gamma_count=gidx.size,
                        grad_sel_idx=gidx[sel], grad_sel=gg[sel].astype(np.float32),
                        grad_sub_idx=gidx[::211], grad_sub=gg[::211].astype(np.float32),
                        grad_outside_max=np.abs(np.delete(grad.ravel(), gidx)).max(), seconds=np.array([t1 - t0]))
    print(f"config_d_grad: {t1 - t0:.0f}s loss {loss:.6e} |g| {np.linalg.norm(gg):.3e} nonzero-ish {sel.size}", flush=True)


def rho0_fixture():
    """Heterogeneous rho0 at config A: the rho0 gradient (GradientParam::rho0,
    gradient.hpp:117-128,213-239; oracle/_ref is built with the F3 compile fix) and the c0
    gradient of the same medium (nt = 393, f_obs = truth data)."""
    from paper_2102_00755_b200.engine import Medium
    sc = scenario.config_a()
    g = sc.grid
    shape = g.shape
    c = [s // 2 for s in shape]
    ix, iy, iz = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    r2 = (ix - c[0] + 3) ** 2 + (iy - c[1]) ** 2 + (iz - c[2] - 2) ** 2
    rho = 1000.0 + 40.0 * np.exp(-r2 / (2 * 5.0 ** 2))
    model = Medium(c0=sc.model.c0, rho0=rho, gamma=sc.model.gamma, c0_min=sc.model.c0_min, c0_max=sc.model.c0_max)
    truth = Medium(c0=sc.truth.c0, rho0=np.full(shape, 1000.0), gamma=sc.model.gamma, c0_min=sc.model.c0_min,
                   c0_max=sc.model.c0_max)
    pos, sig = list(sc.sources.positions), [np.asarray(s) for s in sc.sources.signals]
    sens = list(sc.sensors.positions)
    observed, _ = ref.simulate_forward(g, truth, pos, sig, sens)
    loss, grad_rho = ref.gradient_tr_opts(g, model, pos, sig, sens, observed, 8, param="rho0")
    _, grad_c0 = ref.gradient_time_reversal(g, model, pos, sig, sens, observed, 8)
    gidx = np.flatnonzero(np.asarray(sc.model.gamma).ravel())
    np.savez_compressed(os.path.join(OUT, "config_a_rho0.npz"), rho0=rho.astype(np.float64), observed=observed,
                        loss=loss, grad_rho0=grad_rho.ravel()[gidx], grad_c0=grad_c0.ravel()[gidx], gamma_idx=gidx,
                        grad_rho0_outside_max=np.abs(np.delete(grad_rho.ravel(), gidx)).max())
    print(f"config_a_rho0: loss {loss:.6e} |g_rho0| {np.linalg.norm(grad_rho):.3e}", flush=True)


if __name__ == "__main__":
    if not ref.available():
        sys.exit("oracle/_ref missing: make -C oracle")
    which = sys.argv[1] if len(sys.argv) > 1 else ""
    {"B": config_b_fixture, "D": config_d_fixture, "drift": drift_fixture, "rho0": rho0_fixture,
     "Dgrad": config_d_gradient_fixture, "E0": config_e0_fixture}[which]()
