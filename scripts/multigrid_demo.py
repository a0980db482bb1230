"""BASELINE config 5 / SURVEY §8(d) E: encoded gradients/s on each multigrid level
(2 / 1 / 0.5 mm) and a short coarse-to-fine reconstruction on the device path
(`--quick`: the reconstruction part only).

For each level: one encoded TR gradient timed after a warm-up (device + host API, the same
call a user makes). Then SLBFGS (Algorithm 2, optim.slbfgs_run: nu = 1, H0 = h0 I for the
first step, then the secant scaling) on the 2 mm level with the encoded-gradient estimator
(realization i for iteration i; observed data = forward of the same encoded source on the
truth phantom), the result prolonged to the 1 mm interior with the Blackman-tapered Fourier
interpolation (multigrid.prolong_model) and refined there. Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2102_00755_b200 import multigrid, scenario  # noqa: E402
from paper_2102_00755_b200.engine import GpuEngine, draw_realization, encode  # noqa: E402
from paper_2102_00755_b200.estimators import delay_schedule  # noqa: E402
from paper_2102_00755_b200.optim import slbfgs_run  # noqa: E402


def interior_slices(sc):
    g = sc.grid
    return tuple(slice(g.pml_size[a], g.shape[a] - g.pml_size[a]) for a in range(3))


def rel_err(c, truth, gamma):
    m = gamma.astype(bool)
    return float(np.linalg.norm(c[m] - truth[m]) / np.linalg.norm(truth[m]))


def estimator(eng, sc, base_c0, gam_idx, cache, log):
    """Encoded-gradient estimator with delayed source encoding: realization (seed, iteration k)
    with maximal delay theta; the encoded observed data over nt + ceil(theta/dt) is the
    forward of the same delayed encoded source on the truth phantom (the propagator is
    linear and shift invariant, so this equals sum_i w_i f_i(t - d_i tau))."""
    nt = sc.grid.nt
    dt = sc.grid.dt

    def est(u, theta, k):
        r = draw_realization(sc.n_src, float(theta), dt, scenario.MASTER_SEED, int(k), 0)
        enc, _, nt_ext = encode(sc.sources, None, r, nt)
        if nt_ext != eng.grid.nt:
            eng.set_nt(nt_ext)
        key = (k, nt_ext)
        if key not in cache:
            eng.set_medium(sc.truth)
            eng.set_sources(enc)
            cache.clear()
            cache[key] = eng.forward(0)[0]
        c0 = base_c0.copy()
        c0.ravel()[gam_idx] = np.clip(u, 1350.0, 1800.0)
        m = sc.model
        m.c0 = c0
        eng.set_medium(m)
        eng.set_sources(enc)
        loss, grad = eng.gradient_tr(cache[key], sc.thickness)
        log.append({"iteration": int(k), "tau_s": float(theta), "nt_ext": int(nt_ext), "loss": float(loss)})
        return loss, grad.ravel()[gam_idx]
    return est


def arg(name, default):
    for k, a in enumerate(sys.argv):
        if a == name and k + 1 < len(sys.argv):
            return type(default)(sys.argv[k + 1])
    return default


def main():
    out = {"levels": {}}
    quick = "--quick" in sys.argv
    e1_evals = arg("--e1-evals", 8)       # SLBFGS evaluations on the 1 mm level
    e1_step = arg("--e1-step", 1.0)       # first step on the 1 mm level, m/s
    levels = () if quick else (0, 1, 2)
    for lv in levels:
        sc = scenario.config_e(lv)
        with GpuEngine(sc.grid) as eng:
            enc = sc.encoded(0)
            eng.set_medium(sc.truth)
            eng.set_sources(enc)
            eng.set_sensors(sc.sensors)
            obs, _ = eng.forward(0)
            eng.set_medium(sc.model)
            eng.gradient_tr(obs, sc.thickness)  # warm-up: eager launches
            eng.gradient_tr(obs, sc.thickness)  # warm-up: CUDA-graph capture
            t0 = time.perf_counter()
            eng.gradient_tr(obs, sc.thickness)
            dt = time.perf_counter() - t0
        out["levels"][sc.name] = {"grid": list(sc.grid.shape), "dx_mm": sc.grid.dx[0] * 1e3, "nt": sc.grid.nt,
                                  "n_emitters": sc.n_src, "s_per_gradient": dt, "gradients_per_s": 1.0 / dt}

    # coarse-to-fine: 2 mm (16 evaluations), prolong, 1 mm (8 evaluations), both with the
    # delayed-encoding schedule tau = b (i - 1), b = 2 % of the duration T
    hist = []
    sc0 = scenario.config_e(0)
    gam0 = np.flatnonzero(np.asarray(sc0.model.gamma).ravel())
    base0 = np.asarray(sc0.model.c0, dtype=np.float64).copy()
    b0 = 0.02 * sc0.grid.nt * sc0.grid.dt
    log0 = []
    with GpuEngine(sc0.grid) as eng:
        eng.set_sensors(sc0.sensors)
        est = estimator(eng, sc0, base0, gam0, {}, log0)
        F0, G0 = est(base0.ravel()[gam0], 0.0, 1)
        h0 = 2.0 / np.abs(G0).max()  # first step <= 2 m/s
        res0 = slbfgs_run(est, base0.ravel()[gam0], 16, nu=1.0, h0=h0, bounds=(1350.0, 1800.0),
                          theta=delay_schedule(b0))
    c_coarse = base0.copy()
    c_coarse.ravel()[gam0] = res0.u
    hist.append({"level": sc0.name, "evals": res0.n_evl, "energy": res0.energy, "b_s": b0,
                 "schedule": [(h["iteration"], h["nt_ext"]) for h in log0],
                 "rel_l2_start": rel_err(base0, np.asarray(sc0.truth.c0), sc0.model.gamma),
                 "rel_l2_end": rel_err(c_coarse, np.asarray(sc0.truth.c0), sc0.model.gamma)})
    sc1 = scenario.config_e(1)
    s0, s1 = interior_slices(sc0), interior_slices(sc1)
    fine_int = [sc1.grid.shape[a] - 2 * sc1.grid.pml_size[a] for a in range(3)]
    up = multigrid.prolong_model(c_coarse[s0], fine_int)
    c1 = np.asarray(sc1.model.c0, dtype=np.float64).copy()
    gam1_mask = np.asarray(sc1.model.gamma).astype(bool)
    c1_int = c1[s1]
    c1_int[gam1_mask[s1]] = np.clip(up[gam1_mask[s1]], 1350.0, 1800.0)
    c1[s1] = c1_int
    gam1 = np.flatnonzero(gam1_mask.ravel())
    b1 = 0.02 * sc1.grid.nt * sc1.grid.dt
    log1 = []
    with GpuEngine(sc1.grid) as eng:
        eng.set_sensors(sc1.sensors)
        est = estimator(eng, sc1, c1, gam1, {}, log1)
        F1, G1 = est(c1.ravel()[gam1], 0.0, 1)
        res1 = slbfgs_run(est, c1.ravel()[gam1], e1_evals, nu=1.0, h0=e1_step / np.abs(G1).max(),
                          bounds=(1350.0, 1800.0), theta=delay_schedule(b1))
    c_fine = c1.copy()
    c_fine.ravel()[gam1] = res1.u
    water = np.asarray(sc1.model.c0, dtype=np.float64)
    hist.append({"level": sc1.name, "evals": res1.n_evl, "first_step_m_s": e1_step, "energy": res1.energy, "b_s": b1,
                 "schedule": [(h["iteration"], h["nt_ext"]) for h in log1],
                 "rel_l2_water_init": rel_err(water, np.asarray(sc1.truth.c0), sc1.model.gamma),
                 "rel_l2_prolonged_init": rel_err(c1, np.asarray(sc1.truth.c0), sc1.model.gamma),
                 "rel_l2_end": rel_err(c_fine, np.asarray(sc1.truth.c0), sc1.model.gamma)})
    out["multigrid_reconstruction"] = hist
    print(json.dumps(out))


if __name__ == "__main__":
    main()
