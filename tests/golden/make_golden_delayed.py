"""Delayed / conventional source-encoding fixtures from the REFERENCE itself (oracle/_ref).

SPEC.md:296-313 defines the encoded super-source s^ = sum w_i s_i(t - d_i tau) and data
f^ = sum w_i f_i(t - d_i tau) on the extended duration nt + ceil(tau/dt); the reference has
no encoding code, so the oracle runs its own compute_gradient on the
EXPANDED SourceSet (each delayed signal with d_i tau / dt zeros prepended, weights folded in)
over the extended grid — the exact inputs the device path builds on the fly.

    python tests/golden/make_golden_delayed.py      (~50 min single-threaded)

delayed_encoding.npz
  small 3-D problem (scenario.encoding_problem: 24^3 interior -> 64^3, 2 emitters, 6 receivers, ball gamma r = 8):
  * per-source observed data f_i (truth medium), nt = 768 (every field has left the domain)
  * the tau = 2T, d = (0, 1), w = (+1, -1) encoded gradient and loss over nt_ext = 3 nt
    (the second emitter fires after the first's field has left the domain)
  * the exact 2-source gradient sum_i grad D_i and loss sum_i D_i (SPEC.md:304 bar 1e-3)
unbiased_encoding.npz
  4 emitters of the same problem, tau = 0: the full gradient sum_i grad D_i (the target of
  the 1/sqrt(n) Monte-Carlo check) and per-source observed data.
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
from paper_2102_00755_b200.engine import Medium  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


# The tau = 2T check needs every single-source field to have left the domain within T: the
# pulse (peak near sample 200, ~400 samples long) plus one domain crossing (~260 steps) -> nt 768
DELAYED_NT = 768


def small_problem(n_src, nt=None):
    return scenario.encoding_problem(n_src, nt)


def with_nt(g, nt):
    h = capi.UstfwiGrid.from_buffer_copy(g)
    h.nt = int(nt)
    return h


def delayed_fixture():
    g, model, truth, srcs, sens, pulse = small_problem(2, DELAYED_NT)
    nt = g.nt
    t0 = time.time()
    f = [ref.simulate_forward(g, truth, [s], [pulse], sens)[0] for s in srcs]
    # exact sum of the single-source gradients (and losses)
    singles = [ref.gradient_time_reversal(g, model, [s], [pulse], sens, f[i], 8) for i, s in enumerate(srcs)]
    t1 = time.time()
    w = np.array([1.0, -1.0])
    ext = 2 * nt                                # tau = 2T -> ceil(tau/dt) = 2 nt
    d = np.array([0, ext])
    nt_ext = nt + ext
    ge = with_nt(g, nt_ext)
    sig = [w[i] * np.concatenate([np.zeros(d[i]), pulse]) for i in range(2)]
    f_hat = np.zeros((len(sens), nt_ext))
    for i in range(2):
        f_hat[:, d[i]:d[i] + nt] += w[i] * f[i]
    loss_e, grad_e = ref.gradient_time_reversal(ge, model, srcs, sig, sens, f_hat, 8)
    t2 = time.time()
    gidx = np.flatnonzero(np.asarray(model.gamma).ravel())
    np.savez_compressed(os.path.join(OUT, "delayed_encoding.npz"), nt=nt, ext=ext, weights=w, delay_steps=d,
                        f=np.stack(f), loss_enc=loss_e, grad_enc=grad_e.ravel()[gidx],
                        loss_sum=sum(s[0] for s in singles), grad_sum=sum(s[1] for s in singles).ravel()[gidx],
                        gamma_idx=gidx, seconds=np.array([t1 - t0, t2 - t1]))
    cross = np.linalg.norm(grad_e - sum(s[1] for s in singles)) / np.linalg.norm(sum(s[1] for s in singles))
    print(f"delayed: singles {t1 - t0:.0f}s encoded {t2 - t1:.0f}s; reference cross-talk rel l2 {cross:.2e}", flush=True)


def unbiased_fixture():
    g, model, truth, srcs, sens, pulse = small_problem(4)
    f = [ref.simulate_forward(g, truth, [s], [pulse], sens)[0] for s in srcs]
    singles = [ref.gradient_time_reversal(g, model, [s], [pulse], sens, f[i], 8) for i, s in enumerate(srcs)]
    gidx = np.flatnonzero(np.asarray(model.gamma).ravel())
    full = sum(s[1] for s in singles)
    np.savez_compressed(os.path.join(OUT, "unbiased_encoding.npz"), f=np.stack(f), grad_full=full.ravel()[gidx],
                        loss_full=sum(s[0] for s in singles), gamma_idx=gidx, nt=g.nt)
    print(f"unbiased: |full| {np.linalg.norm(full):.3e}", flush=True)


if __name__ == "__main__":
    if not ref.available():
        sys.exit("oracle/_ref missing: make -C oracle")
    which = sys.argv[1:] or ["delayed", "unbiased"]
    if "delayed" in which:
        delayed_fixture()
    if "unbiased" in which:
        unbiased_fixture()
