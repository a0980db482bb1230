"""Profiling driver: a few steps of the device engine on a config grid (default D's
480x480x256) with a homogeneous medium and a cheap setup, for ncu / nsys-free timing.

    python scripts/prof_step.py [--config D] [--nt 12] [--grad]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2102_00755_b200 import capi
from paper_2102_00755_b200.engine import GpuEngine, Medium, SensorArray, SourceSet

DIMS = {"A": ([44, 44, 44], 1e-3), "B": ([108, 108, 108], 1e-3), "C": ([236, 236, 236], 1e-3),
        "D": ([442, 442, 222], 0.5e-3)}

p = argparse.ArgumentParser()
p.add_argument("--config", default="D")
p.add_argument("--nt", type=int, default=12)
p.add_argument("--grad", action="store_true")
a = p.parse_args()
interior, dx = DIMS[a.config]
g = capi.make_grid(interior, dx, 1800.0, 1e-3)
g.nt = a.nt
sh = g.shape
c = [s // 2 for s in sh]
gamma = capi.ball_mask(sh, c, min(sh) / 4)
m = Medium(c0=np.full(sh, 1500.0), rho0=np.full(sh, 1000.0), gamma=gamma)
pulse = capi.synth_source_pulse(g, 0.8, 1350.0)
f = lambda x, y, z: (x * sh[1] + y) * sh[2] + z
src = SourceSet([f(sh[0] // 8, c[1], c[2])], [pulse])
sens = SensorArray([f(7 * sh[0] // 8, c[1], c[2]), f(c[0], sh[1] // 8, c[2])])
with GpuEngine(g) as eng:
    eng.set_medium(m)
    eng.set_sources(src)
    eng.set_sensors(sens)
    t0 = time.time()
    if a.grad:
        eng.gradient_tr(np.zeros((2, g.nt)), 4)
    else:
        eng.forward(0)
    eng.synchronize()
    print(f"{a.config} nt={a.nt} grad={a.grad}: {time.time() - t0:.3f}s, {eng.launch_count()} launches")
