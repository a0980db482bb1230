"""Tiny device workloads for compute-sanitizer (memcheck / racecheck / synccheck), SURVEY §5.2:
config A geometry (64^3: the 64-point pencils, nz = 64 rows) for a short TR gradient with the
CUDA graph path, the stepper API and the rho0 gradient, plus two small grids that select the
480-point x and y pencils and the nz = 256 row kernels (the config-D kernels). Only the
engine library is loaded (no torch).

    compute-sanitizer --tool memcheck python scripts/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2102_00755_b200 import capi, scenario
from paper_2102_00755_b200.engine import GpuEngine, Medium, SensorArray, SourceSet

sc = scenario.config_a(nt=int(os.environ.get("SAN_NT", "12")))
obs = np.zeros((len(sc.sensors.positions), sc.grid.nt))
with GpuEngine(sc.grid) as eng:
    eng.set_medium(sc.model)
    eng.set_sources(sc.encoded(0))
    eng.set_sensors(sc.sensors)
    for _ in range(3):  # eager, graph capture, graph replay
        loss, grad = eng.gradient_tr(obs, 8)
    loss_r, grad_r = eng.gradient_tr(obs, 8, param="rho0")
    data, trace = eng.forward(8)
print(f"config A: loss {loss:.4e} rho0 loss {loss_r:.4e} |data| {np.linalg.norm(data):.4e}")

for dims in ([480, 16, 256], [8, 480, 256]):
    g = capi.grid_from(dims, 1e-3, 0.3e-3 / 1800.0, 4, [0, 0, 0], 1800.0)
    sh = g.shape
    f = lambda x, y, z: (x * sh[1] + y) * sh[2] + z
    c = [d // 2 for d in sh]
    m = Medium(c0=np.full(sh, 1500.0), rho0=np.full(sh, 1000.0), gamma=capi.ball_mask(sh, c, 3.0))
    pulse = capi.synth_source_pulse(g, 0.8, 1350.0)
    with GpuEngine(g) as eng:
        eng.set_medium(m)
        eng.set_sources(SourceSet([f(c[0], c[1], c[2] + 5)], [pulse]))
        eng.set_sensors(SensorArray([f(c[0], c[1], c[2] + 8)]))
        loss, grad = eng.gradient_tr(np.zeros((1, g.nt)), 1)
    print(f"{dims}: loss {loss:.4e}")
print("sanitize case done")
