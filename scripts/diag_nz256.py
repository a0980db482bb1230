"""Diagnostic: the nz = 256 small-grid forward against the numpy oracle and oracle/_ref."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ustfwi_oracle as orc, ref
from paper_2102_00755_b200 import capi
from paper_2102_00755_b200.engine import GpuEngine, Medium, SensorArray, SourceSet

dims = [32, 32, 256]
dt = 0.3e-3 / 1800.0
g = capi.grid_from(dims, 1e-3, dt, 70, [4, 4, 10], 1800.0)
sh = g.shape
f = lambda x, y, z: (x * sh[1] + y) * sh[2] + z
rng = np.random.default_rng(11)
c0 = 1480.0 + 60.0 * rng.random(sh)
m = Medium(c0=c0, rho0=np.full(sh, 1000.0))
pulse = capi.synth_source_pulse(g, 0.8, 1350.0)
src = SourceSet([f(16, 16, 40), f(8, 24, 200)], [pulse, -0.6 * pulse])
sens = SensorArray([f(16, 16, 52), f(12, 22, 190), f(20, 10, 46)])  # within reach in 70 steps
with GpuEngine(g) as eng:
    eng.set_medium(m)
    eng.set_sources(src)
    eng.set_sensors(sens)
    data, _ = eng.forward(0)
og = orc.Grid.of(g)
want = orc.simulate_forward(og, c0, m.rho0, list(src.positions), [np.asarray(s) for s in src.signals],
                            list(sens.positions))[0]
r = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
print("gpu vs numpy oracle", r(data, want))
if ref.available():
    class M: pass
    mm = M(); mm.c0, mm.rho0, mm.alpha0, mm.y, mm.gamma, mm.c0_min, mm.c0_max = c0, m.rho0, None, 1.5, None, 1350.0, 1800.0
    wr, _ = ref.simulate_forward(g, mm, list(src.positions), [np.asarray(s) for s in src.signals], list(sens.positions))
    print("gpu vs _ref", r(data, wr), " numpy vs _ref", r(want, wr))
