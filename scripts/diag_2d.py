"""Dev diagnostic: 2-D forward parity vs the reference golden, per-sensor errors."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2102_00755_b200 import capi
from paper_2102_00755_b200.engine import GpuEngine, SourceSet, SensorArray, make_homogeneous_medium, simulate_forward
z = np.load("tests/golden/forward_2d.npz")
g = capi.make_grid([64, 64], 1e-3, 1800.0, 5e-5)
print(g)
m = make_homogeneous_medium(g)
pulse = z["pulse"]
res = simulate_forward(m, SourceSet(list(z["pos"]), [pulse, -0.7 * pulse]), SensorArray(list(z["sens"])), g)
d, r = res.data, z["data"]
for s in range(d.shape[0]):
    print(s, np.linalg.norm(d[s] - r[s]) / np.linalg.norm(r[s]), np.abs(r[s]).max(), np.abs(d[s]).max())
print("total", np.linalg.norm(d - r) / np.linalg.norm(r))
i = np.argmax(np.abs(r[0])); print("peak idx", i, d[0, i-2:i+3], r[0, i-2:i+3])
# single-source 3-D-embedded check: same case as a 3-D grid with nx padded? derivative 2-D
f = np.random.default_rng(0).standard_normal(g.shape)
from oracle import ustfwi_oracle as orc
og = orc.Grid.of(g); oe = orc.SpectralEngine(og)
with GpuEngine(g) as e:
    for ax in range(2):
        for st in ("none", "plus", "minus"):
            a = e.derivative(f, ax, st); b = oe.derivative(f, ax, st)
            print("deriv2d", ax, st, np.linalg.norm(a - b) / np.linalg.norm(b))
