"""The kernel-selection switches (USTFWI_PENCIL_TMA=0: cp.async pencils, USTFWI_ZROW2=0: 8-row
z kernels, USTFWI_GENERIC=1: runtime-plan Stockham kernels, USTFWI_X480=1: 32x15 x pass)
compute the same step: forward traces of a grid that selects the 480-point y pencils and
the nz = 256 z kernels agree across variants (each variant in its own process, the switches
are read once). On a 480 x 480 x 32 grid the three separate pencil launches (default) and the
experimental fused y-x-y chain kernel (USTFWI_CHAIN=1) give the same traces and TR gradient,
and the eager launches (USTFWI_GRAPH=0) the same as the CUDA-graph replay; the SM-partitioned
pair loop (default: green contexts) the same as the shared-SM one (USTFWI_GREEN=0) and as the
other split (USTFWI_GREEN=-72)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r'''
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_2102_00755_b200 import capi
from paper_2102_00755_b200.engine import GpuEngine, Medium, SensorArray, SourceSet
dims = {"x": [480, 16, 256], "y": [8, 480, 256], "xy": [480, 480, 32]}[sys.argv[2]]
g = capi.grid_from(dims, 1e-3, 0.3e-3 / 1800.0, 40, [0, 0, 0], 1800.0)
sh = g.shape
f = lambda x, y, z: (x * sh[1] + y) * sh[2] + z
rng = np.random.default_rng(4)
c0 = 1480.0 + 60.0 * rng.random(sh)
m = Medium(c0=c0, rho0=np.full(sh, 1000.0))
pulse = capi.synth_source_pulse(g, 0.8, 1350.0)
c = [d // 2 for d in sh]
src = SourceSet([f(c[0], c[1], c[2])], [pulse])
sens = SensorArray([f(c[0], c[1], c[2] + 6), f(c[0], min(c[1] + 5, sh[1] - 1), c[2])])
with GpuEngine(g) as eng:
    eng.set_medium(m)
    eng.set_sources(src)
    eng.set_sensors(sens)
    data, _ = eng.forward(0)
    if sys.argv[2] == "xy":  # a TR gradient too (both y-x-y chains, two streams, graph replay)
        m.gamma = capi.ball_mask(sh, c, 6.0)
        eng.set_medium(m)
        for _ in range(3):
            loss, grad = eng.gradient_tr(np.zeros_like(data), 2)
        data = np.concatenate([data.ravel(), grad.ravel()[::97], [loss]])
print(json.dumps(np.asarray(data).tolist()))
'''


def run(env_extra, layout):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, layout], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.array(json.loads(r.stdout.strip().splitlines()[-1]))


@pytest.mark.parametrize("layout,variant", [
    ("y", {"USTFWI_PENCIL_TMA": "0"}), ("y", {"USTFWI_ZROW2": "0"}), ("y", {"USTFWI_GENERIC": "1"}),
    ("x", {"USTFWI_X480": "1"}), ("x", {"USTFWI_PENCIL_TMA": "0"}),
    ("xy", {"USTFWI_CHAIN": "1"}), ("xy", {"USTFWI_GRAPH": "0"}),
    ("y", {"USTFWI_ZFUSE": "1"}), ("x", {"USTFWI_ZFUSE": "1"}),
    ("xy", {"USTFWI_GREEN": "0"}), ("xy", {"USTFWI_GREEN": "0", "USTFWI_GRAPH": "0"}),
    ("xy", {"USTFWI_GREEN": "-72"}),
])
def test_kernel_variants_agree(layout, variant):
    base = run({}, layout)
    other = run(variant, layout)
    assert np.abs(base).max() > 0
    assert np.linalg.norm(other - base) <= 1e-5 * np.linalg.norm(base)
