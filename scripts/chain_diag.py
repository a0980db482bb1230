"""Diagnostics of the fused y-x-y chain kernel on the config-D grid: time per gradient (nt 40)
and the kernel's wait statistics (USTFWI_CHAIN_STATS=1).

    USTFWI_CHAIN_STATS=1 python scripts/chain_diag.py
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2102_00755_b200 import capi
from paper_2102_00755_b200.engine import GpuEngine, Medium, SensorArray, SourceSet

g = capi.make_grid([442, 442, 222], 0.5e-3, 1800.0, 1e-3)
g.nt = 40
sh = g.shape
c = [s // 2 for s in sh]
m = Medium(c0=np.full(sh, 1500.0), rho0=np.full(sh, 1000.0), gamma=capi.ball_mask(sh, c, 60.0))
pulse = capi.synth_source_pulse(g, 0.8, 1350.0)
f = lambda x, y, z: (x * sh[1] + y) * sh[2] + z
with GpuEngine(g) as eng:
    eng.set_medium(m)
    eng.set_sources(SourceSet([f(sh[0] // 8, c[1], c[2])], [pulse]))
    eng.set_sensors(SensorArray([f(7 * sh[0] // 8, c[1], c[2])]))
    obs = np.zeros((1, g.nt))
    eng.upload_observed(obs)
    eng.run_gradient(4)
    eng.synchronize()
    out = (C.c_uint64 * 5)()
    capi.lib().ustfwi_gpu_chain_stats(out)
    t0 = time.time()
    eng.run_gradient(4)
    eng.synchronize()
    t = time.time() - t0
    capi.lib().ustfwi_gpu_chain_stats(out)
    n, units, deferred, wait, mbar = list(out)
    launches = 2 * (3 * g.nt - 3)
    print(f"{os.environ.get('TAG', '')}: {t:.4f} s/grad ({t / (3 * g.nt - 3) * 1e3:.3f} ms/step); per chain launch: "
          f"units {units / max(launches, 1):.0f}, deferred {deferred / max(launches, 1):.1f}, dep-wait "
          f"{wait / max(launches, 1) / max(n, 1) / 1.9e3:.1f} us/CTA, tile-wait {mbar / max(launches, 1) / max(n, 1) / 1.9e3:.1f} us/CTA")
