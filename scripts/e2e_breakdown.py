"""Host-side cost of the end-to-end gradient call at config D, by API step."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_00755_b200 import scenario
from paper_2102_00755_b200.engine import GpuEngine

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 40
sc = scenario.config_d(nt=nt)
enc = sc.encoded(0)
obs = np.zeros((len(sc.sensors.positions), sc.grid.nt))
with GpuEngine(sc.grid) as eng:
    for it in range(3):
        t = [time.perf_counter()]
        eng.set_medium(sc.model); t.append(time.perf_counter())
        eng.set_sources(enc); t.append(time.perf_counter())
        eng.set_sensors(sc.sensors); t.append(time.perf_counter())
        loss, grad = eng.gradient_tr(obs, sc.thickness); t.append(time.perf_counter())
        d = np.diff(t)
        print(f"iter {it}: set_medium {d[0]:.3f} set_sources {d[1]:.3f} set_sensors {d[2]:.3f} gradient+io {d[3]:.3f} s")
