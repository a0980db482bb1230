"""Benchmark of the source-encoded time-reversal c0 gradient (BASELINE.json metric).

One "step" = one full source-encoded TR gradient (forward + time-reversal replay +
adjoint, 3nt-3 simulation steps) of the config named by --config on each GPU; at N>1 GPUs
every rank computes a different encoded realization and the step ends with the NCCL
mini-batch mean (weak scaling). Default workload: config D, 442x442x222 interior at
0.5 mm -> 480x480x256 padded, 1024 emitters + 1024 receivers, nt = 3912.

Arms:
  --impl b200       (default) the device engine (libustfwi_b200.so) through its C ABI
  --impl reference  the reference C++ (oracle/_ref: unmodified headers + FFTW-API shim) on
                    the host cores, bounded per-step sample (see cpu_reference_arm)

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config D]
    torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "voxel-updates/s/GPU & s per SE gradient @442x442x222, 1/2/4/8 B200, % HBM roof"
BYTES_PER_VU_MODEL = 128.0   # B_step per voxel-update (fp32, 4-pass design)
BYTES_CORR_MODEL = 16.0      # per voxel per adjoint+TR pair-step


def ncu_traffic(config_name: str, kernel_class: str):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, averaged over the
    launches of the class) from the committed ncu launch list of this config, if any."""
    cands = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_launches_config{config_name}.json")))
    if not cands:
        return None, None
    p = cands[-1]  # latest round
    try:
        d = json.load(open(p))
        return float(d["class_dram_bytes_per_launch_avg"][kernel_class]), os.path.relpath(p, ROOT)
    except Exception:
        return None, None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.25)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------------------
# CPU reference arm / baseline (oracle/_ref only: this path never loads libustfwi_b200.so)
# ----------------------------------------------------------------------------------------

# interior, dx (m), emitters, nt override (the paper's nt at D); the grid itself
# comes from the reference's own make_grid (grid.hpp:91-103) through oracle/_ref
CONFIG_SPECS = {"A": ([44, 44, 44], 1e-3, 1, None), "B": ([108, 108, 108], 1e-3, 64, None),
                "C": ([236, 236, 236], 1e-3, 256, None), "D": ([442, 442, 222], 0.5e-3, 1024, 3912),
                "E0": ([112, 112, 56], 2e-3, 64, 978), "E1": ([222, 222, 112], 1e-3, 256, 1956)}
# resident fp64 bytes per grid point of one ref_time_steps process: engine multipliers and
# spectra + three steppers + accumulator (measured here: 23.7 GB for a D forward with its
# shell trace; SURVEY §8(d) estimates 28 GiB for a TR gradient) -> 64 doubles per point
REF_BYTES_PER_POINT = 64 * 8


def ref_grid(cfg: str, nt=None):
    from oracle import ref
    interior, dx, _, nt_paper = CONFIG_SPECS[cfg]
    g = ref.make_grid(interior, dx, 1800.0, 2 * max(interior) * dx / 1350.0)
    if nt is not None:
        g.nt = int(nt)
    elif nt_paper:
        g.nt = int(nt_paper)
    return g


def grid_points(g):
    n = 1
    for a in range(g.ndim):
        n *= int(g.dims[a])
    return n


def _cpu_worker(args):
    cfg, k_fwd, k_pair = args
    from types import SimpleNamespace
    from oracle import ref
    g = ref_grid(cfg, nt=16)
    shape = tuple(int(g.dims[a]) for a in range(g.ndim))
    m = SimpleNamespace(c0=np.full(shape, 1500.0), rho0=np.full(shape, 1000.0), alpha0=None, y=1.5, gamma=None,
                        c0_min=1350.0, c0_max=1800.0)
    t_f, t_p = ref.time_steps(g, m, k_fwd, k_pair)
    return t_f, t_p, grid_points(g)


def cpu_reference_sample(cfg: str, k_fwd: int, k_pair: int, procs: int):
    """Each process builds the reference SpectralEngine + WaveSteppers + GradientAccumulator
    (oracle/ref_driver.cpp:ref_time_steps, engine.hpp / gradient.hpp unmodified) on the config
    grid and times k_fwd forward steps and k_pair adjoint+replay pair-steps; `procs`
    single-threaded processes run concurrently (independent realizations). A
    gradient is nt forward + (nt - 1) replay + (nt - 2) adjoint steps, so one forward step and
    one pair step advance 3 voxel-update sweeps."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_cpu_worker, [(cfg, k_fwd, k_pair)] * procs)
    wall = time.perf_counter() - t0
    n = res[0][2]
    tf = max(r[0] for r in res)
    tp = max(r[1] for r in res)
    rate_one = n * 3 / (tf + tp)
    return {"rate_per_core": rate_one, "rate_aggregate": rate_one * procs, "t_fwd_step": tf, "t_pair_step": tp,
            "points": n, "wall": wall}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_procs(cfg: str, cap: int = 32):
    """P = min(nproc, RAM / footprint), capped and with a 0.6 safety factor on
    the available memory."""
    n = grid_points(ref_grid(cfg, nt=2))
    foot = n * REF_BYTES_PER_POINT
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except Exception:
        avail = 16 << 30
    return max(1, min(cpu_cores(), cap, int(0.6 * avail // foot)))


def fft_impl():
    """The FFT the oracle links: the in-repo fp64 FFTW-API shim (FFTW3 is not in the image)."""
    try:
        out = subprocess.run(["ldconfig", "-p"], capture_output=True, text=True, timeout=10).stdout
        sys_fftw = "libfftw3.so" in out
    except Exception:
        sys_fftw = False
    return ("in-repo FFTW-API shim (fp64 mixed-radix Stockham, oracle/fftw3_shim)"
            + ("; a system libfftw3 exists on this host but oracle/_ref was built against the shim" if sys_fftw
               else "; no libfftw3 on this host"))


def cpu_baseline_block(cfg: str, vu_grad: float):
    """The reference on the benchmarked grid: 1 forward + 1 pair step per process, P processes
    ('C and D ... extrapolated'), plus the config-B sample beside it."""
    procs = cpu_procs(cfg)
    r = cpu_reference_sample(cfg, 1, 1, procs)
    sample = (f"reference (oracle/_ref: unmodified headers, FFT = {fft_impl()}) on the config {cfg} grid "
              f"{CONFIG_SPECS[cfg][0]} padded to {r['points']} points: 1 forward + 1 adjoint/replay pair step per "
              f"process, {procs} concurrent single-threaded processes (P = min(nproc, 0.6 RAM / footprint, 32)); "
              f"per core {r['rate_per_core']:.3g} vu/s (fwd step {r['t_fwd_step']:.1f} s, pair step "
              f"{r['t_pair_step']:.1f} s); extrapolated s/gradient {vu_grad / r['rate_aggregate']:.4g}")
    out = {"value": r["rate_aggregate"], "unit": "voxel-updates/s", "cores": procs, "kind": "reference",
           "sample": sample, "extrapolated": True, "s_per_gradient_extrapolated": vu_grad / r["rate_aggregate"],
           "wall_s": r["wall"]}
    if cfg != "B":
        pb = cpu_procs("B")
        rb = cpu_reference_sample("B", 2, 2, pb)
        out["b_grid_sample"] = {"value": rb["rate_aggregate"], "cores": pb, "per_core": rb["rate_per_core"],
                                "s_per_gradient_extrapolated": vu_grad / rb["rate_aggregate"],
                                "sample": "config B grid, 2 fwd + 2 pair steps per process"}
    return out


def ref_config_block(cfg: str, n_gpus: int, batch: int):
    g = ref_grid(cfg)
    interior, dx, n_src, _ = CONFIG_SPECS[cfg]
    n = grid_points(g)
    return {"workload": f"config {cfg}: source-encoded TR c0 gradient, grid {tuple(int(g.dims[a]) for a in range(3))} "
                        f"(interior {tuple(interior)}), dx {dx * 1e3:g} mm, nt {g.nt}, {n_src} emitters + "
                        f"{n_src} receivers, shell thickness 8" + (f", mini-batch of {batch}" if batch else ""),
            "grid": [int(g.dims[a]) for a in range(3)], "nt": int(g.nt), "n_emitters": n_src,
            "voxel_updates_per_gradient": n * (3 * int(g.nt) - 3),
            "parallelism": parallelism(n_gpus, batch), "l2_flush": l2_note(n)}


def parallelism(n_gpus, batch):
    if batch:
        return f"fixed mini-batch of {batch} encoded realizations over {n_gpus} GPU(s), NCCL all-gather + ordered mean"
    return f"dp{n_gpus} (one encoded realization per GPU, NCCL all-gather + ordered mean)" if n_gpus > 1 else "1 GPU"


def l2_note(points):
    return ("inputs larger than L2 (each field >= 126 MB)" if points * 4 > 126e6
            else "working set may be L2-resident at this size")


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (make -C oracle)"}))
        return 0
    g = ref_grid(a.config)
    n = grid_points(g)
    vu_grad = n * (3 * int(g.nt) - 3)
    n_grad = a.batch if a.batch else a.gpus
    cb = cpu_baseline_block(a.config, vu_grad)
    value = cb["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "voxel-updates/s",
        "n_gpus": a.gpus, "steps": 1, "warmup": 0,
        "ms_per_step": n_grad * vu_grad / value * 1e3, "higher_is_better": True,
        "scaling": "strong" if a.batch else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": ref_config_block(a.config, a.gpus, a.batch),
        "s_per_gradient_extrapolated": vu_grad / value,
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "voxel-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": f"one sample (requested --steps {a.steps} --warmup {a.warmup}): a full reference gradient at this "
                f"grid takes hours per core, so the per-step rate is measured on the grid and extrapolated",
    }
    print(json.dumps(line))
    return 0


def config_block(sc, n_gpus, batch=0):
    return {"workload": f"config {sc.name}: source-encoded TR c0 gradient, grid {tuple(sc.grid.shape)} "
                        f"(interior {tuple(sc.grid.shape[a] - 2 * sc.grid.pml_size[a] for a in range(3))}), "
                        f"dx {sc.grid.dx[0] * 1e3:g} mm, nt {sc.grid.nt}, {sc.n_src} emitters + "
                        f"{len(sc.sensors.positions)} receivers, shell thickness {sc.thickness}"
                        + (f", mini-batch of {batch}" if batch else ""),
            "grid": list(sc.grid.shape), "nt": sc.grid.nt, "n_emitters": sc.n_src,
            "n_receivers": len(sc.sensors.positions), "voxel_updates_per_gradient": sc.voxel_updates_per_gradient,
            "parallelism": parallelism(n_gpus, batch), "l2_flush": l2_note(sc.grid.points)}


# ----------------------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------------------

def b200_arm(a):
    import torch
    import torch.distributed as dist

    from paper_2102_00755_b200 import engine as E
    from paper_2102_00755_b200 import scenario

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    dev = local
    sc = scenario.CONFIGS[a.config]() if a.nt is None else scenario.CONFIGS[a.config](nt=a.nt)
    g = sc.grid
    eng = E.GpuEngine(g, device=dev)
    if world > 1:
        uid = [E.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        eng.comm_init(uid[0], world, rank)

    from paper_2102_00755_b200.minibatch import NcclReducer, run_minibatch, shard, slots_per_rank
    # realizations of this rank: weak scaling = realization `rank` (one encoded gradient per GPU
    # per step); --batch B = the fixed mini-batch r = rank, rank + W, ... < B (BASELINE config 3)
    mine = shard(a.batch, world, rank) if a.batch else [rank]
    batch = a.batch if a.batch else world
    slots = slots_per_rank(batch, world)
    eng.set_sensors(sc.sensors)
    # synthetic observed data: forward of each encoded source on the true phantom (setup)
    eng.set_medium(sc.truth)
    encs, obs = {}, {}
    for r in mine:
        encs[r] = sc.encoded(r)
        eng.set_sources(encs[r])
        obs[r], _ = eng.forward(0)
    eng.set_medium(sc.model)
    if len(mine) == 1:
        eng.set_sources(encs[mine[0]])
        eng.upload_observed(obs[mine[0]])
    eng.batch_reserve(slots)
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=dev)

    def one_step():
        # this rank's gradients into its slots, then the deterministic mean over all ranks
        for r in mine:
            if len(mine) > 1:
                eng.set_sources(encs[r])
                eng.upload_observed(obs[r])
            eng.run_gradient_slot(sc.thickness, r // world)
        if world > 1 or batch > 1:
            eng.batch_mean(batch)

    for _ in range(a.warmup):
        one_step()
    eng.synchronize()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    l0 = eng.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        ev0.record(stream)
        for _ in range(a.steps):
            one_step()
        ev1.record(stream)
        ev1.synchronize()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
    launches = eng.launch_count() - l0
    # per-launch-class CUDA-event timing: one extra gradient with profiling on (the engine
    # then serialises adjoint and replay on one stream so each launch is timed alone)
    eng.set_profiling(True)
    eng.run_gradient_slot(sc.thickness, 0)
    stats = eng.kernel_stats()
    prof_ms = sum(v[0] for v in stats.values())
    eng.set_profiling(False)
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    s_per_step = ms / 1e3 / a.steps
    vu = sc.voxel_updates_per_gradient
    n_grad = batch            # gradients of the whole job per step
    value = n_grad * vu / s_per_step

    # end to end through the public API: host medium + encoded sources + observed data in,
    # gradient out (weak: gradient_time_reversal per rank; --batch: the mini-batch driver)
    e2e = None
    if a.e2e_steps > 0:
        e_times = []
        for _ in range(a.e2e_steps):
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            if a.batch or world > 1:
                eng.set_medium(sc.model)
                run_minibatch(eng, lambda r: encs[r], lambda r: obs[r], sc.thickness, batch, world, rank,
                              NcclReducer())
                loss, grad = eng.download_gradient()
            else:
                r0 = mine[0]
                res = E.gradient_time_reversal(sc.model, encs[r0], sc.sensors, obs[r0], g, sc.thickness, engine=eng)
            dt = time.perf_counter() - t0
            tt = torch.tensor([dt], dtype=torch.float64)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_times.append(float(tt.item()))
        te = float(np.median(e_times))
        h2d = sum(obs[r].nbytes + encs[r].weights.nbytes + encs[r].delays.nbytes + len(encs[r].positions) * 8 +
                  sum(np.asarray(x).nbytes for x in encs[r].signals) for r in mine) + \
            3 * g.points * 8  # observed + sources per realization, medium (c0, rho0, gamma)
        d2h = g.points * 8 + 8
        e2e = {"value": n_grad * vu / te, "unit": "voxel-updates/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "s_per_gradient": te / max(1, len(mine))}

    if rank != 0:
        if world > 1:
            dist.barrier()
        return 0

    hbm, peak_kind = peaks()
    # dominant kernel roofline (CUDA events per launch on the engine stream)
    dom = max(stats, key=lambda k: stats[k][0])
    d_ms, d_n, d_b = stats[dom]
    achieved = (d_b / d_n) / (d_ms / d_n / 1e3) / 1e9 if d_n else 0.0
    traffic, traffic_src = ncu_traffic(sc.name, dom)
    kernels = {k: {"ms_total": v[0], "launches": v[1], "ms_per_launch": v[0] / v[1] if v[1] else 0.0,
                   "GB_per_launch": v[2] / v[1] / 1e9 if v[1] else 0.0,
                   "achieved_GBps": (v[2] / v[0] * 1e3 / 1e9) if v[0] else 0.0,
                   "share_of_profiled_gradient": v[0] / prof_ms if prof_ms else 0.0} for k, v in stats.items() if v[1]}
    n = g.points
    b_model = n * (BYTES_PER_VU_MODEL * (3 * g.nt - 3) + BYTES_CORR_MODEL * (g.nt - 2))
    path_gbps = b_model * slots / s_per_step / 1e9   # gradients per GPU per step = slots
    # the engine's own algorithmic bytes per voxel-update (sum over launch classes) and the
    # ncu-measured DRAM bytes of the same launches where a launch list is committed
    alg_bytes = sum(v[2] for v in stats.values())
    meas_bytes, meas_src = 0.0, None
    for k, v in stats.items():
        t, src = ncu_traffic(sc.name, k)
        if t is None:  # classes without a launch-list entry (small auxiliary kernels): model bytes
            meas_bytes += v[2]
            continue
        meas_bytes += t * v[1]
        meas_src = src
    if meas_src is None:
        meas_bytes = None
    line = {
        "metric": METRIC, "value": value, "unit": "voxel-updates/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
        "scaling": "strong" if a.batch else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (breast phantom, golden-spiral bowl, "
                                                     "Rademacher-encoded emitters, observed = forward on truth)",
        "config": config_block(sc, world, a.batch),
        "voxel_updates_per_s_per_gpu": value / world,
        "s_per_gradient": s_per_step * world / n_grad,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "peak_kind": peak_kind,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": d_b / d_n if d_n else 0.0},
        "path_roofline": {"model_bytes_per_gradient": b_model, "model_B_per_voxel_update": b_model / vu,
                          "achieved_GBps": path_gbps, "frac_of_measured": path_gbps / hbm,
                          "frac_of_8TBps": path_gbps / 8000.0,
                          "engine_algorithmic_B_per_voxel_update": alg_bytes / vu,
                          "ncu_dram_B_per_voxel_update": (meas_bytes / vu) if meas_bytes else None,
                          "ncu_dram_note": (f"{meas_src}: per-class DRAM bytes per launch of the first launches "
                                            "(forward steps; the replay's correlation traffic is counted at the "
                                            "forward rate) x launches per gradient") if meas_bytes else None},
        "kernels": kernels,
        "kernel_timing": "CUDA events around every launch of one extra gradient after the timed region "
                         "(adjoint and replay serialised on one stream for that gradient)",
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if world == 1 and a.cpu_baseline:
        try:
            from oracle import ref
            if ref.available():
                line["cpu_baseline"] = cpu_baseline_block(a.config, vu)
        except Exception as e:  # baseline is reported, never blocks the bench line
            line["cpu_baseline"] = {"value": None, "unit": "voxel-updates/s", "cores": 0, "kind": "reference",
                                    "sample": f"failed: {e}"}
    print(json.dumps(line))
    eng.close()
    if world > 1:
        dist.barrier()
    return 0


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="D", choices=["A", "B", "C", "D", "E0", "E1"])
    p.add_argument("--e2e-steps", type=int, default=1)
    p.add_argument("--cpu-baseline", type=int, default=1)
    p.add_argument("--batch", type=int, default=0,
                   help="fixed mini-batch of B encoded realizations sharded over the GPUs (BASELINE config 3); "
                        "0 = one realization per GPU (weak scaling)")
    p.add_argument("--nt", type=int, default=None, help="override nt (development only; not a valid bench number)")
    a = p.parse_args()
    if a.impl == "reference":
        return reference_arm(a)
    return b200_arm(a)


if __name__ == "__main__":
    sys.exit(main())
