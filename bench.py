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
# CPU reference arm / baseline
# ----------------------------------------------------------------------------------------

def _cpu_worker(args):
    cfg, k = args
    from oracle import ref
    from paper_2102_00755_b200 import scenario
    sc = scenario.CONFIGS[cfg](nt=16)
    t_f, t_p = ref.time_steps(sc.grid, sc.model, k, k)
    return t_f, t_p, sc.grid.points


def cpu_reference_sample(cfg: str, k: int, procs: int):
    """Each process builds the reference SpectralEngine + WaveSteppers (engine.hpp) for the
    config grid and times k forward steps and k adjoint+replay pair-steps with the
    GradientAccumulator (oracle/ref_driver.cpp:ref_time_steps). Returns aggregate
    voxel-updates/s over `procs` concurrent single-threaded processes."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_cpu_worker, [(cfg, k)] * procs)
    wall = time.perf_counter() - t0
    per_proc = [(n * 1 / tf + n * 2 / tp) / 2 for tf, tp, n in res]   # mean of fwd and pair rates
    n = res[0][2]
    # voxel-updates of one gradient per step: forward nt, pair (nt-2)*2, + 1 look-ahead
    tf = max(r[0] for r in res)
    tp = max(r[1] for r in res)
    rate_one = n * 3 / (tf + tp)   # one fwd step + one pair step = 3 voxel-update sweeps
    return {"rate_per_core": rate_one, "rate_aggregate": rate_one * procs, "t_fwd_step": tf, "t_pair_step": tp,
            "points": n, "wall": wall, "per_proc": per_proc}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_procs(cfg: str):
    # footprint per reference process ~ (7 state + 6 scratch + 3 rho~ + 2 medium) fp64 fields +
    # 15 complex half-spectrum multiplier arrays (engine.hpp:46-78); config B ~ 1 GiB
    from paper_2102_00755_b200 import scenario
    n = scenario.CONFIGS[cfg](nt=2).grid.points
    foot = n * 8 * (18 + 15 + 4)
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except Exception:
        avail = 16 << 30
    return max(1, min(cpu_cores(), int(0.7 * avail // foot)))


def reference_arm(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import ref
    from paper_2102_00755_b200 import scenario
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (make -C oracle)"}))
        return 0
    sample_cfg = a.cpu_sample_config
    procs = cpu_procs(sample_cfg)
    sc = scenario.CONFIGS[a.config]()
    vu_grad = sc.voxel_updates_per_gradient
    for _ in range(a.warmup):
        cpu_reference_sample(sample_cfg, 1, procs)
    rates, times = [], []
    for _ in range(a.steps):
        r = cpu_reference_sample(sample_cfg, a.cpu_sample_steps, procs)
        rates.append(r["rate_aggregate"])
        times.append(vu_grad / r["rate_aggregate"])
    value = float(np.median(rates))
    sample = (f"config {sample_cfg} grid {tuple(scenario.CONFIGS[sample_cfg](nt=2).grid.shape)}: "
              f"{a.cpu_sample_steps} forward + {a.cpu_sample_steps} adjoint/replay pair steps per process, "
              f"{procs} concurrent 1-thread processes; FFT = in-repo FFTW-API shim (fp64 Stockham), not FFTW; "
              f"per-voxel-update rate extrapolated to the {a.config} gradient")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "voxel-updates/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": float(np.median(times)) * 1e3 / max(1, a.gpus), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(sc, a.gpus),
        "s_per_gradient_extrapolated": float(np.median(times)),
        "cpu_baseline": {"value": value, "unit": "voxel-updates/s", "cores": procs, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "voxel-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def config_block(sc, n_gpus):
    return {"workload": f"config {sc.name}: source-encoded TR c0 gradient, grid {tuple(sc.grid.shape)} "
                        f"(interior {tuple(sc.grid.shape[a] - 2 * sc.grid.pml_size[a] for a in range(3))}), "
                        f"dx {sc.grid.dx[0] * 1e3:g} mm, nt {sc.grid.nt}, {sc.n_src} emitters + "
                        f"{len(sc.sensors.positions)} receivers, shell thickness {sc.thickness}",
            "grid": list(sc.grid.shape), "nt": sc.grid.nt, "n_emitters": sc.n_src,
            "n_receivers": len(sc.sensors.positions), "voxel_updates_per_gradient": sc.voxel_updates_per_gradient,
            "parallelism": f"dp{n_gpus} (one encoded realization per GPU, NCCL mean)" if n_gpus > 1 else "1 GPU",
            "l2_flush": "inputs larger than L2 (each field >= 126 MB at config D)" if sc.grid.points * 4 > 126e6
            else "working set may be L2-resident at this size"}


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

    # realization of this rank (weak scaling: one encoded gradient per GPU per step)
    enc = sc.encoded(rank)
    # synthetic observed data: forward of the encoded source on the true phantom (setup)
    eng.set_medium(sc.truth)
    eng.set_sources(enc)
    eng.set_sensors(sc.sensors)
    observed, _ = eng.forward(0)
    eng.set_medium(sc.model)
    eng.upload_observed(observed)
    stream = torch.cuda.ExternalStream(eng.stream_ptr(), device=dev)

    def one_step(accumulate=False):
        eng.run_gradient(sc.thickness, accumulate=accumulate)
        if world > 1:
            eng.allreduce_mean(world)

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
    eng.run_gradient(sc.thickness)
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
    value = world * vu / s_per_step

    # end to end through the public API: host observed + encoded sources in, gradient out
    e2e = None
    if a.e2e_steps > 0:
        obs_host = np.ascontiguousarray(observed)
        e_times = []
        for _ in range(a.e2e_steps):
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            res = E.gradient_time_reversal(sc.model, enc, sc.sensors, obs_host, g, sc.thickness, engine=eng)
            if world > 1:
                eng.allreduce_mean(world)
            dt = time.perf_counter() - t0
            tt = torch.tensor([dt], dtype=torch.float64)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_times.append(float(tt.item()))
        te = float(np.median(e_times))
        h2d = obs_host.nbytes + enc.weights.nbytes + enc.delays.nbytes + len(enc.positions) * 8 + \
            sum(np.asarray(s).nbytes for s in enc.signals) + 3 * g.points * 8  # observed, sources, medium (c0, rho0, gamma)
        d2h = g.points * 8 + 8
        e2e = {"value": world * vu / te, "unit": "voxel-updates/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "s_per_gradient": te}

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
    path_gbps = b_model / s_per_step / 1e9
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
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (breast phantom, golden-spiral bowl, "
                                                     "Rademacher-encoded emitters, observed = forward on truth)",
        "config": config_block(sc, world),
        "voxel_updates_per_s_per_gpu": value / world,
        "s_per_gradient": s_per_step,
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
                procs = cpu_procs(a.cpu_sample_config)
                r = cpu_reference_sample(a.cpu_sample_config, a.cpu_sample_steps, procs)
                line["cpu_baseline"] = {
                    "value": r["rate_aggregate"], "unit": "voxel-updates/s", "cores": procs, "kind": "reference",
                    "sample": f"reference (oracle/_ref, FFTW-API shim) on config {a.cpu_sample_config} grid: "
                              f"{a.cpu_sample_steps} fwd + {a.cpu_sample_steps} pair steps x {procs} processes; "
                              f"per core {r['rate_per_core']:.3g} vu/s; extrapolated s/gradient at "
                              f"{sc.name}: {vu / r['rate_aggregate']:.4g}"}
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
    p.add_argument("--config", default="D", choices=["A", "B", "C", "D"])
    p.add_argument("--e2e-steps", type=int, default=1)
    p.add_argument("--cpu-baseline", type=int, default=1)
    p.add_argument("--cpu-sample-config", default="B")
    p.add_argument("--cpu-sample-steps", type=int, default=2)
    p.add_argument("--nt", type=int, default=None, help="override nt (development only; not a valid bench number)")
    a = p.parse_args()
    if a.impl == "reference":
        return reference_arm(a)
    return b200_arm(a)


if __name__ == "__main__":
    sys.exit(main())
