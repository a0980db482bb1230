"""Summarise ncu outputs into the JSON files kept under profiles/.

  launches <csv> <out.json> <command...>   the `--metrics gpu__time_duration.sum,dram__bytes_*`
                                          launch list (per-class time share, DRAM bytes per launch)
  full <ncu-rep> <out.json> <command...>   one `--set full` capture: headline metrics per kernel

Kernel classes follow bench.py: pencil AXIS 0 = x_pass, AXIS 1 = y_pass, zvel = z_vel,
zrho_axis + zp = z_rho (bench counts the pair as one z_rho launch)."""
import csv
import io
import json
import re
import subprocess
import sys


def kclass(name):
    m = re.search(r"pencil_(?:fast|tma)_kernel<(\d)", name)
    if m:
        return "x_pass" if m.group(1) == "0" else "y_pass"
    if "zvel" in name:
        return "z_vel"
    if "zrho" in name or "zp_kernel" in name or "zp2_kernel" in name:
        return "z_rho"
    if "pencil" in name:
        return "y_pass"
    return "other"


def short(name):
    return re.sub(r"\(.*", "", name.replace("void ", "").replace("ustfwi_dev::", ""))


def launches(path, out, cmd):
    text = open(path).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    per = {}
    for r in rows:
        d = per.setdefault(r["ID"], {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] = v / 1000.0 if unit == "nsecond" or unit == "ns" else (v if unit in ("usecond", "us") else v * 1000.0)
        else:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d[r["Metric Name"]] = v * scale
    tot = sum(d.get("us", 0) for d in per.values())
    kern, cls = {}, {}
    for d in per.values():
        k = short(d["name"])
        c = kclass(d["name"])
        e = kern.setdefault(k, {"class": c, "launches": 0, "us": 0.0, "rd": 0.0, "wr": 0.0})
        e["launches"] += 1
        e["us"] += d.get("us", 0)
        e["rd"] += d.get("dram__bytes_read.sum", 0)
        e["wr"] += d.get("dram__bytes_write.sum", 0)
        s = cls.setdefault(c, {"us": 0.0, "bytes": 0.0, "launches": 0})
        s["us"] += d.get("us", 0)
        s["bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        # bench counts one z_rho launch per (zrho_axis, zp) pair
        if c != "z_rho" or "zp_kernel" in d["name"] or "zp2_kernel" in d["name"]:
            s["launches"] += 1
    res = {
        "command": " ".join(cmd),
        "note": "first launches of the bench command (setup + forward simulation of the same step kernels); "
                "cold-cache and serialised under ncu: compare shares, not absolutes",
        "class_time_share": {c: round(s["us"] / tot, 4) for c, s in cls.items()},
        "class_dram_bytes_per_launch_avg": {c: round(s["bytes"] / max(1, s["launches"])) for c, s in cls.items()},
        "kernels": {k: {"class": e["class"], "launches": e["launches"], "us_avg": round(e["us"] / e["launches"], 1),
                        "time_share": round(e["us"] / tot, 4),
                        "dram_read_MB_avg": round(e["rd"] / e["launches"] / 1e6, 1),
                        "dram_write_MB_avg": round(e["wr"] / e["launches"] / 1e6, 1)} for k, e in kern.items()},
    }
    json.dump(res, open(out, "w"), indent=1)


FULL = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"]


def full(path, out, cmd):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = {"command": " ".join(cmd), "units": {"gpu__time_duration.sum": units[hdr.index("gpu__time_duration.sum")],
                                               "dram__bytes": units[hdr.index("dram__bytes_read.sum")]},
           "launches": []}
    for d in data:
        e = {"kernel": short(d[hdr.index("Kernel Name")])}
        for k in FULL:
            if k in hdr:
                try:
                    e[k] = float(d[hdr.index(k)].replace(",", ""))
                except ValueError:
                    e[k] = d[hdr.index(k)]
        res["launches"].append(e)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    (launches if mode == "launches" else full)(src, dst, sys.argv[4:])
