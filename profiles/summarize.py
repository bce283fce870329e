#!/usr/bin/env python
"""Summarise ncu captures of bench.py into profiles/ (run here, on the CPU box).

    python profiles/summarize.py --rep gpurun_out/prof_r01.ncu-rep \
        --launches gpurun_out/launches_r01.csv --tag r01

Writes profiles/<tag>_ncu_full.json (per profiled launch: duration, DRAM bytes, throughput,
occupancy, pipe utilisation, stall mix), profiles/<tag>_launches.json (per-kernel share of
the launch list) and profiles/traffic.json (DRAM bytes per launch of the profiled launches,
keyed by the C-ABI launcher, read by bench.py for roofline.traffic).
"""

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
C_API = {"stencil_kernel": "emhd_jv_normalized", "multidot_kernel": "emhd_multidot",
         "update_kernel": "emhd_update", "combine_kernel": "emhd_combine",
         "phi_small_kernel": "emhd_phi_small", "norms_kernel": "emhd_norms",
         "lincomb_kernel": "emhd_lincomb", "arnoldi_finish_kernel": "emhd_arnoldi_finish",
         "div_scalar_kernel": "emhd_div_scalar"}
METRICS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_of_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "stall_long_scoreboard": "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "stall_barrier": "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "stall_short_scoreboard": "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "stall_wait": "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
}
UNITS = {"ns": 1e-3, "us": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1.0, "msecond": 1e3,
         "nsecond": 1e-3}


def base_name(full):
    n = full.split("(")[0].replace("void ", "").strip()
    n = n.split("<")[0]
    return n.split("::")[-1]


def full_capture(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                d[k] = v * UNITS.get(units[i], 1.0) if units[i] in UNITS else v
        res.append(d)
    return res


def launch_list(path):
    per = defaultdict(lambda: {"launches": 0, "us": 0.0})
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ik, im, iv, iu = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", "")) * UNITS.get(r[iu], 1.0)
        k = base_name(r[ik])
        per[k]["launches"] += 1
        per[k]["us"] += v
    tot = sum(x["us"] for x in per.values())
    return {k: dict(v, share=v["us"] / tot) for k, v in sorted(per.items(), key=lambda kv: -kv[1]["us"])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r01")
    a = ap.parse_args()
    if a.rep:
        caps = full_capture(a.rep)
        with open(os.path.join(HERE, f"{a.tag}_ncu_full.json"), "w") as fh:
            json.dump(caps, fh, indent=1)
        traffic = {}
        for c in caps:
            api = C_API.get(base_name(c["kernel"]))
            if base_name(c["kernel"]) == "update_kernel" and "<1" in c["kernel"]:
                api = "emhd_update_finish"      # mode 1 (+ fused column bookkeeping)
            # a kernel profiled more than once (a real launch and a device-gated no-op of the
            # second pass): keep the launch that moved the most bytes
            if api and "dram_read_bytes" in c:
                traffic[api] = max(traffic.get(api, 0.0), c["dram_read_bytes"] + c["dram_write_bytes"])
        with open(os.path.join(HERE, "traffic.json"), "w") as fh:
            json.dump(traffic, fh, indent=1)
        for c in caps:
            print(f"{c['kernel'][:40]:40s} {c.get('duration_us', 0):8.1f} us  "
                  f"DRAM {(c.get('dram_read_bytes', 0) + c.get('dram_write_bytes', 0)) / 1e6:8.1f} MB  "
                  f"{c.get('dram_pct_of_peak', 0):5.1f}% peak  warps {c.get('warps_active_pct', 0):5.1f}%  "
                  f"fp64 {c.get('fp64_pipe_pct', 0):5.1f}%")
    if a.launches:
        ll = launch_list(a.launches)
        with open(os.path.join(HERE, f"{a.tag}_launches.json"), "w") as fh:
            json.dump(ll, fh, indent=1)
        for k, v in ll.items():
            print(f"{k:28s} {v['launches']:6d} launches {v['us']:10.1f} us  share {v['share']:.3f}")


if __name__ == "__main__":
    main()
