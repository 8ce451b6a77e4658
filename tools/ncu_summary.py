#!/usr/bin/env python
"""Summarise ncu captures (.ncu-rep) and launch lists into profiles/.

    python tools/ncu_summary.py --rep gpurun_out/stream_full.ncu-rep --name r1_stream \
        --algo-bytes 6442450944 [--traffic-n 268435456]
    python tools/ncu_summary.py --launches gpurun_out/launches.csv --name r1_launches

Reads the raw page (`ncu -i ... --page raw --csv`) and writes
profiles/<name>.json (selected metrics + warp-stall breakdown) and, for launch
lists, profiles/<name>.csv (kernel, grid, block, duration) with each kernel's
share of the total.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum.per_second", "dram__bytes_write.sum.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__maximum_warps_per_active_cycle_pct",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_warps", "launch__occupancy_limit_blocks",
    "launch__occupancy_limit_barriers", "gpc__cycles_elapsed.max.per_second",
    "lts__t_bytes.sum", "smsp__pcsamp_sample_count",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    kernels = []
    for v in rows[2:]:
        kernels.append({h[i]: (v[i], units[i]) for i in range(len(h))})
    return kernels


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def summarise_rep(rep, algo_bytes):
    res = []
    for k in raw(rep):
        m = {key: {"value": num(k[key][0]), "unit": k[key][1]} for key in KEYS if key in k}
        stalls = {}
        for name, (v, _) in k.items():
            if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith(
                    "_not_issued"):
                x = num(v)
                if x:
                    stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
        total = sum(stalls.values())
        d = {"kernel": k.get("Kernel Name", ("?", ""))[0], "metrics": m,
             "stall_samples": stalls,
             "barrier_stall_fraction": round(stalls.get("barrier", 0) / total, 4) if total else None}
        units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

        def nbytes(key):
            v, u = k.get(key, ("0", "byte"))
            return (num(v) or 0) * units.get(u, 1)
        d["dram_bytes_per_launch"] = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
        if algo_bytes:
            d["algorithmic_bytes_per_launch"] = algo_bytes
            d["traffic_over_algorithmic"] = round(d["dram_bytes_per_launch"] / algo_bytes, 4)
            t = num(k.get("gpu__time_duration.sum", ("0", ""))[0])
            tu = k.get("gpu__time_duration.sum", ("", ""))[1]
            sec = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(tu, 1e-9)
            d["achieved_GBps_under_ncu"] = round(algo_bytes / sec / 1e9, 1)
        res.append(d)
    return res


def summarise_launches(path):
    lines = open(path).read().splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[i:]))
    total = sum(float(r["Metric Value"]) for r in rows)
    out = []
    for r in rows:
        ns = float(r["Metric Value"])
        out.append({"kernel": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"],
                    "ns": ns, "share": round(ns / total, 4)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--group", action="store_true",
                    help="with --launches: one row per kernel (launches, total, mean, share)")
    ap.add_argument("--name", required=True)
    ap.add_argument("--algo-bytes", type=float, default=0)
    ap.add_argument("--traffic-n", type=int, default=0,
                    help="also write profiles/traffic.json for bench.py (elements per launch)")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.rep:
        s = summarise_rep(a.rep, a.algo_bytes)
        with open(os.path.join(ROOT, "profiles", a.name + ".json"), "w") as f:
            json.dump(s, f, indent=1)
        if a.traffic_n:
            with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
                sys.path.insert(0, ROOT)
                from paper_1711_10413_b200.build import sources_sha256
                json.dump({"n": a.traffic_n, "dram_bytes_per_launch": s[0]["dram_bytes_per_launch"],
                           "source": a.name, "sources_sha256": sources_sha256()}, f, indent=1)
        json.dump(s, sys.stdout, indent=1)
    if a.launches:
        s = summarise_launches(a.launches)
        if a.group:
            g = {}
            for r in s:
                e = g.setdefault(r["kernel"], [0, 0.0])
                e[0] += 1
                e[1] += r["ns"]
            total = sum(v[1] for v in g.values()) or 1.0
            with open(os.path.join(ROOT, "profiles", a.name + ".csv"), "w") as f:
                w = csv.writer(f)
                w.writerow(["kernel", "launches", "total_ns", "mean_ns", "share"])
                for k, (n, t) in sorted(g.items(), key=lambda kv: -kv[1][1]):
                    w.writerow([k, n, round(t), round(t / n), round(t / total, 4)])
                    print(f"{t / total:7.4f} {n:5d} {t / n:>12.0f} {k[:90]}")
            return
        with open(os.path.join(ROOT, "profiles", a.name + ".csv"), "w") as f:
            w = csv.writer(f)
            w.writerow(["kernel", "grid", "block", "ns", "share"])
            for r in s:
                w.writerow([r["kernel"], r["grid"], r["block"], r["ns"], r["share"]])
        for r in s:
            print(f'{r["share"]:7.4f} {r["ns"]:>12.0f} {r["kernel"][:90]}')


if __name__ == "__main__":
    main()
