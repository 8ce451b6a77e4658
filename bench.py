#!/usr/bin/env python
"""Benchmark of the implicit data-sharing hot path on B200.

One *step* = one generic-mode target region launch of BASELINE config 4:
``teams`` CTAs (OpenMP teams) of W workers + the reserved master warp; each
team runs kernel_init, pushes its kernel depot on the master's data-sharing
stack, shares 8 scalars through prepare_parallel / the shared-memory args
window, releases its workers with a named barrier, the workers read the
shared-variable list (warp-shuffle broadcast) and stream
``y[i] = fma(c1, x[i], y[i]) + (c2+...+c8)`` over 2^28 fp64 elements on the
cyclic schedule, retire, join, deinit.

Metric: body HBM GB/s (24 algorithmic bytes per element) -- BASELINE.json
"parallel regions/sec + body HBM GB/s vs 8 TB/s; smem bytes/CTA & occupancy".
Config-1 latency (ns per parallel region) and the team region's smem/CTA and
occupancy are reported alongside.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun, one process per GPU; BASELINE config 5): strong scaling
by default -- 2^28 elements in total, rank r owns [r*N/G, (r+1)*N/G) and its
own teams, no data-path collective (``--scaling weak``: 2^28 per GPU).  The
K steps are timed twice: CUDA events on each rank's stream (max over ranks =
``value``) and a barrier-bracketed wall-clock window (``wall_window``).
Correctness gate at every N: after timing the inputs are regenerated, one
region pass runs, the per-rank checksums of y are all-reduced and compared
with the whole range's expected checksum (tests/golden/config5_checksums.json,
from the C oracle); ``checksum_ok`` is in the line and a mismatch exits 1.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_ELEM = 24  # read x (8) + read y (8) + write y (8)
SEED_X, SEED_Y = 0x5EED01AB, 0x5EED01AC
COEF = [k / 8 for k in range(1, 9)]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--elements", type=int, default=1 << 28, help="elements per GPU (weak) or in total (strong)")
    ap.add_argument("--teams", type=int, default=0, help="0: 148 x teams-per-SM")
    ap.add_argument("--workers", type=int, default=0, help="W (0: tuned default)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong (BASELINE config 5): --elements in total, split over the "
                         "GPUs; weak: --elements per GPU")
    ap.add_argument("--only-stream", action="store_true",
                    help="only the headline stream region (skip configs 1-3 and overheads)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ptxas_regs(kernel_substr):
    log = os.path.join(ROOT, "paper_1711_10413_b200", "_build", "ptxas.log")
    try:
        lines = open(log).read().splitlines()
    except OSError:
        return None
    for i, l in enumerate(lines):
        if "Compiling entry function" in l and kernel_substr in l:
            for m in lines[i + 1:i + 4]:
                if "Used" in m and "registers" in m:
                    return int(m.split("Used")[1].split("registers")[0])
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes ~0.1-0.5 s to start: wait for its first sample
            # so the samples cover the timed region, not the time after it
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def device_ms(stream, launch, reps=3):
    """Device time of what `launch()` enqueues on `stream` (median of
    `reps`, after one untimed run): the GPU spins (~100 us) while the host
    prepares each launch, so the host's argument marshalling never lands
    between the two events."""
    import torch
    times = []
    for i in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(200_000)
            e0.record(stream)
            launch()
            e1.record(stream)
        e1.synchronize()
        if i:
            times.append(e0.elapsed_time(e1))
    return statistics.median(times)


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(n_sample, threads):
    """The C oracle port (fp64, OpenMP over the host's cores) on a bounded sample."""
    import numpy as np
    from oracle import oracle as O
    L = O.lib()
    x = np.empty(n_sample)
    y = np.empty(n_sample)
    L.orc_fill(1, O.ptr(x), n_sample, SEED_X, 0)
    L.orc_fill(1, O.ptr(y), n_sample, SEED_Y, 0)
    coef = np.array(COEF)
    L.orc_stream(1, n_sample, O.ptr(x), O.ptr(y), O.ptr(coef), threads)  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        L.orc_stream(1, n_sample, O.ptr(x), O.ptr(y), O.ptr(coef), threads)
        reps += 1
        el = time.perf_counter() - t0
        if el > 10.0 or reps >= 60:  # ~10 s of CPU work
            break
    gbs = BYTES_PER_ELEM * n_sample * reps / el / 1e9
    # the regions/s half: the config-1 body (1 team x 32 workers, 4 shared
    # scalars, 10^4 regions) as the port runs it -- sequential, one thread
    # (orc_regions: the semantics only, no protocol to execute)
    R = 10_000
    a = np.zeros(32)
    t0 = time.perf_counter()
    L.orc_regions(1, 1, 32, R, O.ptr(a))
    ns_region = (time.perf_counter() - t0) / R * 1e9
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{n_sample} fp64 elements x {reps} passes of the config-4 body "
                      f"(oracle/ompds_oracle.c orc_stream, OpenMP {threads} threads)",
            "regions": {"ns_per_region": round(ns_region, 1), "cores": 1,
                        "sample": f"config 1 body, 1 team x 32 workers, {R} regions "
                                  "(orc_regions, sequential; no runtime protocol)"}}


def run_reference(args):
    """--impl reference: the reference's own CPU path (oracle/_ref, the
    unmodified omplab simulator running the integer analog of the region)."""
    import ctypes as C
    import numpy as np
    rank, world, local = dist_env()
    if rank != 0:
        return
    shim = os.path.join(ROOT, "oracle", "_ref", "libomplab_ref.so")
    threads = os.cpu_count() or 1
    base = {"metric": "stream region body GB/s (config 4, 24 B/elem)", "impl": "reference",
            "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "int32 (reference language is integer-only)", "data": "synthetic",
            "config": {"workload": "config4_stream_region", "teams": 4, "workers": 96,
                       "elements_per_step": None, "parallelism": f"{threads} host threads"}}
    if not os.path.exists(shim):
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libomplab_ref.so not built (needs /root/reference)"}))
        return
    L = C.CDLL(shim)
    L.omplab_ref_stream.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                    C.c_void_p, C.c_int]
    chunk = 4096
    nchunks = 2 * threads
    n = chunk * nchunks
    x = np.array([(int(v) % 201) - 100 for v in range(n)], dtype=np.int64)
    y = np.zeros(n, dtype=np.int64)
    xp, yp = C.c_void_p(x.ctypes.data), C.c_void_p(y.ctypes.data)
    for _ in range(max(args.warmup, 0)):
        assert L.omplab_ref_stream(0, chunk, nchunks, 4, 96, xp, yp, threads) == 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        assert L.omplab_ref_stream(0, chunk, nchunks, 4, 96, xp, yp, threads) == 0
    el = time.perf_counter() - t0
    gbs = BYTES_PER_ELEM * n * args.steps / el / 1e9
    base["value"] = round(gbs, 6)
    base["ms_per_step"] = round(el / args.steps * 1e3, 3)
    base["config"]["elements_per_step"] = n
    # same metric as our arm: config-4 elements processed per second x 24 B
    # (the reference's i32 elements would move 12 B; counting 24 favours it)
    base["config"]["bytes_counted_per_element"] = BYTES_PER_ELEM
    base["cpu_baseline"] = {"value": base["value"], "unit": "GB/s", "cores": threads,
                            "kind": "reference", "cpu_model": cpu_model(),
                            "sample": f"{nchunks} chunks x {chunk} int elements per step, "
                                      "omplab simulate() (Simulator.cpp) per chunk"}
    base["e2e"] = {"value": base["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}
    # the other half of the metric, parallel regions/s: the config-1 analog
    # (1 team x 32 workers, 4 shared int scalars) through the same simulator
    L.omplab_ref_regions.argtypes = [C.c_int, C.c_int, C.c_int]
    L.omplab_ref_regions.restype = C.c_double
    R = 200
    sec = L.omplab_ref_regions(0, 32, R)
    if sec > 0:
        base["regions"] = {"ns_per_region": round(sec * 1e9, 1),
                           "regions_per_s": round(1 / sec, 1),
                           "workload": f"config-1 analog: 1 team x 32 workers, 4 shared int "
                                       f"scalars, {R} regions in a sequential loop, omplab "
                                       "simulate() on one host thread"}
    print(json.dumps(base))


def expected_checksum(n_total, rank):
    """The checksum y must have after one region pass over [0, n_total):
    the committed fixture (tests/golden/config5_checksums.json, generated by
    the C oracle) when it lists n_total, else the oracle checker computed on
    rank 0 (orc_stream_checksum: regenerates the inputs, no buffers)."""
    fx = os.path.join(ROOT, "tests", "golden", "config5_checksums.json")
    try:
        d = json.load(open(fx))
        if d["seed_x"] == SEED_X and d["seed_y"] == SEED_Y and d["coef"] == COEF and \
                str(n_total) in d["checksums"]:
            return int(d["checksums"][str(n_total)], 16), "tests/golden/config5_checksums.json"
    except (OSError, ValueError, KeyError):
        pass
    if rank != 0:
        return None, "oracle (rank 0)"
    import numpy as np
    from oracle import oracle as O  # the checker only
    cf = np.array(COEF)
    v = O.lib().orc_stream_checksum(1, 0, n_total, SEED_X, SEED_Y, O.ptr(cf), 0)
    return int(v), "oracle/ompds_oracle.c orc_stream_checksum (checker)"


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_1711_10413_b200 import _lib as PL  # noqa: F401  (loads the .so: fails loudly)
    from paper_1711_10413_b200 import regions as RG

    rank, world, local = dist_env()
    # OMPDS_BENCH_SHARE_GPU=1 + OMPDS_BENCH_BACKEND=gloo: exercise the N>1 code
    # path with every rank on cuda:0 (a 1-GPU box); never used for numbers.
    if os.environ.get("OMPDS_BENCH_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("OMPDS_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_1711_10413_b200 import sharding
    # strong scaling (default, BASELINE config 5): 2^28 elements in total,
    # rank r owns [r*N/G, (r+1)*N/G); weak: 2^28 per GPU
    n_total = args.elements * world if args.scaling == "weak" else args.elements
    lo, hi = sharding.shard_range(n_total, rank, world)
    n = hi - lo
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    # Tuned on B200 (tools/stream_geom_ab.py): 128-thread teams (W = 96 +
    # the master warp), 7 teams per SM, each thread streaming 2 consecutive
    # 16-byte units of x and of y per iteration (6.88 TB/s; 8 teams/SM with
    # the unit-cyclic schedule gave 6.70).
    workers = args.workers or 96
    teams = args.teams or sms * 7

    x = torch.empty(n, dtype=torch.float64, device=dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def fill():
        # each rank generates its own slice of the global counter-based inputs
        RG.fill_uniform(x, SEED_X, lo, stream=stream)
        RG.fill_uniform(y, SEED_Y, lo, stream=stream)

    fill()
    stream.synchronize()

    def step():
        RG.run_stream(x, y, COEF, teams, workers, stats=False, stream=stream)

    # runtime statistics of one launch (every team: no trap, one region)
    stats_out = RG.run_stream(x, y, COEF, teams, workers, stream=stream)
    stream.synchronize()
    st = stats_out.team_stats()
    assert all(s.trap == 0 and s.regions == 1 for s in st), "stream region trapped"
    smem_bytes = st[0].smem_bytes

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    # Two clocks over the same K steps: CUDA events on the launching stream
    # (device time, max over ranks = `value`), and a wall-clock window
    # bracketed by barriers on every rank -- if ranks did not actually run
    # concurrently (e.g. several ranks sharing one GPU) the window shows it.
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall_ms = (time.perf_counter() - w0) * 1e3
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    # every rank's (event ms, wall ms): a [world, 2] table filled row by row
    # and summed (all_reduce works on CUDA tensors under nccl and gloo alike)
    table = torch.zeros(world, 2, dtype=torch.float64, device=dev)
    table[rank, 0], table[rank, 1] = ms, wall_ms
    if world > 1:
        dist.all_reduce(table)
    gathered = table.cpu().tolist()
    rank_ms = [float(g[0]) for g in gathered]
    ms_max = max(rank_ms)
    wall_max = max(float(g[1]) for g in gathered)
    ms_per_step = ms_max / args.steps
    value = BYTES_PER_ELEM * n_total / (ms_per_step * 1e-3) / 1e9
    per_gpu = [round(BYTES_PER_ELEM * (sharding.shard_range(n_total, r, world)[1]
                                       - sharding.shard_range(n_total, r, world)[0])
                     / (rank_ms[r] / args.steps * 1e-3) / 1e9, 1) for r in range(world)]
    value_wall = BYTES_PER_ELEM * n_total * args.steps / (wall_max * 1e-3) / 1e9

    # Correctness gate (every N): regenerate the inputs, one region pass,
    # all-reduce the per-rank checksums and compare with the whole range's
    # expected checksum (fixture or oracle checker).
    fill()
    step()
    stream.synchronize()
    checksum = sharding.allreduce_checksum(RG.checksum(y, stream=stream), device=dev)
    want, want_src = expected_checksum(n_total, rank)
    if world > 1:  # rank 0's expectation (the oracle checker runs there only)
        wt = torch.tensor(list(sharding.split64(want or 0)) + [int(want is not None)],
                          dtype=torch.int64, device=dev)
        dist.broadcast(wt, 0)
        want = sharding.join64(int(wt[0]), int(wt[1])) if int(wt[2]) else None
    checksum_ok = want is not None and checksum == want
    gate = {"checksum": f"{checksum:#018x}",
            "expected": f"{want:#018x}" if want is not None else None,
            "checksum_ok": checksum_ok, "expected_from": want_src,
            "what": f"sum of y's fp64 bit patterns mod 2^64 after one region pass over "
                    f"[0, {n_total}) with regenerated inputs, per-rank element ranges "
                    f"all-reduced over {world} rank(s)"}

    from paper_1711_10413_b200 import occupancy as OCC
    regions = {} if args.only_stream else regions_section(RG, torch, dist, dev, stream, sms,
                                                          rank, world)
    configs = other_configs(RG, dev, stream, sms) if rank == 0 and not args.only_stream \
        else {}
    regs = ptxas_regs("StreamProgIdEELb1E") or 64
    thr = ((workers + 31) // 32) * 32 + 32
    occ = OCC.occupancy_for("b200", smem_bytes, regs, thr)

    peak, peak_src = measured_peaks()
    if "config2_shared_array" in configs:
        # from the queued steady-state time: it includes the write-back of
        # the dirty lines a single launch leaves in L2
        c2 = configs["config2_shared_array"]
        c2["roofline_frac"] = round(c2["GBps_queued"] / peak, 4)
        c2["roofline_frac_single_launch"] = round(c2["GBps"] / peak, 4)
    roofline = {"bound": "hbm", "achieved": round(value / world, 1), "peak": peak,
                "unit": "GB/s", "frac": round(value / world / peak, 4), "traffic": None,
                "peak_source": peak_src, "peak_nominal": 8000.0,
                "frac_nominal": round(value / world / 8000.0, 4),
                "algorithmic_bytes_per_launch": BYTES_PER_ELEM * n}
    # DRAM bytes per launch from the committed `ncu --set full` capture, used
    # only when it was taken on this exact build (sources hash) and size.
    tr = os.path.join(ROOT, "profiles", "traffic.json")
    roofline["traffic_source"] = None
    if os.path.exists(tr):
        try:
            from paper_1711_10413_b200.build import sources_sha256
            t = json.load(open(tr))
            if t.get("n") == n and t.get("sources_sha256") == sources_sha256():
                roofline["traffic"] = t["dram_bytes_per_launch"]
                roofline["traffic_source"] = (f"profiles/{t['source']}.json (ncu, this build: "
                                              f"sources {t['sources_sha256']})")
                roofline["traffic_over_algorithmic"] = round(
                    t["dram_bytes_per_launch"] / (BYTES_PER_ELEM * n), 4)
            else:
                roofline["traffic_source"] = ("profiles/traffic.json was captured for another "
                                              "build or size: not reported")
        except (OSError, ValueError, KeyError):
            pass

    line = {
        "metric": "stream region body GB/s (config 4, 24 B/elem)",
        "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config4_stream_region", "elements_per_gpu": n,
                   "elements_total": n_total, "teams": teams, "workers": workers,
                   "threads_per_team": ((workers + 31) // 32) * 32 + 32,
                   "shared_scalars": 8, "parallelism": f"element-range shards x{world}",
                   "l2": "inputs (2 x 8 B x n) larger than the 126 MB L2, no flush needed"},
        "roofline": roofline,
        "regions": regions,
        "smem_bytes_per_cta": smem_bytes,
        "smem_layout": "depot 80 + args window 160 + runtime span 49 (reference footprint 289)",
        "regs_per_thread": regs,
        "occupancy": {"model": "b200 row of the reference occupancy model",
                      "teams_by_regs": occ.teams_by_regs, "teams_by_smem": occ.teams_by_smem,
                      "teams_per_sm": occ.actual, "threads_per_team": thr,
                      "grid_teams_per_sm": round(teams / sms, 2),
                      "binding_limit": "registers" if occ.actual == occ.teams_by_regs
                      else "smem" if occ.actual == occ.teams_by_smem else "blocks/threads"},
        "checksum": f"{checksum:#018x}",
        "checksum_ok": checksum_ok,
        "correctness_gate": gate,
        "per_gpu_GBps": per_gpu,
        "aggregate_GBps": round(value, 1),
        "wall_window": {"ms": round(wall_max, 3), "GBps": round(value_wall, 1),
                        "how": "barrier-bracketed host wall clock around the same K steps "
                               "on every rank, max over ranks (the events time each rank's "
                               "own stream; this window also catches ranks that did not "
                               "overlap)"},
        "configs": configs,
        "gpu_launches": args.steps,
        "clocks": clk,
    }
    if not args.no_e2e:
        e = e2e(args, teams, workers, n, dev, world)
        if rank == 0:
            line["e2e"] = e
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(1 << 26, os.cpu_count() or 1)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))
        sys.stdout.flush()
    if not checksum_ok:
        sys.stderr.write(f"bench: checksum mismatch on rank {rank}: {gate}\n")
        sys.exit(1)


def regions_section(RG, torch, dist, dev, stream, sms, rank, world):
    """Config 1 (ns per region, whole-GPU regions/s), the args-list placement
    study and the runtime building blocks' overheads."""
    from paper_1711_10413_b200 import occupancy as OCC
    # config-1 latency: 1 team x 32 workers, R regions in a loop, 4 shared scalars
    R = 10_000
    # config 1 shares 2 int and 2 double scalars (RegionsProg<double>: c1, c2
    # int, c3, c4 and a[] double)
    a = torch.zeros(32, dtype=torch.float64, device=dev)
    smem1 = RG.run_regions(a, 1, 32, 10, stream=stream).team_stats()[0].smem_bytes
    stream.synchronize()
    # A latency-bound region on one SM runs at whatever clock the GPU is at:
    # right after the power-capped config-4 run that is still below max for
    # a while (config 1 measured 407-444 ns across back-to-back runs, flat
    # 407.6 in isolation, tools/cfg1_variance.py).  Let the clock recover,
    # and report the SM clock the probe sees on either side.
    time.sleep(1.0)
    clk_before = RG.probe_overheads(1024, stream=stream)["sm_clock_mhz"]
    ns_per_region = device_ms(stream, lambda: RG.run_regions(a, 1, 32, R, stream=stream)) \
        * 1e6 / R
    # the reference's integer analog (4 int captures, int body) beside it
    ai = torch.zeros(32, dtype=torch.int32, device=dev)
    ns_int = device_ms(stream, lambda: RG.run_regions(ai, 1, 32, R, stream=stream)) * 1e6 / R
    clk_after = RG.probe_overheads(1024, stream=stream)["sm_clock_mhz"]
    # the same protocol on every SM: 64-thread teams (the small-team
    # instantiation, 32 registers, up to 32 teams/SM by the occupancy model),
    # 20 per SM in one wave, 2000 regions each.  20 is the measured optimum
    # (profiles/r2v_cfg1_sweep_preload.json, tools/cfg1_sweep.py: 16/SM 6.40,
    # 18/SM 6.56, 20/SM 6.61, 22/SM 6.52, 24/SM 6.42, 32/SM 6.07 G regions/s;
    # even counts keep the 4 SM sub-partitions balanced, and past ~20 teams
    # the extra barrier-waiting warps cost more issue slots than they hide).
    # With N ranks the team grid (N x T) is sharded by range: rank r launches
    # teams [r*T, (r+1)*T) of the N*T grid (first_team/total_teams), the
    # whole-job rate is N*T*R2 over the slowest rank's time.
    from paper_1711_10413_b200 import occupancy as OCC
    # every team the register file holds (32/SM for the 32-register small-team
    # kernel: the measured optimum, profiles/r2s2_cfg1_ab.txt)
    per_sm1 = OCC.occupancy_for("b200", 265, ptxas_regs("RegionsProgIdEELb1ELb1E") or 52,
                                64).actual
    R2, teams2 = 2000, sms * per_sm1
    a2 = torch.zeros(world * teams2 * 32, dtype=torch.float64, device=dev)
    rng = dict(first_team=rank * teams2, total_teams=world * teams2)
    RG.run_regions(a2, teams2, 32, 10, stream=stream, **rng)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    time.sleep(1.0)  # every SM busy: start from recovered clocks, like the one-team runs
    ms2 = device_ms(stream, lambda: RG.run_regions(a2, teams2, 32, R2, stream=stream, **rng))
    ms2 = torch.tensor([ms2], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms2, op=dist.ReduceOp.MAX)
    agg_regions_per_s = world * teams2 * R2 / (float(ms2.item()) * 1e-3)
    # where the shared-args list lives (PAPER.md: the shared-memory list vs
    # the malloc back-up scheme, "as large as an order of magnitude"): the
    # 4-capture region with the 20-entry window, with a 2-entry window so the
    # list spills to the team's global slab, and spilled to device malloc
    # (window_general: the window list in the general instantiation -- forced
    # by counting per-thread barrier arrivals -- so the placement comparison
    # with the global lists, which only the general instantiation runs, is
    # like for like)
    placement = {}
    for name, pe, alloc, gen in (("window", 20, 0, False), ("window_general", 20, 0, True),
                                 ("global_slab", 2, 0, False), ("device_malloc", 2, 1, False)):
        row = {}
        for label, tm, rr in (("1team", 1, 2000), ("full", teams2, 200)):
            ap = torch.zeros(tm * 32, dtype=torch.float64, device=dev)
            xkw = {"barrier_arrivals": torch.zeros(tm * 64, dtype=torch.int32, device=dev)} \
                if gen else {}
            RG.run_regions(ap, tm, 32, 10, prealloc_entries=pe, list_allocator=alloc,
                           stream=stream, **xkw)
            ms_p = device_ms(stream, lambda: RG.run_regions(
                ap, tm, 32, rr, prealloc_entries=pe, list_allocator=alloc, stream=stream, **xkw))
            row[f"ns_per_region_{label}"] = round(ms_p * 1e6 / rr, 1)
            row[f"regions_per_s_{label}"] = round(tm * rr / (ms_p * 1e-3), 0)
        placement[name] = row
    # north_star's "push/pop + handoff overhead in ns per parallel region":
    # the building blocks timed alone on one SM (ompds_probe_overheads), and
    # the config-1 region split into the bare handoff and the rest (runtime
    # protocol + get-shared-variables + body)
    ov = RG.probe_overheads(8192, stream=stream)
    ov["config1_ns_per_region"] = round(ns_per_region, 1)
    ov["config1_protocol_ns_per_region"] = round(ns_per_region - ov["handoff_ns"], 1)
    # config 3: each worker warp pushes and pops 2 frames per nested region
    ov["config3_push_pop_ns_per_region"] = round(2 * ov["push_pop_pair_slot_ns"], 2)
    ov["config3_bookkeeping_ns_per_region"] = round(2 * ov["push_pop_pair_bookkeeping_ns"], 2)
    ov["how"] = ("one warp per mode, clock64 and %globaltimer over 8192 iterations; iteration i "
                 "pushes 1-2 frames of 40 B x 32 lanes (depth from a hash of i: frame size, "
                 "lanes, depths and slot capacity are kernel arguments), stores and loads one "
                 "word per lane in each, pops them; push_pop_pair_slot/chain = (that loop - the "
                 "same accesses at fixed addresses) per pair; bookkeeping = the push/pop "
                 "dependent chain with no frame access; handoff = release + join named "
                 "barriers between the master and one worker warp")
    # the reference-facing boundary: one omplab::TeamRuntime operation
    # through the stateful team handle (a launch + a stream sync each)
    from paper_1711_10413_b200 import runtime as RT
    rt = RT.TeamRuntime(RT.RuntimeConfig(), 0x2000, RT.RecordingHeap())
    rt.kernelInit(RT.MASTER, 1)
    n_calls = 0
    t0 = time.perf_counter()
    for _ in range(300):
        rt.prepareParallel(RT.MASTER, "wf", 4)
        rt.kernelParallel(RT.WORKER)
        rt.endParallel(RT.WORKER)
        n_calls += 3
    handle_us = (time.perf_counter() - t0) / n_calls * 1e6
    del rt
    return {"ns_per_region": round(ns_per_region, 1),
            "ns_per_region_int_analog": round(ns_int, 1),
            "team_handle_us_per_call": round(handle_us, 2),
            "regions_per_s": round(1e9 / ns_per_region, 1),
            "sm_clock_mhz_around": [clk_before, clk_after],
            "smem_bytes_per_cta": smem1,
            "teams_per_sm": per_sm1,
            "regs_per_thread": ptxas_regs("RegionsProgIdEELb1ELb1E"),
            "workload": "config 1: 1 team x 32 workers, 4 shared scalars (2 int, 2 double), "
                        f"{R} regions in a sequential loop",
            "aggregate_regions_per_s": round(agg_regions_per_s, 0),
            "aggregate_workload": f"{world * teams2} teams x 32 workers x {R2} regions"
                                  + (f", team grid sharded by range over {world} GPUs"
                                     if world > 1 else ""),
            "args_list_placement": placement,
            "overheads": ov}


def other_configs(RG, dev, stream, sms):
    """BASELINE configs 2 and 3 beside the headline (each timed with CUDA
    events on the launching stream; config 2 flushes L2 between launches)."""
    import torch
    out = {}
    # config 2: d[256] fp64 staged by TMA into the depot, parallel-for a[i] += d[i & 255]
    n2 = 1 << 24
    a = torch.zeros(n2, dtype=torch.float64, device=dev)
    d_init = torch.arange(256, dtype=torch.float64, device=dev) * 3 + 1
    # L2 "flush" by READING 256 MB: evicts a[] without leaving dirty lines
    # whose write-back would be charged to the timed kernel
    flush = torch.ones(64 << 20, dtype=torch.int32, device=dev)
    # teams per SM x W: 4 x 224 measured best on this build (tools/
    # config2_queued.py, profiles/r2s2_config2_geometry.txt); override with
    # OMPDS_BENCH_C2=KxW for A/B runs
    k2, w2 = (int(v) for v in os.environ.get("OMPDS_BENCH_C2", "4x224").split("x"))
    t2 = sms * k2
    time.sleep(1.0)  # HBM-bound: start below the power cap the config-4 run left
    times = []
    st = RG.run_shared_array(a, t2, w2, d_init=d_init, stream=stream).team_stats()[0]
    go = RG.prepared_shared_array(a, t2, w2, d_init=d_init, stream=stream)
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.sum()  # same stream
            # keep the GPU busy (~50 us) while the host enqueues e0, the
            # launch and e1, so no host-side launch gap lands between e0 and
            # the kernel (the kernel is ~45 us; a gap would be charged to it)
            torch.cuda._sleep(100_000)
            e0.record(stream)
            go()
            e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms_single = statistics.median(times)
    # Steady state: K x [evict L2; region] queued back to back minus
    # K x [evict L2] alone -- the region's device time without the launch
    # latency a single event-bracketed launch is charged.
    K = 20

    def queued(with_region):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(200_000)  # host enqueues everything while the GPU spins
            e0.record(stream)
            for _ in range(K):
                flush.sum()
                if with_region:
                    go()
            e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)

    queued(True)
    both = statistics.median(queued(True) for _ in range(3))
    alone = statistics.median(queued(False) for _ in range(3))
    ms_queued = (both - alone) / K
    ms = ms_single
    # the placement decision's other side: a zero-byte depot slot puts the
    # kernel frame (d[] included) on the master's global overflow chain;
    # the reserved warp copies d[] there and the body reads it from L1/L2
    st_o = RG.run_shared_array(a, t2, w2, d_init=d_init, depot_capacity=0,
                               stream=stream).team_stats()[0]
    go_o = RG.prepared_shared_array(a, t2, w2, d_init=d_init, stream=stream, depot_capacity=0)
    times_o = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.sum()
            torch.cuda._sleep(100_000)
            e0.record(stream)
            go_o()
            e1.record(stream)
        e1.synchronize()
        times_o.append(e0.elapsed_time(e1))
    ms_o = statistics.median(times_o)
    # the same bytes moved by a plain device copy of the same size (torch
    # copy_ of 2^24 doubles, the same queued [evict; copy] timing): the
    # practical ceiling for a 1:1 read/write stream this short
    src = torch.ones(n2, dtype=torch.float64, device=dev)

    def queued_copy(with_copy):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(200_000)
            e0.record(stream)
            for _ in range(K):
                flush.sum()
                if with_copy:
                    a.copy_(src)
            e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1)
    queued_copy(True)
    ms_copy = (statistics.median(queued_copy(True) for _ in range(3))
               - statistics.median(queued_copy(False) for _ in range(3))) / K
    del src
    out["config2_shared_array_overflow"] = {
        "elements": n2, "teams": t2, "workers": w2, "ms": round(ms_o, 4),
        "GBps": round(16 * n2 / ms_o / 1e6, 1), "depot_capacity": 0,
        "depot_in_smem": st_o.depot_in_smem, "smem_bytes_per_cta": st_o.smem_bytes}
    out["config2_shared_array"] = {
        "elements": n2, "teams": t2, "workers": w2, "ms": round(ms, 4),
        "GBps": round(16 * n2 / ms / 1e6, 1), "bytes_per_element": 16,
        "ms_queued": round(ms_queued, 4),
        "GBps_queued": round(16 * n2 / ms_queued / 1e6, 1),
        "timing": "ms: median of 10 launches, each after an L2 eviction and bracketed by "
                  f"CUDA events; ms_queued: {K} x [L2 evict; region] minus {K} x [L2 evict], "
                  "queued back to back (ncu's kernel duration: 41.7 us, profiles/r2s2g_config2_ncu.json)",
        "smem_bytes_per_cta": st.smem_bytes, "depot_in_smem": st.depot_in_smem,
        "regs_per_thread": ptxas_regs("SharedArrayProgWideIdEELb1E"),
        "staging": ("cp.async.bulk (TMA) of d[256] into the depot slot, completed asynchronously "
                    "(workers wait on the transaction barrier after their first loads of a[])"),
        "units": "32-byte vectors (a[] 32-byte aligned)",
        "roofline_frac": None,
        "same_size_copy_GBps_queued": round(16 * n2 / ms_copy / 1e6, 1),
        "frac_of_same_size_copy": round(ms_copy / ms_queued, 4),
        "l2": "evicted before every launch by reading a 256 MB buffer"}
    del a, flush
    # config 3: nested regions (depth 3) on per-warp data-sharing stacks;
    # "overflow": a zero-byte shared-memory slot puts every frame on the
    # warp's global overflow chain (the placement decision's other side)
    R = 2000
    for key, teams, slot in (("config3_nested_1team", 1, 2048),
                             ("config3_nested_full", sms * 8, 2048),
                             ("config3_nested_1team_overflow", 1, 0)):
        a3 = torch.zeros(teams * 96, dtype=torch.float64, device=dev)
        o3, stacks = RG.run_nested(a3, teams, 96, 10, warp_slot_bytes=slot, stream=stream)
        # timed: the launch only (collecting the warp statistics is host work)
        ms = device_ms(stream, lambda: RG.run_nested(a3, teams, 96, R, warp_slot_bytes=slot,
                                                     stream=stream, collect=False))
        out[key] = {"teams": teams, "workers": 96, "regions": R,
                    "ns_per_region": round(ms * 1e6 / R, 1),
                    "aggregate_regions_per_s": round(teams * R / (ms * 1e-3), 0),
                    "stack_depth": stacks[0][0].max_depth,
                    "frames_in_smem": stacks[0][0].frame_in_smem,
                    "warp_slot_bytes": slot,
                    "smem_bytes_per_cta": o3.team_stats()[0].smem_bytes,
                    "regs_per_thread": ptxas_regs("NestedProgIdEELb1E")}
    return out


def e2e(args, teams, workers, n, dev, world=1):
    """Same region through the C ABI's host-buffer entry point: H2D x,y from
    pinned memory, region, D2H y -- all inside the timed region.  With N
    ranks every rank moves its own shard; the time is the max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_1711_10413_b200 import regions as RG
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    yh = torch.empty(n, dtype=torch.float64).pin_memory()
    xd = torch.empty(n, dtype=torch.float64, device=dev)
    yd = torch.empty(n, dtype=torch.float64, device=dev)
    RG.fill_uniform(xd, SEED_X)
    RG.fill_uniform(yd, SEED_Y)
    xh.copy_(xd)
    yh.copy_(yd)
    stream = torch.cuda.Stream(device=dev)
    RG.run_stream_host(xh, yh, COEF, teams, workers, xd, yd, stream=stream)  # warm
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.e2e_steps):
        RG.run_stream_host(xh, yh, COEF, teams, workers, xd, yd, stream=stream)
    ev1.record(stream)
    ev1.synchronize()
    wall = time.perf_counter() - t0
    ms = ev0.elapsed_time(ev1) / args.e2e_steps
    if world > 1:
        t = torch.tensor([ms, wall], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, wall = float(t[0]), float(t[1])
    value = BYTES_PER_ELEM * n * world / (ms * 1e-3) / 1e9
    # The host link bounds this path: 16 B/element host->device (x, y) and
    # 8 B/element device->host (y).  Measure each direction alone (pinned,
    # one 2 GiB copy, CUDA events); with both directions overlapped the
    # bound is max(16n/h2d, 8n/d2h).
    link = {}
    s2 = torch.cuda.Stream(device=dev)

    def copy_rates(pairs):
        evs = []
        for st, dst, src in pairs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                e0.record(st)
                dst.copy_(src, non_blocking=True)
                e1.record(st)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return [8 * n / (a.elapsed_time(b) * 1e-3) / 1e9 for a, b in evs]

    copy_rates([(stream, xd, xh), (s2, yh, yd)])  # warm
    link["h2d"] = copy_rates([(stream, xd, xh)])[0]
    link["d2h"] = copy_rates([(s2, yh, yd)])[0]
    link["h2d_concurrent"], link["d2h_concurrent"] = copy_rates([(stream, xd, xh), (s2, yh, yd)])
    # independent directions: max(16n/h2d, 8n/d2h); measured concurrency: the
    # 8n bytes of y come back while x and y go in at the concurrent rates,
    # the rest of the 16n inbound bytes at the lone rate
    bound_ind_s = max(16 * n / (link["h2d"] * 1e9), 8 * n / (link["d2h"] * 1e9))
    t_both = 8 * n / (link["d2h_concurrent"] * 1e9)
    rest = max(0.0, 16 * n - link["h2d_concurrent"] * 1e9 * t_both)
    bound_s = max(bound_ind_s, t_both + rest / (link["h2d"] * 1e9))
    bound = BYTES_PER_ELEM * n * world / bound_s / 1e9
    bound_ind = BYTES_PER_ELEM * n * world / bound_ind_s / 1e9
    return {"value": round(value, 2), "unit": "GB/s",
            "h2d_bytes_per_step": 16 * n * world, "d2h_bytes_per_step": 8 * n * world,
            "ms_per_step": round(ms, 3), "wall_ms_per_step": round(wall / args.e2e_steps * 1e3, 3),
            "path": "ompds_run_stream_host (C ABI, pinned host buffers)",
            "link_roofline": {"bound": "host link (PCIe)", "h2d_GBps": round(link["h2d"], 1),
                              "d2h_GBps": round(link["d2h"], 1),
                              "h2d_concurrent_GBps": round(link["h2d_concurrent"], 1),
                              "d2h_concurrent_GBps": round(link["d2h_concurrent"], 1),
                              "bound_GBps": round(bound, 2), "frac": round(value / bound, 4),
                              "bound_independent_GBps": round(bound_ind, 2),
                              "how": "pinned 2 GiB copies, CUDA events, each direction alone "
                                     "and both at once; bound: y's 8n bytes return at the "
                                     "concurrent rates, the rest of the 16n inbound at the "
                                     "lone rate (bound_independent: max(16n/h2d, 8n/d2h))"}}


if __name__ == "__main__":
    main()
