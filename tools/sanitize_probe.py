#!/usr/bin/env python
"""Small invocation of every generic-mode kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) runs on the GPU box:

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_1711_10413_b200 import regions as RG  # noqa: E402


def main():
    dev = "cuda"
    a = torch.zeros(3 * 40, dtype=torch.int32, device=dev)
    RG.run_regions(a, 3, 40, 3, max_events=256)
    a = torch.zeros(2 * 40, dtype=torch.float64, device=dev)
    RG.run_regions(a, 2, 40, 1)
    for cap in (-1, 0):
        s = torch.zeros(4099, dtype=torch.float64, device=dev)
        RG.run_shared_array(s, 4, 64, d_init=torch.arange(256, dtype=torch.float64,
                                                          device=dev), depot_capacity=cap)
    RG.run_shared_array(torch.zeros(1000, dtype=torch.int32, device=dev), 2, 33)
    # TMA-staged d[] read after the transaction barrier: 32-byte units, a
    # 16-byte aligned view (16-byte units), idle workers (n < workers)
    dd = torch.arange(256, dtype=torch.float64, device=dev)
    s = torch.zeros(4099, dtype=torch.float64, device=dev)
    RG.run_shared_array(s[2:4002], 3, 96, d_init=dd)
    RG.run_shared_array(s[:7], 3, 96, d_init=dd)
    RG.run_shared_array(torch.zeros(1000, dtype=torch.int32, device=dev), 2, 64,
                        d_init=torch.arange(256, dtype=torch.int32, device=dev))
    x = torch.ones(5003, dtype=torch.float64, device=dev)
    y = torch.ones(5003, dtype=torch.float64, device=dev)
    RG.run_stream(x, y, [k / 8 for k in range(1, 9)], 4, 96, max_events=512)
    RG.run_stream(x, y, [k / 8 for k in range(1, 9)], 4, 96, prealloc_entries=2)
    # args lists past the window: team slab and device malloc; team ranges
    for alloc in (0, 1):
        a = torch.zeros(2 * 40, dtype=torch.int32, device=dev)
        RG.run_regions(a, 2, 40, 3, prealloc_entries=2, list_allocator=alloc)
    a = torch.zeros(4 * 32, dtype=torch.int32, device=dev)
    RG.run_regions(a, 2, 32, 2, first_team=0, total_teams=4)
    RG.run_regions(a, 2, 32, 2, first_team=2, total_teams=4)
    for slot in (2048, 0):
        n = torch.zeros(2 * 72, dtype=torch.float64, device=dev)
        RG.run_nested(n, 2, 72, 2, warp_slot_bytes=slot)
    import golden_util as G
    from paper_1711_10413_b200 import program as PG
    from test_program import our_layouts, launches
    for stem in ("shared_scalar", "scalars_32", "two_regions", "private_inner"):
        p = next(x for x in G.load("corpus") if x["stem"] == stem)
        t, w, _ = launches(p)[0]
        prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
        bufs = [torch.full((sz,), init, dtype=torch.int32, device=dev)
                for _, sz, init in prog.buffers]
        PG.run_program(prog, bufs)
    # a runaway program trapping at the step limit
    p = next(x for x in G.load("corpus") if x["stem"] == "arrays_1")
    t, w, _ = launches(p)[0]
    prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
    bufs = [torch.full((sz,), init, dtype=torch.int32, device=dev)
            for _, sz, init in prog.buffers]
    PG.run_program(prog, bufs, step_limit=50)
    # two streams with spilled lists at once; the overhead probe
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    arrs = [torch.zeros(8 * 40, dtype=torch.int32, device=dev) for _ in sts]
    torch.cuda.synchronize()
    for st, a in zip(sts, arrs):
        RG.run_regions(a, 8, 40, 4, prealloc_entries=2, stream=st)
    torch.cuda.synchronize()
    for st in sts:
        RG.release_workspace(st)
    RG.probe_overheads(64)
    RG.probe_overheads(64, frame_bytes=256, max_depth=4, lanes=8)
    # nested region programs (per-lane data-sharing stacks, globalized frames)
    import nested_programs as NP
    for p in NP.corpus()[:4]:
        lays = PG.derive_layouts(p["ast"], p["kernel"])
        prog = PG.compile_program(p["ast"], lays, p["kernel"], p["teams"], p["workers"])
        for slot, ovf in ((4096, 32768), (0, 32768)):
            bufs = [torch.zeros(sz, dtype=torch.int32, device=dev) for _, sz, _ in prog.buffers]
            PG.run_program(prog, bufs, stack_slot_bytes=slot, stack_overflow_bytes=ovf)
    # per-thread barrier arrivals (general instantiation)
    a = torch.zeros(2 * 40, dtype=torch.int32, device=dev)
    arr = torch.zeros(2 * 72, dtype=torch.int32, device=dev)
    RG.run_regions(a, 2, 40, 3, barrier_arrivals=arr)
    # the stateful team handle (one launch per protocol call)
    from paper_1711_10413_b200 import runtime as R
    rt = R.TeamRuntime(R.RuntimeConfig(), 0x2000, R.RecordingHeap())
    rt.kernelInit(R.MASTER, 2)
    for nargs in (3, 25):
        rt.prepareParallel(R.MASTER, "wf", nargs)
        for _ in range(2):
            rt.kernelParallel(R.WORKER)
        for _ in range(2):
            rt.endParallel(R.WORKER)
    rt.kernelDeinit(R.MASTER)
    torch.cuda.synchronize()
    print("sanitize probe done")


if __name__ == "__main__":
    main()
