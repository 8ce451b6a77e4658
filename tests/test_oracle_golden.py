"""Pins the C oracle (oracle/ompds_oracle.c) to the reference's own outputs.

Every expectation here comes from tests/golden/*.json, produced by running
the UNMODIFIED reference (compiled in place from /root/reference/proj) --
see oracle/ref/ref_golden.cpp and tests/golden/regen.sh.
"""
import ctypes as C

import numpy as np
import pytest

import golden_util as G
import layout_util as LU
from oracle import oracle as O
from paper_1711_10413_b200 import _lib as P

OPNAMES = {0: "init", 1: "prepare", 2: "parallel", 3: "end", 4: "deinit"}


def _replay(fn, script):
    calls = script["calls"]
    n = len(calls)
    arr = (P.RtCall * max(n, 1))(*[P.RtCall(op, role, arg) for op, role, arg in calls])
    res = (P.RtResult * max(n, 1))()
    ev = (P.Event * 4096)()
    summ = P.RtSummary()
    cfg = P.RuntimeConfig(script["prealloc_entries"], 1 if script["fail_dynamic_alloc"] else 0)
    rc = fn(C.byref(cfg), arr, n, res, ev, 4096, C.byref(summ))
    assert rc == 0
    return list(res[:n]), list(ev[:min(summ.n_events, 4096)]), summ


def trap_string(code):
    return P.lib().ompds_trap_reason(code).decode()


def check_script(script, results, events, summ):
    """Compares one replayed script with the reference's recorded outcome."""
    name = script["name"]
    fn_names = []  # "region<k>" per successful prepare, in order
    for i, (call, want, got) in enumerate(zip(script["calls"], script["results"], results)):
        tag = f"{name} call {i} {OPNAMES[call[0]]}"
        assert (got.status == 0) == want["ok"], tag
        assert trap_string(got.status) == want["trap"], tag
        assert got.heap_live == want["heap_live"], tag
        if not want["ok"]:
            continue
        if call[0] == 1:
            fn_names.append(f"region{len(fn_names)}")
            kind = {"prealloc": P.ADDR_PREALLOC, "dynamic": P.ADDR_DYNAMIC}[want["addr"]]
            assert got.addr_kind == kind, tag
            assert got.live_bytes == want["live_bytes"], tag
        if call[0] == 2:
            kind = {"null": P.ADDR_NULL, "prealloc": P.ADDR_PREALLOC,
                    "dynamic": P.ADDR_DYNAMIC}[want["addr"]]
            assert got.addr_kind == kind, tag
            assert bool(got.participate) == want["participate"], tag
            assert (f"region{got.wf}" if got.wf >= 0 else "") == want["wf"], tag
    assert summ.workers == script["workers"], name
    assert summ.dynamic_allocs == script["dynamic_allocs"], name
    assert summ.dynamic_frees == script["dynamic_frees"], name
    assert summ.leaked_blocks == script["leaked_blocks"], name
    assert bool(summ.terminated) == script["terminated"], name
    got_ev = [[P.EVENT_KIND_NAMES[e.kind], f"region{e.fn}" if e.fn >= 0 else "", e.nargs,
               e.bytes] for e in events]
    assert got_ev == script["events"], name


def test_runtime_scripts_match_reference():
    scripts = G.load("runtime")
    assert len(scripts) > 600
    for s in scripts:
        check_script(s, *_replay(O.lib().orc_rt_replay, s))


def test_every_trap_string_is_exercised():
    seen = {r["trap"] for s in G.load("runtime") for r in s["results"] if not r["ok"]}
    want = {trap_string(c) for c in range(1, 18)}
    assert want <= seen, want - seen


@pytest.mark.parametrize("key", ["layouts", "layouts_o0", "layouts_bad_order"])
def test_layouts_match_reference(key):
    n = 0
    for p in G.programs():
        if p.get(key) is None:
            continue
        out = LU.run_builder(O.lib().orc_layout_build, p["frame_vars"], len(p["layouts"]),
                             LU.PIPE[key])
        assert LU.strip(out) == LU.golden_view(p[key]), (p["stem"], key)
        for g, want in zip(out, p[key]):
            assert (g["overlap_slot"] >= 0) == (want["overlap"] is not None), p["stem"]
        n += 1
    assert n >= 18 + 5 + 89


def test_coloring_demo_miscompile_shape():
    p = next(x for x in G.load("corpus") if x["stem"] == "coloring_demo")
    bad = LU.run_builder(O.lib().orc_layout_build, p["frame_vars"], len(p["layouts"]),
                         P.PIPELINE_BAD_ORDER)
    k = bad[0]
    assert k["total_local"] == 24
    assert k["slots"][0]["owners"] == ["c", "t"] and k["slots"][0]["shared"]
    assert k["overlap_slot"] == 0


def _spec(name):
    g = P.GpuSpec()
    assert P.lib().ompds_gpu_spec_get(name.encode(), C.byref(g)) == 0
    return g


def test_occupancy_grid_matches_reference():
    occ = G.load("occupancy")
    for name, dev in occ["devices"].items():
        g = _spec(name)
        for fp, regs, thr, tr, ts, pot, act, used in dev["occupancy_grid"]:
            o = P.Occupancy()
            O.lib().orc_occupancy_for(C.byref(g), fp, regs, thr, C.byref(o))
            assert (o.teams_by_regs, o.teams_by_smem, o.potential, o.actual, o.smem_used) == \
                (tr, ts, pot, act, used), (name, fp, regs, thr)
        for t, mv, mr in dev["max_shared_vars"]:
            assert O.lib().orc_max_shared_vars(C.byref(g), t) == mv, (name, t)
            assert O.lib().orc_max_regs_for_teams(C.byref(g), t, 128) == mr, (name, t)


def _analog(stem):
    return next(p for p in G.load("analogs") if p["stem"] == stem)


def test_config1_analog_values():
    for stem, regions in [("cfg1_analog", 1), ("cfg1_loop_analog", 5)]:
        p = _analog(stem)
        for run in p["runs"]:
            if not G.race_free_run(run) or run["teams"] != 1:
                continue
            w = run["workers"]
            a = np.zeros(w, dtype=np.int32)
            O.lib().orc_regions(0, 1, w, regions, O.ptr(a))
            want = run["sim"]["globals"]["a"]
            assert a[: len(want)].tolist() == want[:w] and all(v == 0 for v in want[w:])


def test_config2_analog_values():
    p = _analog("cfg2_analog")
    for run in p["runs"]:
        assert G.race_free_run(run)
        a = np.zeros(256, dtype=np.int32)
        O.lib().orc_shared_array(0, 256, O.ptr(a))
        assert a.tolist() == run["sim"]["globals"]["a"]


@pytest.mark.parametrize("n", [1024, 4096])
def test_config4_analog_values(n):
    p = _analog(f"cfg4_analog_{n}")
    x = np.array(p["inputs"]["x"], dtype=np.int32)
    y0 = np.array(p["inputs"]["y"], dtype=np.int32)
    # the golden's counter-based inputs are the oracle's integer fill
    xf = np.zeros(n, dtype=np.int32)
    O.lib().orc_fill(0, O.ptr(xf), n, 0x5eed01ab, 0)
    assert xf.tolist() == x.tolist()
    coef = np.arange(1, 9, dtype=np.int32)
    for run in p["runs"]:
        assert G.race_free_run(run)
        y = y0.copy()
        O.lib().orc_stream(0, n, O.ptr(x), O.ptr(y), O.ptr(coef), 2)
        assert y.tolist() == run["sim"]["globals"]["y"]
        assert x.tolist() == run["sim"]["globals"]["x"]


def test_fill_f64_is_exact_uniform():
    n = 4096
    a = np.zeros(n)
    O.lib().orc_fill(1, O.ptr(a), n, 0x5eed01ab, 7)
    z = np.array([O.lib().orc_splitmix64((0x5eed01ab + 7 + i) & (2**64 - 1)) for i in range(n)],
                 dtype=np.uint64)
    want = (z >> np.uint64(11)).astype(np.float64) * 2.0**-52 - 1.0
    assert np.array_equal(a, want)
    assert a.min() >= -1.0 and a.max() < 1.0


def test_checksum_is_bit_pattern_sum():
    a = np.random.default_rng(0).standard_normal(1000)
    want = int(a.view(np.uint64).sum(dtype=np.uint64))
    assert O.lib().orc_checksum(1, O.ptr(a), a.size) == want


def test_ds_stack_placement_rules():
    # slot 64 B: 16+16 fit, 48 does not -> chain; later small pushes stay on
    # the chain until it is popped back.
    ops = [16, 16, 48, 8, 0, 0, 8, 0, 0, 0]
    lanes = [1] * len(ops)
    n = len(ops)
    ins = (C.c_int32 * n)()
    off = (C.c_int64 * n)()
    md = C.c_int32()
    hw = C.c_int64()
    rc = O.lib().orc_ds_stack(64, 1024, (C.c_int64 * n)(*ops), (C.c_int32 * n)(*lanes), n, ins,
                              off, C.byref(md), C.byref(hw))
    assert rc == 0
    assert list(ins)[:4] == [1, 1, 0, 0] and list(off)[:4] == [0, 16, 0, 48]
    assert ins[6] == 1 and off[6] == 32  # after popping the chain, back in the slot
    assert md.value == 4 and hw.value == 32 + 56


def test_stream_checksum_equals_fill_stream_checksum_and_pins_the_fixture():
    """orc_stream_checksum (the config-5 checker: fill + one region pass +
    checksum of a range, no buffers) equals orc_fill + orc_stream +
    orc_checksum on the same range, for both element types and an offset
    range; and reproduces the committed fixture bench.py gates on."""
    import json
    import os
    import numpy as np
    from oracle import oracle as O
    L = O.lib()
    for elem, coef in ((1, np.array([k / 8 for k in range(1, 9)])),
                       (0, np.arange(1, 9, dtype=np.int32))):
        dt = np.float64 if elem else np.int32
        lo, n = 12_345, 100_003
        x, y = np.empty(n, dt), np.empty(n, dt)
        L.orc_fill(elem, O.ptr(x), n, 0x5eed01ab, lo)
        L.orc_fill(elem, O.ptr(y), n, 0x5eed01ac, lo)
        L.orc_stream(elem, n, O.ptr(x), O.ptr(y), O.ptr(coef), 0)
        assert L.orc_checksum(elem, O.ptr(y), n) == L.orc_stream_checksum(
            elem, lo, lo + n, 0x5eed01ab, 0x5eed01ac, O.ptr(coef), 0)
    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                     "config5_checksums.json")))
    cf = np.array(fx["coef"])
    for n in (1 << 20, 1 << 22):
        got = L.orc_stream_checksum(1, 0, n, fx["seed_x"], fx["seed_y"], O.ptr(cf), 0)
        assert "%#018x" % got == fx["checksums"][str(n)]
    # shards gather to the whole range (sum mod 2^64 over element ranges)
    n = 1 << 22
    from paper_1711_10413_b200 import sharding
    for world in (2, 3, 8):
        acc = 0
        for r in range(world):
            a, b = sharding.shard_range(n, r, world)
            acc = (acc + L.orc_stream_checksum(1, a, b, fx["seed_x"], fx["seed_y"],
                                               O.ptr(cf), 0)) & ((1 << 64) - 1)
        assert "%#018x" % acc == fx["checksums"][str(n)]


def test_ast_oracle_reproduces_the_reference_oracle():
    """oracle/ast_oracle.py (the checker for nested-region programs) is
    pinned against the reference's own sequential oracle: for every corpus,
    generated and analog program the reference compiles correctly, under
    every recorded launch shape, the final mapped arrays are equal."""
    import golden_util as G
    from oracle import ast_oracle as AO
    n = 0
    for p in G.programs():
        if p["stem"].startswith("gen_") and G.reference_broken(p):
            continue
        if "ast" not in p:
            continue
        tgt = p["ast"]["target"]
        for run in p["runs"]:
            o = run.get("oracle")
            if not o or not o.get("ok"):
                continue
            t = run["teams"] if run["teams"] > 0 else (tgt.get("num_teams") or 1)
            w = run["workers"] if run["workers"] > 0 else (tgt.get("thread_limit") or 32)
            got = AO.run(p["ast"], t, w, p.get("inputs"))
            want = {k: v for k, v in o["globals"].items() if k in got}
            assert {k: got[k] for k in want} == want, (p["stem"], t, w)
            n += 1
    assert n >= 190


def test_derived_frame_layouts_equal_the_reference_o0_layouts():
    """program.derive_layouts (frame variables from the AST, for programs
    the reference frontend cannot compile) reproduces the reference's O0
    frame layouts of every program it compiles correctly."""
    import golden_util as G
    from paper_1711_10413_b200 import program as PG
    keys = ("root", "total_local", "total_shared", "has_shared_depot", "slots")
    n = 0
    for p in G.programs():
        if (p["stem"].startswith("gen_") and G.reference_broken(p)) or not p.get("layouts_o0"):
            continue
        got = [{k: g[k] for k in keys} for g in PG.derive_layouts(p["ast"], p["kernel"])]
        assert got == [{k: g[k] for k in keys} for g in p["layouts_o0"]], p["stem"]
        n += 1
    assert n >= 112
