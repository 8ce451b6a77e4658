"""CPU-side tests of the product library: the C ABI loads and exports every
symbol include/ompds.h declares; the host parts of the boundary (frame-layout
descriptor builder, occupancy model, trap strings) match the reference's
golden vectors and the oracle; compute entry points fail loudly without a
GPU instead of falling back to the CPU."""
import ctypes as C
import os
import random
import re

import pytest

import golden_util as G
import layout_util as LU
from oracle import oracle as O
from paper_1711_10413_b200 import _lib as P
from paper_1711_10413_b200 import layout, occupancy, runtime

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ompds.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ompds_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound():
    lib = P.lib()
    declared = header_functions()
    assert len(declared) >= 19
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(P.exported_symbols()) == declared


def test_struct_sizes_match_the_c_abi():
    # sizes implied by the header's field lists (natural alignment, x86-64)
    assert C.sizeof(P.RtCall) == 16
    assert C.sizeof(P.RtResult) == 32
    assert C.sizeof(P.Event) == 32
    assert C.sizeof(P.FrameVar) == 32
    assert C.sizeof(P.DepotSlot) == 32
    assert C.sizeof(P.DepotLayout) == 32
    assert C.sizeof(P.Launch) == 64
    assert C.sizeof(P.TeamStats) == 56
    assert C.sizeof(P.OverheadProbe) == 96


def test_trap_strings_are_the_reference_strings():
    strings = {r["trap"] for s in G.load("runtime") for r in s["results"] if not r["ok"]}
    assert {runtime.trap_reason(c) for c in range(1, 18)} == strings


@pytest.mark.parametrize("key", ["layouts", "layouts_o0", "layouts_bad_order"])
def test_product_layout_builder_matches_reference(key):
    for p in G.programs():
        if p.get(key) is None:
            continue
        out = LU.run_builder(P.lib().ompds_layout_build, p["frame_vars"], len(p["layouts"]),
                             LU.PIPE[key])
        assert LU.strip(out) == LU.golden_view(p[key]), (p["stem"], key)


def test_product_layout_builder_matches_oracle_on_random_frames():
    rng = random.Random(0x5eed01ab)
    for trial in range(400):
        n = rng.randint(0, 14)
        ngroups = rng.randint(1, 3)
        fv = []
        for i in range(n):
            first = rng.randint(-1, 30)
            fv.append({"group": rng.randrange(ngroups), "func": rng.randint(0, 1),
                       "name": f"v{i}", "bytes": rng.choice([4, 8, 12, 384, 1024, 0 + 4]),
                       "escapes": rng.random() < 0.3, "pinned": rng.random() < 0.2,
                       "def_pos": i, "first": first,
                       "last": first + rng.randint(0, 10) if first >= 0 else -1})
        for pipe in (0, 1, 2):
            a = LU.run_builder(P.lib().ompds_layout_build, fv, ngroups, pipe)
            b = LU.run_builder(O.lib().orc_layout_build, fv, ngroups, pipe)
            assert a == b, (trial, pipe)


def test_frame_block_and_manifest_render_like_the_reference():
    p = next(x for x in G.load("corpus") if x["stem"] == "shared_scalar")
    fv = [layout.FrameVar(v["name"], v["bytes"], v["group"], v["func"], v["escapes"], v["pinned"],
                          v["def_pos"], v["first"], v["last"]) for v in p["frame_vars"]]
    lays = layout.build_layouts(fv, len(p["layouts"]))
    golden_sir = open(os.path.join("/root/reference/proj/tests/golden/shared_scalar.sir")).read() \
        if os.path.exists("/root/reference/proj/tests/golden/shared_scalar.sir") else None
    text = "".join("\n" + layout.frame_block(layout.FrameGroup(r, m), l)
                   for (r, m), l in zip(G.frame_groups(p), lays))
    want = ("\nframe @__omp_offload_shared_scalar members [@__omp_offload_shared_scalar, "
            "@__omp_worker] {\n  slot 0: offset 0, size 8, align 8, shared, %c\n"
            "  slot 1: offset 8, size 8, align 8, local, %wf.addr\n"
            "  slot 2: offset 16, size 8, align 8, local, %args.addr\n  total 24, mirrored\n}\n")
    assert text.startswith(want)
    if golden_sir is not None:  # byte-equal to the reference's golden frame blocks
        assert golden_sir.endswith(text)
    m = layout.manifest_depot(lays[0])
    gm = p["manifest"]
    for k in ("depot", "stack_bytes", "prealloc_entries", "prealloc_bytes", "runtime_bytes",
              "shared_footprint"):
        assert m[k] == gm[k], k


@pytest.mark.parametrize("stem", ["shared_scalar", "two_regions", "seq_only"])
def test_frame_blocks_byte_equal_reference_golden_sir(stem):
    """All frame blocks of the reference's golden .sir modules
    (proj/tests/golden/*.sir, IRTests.cpp:169-178) rendered from our layouts."""
    path = f"/root/reference/proj/tests/golden/{stem}.sir"
    if not os.path.exists(path):
        pytest.skip("reference not mounted")
    p = next(x for x in G.load("corpus") if x["stem"] == stem)
    fv = [layout.FrameVar(v["name"], v["bytes"], v["group"], v["func"], v["escapes"], v["pinned"],
                          v["def_pos"], v["first"], v["last"]) for v in p["frame_vars"]]
    lays = layout.build_layouts(fv, len(p["layouts"]))
    text = "".join("\n" + layout.frame_block(layout.FrameGroup(r, m), l)
                   for (r, m), l in zip(G.frame_groups(p), lays))
    golden = open(path).read()
    assert golden.endswith(text)
    assert golden[: len(golden) - len(text)].rstrip().endswith("}")  # last function body
    # and the parser reads the reference's text back into the same layouts
    parsed = layout.parse_frame_blocks(golden)
    assert [(g.root, g.members) for g, _ in parsed] == [(r, m) for r, m in G.frame_groups(p)]
    assert [l for _, l in parsed] == lays


def test_frame_block_round_trip_over_all_programs():
    for p in G.programs():
        fv = [layout.FrameVar(v["name"], v["bytes"], v["group"], v["func"], v["escapes"],
                              v["pinned"], v["def_pos"], v["first"], v["last"])
              for v in p["frame_vars"]]
        for pipe in ("default", "bad_order"):
            lays = layout.build_layouts(fv, len(p["layouts"]), pipe)
            groups = [layout.FrameGroup(r, m) for r, m in G.frame_groups(p)]
            text = "".join(layout.frame_block(g, l) for g, l in zip(groups, lays))
            back = layout.parse_frame_blocks(text)
            assert [g for g, _ in back] == groups
            assert [l for _, l in back] == lays, p["stem"]


def test_audit_flags_the_bad_order_overlap():
    p = next(x for x in G.load("corpus") if x["stem"] == "coloring_demo")
    fv = [layout.FrameVar(v["name"], v["bytes"], v["group"], v["func"], v["escapes"], v["pinned"],
                          v["def_pos"], v["first"], v["last"]) for v in p["frame_vars"]]
    roots = [r for r, _ in G.frame_groups(p)]
    bad = layout.build_layouts(fv, len(roots), "bad_order")
    diags = layout.audit(bad, roots)
    want = p["bad_order_audit"]
    assert [(d["rule"], d["message"]) for d in diags] == [(d["rule"], d["message"]) for d in want]
    assert layout.audit(layout.build_layouts(fv, len(roots)), roots) == []


def test_occupancy_tables_match_reference_csv():
    occ = G.load("occupancy")
    assert occupancy.footprint_scalars_csv() == occ["footprint_scalars_csv"]
    assert occupancy.footprint_arrays_csv() == occ["footprint_arrays_csv"]
    for name, dev in occ["devices"].items():
        assert occupancy.occupancy_scalars_csv(name) == dev["occupancy_scalars_csv"], name
        assert occupancy.occupancy_arrays_csv(name) == dev["occupancy_arrays_csv"], name
        assert occupancy.max_vars_csv(name) == dev["max_vars_csv"], name
        for fp, regs, thr, tr, ts, pot, act, used in dev["occupancy_grid"]:
            o = occupancy.occupancy_for(name, fp, regs, thr)
            assert (o.teams_by_regs, o.teams_by_smem, o.potential, o.actual, o.smem_used) == \
                (tr, ts, pot, act, used)


def test_paper_footprints_and_capacity_law():
    # AcceptanceMain.cpp:88-90 and the 200-round byte law of RuntimeTests.cpp:235-252
    for n, total in zip([1, 2, 4, 8, 16, 32, 64], [233, 241, 257, 289, 353, 481, 737]):
        assert layout.shared_footprint(8 * n + 16) == total
    for k, total in zip([1, 2, 3, 4], [617, 1001, 1385, 1769]):
        assert layout.shared_footprint(384 * k + 24) == total
    for n in range(0, 129):
        assert runtime.dynamic_args_bytes(n) == (0 if n <= 20 else 8 * n)
    assert runtime.dynamic_args_bytes(5, 4) == 40


def test_b200_occupancy_row():
    # 265-byte team region (config 1 loop layout) at 64 threads, 32 regs:
    # the 32-CTA limit binds; at 40 regs the register file does: 1280
    # registers per warp, 12 warps in each 16K sub-partition = 24 teams (not
    # 65536 / 2560 = 25: a 25th team per SM measured as a partial second
    # wave, profiles/r2e_cfg1.json)
    o = occupancy.occupancy_for("b200", 265, 32, 64)
    assert o.actual == 32
    assert occupancy.occupancy_for("b200", 265, 40, 64).actual == 24
    assert occupancy.max_regs_for_teams("b200", 24, 64) == 40
    assert occupancy.max_regs_for_teams("b200", 25, 64) == 32
    # 1024-thread teams: the 2048-threads/SM limit binds (2 teams/SM).
    o = occupancy.occupancy_for("b200", 289, 32, 1024)
    assert o.potential == 2 and o.actual == 2
    # registers are allocated per warp, 8 per thread at a time: the
    # config-1 kernel at 49 registers x 64 threads fits 18 teams per SM --
    # ncu's launch__occupancy_limit_registers for it (profiles/r1d_regions_ncu.json);
    # the config-4 kernel at 64 x 128 fits 8 (ncu: 8)
    assert occupancy.occupancy_for("b200", 265, 49, 64).teams_by_regs == 18
    assert occupancy.occupancy_for("b200", 289, 64, 128).teams_by_regs == 8
    assert occupancy.max_regs_for_teams("b200", 18, 64) == 56


def test_compute_entry_point_raises_ompds_error_without_gpu():
    if P.lib().ompds_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(P.OmpdsError) as e:
        runtime.replay([(0, 0, 8)])
    assert e.value.code == P.ERR_CUDA


def test_b200_kernel_occupancy_table_from_ptxas_log():
    log = os.path.join(ROOT, "paper_1711_10413_b200", "_build", "ptxas.log")
    csv = occupancy.b200_kernel_occupancy_csv(log)
    rows = [r.split(",") for r in csv.strip().splitlines()[1:]]
    assert {r[0] for r in rows} >= {"RegionsProgIiEELb1ELb1E", "StreamProgIdEELb1E",
                                    "SharedArrayProgIdEELb1E"}
    for r in rows:
        regs, thr = int(r[2]), int(r[3])
        # teams_by_regs: per-warp allocation, registers rounded up to 8, each
        # warp inside one of the four 16K-register sub-partitions
        warps = (thr + 31) // 32
        per_part = 16384 // (((regs + 7) // 8 * 8) * 32)
        assert int(r[5]) == 4 * per_part // warps


@pytest.mark.parametrize("first,teams,total", [(-1, 2, 4), (3, 2, 4), (1, 2, 0), (0, 2, -1)])
def test_team_range_outside_the_grid_is_rejected(first, teams, total):
    """ompds_launch.first_team/total_teams (team-range sharding) are validated
    before anything touches a GPU."""
    import ctypes as C
    launch = P.Launch(teams, 32, 20, 0, -1, 0, 0, None, 0, first, total, 0, None)
    rc = P.lib().ompds_run_regions(C.byref(launch), 0, 1, C.c_void_p(16), None, None)
    assert rc == P.ERR_INVALID


def test_overhead_probe_validates_before_touching_a_gpu():
    import ctypes as C
    L = P.lib()
    for bad in (dict(iterations=0), dict(iterations=(1 << 20) + 1),
                dict(iterations=16, frame_bytes=6), dict(iterations=16, frame_bytes=512),
                dict(iterations=16, max_depth=5), dict(iterations=16, lanes=33)):
        p = P.OverheadProbe(**bad)
        assert L.ompds_probe_overheads(C.byref(p), None) == P.ERR_INVALID, bad
    assert L.ompds_probe_overheads(None, None) == P.ERR_INVALID
    if L.ompds_device_count() == 0:
        p = P.OverheadProbe(iterations=16)
        assert L.ompds_probe_overheads(C.byref(p), None) == P.ERR_CUDA


def test_team_handle_validates_and_needs_a_gpu():
    """ompds_team_create: invalid configurations are refused on the host;
    without a GPU there is no handle (no host fallback)."""
    import ctypes as C
    L = P.lib()
    h = C.c_void_p()
    cfg = P.RuntimeConfig(-1, 0)
    assert L.ompds_team_create(C.byref(cfg), 0x2000, P.AllocFn(), P.ReleaseFn(), None,
                               C.byref(h)) == P.ERR_INVALID
    cfg = P.RuntimeConfig(20, 0)
    alloc = P.AllocFn(lambda n, u: 0x1000)
    assert L.ompds_team_create(C.byref(cfg), 0x2000, alloc, P.ReleaseFn(), None,
                               C.byref(h)) == P.ERR_INVALID  # one callback without the other
    assert L.ompds_team_kernel_init(None, 0, 8) == P.ERR_INVALID
    if L.ompds_device_count() == 0:
        assert L.ompds_team_create(C.byref(cfg), 0x2000, P.AllocFn(), P.ReleaseFn(), None,
                                   C.byref(h)) == P.ERR_CUDA
        assert not h.value


def test_element_misaligned_pointers_are_rejected_before_a_gpu():
    """16-byte-unaligned views are served (element-wise variant); pointers
    not aligned to the element itself are invalid."""
    import ctypes as C
    launch = P.Launch(2, 32, 20, 0, -1, 0, 0, None, 0, 0, 0, 0, None)
    coef = (C.c_double * 8)()
    rc = P.lib().ompds_run_stream(C.byref(launch), 1, 10, C.c_void_p(4100), C.c_void_p(8192),
                                  coef, None, None)
    assert rc == P.ERR_INVALID
    rc = P.lib().ompds_run_shared_array(C.byref(launch), 0, 10, C.c_void_p(4098), None, None,
                                        None)
    assert rc == P.ERR_INVALID
    assert P.lib().ompds_run_regions(C.byref(launch), 1, 2, C.c_void_p(4100), None,
                                     None) == P.ERR_INVALID
