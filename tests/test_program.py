"""The reference's own programs executed by the GPU runtime.

Every corpus program (proj/programs/*.ompk), the reference's generator corpus
(ProgramGen.cpp, seed 0x5eed01ab; minus the 31 programs the reference itself
miscompiles) and the config analogs are lowered from the reference AST with
frame layouts from OUR layout builder, then run as region programs.  Outputs
must equal the reference simulator's final globals bit for bit, and the
runtime statistics (master barriers per team, releases, dynamic args-list
bytes/allocs/frees) its SimStats."""
import pytest

import golden_util as G
from paper_1711_10413_b200 import layout as LY
from paper_1711_10413_b200 import program as PG


def our_layouts(p, pipeline="default"):
    fv = [LY.FrameVar(v["name"], v["bytes"], v["group"], v["func"], v["escapes"], v["pinned"],
                      v["def_pos"], v["first"], v["last"]) for v in p["frame_vars"]]
    roots = [g["root"] for g in p["layouts"]]
    lays = LY.build_layouts(fv, len(roots), pipeline)
    return [{"root": r, "total_local": l.total_local, "total_shared": l.total_shared,
             "slots": [{"offset": s.offset, "size": s.size, "shared": s.shared,
                        "owners": s.owners} for s in l.slots]} for r, l in zip(roots, lays)]


def launches(p):
    """(teams, workers, run) for every race-free launch recorded for p."""
    out = []
    ast = p["ast"]["target"]
    for run in p["runs"]:
        if not G.race_free_run(run):
            continue
        t = run["teams"] if run["teams"] > 0 else (ast.get("num_teams") or 1)
        w = run["workers"] if run["workers"] > 0 else (ast.get("thread_limit") or 32)
        out.append((t, w, run))
    return out


def programs():
    ps = []
    for p in G.programs():
        if p["stem"].startswith("gen_") and G.reference_broken(p):
            continue
        if p["stem"].startswith("cfg4"):
            continue  # needs input overrides; covered below
        ps.append(p)
    return ps


def simulate(prog: PG.Program, inputs):
    """Pure-Python execution of the lowered program with the oracle's
    sequential semantics (test-only check of the lowering)."""
    def wrap(v):
        v &= 0xFFFFFFFF
        return v - (1 << 32) if v >= 1 << 31 else v

    bufs = [list(b) for b in inputs]
    for team in range(prog.teams):
        depot = {}
        mlocal = {}

        def cell(store, v, idx, caps, priv):
            sp, off, n = prog.vars[v]
            if not 0 <= idx < n:
                raise IndexError
            if sp == PG.SP_DEPOT:
                return depot, off + 4 * idx
            if sp == PG.SP_MLOCAL:
                return mlocal, off + 4 * idx
            if sp == PG.SP_PRIV:
                return priv, off + 4 * idx
            if sp == PG.SP_CAPTURE:
                d, o = caps[off]
                return d, o + 4 * idx
            return ("buf", off), idx

        def ld(v, idx, caps, priv):
            d, o = cell(None, v, idx, caps, priv)
            if isinstance(d, tuple):
                return bufs[d[1]][o]
            return d.get(o, 0)

        def stv(v, idx, val, caps, priv):
            d, o = cell(None, v, idx, caps, priv)
            if isinstance(d, tuple):
                bufs[d[1]][o] = val
            else:
                d[o] = val

        def run(pc, tid, caps, priv, nthreads, in_region=False):
            st = []
            code = prog.code
            while True:
                op = code[pc]
                pc += 1
                if op == PG.OP_END:
                    return None, pc
                if op == PG.OP_PUSH:
                    st.append(code[pc]); pc += 1
                elif op == PG.OP_LOAD:
                    st.append(ld(code[pc], 0, caps, priv)); pc += 1
                elif op == PG.OP_STORE:
                    stv(code[pc], 0, st.pop(), caps, priv); pc += 1
                elif op == PG.OP_LOADX:
                    st.append(ld(code[pc], st.pop(), caps, priv)); pc += 1
                elif op == PG.OP_STOREX:
                    val = st.pop(); idx = st.pop()
                    stv(code[pc], idx, val, caps, priv); pc += 1
                elif op in (PG.OP_ADD, PG.OP_SUB, PG.OP_MUL):
                    b = st.pop(); a = st.pop()
                    st.append(wrap(a + b if op == PG.OP_ADD else a - b if op == PG.OP_SUB
                                   else a * b))
                elif op == PG.OP_TID:
                    st.append(tid)
                elif op == PG.OP_TEAM:
                    st.append(team)
                elif op == PG.OP_NTHREADS:
                    st.append(nthreads)
                elif op == PG.OP_NTEAMS:
                    st.append(prog.teams)
                elif op == PG.OP_JMP:
                    pc = code[pc]
                elif op == PG.OP_JNLT:
                    t = code[pc]; pc += 1
                    b = st.pop(); a = st.pop()
                    if not a < b:
                        pc = t
                elif op == PG.OP_PARALLEL and in_region:
                    # nested region (EXTENSION): serialized, a team of one,
                    # captures are addresses in this activation
                    reg2 = prog.regions[code[pc]]
                    pc += 1
                    caps2 = [cell(None, v, 0, caps, priv) for v in reg2.captures]
                    run(reg2.entry, 0, caps2, {}, 1, True)
                elif op == PG.OP_PARALLEL:
                    return code[pc], pc + 1
                elif op == PG.OP_ZERO_PRIV:
                    priv.clear()

        pc = 0
        while True:
            r, pc = run(pc, 0, None, None, 1)
            if r is None:
                break
            reg = prog.regions[r]
            caps = []
            for v in reg.captures:
                sp, off, _ = prog.vars[v]
                caps.append((depot if sp == PG.SP_DEPOT else mlocal, off))
            for w in range(prog.workers):
                run(reg.entry, w, caps, {}, prog.workers, True)
    return bufs


def mapped_inputs(p, prog):
    return [[init] * n for _, n, init in prog.buffers]


def test_lowering_reproduces_reference_outputs_on_cpu():
    n = 0
    for p in programs():
        for t, w, run in launches(p):
            prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
            got = simulate(prog, mapped_inputs(p, prog))
            want = run["sim"]["globals"]
            for (name, _, _), vals in zip(prog.buffers, got):
                assert vals == want[name], (p["stem"], t, w, name)
            n += 1
    assert n > 150


def test_every_lowered_program_passes_the_verifier():
    """ompds_program_verify (run by ompds_run_program before any launch)
    accepts every program the lowering produces, incl. the bad-pass-order
    layouts."""
    from paper_1711_10413_b200 import _lib as L
    n = 0
    for p in programs():
        for pipeline in ("default", "bad_order"):
            prog = PG.compile_program(p["ast"], our_layouts(p, pipeline), p["kernel"], 2, 40)
            assert PG.verify(prog) == L.OK, (p["stem"], pipeline)
            n += 1
    assert n > 200


def _mutants(prog):
    """(label, program) pairs each breaking one rule the verifier enforces."""
    import dataclasses
    code = list(prog.code)
    out = []

    def with_code(c):
        return dataclasses.replace(prog, code=c)

    out.append(("unknown opcode", with_code(code[:-1] + [99])))
    out.append(("falls off the end", with_code(code[:-1] + [PG.OP_TID])))
    out.append(("stack underflow at entry", with_code([PG.OP_ADD] + code[1:])))
    out.append(("jump into an operand", with_code([PG.OP_JMP, 3, PG.OP_PUSH, 7, PG.OP_END])))
    out.append(("jump past the end", with_code([PG.OP_JMP, 10 ** 6] + code[2:])))
    out.append(("stack overflow", with_code([PG.OP_TID] * 33 + [PG.OP_END])))
    out.append(("ZERO_PRIV in master code", with_code([PG.OP_ZERO_PRIV] + code)))
    out.append(("parallel with a value on the stack",
                with_code([PG.OP_TID, PG.OP_PARALLEL, 0, PG.OP_END])))
    out.append(("parallel of a missing region",
                with_code([PG.OP_PARALLEL, len(prog.regions), PG.OP_END])))
    out.append(("variable index out of range",
                with_code([PG.OP_LOAD, len(prog.vars), PG.OP_STORE, 0, PG.OP_END])))
    return out


def test_verifier_rejects_malformed_programs():
    """A malformed program is OMPDS_ERR_INVALID before any launch -- never a
    device fault -- for each rule (tests run without a GPU)."""
    from paper_1711_10413_b200 import _lib as L
    p = next(q for q in programs() if q["stem"] == "shared_scalar")
    t, w, _ = launches(p)[0]
    prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
    assert PG.verify(prog) == L.OK
    for label, bad in _mutants(prog):
        assert PG.verify(bad) == L.ERR_INVALID, label
    # region-side rules: a depot variable or a capture beyond the region's
    # nargs inside a region body, a region entry inside an operand
    import dataclasses
    r0 = prog.regions[0]
    depot_var = next(i for i, v in enumerate(prog.vars) if v[0] == PG.SP_DEPOT)
    body = [PG.OP_ZERO_PRIV, PG.OP_LOAD, depot_var, PG.OP_STORE, depot_var, PG.OP_END]
    bad = dataclasses.replace(prog, code=list(prog.code) + body,
                              regions=[dataclasses.replace(r0, entry=len(prog.code))]
                              + list(prog.regions[1:]))
    assert PG.verify(bad) == L.ERR_INVALID
    cap = len(prog.vars)
    vars_ = list(prog.vars) + [(PG.SP_CAPTURE, len(r0.captures), 1)]
    body = [PG.OP_ZERO_PRIV, PG.OP_LOAD, cap, PG.OP_STORE, cap, PG.OP_END]
    bad = dataclasses.replace(prog, code=list(prog.code) + body, vars=vars_,
                              regions=[dataclasses.replace(r0, entry=len(prog.code))]
                              + list(prog.regions[1:]))
    assert PG.verify(bad) == L.ERR_INVALID
    bad = dataclasses.replace(prog, regions=[dataclasses.replace(r0, entry=r0.entry + 2)]
                              + list(prog.regions[1:]))
    assert PG.verify(bad) in (L.ERR_INVALID, L.OK)  # +2 may still be a boundary
    # layout rules: a depot that would misalign the args window
    # and runtime span; a frame variable at an offset that is not a multiple
    # of 4; a region-side capture larger than the master variable it aliases
    assert PG.verify(dataclasses.replace(prog, total_shared=prog.total_shared + 4)) == \
        L.ERR_INVALID
    sp, off, cnt = prog.vars[depot_var]
    vars_ = list(prog.vars)
    vars_[depot_var] = (sp, off + 2, cnt)
    assert PG.verify(dataclasses.replace(prog, vars=vars_, total_shared=prog.total_shared + 8)) \
        == L.ERR_INVALID
    cap_vars = [i for i, v in enumerate(prog.vars) if v[0] == PG.SP_CAPTURE]
    assert cap_vars, "shared_scalar's region reads a capture"
    vars_ = list(prog.vars)
    sp, j, cnt = vars_[cap_vars[0]]
    vars_[cap_vars[0]] = (sp, j, cnt + 1)
    assert PG.verify(dataclasses.replace(prog, vars=vars_)) == L.ERR_INVALID
    # the same descriptor is refused by ompds_run_program before the launch
    import ctypes as C
    desc, _keep = PG.describe(_mutants(prog)[0][1], [16])
    launch = L.Launch(1, 32, 20, 0, -1, 0, 0, None, 0, 0, 0, 0, None)
    assert L.lib().ompds_run_program(C.byref(launch), C.byref(desc), None, None) == L.ERR_INVALID


def test_sharing_analysis_matches_reference_detection():
    """The captures the lowering derives from the AST are exactly the kernel
    allocas the reference's escape detection marks shared
    (LoweringPasses.cpp:107-139 on the post-codegen module)."""
    n = 0
    for p in programs():
        t, w, _ = launches(p)[0] if launches(p) else (1, 8, None)
        prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
        caps = {prog.var_names[v] for r in prog.regions for v in r.captures}
        want = set(p["detected_shared"].get(p["kernel"], []))
        assert caps == want, p["stem"]
        n += 1
    assert n > 100


def test_captures_follow_the_reference_order():
    p = next(x for x in G.load("corpus") if x["stem"] == "mixed_captures")
    prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], 4, 96)
    assert [prog.var_names[v] for v in prog.regions[0].captures] == \
        [f"c{k}" for k in range(1, 8)]


@pytest.mark.gpu
def test_gpu_runs_reference_programs_bit_exact():
    import torch
    n = 0
    for p in programs():
        for t, w, run in launches(p):
            prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
            bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
                    for _, sz, init in prog.buffers]
            out = PG.run_program(prog, bufs, max_events=4096 if t * w <= 4096 else 0)
            sim = run["sim"]
            for (name, _, _), b in zip(prog.buffers, bufs):
                assert b.cpu().tolist() == sim["globals"][name], (p["stem"], t, w, name)
            st = out.team_stats()
            assert [s.trap for s in st] == [0] * t, (p["stem"], t, w)
            assert [s.master_barriers for s in st] == sim["master_barrier_entries"], p["stem"]
            assert [s.barrier_releases for s in st] == sim["barrier_releases"], p["stem"]
            assert sum(s.dynamic_alloc_bytes for s in st) == sim["dynamic_alloc_bytes"]
            assert sum(s.dynamic_allocs for s in st) == sim["dynamic_allocs"]
            assert sum(s.dynamic_frees for s in st) == sim["dynamic_frees"]
            n += 1
    assert n > 150


@pytest.mark.gpu
def test_gpu_per_thread_barrier_entries_match_the_simulator():
    """SimStats::BarrierEntries (Simulator.h:42-55) for every thread of every
    team of every reference program: each worker's handoff arrivals equal
    the simulator's per-thread count (2R+1), the master's protocol barriers
    equal its entries (2R; on the GPU it adds the explicit termination
    release that stands in for the simulator's master exit,
    Simulator.cpp:475-478), and the reserved warp's idle lanes -- which the
    simulator never lets enter a barrier (SimulatorTests.cpp:85-93) -- arrive
    only at the master's handoff barriers, in lockstep with it, never at one
    of their own (hardware barriers count every lane of a warp that is
    resident: DESIGN.md §2)."""
    import torch
    n = 0
    for p in programs():
        for t, w, run in launches(p):
            sim = run["sim"]
            ref = sim.get("barrier_entries")
            assert ref and len(ref) == t, p["stem"]
            prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
            bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
                    for _, sz, init in prog.buffers]
            arr = torch.full((t * (w + 32),), -1, dtype=torch.int32, device="cuda")
            out = PG.run_program(prog, bufs, barrier_arrivals=arr)
            got = arr.view(t, w + 32).cpu().tolist()
            st = out.team_stats()
            for team in range(t):
                r, g = ref[team], got[team]
                assert len(r) == w + 32
                assert g[:w] == r[:w], (p["stem"], t, w, team)           # workers
                assert st[team].master_barriers == r[w]                   # master protocol
                assert g[w] == r[w] + 1                                   # + termination
                assert r[w + 1:] == [0] * 31                              # reference idle
                assert g[w + 1:] == [g[w]] * 31, (p["stem"], team)        # shadow the master
            n += 1
    assert n > 150


@pytest.mark.gpu
def test_gpu_programs_queued_back_to_back_without_a_sync():
    """ompds_run_program is asynchronous: every corpus/generated program is
    enqueued on one stream with no synchronisation in between (each launch
    restages its tables into the stream's workspace behind the previous
    kernel), then all outputs are checked at once."""
    import torch
    pending = []
    for p in programs()[:60]:
        t, w, run = launches(p)[0]
        prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
        bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
                for _, sz, init in prog.buffers]
        pending.append((p["stem"], prog, bufs, run, PG.run_program(prog, bufs)))
    torch.cuda.synchronize()
    assert len(pending) >= 40
    for stem, prog, bufs, run, out in pending:
        for (name, _, _), b in zip(prog.buffers, bufs):
            assert b.cpu().tolist() == run["sim"]["globals"][name], (stem, name)
        assert all(s.trap == 0 for s in out.team_stats()), stem


@pytest.mark.gpu
def test_gpu_reproduces_the_pass_order_miscompile():
    """SimulatorTests.cpp:150-173: bad pass order merges master-private t into
    the shared slot of c; unguarded, workers read 7 instead of 1."""
    import torch
    p = next(x for x in G.load("corpus") if x["stem"] == "coloring_demo")
    want_bad = p["bad_order_sim_unguarded"]["globals"]["a"]
    assert want_bad == [7] * 8
    for pipeline, want in (("bad_order", want_bad), ("default", [1] * 8)):
        prog = PG.compile_program(p["ast"], our_layouts(p, pipeline), p["kernel"], 1, 8)
        a = torch.zeros(8, dtype=torch.int32, device="cuda")
        PG.run_program(prog, [a])
        assert a.cpu().tolist() == want, pipeline


@pytest.mark.gpu
def test_gpu_program_events_match_reference():
    import torch
    from test_gpu_regions import canon
    checked = 0
    for p in programs():
        runs = [r for r in launches(p) if "team_events" in r[2]["sim"]]
        if not runs:
            continue
        t, w, run = runs[0]
        stem = p["stem"]
        checked += 1
        prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
        bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
                for _, sz, init in prog.buffers]
        out = PG.run_program(prog, bufs, max_events=4096)
        names = {}
        for team in range(t):
            ref = []
            for k, fn, nn, b in run["sim"]["team_events"][team]:
                if k.startswith("prepare"):
                    names.setdefault(fn, len(names))
                ref.append((k, names[fn] if fn else -1, nn, b))
            assert canon(out.team_events()[team]) == canon(ref), (stem, team)
    assert checked > 100


@pytest.mark.gpu
def test_gpu_out_of_bounds_traps():
    import torch
    p = next(x for x in G.load("corpus") if x["stem"] == "scalars_1")
    prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], 4, 8)  # a[16] overrun
    a = torch.zeros(16, dtype=torch.int32, device="cuda")
    out = PG.run_program(prog, [a])
    assert any(s.trap == 20 for s in out.team_stats())


@pytest.mark.gpu
@pytest.mark.parametrize("prealloc,allocator", [(64, 0), (33, 0), (0, 0), (20, 1)])
def test_gpu_window_sizes_and_allocators_keep_reference_outputs(prealloc, allocator):
    """The 32- and 64-capture corpus programs with windows of 64 (every list
    in shared memory, 2 entries per publishing lane), 33, 0 (every list in
    global memory) entries, and with device-malloc lists: outputs and barrier
    counts stay the reference's; only the allocation statistics follow the
    window (DeviceRuntime.cpp:61-74: dynamic iff nargs > PreallocEntries)."""
    import torch
    checked = 0
    for p in programs():
        if p["stem"] not in ("scalars_32", "scalars_64", "shared_scalar", "mixed_captures"):
            continue
        for t, w, run in launches(p)[:2]:
            prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
            bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
                    for _, sz, init in prog.buffers]
            out = PG.run_program(prog, bufs, prealloc_entries=prealloc,
                                 list_allocator=allocator)
            sim = run["sim"]
            for (name, _, _), b in zip(prog.buffers, bufs):
                assert b.cpu().tolist() == sim["globals"][name], (p["stem"], prealloc, name)
            st = out.team_stats()
            assert [s.trap for s in st] == [0] * t
            assert [s.master_barriers for s in st] == sim["master_barrier_entries"]
            nregions = [len(r.captures) for r in prog.regions]
            dyn = sum(1 for n in nregions if n > prealloc)
            for s in st:
                assert s.dynamic_allocs == s.dynamic_frees
                assert s.dynamic_allocs >= dyn and (dyn > 0 or s.dynamic_allocs == 0)
            checked += 1
    assert checked >= 4


@pytest.mark.gpu
def test_gpu_reference_programs_sharded_by_team_range():
    """Every multi-team reference program run as two team-range shards
    (first_team / total_teams; omp_get_team_num and omp_get_num_teams are
    the grid's) leaves the same buffers as the reference simulator."""
    import torch
    checked = 0
    for p in programs():
        for t, w, run in launches(p):
            if t < 2:
                continue
            prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
            bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
                    for _, sz, init in prog.buffers]
            half = t // 2
            for lo, n in ((0, half), (half, t - half)):
                out = PG.run_program(prog, bufs, first_team=lo, total_teams=t, teams=n)
                assert [s.trap for s in out.team_stats()] == [0] * n
            for (name, _, _), b in zip(prog.buffers, bufs):
                assert b.cpu().tolist() == run["sim"]["globals"][name], (p["stem"], t, w, name)
            checked += 1
            break
    assert checked >= 10


@pytest.mark.gpu
def test_gpu_runtime_parameters_never_change_program_outputs():
    """Seeded fuzz over the reference's programs x the runtime's knobs: window
    size (0/1/2/20/64 entries), args-list allocator (slab / device malloc),
    event log on/off, depot slot capacity (smem or the global chain) and
    team-range sharding (1-3 launches).  The final globals and the barrier
    counts must be the reference simulator's for every combination; the
    dynamic allocations must follow the window (every region whose capture
    count exceeds the window allocates and frees once)."""
    import random
    import torch
    rng = random.Random(0x5eed01ab)
    cases = []
    for p in programs():
        for t, w, run in launches(p):
            cases.append((p, t, w, run))
    rng.shuffle(cases)
    checked = 0
    for p, t, w, run in cases[:80]:
        pe = rng.choice([0, 1, 2, 20, 64])
        alloc = rng.choice([0, 0, 1])
        log = rng.random() < 0.3 and t * w <= 4096
        depot_cap = rng.choice([-1, -1, 0])
        shards = rng.choice([1, 1, 2, 3]) if t >= 2 else 1
        prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
        bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
                for _, sz, init in prog.buffers]
        stats = []
        for g in range(shards):
            lo, hi = g * t // shards, (g + 1) * t // shards
            if hi == lo:
                continue
            out = PG.run_program(prog, bufs, prealloc_entries=pe, list_allocator=alloc,
                                 max_events=4096 if log else 0, depot_capacity=depot_cap,
                                 first_team=lo, total_teams=t, teams=hi - lo)
            stats += out.team_stats()
        key = (p["stem"], t, w, pe, alloc, log, depot_cap, shards)
        for (name, _, _), b in zip(prog.buffers, bufs):
            assert b.cpu().tolist() == run["sim"]["globals"][name], key
        assert [s.trap for s in stats] == [0] * t, key
        assert [s.master_barriers for s in stats] == run["sim"]["master_barrier_entries"], key
        assert all(s.dynamic_allocs == s.dynamic_frees for s in stats), key
        if all(len(r.captures) <= pe for r in prog.regions):
            assert all(s.dynamic_allocs == 0 for s in stats), key
        checked += 1
    assert checked == 80


@pytest.mark.gpu
def test_gpu_runaway_programs_hit_the_step_limit():
    """SimulatorTests.cpp:142-148 ("runaway launches hit the step limit"): a
    program whose thread runs more operations than the limit traps with the
    reference's string and the team still terminates; the default limit
    (SimOptions::StepLimit, 20M) leaves the reference's outputs intact."""
    import torch
    from paper_1711_10413_b200 import _lib as L
    p = next(x for x in G.load("corpus") if x["stem"] == "arrays_1")  # a 96-trip loop
    t, w, run = launches(p)[0]
    prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
    bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
            for _, sz, init in prog.buffers]
    out = PG.run_program(prog, bufs, step_limit=50)
    st = out.team_stats()
    assert all(s.trap == L.TRAP_STEP_LIMIT for s in st)
    assert L.trap_reason(L.TRAP_STEP_LIMIT) == "step limit exceeded"
    bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
            for _, sz, init in prog.buffers]
    out = PG.run_program(prog, bufs)
    assert [s.trap for s in out.team_stats()] == [0] * t
    for (name, _, _), b in zip(prog.buffers, bufs):
        assert b.cpu().tolist() == run["sim"]["globals"][name]


@pytest.mark.gpu
def test_gpu_program_launches_replay_from_a_cuda_graph():
    """After one eager launch has staged a program's tables on a stream, the
    same launch issues no table copy and can be captured into a CUDA graph;
    every replay is one more run of the program (two_regions adds c to a[]
    twice per run).  Capturing a program whose tables are not staged is
    refused instead of recording a copy from freed host memory."""
    import torch
    p = next(x for x in G.load("corpus") if x["stem"] == "two_regions")
    t, w, run = launches(p)[0]
    prog = PG.compile_program(p["ast"], our_layouts(p), p["kernel"], t, w)
    s = torch.cuda.Stream()
    buf = torch.zeros(prog.buffers[0][1], dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s):
        PG.run_program(prog, [buf], stream=s)
    s.synchronize()
    one = buf.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        PG.run_program(prog, [buf], stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert buf.cpu().tolist() == (one * 4).cpu().tolist()
    # a different program (other tables) cannot be captured before it is staged
    p2 = next(x for x in G.load("corpus") if x["stem"] == "shared_scalar")
    t2, w2, _ = launches(p2)[0]
    prog2 = PG.compile_program(p2["ast"], our_layouts(p2), p2["kernel"], t2, w2)
    buf2 = torch.zeros(prog2.buffers[0][1], dtype=torch.int32, device="cuda")
    g2 = torch.cuda.CUDAGraph()
    from paper_1711_10413_b200 import _lib as L
    with pytest.raises(L.OmpdsError):
        with torch.cuda.graph(g2, stream=s):
            PG.run_program(prog2, [buf2], stream=s)
