"""GPU parity of the generic-mode region kernels (configs 1, 2, 4) through the
C ABI: integer analogs bit-exact against the reference's own simulator output
(tests/golden/analogs.json), fp64 bodies against the C oracle (bit-exact: the
kernels and the oracle use the same explicit fma / add order; the stated
tolerance would be 1e-12 relative), runtime statistics against the
reference's barrier / allocation laws."""
import functools

import numpy as np
import pytest
import torch

import golden_util as G
from oracle import oracle as O
from paper_1711_10413_b200 import regions as RG

pytestmark = pytest.mark.gpu
DEV = "cuda"
RTOL_F64 = 1e-12  # north_star tolerance for fp64 bodies; we also require bit equality


def analog(stem):
    return next(p for p in G.load("analogs") if p["stem"] == stem)


def canon(events, fn_of=None):
    """Orders each region's worker events like the reference's round-robin
    simulator: fetches, then retires by decreasing `remaining`, then free."""
    out, seg = [], []
    order = {"fetch": 0, "retire": 1, "dynamic_free": 2}

    def flush():
        seg.sort(key=lambda e: (order[e[0]], -e[2] if e[0] == "retire" else 0))
        out.extend(seg)
        seg.clear()

    for e in events:
        kind, fn, nargs, nbytes = e
        fn = fn_of(fn) if fn_of else fn
        if kind in order:
            seg.append((kind, fn, nargs, nbytes))
        else:
            flush()
            out.append((kind, fn, nargs, nbytes))
    flush()
    return out


# --------------------------------------------------------------------------- config 1

@pytest.mark.parametrize("stem,regions", [("cfg1_analog", 1), ("cfg1_loop_analog", 5)])
def test_config1_int_analog_matches_reference(stem, regions):
    p = analog(stem)
    for run in p["runs"]:
        if run["teams"] != 1 or not G.race_free_run(run):
            continue
        w = run["workers"]
        a = torch.zeros(len(run["sim"]["globals"]["a"]), dtype=torch.int32, device=DEV)
        out = RG.run_regions(a, 1, w, regions, max_events=4096)
        assert a.cpu().tolist() == run["sim"]["globals"]["a"]
        st = out.team_stats()[0]
        assert st.trap == 0
        assert st.master_barriers == run["sim"]["master_barrier_entries"][0] == 2 * regions
        assert st.barrier_releases == run["sim"]["barrier_releases"][0] == 2 * regions + 1
        assert st.regions == regions and st.dynamic_allocs == 0 and st.depot_in_smem
        # team region = depot (layout) + 160 + 49, the reference footprint
        depot = next(l for l in p["layouts"] if l["root"] == p["kernel"])["total_shared"]
        assert st.smem_bytes == p["manifest"]["shared_footprint"] == depot + 209
        # event log == the reference TeamRuntime's, per region in canonical order
        ours = canon(out.team_events()[0])
        ref = run["sim"]["team_events"][0]
        names = {}
        ref_ev = []
        for k, fn, n, b in ref:
            if k.startswith("prepare"):
                names.setdefault(fn, len(names))
            ref_ev.append((k, names[fn] if fn else -1, n, b))
        assert ours == canon(ref_ev)


@pytest.mark.parametrize("teams,workers,regions", [(1, 32, 1), (3, 40, 7), (148, 96, 3),
                                                   (2, 992, 2), (5, 1, 4), (4, 40, 0),
                                                   (148 * 18, 32, 50),
                                                   (148 * 32, 32, 2000)])  # bench's whole-GPU grid
def test_config1_f64_and_int_match_oracle(teams, workers, regions):
    for dt, elem in ((torch.float64, 1), (torch.int32, 0)):
        a = torch.zeros(teams * workers, dtype=dt, device=DEV)
        out = RG.run_regions(a, teams, workers, regions)
        want = np.zeros(teams * workers, dtype=np.float64 if elem else np.int32)
        O.lib().orc_regions(elem, teams, workers, regions, O.ptr(want))
        assert np.array_equal(a.cpu().numpy(), want)
        for st in out.team_stats():
            assert (st.trap, st.master_barriers, st.barrier_releases, st.regions) == \
                (0, 2 * regions, 2 * regions + 1, regions)


@pytest.mark.gpu
@pytest.mark.parametrize("teams,workers,regions", [(1, 32, 5), (3, 40, 7), (148 * 20, 32, 20)])
@pytest.mark.parametrize("depot_capacity", [0, -1])
def test_config1_preloaded_entries_with_the_depot_in_smem_or_global(teams, workers, regions,
                                                                    depot_capacity):
    """Config 1 takes list entries 0-3 with the team state and dereferences
    the captures with broadcast loads (kPreloadEntries): with the master's
    depot in its smem slot the entries point into shared memory, with a
    zero-byte slot into the team's global chain -- the same values either way,
    on the small-team kernel (W = 32) and the general-size one (W = 40)."""
    for dt, elem in ((torch.float64, 1), (torch.int32, 0)):
        a = torch.zeros(teams * workers, dtype=dt, device=DEV)
        out = RG.run_regions(a, teams, workers, regions, depot_capacity=depot_capacity)
        want = np.zeros(teams * workers, dtype=np.float64 if elem else np.int32)
        O.lib().orc_regions(elem, teams, workers, regions, O.ptr(want))
        assert np.array_equal(a.cpu().numpy(), want)
        for st in out.team_stats():
            assert st.trap == 0 and st.regions == regions
            assert st.depot_in_smem == (depot_capacity != 0)


# --------------------------------------------------------------------------- config 2

def test_config2_int_analog_matches_reference():
    p = analog("cfg2_analog")
    for run in p["runs"]:
        for staged in (False, True):
            a = torch.zeros(256, dtype=torch.int32, device=DEV)
            d_init = (torch.arange(256, dtype=torch.int32, device=DEV) * 3 + 1) if staged else None
            out = RG.run_shared_array(a, run["teams"], run["workers"], d_init=d_init)
            assert a.cpu().tolist() == run["sim"]["globals"]["a"]
            for st in out.team_stats():
                assert st.trap == 0 and st.depot_in_smem
                assert st.smem_bytes == p["manifest"]["shared_footprint"] == 1048 + 209
                assert st.master_barriers == 2


@pytest.mark.parametrize("capacity", [-1, 1024, 0])
def test_config2_f64_placement_and_values(capacity):
    n = (1 << 20) + 3
    a = torch.empty(n, dtype=torch.float64, device=DEV)
    RG.fill_uniform(a, 0x5eed01ac)
    want = np.empty(n)
    O.lib().orc_fill(1, O.ptr(want), n, 0x5eed01ac, 0)
    assert np.array_equal(a.cpu().numpy(), want)
    d_init = torch.arange(256, dtype=torch.float64, device=DEV) * 3 + 1
    out = RG.run_shared_array(a, 148, 224, d_init=d_init, depot_capacity=capacity)
    O.lib().orc_shared_array(1, n, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want)
    in_smem = capacity < 0 or capacity >= 2072
    for st in out.team_stats():
        assert st.trap == 0
        assert st.depot_in_smem == in_smem  # slot vs global-overflow decision
        assert st.depot_offset == 0
        expect_depot = 2072 if capacity < 0 else capacity
        assert st.smem_bytes == expect_depot + 160 + 49


def test_config2_master_loop_equals_tma_staging():
    n = 4096 * 7 + 1
    a1 = torch.zeros(n, dtype=torch.float64, device=DEV)
    a2 = torch.zeros(n, dtype=torch.float64, device=DEV)
    RG.run_shared_array(a1, 16, 64)
    RG.run_shared_array(a2, 16, 64, d_init=torch.arange(256, dtype=torch.float64,
                                                        device=DEV) * 3 + 1)
    assert torch.equal(a1, a2)


# --------------------------------------------------------------------------- config 4

@pytest.mark.parametrize("n", [1024, 4096])
def test_config4_int_analog_matches_reference(n):
    p = analog(f"cfg4_analog_{n}")
    for run in p["runs"]:
        x = torch.tensor(p["inputs"]["x"], dtype=torch.int32, device=DEV)
        y = torch.tensor(p["inputs"]["y"], dtype=torch.int32, device=DEV)
        out = RG.run_stream(x, y, list(range(1, 9)), run["teams"], run["workers"],
                            max_events=4096)
        assert y.cpu().tolist() == run["sim"]["globals"]["y"]
        for t, st in enumerate(out.team_stats()):
            assert st.trap == 0 and st.master_barriers == 2 and st.barrier_releases == 3
            assert st.smem_bytes == p["manifest"]["shared_footprint"] == 80 + 209
            ours = canon(out.team_events()[t])
            ref = run["sim"]["team_events"][t] if "team_events" in run["sim"] else None
            if ref is not None:
                assert [e[0] for e in ours] == [e[0] for e in canon(
                    [(k, -1, nn, b) for k, _, nn, b in ref])]


def _f64_inputs(n, first=0):
    x = torch.empty(n, dtype=torch.float64, device=DEV)
    y = torch.empty(n, dtype=torch.float64, device=DEV)
    RG.fill_uniform(x, 0x5eed01ab, first)
    RG.fill_uniform(y, 0x5eed01ac, first)
    return x, y


COEF = [k / 8 for k in range(1, 9)]


@pytest.mark.parametrize("teams,workers", [(148, 224), (296, 992), (7, 33), (1, 1)])
def test_config4_f64_bitwise_vs_oracle(teams, workers):
    n = (1 << 20) + 5
    x, y = _f64_inputs(n)
    xs, ys = x.cpu().numpy().copy(), y.cpu().numpy().copy()
    out = RG.run_stream(x, y, COEF, teams, workers)
    O.lib().orc_stream(1, n, O.ptr(xs), O.ptr(ys), O.ptr(np.array(COEF)), 0)
    got = y.cpu().numpy()
    assert np.allclose(got, ys, rtol=RTOL_F64, atol=0)
    assert np.array_equal(got.view(np.uint64), ys.view(np.uint64))
    assert all(s.trap == 0 and s.regions == 1 for s in out.team_stats())


def test_config4_spilled_args_list_and_alloc_failure():
    n = 100_003
    x, y = _f64_inputs(n)
    y0 = y.clone()
    ref = y.clone()
    RG.run_stream(x, ref, COEF, 64, 96)
    out = RG.run_stream(x, y, COEF, 64, 96, prealloc_entries=2, max_events=1024)
    assert torch.equal(y, ref)
    for t, st in enumerate(out.team_stats()):
        assert (st.dynamic_allocs, st.dynamic_frees, st.dynamic_alloc_bytes) == (1, 1, 64)
        ev = canon(out.team_events()[t])
        assert ev[1] == ("prepare_dynamic", 0, 8, 64) and ev[-2] == ("dynamic_free", -1, 0, 64)
    y2 = y0.clone()
    out = RG.run_stream(x, y2, COEF, 64, 96, prealloc_entries=2, fail_dynamic_alloc=True)
    assert torch.equal(y2, y0)  # no region ran
    assert all(st.trap == 9 and st.regions == 0 for st in out.team_stats())


def test_config4_host_buffer_entry_point_matches_oracle():
    n = (1 << 24) + 5  # three pipelined chunks
    x, y = _f64_inputs(n)
    xh = x.cpu().pin_memory()
    yh = y.cpu().pin_memory()
    xs, ys = xh.numpy().copy(), yh.numpy().copy()
    xd = torch.empty_like(x)
    yd = torch.empty_like(y)
    RG.run_stream_host(xh, yh, COEF, 148, 992, xd, yd)
    O.lib().orc_stream(1, n, O.ptr(xs), O.ptr(ys), O.ptr(np.array(COEF)), 0)
    assert np.array_equal(yh.numpy().view(np.uint64), ys.view(np.uint64))


@functools.lru_cache(maxsize=None)
def _full_size_oracle_checksum(n):
    xs = np.empty(n)
    ys = np.empty(n)
    O.lib().orc_fill(1, O.ptr(xs), n, 0x5eed01ab, 0)
    O.lib().orc_fill(1, O.ptr(ys), n, 0x5eed01ac, 0)
    O.lib().orc_stream(1, n, O.ptr(xs), O.ptr(ys), O.ptr(np.array(COEF)), 0)
    return O.lib().orc_checksum(1, O.ptr(ys), n)


@pytest.mark.parametrize("teams,workers", [(296, 992), (148 * 7, 96)])  # 2nd: bench.py's grid
def test_config4_full_size_checksum_vs_oracle(teams, workers):
    n = 1 << 28
    x, y = _f64_inputs(n)
    RG.run_stream(x, y, COEF, teams, workers, stats=False)
    torch.cuda.synchronize()
    got = RG.checksum(y)
    del x, y
    assert got == _full_size_oracle_checksum(n)


# --------------------------------------------------------------------------- config 5

@pytest.mark.parametrize("world", [2, 4, 8])
def test_config5_shards_on_one_gpu_gather_to_whole_checksum(world):
    """Config 5 on one GPU: each shard g of the element range runs the region
    with its own teams on inputs generated for [lo, hi) (first = lo, as each
    rank of bench.py does); the shards' checksums summed mod 2^64 -- what the
    all-reduce gathers -- equal the oracle's whole-range checksum, and every
    element equals the unsharded oracle bit for bit."""
    from paper_1711_10413_b200 import sharding
    n = (1 << 22) + 13
    teams_total = 148 * 8
    parts, total = [], 0
    for g in range(world):
        lo, hi = sharding.shard_range(n, g, world)
        x, y = _f64_inputs(hi - lo, first=lo)
        teams = max(1, sharding.shard_range(teams_total, g, world)[1]
                    - sharding.shard_range(teams_total, g, world)[0])
        out = RG.run_stream(x, y, COEF, teams, 96)
        assert all(s.trap == 0 and s.regions == 1 for s in out.team_stats())
        total = (total + RG.checksum(y)) & sharding.MASK64
        parts.append(y.cpu().numpy())
    xs = np.empty(n)
    ys = np.empty(n)
    O.lib().orc_fill(1, O.ptr(xs), n, 0x5eed01ab, 0)
    O.lib().orc_fill(1, O.ptr(ys), n, 0x5eed01ac, 0)
    O.lib().orc_stream(1, n, O.ptr(xs), O.ptr(ys), O.ptr(np.array(COEF)), 0)
    assert total == O.lib().orc_checksum(1, O.ptr(ys), n)
    assert np.array_equal(np.concatenate(parts).view(np.uint64), ys.view(np.uint64))


# --------------------------------------------------------------------------- list allocators

@pytest.mark.parametrize("allocator", [0, 1])
@pytest.mark.parametrize("teams,workers,log", [(3, 40, True), (148, 32, False), (2, 96, False)])
def test_args_lists_past_the_window_slab_and_malloc(allocator, teams, workers, log):
    """4 captures with a 2-entry window: every region's list goes to global
    memory -- the team slab or device malloc (the paper's back-up scheme) --
    and is freed by the last retirement; values, barrier counts and the
    allocation statistics are the reference's either way."""
    from paper_1711_10413_b200 import _lib as L
    regions = 5
    a = torch.zeros(teams * workers, dtype=torch.int32, device=DEV)
    out = RG.run_regions(a, teams, workers, regions, prealloc_entries=2,
                         max_events=1024 if log else 0, list_allocator=allocator)
    want = np.zeros(teams * workers, dtype=np.int32)
    O.lib().orc_regions(0, teams, workers, regions, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want)
    for t, st in enumerate(out.team_stats()):
        assert (st.trap, st.master_barriers, st.barrier_releases, st.regions) == \
            (0, 2 * regions, 2 * regions + 1, regions)
        assert (st.dynamic_allocs, st.dynamic_frees, st.dynamic_alloc_bytes) == \
            (regions, regions, regions * 32)
        if log:
            ev = canon(out.team_events()[t])
            assert sum(1 for e in ev if e[0] == "prepare_dynamic") == regions
            assert sum(1 for e in ev if e[0] == "dynamic_free") == regions
    assert L.LIST_MALLOC == allocator or allocator == L.LIST_SLAB


# --------------------------------------------------------------------------- team ranges

@pytest.mark.parametrize("shards", [2, 3])
def test_team_grid_sharded_by_range_equals_one_launch(shards):
    """The north_star's multi-GPU partition for team-indexed programs: each
    shard launches teams [g*T/G, (g+1)*T/G) of a T-team grid (first_team,
    total_teams); omp_get_team_num() is the global team, so the shards
    together write exactly what one launch of T teams writes."""
    from paper_1711_10413_b200 import sharding
    teams, workers, regions = 7, 40, 3
    for dt, elem in ((torch.int32, 0), (torch.float64, 1)):
        a = torch.zeros(teams * workers, dtype=dt, device=DEV)
        for g in range(shards):
            lo, hi = sharding.shard_range(teams, g, shards)
            out = RG.run_regions(a, hi - lo, workers, regions, first_team=lo, total_teams=teams)
            assert all(s.trap == 0 and s.regions == regions for s in out.team_stats())
        want = np.zeros(teams * workers, dtype=np.float64 if elem else np.int32)
        O.lib().orc_regions(elem, teams, workers, regions, O.ptr(want))
        assert np.array_equal(a.cpu().numpy(), want)


# --------------------------------------------------------------------------- trace

@pytest.mark.parametrize("teams,workers", [(2, 32), (3, 96)])
def test_event_trace_times_follow_the_handoff_barriers(teams, workers):
    """The event log's device timestamps (ompds_event.t_ns, %globaltimer)
    respect what the barriers guarantee: init <= prepare(r) <= every fetch of
    r (release), every retire of r <= prepare(r+1) (join), last retire <=
    deinit -- per team; fetch/retire order across warps is free."""
    regions = 4
    a = torch.zeros(teams * workers, dtype=torch.int32, device=DEV)
    out = RG.run_regions(a, teams, workers, regions, max_events=2048)
    for ev in out.team_events(times=True):
        kinds = [e[0] for e in ev]
        assert kinds[0] == "init" and kinds[-1] == "deinit"
        t = [e[4] for e in ev]
        assert all(x > 0 for x in t)
        # split into regions at each prepare
        starts = [i for i, k in enumerate(kinds) if k.startswith("prepare")]
        assert len(starts) == regions
        bounds = starts + [len(ev) - 1]
        assert t[0] <= t[starts[0]]
        for r in range(regions):
            p, nxt = bounds[r], bounds[r + 1]
            body = range(p + 1, nxt)
            assert all(t[p] <= t[i] for i in body), r
            assert all(t[i] <= t[nxt] for i in body), r
            assert sum(1 for i in body if kinds[i] == "fetch") == workers
            assert sum(1 for i in body if kinds[i] == "retire") == workers


def test_concurrent_launches_on_two_streams_do_not_share_the_slab():
    """Args lists past the window live in the per-team slab of a workspace
    that is per (device, stream): two launches in flight on two streams,
    both spilling every region's list, still produce the oracle's values."""
    teams, workers, regions = 148, 64, 20
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    arrays = []
    for st in streams:
        a = torch.zeros(teams * workers, dtype=torch.int32, device=DEV)
        arrays.append(a)
    torch.cuda.synchronize()
    for st, a in zip(streams, arrays):
        outs.append(RG.run_regions(a, teams, workers, regions, prealloc_entries=2, stream=st))
    torch.cuda.synchronize()
    want = np.zeros(teams * workers, dtype=np.int32)
    O.lib().orc_regions(0, teams, workers, regions, O.ptr(want))
    for a, out in zip(arrays, outs):
        assert np.array_equal(a.cpu().numpy(), want)
        assert all((s.trap, s.dynamic_allocs, s.dynamic_frees) == (0, regions, regions)
                   for s in out.team_stats())


@pytest.mark.gpu
def test_release_workspace_then_relaunch_on_the_same_stream():
    """ompds_release_workspace frees a stream's slabs and chains after its
    work; the next launch on that stream reallocates and is exact, and
    releasing a stream the library never used is a no-op."""
    teams, workers, regions = 64, 40, 6
    st = torch.cuda.Stream()
    want = np.zeros(teams * workers, dtype=np.int32)
    O.lib().orc_regions(0, teams, workers, regions, O.ptr(want))
    for _ in range(2):
        a = torch.zeros(teams * workers, dtype=torch.int32, device=DEV)
        torch.cuda.synchronize()
        out = RG.run_regions(a, teams, workers, regions, prealloc_entries=2, stream=st)
        RG.release_workspace(st)
        assert np.array_equal(a.cpu().numpy(), want)
        assert all((s.trap, s.dynamic_allocs, s.dynamic_frees) == (0, regions, regions)
                   for s in out.team_stats())
    RG.release_workspace(torch.cuda.Stream())


@pytest.mark.gpu
def test_region_launches_replay_from_a_cuda_graph():
    """After one eager launch on a stream (which sizes the stream's
    workspace), the config-4 region and a config-1 grid with spilled args
    lists can be captured into a CUDA graph and replayed: every replay is one
    more region pass, bit-exact against the oracle."""
    n, teams, workers, replays = (1 << 18) + 3, 148, 96, 3
    x, y = _f64_inputs(n)
    s = torch.cuda.Stream()
    a = torch.zeros(8 * 40, dtype=torch.int32, device=DEV)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        RG.run_stream(x, y, COEF, teams, workers, stats=False, stream=s)  # eager warm-up
        RG.run_regions(a, 8, 40, 3, prealloc_entries=2, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        RG.run_stream(x, y, COEF, teams, workers, stats=False, stream=s)
        RG.run_regions(a, 8, 40, 3, prealloc_entries=2, stream=s)
    for _ in range(replays):
        g.replay()
    torch.cuda.synchronize()
    xs = np.empty(n)
    ys = np.empty(n)
    O.lib().orc_fill(1, O.ptr(xs), n, 0x5eed01ab, 0)
    O.lib().orc_fill(1, O.ptr(ys), n, 0x5eed01ac, 0)
    for _ in range(1 + replays):
        O.lib().orc_stream(1, n, O.ptr(xs), O.ptr(ys), O.ptr(np.array(COEF)), 0)
    assert np.array_equal(y.cpu().numpy().view(np.uint64), ys.view(np.uint64))
    want = np.zeros(8 * 40, dtype=np.int32)
    O.lib().orc_regions(0, 8, 40, 3, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want * (1 + replays))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,ox,oy", [(torch.float64, 1, 1), (torch.float64, 1, 0),
                                         (torch.float64, 0, 1), (torch.int32, 1, 1),
                                         (torch.int32, 2, 3), (torch.int32, 3, 0)])
def test_config4_views_not_16_byte_aligned(dtype, ox, oy):
    """Views starting mid-vector (x[1:], ...) take the element-wise variant
    of the region; results equal the oracle and the neighbours of the view
    are untouched."""
    n = 100_003
    elem = 1 if dtype == torch.float64 else 0
    bx = torch.empty(n + 4, dtype=dtype, device=DEV)
    by = torch.empty(n + 4, dtype=dtype, device=DEV)
    RG.fill_uniform(bx, 0x5eed01ab)
    RG.fill_uniform(by, 0x5eed01ac)
    before = by.cpu().numpy().copy()
    x, y = bx[ox:ox + n], by[oy:oy + n]
    coef = COEF if elem else [k + 1 for k in range(8)]
    out = RG.run_stream(x, y, coef, 148, 96)
    torch.cuda.synchronize()
    xs = bx.cpu().numpy()[ox:ox + n].copy()
    ys = before[oy:oy + n].copy()
    cf = np.array(coef, dtype=np.float64 if elem else np.int32)
    O.lib().orc_stream(elem, n, O.ptr(xs), O.ptr(ys), O.ptr(cf), 0)
    got = by.cpu().numpy()
    view = np.uint64 if elem else np.uint32
    assert np.array_equal(got[oy:oy + n].view(view), ys.view(view))
    assert np.array_equal(got[:oy], before[:oy]) and np.array_equal(got[oy + n:], before[oy + n:])
    assert all(s.trap == 0 and s.regions == 1 for s in out.team_stats())


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,off", [(torch.float64, 1), (torch.int32, 1), (torch.int32, 2)])
def test_config2_view_not_16_byte_aligned(dtype, off):
    n = 70_001
    base = torch.empty(n + 4, dtype=dtype, device=DEV)
    RG.fill_uniform(base, 0x5eed01ac)
    before = base.cpu().numpy().copy()
    d_init = torch.arange(256, dtype=dtype, device=DEV) * 3 + 1
    RG.run_shared_array(base[off:off + n], 37, 64, d_init=d_init)
    torch.cuda.synchronize()
    d = d_init.cpu().numpy()
    want = before.copy()
    if dtype == torch.float64:
        want[off:off + n] = before[off:off + n] + d[np.arange(n) & 255]
    else:
        want[off:off + n] = (before[off:off + n].astype(np.int64)
                             + d[np.arange(n) & 255]).astype(np.int32)
    got = base.cpu().numpy()
    assert np.array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("teams,workers", [(592, 224), (296, 480)])
def test_config2_bench_grid_full_size_matches_oracle(teams, workers):
    """Config 2 as the bench runs it (592 teams x 224 workers; the earlier
    296 x 480 grid too), 2^24 doubles, d[] staged by TMA."""
    n = 1 << 24
    a = torch.empty(n, dtype=torch.float64, device=DEV)
    RG.fill_uniform(a, 0x5eed01ac)
    d_init = torch.arange(256, dtype=torch.float64, device=DEV) * 3 + 1
    out = RG.run_shared_array(a, teams, workers, d_init=d_init)
    want = np.empty(n)
    O.lib().orc_fill(1, O.ptr(want), n, 0x5eed01ac, 0)
    O.lib().orc_shared_array(1, n, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want)
    assert all(s.trap == 0 and s.depot_in_smem and s.smem_bytes == 2281
               for s in out.team_stats())


@pytest.mark.gpu
@pytest.mark.parametrize("elem", [0, 1])
def test_config4_past_2_pow_31_elements_checksum_vs_oracle(elem):
    """Maximum-size edge: 2^31 + 5 elements (64-bit element, unit and
    block indices in the parallel-for), the bench grid; the oracle's
    checksum is accumulated over 2^26-element chunks regenerated from the
    same counter-based inputs, so host memory stays small."""
    n = (1 << 31) + 5
    dt, npdt = (torch.float64, np.float64) if elem else (torch.int32, np.int32)
    coef = COEF if elem else [k + 1 for k in range(8)]
    x = torch.empty(n, dtype=dt, device=DEV)
    y = torch.empty(n, dtype=dt, device=DEV)
    RG.fill_uniform(x, 0x5eed01ab)
    RG.fill_uniform(y, 0x5eed01ac)
    RG.run_stream(x, y, coef, 148 * 7, 96, stats=False)
    torch.cuda.synchronize()
    got = RG.checksum(y)
    del x, y
    torch.cuda.empty_cache()
    want, chunk = 0, 1 << 26
    xs = np.empty(chunk, dtype=npdt)
    ys = np.empty(chunk, dtype=npdt)
    cf = np.array(coef, dtype=npdt)
    for lo in range(0, n, chunk):
        m = min(chunk, n - lo)
        O.lib().orc_fill(elem, O.ptr(xs), m, 0x5eed01ab, lo)
        O.lib().orc_fill(elem, O.ptr(ys), m, 0x5eed01ac, lo)
        O.lib().orc_stream(elem, m, O.ptr(xs), O.ptr(ys), O.ptr(cf), 0)
        want = (want + O.lib().orc_checksum(elem, O.ptr(ys), m)) & ((1 << 64) - 1)
    assert got == want


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 2, 3, 17, 1023])
def test_config2_and_4_tiny_and_empty_ranges(n):
    """Empty and tiny element ranges (fewer elements than one warp, than the
    vector width): the region still runs once per team, the elements that
    exist equal the oracle."""
    x, y = _f64_inputs(n)
    out = RG.run_stream(x, y, COEF, 37, 96)
    xs = np.empty(n)
    ys = np.empty(n)
    O.lib().orc_fill(1, O.ptr(xs), n, 0x5eed01ab, 0)
    O.lib().orc_fill(1, O.ptr(ys), n, 0x5eed01ac, 0)
    O.lib().orc_stream(1, n, O.ptr(xs), O.ptr(ys), O.ptr(np.array(COEF)), 0)
    assert np.array_equal(y.cpu().numpy().view(np.uint64), ys.view(np.uint64))
    assert all(s.trap == 0 and s.regions == 1 for s in out.team_stats())
    a = torch.empty(n, dtype=torch.float64, device=DEV)
    RG.fill_uniform(a, 0x5eed01ac)
    out = RG.run_shared_array(a, 5, 64)
    want = np.empty(n)
    O.lib().orc_fill(1, O.ptr(want), n, 0x5eed01ac, 0)
    O.lib().orc_shared_array(1, n, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want)
    assert all(s.trap == 0 and s.regions == 1 for s in out.team_stats())


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,off", [(torch.float64, 1), (torch.int32, 1), (torch.int32, 3)])
def test_config2_d_init_view_not_16_byte_aligned(dtype, off):
    """d_init = base[off:off+256] is aligned to its element but not to 16
    bytes: the TMA bulk copy needs a 16-byte aligned source, so the reserved
    warp copies it instead; results equal the staged-by-TMA run."""
    n = 50_003
    base = torch.arange(300, dtype=dtype, device=DEV) * 3 + 1
    d_init = base[off:off + 256]
    assert d_init.data_ptr() % 16 != 0
    a = torch.zeros(n, dtype=dtype, device=DEV)
    out = RG.run_shared_array(a, 37, 64, d_init=d_init)
    torch.cuda.synchronize()
    d = d_init.cpu().numpy()
    want = d[np.arange(n) & 255]
    assert np.array_equal(a.cpu().numpy(), want)
    st = out.team_stats()
    assert all(s.trap == 0 and s.depot_in_smem for s in st)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,off_bytes", [(torch.float64, 0), (torch.float64, 16),
                                             (torch.float64, 48), (torch.int32, 16),
                                             (torch.int32, 32)])
def test_config2_32_and_16_byte_aligned_views(dtype, off_bytes):
    """a[] 32-byte aligned runs the 32-byte-unit body, 16-byte aligned the
    16-byte one; d[] arrives by TMA and is read after the transaction
    barrier while the first loads of a[] are in flight: both equal the
    oracle bit for bit."""
    n = 123_457
    esz = torch.tensor([], dtype=dtype).element_size()
    off = off_bytes // esz
    base = torch.empty(n + 16, dtype=dtype, device=DEV)
    assert base.data_ptr() % 256 == 0
    RG.fill_uniform(base, 0x5eed01ac)
    before = base.cpu().numpy().copy()
    d_init = torch.arange(256, dtype=dtype, device=DEV) * 3 + 1
    out = RG.run_shared_array(base[off:off + n], 2 * 148, 480, d_init=d_init)
    torch.cuda.synchronize()
    d = d_init.cpu().numpy()
    want = before.copy()
    if dtype == torch.float64:
        want[off:off + n] = before[off:off + n] + d[np.arange(n) & 255]
    else:
        want[off:off + n] = (before[off:off + n].astype(np.int64)
                             + d[np.arange(n) & 255]).astype(np.int32)
    assert np.array_equal(base.cpu().numpy().view(np.uint8), want.view(np.uint8))
    assert all(s.trap == 0 and s.depot_in_smem for s in out.team_stats())


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 5, 300, 4096])
def test_config2_tma_staging_with_idle_workers(n):
    """Fewer elements than workers: most workers never read d[] (never wait
    on the staging barrier); the master waits for the copy before its team
    retires, and the elements that exist equal the oracle."""
    a = torch.empty(n, dtype=torch.float64, device=DEV)
    RG.fill_uniform(a, 0x5eed01ac)
    d_init = torch.arange(256, dtype=torch.float64, device=DEV) * 3 + 1
    out = RG.run_shared_array(a, 2 * 148, 480, d_init=d_init)
    want = np.empty(n)
    O.lib().orc_fill(1, O.ptr(want), n, 0x5eed01ac, 0)
    O.lib().orc_shared_array(1, n, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want)
    assert all(s.trap == 0 and s.regions == 1 for s in out.team_stats())


@pytest.mark.gpu
def test_graph_survives_a_larger_eager_launch():
    """A graph captured after one eager launch keeps replaying correctly after
    a later, larger eager launch on the same stream grew the workspace: the
    superseded buffers are retired, not freed."""
    s = torch.cuda.Stream()
    a = torch.zeros(4 * 40, dtype=torch.int32, device=DEV)
    with torch.cuda.stream(s):
        RG.run_regions(a, 4, 40, 3, prealloc_entries=2, stream=s)  # sizes the slabs
    s.synchronize()
    a.zero_()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        RG.run_regions(a, 4, 40, 3, prealloc_entries=2, stream=s)
    # a much larger grid on the same stream: the team slabs grow
    big = torch.zeros(4096 * 40, dtype=torch.int32, device=DEV)
    with torch.cuda.stream(s):
        RG.run_regions(big, 4096, 40, 3, prealloc_entries=2, stream=s)
    s.synchronize()
    junk = [torch.full((1 << 20,), -1, dtype=torch.int32, device=DEV) for _ in range(8)]
    torch.cuda.synchronize()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    want = np.zeros(4 * 40, dtype=np.int32)
    O.lib().orc_regions(0, 4, 40, 3, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want * 2)
    want_big = np.zeros(4096 * 40, dtype=np.int32)
    O.lib().orc_regions(0, 4096, 40, 3, O.ptr(want_big))
    assert np.array_equal(big.cpu().numpy(), want_big)
    del junk
