"""Config 3: nested parallel regions on per-warp data-sharing stacks.

The reference rejects nested parallelism at parse time (DslParser.cpp:846-849;
pinned below from tests/golden/analogs.json), so the C oracle's restatement
 is the oracle: region values, and the placement of
every data-sharing frame (shared-memory slot vs global overflow chain,
offset, stack depth, high-water mark) predicted by orc_ds_stack."""
import ctypes as C

import numpy as np
import pytest

import golden_util as G
from oracle import oracle as O


def test_reference_rejects_nesting():
    p = next(x for x in G.load("analogs") if x["stem"] == "cfg3_nested")
    assert not p["compile_ok"]
    assert p["diags"][0]["rule"] == "nested-parallel-unsupported"


@pytest.mark.parametrize("regions", [1, 3])
def test_oracle_closed_form(regions):
    teams, w = 2, 40
    a = np.zeros(teams * w, dtype=np.int32)
    O.lib().orc_nested(0, teams, w, regions, O.ptr(a))
    want = np.array([sum(4 * i + 5 * c + 12 * (i % 8 + 1) + 1 for c in range(1, regions + 1))
                     for t in range(teams) for i in range(w)], dtype=np.int32)
    assert np.array_equal(a, want)
    b = np.zeros(teams * w)
    O.lib().orc_nested(1, teams, w, regions, O.ptr(b))
    assert np.array_equal(b, want.astype(np.float64))


def predict_stack(slot_cap, ovf_cap, l1, l2):
    """Per-warp frame placement for one region: push L1, push L2, pop, pop."""
    ops = [l1, l2, 0, 0]
    lanes = [32, 32, 32, 32]
    n = 4
    ins = (C.c_int32 * n)()
    off = (C.c_int64 * n)()
    md = C.c_int32()
    hw = C.c_int64()
    st = O.lib().orc_ds_stack(slot_cap, ovf_cap, (C.c_int64 * n)(*ops), (C.c_int32 * n)(*lanes),
                              n, ins, off, C.byref(md), C.byref(hw))
    return st, [ins[0], ins[1]], [off[0], off[1]], md.value, hw.value


@pytest.mark.gpu
@pytest.mark.parametrize("elem", [0, 1])
@pytest.mark.parametrize("slot", [2048, 1536, 1400, 1024, 600, 0])
def test_gpu_nested_values_and_stack_placement(elem, slot):
    import torch
    from paper_1711_10413_b200 import regions as RG
    teams, workers, regions = 5, 72, 3
    dt = torch.float64 if elem else torch.int32
    a = torch.zeros(teams * workers, dtype=dt, device="cuda")
    out, stacks = RG.run_nested(a, teams, workers, regions, warp_slot_bytes=slot,
                                warp_overflow_bytes=4096)
    want = np.zeros(teams * workers, dtype=np.float64 if elem else np.int32)
    O.lib().orc_nested(elem, teams, workers, regions, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want)
    l1 = 8 + 4 * (8 if elem else 4)   # frame group of L1: e (8-byte slot) + v[4]
    l2 = 8                            # frame group of L2: f
    # the launcher rounds slot capacities up to 16 bytes
    st, ins, off, md, hw = predict_stack((slot + 15) // 16 * 16, 4096, l1, l2)
    assert st == 0
    for t in range(teams):
        for ws in stacks[t]:
            assert ws.status == 0
            assert ws.frame_in_smem == [bool(x) for x in ins]
            assert ws.frame_offset == off
            assert (ws.max_depth, ws.high_water) == (md, hw)
    for s in out.team_stats():
        assert s.trap == 0 and s.regions == regions and s.master_barriers == 2 * regions
        depot = 8 + 8 * (8 if elem else 4) + 16
        region = depot + 209
        if slot:
            region = (region + 15) // 16 * 16 + 3 * ((slot + 15) // 16) * 16
        assert s.smem_bytes == region


@pytest.mark.gpu
@pytest.mark.parametrize("elem", [0, 1])
def test_gpu_nested_master_depot_on_the_global_chain(elem):
    """The nested program's two captures (c, s[]) read through list entries
    preloaded with the team state: with a zero-byte master slot they point
    into the team's global chain; the values equal the oracle."""
    import torch
    from paper_1711_10413_b200 import regions as RG
    teams, workers, regions = 7, 96, 4
    dt = torch.float64 if elem else torch.int32
    a = torch.zeros(teams * workers, dtype=dt, device="cuda")
    out, _ = RG.run_nested(a, teams, workers, regions, depot_capacity=0)
    want = np.zeros(teams * workers, dtype=np.float64 if elem else np.int32)
    O.lib().orc_nested(elem, teams, workers, regions, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want)
    assert all(s.trap == 0 and not s.depot_in_smem for s in out.team_stats())


@pytest.mark.gpu
@pytest.mark.parametrize("prealloc", [2, 3, 4])
def test_gpu_nested_small_windows(prealloc):
    """The nested program stages 2 captures; with a window of fewer than 4
    entries it runs on the general instantiation (no entry preload past the
    window), with 4 or more on the lean one; the values equal the oracle."""
    import torch
    from paper_1711_10413_b200 import regions as RG
    teams, workers, regions = 3, 64, 3
    a = torch.zeros(teams * workers, dtype=torch.float64, device="cuda")
    out, _ = RG.run_nested(a, teams, workers, regions, prealloc_entries=prealloc)
    want = np.zeros(teams * workers, dtype=np.float64)
    O.lib().orc_nested(1, teams, workers, regions, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want)
    assert all(s.trap == 0 and s.regions == regions for s in out.team_stats())


@pytest.mark.gpu
def test_gpu_nested_overflow_chain_exhausted():
    import torch
    from paper_1711_10413_b200 import regions as RG
    a = torch.zeros(2 * 64, dtype=torch.float64, device="cuda")
    out, stacks = RG.run_nested(a, 2, 64, 1, warp_slot_bytes=0, warp_overflow_bytes=512)
    st, *_ = predict_stack(0, 512, 40, 8)
    assert st == 18
    assert all(ws.status == 18 for t in stacks for ws in t)
    assert torch.count_nonzero(a).item() == 0  # the nested body never ran


@pytest.mark.gpu
def test_gpu_nested_stack_statistics_on_a_side_stream():
    """The warp statistics are written by each warp's last region; reading
    them must wait for a launch issued on another stream."""
    import torch
    from paper_1711_10413_b200 import regions as RG
    a = torch.zeros(96, dtype=torch.float64, device="cuda")
    _, stacks = RG.run_nested(a, 1, 96, 300, stream=torch.cuda.Stream())
    st, ins, off, md, hw = predict_stack(2048, 4096, 40, 8)
    for ws in stacks[0]:
        assert ws.status == 0 and ws.max_depth == md == 2
        assert ws.frame_in_smem == [bool(x) for x in ins] and ws.frame_offset == off


@pytest.mark.gpu
@pytest.mark.parametrize("elem", [0, 1])
def test_gpu_nested_whole_gpu_grid_matches_oracle(elem):
    """The bench's config-3 grid (8 teams per SM x 96 workers) for 20 nested
    regions: every element equals the oracle, every warp's stack matches."""
    import torch
    from paper_1711_10413_b200 import regions as RG
    teams = torch.cuda.get_device_properties(0).multi_processor_count * 8
    workers, regions = 96, 20
    dt = torch.float64 if elem else torch.int32
    a = torch.zeros(teams * workers, dtype=dt, device="cuda")
    out, stacks = RG.run_nested(a, teams, workers, regions)
    want = np.zeros(teams * workers, dtype=np.float64 if elem else np.int32)
    O.lib().orc_nested(elem, teams, workers, regions, O.ptr(want))
    assert np.array_equal(a.cpu().numpy(), want)
    assert all(ws.status == 0 and ws.frame_in_smem == [True, True]
               for t in stacks for ws in t)
    assert all(s.trap == 0 and s.regions == regions for s in out.team_stats())
