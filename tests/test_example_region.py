"""A user-defined region program (examples/reduction_region.cu) compiled
against the runtime headers: three parallel regions per team share kernel
locals by reference -- the workers' atomics on the shared `sum` / `cnt` are
what the master reads after each join, the master's write of `thr` between
the regions is what the second region's workers read, and the third region
uses an `omp barrier` among its workers before one of them totals the
per-warp partials in a shared array."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1711_10413_b200 import _lib as L
from paper_1711_10413_b200 import build as B


def lib():
    path = B.build_example()
    lb = C.CDLL(path)
    lb.example_reduction.argtypes = [C.POINTER(L.Launch), C.c_void_p, C.c_int64, C.c_void_p,
                                     C.c_void_p]
    lb.example_reduction.restype = C.c_int32
    lb.example_misdeclared.argtypes = [C.POINTER(L.Launch), C.c_int32, C.c_void_p, C.c_void_p]
    lb.example_misdeclared.restype = C.c_int32
    return lb


def test_example_library_exports_its_entry_point():
    lb = lib()
    assert hasattr(lb, "example_reduction")
    assert os.path.basename(B.EXAMPLE_LIB) == "libompds_example.so"


def _expected(x, teams):
    n = len(x)
    out = []
    for t in range(teams):
        lo, hi = n * t // teams, n * (t + 1) // teams
        s = int(x[lo:hi].astype(np.int64).sum())
        c = hi - lo
        thr = 0 if c == 0 else (abs(s) // c) * (1 if s >= 0 else -1)  # C division
        out += [s, int((x[lo:hi].astype(np.int64) > thr).sum()), s]
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("teams,workers,n", [(1, 32, 1000), (4, 96, 100_003), (296, 480, 1 << 22),
                                             (3, 1, 17)])
def test_example_region_program_matches_numpy(teams, workers, n):
    import torch
    from paper_1711_10413_b200 import regions as RG
    x = torch.empty(n, dtype=torch.int32, device="cuda")
    RG.fill_uniform(x, 0x5eed01ab)
    out = torch.zeros(3 * teams, dtype=torch.int64, device="cuda")
    res = RG.Outputs(teams, x.device, 0)
    launch = RG.make_launch(teams, workers)
    L.check(lib().example_reduction(C.byref(launch), C.c_void_p(x.data_ptr()), n,
                                    C.c_void_p(out.data_ptr()), res.stats_ptr()),
            "example_reduction")
    torch.cuda.synchronize()
    assert out.cpu().tolist() == _expected(x.cpu().numpy(), teams)
    for st in res.team_stats():
        # three regions: 6 master barriers, 7 releases; team region = the
        # 304-byte depot + 160 B window + 49 B runtime span
        assert (st.trap, st.master_barriers, st.barrier_releases, st.regions) == (0, 6, 7, 3)
        assert st.smem_bytes == 304 + 160 + 49 and st.depot_in_smem


def _nested_lib():
    lb = lib()
    lb.example_nested.argtypes = [C.POINTER(L.Launch), C.c_void_p, C.c_int32, C.c_int64,
                                  C.c_int64, C.c_void_p]
    lb.example_nested.restype = C.c_int32
    return lb


def test_example_library_exports_the_nested_program():
    assert hasattr(_nested_lib(), "example_nested")


@pytest.mark.gpu
@pytest.mark.parametrize("teams,workers,slot,ovf", [(1, 96, 4096, 4096), (37, 40, 4096, 4096),
                                                    (148, 96, 0, 8192), (5, 33, 1024, 8192)])
def test_example_nested_program_matches_the_config3_oracle(teams, workers, slot, ovf):
    """Nested regions through the device API (push_frame / pop_frame /
    parallel_serialized) compute the config-3 program exactly like the
    C oracle (orc_nested) -- frames in the warps' shared-memory slots, on
    the overflow chains, or spilling from one to the other."""
    import torch
    from oracle import oracle as O
    from paper_1711_10413_b200 import regions as RG
    regions = 4
    a = torch.zeros(teams * workers, dtype=torch.float64, device="cuda")
    res = RG.Outputs(teams, a.device, 0)
    launch = RG.make_launch(teams, workers)
    L.check(_nested_lib().example_nested(C.byref(launch), C.c_void_p(a.data_ptr()), regions,
                                         slot, ovf, res.stats_ptr()), "example_nested")
    torch.cuda.synchronize()
    want = np.zeros(teams * workers)
    O.lib().orc_nested(1, teams, workers, regions, O.ptr(want))
    assert all(s.trap == 0 for s in res.team_stats())
    assert np.array_equal(a.cpu().numpy(), want)


@pytest.mark.gpu
@pytest.mark.parametrize("workers", [32, 96])
def test_lean_refused_prepare_does_not_rerun_the_previous_region(workers):
    """The lean instantiation defers a region's return to Idle to the next
    staging store; a prepare it refuses (more entries than the launch
    declared) must still leave the workers nothing staged: region 0's body
    runs once per worker, the team traps, 2 handoffs per region reached."""
    import torch
    from paper_1711_10413_b200 import regions as RG
    teams = 3
    runs = torch.zeros(teams, dtype=torch.int64, device="cuda")
    res = RG.Outputs(teams, runs.device, 0)
    launch = RG.make_launch(teams, workers)
    # 25 entries: past the 20-entry window the lean launch was sized for
    L.check(lib().example_misdeclared(C.byref(launch), 25, C.c_void_p(runs.data_ptr()),
                                      res.stats_ptr()), "example_misdeclared")
    torch.cuda.synchronize()
    assert runs.cpu().tolist() == [workers] * teams
    for st in res.team_stats():
        assert st.trap == L.ERR_INVALID  # no list allocator in the lean launch
        assert st.regions == 1
        assert st.master_barriers == 4
    # a negative count: the reference's own trap, even though the state word
    # still shows region 0 staged (the lean completion is deferred)
    runs.zero_()
    L.check(lib().example_misdeclared(C.byref(launch), -1, C.c_void_p(runs.data_ptr()),
                                      res.stats_ptr()), "example_misdeclared")
    torch.cuda.synchronize()
    assert runs.cpu().tolist() == [workers] * teams
    assert all(st.trap == 8 and st.regions == 1  # OMPDS_TRAP_NEGATIVE_NARGS
               for st in res.team_stats())
    # a second region that fits the window: both regions run
    runs.zero_()
    L.check(lib().example_misdeclared(C.byref(launch), 1, C.c_void_p(runs.data_ptr()),
                                      res.stats_ptr()), "example_misdeclared")
    torch.cuda.synchronize()
    assert runs.cpu().tolist() == [2 * workers] * teams
    assert all(st.trap == 0 and st.regions == 2 for st in res.team_stats())
