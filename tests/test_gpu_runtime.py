"""GPU parity of the device runtime protocol (csrc/ompds_device.cuh) against
the reference TeamRuntime's recorded outcomes (tests/golden/runtime.json) and
the C oracle.  Calls go through the C ABI (ompds_rt_replay)."""
import ctypes as C
import random

import pytest

import golden_util as G
from oracle import oracle as O
from paper_1711_10413_b200 import _lib as P
from paper_1711_10413_b200 import runtime as R
from test_oracle_golden import _replay, check_script

pytestmark = pytest.mark.gpu


def test_device_runtime_matches_reference_scripts():
    scripts = G.load("runtime")
    for s in scripts:
        check_script(s, *_replay(P.lib().ompds_rt_replay, s))


def test_device_runtime_matches_oracle_on_long_fuzz():
    rng = random.Random(1234)
    for trial in range(60):
        calls = [(0, 0, rng.randint(1, 64))] if rng.random() < 0.9 else []
        for _ in range(rng.randint(50, 300)):
            op = rng.choice([1, 2, 2, 2, 3, 3, 3, 4])
            role = 0 if op in (1, 4) else 1
            if rng.random() < 0.05:
                role ^= 1
            arg = rng.randint(-1, 70) if op == 1 else 0
            calls.append((op, role, arg))
        pe = rng.choice([0, 1, 4, 20, 20, 20, 64])
        fail = rng.random() < 0.1
        script = {"calls": calls, "prealloc_entries": pe, "fail_dynamic_alloc": fail}
        a = _replay(P.lib().ompds_rt_replay, script)
        b = _replay(O.lib().orc_rt_replay, script)
        for x, y in zip(a[0], b[0]):
            assert (x.status, x.addr_kind, x.wf, x.participate, x.live_bytes, x.heap_live) == \
                (y.status, y.addr_kind, y.wf, y.participate, y.live_bytes, y.heap_live)
        assert [(e.kind, e.fn, e.nargs, e.bytes) for e in a[1]] == \
            [(e.kind, e.fn, e.nargs, e.bytes) for e in b[1]]


# proj/tests/RuntimeTests.cpp, through the TeamRuntime mirror -------------------

def live(workers=8, cfg=None, heap=None):
    rt = R.TeamRuntime(cfg or R.RuntimeConfig(), prealloc_base=0x2000, heap=heap)
    assert rt.kernelInit(R.MASTER, workers).ok
    return rt


def drain(rt):
    res, wf, addr, part = rt.kernelParallel(R.WORKER)
    assert res.ok and part
    assert rt.endParallel(R.WORKER).ok


def test_init_accepts_one_master_call_and_nothing_else():
    rt = R.TeamRuntime(R.RuntimeConfig(), 0x2000)
    assert not rt.kernelInit(R.WORKER, 8).ok
    assert not rt.kernelInit(R.MASTER, 0).ok
    assert rt.kernelInit(R.MASTER, 8).ok
    assert not rt.kernelInit(R.MASTER, 8).ok
    assert rt.workerCount() == 8


def test_small_capture_lists_use_the_preallocated_window():
    rt = live()
    for n in (0, 1, 19, 20):
        res, addr = rt.prepareParallel(R.MASTER, "wf", n)
        assert res.ok and addr == 0x2000
        drain(rt)
    assert rt.dynamicAllocs() == 0


def test_oversized_capture_lists_fall_back_to_global_memory():
    rt = live()
    for n, nbytes in ((21, 168), (32, 256), (64, 512), (128, 1024)):
        res, addr = rt.prepareParallel(R.MASTER, "wf", n)
        assert res.ok and addr != 0x2000
        assert rt.events()[-1].kind == "prepare_dynamic" and rt.events()[-1].bytes == nbytes
        drain(rt)
        assert rt.events()[-1].str() == f"free bytes={nbytes}"
    assert rt.dynamicAllocs() == 4 and rt.dynamicFrees() == 4 and rt.leakedBlocks() == 0


def test_window_boundary_is_exactly_the_entry_count():
    rt = live(cfg=R.RuntimeConfig(prealloc_entries=4))
    res, addr = rt.prepareParallel(R.MASTER, "wf", 4)
    assert res.ok and addr == 0x2000
    drain(rt)
    res, addr = rt.prepareParallel(R.MASTER, "wf", 5)
    assert res.ok and addr != 0x2000
    assert rt.events()[-1].bytes == 40


def test_failing_global_allocation_is_a_trap():
    rt = live(cfg=R.RuntimeConfig(fail_dynamic_alloc=True))
    res, _ = rt.prepareParallel(R.MASTER, "wf", 21)
    assert not res.ok and res.trap_reason == "shared-args-alloc-failed"


def test_termination_sentinel_and_event_order():
    rt = live()
    res, _ = rt.prepareParallel(R.MASTER, "region0", 21)
    assert res.ok
    res, wf, _, part = rt.kernelParallel(R.WORKER)
    assert wf == "region0"
    assert rt.endParallel(R.WORKER).ok
    assert rt.kernelDeinit(R.MASTER).ok
    res, wf, addr, part = rt.kernelParallel(R.WORKER)
    assert res.ok and wf == "" and addr == 0 and not part and rt.terminated()
    assert [e.kind for e in rt.events()] == ["init", "prepare_dynamic", "fetch", "retire",
                                             "dynamic_free", "deinit"]


def test_byte_law_for_every_count():
    rng = random.Random(1234)
    for _ in range(50):
        n = rng.randint(0, 128)
        rt = live()
        res, addr = rt.prepareParallel(R.MASTER, "wf", n)
        assert res.ok
        dyn = rt.events()[-1].bytes
        assert dyn == R.dynamic_args_bytes(n)
        assert (addr == 0x2000) == (n <= 20)


def test_allocator_sees_exactly_the_reference_calls():
    """The injected SharedArgsAllocator (RuntimeTests.cpp:19-42's
    RecordingHeap): allocate(8*nargs) once per spilled region, the list
    address returned is the allocator's block, release(that address) at the
    last retirement -- with 3 workers, only the third retire frees."""
    heap = R.RecordingHeap()
    rt = live(workers=3, heap=heap)
    res, addr = rt.prepareParallel(R.MASTER, "wf", 40)
    assert res.ok and heap.live_bytes == {addr: 320} and heap.allocs == 1
    for _ in range(3):
        res, wf, a, part = rt.kernelParallel(R.WORKER)
        assert res.ok and wf == "wf" and a == addr and part
    for k in range(3):
        assert rt.endParallel(R.WORKER).ok
        assert (addr in heap.live_bytes) == (k < 2)
    assert heap.frees == 1 and rt.leakedBlocks() == 0
    # FailDynamicAlloc never reaches the heap; an exhausted heap traps and
    # leaves the team Idle
    h2 = R.RecordingHeap()
    rt2 = live(cfg=R.RuntimeConfig(fail_dynamic_alloc=True), heap=h2)
    res, _ = rt2.prepareParallel(R.MASTER, "wf", 21)
    assert res.trap_reason == "shared-args-alloc-failed" and h2.allocs == 0
    h3 = R.RecordingHeap(fail_all=True)
    rt3 = live(heap=h3)
    res, _ = rt3.prepareParallel(R.MASTER, "wf", 21)
    assert res.trap_reason == "shared-args-alloc-failed"
    h3.fail_all = False
    res, addr = rt3.prepareParallel(R.MASTER, "wf", 21)
    assert res.ok and h3.live_bytes == {addr: 168}


def test_handle_calls_are_constant_time():
    """No history replay: the 1000th region costs what the 10th does."""
    import time
    rt = live(workers=1)

    def region():
        assert rt.prepareParallel(R.MASTER, "wf", 2)[0].ok
        assert rt.kernelParallel(R.WORKER)[0].ok
        assert rt.endParallel(R.WORKER).ok

    for _ in range(10):
        region()
    t0 = time.perf_counter()
    for _ in range(50):
        region()
    early = time.perf_counter() - t0
    for _ in range(900):
        region()
    t0 = time.perf_counter()
    for _ in range(50):
        region()
    late = time.perf_counter() - t0
    assert late < 3 * early, (early, late)
    assert len(rt.events()) == 1 + 3 * 1010


def test_handle_rejects_bad_arguments_and_traps_leave_state():
    """C-ABI edge cases of the team handle: an out-of-range role or work
    function id is OMPDS_ERR_INVALID before any launch; a trapped call
    leaves the phase, counters and event log exactly as they were."""
    import ctypes as C
    lib = P.lib()
    rt = live(workers=2)
    h = rt._h
    addr = C.c_uint64()
    assert lib.ompds_team_prepare_parallel(h, 7, 0, 1, C.byref(addr)) == P.ERR_INVALID
    assert lib.ompds_team_prepare_parallel(h, R.MASTER, 1 << 23, 1, C.byref(addr)) == \
        P.ERR_INVALID
    assert lib.ompds_team_prepare_parallel(h, R.MASTER, -1, 1, C.byref(addr)) == P.ERR_INVALID
    n_events = len(rt.events())
    # traps: fetch with nothing staged, end with nothing active, worker deinit
    assert rt.kernelParallel(R.WORKER)[0].trap_reason == \
        "protocol error: kernel_parallel with no staged region"
    assert rt.endParallel(R.WORKER).trap_reason == \
        "protocol error: end_parallel with no active region"
    assert rt.kernelDeinit(R.WORKER).trap_reason == \
        "protocol error: kernel_deinit from a worker thread"
    assert len(rt.events()) == n_events and not rt.terminated()
    # the largest work-function id (24-bit field in the state word) round-trips
    big = (1 << 23) - 1
    assert lib.ompds_team_prepare_parallel(h, R.MASTER, big, 3, C.byref(addr)) == 0
    fn = C.c_int32()
    part = C.c_int32()
    assert lib.ompds_team_kernel_parallel(h, R.WORKER, C.byref(fn), C.byref(addr),
                                          C.byref(part)) == 0
    assert fn.value == big and part.value == 1 and addr.value == 0x2000
