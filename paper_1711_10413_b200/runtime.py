"""Host mirror of ``omplab::TeamRuntime`` (proj/include/omplab/DeviceRuntime.h:81-119).

Same names, argument meaning and error behaviour as the reference class:
every operation returns an :class:`RtResult` (``ok`` / ``trap_reason`` with the
reference's exact strings), nothing raises on a protocol violation.  The
operations execute on the GPU: each instance owns one team handle
(``ompds_team_create``) whose state lives in device memory, and each call
runs the team's ``__device__`` protocol function once -- the same state
machine the generic-mode kernels inline (csrc/ompds_device.cuh) -- so this
class is a thin, synchronous view of the device runtime, not a host
re-implementation.  ``replay`` runs a whole call script in one launch
(``ompds_rt_replay``), for the recorded-script parity tests.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

from . import _lib as L

DEFAULT_PREALLOC_ENTRIES = L.DEFAULT_PREALLOC_ENTRIES
SHARED_ARG_ENTRY_BYTES = L.SHARED_ARG_ENTRY_BYTES
RUNTIME_PRIVATE_BYTES = L.RUNTIME_PRIVATE_BYTES

MASTER = L.ROLE_MASTER
WORKER = L.ROLE_WORKER


def dynamic_args_bytes(nargs: int, prealloc_entries: int = DEFAULT_PREALLOC_ENTRIES) -> int:
    """DeviceRuntime.h:35-38 -- bytes a region allocates outside the window."""
    return int(L.lib().ompds_dynamic_args_bytes(nargs, prealloc_entries))


def trap_reason(code: int) -> str:
    return L.lib().ompds_trap_reason(code).decode()


@dataclass
class RuntimeConfig:  # DeviceRuntime.h:40-43
    prealloc_entries: int = DEFAULT_PREALLOC_ENTRIES
    fail_dynamic_alloc: bool = False


@dataclass
class RtResult:  # DeviceRuntime.h:56-62
    ok: bool = True
    trap_reason: str = ""
    code: int = 0


@dataclass
class RuntimeEvent:  # DeviceRuntime.h:64-79
    kind: str
    fn: str = ""
    nargs: int = 0
    bytes: int = 0

    def str(self) -> str:  # DeviceRuntime.cpp:12-31
        k = self.kind
        if k == "init":
            return f"init workers={self.nargs}"
        if k == "prepare_prealloc":
            return f"prepare {self.fn} nargs={self.nargs} prealloc"
        if k == "prepare_dynamic":
            return f"prepare {self.fn} nargs={self.nargs} dynamic bytes={self.bytes}"
        if k == "fetch":
            return f"fetch {self.fn}"
        if k == "retire":
            return f"retire remaining={self.nargs}"
        if k == "dynamic_free":
            return f"free bytes={self.bytes}"
        if k == "deinit":
            return "deinit"
        return "?"


@dataclass
class ReplayOutcome:
    results: List[L.RtResult]
    events: List[L.Event]
    summary: L.RtSummary


def replay(calls: Sequence[Tuple[int, int, int]], prealloc_entries: int = DEFAULT_PREALLOC_ENTRIES,
           fail_dynamic_alloc: bool = False, max_events: int = 4096) -> ReplayOutcome:
    """Runs (op, role, arg) calls in order on the device runtime of one team."""
    lib = L.lib()
    n = len(calls)
    arr = (L.RtCall * max(n, 1))(*[L.RtCall(op, role, arg) for op, role, arg in calls])
    res = (L.RtResult * max(n, 1))()
    ev = (L.Event * max(max_events, 1))()
    summ = L.RtSummary()
    cfg = L.RuntimeConfig(prealloc_entries, 1 if fail_dynamic_alloc else 0)
    L.check(lib.ompds_rt_replay(C.byref(cfg), arr, n, res, ev, max_events, C.byref(summ)),
            "ompds_rt_replay")
    n_ev = min(summ.n_events, max_events)
    return ReplayOutcome(list(res[:n]), list(ev[:n_ev]), summ)


class SharedArgsAllocator:
    """DeviceRuntime.h:46-52: hooks for shared-args lists past the window.

    ``allocate(nbytes)`` returns a non-zero block address, or 0 when the heap
    is exhausted; ``release(addr)`` gets back exactly such an address.  The
    runtime only stages and compares list addresses, so any distinct
    non-zero integers will do (as in the reference's RecordingHeap)."""

    def allocate(self, nbytes: int) -> int:  # pragma: no cover - interface
        raise NotImplementedError

    def release(self, addr: int) -> None:  # pragma: no cover - interface
        raise NotImplementedError


class RecordingHeap(SharedArgsAllocator):
    """The reference's test heap (RuntimeTests.cpp:19-42): distinct
    addresses, live blocks by address, allocation / free counts."""

    def __init__(self, fail_all: bool = False, first: int = 0x1000):
        self.fail_all = fail_all
        self.next = first
        self.live_bytes = {}
        self.allocs = 0
        self.frees = 0

    def allocate(self, nbytes: int) -> int:
        if self.fail_all:
            return 0
        addr = self.next
        self.next += nbytes + 64
        self.live_bytes[addr] = nbytes
        self.allocs += 1
        return addr

    def release(self, addr: int) -> None:
        if addr not in self.live_bytes:
            raise AssertionError(f"release of an address that is not live: {addr:#x}")
        del self.live_bytes[addr]
        self.frees += 1


class TeamRuntime:
    """omplab::TeamRuntime(RuntimeConfig, PreallocBase, SharedArgsAllocator&)
    over one GPU-resident team handle (``ompds_team_*``).

    Every call runs the team's __device__ protocol function once (O(1) per
    call, no history replay).  ``heap`` is called where the reference calls
    it (DeviceRuntime.cpp:61-74, 108-121); by default a :class:`RecordingHeap`.
    Methods return what the reference's out-parameters carry: e.g.
    ``prepareParallel`` -> (RtResult, ArgsAddr).
    """

    def __init__(self, config: Optional[RuntimeConfig] = None, prealloc_base: int = 0x2000,
                 heap: Optional[SharedArgsAllocator] = None):
        self.config = config or RuntimeConfig()
        self.prealloc_base = prealloc_base
        self.heap = heap if heap is not None else RecordingHeap()
        self._fn_names: List[str] = []
        self._fn_ids = {}
        self._events: List[RuntimeEvent] = []
        self._summary = L.RtSummary()
        self._evbuf = (L.Event * 8)()  # reused by every call's log fetch
        self._evtotal = C.c_int32()
        heap_ref = self.heap
        # keep the ctypes trampolines alive as long as the handle
        self._alloc = L.AllocFn(lambda nbytes, _u: int(heap_ref.allocate(int(nbytes))))
        self._release = L.ReleaseFn(lambda addr, _u: heap_ref.release(int(addr)))
        cfg = L.RuntimeConfig(self.config.prealloc_entries,
                              1 if self.config.fail_dynamic_alloc else 0)
        h = C.c_void_p()
        L.check(L.lib().ompds_team_create(C.byref(cfg), prealloc_base, self._alloc,
                                          self._release, None, C.byref(h)), "ompds_team_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and L._lib is not None:
            L._lib.ompds_team_destroy(h)
            self._h = None

    # -- internals ---------------------------------------------------------
    def _done(self, status: int) -> RtResult:
        if status >= L.ERR_CUDA:
            L.check(status, "ompds_team")
        if status != 0:
            return RtResult(False, trap_reason(status), status)
        lib = L.lib()
        lib.ompds_team_summary(self._h, C.byref(self._summary))
        if self._summary.n_events <= len(self._events):
            return RtResult()  # nothing new in the log
        buf = self._evbuf
        total = self._evtotal
        while True:
            first = len(self._events)
            st = lib.ompds_team_events(self._h, first, buf, 8, C.byref(total))
            for e in buf[:max(0, min(8, total.value - first))]:
                fn = self._fn_names[e.fn] if 0 <= e.fn < len(self._fn_names) else ""
                self._events.append(RuntimeEvent(L.EVENT_KIND_NAMES[e.kind], fn, e.nargs,
                                                 e.bytes))
            if st != L.ERR_CAPACITY:
                break
        return RtResult()

    def _intern(self, fn: str) -> int:
        if fn not in self._fn_ids:
            self._fn_ids[fn] = len(self._fn_names)
            self._fn_names.append(fn)
        return self._fn_ids[fn]

    # -- the reference API -------------------------------------------------
    def kernelInit(self, role: int, worker_count: int) -> RtResult:
        return self._done(L.lib().ompds_team_kernel_init(self._h, role, worker_count))

    def prepareParallel(self, role: int, fn: str, nargs: int) -> Tuple[RtResult, int]:
        """Returns (RtResult, ArgsAddr)."""
        addr = C.c_uint64()
        res = self._done(L.lib().ompds_team_prepare_parallel(self._h, role, self._intern(fn),
                                                             nargs, C.byref(addr)))
        return res, (addr.value if res.ok else 0)

    def kernelParallel(self, role: int) -> Tuple[RtResult, str, int, bool]:
        """Returns (RtResult, WfName, ArgsAddr, Participate)."""
        fn, part, addr = C.c_int32(-1), C.c_int32(0), C.c_uint64()
        res = self._done(L.lib().ompds_team_kernel_parallel(self._h, role, C.byref(fn),
                                                            C.byref(addr), C.byref(part)))
        if not res.ok:
            return res, "", 0, False
        wf = self._fn_names[fn.value] if fn.value >= 0 else ""
        return res, wf, addr.value, bool(part.value)

    def endParallel(self, role: int) -> RtResult:
        return self._done(L.lib().ompds_team_end_parallel(self._h, role))

    def kernelDeinit(self, role: int) -> RtResult:
        return self._done(L.lib().ompds_team_kernel_deinit(self._h, role))

    # -- accessors (DeviceRuntime.h:97-102) --------------------------------
    def workerCount(self) -> int:
        return self._summary.workers

    def dynamicAllocs(self) -> int:
        return self._summary.dynamic_allocs

    def dynamicFrees(self) -> int:
        return self._summary.dynamic_frees

    def leakedBlocks(self) -> int:
        return self._summary.leaked_blocks

    def terminated(self) -> bool:
        return bool(self._summary.terminated)

    def events(self) -> List[RuntimeEvent]:
        return list(self._events)
