"""Host mirror of ``omplab::TeamRuntime`` (proj/include/omplab/DeviceRuntime.h:81-119).

Same names, argument meaning and error behaviour as the reference class:
every operation returns an :class:`RtResult` (``ok`` / ``trap_reason`` with the
reference's exact strings), nothing raises on a protocol violation.  The
operations execute on the GPU: each call replays the team's call history
through ``ompds_rt_replay`` -- the same ``__device__`` state machine the
generic-mode kernels inline (csrc/ompds_device.cuh) -- so this class is a
thin, synchronous view of the device runtime, not a host re-implementation.
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


class TeamRuntime:
    """omplab::TeamRuntime with the device runtime behind it.

    ``prealloc_base`` is reported as the args address of regions that fit the
    shared-memory window (the reference's PreallocBase); regions that spill
    report a distinct non-zero address per live block.
    """

    def __init__(self, config: Optional[RuntimeConfig] = None, prealloc_base: int = 0x2000):
        self.config = config or RuntimeConfig()
        self.prealloc_base = prealloc_base
        self._calls: List[Tuple[int, int, int]] = []
        self._fn_names: List[str] = []
        self._last: Optional[ReplayOutcome] = None

    # -- internals ---------------------------------------------------------
    def _run(self, op: int, role: int, arg: int) -> Tuple[RtResult, L.RtResult]:
        self._calls.append((op, role, int(arg)))
        out = replay(self._calls, self.config.prealloc_entries, self.config.fail_dynamic_alloc)
        self._last = out
        r = out.results[-1]
        if r.status != 0:
            self._calls.pop()  # a trap leaves the state untouched
            return RtResult(False, trap_reason(r.status), r.status), r
        return RtResult(), r

    def _addr(self, kind: int) -> int:
        if kind == L.ADDR_PREALLOC:
            return self.prealloc_base
        if kind == L.ADDR_DYNAMIC:
            return 0x4000_0000 + 0x100 * len(self._fn_names)
        return 0

    # -- the reference API -------------------------------------------------
    def kernelInit(self, role: int, worker_count: int) -> RtResult:
        return self._run(L.OP_KERNEL_INIT, role, worker_count)[0]

    def prepareParallel(self, role: int, fn: str, nargs: int) -> Tuple[RtResult, int]:
        """Returns (RtResult, ArgsAddr)."""
        res, raw = self._run(L.OP_PREPARE_PARALLEL, role, nargs)
        if not res.ok:
            return res, 0
        self._fn_names.append(fn)
        return res, self._addr(raw.addr_kind)

    def kernelParallel(self, role: int) -> Tuple[RtResult, str, int, bool]:
        """Returns (RtResult, WfName, ArgsAddr, Participate)."""
        res, raw = self._run(L.OP_KERNEL_PARALLEL, role, 0)
        if not res.ok:
            return res, "", 0, False
        wf = self._fn_names[raw.wf] if raw.wf >= 0 else ""
        return res, wf, self._addr(raw.addr_kind), bool(raw.participate)

    def endParallel(self, role: int) -> RtResult:
        return self._run(L.OP_END_PARALLEL, role, 0)[0]

    def kernelDeinit(self, role: int) -> RtResult:
        return self._run(L.OP_KERNEL_DEINIT, role, 0)[0]

    # -- accessors (DeviceRuntime.h:97-102) --------------------------------
    def _summary(self) -> L.RtSummary:
        if self._last is None or (self._last.results and self._last.results[-1].status):
            self._last = replay(self._calls, self.config.prealloc_entries,
                                self.config.fail_dynamic_alloc)
        return self._last.summary

    def workerCount(self) -> int:
        return self._summary().workers

    def dynamicAllocs(self) -> int:
        return self._summary().dynamic_allocs

    def dynamicFrees(self) -> int:
        return self._summary().dynamic_frees

    def leakedBlocks(self) -> int:
        return self._summary().leaked_blocks

    def terminated(self) -> bool:
        return bool(self._summary().terminated)

    def events(self) -> List[RuntimeEvent]:
        self._summary()
        out = []
        for e in self._last.events:
            kind = L.EVENT_KIND_NAMES[e.kind]
            fn = self._fn_names[e.fn] if e.fn >= 0 and e.fn < len(self._fn_names) else ""
            out.append(RuntimeEvent(kind, fn, e.nargs, e.bytes))
        return out
