"""Generic-mode target-region launches (BASELINE.json configs 1, 2, 4, 5).

Thin wrappers over the C ABI that take torch CUDA tensors (torch is used for
device memory and streams only).  Each call launches one sm_100a kernel in
which every CTA is an OpenMP team running the data-sharing protocol:
kernel_init -> push the kernel depot on the master's data-sharing stack ->
sequential code -> prepare_parallel + publish &captures -> named-barrier
release -> workers fetch, get-shared-variables (warp-shuffle broadcast), run
the region, retire -> join -> ... -> kernel_deinit -> termination release.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import torch

from . import _lib as L

ELEM = {torch.int32: L.ELEM_I32, torch.float64: L.ELEM_F64}


@dataclass
class TeamStats:
    trap: int
    master_barriers: int
    barrier_releases: int
    regions: int
    dynamic_alloc_bytes: int
    dynamic_allocs: int
    dynamic_frees: int
    depot_in_smem: bool
    n_events: int
    depot_offset: int
    smem_bytes: int


STATS_DTYPE_BYTES = C.sizeof(L.TeamStats)
EVENT_BYTES = C.sizeof(L.Event)


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if not t.is_cuda:
            raise ValueError("device tensors required (there is no CPU path)")
        if not t.is_contiguous():
            raise ValueError("contiguous tensors required")


def make_launch(teams: int, workers: int, prealloc_entries: int = L.DEFAULT_PREALLOC_ENTRIES,
                fail_dynamic_alloc: bool = False, depot_capacity: int = -1,
                log_events: bool = False, max_events: int = 0,
                stream: Optional[torch.cuda.Stream] = None,
                list_allocator: int = L.LIST_SLAB, first_team: int = 0,
                total_teams: int = 0,
                barrier_arrivals: Optional[torch.Tensor] = None) -> L.Launch:
    cur = torch.cuda.current_stream()
    if stream is not None and stream.cuda_stream != cur.cuda_stream:
        # outputs/inputs prepared on the current stream must be ready first
        stream.wait_stream(cur)
    s = stream.cuda_stream if stream is not None else cur.cuda_stream
    if barrier_arrivals is not None:
        _require_cuda(barrier_arrivals)
        if barrier_arrivals.dtype != torch.int32 or \
                barrier_arrivals.numel() < teams * (workers + L.RESERVED_WARP):
            raise ValueError("barrier_arrivals: int32, teams x (workers + 32)")
    return L.Launch(teams, workers, prealloc_entries, 1 if fail_dynamic_alloc else 0,
                    depot_capacity, 1 if log_events else 0, max_events if log_events else 0,
                    C.c_void_p(s), list_allocator, first_team, total_teams, 0,
                    C.c_void_p(barrier_arrivals.data_ptr()) if barrier_arrivals is not None
                    else None)


def _used_on(stream: Optional[torch.cuda.Stream], *ts) -> None:
    """Buffers allocated on the current stream and written by a launch on a
    side stream: tell the caching allocator, so a buffer the caller drops
    is not handed out again while the launch still writes it."""
    if stream is None or stream.cuda_stream == torch.cuda.current_stream().cuda_stream:
        return
    for t in ts:
        if t is not None:
            t.record_stream(stream)


class Outputs:
    """Device buffers for per-team statistics and event logs."""

    def __init__(self, teams: int, device, max_events: int = 0):
        self.teams = teams
        self.max_events = max_events
        self.stats = torch.zeros(teams * STATS_DTYPE_BYTES, dtype=torch.uint8, device=device)
        self.events = (torch.zeros(max(teams * max_events, 1) * EVENT_BYTES, dtype=torch.uint8,
                                   device=device) if max_events else None)

    def used_on(self, stream: Optional[torch.cuda.Stream]) -> None:
        _used_on(stream, self.stats, self.events)

    def stats_ptr(self):
        return C.c_void_p(self.stats.data_ptr())

    def events_ptr(self):
        return C.c_void_p(self.events.data_ptr()) if self.events is not None else None

    def team_stats(self) -> List[TeamStats]:
        torch.cuda.synchronize(self.stats.device)  # the launch may be on another stream
        raw = bytes(self.stats.cpu().numpy().tobytes())
        arr = (L.TeamStats * self.teams).from_buffer_copy(raw)
        return [TeamStats(s.trap, s.master_barriers, s.barrier_releases, s.regions,
                          s.dynamic_alloc_bytes, s.dynamic_allocs, s.dynamic_frees,
                          bool(s.depot_in_smem), s.n_events, s.depot_offset, s.smem_bytes)
                for s in arr]

    def team_events(self, times: bool = False) -> List[List[tuple]]:
        """Per team: (kind, fn, nargs, bytes) in log order, the reference's
        RuntimeEvent fields; times=True appends the device time (ns)."""
        if self.events is None:
            return [[] for _ in range(self.teams)]
        stats = self.team_stats()
        raw = bytes(self.events.cpu().numpy().tobytes())
        arr = (L.Event * (self.teams * self.max_events)).from_buffer_copy(raw)
        out = []
        for t in range(self.teams):
            n = min(stats[t].n_events, self.max_events)
            base = t * self.max_events
            out.append([(L.EVENT_KIND_NAMES[e.kind], e.fn, e.nargs, e.bytes) +
                        ((e.t_ns,) if times else ())
                        for e in arr[base:base + n]])
        return out


def _require_team_array(a: torch.Tensor, teams: int, workers: int, kw) -> None:
    """a[] is indexed by the grid's team number: one element per worker of
    every team of the grid (total_teams when the launch is a team range)."""
    grid = max(kw.get("total_teams") or 0, kw.get("first_team", 0) + teams, teams)
    if a.numel() < grid * workers:
        raise ValueError(f"a needs {grid} x {workers} elements, has {a.numel()}")


def run_regions(a: torch.Tensor, teams: int, workers: int, regions: int, **kw) -> Outputs:
    """Config 1: ``regions`` parallel regions sharing 4 scalars per team."""
    _require_cuda(a)
    _require_team_array(a, teams, workers, kw)
    max_events = kw.pop("max_events", 0)
    out = Outputs(teams, a.device, max_events)
    launch = make_launch(teams, workers, log_events=max_events > 0, max_events=max_events, **kw)
    L.check(L.lib().ompds_run_regions(C.byref(launch), ELEM[a.dtype], regions,
                                      C.c_void_p(a.data_ptr()), out.stats_ptr(),
                                      out.events_ptr()), "ompds_run_regions")
    out.used_on(kw.get("stream"))
    return out


def run_shared_array(a: torch.Tensor, teams: int, workers: int,
                     d_init: Optional[torch.Tensor] = None, **kw) -> Outputs:
    """Config 2: d[256] in the depot, ``parallel for i: a[i] += d[i & 255]``."""
    _require_cuda(a)
    if d_init is not None:
        _require_cuda(d_init)
        if d_init.dtype != a.dtype or d_init.numel() != 256:
            raise ValueError("d_init: 256 elements of a's dtype")
    max_events = kw.pop("max_events", 0)
    out = Outputs(teams, a.device, max_events)
    launch = make_launch(teams, workers, log_events=max_events > 0, max_events=max_events, **kw)
    dp = C.c_void_p(d_init.data_ptr()) if d_init is not None else None
    L.check(L.lib().ompds_run_shared_array(C.byref(launch), ELEM[a.dtype], a.numel(),
                                           C.c_void_p(a.data_ptr()), dp, out.stats_ptr(),
                                           out.events_ptr()), "ompds_run_shared_array")
    out.used_on(kw.get("stream"))
    return out


@dataclass
class WarpStack:
    frame_in_smem: List[bool]
    frame_offset: List[int]
    status: int
    max_depth: int
    high_water: int


def run_nested(a: torch.Tensor, teams: int, workers: int, regions: int,
               warp_slot_bytes: int = 2048, warp_overflow_bytes: int = 4096,
               collect: bool = True, **kw):
    """Config 3: nested regions (depth 3) on per-warp data-sharing stacks.

    Returns (Outputs, per-team list of per-warp :class:`WarpStack`); with
    collect=False the launch is only enqueued (no wait, stacks None) -- for
    timing the kernel alone."""
    _require_cuda(a)
    _require_team_array(a, teams, workers, kw)
    max_events = kw.pop("max_events", 0)
    out = Outputs(teams, a.device, max_events)
    warps = (workers + 31) // 32
    ws = torch.zeros(teams * warps * C.sizeof(L.WarpStackStats), dtype=torch.uint8,
                     device=a.device)
    launch = make_launch(teams, workers, log_events=max_events > 0, max_events=max_events, **kw)
    L.check(L.lib().ompds_run_nested(C.byref(launch), ELEM[a.dtype], regions, warp_slot_bytes,
                                     warp_overflow_bytes, C.c_void_p(a.data_ptr()),
                                     out.stats_ptr(), C.c_void_p(ws.data_ptr()),
                                     out.events_ptr()), "ompds_run_nested")
    out.used_on(kw.get("stream"))
    _used_on(kw.get("stream"), ws)
    if not collect:
        return out, None
    torch.cuda.synchronize(a.device)  # the launch may be on another stream
    raw = bytes(ws.cpu().numpy().tobytes())
    arr = (L.WarpStackStats * (teams * warps)).from_buffer_copy(raw)
    stacks = [[WarpStack([bool(x) for x in s.frame_in_smem], list(s.frame_offset), s.status,
                         s.max_depth, s.high_water) for s in arr[t * warps:(t + 1) * warps]]
              for t in range(teams)]
    return out, stacks


def prepared_shared_array(a: torch.Tensor, teams: int, workers: int,
                          d_init: Optional[torch.Tensor] = None,
                          stream: Optional[torch.cuda.Stream] = None,
                          depot_capacity: int = -1):
    """A zero-argument callable that only issues the config-2 launch (all
    arguments marshalled up front), for timing without host overhead."""
    _require_cuda(a)
    launch = make_launch(teams, workers, stream=stream, depot_capacity=depot_capacity)
    dp = C.c_void_p(d_init.data_ptr()) if d_init is not None else None
    ap = C.c_void_p(a.data_ptr())
    fn = L.lib().ompds_run_shared_array
    elem, n = ELEM[a.dtype], a.numel()
    lref = C.byref(launch)

    def go():
        L.check(fn(lref, elem, n, ap, dp, None, None), "ompds_run_shared_array")
    go.launch = launch  # keep the struct alive
    return go


def coef_buffer(dtype: torch.dtype, coef) -> C.Array:
    if dtype == torch.float64:
        return (C.c_double * 8)(*[float(c) for c in coef])
    return (C.c_int32 * 8)(*[int(c) for c in coef])


def run_stream(x: torch.Tensor, y: torch.Tensor, coef, teams: int, workers: int,
               stats: bool = True, **kw) -> Optional[Outputs]:
    """Config 4: ``y = fma(c1, x, y) + (c2+...+c8)`` over all elements."""
    _require_cuda(x, y)
    if x.dtype != y.dtype or x.numel() != y.numel():
        raise ValueError("x and y: same dtype and length")
    max_events = kw.pop("max_events", 0)
    out = Outputs(teams, x.device, max_events) if stats else None
    launch = make_launch(teams, workers, log_events=max_events > 0, max_events=max_events, **kw)
    cb = coef_buffer(x.dtype, coef)
    L.check(L.lib().ompds_run_stream(C.byref(launch), ELEM[x.dtype], x.numel(),
                                     C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), cb,
                                     out.stats_ptr() if out else None,
                                     out.events_ptr() if out else None), "ompds_run_stream")
    if out is not None:
        out.used_on(kw.get("stream"))
    return out


def run_stream_host(x_host: torch.Tensor, y_host: torch.Tensor, coef, teams: int, workers: int,
                    x_dev: torch.Tensor, y_dev: torch.Tensor,
                    stream: Optional[torch.cuda.Stream] = None) -> None:
    """Config 4 end to end from host buffers (H2D, region, D2H, synchronise)."""
    launch = make_launch(teams, workers, stream=stream)
    cb = coef_buffer(x_host.dtype, coef)
    L.check(L.lib().ompds_run_stream_host(C.byref(launch), ELEM[x_host.dtype], x_host.numel(),
                                          C.c_void_p(x_host.data_ptr()),
                                          C.c_void_p(y_host.data_ptr()), cb,
                                          C.c_void_p(x_dev.data_ptr()),
                                          C.c_void_p(y_dev.data_ptr())), "ompds_run_stream_host")


def fill_uniform(t: torch.Tensor, seed: int, first: int = 0,
                 stream: Optional[torch.cuda.Stream] = None) -> None:
    _require_cuda(t)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    L.check(L.lib().ompds_fill_uniform(ELEM[t.dtype], C.c_void_p(t.data_ptr()), t.numel(),
                                       seed, first, C.c_void_p(s)), "ompds_fill_uniform")


def probe_overheads(iterations: int = 8192, frame_bytes: int = 40, max_depth: int = 2,
                    lanes: int = 32, seed: int = 0x5eed01ab,
                    stream: Optional[torch.cuda.Stream] = None) -> dict:
    """The runtime's building blocks on one SM (ompds_probe_overheads):
    cycles and ns per data-sharing stack push + pop pair -- frames in the
    smem slot / on the global chain, net of the same store + load at fixed
    addresses, and the bookkeeping's own dependent chain -- and per bare
    region handoff (release + join barriers).  Depths vary per iteration
    (1..max_depth from a hash of the iteration and `seed`)."""
    p = L.OverheadProbe(iterations, frame_bytes, lanes, max_depth, seed & 0xFFFFFFFF, 0)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    L.check(L.lib().ompds_probe_overheads(C.byref(p), C.c_void_p(s)), "ompds_probe_overheads")
    ns = 1e3 / p.sm_clock_mhz if p.sm_clock_mhz > 0 else float("nan")
    per_it = p.pairs / p.iterations  # pairs per iteration

    def pair(mode, base):
        return (mode - base) / per_it
    slot = pair(p.slot_cycles, p.smem_baseline_cycles)
    chain = pair(p.chain_cycles, p.global_baseline_cycles)
    book = pair(p.bookkeeping_cycles, p.bookkeeping_baseline_cycles)
    # what a frame on the chain costs against one in the slot, per pair (the
    # placement decision), including its store + load
    placement = pair(p.chain_cycles, p.slot_cycles)
    return {"iterations": p.iterations, "frame_bytes_per_lane": p.frame_bytes,
            "lanes": p.lanes, "max_depth": p.max_depth, "pairs_per_iteration": round(per_it, 4),
            "sm_clock_mhz": round(p.sm_clock_mhz, 1),
            "cycles_per_iteration": {
                "smem_baseline": round(p.smem_baseline_cycles, 2), "slot": round(p.slot_cycles, 2),
                "global_baseline": round(p.global_baseline_cycles, 2),
                "chain": round(p.chain_cycles, 2), "bookkeeping": round(p.bookkeeping_cycles, 2),
                "bookkeeping_baseline": round(p.bookkeeping_baseline_cycles, 2)},
            "push_pop_pair_slot_cycles": round(slot, 2),
            "push_pop_pair_slot_ns": round(slot * ns, 2),
            "push_pop_pair_chain_cycles": round(chain, 2),
            "push_pop_pair_chain_ns": round(chain * ns, 2),
            "push_pop_pair_bookkeeping_cycles": round(book, 2),
            "push_pop_pair_bookkeeping_ns": round(book * ns, 2),
            "chain_vs_slot_per_pair_cycles": round(placement, 2),
            "handoff_cycles": round(p.handoff_cycles, 2),
            "handoff_ns": round(p.handoff_cycles * ns, 2)}


def release_workspace(stream: Optional[torch.cuda.Stream] = None) -> None:
    """Frees the library's device workspace kept for `stream` on the current
    device (waits for the stream first); the next launch reallocates."""
    s = (stream or torch.cuda.current_stream()).cuda_stream
    L.check(L.lib().ompds_release_workspace(C.c_void_p(s)), "ompds_release_workspace")


def checksum(t: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> int:
    """Sum of the elements' bit patterns mod 2^64 (order independent, exact)."""
    _require_cuda(t)
    out = torch.zeros(1, dtype=torch.int64, device=t.device)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    L.check(L.lib().ompds_checksum(ELEM[t.dtype], C.c_void_p(t.data_ptr()), t.numel(),
                                   C.c_void_p(out.data_ptr()), C.c_void_p(s)), "ompds_checksum")
    (stream or torch.cuda.current_stream()).synchronize()
    return int(out.item()) & ((1 << 64) - 1)
