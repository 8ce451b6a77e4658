"""ctypes binding of the C ABI in ``include/ompds.h``.

Loads the in-tree ``_build/libompds_b200.so`` (built by ``build.py`` /
``__graft_entry__.build()``).  There is no fallback: if the library is
missing this module raises, and every compute entry point reports
``OMPDS_ERR_CUDA`` when no GPU is usable.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OMPDS_LIB_PATH") or os.path.join(HERE, "_build", "libompds_b200.so")

# ---------------------------------------------------------------------------
# constants (ompds.h)
# ---------------------------------------------------------------------------
DEFAULT_PREALLOC_ENTRIES = 20
SHARED_ARG_ENTRY_BYTES = 8
RUNTIME_PRIVATE_BYTES = 49
RESERVED_WARP = 32

OK = 0
ERR_CUDA = 100
ERR_INVALID = 101
ERR_CAPACITY = 102

ROLE_MASTER, ROLE_WORKER = 0, 1
OP_KERNEL_INIT, OP_PREPARE_PARALLEL, OP_KERNEL_PARALLEL, OP_END_PARALLEL, OP_KERNEL_DEINIT = range(5)
ADDR_NULL, ADDR_PREALLOC, ADDR_DYNAMIC = range(3)
EV_INIT, EV_PREPARE_PREALLOC, EV_PREPARE_DYNAMIC, EV_FETCH, EV_RETIRE, EV_DYNAMIC_FREE, EV_DEINIT = range(7)
EVENT_KIND_NAMES = ["init", "prepare_prealloc", "prepare_dynamic", "fetch", "retire",
                    "dynamic_free", "deinit"]
VAR_ESCAPES, VAR_PINNED = 1, 2
PIPELINE_DEFAULT, PIPELINE_O0, PIPELINE_BAD_ORDER = range(3)
ELEM_I32, ELEM_F64 = 0, 1
TRAP_STACK_OVERFLOW, TRAP_STACK_UNDERFLOW, TRAP_OUT_OF_BOUNDS, TRAP_STEP_LIMIT = 18, 19, 20, 21
LIST_SLAB, LIST_MALLOC = 0, 1


class RuntimeConfig(C.Structure):
    _fields_ = [("prealloc_entries", C.c_int32), ("fail_dynamic_alloc", C.c_int32)]


class RtCall(C.Structure):
    _fields_ = [("op", C.c_int32), ("role", C.c_int32), ("arg", C.c_int64)]


class RtResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("addr_kind", C.c_int32), ("wf", C.c_int32),
                ("participate", C.c_int32), ("live_bytes", C.c_int64), ("heap_live", C.c_int64)]


class Event(C.Structure):
    _fields_ = [("kind", C.c_int32), ("fn", C.c_int32), ("nargs", C.c_int64), ("bytes", C.c_int64),
                ("t_ns", C.c_int64)]


class RtSummary(C.Structure):
    _fields_ = [("workers", C.c_int32), ("terminated", C.c_int32),
                ("dynamic_allocs", C.c_int64), ("dynamic_frees", C.c_int64),
                ("leaked_blocks", C.c_int64), ("n_events", C.c_int32), ("_pad", C.c_int32)]


class FrameVar(C.Structure):
    _fields_ = [("group", C.c_int32), ("func", C.c_int32), ("flags", C.c_uint32),
                ("def_pos", C.c_int32), ("bytes", C.c_int64), ("live_first", C.c_int32),
                ("live_last", C.c_int32)]


class DepotSlot(C.Structure):
    _fields_ = [("offset", C.c_int64), ("size", C.c_int64), ("align", C.c_int32),
                ("shared", C.c_int32), ("owner_begin", C.c_int32), ("n_owners", C.c_int32)]


class DepotLayout(C.Structure):
    _fields_ = [("total_local", C.c_int64), ("total_shared", C.c_int64),
                ("has_shared_depot", C.c_int32), ("slot_begin", C.c_int32),
                ("n_slots", C.c_int32), ("overlap_slot", C.c_int32)]


class GpuSpec(C.Structure):
    _fields_ = [("shared_bytes_per_sm", C.c_int64), ("registers_per_sm", C.c_int64),
                ("max_blocks_per_sm", C.c_int64), ("warp_size", C.c_int32),
                ("max_regs_per_thread", C.c_int32), ("max_threads_per_sm", C.c_int64),
                ("reserved_smem_per_block", C.c_int64), ("reg_alloc_unit", C.c_int32),
                ("reg_partitions", C.c_int32)]


class Occupancy(C.Structure):
    _fields_ = [("teams_by_regs", C.c_int64), ("teams_by_smem", C.c_int64),
                ("potential", C.c_int64), ("actual", C.c_int64), ("smem_used", C.c_int64)]


class Launch(C.Structure):
    _fields_ = [("teams", C.c_int32), ("workers", C.c_int32), ("prealloc_entries", C.c_int32),
                ("fail_dynamic_alloc", C.c_int32), ("depot_capacity", C.c_int64),
                ("log_events", C.c_int32), ("max_events", C.c_int32), ("stream", C.c_void_p),
                ("list_allocator", C.c_int32), ("first_team", C.c_int32),
                ("total_teams", C.c_int32), ("reserved0", C.c_int32),
                ("barrier_arrivals", C.c_void_p)]


class Manifest(C.Structure):
    _fields_ = [("kernel", C.c_char_p), ("teams", C.c_int32), ("workers", C.c_int32),
                ("prealloc_entries", C.c_int32), ("has_layout", C.c_int32),
                ("layout", C.POINTER(DepotLayout)), ("slots", C.POINTER(DepotSlot)),
                ("owners", C.POINTER(C.c_int32)), ("var_names", C.POINTER(C.c_char_p))]


class ManifestInfo(C.Structure):
    _fields_ = [("kernel", C.c_int64), ("teams", C.c_int32), ("workers", C.c_int32),
                ("total_local", C.c_int64), ("total_shared", C.c_int64),
                ("mirrored", C.c_int32), ("prealloc_entries", C.c_int32),
                ("stack_bytes", C.c_int64), ("prealloc_bytes", C.c_int64),
                ("runtime_bytes", C.c_int64), ("shared_footprint", C.c_int64),
                ("n_slots", C.c_int32), ("n_owners", C.c_int32)]


class OverheadProbe(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("frame_bytes", C.c_int32), ("lanes", C.c_int32),
                ("max_depth", C.c_int32), ("seed", C.c_uint32), ("reserved0", C.c_int32),
                ("sm_clock_mhz", C.c_double), ("pairs", C.c_double),
                ("smem_baseline_cycles", C.c_double), ("slot_cycles", C.c_double),
                ("global_baseline_cycles", C.c_double), ("chain_cycles", C.c_double),
                ("bookkeeping_cycles", C.c_double), ("bookkeeping_baseline_cycles", C.c_double),
                ("handoff_cycles", C.c_double)]


class TeamStats(C.Structure):
    _fields_ = [("trap", C.c_int32), ("master_barriers", C.c_int32),
                ("barrier_releases", C.c_int32), ("regions", C.c_int32),
                ("dynamic_alloc_bytes", C.c_int64), ("dynamic_allocs", C.c_int32),
                ("dynamic_frees", C.c_int32), ("depot_in_smem", C.c_int32),
                ("n_events", C.c_int32), ("depot_offset", C.c_int64), ("smem_bytes", C.c_int64)]


class WarpStackStats(C.Structure):
    _fields_ = [("frame_in_smem", C.c_int32 * 2), ("frame_offset", C.c_int64 * 2),
                ("status", C.c_int32), ("max_depth", C.c_int32), ("high_water", C.c_int64)]


class ProgVar(C.Structure):
    _fields_ = [("space", C.c_int32), ("index", C.c_int32), ("count", C.c_int32),
                ("_pad", C.c_int32)]


class ProgRegion(C.Structure):
    _fields_ = [("entry", C.c_int32), ("n_captures", C.c_int32), ("cap_begin", C.c_int32),
                ("parent", C.c_int32), ("frame_bytes", C.c_int32), ("flags", C.c_int32)]


REGION_GLOBALIZE = 1


class Program(C.Structure):
    _fields_ = [("code", C.POINTER(C.c_int32)), ("n_code", C.c_int64),
                ("vars", C.POINTER(ProgVar)), ("n_vars", C.c_int32), ("n_regions", C.c_int32),
                ("regions", C.POINTER(ProgRegion)), ("captures", C.POINTER(C.c_int32)),
                ("n_captures", C.c_int32), ("n_buffers", C.c_int32),
                ("buffers", C.POINTER(C.c_void_p)), ("total_shared", C.c_int64),
                ("total_local", C.c_int64), ("priv_bytes", C.c_int64),
                ("step_limit", C.c_int64), ("stack_slot_bytes", C.c_int64),
                ("stack_overflow_bytes", C.c_int64)]


AllocFn = C.CFUNCTYPE(C.c_uint64, C.c_int64, C.c_void_p)   # ompds_alloc_fn
ReleaseFn = C.CFUNCTYPE(None, C.c_uint64, C.c_void_p)        # ompds_release_fn

# Every symbol include/ompds.h declares, with its signature.
_P = C.c_void_p
_SIGS = {
    "ompds_trap_reason": (C.c_char_p, [C.c_int32]),
    "ompds_last_error": (C.c_char_p, []),
    "ompds_version": (C.c_uint32, []),
    "ompds_device_count": (C.c_int32, []),
    "ompds_release_workspace": (C.c_int32, [C.c_void_p]),
    "ompds_rt_replay": (C.c_int32, [C.POINTER(RuntimeConfig), C.POINTER(RtCall), C.c_int32,
                                     C.POINTER(RtResult), C.POINTER(Event), C.c_int32,
                                     C.POINTER(RtSummary)]),
    "ompds_team_create": (C.c_int32, [C.POINTER(RuntimeConfig), C.c_uint64, AllocFn, ReleaseFn,
                                       C.c_void_p, C.POINTER(C.c_void_p)]),
    "ompds_team_destroy": (C.c_int32, [C.c_void_p]),
    "ompds_team_kernel_init": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32]),
    "ompds_team_prepare_parallel": (C.c_int32, [C.c_void_p, C.c_int32, C.c_int32, C.c_int64,
                                                 C.POINTER(C.c_uint64)]),
    "ompds_team_kernel_parallel": (C.c_int32, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32),
                                                C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]),
    "ompds_team_end_parallel": (C.c_int32, [C.c_void_p, C.c_int32]),
    "ompds_team_kernel_deinit": (C.c_int32, [C.c_void_p, C.c_int32]),
    "ompds_team_summary": (C.c_int32, [C.c_void_p, C.POINTER(RtSummary)]),
    "ompds_team_events": (C.c_int32, [C.c_void_p, C.c_int32, C.POINTER(Event), C.c_int32,
                                       C.POINTER(C.c_int32)]),
    "ompds_dynamic_args_bytes": (C.c_int64, [C.c_int64, C.c_int32]),
    "ompds_layout_build": (C.c_int32, [C.POINTER(FrameVar), C.c_int32, C.c_int32, C.c_int32,
                                        C.POINTER(DepotLayout), C.POINTER(DepotSlot), C.c_int32,
                                        C.POINTER(C.c_int32), C.c_int32]),
    "ompds_shared_footprint": (C.c_int64, [C.c_int64, C.c_int32]),
    "ompds_manifest_write": (C.c_int32, [C.POINTER(Manifest), C.c_char_p, C.c_int64,
                                          C.POINTER(C.c_int64)]),
    "ompds_manifest_parse": (C.c_int32, [C.c_char_p, C.c_int64, C.POINTER(ManifestInfo),
                                          C.POINTER(DepotSlot), C.c_int32,
                                          C.POINTER(C.c_int64), C.c_int32, C.c_char_p,
                                          C.c_int64]),
    "ompds_gpu_spec_get": (C.c_int32, [C.c_char_p, C.POINTER(GpuSpec)]),
    "ompds_occupancy_for": (C.c_int32, [C.POINTER(GpuSpec), C.c_int64, C.c_int32, C.c_int32,
                                         C.POINTER(Occupancy)]),
    "ompds_max_regs_for_teams": (C.c_int64, [C.POINTER(GpuSpec), C.c_int64, C.c_int32]),
    "ompds_max_shared_vars": (C.c_int64, [C.POINTER(GpuSpec), C.c_int64]),
    "ompds_run_regions": (C.c_int32, [C.POINTER(Launch), C.c_int32, C.c_int32, _P, _P, _P]),
    "ompds_run_shared_array": (C.c_int32, [C.POINTER(Launch), C.c_int32, C.c_int64, _P, _P,
                                            _P, _P]),
    "ompds_run_stream": (C.c_int32, [C.POINTER(Launch), C.c_int32, C.c_int64, _P, _P, _P, _P,
                                      _P]),
    "ompds_run_nested": (C.c_int32, [C.POINTER(Launch), C.c_int32, C.c_int32, C.c_int64,
                                      C.c_int64, _P, _P, _P, _P]),
    "ompds_program_verify": (C.c_int32, [C.POINTER(Program)]),
    "ompds_run_program": (C.c_int32, [C.POINTER(Launch), C.POINTER(Program), _P, _P]),
    "ompds_run_stream_host": (C.c_int32, [C.POINTER(Launch), C.c_int32, C.c_int64, _P, _P, _P,
                                           _P, _P]),
    "ompds_fill_uniform": (C.c_int32, [C.c_int32, _P, C.c_int64, C.c_uint64, C.c_int64, _P]),
    "ompds_checksum": (C.c_int32, [C.c_int32, _P, C.c_int64, _P, _P]),
    "ompds_probe_overheads": (C.c_int32, [C.POINTER(OverheadProbe), _P]),
    "ompds_team_smem_bytes": (C.c_int64, [C.c_int64, C.c_int32]),
}

_lib = None


class OmpdsError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        detail = ""
        if _lib is not None:
            if code == ERR_CUDA:
                detail = _lib.ompds_last_error().decode()
            else:
                detail = _lib.ompds_trap_reason(code).decode()
        super().__init__(f"{where}: status {code}: {detail}")


def lib():
    """The loaded library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run paper_1711_10413_b200.build.build() "
                "(or __graft_entry__.build()) -- there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(code: int, where: str) -> None:
    if code != OK:
        raise OmpdsError(code, where)


def exported_symbols():
    return list(_SIGS)


def trap_reason(code: int) -> str:
    """The trap string of a status code (1..17: the reference's, byte for byte)."""
    return lib().ompds_trap_reason(code).decode()
