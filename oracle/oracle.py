"""ctypes loader for the C oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libompds_oracle.so")
REF_SHIM = os.path.join(HERE, "_ref", "libomplab_ref.so")

_lib = None


def build() -> str:
    src = [os.path.join(HERE, "ompds_oracle.c"), os.path.join(HERE, "ompds_oracle.h"),
           os.path.join(os.path.dirname(HERE), "include", "ompds.h")]  # shared ABI structs
    if os.path.exists(LIB_PATH) and all(os.path.getmtime(s) <= os.path.getmtime(LIB_PATH)
                                        for s in src):
        return LIB_PATH
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        from paper_1711_10413_b200 import _lib as P  # struct shapes only
        L = C.CDLL(LIB_PATH)
        L.orc_rt_replay.argtypes = [C.POINTER(P.RuntimeConfig), C.POINTER(P.RtCall), C.c_int32,
                                    C.POINTER(P.RtResult), C.POINTER(P.Event), C.c_int32,
                                    C.POINTER(P.RtSummary)]
        L.orc_layout_build.argtypes = [C.POINTER(P.FrameVar), C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(P.DepotLayout), C.POINTER(P.DepotSlot),
                                       C.c_int32, C.POINTER(C.c_int32), C.c_int32]
        L.orc_occupancy_for.argtypes = [C.POINTER(P.GpuSpec), C.c_int64, C.c_int32, C.c_int32,
                                        C.POINTER(P.Occupancy)]
        L.orc_max_regs_for_teams.argtypes = [C.POINTER(P.GpuSpec), C.c_int64, C.c_int32]
        L.orc_max_regs_for_teams.restype = C.c_int64
        L.orc_max_shared_vars.argtypes = [C.POINTER(P.GpuSpec), C.c_int64]
        L.orc_max_shared_vars.restype = C.c_int64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_fill.argtypes = [C.c_int32, C.c_void_p, C.c_int64, C.c_uint64, C.c_int64]
        L.orc_checksum.argtypes = [C.c_int32, C.c_void_p, C.c_int64]
        L.orc_checksum.restype = C.c_uint64
        L.orc_regions.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
        L.orc_shared_array.argtypes = [C.c_int32, C.c_int64, C.c_void_p]
        L.orc_stream.argtypes = [C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_int32]
        L.orc_max_threads.restype = C.c_int32
        L.orc_stream_checksum.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_uint64,
                                          C.c_uint64, C.c_void_p, C.c_int32]
        L.orc_stream_checksum.restype = C.c_uint64
        L.orc_nested.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
        L.orc_ds_stack.argtypes = [C.c_int64, C.c_int64, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int64)]
        _lib = L
    return _lib


def ptr(a):
    """numpy array -> void*"""
    return C.c_void_p(a.ctypes.data)
