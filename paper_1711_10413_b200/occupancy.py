"""Shared-memory occupancy model (proj/include/omplab/Occupancy.h,
proj/src/Occupancy.cpp) over the C ABI, plus a ``b200`` device row.

The per-team footprint is the team region the sm_100a kernels actually
allocate as dynamic shared memory: depot + 8*PreallocEntries + 49 bytes.
For ``b200`` the model adds the 1 KB of shared memory the hardware reserves
per CTA and the 2048-threads-per-SM limit, which the K40/P100 model does not
have (their rows reproduce the paper's tables unchanged).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List

from . import _lib as L

SCALARS_FIXTURE_VARS = [1, 2, 4, 8, 16, 32, 64]  # Occupancy.cpp:38
ARRAYS_FIXTURE_VARS = [1, 2, 3, 4]               # Occupancy.cpp:39
MAX_VARS_TEAM_POINTS = [16, 15, 14, 13, 12, 8, 4, 2, 1]  # Occupancy.cpp:40
FIXTURE_THREADS_PER_TEAM = 128                   # Occupancy.h:59
# Register counts the paper measured for the fixture kernels (Occupancy.cpp:63-75).
_K40_SCALAR_REGS = [36, 36, 36, 36, 40, 72, 136]
_P100_SCALAR_REGS = [31, 31, 31, 31, 40, 71, 135]
KNOWN_GPUS = ["k40-16k", "k40-32k", "k40-48k", "p100", "b200"]


@dataclass
class OccupancyResult:
    teams_by_regs: int
    teams_by_smem: int
    potential: int
    actual: int
    smem_used: int


def gpu_spec(name: str) -> L.GpuSpec:
    g = L.GpuSpec()
    L.check(L.lib().ompds_gpu_spec_get(name.encode(), C.byref(g)), f"gpu_spec({name})")
    return g


def occupancy_for(gpu: str, footprint: int, regs: int, threads: int) -> OccupancyResult:
    o = L.Occupancy()
    g = gpu_spec(gpu)
    L.check(L.lib().ompds_occupancy_for(C.byref(g), footprint, regs, threads, C.byref(o)),
            "ompds_occupancy_for")
    return OccupancyResult(o.teams_by_regs, o.teams_by_smem, o.potential, o.actual, o.smem_used)


def max_regs_for_teams(gpu: str, teams: int, threads: int = FIXTURE_THREADS_PER_TEAM) -> int:
    g = gpu_spec(gpu)
    return int(L.lib().ompds_max_regs_for_teams(C.byref(g), teams, threads))


def max_shared_vars(gpu: str, teams: int) -> int:
    g = gpu_spec(gpu)
    return int(L.lib().ompds_max_shared_vars(C.byref(g), teams))


def _footprint(depot: int) -> int:
    return int(L.lib().ompds_shared_footprint(depot, L.DEFAULT_PREALLOC_ENTRIES))


def scalars_fixture_depot(n: int) -> int:  # Occupancy.cpp:42-49
    return 8 * n + 16


def arrays_fixture_depot(k: int) -> int:  # Occupancy.cpp:51-58
    return 384 * k + 24


def scalars_fixture_regs(gpu: str, n: int) -> int:
    k40 = gpu.startswith("k40")
    if n in SCALARS_FIXTURE_VARS:
        i = SCALARS_FIXTURE_VARS.index(n)
        return _K40_SCALAR_REGS[i] if k40 else _P100_SCALAR_REGS[i]
    return 36 if k40 else 31


def arrays_fixture_regs(gpu: str, k: int) -> int:
    return 36 if gpu.startswith("k40") else 30


def dynamic_args_bytes(n: int) -> int:
    return int(L.lib().ompds_dynamic_args_bytes(n, L.DEFAULT_PREALLOC_ENTRIES))


def footprint_scalars_csv() -> str:  # Occupancy.cpp:107-119
    rows = ["vars,stack,prealloc,private,total,source"]
    for n in [0] + SCALARS_FIXTURE_VARS:
        d = scalars_fixture_depot(n)
        rows.append(f"{n},{d},160,49,{_footprint(d)},{'model' if n == 0 else 'measured'}")
    return "\n".join(rows) + "\n"


def footprint_arrays_csv() -> str:  # Occupancy.cpp:121-130
    rows = ["arrays,stack,prealloc,private,total,source"]
    for k in ARRAYS_FIXTURE_VARS:
        d = arrays_fixture_depot(k)
        rows.append(f"{k},{d},160,49,{_footprint(d)},measured")
    return "\n".join(rows) + "\n"


def _occ_rows(gpu: str, vars_: List[int], depot, regs) -> str:
    rows = ["vars,regs,dynamic,total,teams_by_regs,teams_by_smem,potential,actual,smem_used"]
    for n in vars_:
        fp = _footprint(depot(n))
        r = regs(gpu, n)
        o = occupancy_for(gpu, fp, r, FIXTURE_THREADS_PER_TEAM)
        rows.append(f"{n},{r},{dynamic_args_bytes(n)},{fp},{o.teams_by_regs},{o.teams_by_smem},"
                    f"{o.potential},{o.actual},{o.smem_used}")
    return "\n".join(rows) + "\n"


def occupancy_scalars_csv(gpu: str) -> str:  # Occupancy.cpp:132-147
    return _occ_rows(gpu, SCALARS_FIXTURE_VARS, scalars_fixture_depot, scalars_fixture_regs)


def occupancy_arrays_csv(gpu: str) -> str:  # Occupancy.cpp:149-162
    s = _occ_rows(gpu, ARRAYS_FIXTURE_VARS, arrays_fixture_depot, arrays_fixture_regs)
    return s.replace("vars,regs", "arrays,regs", 1)


def ptxas_registers(log_path: str) -> dict:
    """Registers per thread of every kernel in a ``ptxas -v`` log (the
    in-tree build writes ``_build/ptxas.log``), keyed by mangled name."""
    out = {}
    name = None
    for line in open(log_path).read().splitlines():
        if "Compiling entry function" in line:
            name = line.split("'")[1]
        elif name and "Used" in line and "registers" in line:
            out[name] = int(line.split("Used")[1].split("registers")[0])
            name = None
    return out


# (kernel instantiation, what it runs, threads per team, team region bytes);
# "ELb1ELb0E" = the lean instantiation the config launchers use, "ELb0ELb0E" =
# the general one (event log / allocation hook / spilled lists / programs),
# "ELb1ELb1E" = the lean small-team one (64 threads, 32 teams/SM bound) a
# program opting into kSmallTeams gets for W <= 32
B200_KERNELS = [
    ("RegionsProgIiEELb1ELb1E", "config1 int (loop layout) lean small-team", 64, 56 + 160 + 49),
    ("RegionsProgIdEELb1ELb1E", "config1 int+f64 (loop layout) lean small-team", 64,
     56 + 160 + 49),
    ("RegionsProgIdEELb1ELb0E", "config1 lean W>32", 64, 56 + 160 + 49),
    ("RegionsProgIdEELb0ELb0E", "config1 general", 64, 56 + 160 + 49),
    ("SharedArrayProgWideIdEELb1E", "config2 f64 lean (32-byte units; a[] 32-byte aligned)", 512,
     2072 + 160 + 49),
    ("SharedArrayProgIdEELb1E", "config2 f64 lean (16-byte units)", 512, 2072 + 160 + 49),
    ("NestedProgIdEELb1E", "config3 f64 (2 KB warp slots x 3) lean", 128,
     96 * 0 + 304 + 3 * 2048),
    ("StreamProgIdEELb1E", "config4 f64 lean", 128, 80 + 160 + 49),
    ("ProgramProgELb0E", "reference programs (scalars_4 footprint)", 128, 48 + 160 + 49),
]


def b200_kernel_occupancy_csv(log_path: str) -> str:
    """The paper's occupancy table for our own sm_100a kernels on B200:
    registers from ptxas, footprint = the team region each launch requests."""
    regs = ptxas_registers(log_path)
    rows = ["kernel,config,regs,threads,footprint,teams_by_regs,teams_by_smem,potential,actual,"
            "smem_used,binding"]
    for key, cfg, thr, fp in B200_KERNELS:
        r = next((v for k, v in regs.items() if key in k), None)
        if r is None:
            continue
        o = occupancy_for("b200", fp, r, thr)
        binding = ("registers" if o.actual == o.teams_by_regs else
                   "shared memory" if o.actual == o.teams_by_smem else "threads/blocks")
        rows.append(f"{key},{cfg},{r},{thr},{fp},{o.teams_by_regs},{o.teams_by_smem},"
                    f"{o.potential},{o.actual},{o.smem_used},{binding}")
    return "\n".join(rows) + "\n"


def max_vars_csv(gpu: str) -> str:  # Occupancy.cpp:164-170
    rows = ["teams,max_regs,max_vars"]
    for t in MAX_VARS_TEAM_POINTS:
        rows.append(f"{t},{max_regs_for_teams(gpu, t)},{max_shared_vars(gpu, t)}")
    return "\n".join(rows) + "\n"
