"""Frame-layout descriptors: ``DepotSlot`` / ``DepotLayout`` / ``FrameGroup``
(proj/include/omplab/IR.h:219-254) built by the C-ABI frame pipeline
(``ompds_layout_build``; LoweringPasses.cpp buildDepots :264-305,
lowerSharedFrames :345-380, colorStack :458-538, repackOffsets :556-593).

Also the descriptor exports the reference produces: the ``.sir`` frame block
(IRPrinter.cpp:191-218) and the manifest's depot section
(Compiler.cpp:112-155), and the layout audit (LoweringPasses.cpp:617-665).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

from . import _lib as L

PIPELINES = {"default": L.PIPELINE_DEFAULT, "o0": L.PIPELINE_O0, "bad_order": L.PIPELINE_BAD_ORDER}


@dataclass
class FrameVar:
    """One alloca of the post-codegen module, in emission order."""
    name: str
    bytes: int
    group: int = 0
    func: int = 0
    escapes: bool = False
    pinned: bool = False
    def_pos: int = -1
    first: int = -1
    last: int = -1


@dataclass
class DepotSlot:  # IR.h:219-228
    offset: int
    size: int
    align: int = 8
    shared: bool = False
    owners: List[str] = field(default_factory=list)


@dataclass
class DepotLayout:  # IR.h:230-244
    slots: List[DepotSlot]
    total_local: int
    total_shared: int
    has_shared_depot: bool
    overlap_slot: int = -1

    def stack_bytes(self) -> int:
        return self.total_local

    def find_shared_local_overlap(self) -> Optional[str]:  # IR.cpp:228-242
        if self.overlap_slot < 0:
            return None
        s = self.slots[self.overlap_slot]
        return (f"slot {self.overlap_slot} at offset {s.offset} hosts"
                + "".join(f" %{o}" for o in s.owners))


@dataclass
class FrameGroup:  # IR.h:249-254
    root: str
    members: List[str]


def build_layouts(vars_: Sequence[FrameVar], n_groups: int,
                  pipeline: str = "default") -> List[DepotLayout]:
    """Runs the frame pipeline over ``vars_`` and returns one layout per group."""
    lib = L.lib()
    n = len(vars_)
    arr = (L.FrameVar * max(n, 1))()
    for i, v in enumerate(vars_):
        flags = (L.VAR_ESCAPES if v.escapes else 0) | (L.VAR_PINNED if v.pinned else 0)
        arr[i] = L.FrameVar(v.group, v.func, flags, v.def_pos, v.bytes, v.first, v.last)
    lays = (L.DepotLayout * max(n_groups, 1))()
    slots = (L.DepotSlot * max(n, 1))()
    owners = (C.c_int32 * max(n, 1))()
    L.check(lib.ompds_layout_build(arr, n, n_groups, PIPELINES[pipeline], lays, slots, max(n, 1),
                                   owners, max(n, 1)), "ompds_layout_build")
    out = []
    for g in range(n_groups):
        lay = lays[g]
        ss = []
        for k in range(lay.slot_begin, lay.slot_begin + lay.n_slots):
            s = slots[k]
            names = [vars_[owners[j]].name for j in range(s.owner_begin, s.owner_begin + s.n_owners)]
            ss.append(DepotSlot(s.offset, s.size, s.align, bool(s.shared), names))
        out.append(DepotLayout(ss, lay.total_local, lay.total_shared, bool(lay.has_shared_depot),
                               lay.overlap_slot))
    return out


def shared_footprint(total_shared: int, prealloc_entries: int = L.DEFAULT_PREALLOC_ENTRIES) -> int:
    """Simulator.cpp:281-284 / Occupancy.h:49-51: depot + window + runtime span."""
    return int(L.lib().ompds_shared_footprint(total_shared, prealloc_entries))


def audit(layouts: Sequence[DepotLayout], roots: Sequence[str]) -> List[Dict[str, str]]:
    """layout-overlap / mirror-mismatch findings (LoweringPasses.cpp:617-640)."""
    diags = []
    for lay, root in zip(layouts, roots):
        ov = lay.find_shared_local_overlap()
        if ov:
            diags.append({"rule": "layout-overlap", "message": ov, "function": root})
        if lay.total_shared != lay.total_local:
            diags.append({"rule": "mirror-mismatch",
                          "message": f"shared depot size {lay.total_shared} does not mirror "
                                     f"local depot size {lay.total_local}",
                          "function": root})
    return diags


def frame_block(group: FrameGroup, lay: DepotLayout) -> str:
    """The ``.sir`` frame block for one group (IRPrinter.cpp:191-218)."""
    out = [f"frame @{group.root} members [" + ", ".join(f"@{m}" for m in group.members) + "] {"]
    for i, s in enumerate(lay.slots):
        line = (f"  slot {i}: offset {s.offset}, size {s.size}, align {s.align}, "
                + ("shared" if s.shared else "local"))
        line += "".join(f", %{o}" for o in s.owners)
        out.append(line)
    out.append(f"  total {lay.total_local}" + (", mirrored" if lay.has_shared_depot else ""))
    out.append("}")
    return "\n".join(out) + "\n"


def parse_frame_blocks(text: str):
    """Parses every ``frame @root members [...] { ... }`` block of a ``.sir``
    module (IRParser.cpp:689-795) into (FrameGroup, DepotLayout) pairs."""
    import re
    out = []
    lines = text.splitlines()
    i = 0
    head = re.compile(r"^frame @(\S+) members \[(.*)\] \{$")
    slot = re.compile(r"^  slot (\d+): offset (\d+), size (\d+), align (\d+), (shared|local)(.*)$")
    tot = re.compile(r"^  total (\d+)(, mirrored)?$")
    while i < len(lines):
        m = head.match(lines[i])
        if not m:
            i += 1
            continue
        members = [x.strip().lstrip("@") for x in m.group(2).split(",") if x.strip()]
        slots = []
        i += 1
        while True:
            sm = slot.match(lines[i])
            if sm:
                if int(sm.group(1)) != len(slots):
                    raise ValueError(f"frame @{m.group(1)}: slot {sm.group(1)} out of order")
                owners = [o.strip().lstrip("%") for o in sm.group(6).split(",") if o.strip()]
                slots.append(DepotSlot(int(sm.group(2)), int(sm.group(3)), int(sm.group(4)),
                                       sm.group(5) == "shared", owners))
                i += 1
                continue
            tm = tot.match(lines[i])
            if not tm:
                raise ValueError(f"frame @{m.group(1)}: malformed line {lines[i]!r}")
            total = int(tm.group(1))
            if lines[i + 1] != "}":
                raise ValueError(f"frame @{m.group(1)}: missing closing brace")
            i += 2
            break
        ov = next((k for k, s in enumerate(slots) if s.shared and len(s.owners) > 1), -1)
        out.append((FrameGroup(m.group(1), members),
                    DepotLayout(slots, total, total, bool(tm.group(2)), ov)))
    return out


@dataclass
class Manifest:  # Compiler.cpp:112-155
    kernel: str
    teams: int
    workers: int
    depot: DepotLayout
    prealloc_entries: int
    prealloc_bytes: int
    runtime_bytes: int
    shared_footprint: int
    stack_bytes: int


def manifest_text(vars_: Sequence[FrameVar], n_groups: int, kernel: str, teams: int,
                  workers: int, pipeline: str = "default",
                  prealloc_entries: int = L.DEFAULT_PREALLOC_ENTRIES,
                  kernel_group: int = 0) -> str:
    """The reference compiler's manifest JSON (``manifestJson``, byte for
    byte) for the kernel frame group of ``vars_``, via the C ABI's frame
    pipeline and ``ompds_manifest_write``."""
    lib = L.lib()
    n = len(vars_)
    arr = (L.FrameVar * max(n, 1))()
    for i, v in enumerate(vars_):
        flags = (L.VAR_ESCAPES if v.escapes else 0) | (L.VAR_PINNED if v.pinned else 0)
        arr[i] = L.FrameVar(v.group, v.func, flags, v.def_pos, v.bytes, v.first, v.last)
    lays = (L.DepotLayout * max(n_groups, 1))()
    slots = (L.DepotSlot * max(n, 1))()
    owners = (C.c_int32 * max(n, 1))()
    L.check(lib.ompds_layout_build(arr, n, n_groups, PIPELINES[pipeline], lays, slots, max(n, 1),
                                   owners, max(n, 1)), "ompds_layout_build")
    names = (C.c_char_p * max(n, 1))(*[v.name.encode() for v in vars_])
    has = 0 <= kernel_group < n_groups
    m = L.Manifest(kernel.encode(), teams, workers, prealloc_entries, 1 if has else 0,
                   C.pointer(lays[kernel_group]) if has else None, slots, owners, names)
    size = C.c_int64()
    buf = C.create_string_buffer(4096)
    rc = lib.ompds_manifest_write(C.byref(m), buf, len(buf), C.byref(size))
    if rc == L.ERR_CAPACITY:
        buf = C.create_string_buffer(size.value + 1)
        rc = lib.ompds_manifest_write(C.byref(m), buf, len(buf), C.byref(size))
    L.check(rc, "ompds_manifest_write")
    return buf.raw[:size.value].decode()


def parse_manifest(text: str) -> Manifest:
    """Reads manifest JSON back (``ompds_manifest_parse``: any key order and
    whitespace; the reference's size laws are checked)."""
    lib = L.lib()
    raw = text.encode()
    info = L.ManifestInfo()
    cap_s, cap_o, cap_n = 64, 256, 1 << 14
    for _ in range(2):
        slots = (L.DepotSlot * cap_s)()
        onames = (C.c_int64 * cap_o)()
        names = C.create_string_buffer(cap_n)
        rc = lib.ompds_manifest_parse(raw, len(raw), C.byref(info), slots, cap_s, onames, cap_o,
                                      names, cap_n)
        if rc != L.ERR_CAPACITY:
            break
        cap_s, cap_o, cap_n = max(info.n_slots, 1), max(info.n_owners, 1), len(raw) + 1
    L.check(rc, "ompds_manifest_parse")

    def name_at(off):
        end = names.raw.index(b"\0", off)
        return names.raw[off:end].decode()
    ss = []
    for k in range(info.n_slots):
        s = slots[k]
        ss.append(DepotSlot(s.offset, s.size, s.align, bool(s.shared),
                            [name_at(onames[j]) for j in range(s.owner_begin,
                                                               s.owner_begin + s.n_owners)]))
    depot = DepotLayout(ss, info.total_local, info.total_shared, bool(info.mirrored))
    return Manifest(name_at(info.kernel), info.teams, info.workers, depot, info.prealloc_entries,
                    info.prealloc_bytes, info.runtime_bytes, info.shared_footprint,
                    info.stack_bytes)


def manifest_depot(lay: DepotLayout, prealloc_entries: int = L.DEFAULT_PREALLOC_ENTRIES) -> dict:
    """The depot part of the reference manifest (Compiler.cpp:112-155)."""
    return {
        "depot": {
            "slots": [{"offset": s.offset, "size": s.size, "align": s.align, "shared": s.shared,
                       "owners": list(s.owners)} for s in lay.slots],
            "total_local": lay.total_local,
            "total_shared": lay.total_shared,
            "mirrored": lay.has_shared_depot,
        },
        "stack_bytes": lay.total_local,
        "prealloc_entries": prealloc_entries,
        "prealloc_bytes": prealloc_entries * L.SHARED_ARG_ENTRY_BYTES,
        "runtime_bytes": L.RUNTIME_PRIVATE_BYTES,
        "shared_footprint": shared_footprint(lay.total_shared, prealloc_entries),
    }
