"""Shared helpers: run a frame-pipeline implementation over the golden
frame_vars of a reference program and render the result like the golden."""
import ctypes as C

from paper_1711_10413_b200 import _lib as P

PIPE = {"layouts": P.PIPELINE_DEFAULT, "layouts_o0": P.PIPELINE_O0,
        "layouts_bad_order": P.PIPELINE_BAD_ORDER}


def frame_var_array(fvars):
    arr = (P.FrameVar * max(len(fvars), 1))()
    for i, v in enumerate(fvars):
        flags = (P.VAR_ESCAPES if v["escapes"] else 0) | (P.VAR_PINNED if v["pinned"] else 0)
        arr[i] = P.FrameVar(v["group"], v["func"], flags, v["def_pos"], v["bytes"], v["first"],
                            v["last"])
    return arr


def run_builder(fn, fvars, n_groups, pipeline):
    n = len(fvars)
    arr = frame_var_array(fvars)
    lays = (P.DepotLayout * max(n_groups, 1))()
    slots = (P.DepotSlot * max(n, 1))()
    owners = (C.c_int32 * max(n, 1))()
    rc = fn(arr, n, n_groups, pipeline, lays, slots, max(n, 1), owners, max(n, 1))
    assert rc == 0, rc
    out = []
    for g in range(n_groups):
        L = lays[g]
        ss = []
        for k in range(L.slot_begin, L.slot_begin + L.n_slots):
            s = slots[k]
            ss.append({"offset": s.offset, "size": s.size, "align": s.align,
                       "shared": bool(s.shared),
                       "owners": [fvars[owners[j]]["name"]
                                  for j in range(s.owner_begin, s.owner_begin + s.n_owners)]})
        out.append({"slots": ss, "total_local": L.total_local, "total_shared": L.total_shared,
                    "has_shared_depot": bool(L.has_shared_depot),
                    "overlap_slot": L.overlap_slot})
    return out


def golden_view(layouts):
    return [{"slots": g["slots"], "total_local": g["total_local"],
             "total_shared": g["total_shared"], "has_shared_depot": g["has_shared_depot"]}
            for g in layouts]


def strip(out):
    return [{k: v for k, v in g.items() if k != "overlap_slot"} for g in out]
