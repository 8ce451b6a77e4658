"""Manifest JSON (Compiler.cpp:112-155, §8(f) row 1): the C ABI's writer
reproduces the reference compiler's text byte for byte for every corpus and
generated program (from our own frame pipeline's layouts), the reader parses
the reference's text back to the golden values, and malformed manifests are
refused."""
import json

import pytest

import golden_util as G
from paper_1711_10413_b200 import layout


def _vars(p):
    return [layout.FrameVar(v["name"], v["bytes"], v["group"], v["func"], v["escapes"],
                            v["pinned"], v["def_pos"], v["first"], v["last"])
            for v in p["frame_vars"]]


def _programs():
    return [p for p in G.programs() if p.get("manifest_text")]


def test_writer_is_byte_identical_to_the_reference():
    n = 0
    for p in _programs():
        m = p["manifest"]
        text = layout.manifest_text(_vars(p), len(p["layouts"]), m["kernel"],
                                    m["launch"]["teams"], m["launch"]["workers"])
        assert text == p["manifest_text"], p["stem"]
        n += 1
    assert n >= 18 + 89


def test_reader_recovers_the_reference_values():
    for p in _programs():
        got = layout.parse_manifest(p["manifest_text"])
        m = p["manifest"]
        assert got.kernel == m["kernel"]
        assert (got.teams, got.workers) == (m["launch"]["teams"], m["launch"]["workers"])
        d = m["depot"]
        assert [(s.offset, s.size, s.align, s.shared, s.owners) for s in got.depot.slots] == \
            [(s["offset"], s["size"], s["align"], s["shared"], s["owners"]) for s in d["slots"]]
        assert (got.depot.total_local, got.depot.total_shared, got.depot.has_shared_depot) == \
            (d["total_local"], d["total_shared"], d["mirrored"])
        assert (got.stack_bytes, got.prealloc_entries, got.prealloc_bytes, got.runtime_bytes,
                got.shared_footprint) == (m["stack_bytes"], m["prealloc_entries"],
                                          m["prealloc_bytes"], m["runtime_bytes"],
                                          m["shared_footprint"])


def test_reader_accepts_any_layout_of_the_json_and_round_trips():
    p = next(q for q in _programs() if q["stem"] == "mixed_captures")
    compact = json.dumps(json.loads(p["manifest_text"]), separators=(",", ":"))
    reordered = json.dumps(dict(reversed(list(json.loads(p["manifest_text"]).items()))))
    a = layout.parse_manifest(p["manifest_text"])
    assert layout.parse_manifest(compact) == a == layout.parse_manifest(reordered)
    # write -> parse -> the same manifest; the other pipelines' kernel layouts too
    for pipe in ("default", "o0", "bad_order"):
        m = p["manifest"]
        t = layout.manifest_text(_vars(p), len(p["layouts"]), m["kernel"], m["launch"]["teams"],
                                 m["launch"]["workers"], pipeline=pipe)
        back = layout.parse_manifest(t)
        assert layout.manifest_text(_vars(p), len(p["layouts"]), back.kernel, back.teams,
                                    back.workers, pipeline=pipe) == t


@pytest.mark.parametrize("mutate", [
    lambda d: d.pop("kernel"),
    lambda d: d["depot"].pop("slots"),
    lambda d: d.__setitem__("shared_footprint", d["shared_footprint"] + 1),
    lambda d: d.__setitem__("stack_bytes", d["stack_bytes"] + 8),
    lambda d: d["depot"]["slots"][0].__setitem__("offset", 8),
    lambda d: d["depot"]["slots"][0].__setitem__("size", "8"),
    lambda d: d.__setitem__("runtime_bytes", 48),
    lambda d: d.__setitem__("prealloc_bytes", 8),
    lambda d: d["depot"].__setitem__("mirrored", 1),
])
def test_reader_refuses_malformed_manifests(mutate):
    from paper_1711_10413_b200 import _lib as L
    p = next(q for q in _programs() if q["stem"] == "shared_scalar")
    d = json.loads(p["manifest_text"])
    mutate(d)
    with pytest.raises(L.OmpdsError):
        layout.parse_manifest(json.dumps(d))


@pytest.mark.parametrize("text", ["", "{", "[]", '{"kernel": "k"', "nul", '{"a": 1,}',
                                  '{"a": 1.5}', '{"a": "\\x"}'])
def test_reader_refuses_broken_json(text):
    from paper_1711_10413_b200 import _lib as L
    with pytest.raises(L.OmpdsError):
        layout.parse_manifest(text)
