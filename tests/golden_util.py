"""Loads the reference golden vectors (tests/golden/*.json, produced from the
unmodified reference by oracle/ref/ref_golden.cpp via tests/golden/regen.sh)."""
import functools
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def load(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def programs(include_generated=True, only_ok=True):
    out = list(load("corpus")) + list(load("analogs"))
    if include_generated:
        out += list(load("generated"))
    if only_ok:
        out = [p for p in out if p.get("compile_ok")]
    return out


def race_free_run(run):
    """A launch whose simulator output equals the sequential oracle's."""
    s, o = run["sim"], run["oracle"]
    return s["ok"] and o["ok"] and s["globals"] == o["globals"]


def reference_broken(p):
    """The 31 generated programs hit by the reference's name-shadowing bug
    (AstLowering.cpp:237-242): two or more `for (int i` loops."""
    return p["source"].count("for (int i") >= 2


def frame_groups(p):
    """Group roots/members in the reference's order."""
    return [(g["root"], g["members"]) for g in p["layouts"]]
