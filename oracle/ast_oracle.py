"""Sequential AST oracle for region programs, with nested regions.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): tests use it as the
checker for programs the reference cannot run; the product never imports it.

Restates the reference's sequential oracle (proj/src/SequentialOracle.cpp)
on the frontend's AST (dumpAst JSON): every team runs the target body
sequentially with fresh kernel-scope variables (:182-196; unmapped host
scalars are per-team copies of the host value, mapped arrays are global);
a bare ``parallel`` runs its body once per worker w with
omp_get_thread_num() = w (:150-172); a ``parallel for`` gives worker w the
iterations init + team*W + w, stepping W*teams (:151-166, the strip-mining
of AstLowering.cpp:429-462).  Integers are int32 with wrap-around after
every operation, as the simulator stores them (Simulator.cpp:29-42); the
reference oracle computes in int64, which agrees on every program without
overflow (tests/test_oracle_golden.py pins this module against the
reference's recorded oracle outputs).

EXTENSION (the reference rejects nesting,
DslParser.cpp:846-849): a region met inside a region body is serialized on
the encountering thread -- a team of one, as the LLVM device runtime the
paper targets does -- so its body runs once with omp_get_thread_num() = 0,
and a nested ``parallel for`` runs all its iterations, init to bound in
order, on that thread.  Variables of enclosing scopes are shared by
reference (the nested region writes the encountering thread's locals).
"""
from __future__ import annotations

from typing import Dict, List


def _wrap(v: int) -> int:
    v &= 0xFFFFFFFF
    return v - (1 << 32) if v & 0x80000000 else v


class _Cell:
    __slots__ = ("vals",)

    def __init__(self, n: int, fill: int = 0):
        self.vals = [fill] * n


class _Scope:
    def __init__(self, parent=None):
        self.parent = parent
        self.vars: Dict[str, _Cell] = {}

    def lookup(self, name):
        s = self
        while s is not None:
            if name in s.vars:
                return s.vars[name]
            s = s.parent
        raise KeyError(name)


def run(ast: dict, teams: int, workers: int, overrides=None) -> Dict[str, List[int]]:
    """Final contents of the mapped arrays after the target region."""
    target = ast["target"]
    maps = {m["name"] for m in target["maps"]}
    glob = _Scope()
    host = {h["name"]: h for h in ast["host"]}
    for h in ast["host"]:
        if h["name"] in maps:
            n = h.get("array_size", 1)
            glob.vars[h["name"]] = _Cell(n, h["init"])
    for name, vals in (overrides or {}).items():
        cell = glob.vars[name]
        cell.vals = [_wrap(v) for v in (vals if len(vals) == len(cell.vals)
                                        else vals * len(cell.vals))]

    def ev(e, sc, tid):
        k = e["kind"]
        if k == "int":
            return _wrap(e["value"])
        if k == "var":
            return sc.lookup(e["name"]).vals[0]
        if k == "index":
            cell = sc.lookup(e["name"])
            i = ev(e["index"], sc, tid)
            if not 0 <= i < len(cell.vals):
                raise IndexError(f"{e['name']}[{i}]")
            return cell.vals[i]
        if k == "binary":
            a, b = ev(e["lhs"], sc, tid), ev(e["rhs"], sc, tid)
            return _wrap(a + b if e["op"] == "+" else a - b if e["op"] == "-" else a * b)
        if k == "thread_num":
            return tid["thread"]
        if k == "team_num":
            return tid["team"]
        raise ValueError(k)

    def exec_body(body, sc, tid):
        for st in body:
            exec_stmt(st, sc, tid)

    def exec_stmt(st, sc, tid):
        k = st["kind"]
        if k == "decl":
            n = st.get("array_size", 1)
            init = st.get("init")
            if "array_size" in st:
                sc.vars[st["name"]] = _Cell(n, _wrap(init["value"]) if init else 0)
            else:
                sc.vars[st["name"]] = _Cell(1, ev(init, sc, tid) if init else 0)
        elif k == "assign":
            cell = sc.lookup(st["name"])
            i = ev(st["index"], sc, tid) if "index" in st else 0
            if not 0 <= i < len(cell.vals):
                raise IndexError(f"{st['name']}[{i}]")
            v = ev(st["value"], sc, tid)
            cell.vals[i] = _wrap(cell.vals[i] + v) if st["compound"] else v
        elif k == "for":
            inner = _Scope(sc)
            inner.vars[st["counter"]] = _Cell(1, ev(st["init"], sc, tid))
            c = inner.vars[st["counter"]]
            while c.vals[0] < ev(st["bound"], inner, tid):
                exec_body(st.get("body", []), _Scope(inner), tid)
                c.vals[0] = _wrap(c.vals[0] + 1)
        elif k == "block":
            exec_body(st.get("body", []), _Scope(sc), tid)
        elif k in ("parallel", "parallel_for"):
            nested = tid["in_region"]
            team = tid["team"]
            for w in ([0] if nested else range(workers)):
                t2 = {"thread": w, "team": team, "in_region": True}
                if k == "parallel":
                    exec_body(st.get("body", []), _Scope(sc), t2)
                    continue
                loop = st["body"][0]
                rs = _Scope(sc)
                start = ev(loop["init"], sc, t2)
                if nested:  # EXTENSION: the team of one runs every iteration
                    step = 1
                else:       # SequentialOracle.cpp:151-166
                    start = _wrap(start + team * workers + w)
                    step = workers * teams
                rs.vars[loop["counter"]] = _Cell(1, start)
                c = rs.vars[loop["counter"]]
                while c.vals[0] < ev(loop["bound"], rs, t2):
                    exec_body(loop.get("body", []), _Scope(rs), t2)
                    c.vals[0] = _wrap(c.vals[0] + step)
        else:
            raise ValueError(k)

    refd = set()

    def walk(x):
        if isinstance(x, dict):
            if x.get("kind") in ("var", "index", "assign"):
                refd.add(x.get("name"))
            for v in x.values():
                walk(v)
        elif isinstance(x, list):
            for v in x:
                walk(v)
    walk(target["body"])
    for team in range(teams):
        ks = _Scope(glob)
        for name, h in host.items():  # per-team firstprivate copies
            if name not in maps and name in refd:
                ks.vars[name] = _Cell(1, _wrap(h["init"]))
        exec_body(target["body"], ks, {"thread": 0, "team": team, "in_region": False})
    return {name: glob.vars[name].vals for name in maps}
