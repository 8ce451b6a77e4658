"""Region programs with nested parallel regions (EXTENSION: the reference
frontend rejects nesting, proj/src/DslParser.cpp:846-849), written as the
frontend's AST (dumpAst JSON shape) with a small builder, plus a seeded
generator of race-free nested programs.

Each program's worker w of team t writes only a[t*W + w] (through a local
`me` captured from its outer region, since omp_get_thread_num() is 0 inside
a serialized nested region), so the programs are race-free and their
results are defined by oracle/ast_oracle.py.
"""
import random


def num(v):
    return {"kind": "int", "value": v}


def var(n):
    return {"kind": "var", "name": n}


def at(n, i):
    return {"kind": "index", "name": n, "index": i}


def bin_(op, a, b):
    return {"kind": "binary", "op": op, "lhs": a, "rhs": b}


def add(a, b):
    return bin_("+", a, b)


def mul(a, b):
    return bin_("*", a, b)


TID = {"kind": "thread_num"}
TEAM = {"kind": "team_num"}


def decl(n, init=None, size=None):
    d = {"kind": "decl", "name": n}
    if size is not None:
        d["array_size"] = size
        d["init"] = num(init or 0)
    elif init is not None:
        d["init"] = init
    return d


def assign(n, val, index=None, compound=False):
    d = {"kind": "assign", "name": n, "value": val, "compound": compound}
    if index is not None:
        d["index"] = index
    return d


def loop(counter, init, bound, *body):
    return {"kind": "for", "counter": counter, "init": init, "bound": bound,
            "body": [{"kind": "block", "body": list(body)}]}


def par(*body):
    return {"kind": "parallel", "body": [{"kind": "block", "body": list(body)}]}


def pfor(counter, init, bound, *body):
    return {"kind": "parallel_for",
            "body": [{"kind": "for", "counter": counter, "init": init, "bound": bound,
                      "body": [{"kind": "block", "body": list(body)}]}]}


def program(stem, teams, workers, body, host=None):
    host = host or []
    n = teams * workers
    ast = {"host": [{"name": "a", "array_size": n, "init": 0}] + host,
           "target": {"body": body, "maps": [{"name": "a", "length": n, "dir": "tofrom"}],
                      "num_teams": teams, "thread_limit": workers}}
    return {"stem": stem, "ast": ast, "kernel": f"__omp_offload_{stem}", "teams": teams,
            "workers": workers}


def _slot(workers):
    """a[] index of the current outer worker: team * W + me."""
    return add(mul(TEAM, num(workers)), var("me"))


def corpus():
    out = []
    W, T = 8, 2
    # a local of the outer region captured (and written) by a nested region
    out.append(program("nest_shared_local", T, W, [
        decl("c", num(3)),
        par(decl("me", TID),
            decl("e", add(TID, var("c"))),
            par(assign("e", num(1), compound=True)),
            assign("a", var("e"), _slot(W), compound=True))]))
    # a nested parallel-for filling an outer region's array
    out.append(program("nest_parallel_for", T, W, [
        par(decl("me", TID),
            decl("s", 0, 4),
            pfor("j", num(0), num(4),
                 assign("s", mul(var("j"), add(var("me"), num(1))), var("j"))),
            assign("a", add(at("s", num(1)), at("s", num(3))), _slot(W)))]))
    # the config-3 program of DESIGN.md §7 (int): depth 3, scalars and arrays
    body3 = [
        decl("c", num(1)),
        decl("s", 0, 8),
        loop("k", num(0), num(8), assign("s", add(var("k"), num(1)), var("k"))),
        loop("r", num(0), num(3),
             par(decl("me", TID),
                 decl("e", add(TID, var("c"))),
                 decl("v", 0, 4),
                 loop("j", num(0), num(4),
                      assign("v", mul(at("s", var("me")), add(var("j"), num(1))), var("j"))),
                 par(decl("f", add(var("e"), at("v", num(3)))),
                     par(assign("a", add(var("f"), var("c")), _slot(W), compound=True),
                         assign("f", mul(var("f"), num(2)))),
                     assign("v", var("f"), num(0)),
                     assign("e", num(1), compound=True)),
                 assign("a", add(at("v", num(0)), var("e")), _slot(W), compound=True)),
             assign("c", num(1), compound=True)),
    ]
    out.append(program("nest_config3", T, W, body3))
    # divergent nesting: worker `me` enters me nested regions
    out.append(program("nest_divergent", T, W, [
        decl("c", num(5)),
        par(decl("me", TID),
            decl("x", num(0)),
            loop("k", num(0), var("me"),
                 par(assign("x", add(var("k"), var("c")), compound=True))),
            assign("a", var("x"), _slot(W), compound=True))]))
    # a kernel variable reaching a depth-2 region through its parent
    out.append(program("nest_kernel_capture", 1, 32, [
        decl("c", num(7)),
        decl("d", num(2)),
        par(decl("me", TID),
            par(decl("t", num(0)),
                par(assign("t", mul(var("c"), var("d")))),
                assign("a", add(var("t"), var("me")), add(mul(TEAM, num(32)), var("me"))))),
        assign("c", num(1), compound=True)]))
    # a host firstprivate scalar, a nested region with no captures
    out.append(program("nest_host_scalar", 3, 4, [
        par(decl("me", TID),
            par(decl("z", num(4))),
            assign("a", add(var("h"), var("me")), _slot(4)))],
        host=[{"name": "h", "init": 11}]))
    return out


def generate(n, seed=0x5eed01ab):
    """Seeded random nested programs: an outer region per worker with 1-2
    locals, nested regions (parallel / parallel for, depth up to 3) that read
    kernel scalars and enclosing locals and update enclosing locals and their
    own, some inside sequential loops whose trip count is the worker's id;
    every write to a[] goes to the worker's own slot."""
    rng = random.Random(seed)
    out = []
    for i in range(n):
        T = rng.choice([1, 2, 3])
        W = rng.choice([1, 4, 8, 32, 40])
        kvars = [f"k{j}" for j in range(rng.randint(0, 3))]
        body = [decl(k, num(rng.randint(-5, 9))) for k in kvars]

        def expr(names, depth=0):
            c = rng.random()
            if not names or c < 0.25 or depth > 2:
                return num(rng.randint(-4, 9))
            if c < 0.6:
                return var(rng.choice(names))
            return bin_(rng.choice("+-*"), expr(names, depth + 1), expr(names, depth + 1))

        counter = [0]

        def fresh(p):
            counter[0] += 1
            return f"{p}{counter[0]}"

        def region_body(names, level):
            """Statements of a region at nesting `level` (1 = outer)."""
            st = []
            mine = []
            for _ in range(rng.randint(1, 2)):
                n_ = fresh("x")
                st.append(decl(n_, expr(names + mine)))
                mine.append(n_)
            visible = names + mine
            for _ in range(rng.randint(1, 3)):
                c = rng.random()
                if c < 0.35 and level < 3:
                    inner = region_body(visible, level + 1)
                    if rng.random() < 0.5:
                        st.append(par(*inner))
                    else:
                        j = fresh("j")
                        st.append(pfor(j, num(0), num(rng.randint(0, 3)), *inner))
                elif c < 0.55 and level < 3:
                    # a nested region inside a sequential loop: with W <= 8 the
                    # trip count is the worker's own id, so the lanes of a
                    # warp enter different numbers of nested activations
                    k = fresh("q")
                    inner = region_body(visible, level + 1)
                    bound = var("me") if W <= 8 else num(rng.randint(0, 2))
                    st.append(loop(k, num(0), bound, par(*inner)))
                elif mine:
                    st.append(assign(rng.choice(mine), expr(visible), compound=rng.random() < 0.5))
                if rng.random() < 0.5:
                    # an enclosing local updated by this (serialized) region
                    tgt = rng.choice(visible)
                    # kernel scalars are shared by all workers; `me` names the slot
                    if tgt not in kvars and tgt != "me":
                        st.append(assign(tgt, expr(visible), compound=True))
            st.append(assign("a", expr(visible), _slot(W), compound=True))
            return st

        outer = [decl("me", TID)] + region_body(["me"] + kvars, 1)
        body.append(par(*outer))
        if kvars and rng.random() < 0.5:
            body.append(assign(kvars[0], num(1), compound=True))
            body.append(par(decl("me", TID), assign("a", var(kvars[0]), _slot(W), compound=True)))
        out.append(program(f"nest_gen_{i}", T, W, body))
    return out
