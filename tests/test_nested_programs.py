"""Nested parallel regions as a runtime facility (EXTENSION):
programs whose region bodies contain `parallel` / `parallel for` run on the
GPU runtime -- each nested region serialized on the encountering thread,
its capture list published on the thread's data-sharing stack and read back
with get-shared-variables, the locals it captures globalized onto that stack
-- and equal the sequential AST oracle (oracle/ast_oracle.py, pinned against
the reference's oracle on every program the reference compiles)."""
import numpy as np
import pytest

import nested_programs as NP
from oracle import ast_oracle as AO
from paper_1711_10413_b200 import _lib as L
from paper_1711_10413_b200 import program as PG


def _compile(p):
    lays = PG.derive_layouts(p["ast"], p["kernel"])
    return PG.compile_program(p["ast"], lays, p["kernel"], p["teams"], p["workers"])


def _programs():
    return NP.corpus() + NP.generate(80)


def test_nested_programs_lower_verify_and_simulate_like_the_oracle():
    """CPU: every nested program lowers, passes the verifier, and the
    lowered bytecode (test-side interpreter) leaves the AST oracle's result."""
    import test_program as TP
    n_nested = 0
    for p in _programs():
        prog = _compile(p)
        assert PG.verify(prog) == L.OK, p["stem"]
        got = dict(zip([b[0] for b in prog.buffers],
                       TP.simulate(prog, TP.mapped_inputs(p, prog))))
        assert got["a"] == AO.run(p["ast"], p["teams"], p["workers"])["a"], p["stem"]
        n_nested += prog.nested()
    assert n_nested >= 50


def test_nested_frames_are_globalized_and_captures_ordered():
    """The frame pipeline marks an outer region's locals that a nested
    region captures as shared (they escape, LoweringPasses.cpp:107-139); the
    region then carries GLOBALIZE and the nested region captures them from
    the encountering activation, kernel variables first."""
    p = next(q for q in NP.corpus() if q["stem"] == "nest_config3")
    lays = PG.derive_layouts(p["ast"], p["kernel"])
    outer = next(g for g in lays if g["root"] == "__omp_outlined.0")
    shared = {o for s in outer["slots"] if s["shared"] for o in s["owners"]}
    assert shared == {"me", "e", "v"}  # L2 and L3 read them
    prog = PG.compile_program(p["ast"], lays, p["kernel"], p["teams"], p["workers"])
    r0, r1, r2 = prog.regions
    assert (r0.parent, r1.parent, r2.parent) == (-1, 0, 1)
    assert r0.globalize and r1.globalize and not r2.globalize
    assert [prog.var_names[v] for v in r0.captures] == ["c", "s"]
    names1 = [prog.var_names[v] for v in r1.captures]
    assert names1 == ["&c", "me", "e", "v"]  # c via the parent's capture
    assert [prog.var_names[v] for v in r2.captures] == ["&c", "&me", "f"]


def test_nested_verifier_rules():
    import dataclasses
    p = next(q for q in NP.corpus() if q["stem"] == "nest_shared_local")
    prog = _compile(p)
    assert PG.verify(prog) == L.OK
    r0, r1 = prog.regions
    # a nested region staged by the master, or one whose parent is not the
    # region that runs its PARALLEL
    bad = dataclasses.replace(prog, regions=[r0, dataclasses.replace(r1, parent=-1)])
    assert PG.verify(bad) == L.ERR_INVALID
    # a parent that is not an earlier region (a cycle)
    bad = dataclasses.replace(prog, regions=[dataclasses.replace(r0, parent=1), r1])
    assert PG.verify(bad) == L.ERR_INVALID
    # a private variable outside the region's frame
    bad = dataclasses.replace(prog, regions=[dataclasses.replace(r0, frame_bytes=0), r1])
    assert PG.verify(bad) == L.ERR_INVALID
    # nesting without data-sharing stacks
    import ctypes as C
    desc, _keep = PG.describe(prog, [16], stack_slot_bytes=0, stack_overflow_bytes=0)
    assert L.lib().ompds_program_verify(C.byref(desc)) == L.ERR_INVALID


def test_config3_program_equals_the_config3_oracle():
    """The DSL form of the config-3 program means what the
    hand-written NestedProg kernel and its C oracle orc_nested compute."""
    from oracle import oracle as O
    p = next(q for q in NP.corpus() if q["stem"] == "nest_config3")
    want = np.zeros(p["teams"] * p["workers"], dtype=np.int32)
    O.lib().orc_nested(0, p["teams"], p["workers"], 3, O.ptr(want))
    assert AO.run(p["ast"], p["teams"], p["workers"])["a"] == want.tolist()


@pytest.mark.gpu
def test_gpu_nested_programs_match_the_oracle():
    import torch
    n = 0
    for p in _programs():
        prog = _compile(p)
        bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
                for _, sz, init in prog.buffers]
        out = PG.run_program(prog, bufs)
        st = out.team_stats()
        assert [s.trap for s in st] == [0] * p["teams"], (p["stem"], [s.trap for s in st])
        got = {name: b.cpu().tolist() for (name, _, _), b in zip(prog.buffers, bufs)}
        assert got["a"] == AO.run(p["ast"], p["teams"], p["workers"])["a"], p["stem"]
        n += prog.nested()
    assert n >= 50


@pytest.mark.gpu
@pytest.mark.parametrize("slot,ovf", [(0, 32768), (4096, 0), (1024, 4096)])
def test_gpu_nested_stack_placement_never_changes_results(slot, ovf):
    """Frames in each lane's shared-memory slot, all on the global overflow
    chain, or spilling from one to the other: the same results."""
    import torch
    for p in NP.corpus() + NP.generate(20, seed=7):
        prog = _compile(p)
        bufs = [torch.full((sz,), init, dtype=torch.int32, device="cuda")
                for _, sz, init in prog.buffers]
        out = PG.run_program(prog, bufs, stack_slot_bytes=slot, stack_overflow_bytes=ovf)
        assert all(s.trap == 0 for s in out.team_stats()), p["stem"]
        assert bufs[0].cpu().tolist() == AO.run(p["ast"], p["teams"], p["workers"])["a"], \
            (p["stem"], slot, ovf)


@pytest.mark.gpu
def test_gpu_nested_stack_exhaustion_traps():
    """A lane whose data-sharing stack cannot hold a nested region's list or
    frame traps with the stack-overflow code instead of corrupting memory."""
    import torch
    p = next(q for q in NP.corpus() if q["stem"] == "nest_config3")
    prog = _compile(p)
    bufs = [torch.zeros(sz, dtype=torch.int32, device="cuda") for _, sz, _ in prog.buffers]
    out = PG.run_program(prog, bufs, stack_slot_bytes=256, stack_overflow_bytes=0)
    assert any(s.trap == L.TRAP_STACK_OVERFLOW for s in out.team_stats())
