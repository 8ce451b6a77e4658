"""Region programs: the reference's kernel language executed by the sm_100a
generic-mode runtime.

A program is the reference frontend's AST (``dumpAst`` JSON,
proj/src/DslParser.cpp:986-1035 -- the frontend itself stays out of scope)
plus the frame layouts of its frame groups.  This module lowers it to a small
stack bytecode the device interprets *inside* the real protocol: the master
lane runs the sequential code; every ``parallel`` / ``parallel for`` becomes
a region staged with prepare_parallel, whose captures (kernel-frame variables
the region references, in kernel alloca order -- Codegen.cpp:173-201) are
published through the shared-args list and read by the workers with
get-shared-variables.  Variables live where the frame layout puts them:

* kernel frame group, shared-resident slot  -> the team's depot (shared memory)
* kernel frame group, local slot            -> the master's local depot mirror
* outlined-function frame group             -> the worker thread's private frame
* mapped host arrays                        -> device buffers

so a layout produced by a hazardous pass order (two variables merged into one
shared slot) misbehaves on the GPU exactly as in the reference
(SimulatorTests.cpp:150-173).  Integer semantics are the simulator's: i32
storage and i32 wrap-around after every operation (Simulator.cpp:29-42).
Parallel-for iterations are strip-mined cyclically: start = init + team*W +
tid, stride = W*teams (AstLowering.cpp:429-462).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from . import _lib as L

# opcodes (must match csrc/ompds_kernels.cu ProgramProg)
OP_END, OP_PUSH, OP_LOAD, OP_STORE, OP_LOADX, OP_STOREX, OP_ADD, OP_SUB, OP_MUL, \
    OP_TID, OP_TEAM, OP_NTHREADS, OP_NTEAMS, OP_JMP, OP_JNLT, OP_PARALLEL, OP_ZERO_PRIV = range(17)
# variable spaces
SP_DEPOT, SP_MLOCAL, SP_PRIV, SP_CAPTURE, SP_GLOBAL = range(5)


class CompileError(Exception):
    pass


@dataclass
class Region:
    entry: int
    captures: List[int]  # var-table indices in the encountering context, in capture order
    parent: int = -1     # -1: staged by the master; else the encountering region (nested)
    frame_bytes: int = 0  # its outlined function's frame (TotalLocal)
    globalize: bool = False  # its frame holds locals a nested region captures


@dataclass
class Program:
    code: List[int]
    vars: List[Tuple[int, int, int]]          # (space, offset/index, elements)
    var_names: List[str]
    regions: List[Region]
    buffers: List[Tuple[str, int, int]]       # (name, elements, init)
    total_shared: int
    total_local: int
    priv_bytes: int
    teams: int
    workers: int

    def nested(self) -> bool:
        """Some region nests or globalizes: the lanes need data-sharing stacks."""
        return any(r.parent >= 0 or r.globalize for r in self.regions)


def _layout_slots(layouts, root) -> Dict[str, Tuple[int, bool]]:
    """owner name -> (slot offset, shared) for the group rooted at `root`."""
    out = {}
    for g in layouts:
        if g["root"] != root:
            continue
        for s in g["slots"]:
            for o in s["owners"]:
                out[o] = (s["offset"], bool(s["shared"]))
    return out


class _Compiler:
    def __init__(self, ast, layouts, kernel_root, teams, workers):
        self.ast = ast
        self.layouts = layouts
        self.kernel_root = kernel_root
        self.teams = teams
        self.workers = workers
        self.code: List[int] = []
        self.vars: List[Tuple[int, int, int]] = []
        self.var_names: List[str] = []
        self.regions: List[Region] = []
        self.kslots = _layout_slots(layouts, kernel_root)
        maps = {m["name"] for m in ast["target"]["maps"]}
        self.buffers = []
        self.global_idx = {}
        for h in ast["host"]:
            if h["name"] in maps:
                self.global_idx[h["name"]] = len(self.buffers)
                self.buffers.append((h["name"], h.get("array_size", 1), h["init"]))
        self.host = {h["name"]: h for h in ast["host"]}
        # kernel-scope variables in alloca emission order (AstLowering.cpp:23-52)
        self.kvars: Dict[str, int] = {}
        self.kelems: Dict[str, int] = {}
        # the region tree in lowering order (derive_frame_vars's numbering):
        # AST statement -> (region id, parent id), and each region's captures
        # (names from enclosing scopes its subtree references), precomputed
        # so a parent captures what its nested regions need
        self.rid_of: Dict[int, int] = {}
        self.tree: List[Tuple[dict, int]] = []
        queue = [(st, -1) for st in _regions_in(ast["target"]["body"], [])]
        while queue:
            st, parent = queue.pop(0)
            self.rid_of[id(st)] = len(self.tree)
            self.tree.append((st, parent))
            queue += [(n, len(self.tree) - 1) for n in _regions_in(_region_body(st), [])]
        self.cap_names: List[List[str]] = []
        self.nested_src: Dict[int, List[int]] = {}

    # -- variable table ----------------------------------------------------
    def _var(self, name, space, off, elems):
        self.vars.append((space, off, elems))
        self.var_names.append(name)
        return len(self.vars) - 1

    def _kernel_var(self, name, elems):
        if name not in self.kslots:
            raise CompileError(f"no kernel frame slot for {name}")
        off, shared = self.kslots[name]
        idx = self._var(name, SP_DEPOT if shared else SP_MLOCAL, off, elems)
        self.kvars[name] = idx
        self.kelems[name] = elems
        return idx

    def emit(self, *w):
        self.code.extend(int(x) for x in w)

    # -- references ---------------------------------------------------------
    def resolve(self, name, scope):
        """Var-table index of `name` in `scope` (a dict for region code)."""
        if scope is not None and name in scope["locals"]:
            return scope["locals"][name]
        if scope is not None and name in scope["capnames"]:
            # a variable of an enclosing scope (the kernel's, or -- nested --
            # an enclosing region's) referenced from a region is a capture
            return scope["capvar"](name)
        if name in self.kvars and scope is None:
            return self.kvars[name]
        if name in self.global_idx:
            return self._global_var(name)
        raise CompileError(f"unresolved {name}")

    def _global_var(self, name):
        key = ("@", name)
        if not hasattr(self, "_gv"):
            self._gv = {}
        if name not in self._gv:
            b = self.global_idx[name]
            self._gv[name] = self._var("@" + name, SP_GLOBAL, b, self.buffers[b][1])
        return self._gv[name]

    # -- expressions ----------------------------------------------------------
    def expr(self, e, scope, in_region):
        k = e["kind"]
        if k == "int":
            self.emit(OP_PUSH, e["value"])
        elif k == "var":
            self.emit(OP_LOAD, self.resolve(e["name"], scope))
        elif k == "index":
            self.expr(e["index"], scope, in_region)
            self.emit(OP_LOADX, self.resolve(e["name"], scope))
        elif k == "binary":
            self.expr(e["lhs"], scope, in_region)
            self.expr(e["rhs"], scope, in_region)
            self.emit({"+": OP_ADD, "-": OP_SUB, "*": OP_MUL}[e["op"]])
        elif k == "thread_num":
            if in_region:
                self.emit(OP_TID)
            else:
                self.emit(OP_PUSH, 0)
        elif k == "team_num":
            self.emit(OP_TEAM)
        else:
            raise CompileError(f"expression kind {k}")

    # -- statements -----------------------------------------------------------
    def stmt(self, s, scope, in_region):
        k = s["kind"]
        if k == "decl":
            elems = s.get("array_size", 1)
            if scope is None:
                v = self._kernel_var(s["name"], elems)
            else:
                v = self._priv_var(s["name"], elems, scope)
            init = s.get("init")
            if "array_size" in s:
                fill = init["value"] if init else 0
                if init and init["kind"] != "int":
                    raise CompileError("array initializer must be a constant")
                if fill:
                    for i in range(elems):
                        self.emit(OP_PUSH, i, OP_PUSH, fill, OP_STOREX, v)
            elif init is not None:
                self.expr(init, scope, in_region)
                self.emit(OP_STORE, v)
        elif k == "assign":
            v = self.resolve(s["name"], scope)
            if "index" in s:
                self.expr(s["index"], scope, in_region)
                if s["compound"]:
                    self.expr(s["index"], scope, in_region)
                    self.emit(OP_LOADX, v)
                    self.expr(s["value"], scope, in_region)
                    self.emit(OP_ADD)
                else:
                    self.expr(s["value"], scope, in_region)
                self.emit(OP_STOREX, v)
            else:
                if s["compound"]:
                    self.emit(OP_LOAD, v)
                    self.expr(s["value"], scope, in_region)
                    self.emit(OP_ADD)
                else:
                    self.expr(s["value"], scope, in_region)
                self.emit(OP_STORE, v)
        elif k == "for":
            if scope is None:
                v = self._kernel_var(s["counter"], 1)
            else:
                v = self._priv_var(s["counter"], 1, scope)
            self.expr(s["init"], scope, in_region)
            self.emit(OP_STORE, v)
            top = len(self.code)
            self.emit(OP_LOAD, v)
            self.expr(s["bound"], scope, in_region)
            self.emit(OP_JNLT, 0)
            patch = len(self.code) - 1
            for b in s.get("body", []):
                self.stmt(b, scope, in_region)
            self.emit(OP_LOAD, v, OP_PUSH, 1, OP_ADD, OP_STORE, v, OP_JMP, top)
            self.code[patch] = len(self.code)
        elif k in ("parallel", "parallel_for"):
            r = self.rid_of[id(s)]
            if scope is not None:
                # nested (EXTENSION): the encountering region publishes the
                # addresses of the nested region's captures from its own
                # activation -- its locals or its own captures
                if self.tree[r][1] != scope["rid"]:
                    raise CompileError("region tree mismatch")
                self.nested_src[r] = [self.resolve(n, scope) for n in self.cap_names[r]]
            self.emit(OP_PARALLEL, r)
            self.pending.append((r, s))
        elif k == "block":
            for b in s.get("body", []):
                self.stmt(b, scope, in_region)
        else:
            raise CompileError(f"statement kind {k}")

    def _priv_var(self, name, elems, scope):
        slots = scope["pslots"]
        if name not in slots:
            raise CompileError(f"no private frame slot for {name}")
        v = self._var(name, SP_PRIV, slots[name][0], elems)
        scope["locals"][name] = v
        return v

    def _capture_names(self):
        """Per region: the names of enclosing-scope variables its subtree
        references, in capture order -- kernel variables in kernel alloca
        order (Codegen.cpp:173-201), then (nested regions, EXTENSION) the
        enclosing regions' locals, outermost region first, each in its
        declaration order."""
        local_names = []
        for st, _ in self.tree:
            ls = [st["body"][0]["counter"]] if st["kind"] == "parallel_for" else []
            local_names.append([n for n, _ in _decls(_region_body(st), [(x, 1) for x in ls])])
        # names declared anywhere in a region's subtree (its own locals and
        # its nested regions'): references to them are not captures of it
        below = [set(ln) for ln in local_names]
        for r in reversed(range(len(self.tree))):
            p = self.tree[r][1]
            if p >= 0:
                below[p] |= below[r]
        out = []
        for r, (st, parent) in enumerate(self.tree):
            refs = _names_in(st, set()) - below[r] - set(self.global_idx)
            chain = []  # ancestors, outermost first
            p = parent
            while p >= 0:
                chain.insert(0, p)
                p = self.tree[p][1]
            keyed = []
            for name in refs:
                home = next((p for p in reversed(chain) if name in local_names[p]), None)
                if home is not None:
                    keyed.append(((1, chain.index(home), local_names[home].index(name)), name))
                elif name in self.kvars:
                    keyed.append(((0, self.kvars[name], 0), name))
                else:
                    raise CompileError(f"unresolved {name}")
            out.append([n for _, n in sorted(keyed)])
        return out

    def region(self, r, s):
        root = f"__omp_outlined.{r}"
        parent = self.tree[r][1]
        group = next((g for g in self.layouts if g["root"] == root), None)
        scope = {"locals": {}, "caps": {}, "pslots": _layout_slots(self.layouts, root), "rid": r}
        names = self.cap_names[r]
        capvars: Dict[str, int] = {}

        def capvar(name):
            if name not in capvars:
                if name not in names:
                    raise CompileError(f"{name} is not a capture of region {r}")
                src = self.kvars.get(name)
                elems = self.kelems[name] if src is not None and parent < 0 else \
                    self._elems_of_capture(r, name)
                capvars[name] = self._var("&" + name, SP_CAPTURE, names.index(name), elems)
            return capvars[name]

        scope["capvar"] = capvar
        scope["capnames"] = set(names)
        entry = len(self.code)
        self.emit(OP_ZERO_PRIV)
        if s["kind"] == "parallel_for":
            loop = s["body"][0]
            v = self._priv_var(loop["counter"], 1, scope)
            self.expr(loop["init"], scope, True)
            if parent < 0:
                # start = init + (team * nt + tid); stride = nt * nteams
                # (AstLowering.cpp:429-462)
                self.emit(OP_TEAM, OP_NTHREADS, OP_MUL, OP_TID, OP_ADD, OP_ADD, OP_STORE, v)
            else:
                # nested: the team of one runs every iteration (start = init +
                # tid, stride = nt, with tid 0 and nt 1)
                self.emit(OP_TID, OP_ADD, OP_STORE, v)
            top = len(self.code)
            self.emit(OP_LOAD, v)
            self.expr(loop["bound"], scope, True)
            self.emit(OP_JNLT, 0)
            patch = len(self.code) - 1
            for b in loop.get("body", []):
                self.stmt(b, scope, True)
            if parent < 0:
                self.emit(OP_LOAD, v, OP_NTHREADS, OP_NTEAMS, OP_MUL, OP_ADD, OP_STORE, v,
                          OP_JMP, top)
            else:
                self.emit(OP_LOAD, v, OP_NTHREADS, OP_ADD, OP_STORE, v, OP_JMP, top)
            self.code[patch] = len(self.code)
        else:
            for b in s.get("body", []):
                self.stmt(b, scope, True)
        self.emit(OP_END)
        self.scopes[r] = scope
        caps = [self.kvars[n] for n in names] if parent < 0 else None
        self.regions[r] = Region(entry, caps, parent,
                                 group["total_local"] if group else 0,
                                 bool(group and any(sl["shared"] for sl in group["slots"])))

    def _elems_of_capture(self, r, name):
        """Elements of the variable a nested region's capture aliases."""
        p = self.tree[r][1]
        while p >= 0:
            sc = self.scopes.get(p)
            if sc is not None and name in sc["locals"]:
                return self.vars[sc["locals"][name]][2]
            p = self.tree[p][1]
        return self.kelems[name]

    def compile(self) -> Program:
        self.pending = []
        self.scopes: Dict[int, dict] = {}
        self.regions = [Region(-1, []) for _ in self.tree]
        # unmapped host scalars referenced by the target become kernel allocas
        # initialised with their host value (AstLowering.cpp:31-37)
        refd = set()

        def walk(x):
            if isinstance(x, dict):
                if x.get("kind") in ("var", "index") or x.get("kind") == "assign":
                    refd.add(x.get("name"))
                for v in x.values():
                    walk(v)
            elif isinstance(x, list):
                for v in x:
                    walk(v)

        walk(self.ast["target"]["body"])
        for h in self.ast["host"]:
            if h["name"] in self.global_idx or h["name"] not in refd:
                continue
            if "array_size" in h:
                raise CompileError("unmapped host array")
            v = self._kernel_var(h["name"], 1)
            self.emit(OP_PUSH, h["init"], OP_STORE, v)
        for s in self.ast["target"]["body"]:
            self.stmt(s, None, False)
        self.emit(OP_END)
        self.cap_names = self._capture_names()
        i = 0
        while i < len(self.pending):  # nested regions are appended as found
            r, s = self.pending[i]
            self.region(r, s)
            i += 1
        for r, src in self.nested_src.items():
            self.regions[r].captures = src
        kl = next(g for g in self.layouts if g["root"] == self.kernel_root)
        priv = max([g["total_local"] for g in self.layouts if g["root"] != self.kernel_root] + [0])
        return Program(self.code, self.vars, self.var_names, self.regions, self.buffers,
                       kl["total_shared"], kl["total_local"], priv, self.teams, self.workers)


# ---------------------------------------------------------------------------
# Frame variables from the AST (the input of the frame pipeline,
# ompds_layout_build), for programs the reference frontend cannot compile
# (nested regions).  Order and groups follow the reference's lowering and
# codegen (AstLowering.cpp:23-52, 322-345, 375-400;
# Codegen.cpp:413-430; LoweringPasses.cpp:270-280): the kernel frame group
# (0) holds the referenced unmapped host scalars in host order, then the
# target body's declarations and sequential loop counters in source order
# (function 0), then __omp_worker's wf.addr / args.addr (function 1, 8 B,
# pinned); region r owns groups 1 + 2r (its outlined function: a
# parallel-for's counter, then the body's declarations in source order) and
# 2 + 2r (its wrapper, no allocas).  A variable escapes when a region
# captures it: a kernel variable any region references, or -- EXTENSION --
# a region local a nested region references.  Liveness is not derived (no
# IR), so these layouts are the O0 pipeline's (no stack coloring).
# Regions are numbered in lowering order: the kernel's in source order,
# then each region's nested ones as its body is lowered.
# ---------------------------------------------------------------------------

def _names_in(x, out):
    if isinstance(x, dict):
        if x.get("kind") in ("var", "index", "assign"):
            out.add(x.get("name"))
        for v in x.values():
            _names_in(v, out)
    elif isinstance(x, list):
        for v in x:
            _names_in(v, out)
    return out


def _decls(body, out):
    """Declarations (name, elements) of a statement list in source order,
    descending into blocks and sequential loops but not into regions."""
    for st in body:
        k = st["kind"]
        if k == "decl":
            out.append((st["name"], st.get("array_size", 1)))
        elif k == "for":
            out.append((st["counter"], 1))
            _decls(st.get("body", []), out)
        elif k == "block":
            _decls(st.get("body", []), out)
    return out


def _regions_in(body, out):
    """Region statements directly inside `body` (not inside other regions)."""
    for st in body:
        k = st["kind"]
        if k in ("parallel", "parallel_for"):
            out.append(st)
        elif k in ("for", "block"):
            _regions_in(st.get("body", []), out)
    return out


def _region_body(st):
    return st["body"][0].get("body", []) if st["kind"] == "parallel_for" else st.get("body", [])


def derive_frame_vars(ast: dict, kernel_name: str):
    """(frame vars, group roots, group members) of `ast`; see above."""
    from . import layout as LY
    target = ast["target"]
    maps = {m["name"] for m in target["maps"]}
    refd = _names_in(target["body"], set())
    kernel_decls = [(h["name"], 1) for h in ast["host"]
                    if h["name"] not in maps and h["name"] in refd]
    kernel_decls += _decls(target["body"], [])
    # regions in lowering order, with their enclosing region (-1: the kernel)
    regions = []
    queue = [(st, -1) for st in _regions_in(target["body"], [])]
    while queue:
        st, parent = queue.pop(0)
        r = len(regions)
        regions.append((st, parent))
        queue += [(n, r) for n in _regions_in(_region_body(st), [])]

    def locals_of(st):
        out = [(st["body"][0]["counter"], 1)] if st["kind"] == "parallel_for" else []
        return _decls(_region_body(st), out)

    # what each region references, including its nested regions' references
    refs = [_names_in(st, set()) for st, _ in regions]
    kernel_names = {n for n, _ in kernel_decls}
    escapes_k = set()
    escapes_r = [set() for _ in regions]
    for r, (st, parent) in enumerate(regions):
        own = {n for n, _ in locals_of(st)}
        # a name resolves to the innermost enclosing scope that declares it
        for name in refs[r]:
            if name in own:
                continue
            p = parent
            while p >= 0 and name not in {n for n, _ in locals_of(regions[p][0])}:
                p = regions[p][1]
            if p >= 0:
                escapes_r[p].add(name)
            elif name in kernel_names:
                escapes_k.add(name)
    fv = []
    for name, el in kernel_decls:
        fv.append(LY.FrameVar(name, 4 * el, 0, 0, name in escapes_k))
    fv.append(LY.FrameVar("wf.addr", 8, 0, 1, False, True))
    fv.append(LY.FrameVar("args.addr", 8, 0, 1, False, True))
    roots = [kernel_name]
    members = [[kernel_name, "__omp_worker"]]
    for r, (st, _) in enumerate(regions):
        for name, el in locals_of(st):
            fv.append(LY.FrameVar(name, 4 * el, 1 + 2 * r, 0, name in escapes_r[r]))
        roots += [f"__omp_outlined.{r}", f"__omp_outlined.{r}_wrapper"]
        members += [[f"__omp_outlined.{r}"], [f"__omp_outlined.{r}_wrapper"]]
    return fv, roots, members, [p for _, p in regions]


def derive_layouts(ast: dict, kernel_name: str, pipeline: str = "o0"):
    """The program's frame layouts (the shape compile_program takes) from
    derive_frame_vars and the C-ABI frame pipeline."""
    from . import layout as LY
    fv, roots, _, _ = derive_frame_vars(ast, kernel_name)
    lays = LY.build_layouts(fv, len(roots), pipeline)
    return [{"root": r, "total_local": l.total_local, "total_shared": l.total_shared,
             "has_shared_depot": l.has_shared_depot,
             "slots": [{"offset": s.offset, "size": s.size, "align": s.align, "shared": s.shared,
                        "owners": s.owners} for s in l.slots]} for r, l in zip(roots, lays)]


def compile_program(ast: dict, layouts: Sequence[dict], kernel_root: str, teams: int,
                    workers: int) -> Program:
    """Lowers a reference AST (dumpAst JSON) + its frame layouts."""
    return _Compiler(ast, layouts, kernel_root, teams, workers).compile()


# Per worker warp, for programs with nested regions: the lanes' data-sharing
# stacks (a 1/32 share of each per lane).
STACK_SLOT_BYTES = 4096
STACK_OVERFLOW_BYTES = 32768


def describe(prog: Program, buffer_ptrs, step_limit: int = 0,
             stack_slot_bytes: Optional[int] = None,
             stack_overflow_bytes: Optional[int] = None):
    """The ompds_program descriptor of `prog` (and the ctypes arrays it
    points into, which must outlive it)."""
    nested = prog.nested()
    if stack_slot_bytes is None:
        stack_slot_bytes = STACK_SLOT_BYTES if nested else 0
    if stack_overflow_bytes is None:
        stack_overflow_bytes = STACK_OVERFLOW_BYTES if nested else 0
    code = (C.c_int32 * max(len(prog.code), 1))(*prog.code)
    vars_ = (L.ProgVar * max(len(prog.vars), 1))(*[L.ProgVar(s, o, n, 0) for s, o, n in prog.vars])
    caps = [c for r in prog.regions for c in r.captures]
    regs = []
    k = 0
    for r in prog.regions:
        regs.append(L.ProgRegion(r.entry, len(r.captures), k, r.parent, r.frame_bytes,
                                 L.REGION_GLOBALIZE if r.globalize else 0))
        k += len(r.captures)
    regs_a = (L.ProgRegion * max(len(regs), 1))(*regs)
    caps_a = (C.c_int32 * max(len(caps), 1))(*caps)
    bufs = (C.c_void_p * max(len(buffer_ptrs), 1))(*buffer_ptrs)
    desc = L.Program(code=code, n_code=len(prog.code), vars=vars_, n_vars=len(prog.vars),
                     n_regions=len(regs), regions=regs_a, captures=caps_a, n_captures=len(caps),
                     n_buffers=len(buffer_ptrs), buffers=bufs, total_shared=prog.total_shared,
                     total_local=prog.total_local, priv_bytes=prog.priv_bytes,
                     step_limit=step_limit, stack_slot_bytes=stack_slot_bytes,
                     stack_overflow_bytes=stack_overflow_bytes)
    return desc, (code, vars_, regs_a, caps_a, bufs)


def verify(prog: Program) -> int:
    """ompds_program_verify on the program (no GPU needed); OMPDS_OK or
    OMPDS_ERR_INVALID."""
    desc, _keep = describe(prog, [16 * (k + 1) for k in range(len(prog.buffers))])
    return L.lib().ompds_program_verify(C.byref(desc))


def run_program(prog: Program, buffers, prealloc_entries: int = L.DEFAULT_PREALLOC_ENTRIES,
                fail_dynamic_alloc: bool = False, depot_capacity: int = -1,
                max_events: int = 0, stream=None, list_allocator: int = L.LIST_SLAB,
                first_team: int = 0, total_teams: int = 0, teams: int = 0,
                step_limit: int = 0, barrier_arrivals=None,
                stack_slot_bytes: Optional[int] = None,
                stack_overflow_bytes: Optional[int] = None):
    """Launches the program: `buffers` are int32 CUDA tensors, one per mapped
    array, in host declaration order.  Returns regions.Outputs."""
    import torch
    from . import regions as RG
    if len(buffers) != len(prog.buffers):
        raise ValueError("one device buffer per mapped array")
    for b, (name, n, _) in zip(buffers, prog.buffers):
        if b.dtype != torch.int32 or b.numel() != n or not b.is_cuda:
            raise ValueError(f"buffer {name}: int32[{n}] on cuda expected")
    desc, _keep = describe(prog, [b.data_ptr() for b in buffers], step_limit,
                           stack_slot_bytes, stack_overflow_bytes)
    out = RG.Outputs(teams or prog.teams, buffers[0].device if buffers else "cuda", max_events)
    launch = RG.make_launch(teams or prog.teams, prog.workers, prealloc_entries,
                            fail_dynamic_alloc, depot_capacity, max_events > 0, max_events,
                            stream, list_allocator, first_team, total_teams,
                            barrier_arrivals)
    L.check(L.lib().ompds_run_program(C.byref(launch), C.byref(desc), out.stats_ptr(),
                                      out.events_ptr()), "ompds_run_program")
    out.used_on(stream)
    return out
