"""TEST INFRASTRUCTURE -- the CPU oracle's front end (never the product path).

Restates the reference's md_hom semantics so the CUDA path can be checked
against it.  Only tests/, `__graft_entry__.smoke()` and bench.py's
cpu_baseline / `--impl reference` legs may import this module.

What is restated here (Python), and where it comes from:

* ``Affine.parse``              proj/src/views.cpp:45-99     index expressions
* ``parse_scalar`` / typecheck  proj/src/scalar_expr.cpp:93-205, 208-346
* ``compile_node``              proj/src/engine.cpp:34-81    stack bytecode
* ``infer_buffer_sizes``        proj/src/views.cpp:164-184
* ``collapsed_ranges``          proj/src/highlevel.cpp:65-75
* ``validate_md_hom``           proj/src/highlevel.cpp:72-102
* ``execute``                   proj/src/engine.cpp:222-375 (engine::run); the hot
                                loop, prefix pass and output scatter run in the C
                                restatement oracle/mdh_oracle.c
* ``make_inputs``               proj/tests/support.hpp:32-51
* ``buffers_match``             proj/tests/support.hpp:53-80 with value.hpp:63-67

Pinned against: the 17 frozen reference vectors (tests/golden/reference_data/
refs, proj/data/refs) and, when oracle/_ref is built, the unmodified reference
library itself (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
DIM_NAMES = "ijklmnopqrstuvw"  # views.cpp:11


class OracleError(Exception):
    """Mirror of mdh::Error (error.hpp:9-17): a stable code plus a message."""

    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


def fail(code: str, msg: str):
    raise OracleError(code, msg)


# --------------------------------------------------------------------------
# Affine index functions (views.hpp:15-31, views.cpp:21-99)
# --------------------------------------------------------------------------
@dataclass
class Affine:
    c0: int
    coeff: List[int]

    def min_over(self, sizes: Sequence[int]) -> int:
        v = self.c0
        for c, n in zip(self.coeff, sizes):
            v += 0 if c >= 0 else c * (n - 1)
        return v

    def max_over(self, sizes: Sequence[int]) -> int:
        v = self.c0
        for c, n in zip(self.coeff, sizes):
            v += c * (n - 1) if c >= 0 else 0
        return v

    @staticmethod
    def parse(text: str, D: int) -> "Affine":
        a = Affine(0, [0] * D)
        pos = 0
        n = len(text)

        def skip():
            nonlocal pos
            while pos < n and text[pos].isspace():
                pos += 1

        def die(msg):
            fail("ParseError", f"{msg} at column {pos + 1} in index expression '{text}'")

        first = True
        while True:
            skip()
            if pos >= n:
                if first:
                    die("empty index expression")
                break
            sign = 1
            if text[pos] in "+-":
                sign = -1 if text[pos] == "-" else 1
                pos += 1
                skip()
            elif not first:
                die("expected '+' or '-'")
            first = False
            k = 1
            have_int = False
            if pos < n and text[pos].isdigit():
                k = 0
                while pos < n and text[pos].isdigit():
                    k = k * 10 + int(text[pos])
                    pos += 1
                have_int = True
                skip()
                if pos < n and text[pos] == "*":
                    pos += 1
                    skip()
                else:
                    a.c0 += sign * k
                    continue
            if pos >= n or text[pos] not in DIM_NAMES:
                die("expected index name")
            d = DIM_NAMES.index(text[pos]) + 1
            if d > D:
                die("index name beyond dimension count")
            pos += 1
            skip()
            if not have_int and pos < n and text[pos] == "*":
                pos += 1
                skip()
                if pos >= n or not text[pos].isdigit():
                    die("expected integer factor")
                k = 0
                while pos < n and text[pos].isdigit():
                    k = k * 10 + int(text[pos])
                    pos += 1
            a.coeff[d - 1] += sign * k
        return a


def parse_access(text: str, D: int) -> List[Affine]:
    return [Affine.parse(part, D) for part in text.split(",")]


# --------------------------------------------------------------------------
# Scalar function language (scalar_expr.hpp, scalar_expr.cpp)
# --------------------------------------------------------------------------
I64, F64 = "i64", "f64"


@dataclass
class Node:
    kind: str  # Lit In Idx Add Sub Mul Div Min Max Abs Cmp Select
    args: list = field(default_factory=list)
    float_lit: bool = False
    ival: int = 0
    fval: float = 0.0
    buf: int = 0
    acc: int = 0
    dim: int = 0
    type: str = I64


class _Lexer:
    def __init__(self, s: str):
        self.s, self.pos, self.line, self.col = s, 0, 1, 1

    def die(self, msg):
        fail("ParseError", f"{msg} at line {self.line}, column {self.col}")

    def skip_ws(self):
        s = self.s
        while self.pos < len(s) and s[self.pos] in " \t\n\r":
            if s[self.pos] == "\n":
                self.line += 1
                self.col = 1
            else:
                self.col += 1
            self.pos += 1

    def peek(self):
        self.skip_ws()
        return self.s[self.pos] if self.pos < len(self.s) else "\0"

    def advance(self, n):
        self.pos += n
        self.col += n

    def eat(self, c):
        if self.peek() != c:
            return False
        self.advance(1)
        return True

    def expect(self, c):
        if not self.eat(c):
            self.die(f"expected '{c}'")

    def ident(self):
        self.skip_ws()
        st = self.pos
        while self.pos < len(self.s) and (self.s[self.pos].isalpha() or self.s[self.pos] == "_"):
            self.advance(1)
        if st == self.pos:
            self.die("expected identifier")
        return self.s[st:self.pos]

    def number(self) -> Node:
        self.skip_ws()
        s, st = self.s, self.pos
        is_float = False
        while self.pos < len(s) and s[self.pos].isdigit():
            self.advance(1)
        if st == self.pos:
            self.die("expected number")
        if self.pos < len(s) and s[self.pos] == ".":
            is_float = True
            self.advance(1)
            while self.pos < len(s) and s[self.pos].isdigit():
                self.advance(1)
        if self.pos < len(s) and s[self.pos] in "eE":
            is_float = True
            self.advance(1)
            if self.pos < len(s) and s[self.pos] in "+-":
                self.advance(1)
            dg = self.pos
            while self.pos < len(s) and s[self.pos].isdigit():
                self.advance(1)
            if dg == self.pos:
                self.die("expected exponent digits")
        text = s[st:self.pos]
        if is_float:
            return Node("Lit", float_lit=True, fval=float(text), type=F64)
        v = int(text)
        return Node("Lit", ival=v, fval=float(v), type=I64)

    def small_int(self):
        n = self.number()
        if n.float_lit:
            self.die("expected integer")
        return n.ival


def _primary(lx: _Lexer) -> Node:
    c = lx.peek()
    if c == "(":
        lx.advance(1)
        e = _expr(lx)
        lx.expect(")")
        return e
    if c == "-":
        lx.advance(1)
        inner = _primary(lx)
        if inner.kind == "Lit":
            inner.ival, inner.fval = -inner.ival, -inner.fval
            return inner
        return Node("Sub", [Node("Lit"), inner])
    if c.isdigit():
        return lx.number()
    name = lx.ident()
    if name == "in":
        lx.expect("(")
        b = lx.small_int()
        lx.expect(",")
        a = lx.small_int()
        lx.expect(")")
        return Node("In", buf=b, acc=a)
    if name == "idx":
        lx.expect("(")
        d = lx.small_int()
        lx.expect(")")
        return Node("Idx", dim=d, type=I64)
    arity = {"min": ("Min", 2), "max": ("Max", 2), "cmp": ("Cmp", 2), "abs": ("Abs", 1),
             "select": ("Select", 3)}
    if name not in arity:
        lx.die(f"unknown function '{name}'")
    kind, n = arity[name]
    lx.expect("(")
    args = []
    for i in range(n):
        if i:
            lx.expect(",")
        args.append(_expr(lx))
    lx.expect(")")
    return Node(kind, args)


def _term(lx):
    e = _primary(lx)
    while True:
        c = lx.peek()
        if c not in "*/":
            return e
        lx.advance(1)
        e = Node("Mul" if c == "*" else "Div", [e, _primary(lx)])


def _expr(lx):
    e = _term(lx)
    while True:
        c = lx.peek()
        if c not in "+-":
            return e
        lx.advance(1)
        e = Node("Add" if c == "+" else "Sub", [e, _term(lx)])


def parse_scalar(text: str) -> List[Tuple[int, int, Node]]:
    """ScalarExpr::parse (scalar_expr.cpp:318-339) -> [(buf, acc, expr)]."""
    lx = _Lexer(text)
    out = []
    while True:
        if lx.peek() == "\0":
            break
        if lx.ident() != "out":
            lx.die("expected 'out'")
        lx.expect("(")
        b = lx.small_int()
        lx.expect(",")
        a = lx.small_int()
        lx.expect(")")
        lx.expect("=")
        out.append((b, a, _expr(lx)))
        if not lx.eat(";"):
            break
    if lx.peek() != "\0":
        lx.die("trailing input")
    if not out:
        lx.die("expected at least one out(...) assignment")
    return out


def _coerce_float(e: Node) -> bool:
    """scalar_expr.cpp:208-232."""
    if e.kind == "Lit":
        if e.float_lit:
            return True
        e.fval = float(e.ival)
        e.type = F64
        return True
    if e.kind in ("In", "Idx", "Cmp"):
        return e.type == F64
    if e.kind == "Select":
        ok = _coerce_float(e.args[1]) and _coerce_float(e.args[2])
        if ok:
            e.type = F64
        return ok
    for a in e.args:
        if not _coerce_float(a):
            return False
    e.type = F64
    return True


def _unify(a: Node, b: Node, what: str) -> str:
    if a.type == b.type:
        return a.type
    intside = a if a.type == I64 else b
    if not _coerce_float(intside):
        fail("MixedTypes", f"{what} mixes i64 and f64 operands")
    return F64


def _type_expr(e: Node, in_types, in_counts, D):
    for a in e.args:
        _type_expr(a, in_types, in_counts, D)
    k = e.kind
    if k == "Lit":
        e.type = F64 if e.float_lit else I64
    elif k == "In":
        if not (1 <= e.buf <= len(in_types)):
            fail("IndexOutOfBounds", f"in({e.buf},_) references a missing input buffer")
        if not (1 <= e.acc <= in_counts[e.buf - 1]):
            fail("IndexOutOfBounds", f"in({e.buf},{e.acc}) references a missing access")
        e.type = in_types[e.buf - 1]
    elif k == "Idx":
        if not (1 <= e.dim <= D):
            fail("DimOutOfRange", f"idx({e.dim}) with {D} dimensions")
        e.type = I64
    elif k == "Abs":
        e.type = e.args[0].type
    elif k == "Cmp":
        _unify(e.args[0], e.args[1], "cmp")
        e.type = I64
    elif k == "Select":
        if e.args[0].type != I64:
            fail("MixedTypes", "select condition must be i64")
        e.type = _unify(e.args[1], e.args[2], "select")
    else:
        e.type = _unify(e.args[0], e.args[1], "arithmetic")


# --------------------------------------------------------------------------
# Computation (highlevel.hpp:16-32) parsed from the reference JSON dialect
# (json_io.cpp:298-328)
# --------------------------------------------------------------------------
@dataclass
class ViewBuffer:
    name: str
    type: str
    rank: int
    accesses: List[List[Affine]]


FOLD = {"+": 0, "-": 1, "*": 2, "mul": 2, "/": 3, "min": 4, "max": 5}
ASSOC_COMM = {"+", "*", "mul", "min", "max"}  # BinOp::named, mda.cpp:75-83


@dataclass
class Computation:
    name: str
    dim_names: List[str]
    sizes: List[int]
    inputs: List[ViewBuffer]
    outputs: List[ViewBuffer]
    scalar_text: str
    combine: List[Tuple[str, Optional[str]]]  # ("cc", None) | ("pw", op) | ("ps", op)
    assigns: list = field(default_factory=list)

    @property
    def D(self):
        return len(self.sizes)

    @staticmethod
    def from_json(text) -> "Computation":
        j = json.loads(text) if isinstance(text, str) else text
        D = len(j["sizes"])
        if len(j["dims"]) != D:
            fail("ParseError", f"computation '{j['name']}': dims and sizes disagree in length")

        def vb(b):
            if b["type"] not in (I64, F64):
                fail("ParseError", f"unknown element type '{b['type']}' (expected i64 or f64)")
            return ViewBuffer(b["name"], b["type"], int(b["rank"]),
                              [parse_access(a, D) for a in b["accesses"]])

        comb = []
        for d, s in enumerate(j["combine"]):
            if s == "cc":
                comb.append(("cc", None))
            elif s.startswith("pw:") or s.startswith("ps:"):
                op = s[3:]
                if op not in FOLD:
                    fail("UnknownOperator", f"unknown binary operator '{op}'")
                comb.append((s[:2], op))
            else:
                fail("ParseError", f"combine operator {d + 1}: '{s}' is not cc, pw:<op>, or ps:<op>")
        c = Computation(j["name"], list(j["dims"]), [int(x) for x in j["sizes"]],
                        [vb(b) for b in j["inputs"]], [vb(b) for b in j["outputs"]],
                        j["scalar"], comb)
        c.typecheck()
        c.validate_structure()
        return c

    def to_json(self) -> dict:
        def acc_text(acc):
            parts = []
            for a in acc:
                terms = []
                for d, k in enumerate(a.coeff):
                    if k:
                        terms.append(("-" if k < 0 else "+") + (f"{abs(k)}*" if abs(k) != 1 else "")
                                     + DIM_NAMES[d])
                if a.c0 or not terms:
                    terms.append(("-" if a.c0 < 0 else "+") + str(abs(a.c0)))
                t = "".join(terms)
                parts.append(t[1:] if t.startswith("+") else t)
            return ", ".join(parts)

        def vbj(b):
            return {"name": b.name, "type": b.type, "rank": b.rank,
                    "accesses": [acc_text(a) for a in b.accesses]}

        return {"name": self.name, "dims": self.dim_names, "sizes": self.sizes,
                "inputs": [vbj(b) for b in self.inputs], "outputs": [vbj(b) for b in self.outputs],
                "scalar": self.scalar_text,
                "combine": [k if k == "cc" else f"{k}:{op}" for k, op in self.combine]}

    # scalar_expr.cpp:346-381 (typecheck, canonical (buf, acc) order)
    def typecheck(self):
        assigns = parse_scalar(self.scalar_text)
        in_types = [b.type for b in self.inputs]
        in_counts = [len(b.accesses) for b in self.inputs]
        seen = [[False] * len(b.accesses) for b in self.outputs]
        for b, a, e in assigns:
            if not (1 <= b <= len(self.outputs)):
                fail("IndexOutOfBounds", f"out({b},_) references a missing output buffer")
            if not (1 <= a <= len(self.outputs[b - 1].accesses)):
                fail("IndexOutOfBounds", f"out({b},{a}) references a missing access")
            if seen[b - 1][a - 1]:
                fail("IndexOutOfBounds", f"out({b},{a}) assigned twice")
            seen[b - 1][a - 1] = True
            _type_expr(e, in_types, in_counts, self.D)
            want = self.outputs[b - 1].type
            if e.type != want:
                if want == F64 and _coerce_float(e):
                    continue
                fail("MixedTypes", f"out({b},{a}) expression type {e.type} does not match buffer type {want}")
        for b, row in enumerate(seen):
            for a, s in enumerate(row):
                if not s:
                    fail("IndexOutOfBounds", f"out({b + 1},{a + 1}) never assigned")
        self.assigns = sorted(assigns, key=lambda t: (t[0], t[1]))

    # highlevel.cpp:15-59
    def validate_structure(self):
        D = self.D
        if D == 0:
            fail("DimOutOfRange", f"computation '{self.name}' has no dimensions")
        for d, n in enumerate(self.sizes):
            if n < 1:
                fail("OutOfRange", f"dimension {d + 1} of '{self.name}' has non-positive size")
        if len(self.combine) != D:
            fail("DimOutOfRange", "combine operator count mismatch")
        for side, bufs in (("input", self.inputs), ("output", self.outputs)):
            if not bufs:
                fail("IndexOutOfBounds", f"'{self.name}' has no {side} buffers")
            for b in bufs:
                if b.rank < 1:
                    fail("DimOutOfRange", f"buffer '{b.name}' has rank {b.rank}")
                if not b.accesses:
                    fail("IndexOutOfBounds", f"buffer '{b.name}' has no accesses")
                for a in b.accesses:
                    if len(a) != b.rank:
                        fail("DimOutOfRange", f"buffer '{b.name}' access arity does not match rank")

    def collapsed_sizes(self) -> List[int]:
        return [1 if k == "pw" else n for n, (k, _) in zip(self.sizes, self.combine)]

    def fold_op(self) -> Optional[str]:
        for k, op in self.combine:
            if k != "cc":
                return op
        return None


def validate_md_hom(c: Computation) -> List[Tuple[str, str, int, int]]:
    """highlevel.cpp:72-102: every non-cc dim shares one assoc+comm op."""
    viol = []
    first = 0
    for d, (k, op) in enumerate(c.combine, start=1):
        if k == "cc":
            continue
        if op not in ASSOC_COMM:
            viol.append(("MixedIncompatibleOperators",
                         f"dimension {d} folds with '{op}', which is not associative and commutative", d, d))
            continue
        if first == 0:
            first = d
            continue
        if FOLD[c.combine[first - 1][1]] != FOLD[op]:
            viol.append(("MixedIncompatibleOperators",
                         f"dimensions {first} and {d} fold with different operators", first, d))
    return viol


def infer_buffer_sizes(bufs: Sequence[ViewBuffer], sizes: Sequence[int]) -> List[List[int]]:
    """views.cpp:164-184 over the box [0, N_d) per dimension."""
    out = []
    for b in bufs:
        dims = [0] * b.rank
        for acc in b.accesses:
            for r, a in enumerate(acc):
                lo = a.min_over(sizes)
                if lo < 0:
                    fail("NegativeIndexReachable", f"buffer '{b.name}' access reaches coordinate {lo}")
                dims[r] = max(dims[r], a.max_over(sizes) + 1)
        out.append(dims)
    return out


def input_shapes(c: Computation):
    return infer_buffer_sizes(c.inputs, c.sizes)


def output_shapes(c: Computation):
    return infer_buffer_sizes(c.outputs, c.collapsed_sizes())


# --------------------------------------------------------------------------
# Bytecode (engine.cpp:34-81)
# --------------------------------------------------------------------------
OPS = ["LIT_I", "LIT_F", "IN_I", "IN_F", "IDX", "ADD_I", "ADD_F", "SUB_I", "SUB_F", "MUL_I", "MUL_F",
       "DIV_I", "DIV_F", "MIN_I", "MIN_F", "MAX_I", "MAX_F", "ABS_I", "ABS_F", "CMP_I", "CMP_F", "SELECT"]
OPC = {n: i for i, n in enumerate(OPS)}


class Instr(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("arg", ctypes.c_int32), ("ilit", ctypes.c_int64),
                ("flit", ctypes.c_double)]


def comp_offset(bufs: Sequence[ViewBuffer], b: int, a: int) -> int:
    """ViewSpec::comp_offset (views.cpp:152-157), 1-based (b, a)."""
    return sum(len(x.accesses) for x in bufs[:b - 1]) + (a - 1)


def compile_node(e: Node, out: list, inputs: Sequence[ViewBuffer]) -> int:
    f = e.type == F64
    k = e.kind
    if k == "Lit":
        out.append(("LIT_F", 0, 0, e.fval) if f else ("LIT_I", 0, e.ival, 0.0))
        return 1
    if k == "In":
        out.append(("IN_F" if f else "IN_I", comp_offset(inputs, e.buf, e.acc), 0, 0.0))
        return 1
    if k == "Idx":
        out.append(("IDX", e.dim - 1, 0, 0.0))
        return 1
    if k == "Abs":
        d = compile_node(e.args[0], out, inputs)
        out.append(("ABS_F" if f else "ABS_I", 0, 0, 0.0))
        return d
    if k == "Cmp":
        d1 = compile_node(e.args[0], out, inputs)
        d2 = compile_node(e.args[1], out, inputs)
        out.append(("CMP_F" if e.args[0].type == F64 else "CMP_I", 0, 0, 0.0))
        return max(d1, 1 + d2)
    if k == "Select":
        d1 = compile_node(e.args[0], out, inputs)
        d2 = compile_node(e.args[1], out, inputs)
        d3 = compile_node(e.args[2], out, inputs)
        out.append(("SELECT", 0, 0, 0.0))
        return max(d1, 1 + d2, 2 + d3)
    d1 = compile_node(e.args[0], out, inputs)
    d2 = compile_node(e.args[1], out, inputs)
    name = {"Add": "ADD", "Sub": "SUB", "Mul": "MUL", "Div": "DIV", "Min": "MIN", "Max": "MAX"}[k]
    out.append((name + ("_F" if f else "_I"), 0, 0, 0.0))
    return max(d1, 1 + d2)


# --------------------------------------------------------------------------
# C restatement binding
# --------------------------------------------------------------------------
_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "libmdh_oracle.so")
        if not os.path.exists(path):
            build()
        _lib = ctypes.CDLL(path)
    return _lib


def build():
    import subprocess
    subprocess.check_call(["make", "-s", "-C", _HERE, "oracle"])


def _ptrs(arrs):
    return (ctypes.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])


def _i64(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def _i32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def lex_plan(sizes):
    """engine.cpp:215-220: one loop per dimension, ascending."""
    return [(d, n, 1) for d, n in enumerate(sizes)]


def execute(c: Computation, inputs: Sequence[np.ndarray], plan=None):
    """engine::run (engine.cpp:222-375).  `inputs` are int64 / float64 arrays
    of at least the inferred extents.  Returns [(values, defined_mask)] per
    output buffer, at the inferred output extents."""
    viol = validate_md_hom(c)
    if viol:
        fail("MixedIncompatibleOperators", viol[0][1])
    D = c.D
    plan = plan or lex_plan(c.sizes)
    prod = [1] * D
    for d, cnt, _ in plan:
        prod[d] *= cnt
    for d in range(D):
        if prod[d] != c.sizes[d]:
            fail("InvalidConfig", f"nest loop counts over dimension {d + 1} cover {prod[d]} of {c.sizes[d]}")
    need = input_shapes(c)
    if len(inputs) != len(c.inputs):
        fail("BufferTooSmall", f"expected {len(c.inputs)} input buffers, got {len(inputs)}")
    arrs = []
    for b, (vb, x) in enumerate(zip(c.inputs, inputs)):
        x = np.ascontiguousarray(x, dtype=np.float64 if vb.type == F64 else np.int64)
        if x.ndim != vb.rank:
            fail("BufferTooSmall", f"input buffer '{vb.name}' rank mismatch")
        for r in range(vb.rank):
            if x.shape[r] < need[b][r]:
                fail("BufferTooSmall", f"input buffer '{vb.name}' extent {x.shape[r]} < required {need[b][r]}")
        arrs.append(x)
    # AccessPlan per (buffer, access): engine.cpp:266-286
    acc_data, c0s, cjs = [], [], []
    for vb, x in zip(c.inputs, arrs):
        strides = [1] * vb.rank
        for r in range(vb.rank - 2, -1, -1):
            strides[r] = strides[r + 1] * x.shape[r + 1]
        for acc in vb.accesses:
            acc_data.append(x)
            c0s.append(sum(strides[r] * acc[r].c0 for r in range(vb.rank)))
            cjs.append([sum(strides[r] * acc[r].coeff[d] for r in range(vb.rank)) for d in range(D)])
    # programs
    code, starts, lens, pf = [], [], [], []
    max_depth = 1
    for _, _, e in c.assigns:
        prog = []
        max_depth = max(max_depth, compile_node(e, prog, c.inputs))
        starts.append(len(code))
        lens.append(len(prog))
        pf.append(1 if e.type == F64 else 0)
        code.extend(prog)
    instrs = (Instr * len(code))(*[Instr(OPC[o], a, il, fl) for o, a, il, fl in code])
    # accumulator over collapsed ranges (engine.cpp:313-335)
    coll = c.collapsed_sizes()
    acc_stride = [0] * D
    cells = 1
    for d in range(D - 1, -1, -1):
        if c.combine[d][0] != "pw":
            acc_stride[d] = cells
            cells *= coll[d]
    acc_vals = [np.zeros(cells, dtype=np.float64 if f else np.int64) for f in pf]
    acc_def = np.zeros(cells, dtype=np.uint8)
    fold = FOLD[c.fold_op()] if c.fold_op() else 0
    err = ctypes.create_string_buffer(512)
    L = lib()
    if cells > 0:
        rc = L.oracle_run(
            ctypes.c_int(D), ctypes.c_int(len(acc_data)), _ptrs(acc_data), _i64(c0s).ctypes.data_as(ctypes.c_void_p),
            _i64(np.array(cjs, dtype=np.int64).reshape(-1)).ctypes.data_as(ctypes.c_void_p),
            ctypes.c_int(len(pf)), _i32(starts).ctypes.data_as(ctypes.c_void_p),
            _i32(lens).ctypes.data_as(ctypes.c_void_p), instrs, _i32(pf).ctypes.data_as(ctypes.c_void_p),
            ctypes.c_int(max_depth), _i64(acc_stride).ctypes.data_as(ctypes.c_void_p), _ptrs(acc_vals),
            acc_def.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(fold), ctypes.c_int(len(plan)),
            _i32([p[0] for p in plan]).ctypes.data_as(ctypes.c_void_p),
            _i64([p[1] for p in plan]).ctypes.data_as(ctypes.c_void_p),
            _i64([p[2] for p in plan]).ctypes.data_as(ctypes.c_void_p), err, ctypes.c_int(512))
        if rc:
            code_, _, msg = err.value.decode().partition(": ")
            fail(code_, msg)
    # prefix dims (engine.cpp:337-353)
    for d in range(D):
        if c.combine[d][0] != "ps":
            continue
        L.oracle_prefix(ctypes.c_int64(cells), ctypes.c_int64(acc_stride[d]), ctypes.c_int64(coll[d]),
                        ctypes.c_int(len(pf)), _i32(pf).ctypes.data_as(ctypes.c_void_p), _ptrs(acc_vals),
                        acc_def.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(fold))
    # output view scatter (views.cpp:242-275)
    oshapes = output_shapes(c)
    outs = [np.zeros(s, dtype=np.float64 if vb.type == F64 else np.int64) for vb, s in zip(c.outputs, oshapes)]
    defs = [np.zeros(s, dtype=np.uint8) for s in oshapes]
    oc0, ocj, comp_of, odata, odef = [], [], [], [], []
    comp = 0
    for b, vb in enumerate(c.outputs):
        shp = oshapes[b]
        strides = [1] * vb.rank
        for r in range(vb.rank - 2, -1, -1):
            strides[r] = strides[r + 1] * shp[r + 1]
        for acc in vb.accesses:
            oc0.append(sum(strides[r] * acc[r].c0 for r in range(vb.rank)))
            ocj.append([sum(strides[r] * acc[r].coeff[d] for r in range(vb.rank)) for d in range(D)])
            comp_of.append(comp)
            odata.append(outs[b])
            odef.append(defs[b])
            comp += 1
    rc = L.oracle_scatter(ctypes.c_int(D), _i64(coll).ctypes.data_as(ctypes.c_void_p),
                          _i64(acc_stride).ctypes.data_as(ctypes.c_void_p), ctypes.c_int(len(oc0)),
                          _i64(oc0).ctypes.data_as(ctypes.c_void_p),
                          _i64(np.array(ocj, dtype=np.int64).reshape(-1)).ctypes.data_as(ctypes.c_void_p),
                          _i32(comp_of).ctypes.data_as(ctypes.c_void_p), _i32(pf).ctypes.data_as(ctypes.c_void_p),
                          _ptrs(odata), _ptrs(odef), _ptrs(acc_vals), err, ctypes.c_int(512))
    if rc:
        code_, _, msg = err.value.decode().partition(": ")
        fail(code_, msg)
    return list(zip(outs, [d.astype(bool) for d in defs]))


def make_inputs(c: Computation, seed: int) -> List[np.ndarray]:
    """support.hpp:32-51: values below(11) - 5 from mt19937_64, x0.25 for f64."""
    shapes = input_shapes(c)
    ks = [np.zeros(int(np.prod(s)), dtype=np.int64) for s in shapes]
    counts = _i64([k.size for k in ks])
    lib().oracle_make_inputs(ctypes.c_uint64(seed), ctypes.c_int(len(ks)), counts.ctypes.data_as(ctypes.c_void_p),
                             _ptrs(ks))
    out = []
    for vb, k, s in zip(c.inputs, ks, shapes):
        out.append((0.25 * k.astype(np.float64) if vb.type == F64 else k).reshape(s))
    return out


def mt19937_64(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=np.uint64)
    lib().oracle_mt64(ctypes.c_uint64(seed), ctypes.c_int64(n), out.ctypes.data_as(ctypes.c_void_p))
    return out


def nearly_equal(a, b, rel_tol):
    """value.hpp:63-67, vectorised."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)
    return (a == b) | (np.abs(a - b) <= rel_tol * scale)


def buffers_match(got, want, rel_tol):
    """support.hpp:53-80.  got/want: [(values, defined)]; returns (ok, why)."""
    if len(got) != len(want):
        return False, "output buffer count differs"
    for b, ((gv, gd), (wv, wd)) in enumerate(zip(got, want)):
        if tuple(gv.shape) != tuple(wv.shape):
            return False, f"dims differ on buffer {b}"
        if not np.array_equal(gd, wd):
            return False, f"definedness differs on buffer {b}"
        m = wd.astype(bool)
        if np.issubdtype(wv.dtype, np.integer):
            bad = (gv != wv) & m
        else:
            bad = ~nearly_equal(gv, wv, rel_tol) & m
        if bad.any():
            t = int(np.flatnonzero(bad.ravel())[0])
            return False, f"buffer {b} cell {t}: {gv.ravel()[t]} != {wv.ravel()[t]}"
    return True, ""


# --------------------------------------------------------------------------
# ++ slicing (the homomorphic property; test_highlevel.cpp:203-211)
# --------------------------------------------------------------------------
def concat_slice(c: Computation, dim: int, lo: int, hi: int) -> Tuple[Computation, List[List[int]]]:
    """The md_hom restricted to [lo, hi) of concatenation dimension `dim`
    (0-based), re-indexed to start at 0: sizes[dim] = hi - lo and every
    affine access gets c0 += coeff[dim] * lo.  The sub-problem reads the SAME
    (full) input buffers.  Returns (sub_computation, out_shift) where
    out_shift[b][r] is the coordinate offset of the sub-result inside output
    buffer b (valid when each output rank depends on `dim` through one coeff).
    """
    if c.combine[dim][0] != "cc":
        fail("InvalidConfig", "can only slice a concatenation dimension")
    import copy
    s = copy.deepcopy(c)
    s.sizes[dim] = hi - lo
    for vb in s.inputs:
        for acc in vb.accesses:
            for a in acc:
                a.c0 += a.coeff[dim] * lo
    shifts = [[a.coeff[dim] * lo for a in vb.accesses[0]] for vb in c.outputs]
    return s, shifts


def pw_outer_plan(c: Computation):
    """A nest with the point-wise dims outermost (in their own order), then the
    other dims.  Every result cell still folds its fiber in ascending lex
    order over the pw dims, so the values are identical to lex_plan's
    (engine.cpp:177-189 folds in visit order); only the cache behaviour of
    the oracle changes."""
    pw = [d for d in range(c.D) if c.combine[d][0] == "pw"]
    rest = [d for d in range(c.D) if c.combine[d][0] != "pw"]
    return [(d, c.sizes[d], 1) for d in pw + rest]


def execute_slice(c: Computation, inputs, dim: int, lo: int, hi: int):
    """Oracle outputs of the [lo, hi) slab of cc-dimension `dim`, plus the
    per-output-buffer coordinate offset of that slab in the full result."""
    s, shifts = concat_slice(c, dim, lo, hi)
    return execute(s, inputs, pw_outer_plan(s)), shifts


def execute_box(c: Computation, inputs, box):
    """Oracle outputs on a box of cc dims {dim: (lo, hi)} (several ++ slices
    composed), with the per-output-buffer coordinate offsets."""
    cur, total = c, None
    for dim, (lo, hi) in sorted(box.items()):
        cur, sh = concat_slice(cur, dim, lo, hi)
        total = sh if total is None else [[a + b for a, b in zip(x, y)] for x, y in zip(total, sh)]
    return execute(cur, inputs, pw_outer_plan(cur)), total
