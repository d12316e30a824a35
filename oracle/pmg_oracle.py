"""Independent CPU oracle for PolyMage-GPU pipelines — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this module.  It shares no code with the CUDA path (paper_1909_07190_b200/): it has its own tokenizer,
parser, type rules and evaluator, and it never imports the product package (nor the reverse).

What it computes (the plain definition the fused GPU kernels must reproduce):
  PAPER.md §2.2: a pipeline is a DAG of stages, "each stage is a function mapping a
  multi-dimensional integer domain to values"; overlapped tiling performs "redundant computations to
  ensure that all the data required to compute the output of a tile (liveouts) is available within
  that tile" — i.e. fusion, OTPW and hybrid tiling (§4, §5) change only WHERE a stage value lives,
  never WHAT it is.  Hence the method's result is exactly the stage-by-stage evaluation below:

      for stage S in topological order (ties: declaration order)
          for every point p of domain(S):
              S[p] = expr_S(p), every read P(q) := P[clamp(q, domain(P))]   # DESIGN.md reading R1
      return the liveouts

Readings of points where the paper is silent (DESIGN.md §"Readings"):
  R1  reads clamp each index to the producer's domain after the index expression is evaluated;
  R3  f32 arithmetic exactly as written, left to right, round-to-nearest per operation, no contraction;
      IEEE '/' and sqrt; float literals are f32(f64(decimal text));
  R4  int32 arithmetic (wraps, two's complement); '/' floors and '%' takes the divisor's sign
      (a == (a/b)*b + a%b); x/0 == 0 and x%0 == 0; a shift count is clamped to [0, 32] first, so
      a<<c == a*2^c mod 2^32 and a>>c == floor(a/2^c) for every int32 count; f32 -> int truncates toward
      zero, saturates to [-2^31, 2^31-1] and maps NaN to 0; narrowing conversions wrap;
  R5  min(a,b) = b<a ? b : a, max(a,b) = b>a ? b : a, lerp(a,b,w) = a*(1-w) + b*w, select is exact.

Evaluation is whole-domain per stage with numpy (vectorised, no blocking, fusion or reordering of any
expression); with precision='f64' every float value is carried in float64 instead (used by the tests
to bound the f32 result against exact arithmetic).  Parity status per function: see DESIGN.md
"Oracle pins"; every function here is pinned by tests/test_oracle_*.py.
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field

import numpy as np

DTYPES = {"f32": np.float32, "i32": np.int32, "i16": np.int16, "u16": np.uint16, "u8": np.uint8}
BUILTINS = {"min": 2, "max": 2, "abs": 1, "absd": 2, "clamp": 3, "select": 3, "lerp": 3, "sqrt": 1,
            "f32": 1, "i32": 1, "i16": 1, "u16": 1, "u8": 1, "sat_u8": 1, "sat_u16": 1}


class OracleError(Exception):
    """Parse / validation / evaluation error; message carries 'line:col' where applicable."""


# ----------------------------------------------------------------------------------------------- lexer
_TOKEN = re.compile(r"""
    (?P<ws>[ \t\r]+) | (?P<comment>\#[^\n]*) | (?P<nl>\n) |
    (?P<num>(\d+\.\d*|\.\d+|\d+)([eE][+-]?\d+)?) |
    (?P<id>[A-Za-z_][A-Za-z_0-9]*) |
    (?P<op>\.\.|<=|>=|==|!=|&&|\|\||<<|>>|[-+*/%()<>,:=\[\]!])
""", re.VERBOSE)


@dataclass
class Tok:
    kind: str
    text: str
    line: int
    col: int


def _lex(text: str):
    toks, pos, line, lstart = [], 0, 1, 0
    while pos < len(text):
        m = _TOKEN.match(text, pos)
        if not m:
            raise OracleError(f"{line}:{pos - lstart + 1}: unexpected character {text[pos]!r}")
        k = m.lastgroup
        if k == "nl":
            toks.append(Tok("nl", "\n", line, pos - lstart + 1))
            line, lstart = line + 1, m.end()
        elif k not in ("ws", "comment"):
            toks.append(Tok(k, m.group(), line, pos - lstart + 1))
        pos = m.end()
    toks.append(Tok("eof", "", line, pos - lstart + 1))
    return toks


# ------------------------------------------------------------------------------------------------- AST
@dataclass
class Num:
    value: float | int
    is_float: bool
    text: str


@dataclass
class Name:          # stage variable or parameter
    name: str


@dataclass
class Call:          # builtin function
    fn: str
    args: list


@dataclass
class Access:        # image / stage read, one index expression per producer dim
    target: str
    args: list
    pos: str = ""


@dataclass
class TableRead:
    table: str
    index: object


@dataclass
class Bin:
    op: str
    a: object
    b: object


@dataclass
class Un:
    op: str
    a: object


@dataclass
class ImageDecl:
    name: str
    extents: list
    dtype: str


@dataclass
class TableDecl:
    name: str
    extent: object
    dtype: str


@dataclass
class StageDecl:
    name: str
    vars: list
    extents: list
    dtype: str
    expr: object
    line: int


@dataclass
class Program:
    params: list = field(default_factory=list)
    images: dict = field(default_factory=dict)
    tables: dict = field(default_factory=dict)
    stages: dict = field(default_factory=dict)      # declaration order preserved
    liveouts: list = field(default_factory=list)

    # ---- structure helpers (pure) ----
    def producers(self, stage: str) -> list:
        out = []
        _collect_accesses(self.stages[stage].expr, out)
        return [a.target for a in out if a.target in self.stages]

    def topo_order(self) -> list:
        """Producers before consumers; ties broken by declaration order."""
        order, done = [], set()
        names = list(self.stages)
        while len(order) < len(names):
            for n in names:
                if n not in done and all(p in done for p in self.producers(n) if p != n):
                    order.append(n)
                    done.add(n)
                    break
            else:  # pragma: no cover - validated at parse time
                raise OracleError("cyclic reference")
        return order


def _collect_accesses(e, out):
    if isinstance(e, Access):
        out.append(e)
        for a in e.args:
            _collect_accesses(a, out)
    elif isinstance(e, TableRead):
        _collect_accesses(e.index, out)
    elif isinstance(e, Call):
        for a in e.args:
            _collect_accesses(a, out)
    elif isinstance(e, Bin):
        _collect_accesses(e.a, out)
        _collect_accesses(e.b, out)
    elif isinstance(e, Un):
        _collect_accesses(e.a, out)


# ---------------------------------------------------------------------------------------------- parser
class _Parser:
    def __init__(self, text):
        self.t = _lex(text)
        self.i = 0
        self.depth = 0

    def peek(self):
        # newlines are insignificant inside parentheses / brackets (statement continuation)
        while self.depth > 0 and self.t[self.i].kind == "nl":
            self.i += 1
        return self.t[self.i]

    def next(self):
        tok = self.peek()
        self.i += 1
        return tok

    def err(self, tok, msg):
        return OracleError(f"{tok.line}:{tok.col}: {msg}")

    def expect(self, text):
        tok = self.next()
        if tok.text != text:
            raise self.err(tok, f"expected {text!r}, found {tok.text or tok.kind!r}")
        if text in "([":
            self.depth += 1
        elif text in ")]":
            self.depth -= 1
        return tok

    def ident(self):
        tok = self.next()
        if tok.kind != "id":
            raise self.err(tok, f"expected identifier, found {tok.text or tok.kind!r}")
        return tok.text

    def end_stmt(self):
        tok = self.next()
        if tok.kind not in ("nl", "eof"):
            raise self.err(tok, f"expected end of statement, found {tok.text!r}")

    # expression grammar (C-like precedence)
    def expr(self):
        return self.binary(0)

    _LEVELS = [["||"], ["&&"], ["==", "!="], ["<", "<=", ">", ">="], ["<<", ">>"], ["+", "-"], ["*", "/", "%"]]

    def binary(self, lvl):
        if lvl == len(self._LEVELS):
            return self.unary()
        a = self.binary(lvl + 1)
        while self.peek().text in self._LEVELS[lvl] and self.peek().kind == "op":
            op = self.next().text
            a = Bin(op, a, self.binary(lvl + 1))
        return a

    def unary(self):
        tok = self.peek()
        if tok.kind == "op" and tok.text in ("-", "!"):
            self.next()
            return Un(tok.text, self.unary())
        return self.primary()

    def primary(self):
        tok = self.next()
        if tok.kind == "num":
            txt = tok.text
            if re.fullmatch(r"\d+", txt):
                return Num(int(txt), False, txt)
            return Num(float(txt), True, txt)
        if tok.kind == "id":
            nxt = self.peek()
            if nxt.text == "(":
                self.expect("(")
                args = []
                if self.peek().text != ")":
                    args.append(self.expr())
                    while self.peek().text == ",":
                        self.next()
                        args.append(self.expr())
                self.expect(")")
                if tok.text in BUILTINS:
                    if len(args) != BUILTINS[tok.text]:
                        raise self.err(tok, f"{tok.text} takes {BUILTINS[tok.text]} arguments")
                    return Call(tok.text, args)
                return Access(tok.text, args, f"{tok.line}:{tok.col}")
            if nxt.text == "[":
                self.expect("[")
                idx = self.expr()
                self.expect("]")
                return TableRead(tok.text, idx)
            return Name(tok.text)
        if tok.text == "(":
            self.depth += 1
            e = self.expr()
            self.expect(")")
            return e
        raise self.err(tok, f"unexpected {tok.text or tok.kind!r}")

    def program(self) -> Program:
        prog = Program()
        while True:
            tok = self.next()
            if tok.kind == "eof":
                break
            if tok.kind == "nl":
                continue
            if tok.kind != "id":
                raise self.err(tok, f"expected a statement, found {tok.text!r}")
            kw = tok.text
            if kw == "param":
                prog.params.append(self.ident())
                while self.peek().text == ",":
                    self.next()
                    prog.params.append(self.ident())
            elif kw == "image":
                name = self.ident()
                self.expect("(")
                ext = [self.expr()]
                while self.peek().text == ",":
                    self.next()
                    ext.append(self.expr())
                self.expect(")")
                self.expect(":")
                prog.images[name] = ImageDecl(name, ext, self.dtype())
            elif kw == "table":
                name = self.ident()
                self.expect("(")
                ext = self.expr()
                self.expect(")")
                self.expect(":")
                prog.tables[name] = TableDecl(name, ext, self.dtype())
            elif kw == "stage":
                name = self.ident()
                self.expect("(")
                vs = [self.ident()]
                while self.peek().text == ",":
                    self.next()
                    vs.append(self.ident())
                self.expect(")")
                self.expect("[")
                ext = [self.expr()]
                while self.peek().text == ",":
                    self.next()
                    ext.append(self.expr())
                self.expect("]")
                self.expect(":")
                dt = self.dtype()
                self.expect("=")
                e = self.expr()
                if len(vs) != len(ext) or not 1 <= len(vs) <= 3:
                    raise self.err(tok, f"stage {name}: {len(vs)} variables but {len(ext)} extents (1-3 dims)")
                if name in prog.stages or name in prog.images or name in prog.tables:
                    raise self.err(tok, f"duplicate name {name!r}")
                prog.stages[name] = StageDecl(name, vs, ext, dt, e, tok.line)
            elif kw == "liveout":
                prog.liveouts.append(self.ident())
                while self.peek().text == ",":
                    self.next()
                    prog.liveouts.append(self.ident())
            else:
                raise self.err(tok, f"unknown statement {kw!r}")
            self.end_stmt()
        return prog

    def dtype(self):
        tok = self.next()
        if tok.text not in DTYPES:
            raise self.err(tok, f"unknown element type {tok.text!r}")
        return tok.text


def parse(text: str) -> Program:
    """Parse and validate pipeline text (grammar: DESIGN.md §"Pipeline language"; extends SPEC.md l.81)."""
    prog = _Parser(text).program()
    _validate(prog)
    return prog


def _validate(prog: Program):
    if not prog.stages:
        raise OracleError("no stages")
    if not prog.liveouts:
        raise OracleError("no liveouts")
    known = set(prog.images) | set(prog.stages)
    for s in prog.stages.values():
        scope = set(s.vars) | set(prog.params)
        _check_names(s.expr, scope, prog, s)
    for lo in prog.liveouts:
        if lo not in prog.stages:
            raise OracleError(f"liveout {lo!r} is not a stage")
    # cycles ("cyclic reference")
    state = {}

    def visit(n, path):
        if state.get(n) == 1:
            raise OracleError(f"cyclic reference: {' -> '.join(path + [n])}")
        if state.get(n) == 2:
            return
        state[n] = 1
        for p in prog.producers(n):
            visit(p, path + [n])
        state[n] = 2

    for n in prog.stages:
        visit(n, [])
    # every stage reachable from a liveout
    seen, todo = set(), list(prog.liveouts)
    while todo:
        n = todo.pop()
        if n in seen:
            continue
        seen.add(n)
        todo.extend(prog.producers(n))
    dead = [n for n in prog.stages if n not in seen]
    if dead:
        raise OracleError(f"stage {dead[0]!r} is unreachable from every liveout")
    _ = known


def _check_names(e, scope, prog, s):
    if isinstance(e, Name):
        if e.name not in scope:
            raise OracleError(f"line {s.line}: undeclared name {e.name!r} in stage {s.name}")
    elif isinstance(e, Access):
        if e.target in prog.images:
            nd = len(prog.images[e.target].extents)
        elif e.target in prog.stages:
            nd = len(prog.stages[e.target].vars)
        else:
            raise OracleError(f"{e.pos}: reference to undeclared stage/image {e.target!r}")
        if len(e.args) != nd:
            raise OracleError(f"{e.pos}: {e.target} has {nd} dims, read with {len(e.args)} indices")
        for a in e.args:
            _check_names(a, scope, prog, s)
    elif isinstance(e, TableRead):
        if e.table not in prog.tables:
            raise OracleError(f"line {s.line}: undeclared table {e.table!r}")
        _check_names(e.index, scope, prog, s)
    elif isinstance(e, Call):
        for a in e.args:
            _check_names(a, scope, prog, s)
    elif isinstance(e, Bin):
        _check_names(e.a, scope, prog, s)
        _check_names(e.b, scope, prog, s)
    elif isinstance(e, Un):
        _check_names(e.a, scope, prog, s)


# ------------------------------------------------------------------------------------------- evaluation
class _V:
    """A value: numpy array (or 0-d) plus its kind, 'i' (int32) or 'f' (float)."""
    __slots__ = ("a", "k")

    def __init__(self, a, k):
        self.a, self.k = a, k


class Evaluator:
    def __init__(self, prog: Program, params: dict, precision: str = "f32"):
        if precision not in ("f32", "f64"):
            raise OracleError("precision must be 'f32' or 'f64'")
        self.p = prog
        self.params = {k: int(v) for k, v in params.items()}
        missing = [n for n in prog.params if n not in self.params]
        if missing:
            raise OracleError(f"missing parameter values: {missing}")
        self.F = np.float32 if precision == "f32" else np.float64
        self.values = {}

    # integer parameter arithmetic for extents (floor division, R4)
    def iext(self, e) -> int:
        v = self._ev(e, {})
        if v.k != "i" or np.ndim(v.a) != 0:
            raise OracleError("extent must be a scalar integer expression")
        return int(v.a)

    def shape_of(self, name):
        if name in self.p.images:
            return tuple(self.iext(x) for x in self.p.images[name].extents)
        if name in self.p.stages:
            return tuple(self.iext(x) for x in self.p.stages[name].extents)
        if name in self.p.tables:
            return (self.iext(self.p.tables[name].extent),)
        raise OracleError(f"unknown {name}")

    def run(self, inputs: dict, keep_all: bool = False) -> dict:
        for name in list(self.p.images) + list(self.p.tables):
            if name not in inputs:
                raise OracleError(f"missing input {name!r}")
            arr = np.asarray(inputs[name])
            decl = self.p.images.get(name) or self.p.tables.get(name)
            if arr.shape != self.shape_of(name):
                raise OracleError(f"shape mismatch for {name}: got {arr.shape}, expected {self.shape_of(name)}")
            if arr.dtype != DTYPES[decl.dtype]:
                raise OracleError(f"dtype mismatch for {name}: got {arr.dtype}, expected {decl.dtype}")
            self.values[name] = arr
        for s in self.p.topo_order():
            self.values[s] = self.eval_stage(s)
        if keep_all:
            return {n: self.values[n] for n in self.p.stages}
        return {n: self.values[n] for n in self.p.liveouts}

    def eval_stage(self, name):
        s = self.p.stages[name]
        shape = self.shape_of(name)
        if min(shape) < 1:
            raise OracleError(f"stage {name} has an empty domain {shape}")
        env = {}
        for d, v in enumerate(s.vars):
            idx_shape = [1] * len(shape)
            idx_shape[d] = shape[d]
            env[v] = _V(np.arange(shape[d], dtype=np.int32).reshape(idx_shape), "i")
        val = self._ev(s.expr, env)
        out = self._store(val, s.dtype)
        return np.ascontiguousarray(np.broadcast_to(out, shape))

    # stage dtype conversion on store (R3/R4)
    def _store(self, v, dtype):
        if dtype == "f32":
            return np.asarray(v.a).astype(self.F) if v.k == "i" else np.asarray(v.a, dtype=self.F)
        iv = self._to_int(v)
        return iv.astype(DTYPES[dtype])            # wraps (two's complement)

    def _to_int(self, v):
        if v.k == "i":
            return np.asarray(v.a, dtype=np.int32)
        # truncate toward zero, saturate to the int32 range, NaN -> 0 (R4)
        t = np.trunc(np.asarray(v.a, dtype=np.float64))
        t = np.where(np.isnan(t), 0.0, np.clip(t, -2147483648.0, 2147483647.0))
        return t.astype(np.int64).astype(np.int32)

    def _to_float(self, v):
        if v.k == "f":
            return np.asarray(v.a, dtype=self.F)
        return np.asarray(v.a).astype(self.F)      # int -> float, round to nearest

    def _promote(self, a, b):
        if a.k == "f" or b.k == "f":
            return _V(self._to_float(a), "f"), _V(self._to_float(b), "f"), "f"
        return _V(np.asarray(a.a, dtype=np.int32), "i"), _V(np.asarray(b.a, dtype=np.int32), "i"), "i"

    def _read(self, name, arr):
        if arr.dtype == np.float32 or arr.dtype == np.float64:
            return _V(arr.astype(self.F, copy=False), "f")
        return _V(arr.astype(np.int32), "i")

    def _ev(self, e, env) -> _V:
        F = self.F
        if isinstance(e, Num):
            if e.is_float:
                return _V(np.asarray(np.float64(e.value)).astype(F), "f")  # f32(f64(text)) (R3)
            return _V(np.asarray(e.value, dtype=np.int32), "i")
        if isinstance(e, Name):
            if e.name in env:
                return env[e.name]
            if e.name in self.params:
                return _V(np.asarray(self.params[e.name], dtype=np.int32), "i")
            raise OracleError(f"undeclared name {e.name!r}")
        if isinstance(e, Access):
            src = self.values[e.target]
            idx = []
            for d, a in enumerate(e.args):
                iv = self._ev(a, env)
                if iv.k != "i":
                    raise OracleError(f"{e.pos}: index {d} of {e.target} is not an integer expression")
                idx.append(np.clip(np.asarray(iv.a, dtype=np.int64), 0, src.shape[d] - 1))  # clamp (R1)
            return self._read(e.target, src[tuple(idx)])
        if isinstance(e, TableRead):
            tab = self.values[e.table]
            iv = self._ev(e.index, env)
            if iv.k != "i":
                raise OracleError(f"table index for {e.table} is not an integer expression")
            return self._read(e.table, tab[np.clip(np.asarray(iv.a, dtype=np.int64), 0, tab.shape[0] - 1)])
        if isinstance(e, Un):
            a = self._ev(e.a, env)
            if e.op == "-":
                return _V(-a.a, a.k) if a.k == "f" else _V(np.negative(np.asarray(a.a, dtype=np.int32)), "i")
            return _V((np.asarray(a.a) == 0).astype(np.int32), "i")
        if isinstance(e, Bin):
            return self._bin(e.op, self._ev(e.a, env), self._ev(e.b, env))
        if isinstance(e, Call):
            return self._call(e, env)
        raise OracleError(f"bad node {e!r}")

    def _bin(self, op, a, b):
        if op in ("&&", "||"):
            x, y = np.asarray(a.a) != 0, np.asarray(b.a) != 0
            return _V((x & y if op == "&&" else x | y).astype(np.int32), "i")
        a, b, k = self._promote(a, b)
        x, y = a.a, b.a
        with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
            if op == "+":
                r = x + y
            elif op == "-":
                r = x - y
            elif op == "*":
                r = x * y
            elif op == "/":
                if k == "i":                          # floor division in int64, wrapped to int32; x/0 = 0 (R4)
                    x64, y64 = np.asarray(x, dtype=np.int64), np.asarray(y, dtype=np.int64)
                    r = np.where(y64 == 0, 0, np.floor_divide(x64, np.where(y64 == 0, 1, y64)))
                    r = r.astype(np.int32)
                else:
                    r = x / y
            elif op == "%":
                if k != "i":
                    raise OracleError("'%' needs integer operands")
                x64, y64 = np.asarray(x, dtype=np.int64), np.asarray(y, dtype=np.int64)
                r = np.where(y64 == 0, 0, np.mod(x64, np.where(y64 == 0, 1, y64))).astype(np.int32)  # x%0 = 0
            elif op in ("<<", ">>"):
                if k != "i":
                    raise OracleError(f"'{op}' needs integer operands")
                c = np.clip(np.asarray(y, dtype=np.int64), 0, 32)      # count clamped to [0, 32] (R4)
                x64 = np.asarray(x, dtype=np.int64)
                r = ((x64 << c) & 0xFFFFFFFF) if op == "<<" else (x64 >> c)
                r = r.astype(np.uint32).view(np.int32) if op == "<<" else r.astype(np.int32)
            elif op in ("<", "<=", ">", ">=", "==", "!="):
                r = {"<": np.less, "<=": np.less_equal, ">": np.greater, ">=": np.greater_equal,
                     "==": np.equal, "!=": np.not_equal}[op](x, y).astype(np.int32)
                return _V(r, "i")
            else:
                raise OracleError(f"unknown operator {op}")
        return _V(np.asarray(r, dtype=np.int32 if k == "i" else self.F), k)

    def _call(self, e, env):
        fn = e.fn
        args = [self._ev(a, env) for a in e.args]
        F = self.F
        if fn in ("min", "max"):
            a, b, k = self._promote(*args)
            r = np.where(b.a < a.a, b.a, a.a) if fn == "min" else np.where(b.a > a.a, b.a, a.a)
            return _V(r, k)
        if fn == "clamp":                         # clamp(x, lo, hi) = min(max(x, lo), hi)  (R5)
            return self._call_v("min", self._call_v("max", args[0], args[1]), args[2])
        if fn == "abs":
            a = args[0]
            return _V(np.abs(a.a), a.k) if a.k == "f" else _V(np.abs(np.asarray(a.a, dtype=np.int32)), "i")
        if fn == "absd":
            d = self._bin("-", args[0], args[1])
            return _V(np.abs(d.a), d.k)
        if fn == "select":
            c = np.asarray(args[0].a) != 0
            a, b, k = self._promote(args[1], args[2])
            return _V(np.where(c, a.a, b.a), k)
        if fn == "lerp":
            a, b, w = (self._to_float(v) for v in args)
            one = np.asarray(1.0, dtype=F)
            with np.errstate(over="ignore", invalid="ignore"):
                r = (a * (one - w)) + (b * w)
            return _V(np.asarray(r, dtype=F), "f")
        if fn == "sqrt":
            with np.errstate(invalid="ignore"):
                return _V(np.sqrt(self._to_float(args[0])), "f")
        if fn == "f32":
            return _V(self._to_float(args[0]), "f")
        if fn == "i32":
            return _V(self._to_int(args[0]), "i")
        if fn in ("i16", "u16", "u8"):
            return _V(self._to_int(args[0]).astype(DTYPES[fn]).astype(np.int32), "i")
        if fn in ("sat_u8", "sat_u16"):
            hi = 255 if fn == "sat_u8" else 65535
            return _V(np.clip(self._to_int(args[0]), 0, hi).astype(np.int32), "i")
        raise OracleError(f"unknown function {fn}")

    def _call_v(self, fn, a, b):
        a, b, k = self._promote(a, b)
        r = np.where(b.a < a.a, b.a, a.a) if fn == "min" else np.where(b.a > a.a, b.a, a.a)
        return _V(np.asarray(r), k)


def evaluate(text_or_prog, params: dict, inputs: dict, precision: str = "f32", keep_all: bool = False) -> dict:
    """Evaluate a pipeline stage by stage on the CPU; returns {liveout: ndarray} (or every stage)."""
    prog = parse(text_or_prog) if isinstance(text_or_prog, str) else text_or_prog
    return Evaluator(prog, params, precision).run(inputs, keep_all=keep_all)


def io_shapes(text_or_prog, params: dict) -> dict:
    """{name: (shape, dtype)} for every image, table and liveout."""
    prog = parse(text_or_prog) if isinstance(text_or_prog, str) else text_or_prog
    ev = Evaluator(prog, params)
    out = {}
    for n, d in list(prog.images.items()) + list(prog.tables.items()):
        out[n] = (ev.shape_of(n), d.dtype)
    for n in prog.liveouts:
        out[n] = (ev.shape_of(n), prog.stages[n].dtype)
    return out
