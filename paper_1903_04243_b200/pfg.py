"""`.pfg` text format for graphs -- the reference's interchange format
(`pforvec/serialize.py`), re-implemented for this IR so
graphs dumped by the reference (e.g. its golden vectorized graphs,
`tests/golden/*.pfg`) load here, run on the B200 executor, and dump back to
byte-identical text.

Grammar (one statement per line, blocks nest with braces):

    stmt    := "var" NAME "=" tensor
             | "%" ID "=" KIND [ "[" attr ("," attr)* "]" ] "(" refs ")"
               [ "ctrl" "[" refs "]" ] [ "{" (SUBNAME "{" graph "}")* "}" ]
             | "outputs" "(" refs ")"          -- ends a graph
    ref     := "%" ID [ ":" PORT ]
    attr    := KEY "=" value
    value   := tensor | dtype | "true" | "false" | "none" | shape | int | float | string
    tensor  := dtype "[" dims "]" "{" items "}"        (f64 / i64 / bool)
    shape   := "[" (INT | "?")* "]"

Node ids are local to each (sub)graph and renumbered densely on load (the
reference does the same: its ids are assigned in file order); attributes are
written in sorted key order; floats use Python's shortest round-trip repr.
"""

from __future__ import annotations

import re

import numpy as np

from .errors import ParseError
from .graph import Block, Graph, Ref
from .tensor import DType, TensorValue

SUBGRAPHS = {"parfor": ("body",), "cond": ("then", "else"), "while": ("cond", "body")}


# ----------------------------------------------------------------------------
# writer

def _float_text(x) -> str:
    x = float(x)
    if x != x:
        return "nan"
    if x in (float("inf"), float("-inf")):
        return "inf" if x > 0 else "-inf"
    return repr(x)


def _tensor_text(v: TensorValue) -> str:
    flat = np.asarray(v.data).reshape(-1)
    if v.dtype == DType.F64:
        body = ",".join(_float_text(x) for x in flat)
    elif v.dtype == DType.I64:
        body = ",".join(str(int(x)) for x in flat)
    else:
        body = ",".join("true" if bool(x) else "false" for x in flat)
    dims = ",".join(str(int(d)) for d in np.shape(v.data))
    return f"{v.dtype.value}[{dims}]{{{body}}}"


def _value_text(v) -> str:
    if isinstance(v, TensorValue):
        return _tensor_text(v)
    if isinstance(v, DType):
        return v.value
    if isinstance(v, (bool, np.bool_)):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return _float_text(v)
    if isinstance(v, str):
        return '"' + v.replace("\\", "\\\\").replace('"', '\\"') + '"'
    if v is None:
        return "none"
    if isinstance(v, (tuple, list)):
        return "[" + ",".join("?" if d is None else str(int(d)) for d in v) + "]"
    raise TypeError(f"pfg: attribute value {v!r} has no text form")


def _ref_text(ref) -> str:
    nid, port = ref
    return f"%{nid}" + (f":{port}" if port else "")


def _emit(g: Graph, depth: int, out: list):
    ind = "  " * depth
    out.extend(f"{ind}var {name} = {_tensor_text(g.variables[name])}" for name in sorted(g.variables))
    for nid in sorted(g.nodes):
        node = g.nodes[nid]
        line = f"{ind}%{nid} = {node.kind}"
        if node.attrs:
            line += "[" + ", ".join(f"{k}={_value_text(node.attrs[k])}"
                                    for k in sorted(node.attrs)) + "]"
        line += "(" + ", ".join(_ref_text(tuple(r)) for r in node.inputs) + ")"
        if node.control_deps:
            line += " ctrl[" + ", ".join(f"%{c}" for c in sorted(node.control_deps)) + "]"
        if node.block is None:
            out.append(line)
            continue
        out.append(line + " {")
        for sub in SUBGRAPHS[node.block.kind]:
            out.append(f"{ind}  {sub} {{")
            _emit(node.block.subgraphs[sub], depth + 2, out)
            out.append(f"{ind}  }}")
        out.append(f"{ind}}}")
    if g.outputs:
        out.append(f"{ind}outputs(" + ", ".join(_ref_text(tuple(r)) for r in g.outputs) + ")")


def dumps(g: Graph) -> str:
    out: list = []
    _emit(g, 0, out)
    return "\n".join(out) + "\n"


def dump(g: Graph, path) -> None:
    with open(path, "w") as fh:
        fh.write(dumps(g))


# ----------------------------------------------------------------------------
# reader

_LEX = re.compile(r"""
    (?P<skip>[ \t\r]+|\#[^\n]*)
  | (?P<newline>\n)
  | (?P<str>"(?:\\.|[^"\\])*")
  | (?P<num>-?(?:\d+\.\d*(?:[eE][+-]?\d+)?|\d+[eE][+-]?\d+|\.\d+(?:[eE][+-]?\d+)?|\d+))
  | (?P<word>-?[A-Za-z_]\w*)
  | (?P<punct>[%=\[\](){},:?])
""", re.VERBOSE)


class _Lexer:
    """Token stream with line/column positions (whitespace, comments and
    line breaks are insignificant)."""

    def __init__(self, text: str):
        self.toks = []
        line, start = 1, 0
        pos = 0
        while pos < len(text):
            m = _LEX.match(text, pos)
            if m is None:
                raise ParseError(f"unexpected character {text[pos]!r}", line, pos - start + 1)
            if m.lastgroup == "newline":
                line, start = line + 1, m.end()
            elif m.lastgroup != "skip":
                self.toks.append((m.lastgroup, m.group(), line, pos - start + 1))
            pos = m.end()
        self.toks.append(("eof", "", line, pos - start + 1))
        self.i = 0

    @property
    def cur(self):
        return self.toks[self.i]

    def look(self, k=0) -> str:
        return self.toks[min(self.i + k, len(self.toks) - 1)][1]

    def take(self):
        t = self.toks[self.i]
        self.i += 1
        return t

    def err(self, msg, tok=None):
        _, text, line, col = tok or self.cur
        raise ParseError(f"{msg} (got {text!r})", line, col)

    def need(self, text: str):
        t = self.take()
        if t[1] != text:
            self.err(f"expected {text!r}", t)
        return t

    def sep_list(self, close: str, item):
        """item (',' item)* up to `close` (consumed)."""
        vals = []
        while self.look() != close:
            vals.append(item())
            if self.look() != close:
                self.need(",")
        self.need(close)
        return vals


def _int(lx: _Lexer) -> int:
    t = lx.take()
    try:
        return int(t[1])
    except ValueError:
        lx.err("expected an integer", t)


def _float(lx: _Lexer) -> float:
    t = lx.take()
    try:
        return float(t[1])  # also 'inf', '-inf', 'nan'
    except ValueError:
        lx.err("expected a number", t)


def _tensor(lx: _Lexer) -> TensorValue:
    t = lx.take()
    try:
        dt = DType(t[1])
    except ValueError:
        lx.err("expected a dtype", t)
    lx.need("[")
    dims = lx.sep_list("]", lambda: _int(lx))
    lx.need("{")
    if dt == DType.F64:
        items = lx.sep_list("}", lambda: _float(lx))
    elif dt == DType.I64:
        items = lx.sep_list("}", lambda: _int(lx))
    else:
        def _bool():
            b = lx.take()
            if b[1] not in ("true", "false"):
                lx.err("expected true/false", b)
            return b[1] == "true"
        items = lx.sep_list("}", _bool)
    return TensorValue(dt, np.array(items, dtype=dt.np_dtype).reshape(tuple(dims)))


def _shape(lx: _Lexer):
    lx.need("[")

    def dim():
        if lx.look() == "?":
            lx.take()
            return None
        return _int(lx)
    return tuple(lx.sep_list("]", dim))


def _value(lx: _Lexer):
    kind, text = lx.cur[0], lx.cur[1]
    if kind == "str":
        lx.take()
        return re.sub(r"\\(.)", r"\1", text[1:-1])
    if text in ("f64", "i64", "bool"):
        if lx.look(1) == "[":
            return _tensor(lx)
        lx.take()
        return DType(text)
    if text in ("true", "false"):
        lx.take()
        return text == "true"
    if text == "none":
        lx.take()
        return None
    if text == "[":
        return _shape(lx)
    if kind == "num":
        return _float(lx) if any(c in text for c in ".eE") else _int(lx)
    lx.err("expected an attribute value")


def _ref(lx: _Lexer, ids: dict) -> tuple:
    lx.need("%")
    t = lx.take()
    try:
        local = int(t[1])
    except ValueError:
        lx.err("expected a node id", t)
    port = 0
    if lx.look() == ":":
        lx.take()
        port = _int(lx)
    if local not in ids:
        lx.err(f"reference to undefined node %{local}", t)
    return ids[local], port


def _graph(lx: _Lexer, g: Graph) -> None:
    ids: dict = {}  # file-local id -> id in g
    while True:
        head = lx.look()
        if head == "var":
            lx.take()
            name = lx.take()[1]
            lx.need("=")
            g.declare_variable(name, _tensor(lx))
        elif head == "%":
            lx.take()
            idt = lx.take()
            try:
                local = int(idt[1])
            except ValueError:
                lx.err("expected a node id", idt)
            lx.need("=")
            kind = lx.take()[1]
            attrs = {}
            if lx.look() == "[":
                lx.take()

                def attr():
                    key = lx.take()[1]
                    lx.need("=")
                    attrs[key] = _value(lx)
                lx.sep_list("]", attr)
            lx.need("(")
            ins = lx.sep_list(")", lambda: _ref(lx, ids))
            ctrl = []
            if lx.look() == "ctrl":
                lx.take()
                lx.need("[")
                ctrl = [r[0] for r in lx.sep_list("]", lambda: _ref(lx, ids))]
            block = None
            if lx.look() == "{":
                lx.take()
                subs = {}
                while lx.look() != "}":
                    sname = lx.take()[1]
                    lx.need("{")
                    sub = Graph()
                    sub.outer_variables = {**g.outer_variables, **g.variables}
                    _graph(lx, sub)
                    lx.need("}")
                    subs[sname] = sub
                lx.need("}")
                if kind not in SUBGRAPHS:
                    lx.err(f"kind {kind!r} takes no block", idt)
                if kind == "while":
                    block = Block(kind, subs, num_carried=len(subs["body"].outputs))
                else:
                    first = subs[SUBGRAPHS[kind][0]]
                    block = Block(kind, subs, out_arity=len(first.outputs))
            node = g.add_node(kind, [Ref(g, n, p) for n, p in ins], attrs, control_deps=ctrl,
                              block=block)
            ids[local] = node.id
        elif head == "outputs":
            lx.take()
            lx.need("(")
            g.set_outputs([Ref(g, n, p) for n, p in lx.sep_list(")", lambda: _ref(lx, ids))])
            return
        else:
            return


def loads(text: str) -> Graph:
    lx = _Lexer(text)
    g = Graph()
    _graph(lx, g)
    if lx.cur[0] != "eof":
        lx.err("trailing input")
    return g


def load(path) -> Graph:
    with open(path) as fh:
        return loads(fh.read())
