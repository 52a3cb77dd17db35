"""Front-end for the kernel language of the reference runtime.

The language (grammar: /root/reference/pkg/src/offloadrt/kernel/lang.py:1-21,
SPEC.md) is kept unchanged so existing ``.k`` programs build here:

    program := kernel*
    kernel  := 'kernel' IDENT '(' [param (',' param)*] ')' block
    param   := IDENT ':' KIND          KIND in buffer_f64 buffer_u32 scalar_f64 scalar_u32
    block   := '{' stmt* '}'
    stmt    := 'let' IDENT '=' expr ';'
             | IDENT '=' expr ';'
             | IDENT '[' expr ']' '=' expr ';'
             | 'if' '(' expr ')' block ['else' block]
             | 'for' IDENT 'in' '0' '..' expr block
             | 'break' 'if' '(' expr ')' ';'
    expr    := or ;  or := and ('||' and)* ;  and := cmp ('&&' cmp)*
    cmp     := add [relop add]           (non-associative)
    add     := mul (('+'|'-') mul)* ;  mul := unary (('*'|'/') unary)*
    unary   := NUMBER | IDENT | IDENT '[' expr ']' | CALL '(' args ')' | '(' expr ')'

Comments run from '#' to end of line.  Every malformed input yields a
CompileError whose message starts with ``line:col:`` — the parser is total.

This is an independent implementation (a single regular-expression lexer,
slotted syntax nodes); only the language is shared.
"""

from __future__ import annotations

import re
from typing import Optional, Union

from ..errors import CompileError

KEYWORDS = frozenset({"kernel", "let", "if", "else", "for", "in", "break"})
KINDS = frozenset({"buffer_f64", "buffer_u32", "scalar_f64", "scalar_u32"})
BUILTINS = frozenset({"gtid", "block_idx", "thread_idx", "grid_dim", "block_dim"})
CALLS = frozenset({"sin", "cos", "sqrt", "abs", "min", "max", "select", "f64", "u32"})

U32_LIMIT = 1 << 32

# Longest alternatives first; ASCII classes only (no unicode digits).
_LEX = re.compile(
    r"""
    (?P<nl>\n)
  | (?P<ws>[ \t\r]+)
  | (?P<comment>\#[^\n]*)
  | (?P<num>[0-9]+(?:\.(?!\.)[0-9]*)?(?:[eE][+-]?[0-9]+)?)
  | (?P<ident>[A-Za-z_][A-Za-z0-9_]*)
  | (?P<punct>\.\.|&&|\|\||<=|>=|==|!=|[(){}\[\],;:=+\-*/<>])
    """,
    re.VERBOSE,
)


class Tok:
    __slots__ = ("kind", "text", "line", "col", "value")

    def __init__(self, kind: str, text: str, line: int, col: int, value=None):
        self.kind = kind  # 'ident' | 'int' | 'float' | 'eof' | keyword | punctuation
        self.text = text
        self.line = line
        self.col = col
        self.value = value

    def __repr__(self):
        return f"Tok({self.kind!r}, {self.text!r}, {self.line}:{self.col})"


def tokenize(source: str) -> list[Tok]:
    out: list[Tok] = []
    pos, line, line_start = 0, 1, 0
    n = len(source)
    while pos < n:
        m = _LEX.match(source, pos)
        col = pos - line_start + 1
        if m is None:
            raise CompileError(f"unexpected character {source[pos]!r}", line, col)
        kind = m.lastgroup
        text = m.group()
        if kind == "nl":
            line += 1
            line_start = m.end()
        elif kind == "num":
            if any(c in text for c in ".eE"):
                out.append(Tok("float", text, line, col, float(text)))
            else:
                v = int(text)
                if v >= U32_LIMIT:
                    raise CompileError(f"integer literal {text} exceeds u32", line, col)
                out.append(Tok("int", text, line, col, v))
        elif kind == "ident":
            out.append(Tok(text if text in KEYWORDS else "ident", text, line, col))
        elif kind == "punct":
            out.append(Tok(text, text, line, col))
        pos = m.end()
    out.append(Tok("eof", "", line, pos - line_start + 1))
    return out


# -- syntax tree ---------------------------------------------------------------
# Plain slotted nodes.  `ty` is filled in by the checker ('f64'|'u32'|'bool').


class Node:
    __slots__ = ("line", "col", "ty")

    def __init__(self, line: int, col: int):
        self.line = line
        self.col = col
        self.ty: Optional[str] = None


class Num(Node):
    __slots__ = ("value", "is_float")

    def __init__(self, value: Union[int, float], is_float: bool, line: int, col: int):
        super().__init__(line, col)
        self.value = value
        self.is_float = is_float


class Name(Node):
    __slots__ = ("ident",)

    def __init__(self, ident: str, line: int, col: int):
        super().__init__(line, col)
        self.ident = ident


class Load(Node):
    __slots__ = ("buf", "index")

    def __init__(self, buf: str, index: Node, line: int, col: int):
        super().__init__(line, col)
        self.buf = buf
        self.index = index


class Bin(Node):
    __slots__ = ("op", "left", "right")

    def __init__(self, op: str, left: Node, right: Node, line: int, col: int):
        super().__init__(line, col)
        self.op = op
        self.left = left
        self.right = right


class Call(Node):
    __slots__ = ("fn", "args")

    def __init__(self, fn: str, args: list, line: int, col: int):
        super().__init__(line, col)
        self.fn = fn
        self.args = args


class Let(Node):
    __slots__ = ("name", "expr")

    def __init__(self, name: str, expr: Node, line: int, col: int):
        super().__init__(line, col)
        self.name = name
        self.expr = expr


class Assign(Node):
    __slots__ = ("name", "expr")

    def __init__(self, name: str, expr: Node, line: int, col: int):
        super().__init__(line, col)
        self.name = name
        self.expr = expr


class Store(Node):
    __slots__ = ("buf", "index", "expr")

    def __init__(self, buf: str, index: Node, expr: Node, line: int, col: int):
        super().__init__(line, col)
        self.buf = buf
        self.index = index
        self.expr = expr


class If(Node):
    __slots__ = ("cond", "then", "orelse")

    def __init__(self, cond: Node, then: list, orelse: list, line: int, col: int):
        super().__init__(line, col)
        self.cond = cond
        self.then = then
        self.orelse = orelse


class For(Node):
    __slots__ = ("var", "bound", "body")

    def __init__(self, var: str, bound: Node, body: list, line: int, col: int):
        super().__init__(line, col)
        self.var = var
        self.bound = bound
        self.body = body


class BreakIf(Node):
    __slots__ = ("cond",)

    def __init__(self, cond: Node, line: int, col: int):
        super().__init__(line, col)
        self.cond = cond


class Kernel(Node):
    __slots__ = ("name", "params", "body")

    def __init__(self, name: str, params: list, body: list, line: int, col: int):
        super().__init__(line, col)
        self.name = name
        self.params = params  # [(name, kind)]
        self.body = body


# -- parser ----------------------------------------------------------------------

_RELOPS = frozenset({"<", "<=", ">", ">=", "==", "!="})


def _shown(tok: Tok) -> str:
    return "end of input" if tok.kind == "eof" else tok.text


class Parser:
    def __init__(self, tokens: list[Tok]):
        self.toks = tokens
        self.i = 0

    @property
    def tok(self) -> Tok:
        return self.toks[self.i]

    def take(self) -> Tok:
        t = self.toks[self.i]
        if t.kind != "eof":
            self.i += 1
        return t

    def want(self, kind: str) -> Tok:
        t = self.tok
        if t.kind != kind:
            raise CompileError(f"expected {kind!r}, found {_shown(t)!r}", t.line, t.col)
        return self.take()

    # program / kernel ----------------------------------------------------------
    def program(self) -> list[Kernel]:
        kernels = []
        while self.tok.kind != "eof":
            kernels.append(self.kernel())
        return kernels

    def kernel(self) -> Kernel:
        kw = self.want("kernel")
        name = self.want("ident")
        self.want("(")
        params = []
        if self.tok.kind != ")":
            while True:
                pname = self.want("ident")
                self.want(":")
                kind = self.want("ident")
                if kind.text not in KINDS:
                    raise CompileError(f"unknown parameter kind {kind.text!r}", kind.line, kind.col)
                params.append((pname.text, kind.text))
                if self.tok.kind != ",":
                    break
                self.take()
        self.want(")")
        return Kernel(name.text, params, self.block(), kw.line, kw.col)

    def block(self) -> list[Node]:
        self.want("{")
        body = []
        while self.tok.kind != "}":
            if self.tok.kind == "eof":
                raise CompileError("unterminated block", self.tok.line, self.tok.col)
            body.append(self.stmt())
        self.take()
        return body

    # statements --------------------------------------------------------------------
    def stmt(self) -> Node:
        t = self.tok
        k = t.kind
        if k == "let":
            self.take()
            name = self.want("ident")
            self.want("=")
            e = self.expr()
            self.want(";")
            return Let(name.text, e, t.line, t.col)
        if k == "if":
            self.take()
            self.want("(")
            cond = self.expr()
            self.want(")")
            then = self.block()
            orelse = []
            if self.tok.kind == "else":
                self.take()
                orelse = self.block()
            return If(cond, then, orelse, t.line, t.col)
        if k == "for":
            self.take()
            var = self.want("ident")
            self.want("in")
            z = self.tok
            if z.kind != "int" or z.value != 0:
                raise CompileError("loop ranges start at 0", z.line, z.col)
            self.take()
            self.want("..")
            bound = self.expr()
            return For(var.text, bound, self.block(), t.line, t.col)
        if k == "break":
            self.take()
            self.want("if")
            self.want("(")
            cond = self.expr()
            self.want(")")
            self.want(";")
            return BreakIf(cond, t.line, t.col)
        if k == "ident":
            self.take()
            if self.tok.kind == "[":
                self.take()
                idx = self.expr()
                self.want("]")
                self.want("=")
                e = self.expr()
                self.want(";")
                return Store(t.text, idx, e, t.line, t.col)
            self.want("=")
            e = self.expr()
            self.want(";")
            return Assign(t.text, e, t.line, t.col)
        raise CompileError(f"expected a statement, found {t.text!r}", t.line, t.col)

    # expressions: one function per precedence level (grammar above) ------------
    def expr(self) -> Node:
        return self._chain(self._and, ("||",))

    def _and(self) -> Node:
        return self._chain(self._cmp, ("&&",))

    def _cmp(self) -> Node:
        left = self._add()
        op = self.tok
        if op.kind in _RELOPS:  # at most one comparison: non-associative
            self.take()
            left = Bin(op.kind, left, self._add(), op.line, op.col)
        return left

    def _add(self) -> Node:
        return self._chain(self._mul, ("+", "-"))

    def _mul(self) -> Node:
        return self._chain(self.unary, ("*", "/"))

    def _chain(self, sub, ops) -> Node:
        left = sub()
        while self.tok.kind in ops:
            op = self.take()
            left = Bin(op.kind, left, sub(), op.line, op.col)
        return left

    def unary(self) -> Node:
        t = self.tok
        if t.kind == "int":
            self.take()
            return Num(t.value, False, t.line, t.col)
        if t.kind == "float":
            self.take()
            return Num(t.value, True, t.line, t.col)
        if t.kind == "(":
            self.take()
            inner = self.expr()
            self.want(")")
            return inner
        if t.kind == "ident":
            self.take()
            nxt = self.tok.kind
            if nxt == "(":
                if t.text not in CALLS:
                    raise CompileError(f"unknown function {t.text!r}", t.line, t.col)
                self.take()
                args = []
                if self.tok.kind != ")":
                    while True:
                        args.append(self.expr())
                        if self.tok.kind != ",":
                            break
                        self.take()
                self.want(")")
                return Call(t.text, args, t.line, t.col)
            if nxt == "[":
                self.take()
                idx = self.expr()
                self.want("]")
                return Load(t.text, idx, t.line, t.col)
            return Name(t.text, t.line, t.col)
        raise CompileError(f"expected an expression, found {_shown(t)!r}", t.line, t.col)


def parse_source(source: str) -> list[Kernel]:
    """Source text -> kernel syntax trees.  Raises CompileError."""
    if not isinstance(source, str):
        raise CompileError("source is not text", 0, 0)
    kernels = Parser(tokenize(source)).program()
    names: set[str] = set()
    for k in kernels:
        if k.name in names:
            raise CompileError(f"duplicate kernel {k.name!r}", k.line, k.col)
        names.add(k.name)
    return kernels
