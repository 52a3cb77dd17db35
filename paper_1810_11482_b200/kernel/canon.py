"""Canonical form of a validated kernel.

Two kernels with the same canonical form compute the same thing: parameter
names become positions, locals become declaration numbers, comments and
layout vanish, and everything that affects IEEE results (operand order,
literal values and types, casts, control flow) is kept.  ``build()`` uses it
to recognise the workloads' kernels — whatever the user named them — and
bind them to the hand-written sm_100a implementations (see bindings.py).
"""

from __future__ import annotations

from .check import KernelIR
from .lang import (
    BUILTINS,
    Assign,
    Bin,
    BreakIf,
    Call,
    For,
    If,
    Let,
    Load,
    Name,
    Num,
    Store,
)


def canonical(ir: KernelIR) -> tuple:
    params = {name: i for i, (name, _) in enumerate(ir.params)}
    scopes: list[dict[str, int]] = [{}]
    counter = [0]

    def declare(name: str) -> int:
        counter[0] += 1
        scopes[-1][name] = counter[0]
        return counter[0]

    def ref(name: str) -> tuple:
        if name in BUILTINS:
            return ("b", name)
        for scope in reversed(scopes):
            if name in scope:
                return ("l", scope[name])
        return ("p", params[name])

    def ex(e) -> tuple:
        if isinstance(e, Num):
            return ("n", bool(e.is_float), float(e.value) if e.is_float else int(e.value))
        if isinstance(e, Name):
            return ref(e.ident)
        if isinstance(e, Load):
            return ("ld", params[e.buf], ex(e.index))
        if isinstance(e, Bin):
            return ("bin", e.op, ex(e.left), ex(e.right))
        if isinstance(e, Call):
            return ("call", e.fn) + tuple(ex(a) for a in e.args)
        raise AssertionError(type(e).__name__)

    def block(body) -> tuple:
        scopes.append({})
        out = tuple(st(s) for s in body)
        scopes.pop()
        return out

    def st(s) -> tuple:
        if isinstance(s, Let):
            value = ex(s.expr)
            return ("let", declare(s.name), value)
        if isinstance(s, Assign):
            return ("set", ref(s.name), ex(s.expr))
        if isinstance(s, Store):
            return ("st", params[s.buf], ex(s.index), ex(s.expr))
        if isinstance(s, If):
            return ("if", ex(s.cond), block(s.then), block(s.orelse))
        if isinstance(s, For):
            bound = ex(s.bound)
            scopes.append({})
            var = declare(s.var)
            body = tuple(st(x) for x in s.body)
            scopes.pop()
            return ("for", var, bound, body)
        if isinstance(s, BreakIf):
            return ("brk", ex(s.cond))
        raise AssertionError(type(s).__name__)

    kinds = tuple(kind for _, kind in ir.params)
    return (kinds, tuple(st(s) for s in ir.body))
