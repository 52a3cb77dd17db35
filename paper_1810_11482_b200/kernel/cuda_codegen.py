"""Lower a validated kernel to CUDA C for NVRTC (kernels with no
hand-written binding).

Semantics follow the reference's executor (/root/reference/pkg/src/
offloadrt/kernel/codegen.py): u32 arithmetic wraps mod 2^32, u32 `/` is
floor division, f64 arithmetic is one IEEE round-to-nearest operation per
source operator (``__dadd_rn`` etc., compiled with --fmad=false), operands
are evaluated left to right with every subexpression hoisted into a
temporary, && and || short-circuit, select() evaluates both arms, min/max
follow Python's builtin (first argument unless the second compares strictly
smaller/greater), u32(f64) truncates toward zero and aborts on NaN or
|x| >= 9.2e18.

Aborts (out-of-bounds index, division by zero, cast range) are reported per
work item into a 2-word record with atomicMin keyed on gtid, so the host
sees the error of the smallest failing gtid — the one the sequential
executor would have hit first.  Differences from the sequential executor:
items run in parallel, so a failing item does not stop the others, and
kernels whose items race on the same locations are not sequentially
consistent (reference test_kernel_fuzz.py:1-4 scopes this out).

Launch ABI of the generated kernel:
    ofl_k(<per param: buffer -> T* ptr, ofl_u64 len | scalar -> value>,
          ofl_u64 total, ofl_u32 nblocks, ofl_u32 bvol,
          unsigned long long* err)
err[0] = min((gtid << 32) | detail), err[1] = min((gtid << 8) | code).
"""

from __future__ import annotations

from .check import KernelIR
from .lang import Assign, Bin, BreakIf, Call, For, If, Let, Load, Name, Num, Store

CODE_OOB, CODE_DIV0, CODE_CAST = 1, 2, 3

_CTYPE = {"f64": "double", "u32": "ofl_u32", "bool": "bool"}
_BUILTIN = {
    "gtid": "gtid",
    "block_idx": "blk",
    "thread_idx": "thr",
    "grid_dim": "nblocks",
    "block_dim": "bvol",
}

PRELUDE = r"""
typedef unsigned int ofl_u32;
typedef unsigned long long ofl_u64;
typedef long long ofl_i64;
#define OFL_ABORT(code, detail) do { \
    atomicMin(&err[0], ((unsigned long long)gtid << 32) | (unsigned long long)(ofl_u32)(detail)); \
    atomicMin(&err[1], ((unsigned long long)gtid << 8) | (unsigned long long)(code)); \
    return; } while (0)
"""


def _lit(num: Num) -> str:
    if num.is_float:
        v = float(num.value)
        if v != v:
            return "(__longlong_as_double(0x7ff8000000000000LL))"
        if v in (float("inf"), float("-inf")):
            return "(1.0/0.0)" if v > 0 else "(-1.0/0.0)"
        return repr(v) if "e" in repr(v) or "." in repr(v) else repr(v) + ".0"
    return f"{int(num.value)}u"


class _Gen:
    def __init__(self, ir: KernelIR):
        self.ir = ir
        self.kinds = dict(ir.params)
        self.lines: list[str] = []
        self.ind = 1
        self.n = 0

    def emit(self, s: str) -> None:
        self.lines.append("    " * self.ind + s)

    def tmp(self, ty: str, expr: str) -> str:
        self.n += 1
        name = f"t{self.n}"
        self.emit(f"{_CTYPE[ty]} {name} = {expr};")
        return name

    # -- expressions --------------------------------------------------------
    def ex(self, e) -> str:
        if isinstance(e, Num):
            return _lit(e)
        if isinstance(e, Name):
            if e.ident in _BUILTIN:
                return _BUILTIN[e.ident]
            return f"p_{e.ident}" if e.ident in self.kinds else f"l_{e.ident}"
        if isinstance(e, Load):
            idx = self.index(e.buf, e.index)
            return self.tmp(e.ty, f"p_{e.buf}[{idx}]")
        if isinstance(e, Bin):
            return self.binop(e)
        if isinstance(e, Call):
            return self.call(e)
        raise AssertionError(type(e).__name__)

    def index(self, buf: str, idx_expr) -> str:
        idx = self.tmp("u32", self.ex(idx_expr))
        self.emit(f"if ((ofl_u64){idx} >= n_{buf}) OFL_ABORT({CODE_OOB}, {idx});")
        return idx

    def binop(self, e: Bin) -> str:
        op = e.op
        if op in ("&&", "||"):
            res = self.tmp("bool", self.ex(e.left))
            self.emit(f"if ({'' if op == '&&' else '!'}{res}) {{")
            self.ind += 1
            r = self.ex(e.right)
            self.emit(f"{res} = {r};")
            self.ind -= 1
            self.emit("}")
            return res
        lt = e.left.ty
        a = self.ex(e.left)
        b = self.ex(e.right)
        if op in ("<", "<=", ">", ">=", "==", "!="):
            return self.tmp("bool", f"({a} {op} {b})")
        if op == "/":
            zero = "0.0" if lt == "f64" else "0u"
            self.emit(f"if ({b} == {zero}) OFL_ABORT({CODE_DIV0}, 0);")
            return self.tmp(lt, f"__ddiv_rn({a}, {b})" if lt == "f64" else f"({a} / {b})")
        if lt == "f64":
            fn = {"+": "__dadd_rn", "-": "__dsub_rn", "*": "__dmul_rn"}[op]
            return self.tmp("f64", f"{fn}({a}, {b})")
        return self.tmp("u32", f"(ofl_u32)({a} {op} {b})")

    def call(self, e: Call) -> str:
        fn = e.fn
        args = [self.ex(a) for a in e.args]
        if fn in ("sin", "cos"):
            return self.tmp("f64", f"{fn}({args[0]})")
        if fn == "sqrt":
            return self.tmp("f64", f"__dsqrt_rn({args[0]})")
        if fn == "abs":
            return self.tmp(e.ty, f"fabs({args[0]})" if e.ty == "f64" else args[0])
        if fn == "min":
            return self.tmp(e.ty, f"(({args[1]} < {args[0]}) ? {args[1]} : {args[0]})")
        if fn == "max":
            return self.tmp(e.ty, f"(({args[1]} > {args[0]}) ? {args[1]} : {args[0]})")
        if fn == "select":
            return self.tmp(e.ty, f"({args[0]} ? {args[1]} : {args[2]})")
        if fn == "f64":
            return self.tmp("f64", f"(double)({args[0]})")
        if fn == "u32":
            if e.args[0].ty == "u32":
                return args[0]
            x = args[0]
            self.emit(f"if (!({x} == {x}) || {x} >= 9.2e18 || {x} <= -9.2e18) OFL_ABORT({CODE_CAST}, 0);")
            return self.tmp("u32", f"(ofl_u32)(unsigned long long)(long long)({x})")
        raise AssertionError(fn)

    # -- statements ---------------------------------------------------------
    def block(self, body) -> None:
        for s in body:
            self.st(s)

    def st(self, s) -> None:
        if isinstance(s, Let):
            v = self.ex(s.expr)
            self.emit(f"{_CTYPE[s.expr.ty]} l_{s.name} = {v};")
        elif isinstance(s, Assign):
            v = self.ex(s.expr)
            self.emit(f"l_{s.name} = {v};")
        elif isinstance(s, Store):
            idx = self.index(s.buf, s.index)
            v = self.ex(s.expr)
            self.emit(f"p_{s.buf}[{idx}] = {v};")
        elif isinstance(s, If):
            c = self.ex(s.cond)
            self.emit(f"if ({c}) {{")
            self.ind += 1
            self.block(s.then)
            self.ind -= 1
            if s.orelse:
                self.emit("} else {")
                self.ind += 1
                self.block(s.orelse)
                self.ind -= 1
            self.emit("}")
        elif isinstance(s, For):
            bound = self.tmp("u32", self.ex(s.bound))
            self.emit(f"for (ofl_u32 l_{s.var} = 0u; l_{s.var} < {bound}; ++l_{s.var}) {{")
            self.ind += 1
            self.block(s.body)
            self.ind -= 1
            self.emit("}")
        elif isinstance(s, BreakIf):
            c = self.ex(s.cond)
            self.emit(f"if ({c}) break;")
        else:
            raise AssertionError(type(s).__name__)

    def generate(self) -> str:
        params = []
        for name, kind in self.ir.params:
            if kind == "buffer_f64":
                params += [f"double* __restrict__ p_{name}", f"ofl_u64 n_{name}"]
            elif kind == "buffer_u32":
                params += [f"ofl_u32* __restrict__ p_{name}", f"ofl_u64 n_{name}"]
            elif kind == "scalar_f64":
                params.append(f"double p_{name}")
            else:
                params.append(f"ofl_u32 p_{name}")
        params += ["ofl_u64 total", "ofl_u32 nblocks", "ofl_u32 bvol", "unsigned long long* err"]
        head = [PRELUDE, 'extern "C" __global__ void ofl_k(' + ", ".join(params) + ") {",
                "  const ofl_u64 stride = (ofl_u64)gridDim.x * blockDim.x;",
                "  for (ofl_u64 item = (ofl_u64)blockIdx.x * blockDim.x + threadIdx.x; "
                "item < total; item += stride) {",
                "    const ofl_u32 gtid = (ofl_u32)item;",
                "    const ofl_u32 blk = (ofl_u32)(item / bvol);",
                "    const ofl_u32 thr = (ofl_u32)(item % bvol);",
                "    (void)blk; (void)thr; (void)nblocks;",
                "    {"]
        self.ind = 3
        self.block(self.ir.body)
        tail = ["    }", "  }", "}"]
        # aliasing between buffer params is legal in the language: drop the
        # __restrict__ promise when two params could point at one buffer
        text = "\n".join(head + self.lines + tail) + "\n"
        return text.replace(" __restrict__", "")


def generate(ir: KernelIR) -> str:
    """CUDA C source with one entry point `ofl_k` for the kernel."""
    return _Gen(ir).generate()
