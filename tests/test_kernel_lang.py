"""Kernel-language front-end (CPU): diagnostics, typing rules, parser
totality, and the canonical-form binding of the workloads' kernels.
Mirrors the reference's test_kernel_lang.py parsing section."""

from __future__ import annotations

import os
import random

import pytest

from paper_1810_11482_b200.bindings import kernel_source, lookup
from paper_1810_11482_b200.errors import CompileError
from paper_1810_11482_b200.kernel import parse_and_validate, parse_source, tokenize
from paper_1810_11482_b200.kernel.canon import canonical

REF_KERNELS = "/root/reference/pkg/src/offloadrt/bench/kernels"


def build(source, name):
    return parse_and_validate(source)[name]


def test_bundled_kernels_parse_and_bind():
    for src, names in (("stencil", ["stencil"]), ("mandelbrot", ["mandelbrot"]),
                       ("sum", ["sum"]), ("partition", ["partition"]),
                       ("stream", ["copy", "scale", "add", "triad"])):
        kernels = parse_and_validate(kernel_source(src))
        for name in names:
            assert lookup(kernels[name]).name == name


@pytest.mark.skipif(not os.path.isdir(REF_KERNELS), reason="reference tree not mounted")
@pytest.mark.parametrize("name", ["stencil", "mandelbrot", "sum", "partition"])
def test_reference_kernel_sources_bind(name):
    """The reference's own .k files bind to the same native kernels."""
    with open(os.path.join(REF_KERNELS, f"{name}.k")) as fh:
        ir = build(fh.read(), name)
    assert lookup(ir).name == name
    assert canonical(ir) == canonical(build(kernel_source(name), name))


def test_canonical_form_ignores_names_and_layout():
    a = "kernel k(x : buffer_f64, n : scalar_u32) { if (gtid < n) { x[gtid] = 1.0; } }"
    b = "# comment\nkernel other(buf:buffer_f64,count:scalar_u32){if(gtid<count){buf[gtid]=1.0;}}"
    assert canonical(build(a, "k")) == canonical(build(b, "other"))
    c = "kernel k(x : buffer_f64, n : scalar_u32) { if (gtid < n) { x[gtid] = 2.0; } }"
    assert canonical(build(a, "k")) != canonical(build(c, "k"))


def test_operand_order_matters_for_binding():
    src = kernel_source("stencil").replace("0.5 * u[gtid - 1] + u[gtid]", "u[gtid] + 0.5 * u[gtid - 1]")
    assert lookup(build(src, "stencil")) is None


def test_parse_error_carries_line_and_col():
    with pytest.raises(CompileError) as err:
        parse_source("kernel broken(x : buffer_f64) {\n    x[0] = ;\n}\n")
    assert str(err.value).startswith("2:")
    assert err.value.line == 2


def test_diagnostics():
    cases = [
        ("kernel k(x : buffer_f64) { x[0] = wat; }", "wat"),
        ("kernel k(x : buffer_f64, n : scalar_u32) { x[0] = n; }", "f64"),
        ("kernel k(x : buffer_u32) { for i in 0 .. x[0] { } }", "loop bound"),
        ("kernel k() { break if (gtid == 0); }", "break"),
        ("kernel k(n : scalar_u32) { n = 3; }", "assignable"),
        ("kernel k() { let a = 1; let a = 2; }", "already defined"),
        ("kernel k(s : scalar_f64) { let a = s + 1; }", "cast"),
        ("kernel k() { if (1) { } }", "boolean"),
        ("kernel k() { let a = nope(1); }", "unknown function"),
        ("kernel k(x : buffer_f64) { let v = x; }", "cannot be used as a value"),
        ("kernel k() { let g = gtid; let b = 1 < 2; }", "numeric"),
        ("kernel k() { for i in 1 .. 3 { } }", "start at 0"),
        ("kernel k() { let t = 1 < 2 < 3; }", "expected"),
    ]
    for src, needle in cases:
        with pytest.raises(CompileError, match=needle):
            parse_and_validate(src)
    with pytest.raises(CompileError, match="kind"):
        parse_source("kernel k(x : buffer_f32) { }")
    with pytest.raises(CompileError, match="duplicate"):
        parse_source("kernel k() { }\nkernel k() { }")
    with pytest.raises(CompileError, match="exceeds u32"):
        parse_source("kernel k() { let a = 4294967296; }")


def test_accepted_programs():
    parse_and_validate("kernel k(n : scalar_u32) { for i in 0 .. n { } }")
    parse_and_validate("kernel k() { for i in 0 .. 17 { } }")
    parse_and_validate("kernel k(s : scalar_f64) { let a = s + f64(1); }")
    parse_and_validate(
        "kernel s(out : buffer_f64, flag : scalar_u32) { if (gtid == 0) {"
        " if (flag == 1) { let t = 2.5; out[0] = t; } else { let t = 7; out[0] = f64(t); } } }"
    )


def test_lexer_numbers():
    kinds = [(t.kind, t.text) for t in tokenize("1..2 1.5 1. 2e3 1e 3.e-2 0")]
    assert kinds[:4] == [("int", "1"), ("..", ".."), ("int", "2"), ("float", "1.5")]
    assert ("float", "1.") in kinds and ("float", "2e3") in kinds and ("float", "3.e-2") in kinds
    assert ("int", "1") in kinds and ("ident", "e") in kinds
    with pytest.raises(CompileError, match="unexpected character"):
        tokenize("let € = 1;")


def test_parser_totality_fuzz():
    rng = random.Random(424242)
    frags = ["kernel", "k", "(", ")", "{", "}", "let", "=", ";", "if", "for", "in", "0", "..",
             "1.5", "buffer_f64", ":", "x", "[", "]", "+", "&&", "sin", "break", "selec", "\x00",
             "€"]
    for _ in range(20_000):
        text = "".join(rng.choice(frags) + rng.choice([" ", ""]) for _ in range(rng.randint(0, 24)))
        try:
            parse_and_validate(text)
        except CompileError:
            pass
    for _ in range(20_000):
        text = "".join(chr(rng.randrange(32, 1000)) for _ in range(rng.randint(0, 60)))
        try:
            parse_and_validate(text)
        except CompileError:
            pass


def test_fuzz_fixtures_parse_and_go_generic(golden):
    """The reference-generated random kernels (tests/golden fuzz) validate
    in this implementation's front end and none is mistaken for a bundled
    workload kernel (they must take the NVRTC path)."""
    from paper_1810_11482_b200 import bindings
    from paper_1810_11482_b200.kernel import parse_and_validate

    assert len(golden["fuzz"]) == 150
    for case in golden["fuzz"]:
        ir = parse_and_validate(case["source"])["fuzzed"]
        assert bindings.lookup(ir) is None
