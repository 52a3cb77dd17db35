"""Differential API fuzzing against the reference itself.

One random plan of operations — buffer creation (valid, zero and negative
sizes), writes and reads at valid and out-of-range offsets, kernel runs of
the bundled programs with well-formed and malformed arguments (wrong arity,
wrong kinds, u32 out of range, counts past the buffers, bad launch shapes),
cross-buffer copies, when_all gates, synchronize, stream creation, unregister
— is executed twice: on the reference's own runtime (``offloadrt``, host
backend, from /root/reference or the offline install in baseline/_ref) and on
this package's runtime on the B200.  Every operation's outcome must agree: the
same exception class (raised at the call or carried by the token) or the same
value, bytes compared exactly (two NaNs count as equal: IEEE leaves the
payload of a propagated NaN open, and x86 and the GPU pick differently).

A run that fails leaves the reference's partial writes (its executor runs
work items one by one until the faulting one) while the CUDA path writes
nothing; such runs' output buffers are excluded from later comparisons
(known differences).  Stencils never alias input and output
(rejected here, sequentially defined there).
"""

from __future__ import annotations

import os
import random
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC_CANDIDATES = ("/root/reference/pkg/src", os.path.join(REPO, "baseline", "_ref"))

SEEDS = range(100)
OPS_PER_PLAN = 80

# kernel -> (program, parameter kinds); element sizes by kind
KERNELS = {
    "copy": ("stream", ["b64", "b64", "u32"]),
    "scale": ("stream", ["b64", "b64", "f64", "u32"]),
    "add": ("stream", ["b64", "b64", "b64", "u32"]),
    "triad": ("stream", ["b64", "b64", "b64", "f64", "u32"]),
    "stencil": ("stencil", ["b64", "b64", "u32"]),
    "stencil2d": ("stencil2d", ["b64", "b64", "u32", "u32"]),
    "sum": ("sum", ["b32", "b32", "u32"]),
    "mandelbrot": ("mandelbrot", ["b32", "u32", "u32", "f64", "f64", "f64", "f64", "f64", "u32"]),
}
OUTPUT_ARG = {"copy": 0, "scale": 0, "add": 0, "triad": 0, "stencil": 1, "stencil2d": 1,
              "sum": 1, "mandelbrot": 0}


def _ref_src():
    for p in REF_SRC_CANDIDATES:
        if os.path.isfile(os.path.join(p, "offloadrt", "__init__.py")):
            return p
    return None


@pytest.fixture(scope="module")
def worlds():
    src = _ref_src()
    if src is None:
        pytest.skip("reference package not importable here (no /root/reference, no baseline/_ref)")
    sys.path.insert(0, src)
    try:
        import offloadrt
        from offloadrt.bench import kernel_source as ref_kernel_source
    except ImportError as exc:  # numba missing, say
        pytest.skip(f"reference not importable: {exc}")
    finally:
        sys.path.remove(src)
    import paper_1810_11482_b200 as ours
    from paper_1810_11482_b200.bindings import kernel_source as our_kernel_source

    sources = {
        "stream": our_kernel_source("stream"),
        "stencil2d": our_kernel_source("stencil2d"),
        "stencil": ref_kernel_source("stencil"),
        "sum": ref_kernel_source("sum"),
        "mandelbrot": ref_kernel_source("mandelbrot"),
    }
    ref_rt = offloadrt.Runtime(backend="host", devices=1)
    our_rt = ours.Runtime(devices=[0])
    yield {
        "ref": (offloadrt, ref_rt, ref_rt.get_all_devices().get()[0]),
        "ours": (ours, our_rt, our_rt.get_all_devices().get()[0]),
        "sources": sources,
    }
    ref_rt.close()
    our_rt.close()


class World:
    """One runtime executing a plan; records an outcome per operation."""

    def __init__(self, pkg, rt, dev, sources):
        self.pkg, self.rt, self.dev, self.sources = pkg, rt, dev, sources
        self.bufs: list = []       # handle or None (unregistered)
        self.progs: dict = {}      # program name -> (handle, built kernels)

    def outcome(self, fn):
        try:
            v = fn()
        except Exception as exc:  # noqa: BLE001 - compared by class
            return ("raise", type(exc).__name__)
        if isinstance(v, self.pkg.CompletionToken):
            try:
                v = v.get(timeout=120)
            except Exception as exc:  # noqa: BLE001
                return ("fail", type(exc).__name__)
        return ("ok", v)

    def program(self, name):
        if name not in self.progs:
            h = self.dev.create_program_with_source(self.sources[name]).get(timeout=120)
            self.progs[name] = (h, set())
        return self.progs[name]


def _f64_bytes(rng, count):
    return np.array([rng.uniform(-1.0, 2.0) for _ in range(count)], np.float64).tobytes()


def _u32_bytes(rng, count):
    return np.array([rng.randrange(0, 2**32) for _ in range(count)], np.uint32).tobytes()


def _plan(seed: int):
    """The operation list (pure data: buffer indices, sizes, payloads)."""
    rng = random.Random(seed)
    ops = []
    sizes = []  # planned size per created buffer slot (creation outcomes must agree)
    for _ in range(OPS_PER_PLAN):
        r = rng.random()
        if r < 0.14 or len(sizes) < 3:
            size = rng.choice([8 * rng.randint(1, 512), 4 * rng.randint(1, 1024),
                               rng.randint(1, 4096), 0, -8])
            ops.append(("create", size))
            if size > 0:
                sizes.append(size)
            continue
        b = rng.randrange(len(sizes))
        size = sizes[b]
        if r < 0.19:  # the whole buffer: f64 values or u32 words
            if rng.random() < 0.5 and size % 8 == 0:
                ops.append(("write", b, 0, _f64_bytes(rng, size // 8)))
            else:
                ops.append(("write", b, 0, bytes(rng.randrange(256) for _ in range(size))
                            if size % 4 else _u32_bytes(rng, size // 4)))
            continue
        if r < 0.34:
            kind = rng.random()
            if kind < 0.45:
                off = 8 * rng.randint(0, size // 8)
                data = _f64_bytes(rng, rng.randint(0, max(0, (size - off) // 8)))
            elif kind < 0.8:
                off = 4 * rng.randint(0, size // 4)
                data = _u32_bytes(rng, rng.randint(0, max(0, (size - off) // 4)))
            else:
                off = rng.choice([rng.randint(0, size), size + rng.randint(1, 9), -1])
                data = bytes(rng.randrange(256) for _ in range(rng.randint(0, 12)))
            ops.append(("write", b, off, data))
        elif r < 0.48:
            off = rng.choice([0, rng.randint(0, size), size + 1, -4])
            n = rng.choice([size - max(0, off), rng.randint(0, max(0, size - max(0, off))),
                            size + 3, -1])
            ops.append(("read", b, off, n))
        elif r < 0.80:
            name = rng.choice(list(KERNELS))
            _, kinds = KERNELS[name]
            args = []
            for k in kinds:
                x = rng.random()
                if k in ("b64", "b32"):
                    args.append(("buf", rng.randrange(len(sizes))) if x > 0.03 else ("u32", 7))
                elif k == "f64":
                    args.append(("f64", rng.uniform(-3, 3)) if x > 0.1 else ("u32", rng.randint(0, 5)))
                else:  # u32: counts / dimensions, mostly within the buffers
                    bufs = [sizes[a[1]] // (8 if kk == "b64" else 4)
                            for a, kk in zip(args, kinds) if a[0] == "buf"]
                    cap = min(bufs) if bufs else 64
                    args.append(("u32", rng.choice([rng.randint(0, cap), rng.randint(0, cap),
                                                    rng.randint(0, 2 * cap + 8), cap]))
                                if x > 0.06 else rng.choice([("u32", -1), ("u32", 2**32),
                                                             ("f64", 1.5), ("buf", 0)]))
            if name == "mandelbrot":  # a sensible viewport and small images mostly
                args[3:8] = [("f64", -2.0), ("f64", 1.0), ("f64", -1.5), ("f64", 1.5), ("f64", 4.0)]
                cap = sizes[args[0][1]] // 4 if args[0][0] == "buf" else 64
                wd = rng.randint(1, 40)
                args[1] = ("u32", wd)
                args[2] = ("u32", rng.randint(1, max(1, cap // wd)) if rng.random() < 0.8
                           else rng.randint(1, 40))
                args[8] = ("u32", rng.randint(0, 80))
            if name in ("stencil", "stencil2d") and args[0] == args[1]:
                args[1] = ("buf", (args[0][1] + 1) % len(sizes)) if args[0][0] == "buf" else args[1]
                if args[0] == args[1]:
                    continue
            if rng.random() < 0.04:
                args = args[:-1] if rng.random() < 0.5 else args + [("u32", 1)]
            block = rng.choice([(32, 1, 1), (64, 1, 1), (128, 1, 1), (8, 4, 1), (16, 2, 2)])
            items = rng.randint(1, 900)
            vol = block[0] * block[1] * block[2]
            grid = ((items + vol - 1) // vol, 1, 1)
            if rng.random() < 0.03:
                grid = rng.choice([(0, 1, 1), (1, 0, 1), (2**20, 2**13, 1)])
            ops.append(("run", name, args, grid, block, rng.random() < 0.06))
        elif r < 0.86:
            d = rng.randrange(len(sizes))
            so = rng.choice([0, rng.randint(0, size), size + 1])
            do = rng.choice([0, rng.randint(0, sizes[d]), -2])
            n = rng.choice([rng.randint(0, 64), min(size, sizes[d]), size + 8])
            ops.append(("copy", b, so, d, do, n))
        elif r < 0.91:
            ops.append(("gate",))
        elif r < 0.94:
            ops.append(("sync",))
        elif r < 0.97:
            ops.append(("stream",))
        else:
            ops.append(("unregister", b))
    return ops


def _execute(w: World, ops, tainted: set, owner: list = None) -> list:
    """Outcomes of the plan; `owner` (if given) gets the op index of each."""
    out = []
    pending = []  # tokens gated by the next "gate"
    for i_op, op in enumerate(ops):
        if owner is not None:
            owner.extend([i_op - 1] * (len(out) - len(owner)))
        kind = op[0]
        if kind == "create":
            res = w.outcome(lambda: w.dev.create_buffer(op[1]))
            if res[0] == "ok":
                w.bufs.append(res[1])
                res = ("ok", res[1].size_bytes)
            out.append(res)
        elif kind == "write":
            b = w.bufs[op[1]]
            if b is None:
                out.append(("skip",))
                continue
            tok = w.outcome(lambda: b.enqueue_write(op[2], op[3]))
            out.append(tok)
            if tok[0] == "ok" and op[2] == 0 and len(op[3]) == b.size_bytes:
                tainted.discard(op[1])  # fully rewritten: comparable again
        elif kind == "read":
            b = w.bufs[op[1]]
            if b is None or op[1] in tainted:
                out.append(("skip",))
                continue
            out.append(w.outcome(lambda: b.enqueue_read(op[2], op[3])))
        elif kind == "run":
            _, name, args, grid, block, gated = op
            if any(a[0] == "buf" and w.bufs[a[1]] is None for a in args):
                out.append(("skip",))
                continue
            prog, built = w.program(KERNELS[name][0])
            if name not in built:
                res = w.outcome(lambda: prog.build(name))
                out.append(("build",) + res)
                built.add(name)
            vals = []
            for a in args:
                if a[0] == "buf":
                    vals.append(w.bufs[a[1]])
                elif a[0] == "f64":
                    vals.append(float(a[1]))
                else:
                    vals.append(int(a[1]))
            if gated:  # issued now, observed at the next gate (stream order holds)
                try:
                    pending.append(prog.run(vals, name, grid, block))
                    res = ("queued",)
                except Exception as exc:  # noqa: BLE001
                    res = ("raise", type(exc).__name__)
            else:
                res = w.outcome(lambda: prog.run(vals, name, grid, block))
            out.append(res)
            # an aborted run (partial writes on the reference side only), or
            # one reading a buffer whose contents already differ, leaves its
            # output incomparable; runs rejected before executing (arity,
            # kinds, u32 range, launch shape) write nothing on either side
            reads_tainted = any(a[0] == "buf" and a[1] in tainted for a in args)
            o = args[OUTPUT_ARG[name]] if OUTPUT_ARG[name] < len(args) else None
            # a gated run may still abort part way: its output is
            # incomparable from the moment it is queued (later operations in
            # stream order may read the reference's partial writes)
            if o is not None and o[0] == "buf" and (
                    res in (("queued",), ("fail", "OobAccessError")) or reads_tainted):
                tainted.add(o[1])
        elif kind == "copy":
            _, s, so, d, do, n = op
            src, dst = w.bufs[s], w.bufs[d]
            if src is None or dst is None or s in tainted:
                out.append(("skip",))
                continue
            out.append(w.outcome(lambda: w.pkg.copy(src, so, dst, do, n)))
        elif kind == "gate":
            toks, pending = pending, []
            out.append(w.outcome(lambda: w.pkg.when_all(toks)))
        elif kind == "sync":
            out.append(w.outcome(lambda: w.dev.synchronize()))
        elif kind == "stream":
            out.append(w.outcome(w.dev.create_stream))
        elif kind == "unregister":
            b = w.bufs[op[1]]
            if b is None:
                out.append(("skip",))
                continue
            out.append(w.outcome(lambda: w.rt.registry.unregister(b.gid)))
            # the handle now names nothing: one more use must fail alike
            out.append(w.outcome(lambda: b.enqueue_read(0, min(8, b.size_bytes))))
            w.bufs[op[1]] = None
    if pending:
        out.append(w.outcome(lambda: w.pkg.when_all(pending)))
    # final state of every live, untainted buffer
    for i, b in enumerate(w.bufs):
        if b is not None and i not in tainted:
            out.append(("final", i) + w.outcome(lambda: b.enqueue_read(0, b.size_bytes)))
    return out


def _same(a, b) -> bool:
    if a == b:
        return True
    if (len(a) == len(b) and a[:-1] == b[:-1] and isinstance(a[-1], bytes)
            and isinstance(b[-1], bytes) and len(a[-1]) == len(b[-1]) and len(a[-1]) % 8 == 0):
        x = np.frombuffer(a[-1], np.float64)
        y = np.frombuffer(b[-1], np.float64)
        return bool(np.all((x.view(np.uint64) == y.view(np.uint64)) | (np.isnan(x) & np.isnan(y))))
    return False


@pytest.mark.parametrize("seed", SEEDS)
def test_random_plan_matches_reference(worlds, seed):
    ops = _plan(seed)
    ref_pkg, ref_rt, ref_dev = worlds["ref"]
    our_pkg, our_rt, our_dev = worlds["ours"]
    t_ref: set = set()
    t_our: set = set()
    got_ref = _execute(World(ref_pkg, ref_rt, ref_dev, worlds["sources"]), ops, t_ref)
    got_our = _execute(World(our_pkg, our_rt, our_dev, worlds["sources"]), ops, t_our)
    assert t_ref == t_our
    assert len(got_ref) == len(got_our)
    for i, (a, b) in enumerate(zip(got_ref, got_our)):
        assert _same(a, b), f"seed {seed} outcome {i}: reference {a!r:.300} vs ours {b!r:.300}"
    # the plan compared real data, not only error classes
    data = [o for o in got_ref if isinstance(o[-1], bytes) and o[-1]]
    assert len(data) >= 2, f"seed {seed}: only {len(data)} data comparisons"
