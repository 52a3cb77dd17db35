"""Generate tests/golden/golden.json by running the REFERENCE implementation.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every expected output below comes from the reference package `offloadrt`
executing the workload through its own public API on its `host` backend
(numba whole-grid executor, /root/reference/pkg/src/offloadrt/kernel/
codegen.py) — never from this repository's code.  STREAM and the T-step heat
equation have no reference kernel; they are produced by the reference
executor running the .k sources in paper_1810_11482_b200/kernels/ (same
language), i.e. the reference's semantics applied to those programs.
Inputs are regenerated from the recorded seeds (numpy default_rng).
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

from offloadrt import Runtime  # noqa: E402  (reference package)
from offloadrt.bench import kernel_source  # noqa: E402

VIEWPORT = (-2.0, 1.0, -1.5, 1.5)


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def mine(name: str) -> str:
    with open(os.path.join(REPO, "paper_1810_11482_b200", "kernels", f"{name}.k")) as fh:
        return fh.read()


def run(device, source, kernel, args, items, block=256):
    prog = device.create_program_with_source(source).get()
    prog.build(kernel).get(timeout=600)
    grid = (max(1, math.ceil(items / block)), 1, 1)
    prog.run(args, kernel, grid, (block, 1, 1)).get(timeout=3600)


def buf_with(device, data: bytes):
    b = device.create_buffer(len(data)).get()
    b.enqueue_write(0, data).get(timeout=600)
    return b


SEMANTICS_SRC = """
kernel semantics(a : buffer_f64, b : buffer_u32, s : scalar_f64, m : scalar_u32) {
    if (gtid < u32(8)) {
        let fi = f64(gtid);
        let x = s * fi + 0.125;
        let wrapped = (m + gtid) * 4294967295;
        let q = (m + 10) / (gtid + 1);
        let picked = select(x > 1.0 && gtid != 3, sqrt(abs(x)), min(x, 2.0));
        let trig = sin(x) * cos(x);
        let clipped = max(u32(x * 100.0), wrapped);
        let acc = 0.0;
        for i in 0 .. 6 {
            acc = acc + f64(i) * 0.5;
            break if (acc > 4.0);
        }
        a[gtid] = picked + trig + acc + f64(q);
        b[gtid] = clipped;
    }
}
"""

# (source, kernel, buffers [(kind, n)], scalars, grid, block)
LANG_CASES = [
    (SEMANTICS_SRC, "semantics", [("f64", 8), ("u32", 8)], [1.75, 123456789], (1, 1, 1), (8, 1, 1)),
    (SEMANTICS_SRC, "semantics", [("f64", 8), ("u32", 8)], [-2.5, 4294967295], (2, 1, 1), (4, 1, 1)),
    ("kernel w(out : buffer_u32, a : scalar_u32, b : scalar_u32) { out[0] = a * b; out[1] = a - b; }",
     "w", [("u32", 2)], [4000000000, 4000000001], (1, 1, 1), (1, 1, 1)),
    ("kernel d(out : buffer_u32, a : scalar_u32, b : scalar_u32) { out[0] = a / b; }",
     "d", [("u32", 1)], [7, 2], (1, 1, 1), (1, 1, 1)),
    ("kernel d(out : buffer_f64, b : scalar_f64) { out[0] = 1.0 / b; }",
     "d", [("f64", 1)], [0.0], (1, 1, 1), (1, 1, 1)),
    ("kernel o(out : buffer_f64, i : scalar_u32) { out[i] = 1.0; }",
     "o", [("f64", 4)], [9], (1, 1, 1), (1, 1, 1)),
    ("kernel n(out : buffer_f64) { out[gtid - 1] = 1.0; }", "n", [("f64", 4)], [], (1, 1, 1), (1, 1, 1)),
    ("""kernel b(blocks : buffer_u32, threads : buffer_u32, dims : buffer_u32) {
    blocks[gtid] = block_idx;
    threads[gtid] = thread_idx;
    if (gtid == 0) { dims[0] = grid_dim; dims[1] = block_dim; }
}""", "b", [("u32", 12), ("u32", 12), ("u32", 2)], [], (3, 1, 1), (2, 2, 1)),
    ("""kernel s(out : buffer_f64, flag : scalar_u32) {
    if (gtid == 0) { let hit = 0.0; if (flag == 1 && out[99] > 0.0) { hit = 1.0; } out[0] = hit; }
}""", "s", [("f64", 4)], [0], (1, 1, 1), (1, 1, 1)),
    ("""kernel s(out : buffer_f64, flag : scalar_u32) {
    if (gtid == 0) { let hit = 0.0; if (flag == 1 && out[99] > 0.0) { hit = 1.0; } out[0] = hit; }
}""", "s", [("f64", 4)], [1], (1, 1, 1), (1, 1, 1)),
    ("""kernel s(out : buffer_f64, flag : scalar_u32) {
    if (gtid == 0) { if (flag == 1) { let t = 2.5; out[0] = t; } else { let t = 7; out[0] = f64(t); } }
}""", "s", [("f64", 1)], [0], (1, 1, 1), (1, 1, 1)),
    ("""kernel l(out : buffer_u32, n : scalar_u32) {
    if (gtid == 0) { let total = 0; for i in 0 .. n { let double = i * 2; total = total + double; } out[0] = total; }
}""", "l", [("u32", 1)], [5], (1, 1, 1), (1, 1, 1)),
    ("kernel c(out : buffer_u32, x : scalar_f64) { out[gtid] = u32(x); }",
     "c", [("u32", 1)], [-3.7], (1, 1, 1), (1, 1, 1)),
    ("kernel c(out : buffer_u32, x : scalar_f64) { out[gtid] = u32(x); }",
     "c", [("u32", 1)], [1e19], (1, 1, 1), (1, 1, 1)),
    ("""kernel poly(y : buffer_f64, x : buffer_f64, n : scalar_u32) {
    if (gtid < n) { let v = x[gtid]; y[gtid] = ((v * 3.0 - 1.5) * v + 0.25) / (v + 2.0); }
}""", "poly", [("f64", 1000), ("f64", 1000)], [1000], (4, 1, 1), (256, 1, 1)),
]


def lang_cases(dev) -> list:
    from offloadrt.errors import OffloadError

    res = []
    for src, name, bufs, scalars, grid, block in LANG_CASES:
        prog = dev.create_program_with_source(src).get()
        prog.build(name).get(timeout=600)
        handles, inits = [], []
        rng = np.random.default_rng(len(res))
        for kind, n in bufs:
            dt = np.float64 if kind == "f64" else np.uint32
            init = (rng.random(n) if kind == "f64" else np.zeros(n)).astype(dt)
            h = dev.create_buffer(n * dt().itemsize).get()
            h.enqueue_write(0, init.tobytes()).get()
            handles.append(h)
            inits.append(init.tobytes().hex())
        err = None
        try:
            prog.run(handles + scalars, name, grid, block).get(timeout=600)
        except OffloadError as exc:
            err = [type(exc).__name__, str(exc)]
        outs = [h.enqueue_read_sync(0, h.size_bytes).hex() for h in handles]
        res.append({"source": src, "kernel": name, "buffers": bufs, "scalars": scalars,
                    "grid": list(grid), "block": list(block), "inputs_hex": inits,
                    "outputs_hex": outs, "error": err})
    return res


STENCIL2D_CASES = ((4, 3, 501, None), (5, 4, 502, None), (64, 48, 503, None),
                   (64, 48, 504, 1000), (63, 47, 505, None), (1, 9, 506, None),
                   (1024, 768, 507, None), (1000, 601, 508, None))


def stencil2d_cases(dev) -> dict:
    """kernels/stencil2d.k executed by the reference (one step, several grid
    shapes incl. odd widths, a partial launch) and 20 ping-pong steps."""
    src = mine("stencil2d")
    cases = []
    for w, h, seed, items in STENCIL2D_CASES:
        x = np.random.default_rng(seed).random(w * h)
        xb, yb = buf_with(dev, x.tobytes()), dev.create_buffer(w * h * 8).get()
        # a partial launch must cover exactly `items` work items: block 8
        run(dev, src, "stencil2d", [xb, yb, w, h], w * h if items is None else items,
            256 if items is None else 8)
        raw = yb.enqueue_read_sync(0, w * h * 8)
        case = {"w": w, "h": h, "seed": seed, "items": items, "sha256": sha(raw)}
        if w * h <= 64:
            case["input"] = x.tolist()
            case["output"] = np.frombuffer(raw, np.float64).tolist()
        cases.append(case)
    heat = []
    for w, h, steps, seed in ((128, 96, 20, 511), (257, 130, 7, 512)):
        x = np.random.default_rng(seed).random(w * h)
        a, b = buf_with(dev, x.tobytes()), dev.create_buffer(w * h * 8).get()
        prog = dev.create_program_with_source(src).get()
        prog.build("stencil2d").get(timeout=600)
        grid = (math.ceil(w * h / 256), 1, 1)
        for s in range(steps):
            s_, d_ = (a, b) if s % 2 == 0 else (b, a)
            prog.run([s_, d_, w, h], "stencil2d", grid, (256, 1, 1))
        final = a if steps % 2 == 0 else b
        heat.append({"w": w, "h": h, "steps": steps, "seed": seed,
                     "sha256": sha(final.enqueue_read_sync(0, w * h * 8))})
    return {"step": cases, "heat": heat}


def fuzz_cases(dev, count: int = 150) -> list:
    """Random well-typed kernels from the reference's own generator
    (pkg/tests/kernelgen.py), run by the reference on ONE work item (no
    write races, so a parallel executor must match bit for bit), with the
    final buffer states and any abort.  sin/cos-free: glibc and CUDA libm may
    differ in the last ulp, which integer casts can amplify."""
    import random

    sys.path.insert(0, "/root/reference/pkg/tests")
    from kernelgen import random_kernel
    from offloadrt.errors import OffloadError

    rng = random.Random(0x1810)
    cases = []
    while len(cases) < count:
        src = random_kernel(rng)
        if "sin(" in src or "cos(" in src:
            continue
        prog = dev.create_program_with_source(src).get()
        prog.build("fuzzed").get(timeout=600)
        irs = __import__("offloadrt.kernel", fromlist=["parse_and_validate"]).parse_and_validate(src)
        params = irs["fuzzed"].params
        vr = np.random.default_rng(len(cases))
        handles, inits, args = [], [], []
        for _, kind in params:
            if kind == "buffer_f64":
                init = vr.uniform(-100.0, 100.0, size=24)
            elif kind == "buffer_u32":
                init = vr.integers(0, 2**32, size=24, dtype=np.uint32)
            else:
                init = None
            if init is not None:
                h = dev.create_buffer(init.nbytes).get()
                h.enqueue_write(0, init.tobytes()).get()
                handles.append(h)
                inits.append(["buf", kind, init.tobytes().hex()])
                args.append(h)
            elif kind == "scalar_f64":
                v = float(vr.uniform(-50.0, 50.0))
                inits.append(["f64", kind, v])
                args.append(v)
            else:
                v = int(vr.integers(0, 2**32))
                inits.append(["u32", kind, v])
                args.append(v)
        err = None
        try:
            prog.run(args, "fuzzed", (1, 1, 1), (1, 1, 1)).get(timeout=600)
        except OffloadError as exc:
            err = [type(exc).__name__, str(exc)]
        outs = [h.enqueue_read_sync(0, h.size_bytes).hex() for h in handles]
        cases.append({"source": src, "args": inits, "outputs_hex": outs, "error": err})
    return cases


DOT_SEQ_SRC = """
# fp32 dot product restated in the reference language (no f32 type,
# lang.py:29): the f64 buffers hold fp32 values, so every product is exact
# in f64 and work item 0 accumulates them in index order (pattern sum.k:3-11).
kernel dot_seq(a : buffer_f64, b : buffer_f64, res : buffer_f64, n : scalar_u32) {
    if (gtid == 0) {
        let acc = 0.0;
        for i in 0 .. n {
            acc = acc + a[i] * b[i];
        }
        res[0] = acc;
    }
}
"""

# (n, seed): BASELINE config 4 inputs are rng(seed).random(n, float32) for a,
# then b; the full 2^31 is beyond the reference's 8-GiB-per-buffer host path,
# so the reference runs prefixes of the same generator family.
DOT_CASES = ((1 << 24, 20180214), ((1 << 24) + 3, 611), (1 << 26, 20180214))

# (n, steps, seed): config 2 (2^28 x 1000, the reference's stencil.k
# iterated ping-pong, harness.py:199-230 inputs) and a 2^20 x 1000 case.
HEAT_LONG = ((1 << 20, 1000, 20180214), (1 << 28, 1000, 20180214))


def dot_long(dev) -> list:
    cases = []
    for n, seed in DOT_CASES:
        rng = np.random.default_rng(seed)
        a = rng.random(n, dtype=np.float32)
        b = rng.random(n, dtype=np.float32)
        ab = buf_with(dev, a.astype(np.float64).tobytes())
        bb = buf_with(dev, b.astype(np.float64).tobytes())
        rb = dev.create_buffer(8).get()
        t1 = time.time()
        run(dev, DOT_SEQ_SRC, "dot_seq", [ab, bb, rb, n], 32, 32)
        res = float(np.frombuffer(rb.enqueue_read_sync(0, 8), np.float64)[0])
        cases.append({"n": n, "seed": seed, "result": res, "result_hex": float.hex(res),
                      "reference_seconds": round(time.time() - t1, 2)})
        print("dot", cases[-1], flush=True)
    return cases


def heat_long(dev, only_small: bool = False) -> list:
    cases = []
    for n, steps, seed in HEAT_LONG:
        if only_small and n > (1 << 20):
            continue
        x = np.random.default_rng(seed).random(n)
        a, b = buf_with(dev, x.tobytes()), dev.create_buffer(n * 8).get()
        del x
        prog = dev.create_program_with_source(kernel_source("stencil")).get()
        prog.build("stencil").get(timeout=600)
        grid = (math.ceil(n / 256), 1, 1)
        t1 = time.time()
        for s in range(steps):
            src, dst = (a, b) if s % 2 == 0 else (b, a)
            prog.run([src, dst, n], "stencil", grid, (256, 1, 1)).get(timeout=3600)
            if s % 50 == 0:
                print(f"heat n={n} step {s} {time.time() - t1:.1f}s", flush=True)
        final = a if steps % 2 == 0 else b
        raw = final.enqueue_read_sync(0, n * 8)
        vals = np.frombuffer(raw, np.float64)
        cases.append({"n": n, "steps": steps, "seed": seed, "sha256": sha(raw),
                      "sum": float(vals.sum()), "max": float(vals.max()),
                      "reference_seconds": round(time.time() - t1, 1)})
        print("heat", cases[-1], flush=True)
        del raw, vals
    return cases


def long_main() -> None:
    """--long: reference outputs for config 2 (full 2^28 x 1000 heat, ~20 min
    on the host backend) and config 4 (sequential fp64 dot of fp32 values),
    written to golden_long.json."""
    path = os.path.join(HERE, "golden_long.json")
    out = {"generator": "tests/golden/make_golden.py --long",
           "reference": "offloadrt (host backend)"}
    small = "--small" in sys.argv
    with Runtime(backend="host") as rt:
        dev = rt.get_all_devices().get()[0]
        out["dot"] = dot_long(dev)
        out["heat"] = heat_long(dev, only_small=small)
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote {path}")


def main() -> None:
    if "--long" in sys.argv:
        return long_main()
    if "--only-fuzz" in sys.argv:  # add/refresh the fuzz section in place
        path = os.path.join(HERE, "golden.json")
        with open(path) as fh:
            out = json.load(fh)
        with Runtime(backend="host") as rt:
            out["fuzz"] = fuzz_cases(rt.get_all_devices().get()[0])
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
        print(f"updated fuzz ({len(out['fuzz'])} kernels) in golden.json")
        return
    if "--only-stencil2d" in sys.argv:  # add/refresh one section in place
        path = os.path.join(HERE, "golden.json")
        with open(path) as fh:
            out = json.load(fh)
        with Runtime(backend="host") as rt:
            out["stencil2d"] = stencil2d_cases(rt.get_all_devices().get()[0])
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
        print("updated stencil2d in golden.json")
        return
    out: dict = {"generator": "tests/golden/make_golden.py", "reference": "offloadrt (host backend)"}
    t0 = time.time()
    with Runtime(backend="host") as rt:
        dev = rt.get_all_devices().get()[0]
        out["stencil2d"] = stencil2d_cases(dev)
        out["fuzz"] = fuzz_cases(dev)

        # -- stencil: hand case + random sizes (test_acceptance.py:62-66) ----
        cases = []
        x = np.array([1.0, 2.0, 3.0, 4.0])
        xb, yb = buf_with(dev, x.tobytes()), dev.create_buffer(32).get()
        run(dev, kernel_source("stencil"), "stencil", [xb, yb, 4], 4, 32)
        cases.append({"n": 4, "input": x.tolist(),
                      "output": np.frombuffer(yb.enqueue_read_sync(0, 32), np.float64).tolist()})
        for n, seed in ((8, 101), (1024, 102), (1 << 20, 103)):
            x = np.random.default_rng(seed).random(n)
            xb, yb = buf_with(dev, x.tobytes()), dev.create_buffer(n * 8).get()
            run(dev, kernel_source("stencil"), "stencil", [xb, yb, n], n, 32)
            raw = yb.enqueue_read_sync(0, n * 8)
            case = {"n": n, "seed": seed, "sha256": sha(raw)}
            if n <= 1024:
                case["output_hex"] = raw.hex()
            cases.append(case)
        out["stencil"] = cases

        # -- heat: T applications, ping-pong (config 2 semantics) ------------
        cases = []
        for n, steps, seed in ((4096, 100, 201), (1 << 16, 10, 202)):
            x = np.random.default_rng(seed).random(n)
            a, b = buf_with(dev, x.tobytes()), dev.create_buffer(n * 8).get()
            prog = dev.create_program_with_source(kernel_source("stencil")).get()
            prog.build("stencil").get(timeout=600)
            grid = (math.ceil(n / 256), 1, 1)
            for s in range(steps):
                src, dst = (a, b) if s % 2 == 0 else (b, a)
                prog.run([src, dst, n], "stencil", grid, (256, 1, 1))
            final = a if steps % 2 == 0 else b
            raw = final.enqueue_read_sync(0, n * 8)
            cases.append({"n": n, "steps": steps, "seed": seed, "sha256": sha(raw)})
        out["heat"] = cases

        # -- sum (test_bench.py:57-59, test_program.py:149-161, acceptance) --
        cases = []
        for values, label in ((np.array([2**32 - 1, 5], np.uint32), "wrap"),
                              (np.ones(1000, np.uint32), "ones")):
            ib, rb = buf_with(dev, values.tobytes()), dev.create_buffer(4).get()
            run(dev, kernel_source("sum"), "sum", [ib, rb, len(values)], 32, 32)
            cases.append({"label": label, "values": values.tolist(),
                          "result": int(np.frombuffer(rb.enqueue_read_sync(0, 4), np.uint32)[0])})
        for n, seed in ((8, 301), (1024, 302), (1 << 20, 303)):
            values = np.random.default_rng(seed).integers(0, 2**32, size=n, dtype=np.uint32)
            ib, rb = buf_with(dev, values.tobytes()), dev.create_buffer(4).get()
            run(dev, kernel_source("sum"), "sum", [ib, rb, n], 32, 32)
            cases.append({"n": n, "seed": seed,
                          "result": int(np.frombuffer(rb.enqueue_read_sync(0, 4), np.uint32)[0])})
        out["sum"] = cases

        # -- mandelbrot (acceptance 16/64/256 @256; hand 3x3; origin) --------
        cases = []
        for w, h, max_iter, vp in (
            (16, 16, 256, VIEWPORT), (64, 64, 256, VIEWPORT), (256, 256, 256, VIEWPORT),
            (24, 16, 256, VIEWPORT), (3, 3, 64, (-0.5, 2.5, -1.5, 1.5)),
            (3, 3, 50, (-1.5, 1.5, -1.5, 1.5)), (960, 540, 2000, VIEWPORT),
        ):
            ob = dev.create_buffer(w * h * 4).get()
            run(dev, kernel_source("mandelbrot"), "mandelbrot",
                [ob, w, h, *vp, 4.0, max_iter], w * h, 256)
            raw = ob.enqueue_read_sync(0, w * h * 4)
            counts = np.frombuffer(raw, np.uint32)
            case = {"width": w, "height": h, "max_iter": max_iter, "viewport": list(vp),
                    "esc": 4.0, "sha256": sha(raw), "sum": int(counts.astype(np.uint64).sum())}
            if w * h <= 4096:
                case["counts"] = counts.tolist()
            cases.append(case)
        if os.environ.get("GOLDEN_FULL_MANDELBROT", "1") == "1":
            w, h, max_iter = 7680, 4320, 2000
            ob = dev.create_buffer(w * h * 4).get()
            t1 = time.time()
            run(dev, kernel_source("mandelbrot"), "mandelbrot",
                [ob, w, h, *VIEWPORT, 4.0, max_iter], w * h, 256)
            raw = ob.enqueue_read_sync(0, w * h * 4)
            counts = np.frombuffer(raw, np.uint32)
            cases.append({"width": w, "height": h, "max_iter": max_iter,
                          "viewport": list(VIEWPORT), "esc": 4.0, "sha256": sha(raw),
                          "sum": int(counts.astype(np.uint64).sum()),
                          "reference_seconds": round(time.time() - t1, 2)})
        out["mandelbrot"] = cases

        # -- partition (acceptance m=1 p=4; backend equivalence offset 17) ---
        cases = []
        for offset, count in ((17, 512), (9, 512), (0, 2_097_152), (4294967000, 1000)):
            ob = dev.create_buffer(count * 8).get()
            run(dev, kernel_source("partition"), "partition", [ob, offset, count], count, 256)
            raw = ob.enqueue_read_sync(0, count * 8)
            vals = np.frombuffer(raw, np.float64)
            case = {"offset": offset, "count": count, "sha256": sha(raw),
                    "max_abs_dev_from_1": float(np.abs(vals - 1.0).max())}
            if count <= 1000:
                case["output_hex"] = raw.hex()
            cases.append(case)
        out["partition"] = cases

        # -- STREAM via the reference executor running kernels/stream.k ------
        cases = []
        n, s = 1 << 20, 3.0
        rng = np.random.default_rng(401)
        b = rng.random(n)
        c = rng.random(n)
        for op, args_of in (
            ("copy", lambda A, B, C: [A, B, n]),
            ("scale", lambda A, B, C: [A, B, s, n]),
            ("add", lambda A, B, C: [A, B, C, n]),
            ("triad", lambda A, B, C: [A, B, C, s, n]),
        ):
            A = dev.create_buffer(n * 8).get()
            B, C = buf_with(dev, b.tobytes()), buf_with(dev, c.tobytes())
            run(dev, mine("stream"), op, args_of(A, B, C), n, 256)
            raw = A.enqueue_read_sync(0, n * 8)
            cases.append({"op": op, "n": n, "seed": 401, "scalar": s, "sha256": sha(raw)})
        out["stream"] = cases

        # -- generic kernel-language semantics (NVRTC path) -----------------
        out["lang"] = lang_cases(dev)

    out["seconds"] = round(time.time() - t0, 1)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote golden.json in {out['seconds']} s")


if __name__ == "__main__":
    sys.exit(main())
