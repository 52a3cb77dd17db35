"""The reference's benchmark harness and CLI, on the CUDA runtime: every
run validates against its oracle before reporting (reference
bench/harness.py:1-7), CSV rows keep the reference's columns."""

from __future__ import annotations

import csv

import numpy as np
import pytest

from paper_1810_11482_b200.bench import (
    MandelbrotConfig,
    PartitionConfig,
    StencilConfig,
    TimingProtocol,
    append_csv,
    run_mandelbrot,
    run_mandelbrot_series,
    run_partition,
    run_stencil,
    run_stream,
    run_sum,
)
from paper_1810_11482_b200.cli import bench_main

pytestmark = pytest.mark.gpu
FAST = TimingProtocol(iterations=3, discard=1)


def test_run_stencil_sum_stream(dev):
    assert run_stencil(StencilConfig(n=100_000), dev, FAST).validated
    assert run_sum(1 << 20, dev, FAST).validated
    r = run_stream("triad", 1 << 22, dev, FAST)
    assert r.validated and r.config["gbs"] > 0


def test_run_partition_alg1(dev, rt2):
    r = run_partition(PartitionConfig(m=1, partitions=4), [dev], FAST)
    assert r.validated and r.n_or_pixels == 2_097_152
    r2 = run_partition(PartitionConfig(m=1, partitions=3), rt2.get_all_devices().get(), FAST)
    assert r2.validated and r2.devices == 2 and r2.n_or_pixels == 2 * 1024 * 256


def test_run_mandelbrot_ppm_and_series(dev, tmp_path):
    path = tmp_path / "m.ppm"
    r = run_mandelbrot(MandelbrotConfig(width=64, height=48), dev, FAST, image_path=path)
    assert r.validated
    data = path.read_bytes()
    assert data.startswith(b"P6\n64 48\n255\n") and len(data) == len(b"P6\n64 48\n255\n") + 64 * 48 * 3
    reports, events = run_mandelbrot_series([32, 64], dev, FAST, async_write=True, out_dir=str(tmp_path))
    assert all(r.validated for r in reports)
    assert {e.kind for e in events} == {"compute", "write"}


def test_csv_and_cli(dev, tmp_path, capsys):
    out = tmp_path / "r.csv"
    append_csv(out, run_sum(1000, dev, FAST))
    assert bench_main(["stencil", "--size", "4096", "--iterations", "2", "--csv", str(out)]) == 0
    assert bench_main(["stream", "--size", "65536", "--iterations", "2", "--csv", str(out)]) == 0
    assert bench_main(["mandelbrot", "--size", "32", "--iterations", "2", "--out-dir", str(tmp_path)]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["benchmark", "backend", "devices", "partitions", "n_or_pixels", "mean_ms", "validated"]
    assert [r[0] for r in rows[1:]] == ["sum", "stencil", "stream_triad"]
    assert all(r[-1] == "1" for r in rows[1:])
    assert "validated=True" in capsys.readouterr().out


def test_dot_multi_single_device(dev):
    from paper_1810_11482_b200.bench import dot_multi

    import oracle

    a = np.random.default_rng(1).random(1 << 20, dtype=np.float32)
    b = np.random.default_rng(2).random(1 << 20, dtype=np.float32)
    got = dot_multi([dev], a, b)
    exp = oracle.dot_f32(a, b)
    assert abs(got - exp) <= 1e-12 * abs(exp)
