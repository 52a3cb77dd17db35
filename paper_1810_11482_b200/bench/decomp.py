"""Pure decomposition arithmetic shared by the multi-device workloads (and
unit-tested on CPU with multi-process gloo, tests/test_multiproc_cpu.py).

* contiguous shards  — STREAM replicas and the dot product (config 1, 4)
* slabs with halos   — heat equation (config 2)
* cyclic rows        — Mandelbrot (config 3)
* i mod k            — the paper's Alg. 1 partitions (harness.py:266-283)
"""

from __future__ import annotations

from dataclasses import dataclass


def shard_bounds(n: int, parts: int) -> list:
    """[b0=0, b1, ..., b_parts=n], contiguous and balanced within one."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    return [n * g // parts for g in range(parts + 1)]


@dataclass(frozen=True)
class Slab:
    lo: int        # first owned global cell
    hi: int        # one past the last owned cell
    left: int      # ghost cells before lo
    right: int     # ghost cells after hi

    @property
    def owned(self) -> int:
        return self.hi - self.lo

    @property
    def length(self) -> int:
        return self.owned + self.left + self.right

    @property
    def start(self) -> int:
        """global index of local cell 0"""
        return self.lo - self.left


def slabs(n: int, parts: int, halo: int) -> list:
    """1-D slab decomposition with `halo` ghosts on every inner side.  Local
    cell 0 / length-1 of a slab is either a global endpoint (held fixed by
    stencil.k) or a ghost refreshed by the exchange every `halo` steps, so
    running the unmodified stencil on each slab for <= halo steps leaves the
    owned cells exactly as the global run would."""
    b = shard_bounds(n, parts)
    out = []
    for g in range(parts):
        left = 0 if g == 0 else halo
        right = 0 if g == parts - 1 else halo
        if b[g + 1] - b[g] < halo + 1:
            raise ValueError("slabs must be longer than the halo")
        out.append(Slab(b[g], b[g + 1], left, right))
    return out


def halo_exchanges(layout: list, halo: int) -> list:
    """(src_part, src_local_cell, dst_part, dst_local_cell, cells) copies that
    refresh every ghost region from its owner."""
    ex = []
    for g in range(len(layout) - 1):
        a, b = layout[g], layout[g + 1]
        # a's last `halo` owned cells -> b's left ghosts
        ex.append((g, a.left + a.owned - halo, g + 1, 0, halo))
        # b's first `halo` owned cells -> a's right ghosts
        ex.append((g + 1, b.left, g, a.left + a.owned, halo))
    return ex


def cyclic_rows(height: int, parts: int, part: int) -> range:
    """Rows of `part` under the cyclic split (row r -> part r mod parts)."""
    return range(part, height, parts)


def partition_device(i: int, devices: int) -> int:
    """Alg. 1: partition i runs on device i mod k (harness.py:266-283)."""
    return i % devices
