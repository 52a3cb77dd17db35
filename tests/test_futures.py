"""Futures laws (CPU), mirroring the reference's test_futures.py: one-shot
transitions, continuation order, error propagation, broken promises,
when_all conjunction — plus the deep when_all chains the overhead sweep
builds (iterative resolution, no recursion limit)."""

from __future__ import annotations

import gc
import random
import threading

import pytest

from paper_1810_11482_b200.errors import AlreadyCompletedError, BrokenPromiseError
from paper_1810_11482_b200.futures import Promise, get, make_failed, make_ready, when_all


class Boom(Exception):
    pass


def test_ready_and_failed():
    assert make_ready(3).get() == 3
    t = make_failed(Boom("x"))
    assert t.is_failed() and isinstance(t.error(), Boom)
    with pytest.raises(Boom):
        t.get()
    assert get(make_ready("v")) == "v"


def test_promise_once():
    p = Promise()
    p.set_value(1)
    with pytest.raises(AlreadyCompletedError):
        p.set_value(2)
    assert not p.try_set_error(Boom())
    assert p.token.get() == 1


def test_broken_promise():
    p = Promise()
    tok = p.token
    del p
    gc.collect()
    with pytest.raises(BrokenPromiseError):
        tok.get(timeout=1)


def test_then_order_and_errors():
    p = Promise()
    order = []
    t1 = p.token.then(lambda v: order.append(1) or v + 1)
    t2 = p.token.then(lambda v: order.append(2) or v * 10)
    t3 = t1.then(lambda v: 1 / 0)
    t4 = t3.then(lambda v: order.append("never"))
    p.set_value(4)
    assert order == [1, 2]
    assert t1.get() == 5 and t2.get() == 40
    with pytest.raises(ZeroDivisionError):
        t4.get()
    assert make_ready(1).then(lambda v: v + 1).get() == 2  # inline on the caller


def test_then_on_pool():
    p = Promise()
    names = []
    t = p.token.then(lambda v: names.append(threading.current_thread().name) or v, on_pool=True)
    p.set_value(9)
    assert t.get(timeout=5) == 9
    assert names[0].startswith("ofl-pool")


def test_when_all_laws():
    assert when_all([]).get() is None
    a, b = Promise(), Promise()
    t = when_all([a.token, b.token])
    assert not t.done()
    a.set_value(1)
    assert not t.done()
    b.set_value(2)
    assert t.get() is None
    c, d = Promise(), Promise()
    u = when_all([c.token, d.token])
    fired = []
    u.then(lambda _: fired.append(1))
    d.set_error(Boom("first"))
    with pytest.raises(Boom):
        u.get()
    c.set_value(0)  # nothing cancelled, nothing re-fired
    assert fired == []


def test_get_timeout():
    p = Promise()
    with pytest.raises(TimeoutError):
        p.token.get(timeout=0.01)
    p.set_value(1)


def test_racing_fulfillers():
    for _ in range(200):
        p = Promise()
        winners = []
        barrier = threading.Barrier(8)

        def go(k):
            barrier.wait()
            if p.try_set_value(k):
                winners.append(k)

        ts = [threading.Thread(target=go, args=(k,)) for k in range(8)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert len(winners) == 1 and p.token.get() == winners[0]


def test_random_then_chains():
    rng = random.Random(7)
    for _ in range(20_000):
        depth = rng.randint(1, 6)
        fail_at = rng.randint(0, depth) if rng.random() < 0.4 else None
        p = Promise()
        tok = p.token
        calls = []
        for level in range(depth):
            def step(x, level=level):
                calls.append(level)
                if fail_at == level + 1:
                    raise Boom(level + 1)
                return x + 1
            tok = tok.then(step)
        if fail_at == 0:
            p.set_error(Boom(0))
        else:
            p.set_value(0)
        if fail_at is None:
            assert tok.get() == depth and calls == list(range(depth))
        else:
            with pytest.raises(Boom):
                tok.get()
            assert calls == list(range(fail_at))


def test_deep_when_all_chain_polled_and_armed():
    n = 50_000
    prev = make_ready(None)
    ps = []
    for _ in range(n):
        p = Promise()
        ps.append(p)
        prev = when_all([prev, p.token])
    armed = prev.then(lambda _: "fired")
    for p in ps[:-1]:
        p.set_value(None)
    assert not prev.done()
    ps[-1].set_value(None)
    assert prev.done() and armed.get() == "fired"


def test_deep_when_all_chain_error():
    prev = make_ready(None)
    ps = []
    for _ in range(10_000):
        p = Promise()
        ps.append(p)
        prev = when_all([prev, p.token])
    ps[5000].set_error(Boom("mid"))
    with pytest.raises(Boom):
        prev.get()
    for i, p in enumerate(ps):
        if i != 5000:
            p.set_value(None)


def test_gid_uniqueness_million():
    from paper_1810_11482_b200.registry import ObjectKind, Registry

    reg = Registry()
    gids = {reg.register(ObjectKind.BUFFER, i) for i in range(1_000_000)}
    assert len(gids) == 1_000_000
    g = next(iter(gids))
    assert reg.resolve_local(g, ObjectKind.BUFFER) is not None
    reg.unregister(g)
    import pytest as _p

    from paper_1810_11482_b200.errors import UnknownGidError

    with _p.raises(UnknownGidError):
        reg.resolve_local(g)
