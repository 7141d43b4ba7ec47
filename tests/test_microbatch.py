"""Thread-safe micro-batch manager (C-ABI hp_mbm_*):
groups become ready exactly when all their prefill micro-batches are done
(make_schedule group membership, pipesim.cpp:22-46), decode tokens are
enqueued in order, duplicate reports are ignored, out-of-order decode
reports are rejected, and concurrent reporters (ctypes drops the GIL, so
the threads really race inside the C++ lock) never lose or duplicate an
enqueue. CPU only."""
import ctypes as C
import random
import threading

import pytest

from paper_2403_01136_b200 import capi


class M:
    def __init__(self, B, eta, xi, n):
        h = C.c_void_p()
        capi.check(capi.lib.hp_mbm_create(B, eta, xi, n, C.byref(h)))
        self.h = h

    def prefill_done(self, k):
        g = C.c_int()
        capi.check(capi.lib.hp_mbm_prefill_done(self.h, k, C.byref(g)))
        return g.value

    def decode_done(self, g, t):
        f = C.c_int()
        capi.check(capi.lib.hp_mbm_decode_done(self.h, g, t, C.byref(f)))
        return bool(f.value)

    def next(self):
        g, t = C.c_int(), C.c_int()
        return (g.value, t.value) if capi.lib.hp_mbm_next(self.h, C.byref(g), C.byref(t)) else None

    def __del__(self):
        capi.lib.hp_mbm_destroy(self.h)


def _groups(B, eta, xi):
    sizes, groups, ng = [], [], None
    buf = (C.c_int * B)()
    gb = (C.c_int * B)()
    nb, ngr = C.c_int(), C.c_int()
    capi.check(capi.lib.hp_host_make_schedule(B, eta, xi, buf, gb, C.byref(nb), C.byref(ngr), B))
    return list(gb[:nb.value]), ngr.value


@pytest.mark.parametrize("B,eta,xi", [(8, 2, 4), (8, 3, 6), (5, 2, 5), (32, 4, 32), (33, 4, 8)])
def test_groups_ready_exactly_when_their_prefill_is_done(B, eta, xi):
    gop, ng = _groups(B, eta, xi)
    m = M(B, eta, xi, 4)
    order = list(range(len(gop)))
    random.Random(B * eta + xi).shuffle(order)
    left = {g: gop.count(g) for g in range(ng)}
    for k in order:
        got = m.prefill_done(k)
        left[gop[k]] -= 1
        assert got == (gop[k] if left[gop[k]] == 0 else -1)
        assert m.prefill_done(k) == -1  # duplicate report: no effect
    ready = []
    while (it := m.next()) is not None:
        ready.append(it)
    assert sorted(ready) == [(g, 1) for g in range(ng)]


def test_decode_tokens_in_order_and_rejections():
    m = M(8, 2, 4, 4)
    with pytest.raises(capi.InvalidArgument):
        m.decode_done(0, 1)  # prefill of group 0 not done
    for k in (0, 1):
        m.prefill_done(k)
    assert m.next() == (0, 1)
    assert not m.decode_done(0, 1)
    assert m.next() == (0, 2)
    with pytest.raises(capi.InvalidArgument):
        m.decode_done(0, 3)  # token 2 not reported yet
    assert not m.decode_done(0, 2)
    assert m.next() == (0, 3)
    assert m.decode_done(0, 3)  # n - 1 = 3: finished
    assert m.next() is None
    with pytest.raises(capi.InvalidArgument):
        m.prefill_done(99)


def test_concurrent_reporters_lose_nothing():
    B, eta, xi, n = 256, 2, 32, 6
    gop, ng = _groups(B, eta, xi)
    m = M(B, eta, xi, n)
    ks = list(range(len(gop)))
    random.Random(5).shuffle(ks)
    ready, lock = [], threading.Lock()

    def worker(part):
        for k in part:
            for _ in range(3):  # duplicates from several reporters
                g = m.prefill_done(k)
                if g >= 0:
                    with lock:
                        ready.append(g)

    th = [threading.Thread(target=worker, args=(ks[i::8],)) for i in range(8)]
    th += [threading.Thread(target=worker, args=(ks[::-1][i::8],)) for i in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert sorted(ready) == list(range(ng))  # every group exactly once
    # drain the decode phase from several consumer threads
    done = []

    def consumer():
        while True:
            it = m.next()
            if it is None:
                with lock:
                    if len(done) == ng * (n - 1):
                        return
                continue
            m.decode_done(*it)
            with lock:
                done.append(it)

    cs = [threading.Thread(target=consumer) for _ in range(4)]
    for t in cs:
        t.start()
    for t in cs:
        t.join(timeout=30)
    assert sorted(done) == sorted((g, t) for g in range(ng) for t in range(1, n))
