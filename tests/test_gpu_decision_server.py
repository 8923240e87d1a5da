"""The persistent decision server (moe_eamc_set_decision_server): the same
prefetch orders as the oracle (policy.cpp:88-126 + engine.cpp:663-668),
bitwise, through the mailbox path -- across collection updates between
decisions (the resident kernel must not read stale collection data), a
storage-width change (relaunch at the new width), idle exits and relaunches,
switching it off, and destroying a handle whose server is resident."""
import ctypes as C
import time

import numpy as np
import pytest

from oracle import Workload

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


def _server(m, e, n):
    from paper_2401_14361_b200 import _lib
    _lib.check(_lib.lib.moe_eamc_set_decision_server(e._h, n))


def _check(m, orc, e, ents, seqs, probe, layer, s):
    order = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=probe), e, layer, True)
    ol, oe, op = orc.prefetch(ents, seqs, probe, layer, True)
    assert np.array_equal(order["layer_idx"], ol)
    assert np.array_equal(order["expert_idx"], oe)
    assert np.array_equal(order["priority"], op)


@pytest.mark.parametrize("L,E,k,P,ctas", [(59, 160, 6, 2000, 64), (32, 8, 2, 300, 16),
                                          (24, 128, 2, 1000, 32)])
def test_server_orders_vs_oracle(m, orc, L, E, k, P, ctas):
    w = Workload(L, E, k, seed=3)
    ents = orc.request_eams(w, P)
    s = m.ModelShape(L, E, k)
    e = m.Eamc(s, m.Phase.decode, P + 50)
    e.append(ents, np.arange(P, dtype=np.uint64))
    _server(m, e, ctas)
    seqs = np.arange(P, dtype=np.uint64)
    base = orc.iteration_probe(w, 4000, 2, L - 1)
    for layer in range(L - 1):  # the engine's call sequence: the probe grows by a row
        pr = base.copy()
        pr[layer + 1:] = 0
        _check(m, orc, e, ents, seqs, pr, layer, s)
    # the collection changes between decisions: appended entries are seen
    more = orc.request_eams(w, 50, start=9000)
    e.append(more, np.arange(P, P + 50, dtype=np.uint64))
    ents2 = np.concatenate([ents, more])
    seqs2 = np.arange(P + 50, dtype=np.uint64)
    for layer in (0, L // 2, L - 2):
        pr = base.copy()
        pr[layer + 1:] = 0
        _check(m, orc, e, ents2, seqs2, pr, layer, s)
    _server(m, e, 0)  # off: the launch path again
    _check(m, orc, e, ents2, seqs2, base, L // 3, s)


def test_server_width_change_idle_and_destroy(m, orc):
    L, E, k, P = 12, 64, 2, 400
    w = Workload(L, E, k, seed=8)
    ents = orc.request_eams(w, P)
    s = m.ModelShape(L, E, k)
    e = m.Eamc(s, m.Phase.decode, P + 1)
    e.append(ents, np.arange(P, dtype=np.uint64))
    _server(m, e, 24)
    seqs = np.arange(P, dtype=np.uint64)
    probe = orc.iteration_probe(w, 77, 2, 5)
    _check(m, orc, e, ents, seqs, probe, 5, s)
    time.sleep(0.2)  # the server idles out (50 ms) and is relaunched on demand
    _check(m, orc, e, ents, seqs, probe, 3, s)
    # an entry with counts > 255 widens the collection: the server relaunches at u16
    big = (ents[7] * 300).astype(np.uint64)
    e.append(big[None], np.array([P], np.uint64))
    assert e.count_bytes() == 2
    ents2 = np.concatenate([ents, big[None]])
    _check(m, orc, e, ents2, np.arange(P + 1, dtype=np.uint64), probe * 100, 5, s)
    for _ in range(50):  # back-to-back requests
        _check(m, orc, e, ents2, np.arange(P + 1, dtype=np.uint64), probe, 6, s)
    del e  # destroyed with its server resident: stops it
    e3 = m.Eamc(s, m.Phase.decode, P)  # decisions on another handle still co-reside
    e3.append(ents, seqs)
    _check(m, orc, e3, ents, seqs, probe, 4, s)


def test_small_server_switches_kinds(m, orc):
    """A small collection is served by the one-CTA server (the k_decision_small
    phases); when it grows past the small path's bound the multi-CTA server
    takes over, and back -- orders bitwise equal to the oracle throughout,
    including collection updates seen by the resident kernel."""
    L, E, k = 32, 8, 2
    w = Workload(L, E, k, seed=23)
    ents = orc.request_eams(w, 900)
    s = m.ModelShape(L, E, k)
    e = m.Eamc(s, m.Phase.decode, 900)
    e.append(ents[:300], np.arange(300, dtype=np.uint64))
    _server(m, e, 8)
    base = orc.iteration_probe(w, 777, 2, L - 1)
    for P in (300, 400, 900, 900):
        if P > e.size():
            e.append(ents[e.size():P], np.arange(e.size(), P, dtype=np.uint64))
        seqs = np.arange(P, dtype=np.uint64)
        for layer in (0, 3, L // 2, L - 2):
            pr = base.copy()
            pr[layer + 1:] = 0
            _check(m, orc, e, ents[:P], seqs, pr, layer, s)
    small = m.Eamc(s, m.Phase.decode, 300)
    small.append(ents[:300], np.arange(300, dtype=np.uint64))
    _server(m, small, 8)
    for j in range(40):  # unrelated probes, every layer: no prefix reuse
        pr = orc.iteration_probe(w, 5000 + j, 2, j % (L - 1))
        _check(m, orc, small, ents[:300], np.arange(300, dtype=np.uint64), pr, j % (L - 1), s)
    # entries replaced in place (at-capacity inserts) while the server is
    # resident and has read them: the next decisions see the new contents
    small.build(ents[300:420])
    want_ent, want_seqs, _ = orc.insert_replay(L, E, 300, ents[:420])
    for j in range(12):
        pr = orc.iteration_probe(w, 6000 + j, 2, j % (L - 1))
        _check(m, orc, small, want_ent, want_seqs, pr, j % (L - 1), s)
    _server(m, small, 0)
    _server(m, e, 0)


@pytest.mark.timeout(300)
def test_concurrent_decisions_two_handles(m, orc):
    """Two handles deciding at once from two host threads (two streams): the
    software-grid-barrier kernels must stay co-resident (two CTAs per SM by
    their shared-memory bound), including the wide-window path (layer 0: listed
    members, staged ranking).  Results equal the sequential ones."""
    import threading
    L, E, k, P = 59, 160, 6, 2000
    w = Workload(L, E, k, seed=13)
    hs, probes = [], []
    for i in range(2):
        ents = orc.request_eams(w, P, start=5000 * i)
        e = m.Eamc(m.ModelShape(L, E, k), m.Phase.decode, P)
        e.append(ents, np.arange(P, dtype=np.uint64))
        hs.append(e)
        probes.append([orc.iteration_probe(w, 700 + 10 * i + j, 2, j % (L - 1)) for j in range(24)])
    s = m.ModelShape(L, E, k)

    def run(i, res):
        for j, pr in enumerate(probes[i]):
            cur = m.Eam(s, m.EamKind.iteration, counts=pr)
            res.append(m.prefetch_order(cur, hs[i], j % (L - 1), True))

    want = [[], []]
    for i in range(2):
        run(i, want[i])
    for _ in range(3):
        got = [[], []]
        ts = [threading.Thread(target=run, args=(i, got[i])) for i in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join(timeout=120)
            assert not t.is_alive(), "concurrent decisions did not finish"
        for i in range(2):
            for a, b in zip(got[i], want[i]):
                assert np.array_equal(a, b)
