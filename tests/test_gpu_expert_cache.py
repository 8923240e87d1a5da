"""Real expert-weight prefetch (moe_expert_cache_*): the
engine's transfer rules over chunked cudaMemcpyAsync.  The slot decisions are
compared with a restatement of engine.cpp's dispatch (try_start_for_gpu,
engine.cpp:306-357; acquire_slot / contention, :429-455; force_slot_for_on_demand,
:462-505) priced by the ORACLE's cache_priority / select_eviction_victim, with
every transfer completed before the next decision (progress(wait_idle)); the
bytes in every resident slot must be that expert's weights."""
import math

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]
INF = math.inf


class EngineModel:
    """engine.cpp's single-GPU dispatch with instantaneous transfers."""

    def __init__(self, orc, L, E, n_slots, req):
        self.orc, self.L, self.E, self.req = orc, L, E, req
        self.slots = [dict(occ=-1, res=0, prot=False, exec=False) for _ in range(n_slots)]
        self.queue = {}

    def cpri(self, fid):
        return self.orc.cache_priority(self.req, fid // self.E, fid % self.E)

    def ordered(self):
        return sorted(self.queue.items(), key=lambda kv: (-kv[1], kv[0]))

    def index(self, fid):
        for i, s in enumerate(self.slots):
            if s["occ"] == fid:
                return i
        return None

    def victim(self):
        res = [(i, s) for i, s in enumerate(self.slots) if s["res"] == 2]
        if not res:
            return None
        v = self.orc.select_victim(self.req, [i for i, _ in res],
                                   [s["occ"] // self.E for _, s in res],
                                   [s["occ"] % self.E for _, s in res],
                                   [int(s["prot"]) for _, s in res],
                                   [int(s["exec"]) for _, s in res])
        return None if v < 0 else v

    def acquire(self, pri):
        for i, s in enumerate(self.slots):
            if s["res"] == 0:
                return i
        v = self.victim()
        if v is not None:
            if pri != INF and self.cpri(self.slots[v]["occ"]) >= pri:
                return None
            self.slots[v] = dict(occ=-1, res=0, prot=False, exec=False)
            return v
        if pri != INF:
            return None
        best = None
        for i, s in enumerate(self.slots):
            if s["occ"] < 0 or s["exec"] or not s["prot"]:
                continue
            p = self.cpri(s["occ"])
            if best is None or p < best[1]:
                best = (i, p)
        assert best is not None
        self.slots[best[0]] = dict(occ=-1, res=0, prot=False, exec=False)
        return best[0]

    def run(self):
        while True:
            started = False
            restart = True
            while restart:
                restart = False
                for fid, pri in self.ordered():
                    if self.index(fid) is not None:
                        del self.queue[fid]
                        restart = True
                        break
                    slot = self.acquire(pri)
                    if slot is None:
                        if pri == INF:
                            continue
                        break
                    self.slots[slot] = dict(occ=fid, res=2, prot=True, exec=False)
                    del self.queue[fid]
                    started = True
                    break
            if not started:
                return

    def submit(self, order):
        self.queue = {int(o["layer_idx"]) * self.E + int(o["expert_idx"]): float(o["priority"])
                      for o in order}
        self.run()


def _order(m, items):
    from paper_2401_14361_b200._lib import CAND_DTYPE
    a = np.zeros(len(items), CAND_DTYPE)
    for i, (l, e, p) in enumerate(items):
        a[i] = (l, e, p)
    return a


def _state(cache):
    out = []
    for i in range(cache.n_slots):
        s = cache.slot(i)
        fid = -1 if s["expert"] is None else (s["expert"].layer_idx * cache.shape.n_experts_per_layer
                                               + s["expert"].expert_idx)
        out.append((fid, s["residency"], s["protected"]))
    return out


def _model_state(md):
    return [(s["occ"], s["res"], s["prot"]) for s in md.slots]


def _check_bytes(cache, w):
    E = cache.shape.n_experts_per_layer
    for i in range(cache.n_slots):
        s = cache.slot(i)
        if s["residency"] == 2:
            ex = s["expert"]
            assert np.array_equal(cache.read_slot(i), w[ex.layer_idx, ex.expert_idx]), (i, ex)


def test_prefetch_order_contention_on_demand(m, orc):
    L, E, nb, n_slots = 4, 8, 64 << 10, 5
    rng = np.random.default_rng(1)
    w = rng.integers(0, 256, size=(L, E, nb), dtype=np.uint8)
    req = rng.integers(0, 9, size=(L, E)).astype(np.uint64)
    s = m.ModelShape(L, E, 2)
    cache = m.ExpertCache(s, w, n_slots, chunk_bytes=16 << 10)
    cache.set_request_eam(m.Eam(s, counts=req))
    md = EngineModel(orc, L, E, n_slots, req)
    # 1) fill from an order (7 candidates, 5 slots: the first five land)
    order = _order(m, [(1, 3, 0.9), (1, 5, 0.8), (2, 0, 0.7), (2, 6, 0.6), (3, 1, 0.5),
                       (3, 2, 0.4), (3, 7, 0.3)])
    cache.submit(order)
    cache.progress(wait_idle=True)
    md.submit(order)
    assert _state(cache) == _model_state(md)
    _check_bytes(cache, w)
    # 2) executions clear protection and reprice (policy.cpp:161-167)
    for (l, e) in [(1, 3), (2, 0), (3, 1)]:
        ptr, hit = cache.acquire(m.ExpertId(l, e))
        assert hit and ptr
        cache.release(m.ExpertId(l, e))
        i = md.index(l * E + e)
        md.slots[i]["prot"] = False
        sl = cache.slot(i)
        if sl["expert"] == m.ExpertId(l, e):
            assert not sl["protected"] and sl["priority"] == orc.cache_priority(req, l, e)
        # the released slot is now an eviction candidate: queued prefetches may
        # take it (the engine's dispatch runs after every event)
        cache.progress(wait_idle=True)
        md.run()
        assert _state(cache) == _model_state(md)
    # 3) a new order: contention decides which victims a prefetch displaces
    order2 = _order(m, [(0, 4, 5.0), (0, 5, 1e-5), (1, 1, 0.05)])
    cache.submit(order2)
    cache.progress(wait_idle=True)
    md.submit(order2)
    assert _state(cache) == _model_state(md)
    _check_bytes(cache, w)
    # 4) on-demand fetch of a non-resident expert (kMaxPriority) always lands
    ptr, hit = cache.acquire(m.ExpertId(3, 6))
    assert not hit and ptr
    md.queue[3 * E + 6] = INF
    md.run()
    md.slots[md.index(3 * E + 6)]["exec"] = True
    assert _state(cache) == _model_state(md)
    _check_bytes(cache, w)
    cache.release(m.ExpertId(3, 6))
    cache.progress(wait_idle=True)
    st = cache.stats()
    assert st["misses"] == 1 and st["hits"] == 3 and st["in_flight"] == 0
    assert st["transfers_started"] == st["transfers_completed"] + st["transfers_cancelled"]
    assert st["bytes_moved"] == st["transfers_completed"] * nb


def test_on_demand_preempts_a_speculative_transfer(m, orc):
    """A 256 MB speculative transfer in 4 MB chunks is cut at a chunk boundary
    by an on-demand fetch, which lands first; the preempted expert is requeued
    at its old priority and lands afterwards."""
    L, E, nb = 2, 4, 256 << 20
    w = np.zeros((L, E, nb), np.uint8)
    for l in range(L):
        for e in range(E):
            w[l, e, ::4096] = 16 * l + e + 1
    s = m.ModelShape(L, E, 1)
    cache = m.ExpertCache(s, w, 3, chunk_bytes=4 << 20)
    cache.set_request_eam(m.Eam(s, counts=np.ones((L, E), np.uint64)))
    cache.submit(_order(m, [(1, 2, 0.7)]))
    ptr, hit = cache.acquire(m.ExpertId(0, 1))  # on demand while (1, 2) is in flight
    assert not hit
    st = cache.stats()
    assert st["preemptions"] == 1 and st["transfers_cancelled"] == 1
    cache.release(m.ExpertId(0, 1))
    cache.progress(wait_idle=True)
    occ = {cache.slot(i)["expert"] for i in range(3)}
    assert m.ExpertId(0, 1) in occ and m.ExpertId(1, 2) in occ
    _check_bytes(cache, w)


def test_decode_loop_with_the_gpu_prefetch_order(m, orc):
    """The engine's per-layer loop on real weights: prefetch order from the GPU
    decision path -> submit -> routed experts acquired (hit or on-demand miss)
    -> released; every acquired slot holds the right bytes."""
    from oracle import Workload
    L, E, k, P = 8, 16, 2, 60
    wl = Workload(L, E, k, seed=4)
    ents = orc.request_eams(wl, P)
    s = m.ModelShape(L, E, k)
    eamc = m.Eamc(s, m.Phase.decode, P)
    eamc.build(ents)
    rng = np.random.default_rng(2)
    w = rng.integers(0, 256, size=(L, E, 32 << 10), dtype=np.uint8)
    cache = m.ExpertCache(s, w, 12, chunk_bytes=8 << 10)
    req = orc.request_eams(wl, 1, start=500)[0]
    cache.set_request_eam(m.Eam(s, counts=req))
    probe = orc.iteration_probe(wl, 501, 1, L - 1)
    for layer in range(L):
        cur = probe.copy()
        cur[layer + 1:] = 0
        order = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=cur), eamc, layer, True)
        cache.submit(order)
        for e in np.nonzero(probe[layer])[0][:k]:
            ex = m.ExpertId(layer, int(e))
            ptr, hit = cache.acquire(ex)
            i = [j for j in range(cache.n_slots) if cache.slot(j)["expert"] == ex][0]
            assert np.array_equal(cache.read_slot(i), w[layer, e])
            cache.release(ex)
        cache.progress()
    st = cache.stats()
    assert st["hits"] + st["misses"] > 0 and st["hits"] > 0, st
