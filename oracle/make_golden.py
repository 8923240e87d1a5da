"""Generate tests/golden/*.npz from the REFERENCE library itself (TEST INFRASTRUCTURE).

Runs oracle/_ref/libmoesim_ref.so -- moesim compiled from /root/reference
sources by oracle/Makefile -- and records inputs and outputs of the path's
functions.  These fixtures pin oracle/ (the C restatement) and the GPU path
on machines where /root/reference is absent (the GPU box).

    python oracle/make_golden.py      # rewrites tests/golden/
"""
from __future__ import annotations

import os
import sys

import ctypes as C

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle import Oracle, RefLib, Workload  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    ref = RefLib()
    orc = Oracle()  # only its generators are used here (pinned below against ref)

    # ---- distances: hand examples (test_eam.cpp:170-225) + random pairs
    pairs_a, pairs_b, dists, shapes = [], [], [], []
    hand = [
        ((2, 2), [[1, 0], [0, 1]], [[1, 0], [1, 0]]),
        ((1, 2), [[1, 0]], [[2, 0]]),
        ((1, 2), [[1, 0]], [[1, 0]]),
        ((2, 2), [[0, 0], [0, 0]], [[0, 0], [0, 0]]),
        ((2, 2), [[1, 0], [0, 0]], [[0, 0], [0, 0]]),
    ]
    for (L, E), a, b in hand:
        a = np.array(a, np.uint64)
        b = np.array(b, np.uint64)
        shapes.append((L, E))
        pairs_a.append(a.ravel())
        pairs_b.append(b.ravel())
        dists.append(ref.distance(a, b))
    rng = orc.rng(17)
    for _ in range(300):
        a = orc.random_eam(rng, 3, 5)
        b = orc.random_eam(rng, 3, 5)
        shapes.append((3, 5))
        pairs_a.append(a.ravel())
        pairs_b.append(b.ravel())
        dists.append(ref.distance(a, b))
    for L, E, seed in [(12, 128, 55), (32, 8, 7), (59, 160, 9), (24, 128, 3)]:
        fam = orc.bench_family(seed, L, E, 40)
        for i in range(20):
            shapes.append((L, E))
            pairs_a.append(fam[2 * i].ravel())
            pairs_b.append(fam[2 * i + 1].ravel())
            dists.append(ref.distance(fam[2 * i], fam[2 * i + 1]))
    flat_a = np.concatenate(pairs_a)
    flat_b = np.concatenate(pairs_b)
    np.savez_compressed(os.path.join(OUT, "distance.npz"), shapes=np.array(shapes, np.uint32),
                        a=flat_a, b=flat_b, d=np.array(dists, np.float64))

    # ---- bench_match checksums (bench.cpp:58-88) and full match results
    cks = []
    for P, L, E, Q, seed in [(300, 32, 8, 200, 55), (1000, 12, 128, 50, 55),
                             (200, 12, 128, 20, 0), (64, 59, 160, 8, 1)]:
        ck, _, _ = ref.bench_match(P, L, E, Q, seed)
        cks.append((P, L, E, Q, seed, ck))
    np.savez_compressed(os.path.join(OUT, "bench_checksum.npz"), rows=np.array(cks, np.uint64))

    # match / match_within on the bench family with the reference Eamc
    P, L, E, Q, seed = 300, 32, 8, 64, 55
    fam = orc.bench_family(seed, L, E, P + Q)
    e = ref.eamc(L, E, 1, 1, P)
    for i in range(P):
        e.insert(fam[i])
    idx, seq, d, f = e.match(fam[P:])
    wi, ws, wd, wn = [], [], [], []
    for q in range(8):
        a, b, c = e.match_within(fam[P + q], 0.01)
        wi.append(a)
        ws.append(b)
        wd.append(c)
        wn.append(len(a))
    np.savez_compressed(os.path.join(OUT, "match_mix.npz"), params=np.array([P, L, E, Q, seed]),
                        idx=idx, seq=seq, d=d, w_n=np.array(wn), w_idx=np.concatenate(wi),
                        w_seq=np.concatenate(ws), w_d=np.concatenate(wd))

    # ---- construction replay (acceptance_main.cpp:192-229: 2x4, capacity 10,
    # 500 random_eam inserts, seed 103) + the documented example
    rng = orc.rng(103)
    eams = np.stack([orc.random_eam(rng, 2, 4) for _ in range(500)])
    e = ref.eamc(2, 4, 1, 1, 10)
    slots = np.array([e.insert(x) for x in eams], np.int64)
    ent, sq = e.entries()
    ex = np.array([[[10, 0, 0, 0]], [[0, 10, 0, 0]], [[0, 0, 10, 0]], [[0, 0, 9, 1]]], np.uint64)
    e2 = ref.eamc(1, 4, 1, 1, 3)
    ex_slots = np.array([e2.insert(x) for x in ex], np.int64)
    np.savez_compressed(os.path.join(OUT, "insert_replay.npz"), eams=eams, slots=slots,
                        entries=ent, seqs=sq, ex=ex, ex_slots=ex_slots)

    # ---- prefetch priorities (policy.cpp:88-126 + engine.cpp:663-668)
    pf = {}
    s = (4, 2)
    e = ref.eamc(4, 2, 1, 1, 4)
    e.insert(np.array([[1, 0], [1, 0], [2, 1], [0, 3]], np.uint64))
    cur = np.array([[1, 0], [1, 0], [0, 0], [0, 0]], np.uint64)
    l_, e_, p_ = e.prefetch(cur, 1, False)
    pf["worked_l"], pf["worked_e"], pf["worked_p"] = l_, e_, p_
    # F2 workload, Mixtral-ish shape, iteration probes
    w = Workload(32, 8, 2, n_groups=24)
    ents = orc.request_eams(w, 60, phase=1)
    e = ref.eamc(32, 8, 2, 1, 60)
    for x in ents:
        e.insert(x)
    probes, layers, outs_l, outs_e, outs_p, outs_n, filt = [], [], [], [], [], [], []
    for r in range(6):
        for it, layer in [(1, 0), (2, 5), (3, 17), (4, 30), (5, 31)]:
            pr = orc.iteration_probe(w, 1000 + r, it, layer)
            for flt in (True, False):
                l_, e_, p_ = e.prefetch(pr, layer, flt)
                probes.append(pr)
                layers.append(layer)
                filt.append(flt)
                outs_l.append(l_)
                outs_e.append(e_)
                outs_p.append(p_)
                outs_n.append(len(l_))
    pf["f2_entries"] = ents
    pf["f2_probes"] = np.stack(probes)
    pf["f2_layers"] = np.array(layers, np.uint32)
    pf["f2_filter"] = np.array(filt, np.uint8)
    pf["f2_n"] = np.array(outs_n)
    pf["f2_l"] = np.concatenate(outs_l)
    pf["f2_e"] = np.concatenate(outs_e)
    pf["f2_p"] = np.concatenate(outs_p)
    np.savez_compressed(os.path.join(OUT, "prefetch.npz"), **pf)

    # ---- cache priority + victim selection (test_policy.cpp:164-193, 330-377)
    reqs, views, victims = [], [], []
    r = orc.rng(0)
    for trial in range(200):
        req = np.zeros((4, 8), np.uint64)
        lib = orc.lib
        for l in range(4):
            for x in range(8):
                if lib.orc_rng_bernoulli(C.byref(r), 0.6):
                    req[l, x] = lib.orc_rng_bounded(C.byref(r), 20)
        used = set()
        slot, lay, exp, prot, pin = [], [], [], [], []
        for s_ in range(8):
            while True:
                ident = (int(lib.orc_rng_bounded(C.byref(r), 4)), int(lib.orc_rng_bounded(C.byref(r), 8)))
                if ident not in used:
                    used.add(ident)
                    break
            slot.append(s_)
            lay.append(ident[0])
            exp.append(ident[1])
            prot.append(int(lib.orc_rng_bernoulli(C.byref(r), 0.2)))
            pin.append(int(lib.orc_rng_bernoulli(C.byref(r), 0.2)))
        reqs.append(req)
        views.append(np.array([slot, lay, exp, prot, pin], np.uint64))
        victims.append(ref.select_victim(req, slot, lay, exp, prot, pin))
    cp_req = np.array([[1, 3], [0, 0], [2, 2]], np.uint64)
    cp = [ref.cache_priority(cp_req, 0, 1), ref.cache_priority(cp_req, 1, 0),
          ref.cache_priority(cp_req, 2, 1)]
    np.savez_compressed(os.path.join(OUT, "eviction.npz"), reqs=np.stack(reqs),
                        views=np.stack(views), victims=np.array(victims, np.int64),
                        cp_req=cp_req, cp=np.array(cp))

    # ---- generated traces (workload.cpp) -> per-iteration counts, pins the
    # oracle's F2/F3 generator; capacity bounds (test_eam.cpp:344-349)
    tr = {}
    for name, w in [("sw", Workload(12, 64, 1, seed=1001)), ("mix", Workload(32, 8, 2, seed=99)),
                    ("ds", Workload(59, 160, 6, n_groups=8, prompt_len=6, decode_len=3,
                                    batch_size=2, seed=5))]:
        tr[name] = np.stack([ref.trace_counts(w, i) for i in range(3)])
    tr["cap"] = np.array([ref.capacity_bound(12, 128, 0.75), ref.capacity_bound(12, 128, 0.98),
                          ref.capacity_bound(1, 1, 0.75), ref.capacity_bound(2, 2, 0.9)], np.uint64)
    np.savez_compressed(os.path.join(OUT, "traces.npz"), **tr)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
