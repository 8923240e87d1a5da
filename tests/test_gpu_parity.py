"""GPU parity: libmoe_eamc (sm_100a kernels, through its C ABI) vs the oracle.

Bar (BASELINE.json north_star): bit-exact counts, match indices / seqs,
distances, window sets, prefetch order and victims.  Distances are compared
BITWISE (stricter than the 1e-5 relative the north star allows), because
the device path reproduces the reference's fp64 operation order on exact
integer sums ("exactness contract").
"""
import numpy as np
import pytest

from oracle import Workload

pytestmark = pytest.mark.gpu


def seqs_of(n):
    return np.arange(n, dtype=np.uint64)


def filled(m, L, E, entries, capacity=None, top_k=1, count_bytes=0):
    e = m.Eamc(m.ModelShape(L, E, top_k), m.Phase.decode, capacity or max(len(entries), 1),
               count_bytes=count_bytes)
    if len(entries):
        slots = e.build(entries)
        assert (slots == -1).all()
    return e


def check_match(m, orc, e, entries, seqs, probes):
    got = e.match_batch(probes)
    idx, seq, d, found = orc.match(entries, seqs, probes)
    assert found.all()
    assert np.array_equal(got["index"], idx), np.nonzero(got["index"] != idx)
    assert np.array_equal(got["seq"], seq)
    assert np.array_equal(got["distance"], d)  # bitwise
    return got


# ---------------------------------------------------------------- distance
def test_distance_golden(m, golden):
    g = golden("distance.npz")
    oa = 0
    for i, (L, E) in enumerate(g["shapes"]):
        n = int(L) * int(E)
        s = m.ModelShape(int(L), int(E))
        a = m.Eam(s, counts=g["a"][oa:oa + n])
        b = m.Eam(s, counts=g["b"][oa:oa + n])
        oa += n
        assert m.eam_distance(a, b) == g["d"][i]
    with pytest.raises(ValueError):
        m.eam_distance(m.Eam(m.ModelShape(1, 2)), m.Eam(m.ModelShape(2, 2)))


# ------------------------------------------------------------------- match
def test_empty_collection_matches_nothing(m):
    e = m.Eamc(m.ModelShape(2, 4), m.Phase.decode, 200)
    assert e.match(m.Eam(m.ModelShape(2, 4), counts=np.ones((2, 4)))) is None
    assert e.match_within(m.Eam(m.ModelShape(2, 4)), 0.01) == []
    with pytest.raises(ValueError):
        e.match(m.Eam(m.ModelShape(3, 4)))


def test_bench_checksums_golden(m, golden):
    for P, L, E, Q, seed, ck in golden("bench_checksum.npz")["rows"]:
        P, L, E, Q, seed = int(P), int(L), int(E), int(Q), int(seed)
        fam = m.gen_bench_family(seed, L, E, P + Q)
        e = filled(m, L, E, fam[:P])
        got = e.match_batch(fam[P:])
        assert int((got["index"] + 1).sum()) == int(ck)


def test_match_golden_mix(m, golden):
    g = golden("match_mix.npz")
    P, L, E, Q, seed = (int(x) for x in g["params"])
    fam = m.gen_bench_family(seed, L, E, P + Q)
    e = filled(m, L, E, fam[:P])
    got = e.match_batch(fam[P:])
    assert np.array_equal(got["index"], g["idx"]) and np.array_equal(got["seq"], g["seq"])
    assert np.array_equal(got["distance"], g["d"])
    o = 0
    for q in range(len(g["w_n"])):
        n = int(g["w_n"][q])
        w = e.match_within(m.Eam(m.ModelShape(L, E), counts=fam[P + q]), 0.01)
        assert [x.index for x in w] == list(g["w_idx"][o:o + n])
        assert [x.seq for x in w] == list(g["w_seq"][o:o + n])
        assert [x.distance for x in w] == list(g["w_d"][o:o + n])
        o += n


@pytest.mark.parametrize("L,E,P,Q,seed", [
    (12, 128, 2000, 96, 55),    # Switch shape (SW), streaming + batch tiles
    (32, 8, 300, 200, 7),       # Mixtral shape (MIX)
    (59, 160, 300, 12, 9),      # DeepSeek-V2 shape (DS)
    (24, 128, 500, 20, 3),      # NLLB shape (NL)
    (3, 5, 77, 33, 1),          # odd tiny shape
    (1, 1, 10, 5, 2),
])
def test_match_bench_family(m, orc, L, E, P, Q, seed):
    fam = m.gen_bench_family(seed, L, E, P + Q)
    e = filled(m, L, E, fam[:P])
    check_match(m, orc, e, fam[:P], seqs_of(P), fam[P:])


@pytest.mark.parametrize("Q", [1, 2, 3, 4, 7, 8, 9, 64, 65, 130])
def test_match_probe_batch_sizes(m, orc, Q):
    L, E, P = 12, 128, 700
    fam = m.gen_bench_family(11, L, E, P + Q)
    e = filled(m, L, E, fam[:P])
    check_match(m, orc, e, fam[:P], seqs_of(P), fam[P:])


def test_match_random_eam_family(m, orc):
    """random_eam family (test_eam.cpp:58-66): dense Bernoulli(0.4) rows."""
    rng = orc.rng(23)
    ents = np.stack([orc.random_eam(rng, 2, 4) for _ in range(100)])
    probes = np.stack([orc.random_eam(rng, 2, 4) for _ in range(20)])
    e = filled(m, 2, 4, ents, capacity=200)
    check_match(m, orc, e, ents, seqs_of(100), probes)
    # a contained entry matches itself at distance 0 (test_eam.cpp:257-261)
    r = e.match(m.Eam(m.ModelShape(2, 4), counts=ents[42]))
    assert r.distance == orc.distance(ents[42], ents[42]) < 1e-15
    first = min(i for i in range(100) if np.array_equal(ents[i], ents[42]))
    assert r.index == first


def test_match_ties_and_duplicates(m, orc):
    """Many exact ties: the oldest seq must win (eam.cpp:123-124); exceeds the
    candidate bucket and exercises the exact fallback pass."""
    L, E = 12, 128
    base = m.gen_bench_family(5, L, E, 40)
    ents = np.concatenate([np.repeat(base[:3], 150, axis=0), base[3:30]])
    rng = np.random.default_rng(0)
    perm = rng.permutation(len(ents))
    ents = ents[perm]
    e = filled(m, L, E, ents)
    probes = np.concatenate([base[:3], base[30:36], base[:3] * 2])  # scaled rows: distance 0
    check_match(m, orc, e, ents, seqs_of(len(ents)), probes)


def test_match_zero_rows(m, orc):
    L, E, P = 6, 16, 400
    fam = m.gen_bench_family(8, L, E, P + 40).copy()
    rng = np.random.default_rng(1)
    z = rng.random((P + 40, L)) < 0.3
    fam[z] = 0
    fam[P + 35:] = 0  # all-zero probes
    fam[:5] = 0       # all-zero entries
    e = filled(m, L, E, fam[:P])
    check_match(m, orc, e, fam[:P], seqs_of(P), fam[P:])


def test_match_wide_counts(m, orc):
    """Counts above 255 widen the device collection to 2-byte storage."""
    L, E, P = 4, 32, 300
    fam = m.gen_bench_family(21, L, E, P + 30).copy()
    e = filled(m, L, E, fam[:P])
    assert e.count_bytes() == 1
    probes = fam[P:] * 37  # up to 1184 > 255
    check_match(m, orc, e, fam[:P], seqs_of(P), probes)
    assert e.count_bytes() == 2
    big = fam[:P].copy()
    big[::7] *= 1500
    e2 = filled(m, L, E, big)
    check_match(m, orc, e2, big, seqs_of(P), fam[P:])
    # 70,000 > 65,535: 4-byte storage, still exact (sum c^2 < 2^53)
    check_match(m, orc, e2, big, seqs_of(P), fam[P:P + 3] * 70000)
    assert e2.count_bytes() == 4
    # a row with sum c^2 >= 2^53 is outside the reference's exact range
    with pytest.raises(m.CountOverflowError):
        e2.match_batch(fam[P:P + 1] * 100_000_000)


def test_match_long_wide_eams(m, orc):
    """2-byte storage with L*E large enough that k_refine takes its
    lane-per-row path (L x 20 chunks of 16 B > the chunk-parallel scratch)."""
    L, E, P = 40, 160, 500
    fam = m.gen_bench_family(31, L, E, P + 20).copy()
    fam[::3] *= 300
    e = filled(m, L, E, fam[:P])
    assert e.count_bytes() == 2
    check_match(m, orc, e, fam[:P], seqs_of(P), fam[P:])
    dup = np.concatenate([fam[:P], np.repeat(fam[P:P + 1], 40, axis=0)])
    e2 = filled(m, L, E, dup)
    check_match(m, orc, e2, dup, seqs_of(len(dup)), fam[P:P + 2])


def test_match_f2_workload(m, orc):
    """Realistic grouped/skewed request EAMs (F2) and iteration probes."""
    w = Workload(12, 64, 1, seed=1001)
    ents = orc.request_eams(w, 300)
    probes = np.stack([orc.iteration_probe(w, 500 + i, 1 + i % 8, i % 12) for i in range(40)])
    e = filled(m, 12, 64, ents)
    check_match(m, orc, e, ents, seqs_of(300), probes)


def test_match_large_collection(m, orc):
    """P = 100k at the Switch shape (> one wave of tiles on every SM)."""
    L, E, P, Q = 12, 128, 100_000, 3
    fam = m.gen_bench_family(55, L, E, P + Q, dtype=np.uint8)
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
    e.append(fam[:P], seqs_of(P))
    got = e.match_batch(fam[P:].astype(np.uint64))
    idx, seq, d, _ = orc.match(fam[:P].astype(np.uint64), seqs_of(P), fam[P:].astype(np.uint64))
    assert np.array_equal(got["index"], idx) and np.array_equal(got["distance"], d)


def test_match_device_api(m, orc):
    import ctypes as C
    import torch
    from paper_2401_14361_b200 import _lib
    L, E, P, Q = 12, 128, 1000, 50
    fam = m.gen_bench_family(3, L, E, P + Q)
    e = filled(m, L, E, fam[:P])
    for dt in (torch.uint8, torch.int16, torch.int64):
        pr = torch.from_numpy(fam[P:].astype(np.int64)).to(dt).cuda()
        out = torch.zeros((Q, 3), dtype=torch.float64, device="cuda")  # 24 B per moe_match
        stream = torch.cuda.current_stream().cuda_stream
        _lib.check(_lib.lib.moe_eamc_match_device(e._h, pr.data_ptr(), pr.element_size(), Q,
                                                  out.data_ptr(), C.c_void_p(stream)))
        torch.cuda.synchronize()
        res = out.cpu().numpy().view(np.uint8).reshape(Q, 24).copy().view(_lib.MATCH_DTYPE)[:, 0]
        idx, seq, d, _ = orc.match(fam[:P], seqs_of(P), fam[P:])
        assert np.array_equal(res["index"], idx) and np.array_equal(res["distance"], d)


# ------------------------------------------------------------ construction
def test_insert_replay_golden(m, orc, golden):
    g = golden("insert_replay.npz")
    s = m.ModelShape(2, 4)
    e = m.Eamc(s, m.Phase.decode, 10)
    slots = e.build(g["eams"])
    assert np.array_equal(slots, g["slots"])
    for i in range(e.size()):
        assert np.array_equal(e.entry(i).counts, g["entries"][i])
        assert e.entry_seq(i) == g["seqs"][i]
    # one-at-a-time inserts return the evicted Eam (eam.cpp:175-177)
    e1 = m.Eamc(m.ModelShape(1, 4), m.Phase.decode, 3)
    ex = g["ex"]
    for x in ex[:3]:
        assert e1.insert(m.Eam(m.ModelShape(1, 4), counts=x)) is None
    ev = e1.insert(m.Eam(m.ModelShape(1, 4), counts=ex[3]))
    assert ev is not None and np.array_equal(ev.counts, ex[2])
    assert e1.size() == 3
    # sqrt(82)*sqrt(82) != 82 in fp64: the reference itself returns 2.2e-16 here
    assert e1.match(m.Eam(m.ModelShape(1, 4), counts=ex[3])).distance == orc.distance(ex[3], ex[3])


def test_insert_validation(m):
    s = m.ModelShape(1, 2)
    e = m.Eamc(s, m.Phase.decode, 2)
    with pytest.raises(ValueError):
        e.insert(m.Eam(s, m.EamKind.iteration, m.Phase.decode))
    with pytest.raises(ValueError):
        e.insert(m.Eam(s, m.EamKind.request, m.Phase.prefill))
    with pytest.raises(ValueError):
        e.insert(m.Eam(m.ModelShape(2, 2)))


@pytest.mark.parametrize("L,E,cap,n,seed", [(24, 128, 50, 400, 3), (12, 128, 200, 900, 55),
                                            (2, 4, 10, 600, 1)])
def test_build_replay_vs_oracle(m, orc, L, E, cap, n, seed):
    eams = m.gen_bench_family(seed, L, E, n)
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, cap)
    slots = e.build(eams)
    ent, sq, want = orc.insert_replay(L, E, cap, eams)
    assert np.array_equal(slots, want)
    for i in range(cap):
        assert e.entry_seq(i) == sq[i]
    assert np.array_equal(e.entry(cap // 2).counts, ent[cap // 2])


def test_build_replay_f2_nllb_shape(m, orc):
    w = Workload(24, 128, 2, seed=1234)
    eams = orc.request_eams(w, 260)
    e = m.Eamc(m.ModelShape(24, 128, 2), m.Phase.decode, 60)
    slots = e.build(eams)
    _, _, want = orc.insert_replay(24, 128, 60, eams)
    assert np.array_equal(slots, want)


def test_build_with_duplicates(m, orc):
    """Tied victims (duplicate entries) resolve to the oldest seq."""
    base = m.gen_bench_family(17, 4, 16, 6)
    eams = np.concatenate([np.repeat(base[:2], 40, axis=0), base[2:], base[:2]])
    e = m.Eamc(m.ModelShape(4, 16), m.Phase.decode, 70)
    slots = e.build(eams)
    _, _, want = orc.insert_replay(4, 16, 70, eams)
    assert np.array_equal(slots, want)


@pytest.mark.parametrize("block", [None, "16", "37"])
def test_blocked_replay_edge_cases(m, orc, monkeypatch, block):
    """Blocked construction replay (screen matrices + one-CTA sequential
    decisions): re-replacement of a slot inside one block, steps that pick
    an entry inserted earlier in the same block, block boundaries, u16
    storage, and a band wider than the candidate list (> 1024 tied slots)."""
    if block:
        monkeypatch.setenv("MOE_REPLAY_BLOCK", block)
    base = m.gen_bench_family(23, 6, 32, 40)
    # repeated incoming EAMs: the same slot is replaced again and again
    eams = np.concatenate([base[:30], np.repeat(base[30:32], 25, axis=0), base[32:], base[:8]])
    for cap in (30, 31):
        e = m.Eamc(m.ModelShape(6, 32), m.Phase.decode, cap)
        slots = e.build(eams)
        ent, sq, want = orc.insert_replay(6, 32, cap, eams)
        assert np.array_equal(slots, want)
        for i in range(cap):
            assert e.entry_seq(i) == sq[i]
            assert np.array_equal(e.entry(i).counts, ent[i])
    wide = m.gen_bench_family(24, 5, 40, 300).copy()
    wide[::3] *= 500  # 2-byte storage
    e = m.Eamc(m.ModelShape(5, 40), m.Phase.decode, 90)
    slots = e.build(wide)
    assert e.count_bytes() == 2
    _, _, want = orc.insert_replay(5, 40, 90, wide)
    assert np.array_equal(slots, want)


def test_blocked_replay_mass_ties(m, orc):
    """1,100 identical entries: every incoming EAM's screen band holds more
    slots than the one-CTA candidate list; the slot-order walk resolves the
    (distance, seq) minimum exactly."""
    base = m.gen_bench_family(25, 3, 16, 4)
    eams = np.concatenate([np.repeat(base[:1], 1100, axis=0), base[1:3], np.repeat(base[:1], 20, axis=0)])
    e = m.Eamc(m.ModelShape(3, 16), m.Phase.decode, 1100)
    slots = e.build(eams)
    _, _, want = orc.insert_replay(3, 16, 1100, eams)
    assert np.array_equal(slots, want)


def test_snapshot_round_trip(m, tmp_path):
    s = m.ModelShape(3, 6, 1)
    empty = m.Eamc(s, m.Phase.prefill, 5)
    p = str(tmp_path / "snap.json")
    empty.save(p)
    back = m.Eamc.load(p)
    assert back.size() == 0 and back.capacity() == 5 and back.phase() == m.Phase.prefill
    full = m.Eamc(s, m.Phase.decode, 64)
    fam = m.gen_bench_family(41, 3, 6, 101)
    full.build(fam[:100])
    full.save(p)
    b1 = m.Eamc.load(p, s)
    assert b1.size() == full.size() and b1.next_seq() == full.next_seq()
    for i in range(b1.size()):
        assert np.array_equal(b1.entry(i).counts, full.entry(i).counts)
        assert b1.entry_seq(i) == full.entry_seq(i)
    b2 = m.Eamc.load(p, s)
    x = m.Eam(s, counts=fam[100])
    assert b1.insert(x) == b2.insert(x)
    with pytest.raises(m.EamcSnapshotError):
        m.Eamc.load(p, m.ModelShape(4, 6, 1))
    open(p, "w").write('{"version": 99}\n')
    with pytest.raises(m.EamcSnapshotError):
        m.Eamc.load(p)
    open(p, "w").write("not json\n")
    with pytest.raises(m.EamcSnapshotError):
        m.Eamc.load(p)


# ---------------------------------------------------------------- policy
def test_prefetch_worked_example(m, golden):
    g = golden("prefetch.npz")
    s = m.ModelShape(4, 2)
    e = m.Eamc(s, m.Phase.decode, 4)
    e.insert(m.Eam(s, counts=[[1, 0], [1, 0], [2, 1], [0, 3]]))
    cur = m.Eam(s, m.EamKind.iteration, counts=[[1, 0], [1, 0], [0, 0], [0, 0]])
    out = m.prefetch_priorities(cur, e, 1)
    assert [c.expert.layer_idx for c in out] == list(g["worked_l"])
    assert [c.expert.expert_idx for c in out] == list(g["worked_e"])
    assert [c.priority for c in out] == list(g["worked_p"])
    assert out[0].expert == m.ExpertId(2, 0) and abs(out[0].priority - 0.500075) < 1e-12
    with pytest.raises(IndexError):
        m.prefetch_priorities(cur, e, 4)
    assert m.prefetch_priorities(cur, m.Eamc(s, m.Phase.decode, 2), 0) == []


def test_prefetch_zero_rows_floor(m):
    """test_policy.cpp:67-82: zero rows -> epsilon floor, ties in ExpertId order."""
    s = m.ModelShape(3, 2)
    e = m.Eamc(s, m.Phase.decode, 2)
    e.insert(m.Eam(s, counts=[[1, 0], [0, 0], [0, 0]]))
    cur = m.Eam(s, m.EamKind.iteration, counts=[[1, 0], [0, 0], [0, 0]])
    out = m.prefetch_priorities(cur, e, 0)
    assert len(out) == 4
    assert out[0].expert == m.ExpertId(1, 0) and out[1].expert == m.ExpertId(1, 1)
    assert m.prefetch_priorities(cur, e, 0, apply_floor_filter=True) == []


def test_prefetch_f2_golden(m, golden):
    g = golden("prefetch.npz")
    s = m.ModelShape(32, 8, 2)
    e = m.Eamc(s, m.Phase.decode, 60)
    e.build(g["f2_entries"])
    o = 0
    for i in range(len(g["f2_n"])):
        n = int(g["f2_n"][i])
        cur = m.Eam(s, m.EamKind.iteration, counts=g["f2_probes"][i])
        out = m.prefetch_order(cur, e, int(g["f2_layers"][i]), bool(g["f2_filter"][i]))
        assert np.array_equal(out["layer_idx"], g["f2_l"][o:o + n])
        assert np.array_equal(out["expert_idx"], g["f2_e"][o:o + n])
        assert np.array_equal(out["priority"], g["f2_p"][o:o + n])  # bitwise
        o += n


@pytest.mark.parametrize("L,E,P,seed", [(59, 160, 200, 5), (12, 128, 1000, 7), (24, 128, 300, 9)])
def test_prefetch_vs_oracle(m, orc, L, E, P, seed):
    w = Workload(L, E, min(6, E), n_groups=12, prompt_len=3, decode_len=4, batch_size=2,
                 seed=seed)
    ents = orc.request_eams(w, P)
    s = m.ModelShape(L, E, min(6, E))
    e = m.Eamc(s, m.Phase.decode, P)
    e.build(ents)
    for r, it, layer in [(900, 1, 0), (901, 2, L // 2), (902, 3, L - 2), (903, 4, L - 1)]:
        pr = orc.iteration_probe(w, r, it, layer)
        for flt in (True, False):
            l, x, p = orc.prefetch(ents, seqs_of(P), pr, layer, flt)
            out = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=pr), e, layer, flt)
            assert np.array_equal(out["layer_idx"], l)
            assert np.array_equal(out["expert_idx"], x)
            assert np.array_equal(out["priority"], p)


def test_prefetch_decode_sequence_incremental(m, orc):
    """The engine's call pattern (engine.cpp:546, :587, :658-678): one decode
    iteration calls prefetch_priorities at l = 0..L-2 with the iteration EAM
    growing by one row; the device reuses the layer-prefix sums of the rows
    that did not change.  Every call must equal the oracle, including after a
    prefix break (next iteration), a repeated / earlier layer, rows beyond the
    current layer, a collection mutation, and u16 storage."""
    L, E, P = 9, 24, 700
    w = Workload(L, E, 3, n_groups=10, prompt_len=3, decode_len=4, batch_size=2, seed=77)
    ents = orc.request_eams(w, P)
    s = m.ModelShape(L, E, 3)
    e = m.Eamc(s, m.Phase.decode, P + 5)
    e.build(ents)
    seqs = list(range(P))

    def check(pr, layer, flt=True, entries=None):
        entries = ents if entries is None else entries
        lx, ex, px = orc.prefetch(entries, np.arange(len(entries), dtype=np.uint64), pr, layer, flt)
        out = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=pr), e, layer, flt)
        assert np.array_equal(out["layer_idx"], lx), layer
        assert np.array_equal(out["expert_idx"], ex), layer
        assert np.array_equal(out["priority"], px), layer

    for it in (1, 2):
        for layer in range(L - 1):
            check(orc.iteration_probe(w, 500 + it, it, layer), layer)
    pr = orc.iteration_probe(w, 600, 2, 4)
    check(pr, 4)
    check(pr, 4)                     # same call again
    check(orc.iteration_probe(w, 600, 2, 6), 6)
    check(orc.iteration_probe(w, 600, 2, 2), 2)  # earlier layer, shared prefix
    full = orc.iteration_probe(w, 601, 2, L - 1)
    check(full, 3)                   # rows beyond the current layer are nonzero
    check(full, 5, flt=False)
    # mutation: an append changes the collection -> the prefix cache is stale
    extra = orc.request_eams(w, P + 3)[P:]
    e.build(extra)
    allents = np.concatenate([ents, extra])
    check(orc.iteration_probe(w, 600, 2, 6), 6, entries=allents)
    check(orc.iteration_probe(w, 600, 2, 7), 7, entries=allents)
    # u16 storage (widened collection)
    big = allents.copy()
    big[::4] *= 300
    e2 = m.Eamc(s, m.Phase.decode, len(big))
    e2.build(big)
    assert e2.count_bytes() == 2
    for layer in (0, 1, 2, 5):
        pr = orc.iteration_probe(w, 700, 3, layer)
        lx, ex, px = orc.prefetch(big, np.arange(len(big), dtype=np.uint64), pr, layer, True)
        out = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=pr), e2, layer, True)
        assert np.array_equal(out["expert_idx"], ex) and np.array_equal(out["priority"], px)
    # a probe wider than the storage width takes the u64 path (widens)
    pr = orc.iteration_probe(w, 701, 3, 3) * 400
    check(pr, 3, entries=allents)


def test_eviction_golden(m, golden):
    g = golden("eviction.npz")
    s = m.ModelShape(4, 8)
    for req, v, want in zip(g["reqs"], g["views"], g["victims"]):
        slots = [m.SlotView(int(v[0][i]), m.ExpertId(int(v[1][i]), int(v[2][i])), bool(v[3][i]),
                            bool(v[4][i])) for i in range(v.shape[1])]
        got = m.select_eviction_victim(slots, m.Eam(s, counts=req))
        assert (got if got is not None else -1) == want
    cs = m.ModelShape(3, 2)
    req = m.Eam(cs, counts=g["cp_req"])
    got = [m.cache_priority(req, m.ExpertId(0, 1)), m.cache_priority(req, m.ExpertId(1, 0)),
           m.cache_priority(req, m.ExpertId(2, 1))]
    assert got == list(g["cp"])
    with pytest.raises(IndexError):
        m.cache_priority(req, m.ExpertId(3, 0))
    assert m.select_eviction_victim([], req) is None


def test_fused_decide(m, orc):
    """K5+K6 in one launch equals prefetch_priorities+filter and the victim."""
    w = Workload(12, 64, 2, seed=31)
    ents = orc.request_eams(w, 100)
    s = m.ModelShape(12, 64, 2)
    e = m.Eamc(s, m.Phase.decode, 100)
    e.build(ents)
    pr = orc.iteration_probe(w, 555, 2, 4)
    req = orc.request_eams(w, 1, start=777)[0]
    slots = [m.SlotView(i, m.ExpertId(i % 12, (7 * i) % 64), i % 5 == 0, i % 7 == 0)
             for i in range(40)]
    order, victim = m.decide(m.Eam(s, m.EamKind.iteration, counts=pr), e, 4, m.Eam(s, counts=req),
                             slots)
    l, x, p = orc.prefetch(ents, seqs_of(100), pr, 4, True)
    assert np.array_equal(order["layer_idx"], l) and np.array_equal(order["priority"], p)
    want = orc.select_victim(req, [v.slot for v in slots],
                             [v.occupant.layer_idx for v in slots],
                             [v.occupant.expert_idx for v in slots],
                             [int(v.prefetch_protected) for v in slots],
                             [int(v.pinned) for v in slots])
    assert (victim if victim is not None else -1) == want


# ---------------------------------------------------------------- tracing
@pytest.mark.parametrize("name,w", [
    ("mix", Workload(32, 8, 2, seed=99)),
    ("ds", Workload(59, 160, 6, n_groups=8, prompt_len=40, decode_len=25, batch_size=2, seed=5)),
])
def test_trace_vs_oracle(m, orc, name, w):
    p = w.params
    picks, offs = [], [0]
    for r in range(6):
        _, pk = orc.trace_picks(w, r)
        picks.append(pk)
        offs.append(offs[-1] + pk.shape[0])
    picks = np.concatenate(picks)
    offs = np.array(offs, np.uint64)
    rc, want = orc.trace(p["L"], p["E"], p["top_k"], picks, offs)
    assert rc == 0
    s = m.ModelShape(p["L"], p["E"], p["top_k"])
    for dt in (np.uint8, np.uint16, np.uint32):
        got = m.trace_requests(s, picks.astype(dt), offs)
        assert np.array_equal(got, want)
    # accumulate semantics (Eam::record adds)
    base = np.ones_like(want)
    got = m.trace_requests(s, picks.astype(np.uint8), offs, counts=base.copy())
    assert np.array_equal(got, want + 1)


def test_trace_all_or_nothing(m):
    s = m.ModelShape(2, 4, 2)
    picks = np.array([[[0, 1], [2, 3]], [[1, 2], [3, 9]]], np.uint8)
    base = np.full((1, 2, 4), 5, np.uint64)
    with pytest.raises(IndexError):
        m.trace_requests(s, picks, np.array([0, 2], np.uint64), counts=base)
    assert (base == 5).all()


# ------------------------------------------------- tensor-core screen path
@pytest.mark.parametrize("L,E,P,Q,seed", [
    (12, 128, 2000, 300, 55),   # SW shape, ragged M and N tiles
    (32, 8, 300, 200, 7),       # MIX
    (59, 160, 300, 130, 9),     # DS (L=59 <= 64 zero-row mask bits)
    (24, 128, 777, 256, 3),     # NL
    (3, 5, 77, 129, 1),
])
def test_match_tensor_core_path(m, orc, monkeypatch, L, E, P, Q, seed):
    monkeypatch.setenv("MOE_TC", "1")
    fam = m.gen_bench_family(seed, L, E, P + Q)
    e = filled(m, L, E, fam[:P])
    check_match(m, orc, e, fam[:P], seqs_of(P), fam[P:])


def test_tensor_core_small_batches_and_edge_cases(m, orc, monkeypatch):
    monkeypatch.setenv("MOE_TC", "1")
    L, E, P = 6, 16, 600
    fam = m.gen_bench_family(8, L, E, P + 200).copy()
    rng = np.random.default_rng(3)
    fam[rng.random((P + 200, L)) < 0.3] = 0
    fam[P + 190:] = 0
    fam[:5] = 0
    fam[100:400] = fam[100]  # mass duplicates -> bucket overflow -> exact pass
    e = filled(m, L, E, fam[:P])
    for Q in (1, 7, 200):
        check_match(m, orc, e, fam[:P], seqs_of(P), fam[P:P + Q])
    check_match(m, orc, e, fam[:P], seqs_of(P), fam[100:160])


def test_tensor_core_wide_counts(m, orc, monkeypatch):
    monkeypatch.setenv("MOE_TC", "1")
    L, E, P = 4, 32, 500
    fam = m.gen_bench_family(21, L, E, P + 150).copy()
    fam[::5] *= 1900  # 2-byte storage, subnormal fp16 normalised values
    e = filled(m, L, E, fam[:P])
    check_match(m, orc, e, fam[:P], seqs_of(P), fam[P:])


def test_tensor_core_f2_and_build(m, orc, monkeypatch):
    monkeypatch.setenv("MOE_TC", "1")
    w = Workload(12, 64, 1, seed=1001)
    ents = orc.request_eams(w, 400)
    probes = np.stack([orc.iteration_probe(w, 500 + i, 1 + i % 8, i % 12) for i in range(150)])
    e = filled(m, 12, 64, ents)
    check_match(m, orc, e, ents, seqs_of(400), probes)
    # replacement steps after a tensor-core-screened build keep the fp16 copy in sync
    e2 = m.Eamc(m.ModelShape(12, 64), m.Phase.decode, 150)
    slots = e2.build(ents)
    _, _, want = orc.insert_replay(12, 64, 150, ents)
    assert np.array_equal(slots, want)
    cur_e, cur_s, _ = orc.insert_replay(12, 64, 150, ents)
    check_match(m, orc, e2, cur_e, cur_s, probes)


def test_device_api_async_width_sentinel_and_overflow(m, orc):
    """The device path never waits on the host: a probe wider than the storage
    width gets the sentinel, and mass ties are resolved by the device-gated
    exact pass."""
    import ctypes as C
    import torch
    from paper_2401_14361_b200 import _lib
    L, E, P = 6, 32, 400
    fam = m.gen_bench_family(12, L, E, P + 10).copy()
    fam[50:300] = fam[50]  # 250 exact duplicates -> bucket overflow for probe 0
    e = filled(m, L, E, fam[:P])
    probes = np.concatenate([fam[50:51], fam[P:P + 8], fam[P + 8:P + 9] * 300])  # last: > 255
    st = torch.cuda.Stream()
    pr = torch.from_numpy(probes.astype(np.int64)).cuda()
    out = torch.zeros((len(probes), 3), dtype=torch.float64, device="cuda")
    with torch.cuda.stream(st):
        _lib.check(_lib.lib.moe_eamc_match_device(e._h, pr.data_ptr(), 8, len(probes),
                                                  out.data_ptr(), C.c_void_p(st.cuda_stream)))
    st.synchronize()
    res = out.cpu().numpy().view(np.uint8).reshape(len(probes), 24).copy().view(
        _lib.MATCH_DTYPE)[:, 0]
    idx, seq, d, _ = orc.match(fam[:P], seqs_of(P), probes[:-1])
    assert np.array_equal(res["index"][:-1], idx) and np.array_equal(res["distance"][:-1], d)
    assert int(res["index"][-1]) == 0xFFFFFFFFFFFFFFFE and np.isnan(res["distance"][-1])
    assert e.count_bytes() == 1  # the device path never widens behind the caller's back
    # the host API widens and answers the same probe exactly
    got = e.match_batch(probes[-1:])
    i2, s2, d2, _ = orc.match(fam[:P], seqs_of(P), probes[-1:])
    assert got["index"][0] == i2[0] and got["distance"][0] == d2[0]


@pytest.mark.parametrize("L,dups", [(6, 250), (3, 200), (12, 70), (1, 240)])
def test_refine_many_tied_candidates(m, orc, L, dups):
    """More than 32 exact ties inside the candidate bucket (<= 256): every one
    must be evaluated; the oldest seq wins (eam.cpp:123-124)."""
    E, P = 32, 400
    fam = m.gen_bench_family(12 + L, L, E, P + 4).copy()
    fam[37:37 + dups] = fam[37]
    rng = np.random.default_rng(L)
    perm = rng.permutation(P)
    ents = fam[:P][perm]
    e = filled(m, L, E, ents)
    for _ in range(3):  # bucket push order is nondeterministic: repeat
        check_match(m, orc, e, ents, seqs_of(P), np.concatenate([fam[37:38], fam[P:P + 3]]))


def test_host_api_pipelined_large_batch(m, orc):
    """> 16 MB of u64 probes: chunked H2D overlapped with matching; probes that
    need a wider storage width are redone synchronously after widening."""
    L, E, P, Q = 12, 128, 600, 2200
    fam = m.gen_bench_family(77, L, E, P + Q).copy()
    probes = fam[P:].copy()
    probes[5::97] *= 300  # > 255: forces the widening redo path
    e = filled(m, L, E, fam[:P])
    check_match(m, orc, e, fam[:P], seqs_of(P), probes)
    assert e.count_bytes() == 2
    check_match(m, orc, e, fam[:P], seqs_of(P), fam[P:])


@pytest.mark.parametrize("groups,chunk", [(None, None), ("3", "77"), ("1", "5000")])
def test_host_api_narrowed_batch(m, orc, monkeypatch, groups, chunk):
    """>= 4 MB of u64 probes: narrowed to the storage width on the host pool,
    chunked DMA, matched in groups; both storage widths; identical to the
    u64 path."""
    if groups:
        monkeypatch.setenv("MOE_MATCH_GROUPS", groups)
        monkeypatch.setenv("MOE_PACK_CHUNK", chunk)
    L, E, P, Q = 12, 128, 700, 2111
    fam = m.gen_bench_family(78, L, E, P + Q).copy()
    e = filled(m, L, E, fam[:P])
    got = check_match(m, orc, e, fam[:P], seqs_of(P), fam[P:])
    assert e.count_bytes() == 1
    monkeypatch.setenv("MOE_HOST_PACK", "0")
    ref = e.match_batch(fam[P:])
    assert np.array_equal(ref["index"], got["index"]) and np.array_equal(ref["distance"], got["distance"])
    monkeypatch.delenv("MOE_HOST_PACK")
    wide = fam[:P].copy()
    wide[::5] *= 400  # 2-byte storage: probes narrowed to u16 on the host
    e2 = filled(m, L, E, wide)
    assert e2.count_bytes() == 2
    check_match(m, orc, e2, wide, seqs_of(P), fam[P:] * 3)


def test_trace_long_and_empty_requests(m, orc):
    """Requests longer than one block's ownership limit (chunked, atomics),
    empty requests, unaligned id ranges, and tokens outside any request."""
    L, E, k = 7, 40, 3
    rng = np.random.default_rng(9)
    T = 41_000
    base = rng.integers(0, E, size=(T, L))
    picks = ((base[:, :, None] + np.arange(k)[None, None, :]) % E).astype(np.uint8)
    offs = np.array([0, 20_001, 20_001, 20_006, 40_999], np.uint64)  # long, empty, short, long
    rc, want = orc.trace(L, E, k, picks.astype(np.uint32), offs)
    assert rc == 0
    s = m.ModelShape(L, E, k)
    for dt in (np.uint8, np.uint16, np.uint32):
        got = m.trace_requests(s, picks.astype(dt), offs)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("L,E,P,n_shards", [(59, 160, 240, 3), (24, 128, 301, 2)])
def test_prefetch_sharded_device_steps(m, orc, L, E, P, n_shards):
    """The P-sharded decision steps through the C ABI, with the
    ranks emulated as shard handles on one GPU: local minima -> min,
    per-shard window aggregates -> sum, order from the sum.  Must equal the
    oracle's prefetch_priorities over the whole collection, bitwise."""
    import ctypes as C

    import torch
    from paper_2401_14361_b200 import _lib
    from paper_2401_14361_b200.sharded import ShardedDecider, shard_range
    w = Workload(L, E, min(6, E), n_groups=12, prompt_len=3, decode_len=4, batch_size=2,
                 seed=31)
    ents = orc.request_eams(w, P)
    s = m.ModelShape(L, E, min(6, E))
    shards = []
    for r in range(n_shards):
        a, b = shard_range(P, r, n_shards)
        e = m.Eamc(s, m.Phase.decode, b - a)
        e.append(ents[a:b], np.arange(a, b, dtype=np.uint64))
        shards.append(e)
    whole = m.Eamc(s, m.Phase.decode, P)
    whole.build(ents)
    st = torch.cuda.Stream()
    sp = C.c_void_p(st.cuda_stream)
    lib = _lib.lib
    for r, it, layer in [(900, 1, 0), (901, 2, L // 2), (902, 3, L - 2), (903, 4, L - 1)]:
        pr = np.ascontiguousarray(orc.iteration_probe(w, r, it, layer), np.uint64)
        for flt in (True, False):
            with torch.cuda.stream(st):
                mins = torch.empty(n_shards, dtype=torch.int64, device="cuda")
                for k, e in enumerate(shards):
                    _lib.check(lib.moe_eamc_window_min_device(e._h, pr.ctypes.data,
                                                              mins[k:].data_ptr(), sp))
                gmin = mins.min().reshape(1)
                aggs = torch.empty((n_shards, L * E), dtype=torch.int64, device="cuda")
                for k, e in enumerate(shards):
                    _lib.check(lib.moe_eamc_window_aggregate_device(
                        e._h, layer, 0.01, gmin.data_ptr(), aggs[k].data_ptr(), sp))
                agg = aggs.sum(0).contiguous()
                out = torch.empty((max((L - layer - 1) * E, 1), 2), dtype=torch.float64,
                                  device="cuda")
                n = torch.zeros(1, dtype=torch.int32, device="cuda")
                _lib.check(lib.moe_eamc_prefetch_order_device(shards[0]._h, agg.data_ptr(),
                                                              layer, int(flt), out.data_ptr(),
                                                              n.data_ptr(), sp))
                k = int(n.item())
                got = out[:k].cpu().numpy().view(np.uint8).reshape(k, 16).copy().view(
                    _lib.CAND_DTYPE)[:, 0]
            ol, ox, op = orc.prefetch(ents, seqs_of(P), pr, layer, flt)
            assert np.array_equal(got["layer_idx"], ol)
            assert np.array_equal(got["expert_idx"], ox)
            assert np.array_equal(got["priority"], op)
            # world size 1: the ShardedDecider equals the unsharded call
            one = ShardedDecider(whole).prefetch_order(pr, layer, flt)
            ref = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=pr), whole, layer, flt)
            assert np.array_equal(one, ref)


def test_match_packed_host_probes(m, orc):
    """moe_eamc_match_packed: narrow (u8 / u16) host probes give the same
    results as the u64 reference-API path; u16 counts above 255 widen."""
    L, E, P = 12, 64, 500
    fam = m.gen_bench_family(19, L, E, P + 40)
    e = filled(m, L, E, fam[:P])
    want = check_match(m, orc, e, fam[:P], seqs_of(P), fam[P:])
    got8 = e.match_batch(fam[P:].astype(np.uint8))
    assert np.array_equal(got8, want)
    wide = (fam[P:] * 20).astype(np.uint16)  # up to 640 > 255
    got16 = e.match_batch(wide)
    idx, seq, d, _ = orc.match(fam[:P], seqs_of(P), wide.astype(np.uint64))
    assert np.array_equal(got16["index"], idx) and np.array_equal(got16["distance"], d)
    assert e.count_bytes() == 2


def test_pipeline_without_pdl():
    """The match / decision pipelines with programmatic dependent launch
    disabled (plain stream order, MOE_PDL=0): the smoke checks still hold."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MOE_PDL="0")
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=root,
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "smoke ok" in r.stdout


@pytest.mark.parametrize("L,E,P,mult", [(32, 8, 300, 1), (8, 16, 1000, 1), (4, 4, 37, 1),
                                        (16, 32, 200, 40)])
def test_prefetch_small_collection(m, orc, L, E, P, mult):
    """Small collections (one or a few CTAs of the fused decision kernel,
    decide.cu); mult > 1 pushes counts past 255 (u16 storage)."""
    w = Workload(L, E, min(2, E), n_groups=6, prompt_len=3, decode_len=4, batch_size=2, seed=L + P)
    ents = orc.request_eams(w, P) * mult
    s = m.ModelShape(L, E, min(2, E))
    e = m.Eamc(s, m.Phase.decode, P)
    e.build(ents)
    for r, it, layer in [(700, 1, 0), (701, 2, L // 2), (702, 3, L - 2), (703, 4, L - 1)]:
        pr = orc.iteration_probe(w, r, it, layer) * mult
        for flt in (True, False):
            ol, ox, op = orc.prefetch(ents, seqs_of(P), pr, layer, flt)
            out = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=pr), e, layer, flt)
            assert np.array_equal(out["layer_idx"], ol)
            assert np.array_equal(out["expert_idx"], ox)
            assert np.array_equal(out["priority"], op)


@pytest.mark.parametrize("L,E,P,mult", [(72, 8, 150, 1), (32, 8, 509, 1), (20, 8, 64, 70000),
                                        (12, 8, 9, 1)])
def test_prefetch_small_cluster_shapes(m, orc, L, E, P, mult):
    """The small-path decision kernel launched as a thread-block cluster
    (size x explicit rows >= 1,024; decide.cu small_body): L > 64 (no
    zero-row mask), entry counts not a multiple of the cluster size, u32
    storage (counts of 70,000), and a collection small enough for one CTA."""
    w = Workload(L, E, 2, n_groups=5, prompt_len=3, decode_len=4, batch_size=2, seed=L * 7 + P)
    ents = orc.request_eams(w, P) * mult
    s = m.ModelShape(L, E, 2)
    e = m.Eamc(s, m.Phase.decode, P)
    e.build(ents)
    for r, it, layer in [(800, 1, 0), (801, 2, L // 3), (802, 3, (2 * L) // 3), (803, 4, L - 2)]:
        pr = orc.iteration_probe(w, r, it, layer) * mult
        ol, ox, op = orc.prefetch(ents, seqs_of(P), pr, layer, True)
        out = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=pr), e, layer, True)
        assert np.array_equal(out["layer_idx"], ol)
        assert np.array_equal(out["expert_idx"], ox)
        assert np.array_equal(out["priority"], op)


def test_prefetch_small_cluster_decode_sequence(m, orc):
    """One decode step on a small collection: the iteration EAM grows by one
    row per call, so the cluster path reuses the stored layer-prefix sums
    (j0 > 0) -- every call's order equals the oracle's."""
    L, E, P = 32, 8, 300
    w = Workload(L, E, 2, n_groups=6, prompt_len=3, decode_len=4, batch_size=2, seed=4242)
    ents = orc.request_eams(w, P)
    s = m.ModelShape(L, E, 2)
    e = m.Eamc(s, m.Phase.decode, P)
    e.build(ents)
    full = orc.iteration_probe(w, 900, 2, L - 1)
    for layer in range(L - 1):
        pr = full.copy()
        pr[layer + 1:] = 0
        ol, ox, op = orc.prefetch(ents, seqs_of(P), pr, layer, True)
        out = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=pr), e, layer, True)
        assert np.array_equal(out["layer_idx"], ol), layer
        assert np.array_equal(out["expert_idx"], ox), layer
        assert np.array_equal(out["priority"], op), layer


@pytest.mark.parametrize("n", ["1", "2"])
def test_prefetch_small_cluster_sizes(n):
    """The small-collection parity cases with other cluster sizes
    (MOE_DEC_CLUSTER: 1 = the one-CTA kernel, 2 = a two-CTA cluster; the
    default is 8), in a subprocess since the switch is read once."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MOE_DEC_CLUSTER=n)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "tests/test_gpu_parity.py", "-k",
                        "small_cluster_shapes or small_cluster_decode or small_collection"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " passed" in r.stdout


def test_concurrent_readers_one_handle(m, orc):
    """match / prefetch are const readers (eam.hpp:89-94): concurrent calls on
    one handle from several host threads give the serial results."""
    from concurrent.futures import ThreadPoolExecutor
    L, E, P = 12, 32, 400
    fam = m.gen_bench_family(23, L, E, P + 64)
    e = filled(m, L, E, fam[:P])
    want = e.match_batch(fam[P:])
    s = m.ModelShape(L, E, 1)
    probes = [fam[P + i].copy() for i in range(8)]  # copies: fam itself is matched too
    for i, pr in enumerate(probes):
        pr[i % (L - 1) + 1:] = 0
    want_pf = [m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=pr), e, i % (L - 1), True)
               for i, pr in enumerate(probes)]

    def work(k):
        ok = True
        for _ in range(5):
            ok &= bool(np.array_equal(e.match_batch(fam[P:]), want))
            i = k % len(probes)
            got = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=probes[i]), e,
                                   i % (L - 1), True)
            ok &= bool(np.array_equal(got, want_pf[i]))
        return ok

    with ThreadPoolExecutor(4) as ex:
        assert all(ex.map(work, range(8)))


@pytest.mark.parametrize("E,offset", [(40, 0), (128, 16), (128, 4)])
def test_match_device_u8_layouts(m, orc, E, offset):
    """Device u8 probes: rows narrower than the storage row (E % 16 != 0: a
    packed copy is made), and base pointers at 16- and 4-byte offsets (only a
    16-byte aligned batch in the storage layout is used in place)."""
    import ctypes as C
    import torch
    from paper_2401_14361_b200 import _lib
    L, P, Q = 6, 700, 40
    fam = m.gen_bench_family(41, L, E, P + Q)
    e = filled(m, L, E, fam[:P])
    flat = torch.zeros(offset + Q * L * E, dtype=torch.uint8, device="cuda")
    flat[offset:] = torch.from_numpy(fam[P:].astype(np.uint8).reshape(-1)).cuda()
    out = torch.zeros((Q, 3), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib.moe_eamc_match_device(e._h, flat.data_ptr() + offset, 1, Q,
                                              out.data_ptr(), None))
    torch.cuda.synchronize()
    res = out.cpu().numpy().view(np.uint8).reshape(Q, 24).copy().view(_lib.MATCH_DTYPE)[:, 0]
    idx, seq, d, _ = orc.match(fam[:P], seqs_of(P), fam[P:])
    assert np.array_equal(res["index"], idx) and np.array_equal(res["distance"], d)


# ------------------------------------------ i8 streaming screen, 1-3 M tiles
@pytest.mark.parametrize("L,E,Q", [(12, 128, 8), (12, 128, 16), (12, 128, 24), (32, 8, 12),
                                   (3, 64, 96), (30, 32, 3)])
def test_match_i8_screen_m_tiles(m, orc, L, E, Q):
    """u8 collections with Q up to three 128-row block-diagonal M tiles take
    the kind::i8 tensor-core screen (its entry norms staged in shared memory):
    bitwise vs the oracle, incl. exact duplicates (ties) and zero rows."""
    P = 3000
    fam = m.gen_bench_family(13, L, E, P + Q).copy()
    fam[P - 40:P] = fam[:40]            # exact duplicate entries: ties by seq
    fam[5, :L // 2] = 0                 # zero rows
    probes = np.concatenate([fam[[0, 7, 2999]], fam[P:P + Q - 3]])
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
    e.append(fam[:P], np.arange(P, dtype=np.uint64))
    assert e.count_bytes() == 1
    check_match(m, orc, e, fam[:P], np.arange(P, dtype=np.uint64), probes)
