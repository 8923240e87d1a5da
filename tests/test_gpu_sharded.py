"""P-sharded collections behind the C ABI (moe_eamc_create_sharded):
every entry point on a sharded handle must give exactly the unsharded Eamc's
answer -- the oracle's, bitwise.  On this one-GPU box the shards share device
0, so the collectives take the device-copy path; the sharded logic (slot
ranges, per-shard matching, gather + lexicographic merge, MIN/SUM reductions,
victim selection across shards) is the same one NCCL drives on distinct GPUs.
"""
import numpy as np
import pytest

from oracle import Workload

pytestmark = pytest.mark.gpu


def seqs_of(n):
    return np.arange(n, dtype=np.uint64)


def _replayed(m, orc, L, E, cap, n, seed, dup_every=0):
    """A collection whose slot order is not seq order (reference insert rule),
    with exact duplicates across the shard boundaries when dup_every > 0."""
    fam = m.gen_bench_family(seed, L, E, n + 96).copy()
    if dup_every:
        fam[cap::dup_every] = fam[0]
    ent, seqs, _ = orc.insert_replay(L, E, cap, fam[:n])
    return ent, seqs, fam[n:]


@pytest.mark.parametrize("L,E,cap,n_shards", [(12, 64, 1500, 3), (32, 8, 300, 4), (59, 160, 200, 2)])
def test_sharded_match_vs_oracle(m, orc, L, E, cap, n_shards):
    ent, seqs, probes = _replayed(m, orc, L, E, cap, cap + 700, 41, dup_every=37)
    probes = np.concatenate([ent[[0, 5, cap // 2, cap - 1]], probes])  # self-matches, ties
    e = m.Eamc.sharded(m.ModelShape(L, E), m.Phase.decode, cap, [0] * n_shards)
    assert e.shard_layout() == (n_shards, False)
    e.append(ent, seqs)
    assert e.size() == cap and e.next_seq() == int(seqs.max()) + 1
    got = e.match_batch(probes)
    idx, sq, d, _ = orc.match(ent, seqs, probes)
    assert np.array_equal(got["index"], idx)
    assert np.array_equal(got["seq"], sq)
    assert np.array_equal(got["distance"], d)
    # wide probes (counts > 255): the u8 shards widen, results stay exact
    wide = probes[:20] * 40
    got = e.match_batch(wide)
    idx, sq, d, _ = orc.match(ent, seqs, wide)
    assert np.array_equal(got["index"], idx) and np.array_equal(got["distance"], d)
    # entries through the facade
    for i in (0, cap // 3, cap - 1):
        assert np.array_equal(e.entry(i).counts, ent[i]) and e.entry_seq(i) == seqs[i]


def test_sharded_partially_filled(m, orc):
    """Capacity 12 over 3 shards with 5 entries: shards 1 and 2 (partly) empty."""
    L, E = 4, 16
    fam = m.gen_bench_family(3, L, E, 40)
    e = m.Eamc.sharded(m.ModelShape(L, E), m.Phase.decode, 12, [0, 0, 0])
    assert e.match(m.Eam(m.ModelShape(L, E), counts=fam[30])) is None  # empty: no match
    e.append(fam[:5], seqs_of(5))
    got = e.match_batch(fam[10:40])
    idx, sq, d, _ = orc.match(fam[:5], seqs_of(5), fam[10:40])
    assert np.array_equal(got["index"], idx) and np.array_equal(got["distance"], d)


@pytest.mark.parametrize("n_shards", [2, 3])
def test_sharded_insert_replay(m, orc, n_shards):
    """Eamc::insert (eam.cpp:152-178) on a sharded handle: appends fill the
    slot ranges in order, at capacity the victim is the global (distance, seq)
    argmin across shards; slots, evicted entries, final contents and seqs equal
    the reference replay, including duplicate (tied) incoming EAMs."""
    L, E, cap = 8, 32, 90
    fam = m.gen_bench_family(17, L, E, 400).copy()
    fam[150::13] = fam[2]  # exact ties with an early entry
    e = m.Eamc.sharded(m.ModelShape(L, E), m.Phase.decode, cap, [0] * n_shards)
    slots = e.build(fam)
    want_ent, want_seqs, want_slots = orc.insert_replay(L, E, cap, fam)
    assert np.array_equal(slots, want_slots)
    assert e.size() == cap and e.next_seq() == len(fam)
    for i in range(cap):
        assert np.array_equal(e.entry(i).counts, want_ent[i])
        assert e.entry_seq(i) == want_seqs[i]
    # single inserts return the evicted Eam
    inc = m.Eam(m.ModelShape(L, E), counts=fam[7])
    ev = e.insert(inc)
    want_ent2, _, want_slot2 = orc.insert_replay(L, E, cap, np.concatenate([fam, fam[7:8]]))
    assert ev is not None and np.array_equal(ev.counts, want_ent[want_slot2[-1]])


@pytest.mark.parametrize("L,E,k,P,n_shards", [(24, 128, 2, 301, 3), (59, 160, 6, 240, 2),
                                               (32, 8, 2, 300, 4)])
def test_sharded_prefetch_and_within_vs_oracle(m, orc, L, E, k, P, n_shards):
    w = Workload(L, E, k, seed=7)
    ents = orc.request_eams(w, P)
    s = m.ModelShape(L, E, k)
    e = m.Eamc.sharded(s, m.Phase.decode, P, [0] * n_shards)
    e.append(ents, seqs_of(P))
    for r, layer in [(900, 0), (901, L // 2), (902, L - 2), (903, L - 1)]:
        probe = orc.iteration_probe(w, r, 2, layer)
        cur = m.Eam(s, m.EamKind.iteration, counts=probe)
        for filt in (True, False):
            order = m.prefetch_order(cur, e, layer, filt)
            ol, oe, op = orc.prefetch(ents, seqs_of(P), probe, layer, filt)
            assert np.array_equal(order["layer_idx"], ol)
            assert np.array_equal(order["expert_idx"], oe)
            assert np.array_equal(order["priority"], op)
        within = e.match_within(cur, 0.01)
        wi, ws, wd = orc.match_within(ents, seqs_of(P), probe, 0.01)
        assert [x.index for x in within] == list(wi)
        assert [x.seq for x in within] == list(ws)
        assert [x.distance for x in within] == list(wd)


def test_sharded_decide_save_clone(m, orc, tmp_path):
    L, E, k, P = 12, 64, 2, 100
    w = Workload(L, E, k, seed=31)
    ents = orc.request_eams(w, P)
    s = m.ModelShape(L, E, k)
    e1 = m.Eamc(s, m.Phase.decode, P)
    e3 = m.Eamc.sharded(s, m.Phase.decode, P, [0, 0, 0])
    e1.build(ents)
    e3.build(ents)
    pr = orc.iteration_probe(w, 555, 2, 4)
    req = orc.request_eams(w, 1, start=777)[0]
    slots = [m.SlotView(i, m.ExpertId(i % 12, (7 * i) % 64), i % 5 == 0, i % 7 == 0)
             for i in range(40)]
    cur = m.Eam(s, m.EamKind.iteration, counts=pr)
    o1, v1 = m.decide(cur, e1, 4, m.Eam(s, counts=req), slots)
    o3, v3 = m.decide(cur, e3, 4, m.Eam(s, counts=req), slots)
    assert np.array_equal(o1, o3) and v1 == v3
    # snapshots of the sharded collection are byte-identical to the unsharded one's
    p1, p3 = tmp_path / "one.json", tmp_path / "sharded.json"
    e1.save(str(p1))
    e3.save(str(p3))
    assert p1.read_bytes() == p3.read_bytes()
    c3 = e3.copy()
    assert c3.shard_layout()[0] == 3 and c3.size() == P and c3.next_seq() == e3.next_seq()
    probes = orc.request_eams(w, 30, start=2000)
    assert np.array_equal(c3.match_batch(probes), e1.match_batch(probes))
