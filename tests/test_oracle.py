"""CPU: the oracle (oracle/eamc_oracle.c, workload_oracle.c) pinned against
golden vectors produced by the reference library itself (oracle/make_golden.py)
and, when oracle/_ref is built, against the live reference."""
import numpy as np
import pytest

from oracle import Workload


def test_distance_golden(orc, golden):
    g = golden("distance.npz")
    oa = ob = 0
    for i, (L, E) in enumerate(g["shapes"]):
        n = int(L) * int(E)
        a = g["a"][oa:oa + n].reshape(L, E)
        b = g["b"][ob:ob + n].reshape(L, E)
        oa += n
        ob += n
        d = orc.distance(a, b)
        assert d == g["d"][i], (i, d, g["d"][i])  # bitwise
    # known answers (test_eam.cpp:170-225)
    assert g["d"][0] == 0.5
    assert g["d"][1] == 0.0 and g["d"][2] == 0.0 and g["d"][3] == 0.0
    assert g["d"][4] == 0.5


def test_bench_checksum_golden(orc, golden):
    for P, L, E, Q, seed, ck in golden("bench_checksum.npz")["rows"]:
        P, L, E, Q, seed = int(P), int(L), int(E), int(Q), int(seed)
        fam = orc.bench_family(seed, L, E, P + Q)
        idx, _, _, found = orc.match(fam[:P], np.arange(P, dtype=np.uint64), fam[P:])
        assert found.all()
        assert int((idx + 1).sum()) == int(ck)


def test_match_golden(orc, golden):
    g = golden("match_mix.npz")
    P, L, E, Q, seed = (int(x) for x in g["params"])
    fam = orc.bench_family(seed, L, E, P + Q)
    seqs = np.arange(P, dtype=np.uint64)
    idx, seq, d, _ = orc.match(fam[:P], seqs, fam[P:])
    assert np.array_equal(idx, g["idx"]) and np.array_equal(seq, g["seq"])
    assert np.array_equal(d, g["d"])
    o = 0
    for q in range(len(g["w_n"])):
        n = int(g["w_n"][q])
        wi, ws, wd = orc.match_within(fam[:P], seqs, fam[P + q], 0.01)
        assert np.array_equal(wi, g["w_idx"][o:o + n])
        assert np.array_equal(ws, g["w_seq"][o:o + n])
        assert np.array_equal(wd, g["w_d"][o:o + n])
        o += n


def test_insert_replay_golden(orc, golden):
    g = golden("insert_replay.npz")
    ent, seqs, slots = orc.insert_replay(2, 4, 10, g["eams"])
    assert np.array_equal(slots, g["slots"])
    assert np.array_equal(ent, g["entries"]) and np.array_equal(seqs, g["seqs"])
    # documented example: newcomer nearest EAM3 evicts slot 2 (test_eam.cpp:273-292)
    _, _, s = orc.insert_replay(1, 4, 3, g["ex"])
    assert list(s) == [-1, -1, -1, 2] == list(g["ex_slots"])


def test_prefetch_golden(orc, golden):
    g = golden("prefetch.npz")
    ent = np.array([[[1, 0], [1, 0], [2, 1], [0, 3]]], np.uint64)
    cur = np.array([[1, 0], [1, 0], [0, 0], [0, 0]], np.uint64)
    l, e, p = orc.prefetch(ent, np.zeros(1, np.uint64), cur, 1, False)
    assert np.array_equal(l, g["worked_l"]) and np.array_equal(e, g["worked_e"])
    assert np.array_equal(p, g["worked_p"])
    assert abs(p[0] - 0.500075) < 1e-12  # test_policy.cpp:46-65
    ents = g["f2_entries"]
    seqs = np.arange(len(ents), dtype=np.uint64)
    o = 0
    for i in range(len(g["f2_n"])):
        n = int(g["f2_n"][i])
        l, e, p = orc.prefetch(ents, seqs, g["f2_probes"][i], int(g["f2_layers"][i]),
                               bool(g["f2_filter"][i]))
        assert np.array_equal(l, g["f2_l"][o:o + n])
        assert np.array_equal(e, g["f2_e"][o:o + n])
        assert np.array_equal(p, g["f2_p"][o:o + n])
        o += n


def test_eviction_golden(orc, golden):
    g = golden("eviction.npz")
    for req, v, want in zip(g["reqs"], g["views"], g["victims"]):
        got = orc.select_victim(req, v[0], v[1], v[2], v[3], v[4])
        assert got == want
    cp = [orc.cache_priority(g["cp_req"], 0, 1), orc.cache_priority(g["cp_req"], 1, 0),
          orc.cache_priority(g["cp_req"], 2, 1)]
    assert cp == list(g["cp"])
    assert abs(cp[0] - 0.7501) < 1e-12  # test_policy.cpp:164-175


def test_trace_generator_golden(orc, golden):
    g = golden("traces.npz")
    cases = {"sw": Workload(12, 64, 1, seed=1001), "mix": Workload(32, 8, 2, seed=99),
             "ds": Workload(59, 160, 6, n_groups=8, prompt_len=6, decode_len=3, batch_size=2,
                            seed=5)}
    for name, w in cases.items():
        for i in range(3):
            counts, picks = orc.trace_picks(w, i)
            assert np.array_equal(counts, g[name][i])
            # the raw picks re-aggregate to the same counts (K1 semantics)
            p = w.params
            offs = np.array([0, picks.shape[0]], np.uint64)
            rc, tot = orc.trace(p["L"], p["E"], p["top_k"], picks, offs)
            assert rc == 0
            assert np.array_equal(tot[0], counts.sum(axis=0))
    cap = g["cap"]
    assert [orc.capacity_bound(12, 128, 0.75), orc.capacity_bound(12, 128, 0.98),
            orc.capacity_bound(1, 1, 0.75), orc.capacity_bound(2, 2, 0.9)] == list(cap)
    assert list(cap[:3]) == [3072, 5635, 2]


def test_trace_all_or_nothing(orc):
    picks = np.array([[[0, 1]], [[1, 5]]], np.uint32)  # expert 5 out of range for E=4
    rc, out = orc.trace(1, 4, 2, picks, np.array([0, 2], np.uint64))
    assert rc == -1 and not out.any()


# ---- live reference (only where oracle/_ref was built) ---------------------
def test_oracle_vs_live_reference(orc, ref):
    rng = orc.rng(4242)
    for _ in range(200):
        a = orc.random_eam(rng, 4, 6)
        b = orc.random_eam(rng, 4, 6)
        assert orc.distance(a, b) == ref.distance(a, b)
    fam = orc.bench_family(9, 12, 128, 330)
    e = ref.eamc(12, 128, 1, 1, 300)
    for x in fam[:300]:
        e.insert(x)
    idx, seq, d, _ = e.match(fam[300:])
    oi, os_, od, _ = orc.match(fam[:300], np.arange(300, dtype=np.uint64), fam[300:])
    assert np.array_equal(idx, oi) and np.array_equal(d, od)


def test_workload_vs_live_reference(orc, ref):
    w = Workload(24, 128, 2, seed=77)
    for i in range(2):
        counts, _ = orc.trace_picks(w, i)
        assert np.array_equal(counts, ref.trace_counts(w, i))
