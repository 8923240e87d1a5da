"""GPU parity at scale and on the paths round 1 left untested (VERDICT r1,
"what's weak" 1-5): the P-sharded matcher's device half (per-shard
moe_eamc_match_device -> moe_match_merge[_device] / ShardedMatcher), the
construction replay at the NL capacity across several blocked-replay blocks,
the step-wise replay fallback (P > 16,384 and L > 64), and prefetch orders
whose candidate count exceeds the one-block ranking.

Everything is compared with the CPU oracle (or the compiled reference,
oracle/_ref) on the same inputs, bitwise.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _matches(t):
    from paper_2401_14361_b200 import _lib
    a = t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)
    return np.ascontiguousarray(a).view(np.uint8).reshape(-1, 24).copy().view(
        _lib.MATCH_DTYPE)[:, 0]


def _replayed_collection(m, orc, L, E, cap, n, seed, dup_every=0):
    """A collection whose slot order is NOT seq order (entries replaced by the
    reference insert rule), plus probes."""
    fam = m.gen_bench_family(seed, L, E, n + 64).copy()
    if dup_every:
        fam[cap::dup_every] = fam[0]  # incoming duplicates of slot 0: exact ties
    ent, seqs, _ = orc.insert_replay(L, E, cap, fam[:n])
    return ent, seqs, fam[n:]


# ------------------------------------------------- P-sharded matching (8e)
@pytest.mark.parametrize("bounds", [(0, 700, 700, 1500, 2000), (0, 1, 999, 2000)])
def test_sharded_match_merge_single_gpu(m, orc, bounds):
    """Shards [b_k, b_k+1) of one collection as separate handles on one GPU
    (one of them empty in the first case, one of size 1 in the second), each
    with its real global seqs and index base; per-shard device matching, then
    the device merge and the host merge.  Cross-shard exact ties (duplicates
    of slot 0 in other shards) must go to the oldest seq (eam.cpp:123-124)."""
    import torch
    from paper_2401_14361_b200 import _lib
    L, E, cap = 12, 64, bounds[-1]
    ent, seqs, probes = _replayed_collection(m, orc, L, E, cap, cap + 900, 41, dup_every=97)
    probes = np.concatenate([ent[[0, 5, cap // 2]], probes])  # self-matches + ties
    Q = len(probes)
    n_parts = len(bounds) - 1
    st = torch.cuda.Stream()
    d_pr = torch.from_numpy(probes.astype(np.uint8)).cuda()
    parts = torch.empty((n_parts * Q, 3), dtype=torch.float64, device="cuda")
    shards = []
    for k in range(n_parts):
        a, b = bounds[k], bounds[k + 1]
        e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, max(b - a, 1))
        if b > a:
            e.append(ent[a:b], seqs[a:b])
        _lib.check(_lib.lib.moe_eamc_set_index_base(e._h, a))
        shards.append(e)
        _lib.check(_lib.lib.moe_eamc_match_device(
            e._h, d_pr.data_ptr(), 1, Q, parts[k * Q:(k + 1) * Q].data_ptr(),
            C.c_void_p(st.cuda_stream)))
    final = torch.empty((Q, 3), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib.moe_match_merge_device(parts.data_ptr(), n_parts, Q, final.data_ptr(),
                                               C.c_void_p(st.cuda_stream)))
    st.synchronize()
    got = _matches(final)
    idx, seq, d, _ = orc.match(ent, seqs, probes)
    assert np.array_equal(got["index"], idx)
    assert np.array_equal(got["seq"], seq)
    assert np.array_equal(got["distance"], d)
    # the host-pointer merge (moe_match_merge) gives the same answer
    hp = _matches(parts)
    hout = np.zeros(Q, _lib.MATCH_DTYPE)
    _lib.check(_lib.lib.moe_match_merge(hp.ctypes.data, n_parts, Q, hout.ctypes.data))
    assert np.array_equal(hout, got)
    # an empty shard reports "none" (index = seq = UINT64_MAX, d = +inf)
    if bounds[1] == bounds[2]:
        p1 = hp[Q:2 * Q]
        assert (p1["index"] == _lib.NONE).all() and np.isinf(p1["distance"]).all()


def test_sharded_matcher_class_single_gpu(m, orc):
    """ShardedMatcher (the product's rank-side object) for every shard of a
    3-way split on one GPU, the collective replaced by an in-process gather
    of the other shards' device results; its merged answer must equal the
    oracle over the whole collection."""
    import torch
    from paper_2401_14361_b200 import _lib
    from paper_2401_14361_b200.sharded import ShardedMatcher, gathered_layout, shard_range
    L, E, P, world = 8, 32, 1203, 3
    ent, seqs, probes = _replayed_collection(m, orc, L, E, P, P + 500, 43, dup_every=53)
    Q = len(probes)
    handles = []
    for r in range(world):
        e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
        handles.append(e)
    mats = []
    d_pr = torch.from_numpy(probes.astype(np.int64)).cuda()
    outs = [torch.empty((Q, 3), dtype=torch.float64, device="cuda") for _ in range(world)]
    st = torch.cuda.Stream()

    def make_gather(r):
        def gather(parts, out):
            for j in range(world):
                if j == r:
                    parts[j * Q:(j + 1) * Q].copy_(out)
                else:
                    _lib.check(_lib.lib.moe_eamc_match_device(
                        handles[j]._h, d_pr.data_ptr(), 8, Q, outs[j].data_ptr(),
                        C.c_void_p(torch.cuda.current_stream().cuda_stream)))
                    parts[j * Q:(j + 1) * Q].copy_(outs[j])
        return gather

    for r in range(world):
        sm = ShardedMatcher(handles[r], r, world, P, gather=make_gather(r))
        a, b = shard_range(P, r, world)
        sm.load_shard(ent[a:b], seqs[a:b])
        mats.append(sm)
    idx, seq, d, _ = orc.match(ent, seqs, probes)
    for r in range(world):
        out = torch.empty((Q, 3), dtype=torch.float64, device="cuda")
        parts = torch.empty(gathered_layout(world, Q), dtype=torch.float64, device="cuda")
        final = torch.empty((Q, 3), dtype=torch.float64, device="cuda")
        res = mats[r].match_device(d_pr, 8, out, parts, final, st)
        st.synchronize()
        got = _matches(res)
        assert np.array_equal(got["index"], idx) and np.array_equal(got["seq"], seq)
        assert np.array_equal(got["distance"], d)
    with pytest.raises(ValueError):
        mats[0].load_shard(ent[:3], seqs[:2])


def test_merge_width_sentinel_poisons_and_matcher_redoes(m, orc):
    """A width sentinel in any part is the merged answer whatever the part
    order; ShardedMatcher.match redoes such probes through the
    synchronous path, which widens the shard, and answers exactly."""
    import torch
    from paper_2401_14361_b200 import _lib
    from paper_2401_14361_b200.sharded import WIDTH_SENTINEL, ShardedMatcher
    Q = 4
    good = np.zeros(Q, _lib.MATCH_DTYPE)
    good["index"], good["seq"], good["distance"] = np.arange(Q), np.arange(Q), 0.25
    bad = good.copy()
    bad["index"][1], bad["seq"][1], bad["distance"][1] = WIDTH_SENTINEL, _lib.NONE, np.nan
    for order in ([good, bad], [bad, good]):
        parts = np.concatenate(order)
        d = torch.from_numpy(parts.view(np.float64).reshape(-1, 3).copy()).cuda()
        out = torch.empty((Q, 3), dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib.moe_match_merge_device(d.data_ptr(), 2, Q, out.data_ptr(), None))
        torch.cuda.synchronize()
        got = _matches(out)
        assert int(got["index"][1]) == WIDTH_SENTINEL and np.isnan(got["distance"][1])
        assert np.array_equal(got["index"][[0, 2, 3]], [0, 2, 3])
    L, E, P = 6, 16, 300
    fam = m.gen_bench_family(44, L, E, P + 6).copy()
    probes = fam[P:].copy()
    probes[2] *= 40  # > 255: the u8 shard cannot represent it on the device path
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
    sm = ShardedMatcher(e, 0, 1, P)
    sm.load_shard(fam[:P], np.arange(P, dtype=np.uint64) * 3 + 1)
    got = sm.match(probes)
    idx, seq, d, _ = orc.match(fam[:P], np.arange(P, dtype=np.uint64) * 3 + 1, probes)
    assert np.array_equal(got["index"], idx) and np.array_equal(got["seq"], seq)
    assert np.array_equal(got["distance"], d)
    assert e.count_bytes() >= 2


# ------------------------------------------------ construction at scale (K7)
def test_nl_replay_at_capacity_multi_block(m, orc, ref):
    """NL shape (L=24, E=128), capacity P=10,000, then 1,100 at-capacity
    inserts: three blocks of the blocked replay (B=512), slots replaced in
    earlier blocks chosen again, and the final slots / entries / seqs equal
    the reference's own Eamc::insert replay (eam.cpp:152-178)."""
    L, E, P, n = 24, 128, 10_000, 1_100
    fam = m.gen_bench_family(3, L, E, P + n)
    inc = fam[P:].copy()
    inc[700:760] = fam[P + 10:P + 70]  # incoming duplicates of entries inserted earlier
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
    e.append(fam[:P].astype(np.uint8), np.arange(P, dtype=np.uint64))
    slots = e.build(inc)
    r = ref.eamc(L, E, 1, 1, P)
    r.fill_bench(3, P)
    want = np.array([r.insert(x) for x in inc], np.int64)
    assert np.array_equal(slots, want)
    ent, seqs = r.entries()
    changed = np.unique(want)
    for i in changed:
        assert e.entry_seq(int(i)) == seqs[i]
        assert np.array_equal(e.entry(int(i)).counts, ent[i])
    assert e.entry_seq(int(np.setdiff1d(np.arange(P), changed)[0])) < P


@pytest.mark.parametrize("L,E,P,n", [(12, 128, 20_000, 300), (70, 8, 300, 500)])
def test_stepwise_replay_fallback(m, orc, L, E, P, n):
    """The per-step replay (P > 16,384, or L > 64), never timed or tested in
    round 1: same slots and seqs as the oracle's sequential insert."""
    fam = m.gen_bench_family(5 + L, L, E, P + n).copy()
    fam[P + 7::41] = fam[3]  # exact duplicates among the incoming EAMs
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
    slots = e.build(fam)
    ent, sq, want = orc.insert_replay(L, E, P, fam)
    assert np.array_equal(slots, want)
    for i in np.unique(want[want >= 0])[:50]:
        assert e.entry_seq(int(i)) == sq[i]
        assert np.array_equal(e.entry(int(i)).counts, ent[i])


# ----------------------------------------------- large prefetch candidate sets
@pytest.mark.parametrize("L,E,P,layer,filt", [
    (40, 512, 60, 0, True),     # 39 * 512 = 19,968 candidates
    (40, 512, 60, 0, False),
    (64, 512, 40, 2, False),    # 61 * 512 = 31,232 candidates (> one block's shared memory)
    (64, 512, 40, 2, True),
])
def test_prefetch_large_candidate_sets(m, orc, L, E, P, layer, filt):
    """prefetch_priorities with (L-l-1)*E beyond the one-block ranking: the
    whole reference order (policy.cpp:106-124), with and without the floor
    filter (engine.cpp:663-668)."""
    fam = m.gen_bench_family(61, L, E, P + 1).copy()
    fam[1:P:3] = fam[0]  # a wide window: many members
    e = m.Eamc(m.ModelShape(L, E, 2), m.Phase.decode, P)
    e.append(fam[:P], np.arange(P, dtype=np.uint64))
    cur = fam[0].copy()
    cur[layer + 1:] = 0
    got = m.prefetch_order(m.Eam(m.ModelShape(L, E, 2), m.EamKind.iteration, counts=cur), e,
                           layer, filt)
    ol, oe, op = orc.prefetch(fam[:P], np.arange(P, dtype=np.uint64), cur, layer, filt)
    assert len(got) == len(ol)
    assert np.array_equal(got["layer_idx"], ol) and np.array_equal(got["expert_idx"], oe)
    assert np.array_equal(got["priority"], op)


# ------------------------------------------- count envelope: u32 storage (A1)
def _ds_request_eams(n, L=59, E=160, k=6, tokens=1_000_000, seed=7):
    """Request-level EAMs of 1M-token DeepSeek-V2 requests (hard
    part 5): every row sums to tokens*k, the hot experts far above 65,535."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, L, E), np.uint64)
    for i in range(n):
        p = rng.dirichlet(np.full(E, 0.3), size=L)
        out[i] = np.stack([rng.multinomial(tokens * k, p[l]) for l in range(L)])
    return out


def test_u32_counts_match_within_prefetch_bitwise(m, orc):
    """1M-token DS request EAMs (counts up to ~10^6) stored as u32: match,
    match_within and prefetch order against the oracle, bitwise; the
    collection widens 1 -> 4 bytes by itself."""
    L, E, P = 59, 160, 40
    ents = _ds_request_eams(P + 4)
    assert ents.max() > 65535 and ents.max() < (1 << 27)
    e = m.Eamc(m.ModelShape(L, E, 6), m.Phase.decode, P)
    e.append(ents[:P], np.arange(P, dtype=np.uint64))
    assert e.count_bytes() == 4
    probes = np.concatenate([ents[P:], ents[:2]])
    got = e.match_batch(probes)
    idx, seq, d, _ = orc.match(ents[:P], np.arange(P, dtype=np.uint64), probes)
    assert np.array_equal(got["index"], idx) and np.array_equal(got["distance"], d)
    # the same probes as u32 arrays ship narrow (probe_bytes 4)
    got32 = e.match_batch(probes.astype(np.uint32))
    assert np.array_equal(got32, got)
    s = m.ModelShape(L, E, 6)
    w = e.match_within(m.Eam(s, counts=probes[0]), 0.01)
    wi, ws, wd = orc.match_within(ents[:P], np.arange(P, dtype=np.uint64), probes[0], 0.01)
    assert [x.index for x in w] == list(wi) and [x.distance for x in w] == list(wd)
    for layer in (0, 30, 57):
        cur = probes[1].copy()
        cur[layer + 1:] = 0
        o = m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=cur), e, layer, True)
        ol, oe, op = orc.prefetch(ents[:P], np.arange(P, dtype=np.uint64), cur, layer, True)
        assert np.array_equal(o["layer_idx"], ol) and np.array_equal(o["expert_idx"], oe)
        assert np.array_equal(o["priority"], op)


def test_u32_counts_construction_and_snapshot(m, orc, tmp_path):
    """Construction replay on a u32 collection (blocked replay, 4-byte rows)
    and a JSON v1 snapshot holding counts > 65,535 round-trips."""
    L, E, cap, n = 12, 128, 60, 260
    fam = m.gen_bench_family(91, L, E, n).copy()
    fam[::4] *= 9000  # up to 288,000 per cell: 4-byte storage
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, cap)
    slots = e.build(fam)
    assert e.count_bytes() == 4
    ent, sq, want = orc.insert_replay(L, E, cap, fam)
    assert np.array_equal(slots, want)
    p = tmp_path / "big.json"
    e.save(str(p))
    e2 = m.Eamc.load(str(p))
    assert e2.count_bytes() == 4 and e2.size() == cap
    for i in (0, cap // 2, cap - 1):
        assert np.array_equal(e2.entry(i).counts, ent[i]) and e2.entry_seq(i) == sq[i]
    probes = fam[:5] * 3
    got = e2.match_batch(probes)
    idx, seq, d, _ = orc.match(ent, sq, probes)
    assert np.array_equal(got["index"], idx) and np.array_equal(got["distance"], d)


def test_overflow_only_past_the_exact_range(m, orc):
    """MOE_ERR_OVERFLOW exactly when a row's sum of squares reaches 2^53
    (where the reference's fp64 sums stop being exact), not before."""
    L, E = 2, 4
    s = m.ModelShape(L, E)
    ok_row = np.array([[67_108_863, 0, 0, 0], [1, 2, 3, 4]], np.uint64)  # (2^26-1)^2 < 2^53
    bad_row = np.array([[94_906_266, 0, 0, 0], [1, 0, 0, 0]], np.uint64)  # > 2^53
    e = m.Eamc(s, m.Phase.decode, 4)
    e.append(np.stack([ok_row, ok_row // 3]), np.arange(2, dtype=np.uint64))
    got = e.match_batch(ok_row[None])
    idx, seq, d, _ = orc.match(np.stack([ok_row, ok_row // 3]), np.arange(2, dtype=np.uint64),
                               ok_row[None])
    assert got["index"][0] == idx[0] and got["distance"][0] == d[0]
    with pytest.raises(m.CountOverflowError):
        e.match_batch(bad_row[None])
    with pytest.raises(m.CountOverflowError):
        e.insert(m.Eam(s, counts=bad_row))
    assert m.eam_distance(m.Eam(s, counts=ok_row), m.Eam(s, counts=ok_row // 3)) == \
        orc.distance(ok_row, ok_row // 3)


# ------------------------------------------ fused decision kernel (K4+K5+K6)
def test_fused_decision_sequence_with_victims(m, orc):
    """moe_decide = ONE cooperative launch (decide.cu): the engine's per-layer
    call sequence (the iteration EAM grows by one row per call, so phase A
    reuses the layer-prefix sums), each call's floor-filtered order and the
    eviction victim over slot views, against the oracle; then an unrelated
    probe (prefix cache miss) and the last layer (no candidates)."""
    from oracle import Workload
    L, E, P = 24, 64, 700
    w = Workload(L, E, 2, n_groups=10, prompt_len=3, decode_len=4, batch_size=2, seed=77)
    ents = orc.request_eams(w, P)
    s = m.ModelShape(L, E, 2)
    e = m.Eamc(s, m.Phase.decode, P)
    e.build(ents)
    req = orc.request_eams(w, 1, start=901)[0]
    slots = [m.SlotView(i, m.ExpertId(i % L, (11 * i) % E), i % 6 == 0, i % 9 == 0)
             for i in range(61)]
    want_v = orc.select_victim(req, [v.slot for v in slots],
                               [v.occupant.layer_idx for v in slots],
                               [v.occupant.expert_idx for v in slots],
                               [int(v.prefetch_protected) for v in slots],
                               [int(v.pinned) for v in slots])
    full = orc.iteration_probe(w, 950, 2, L - 1)
    for layer in list(range(L)) + [5, L - 1]:
        pr = full.copy()
        pr[layer + 1:] = 0
        if layer == 5:
            pr = orc.iteration_probe(w, 951, 3, 5)  # unrelated probe: prefix cache miss
        order, victim = m.decide(m.Eam(s, m.EamKind.iteration, counts=pr), e, layer,
                                 m.Eam(s, counts=req), slots)
        ol, ox, op = orc.prefetch(ents, np.arange(P, dtype=np.uint64), pr, layer, True)
        assert np.array_equal(order["layer_idx"], ol) and np.array_equal(order["expert_idx"], ox)
        assert np.array_equal(order["priority"], op)
        assert (victim if victim is not None else -1) == want_v
    assert len(ol) == 0  # last layer: nothing above it


def test_decision_many_explicit_rows_fallback(m, orc):
    """More explicit probe rows than the fused kernel stages (L = 1,100 > 1,024):
    the row-parallel exact distance pass feeds the kernel's aggregation and
    order phases; same order as the reference."""
    L, E, P = 1100, 4, 50
    fam = m.gen_bench_family(19, L, E, P + 1).copy()
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
    e.append(fam[:P], np.arange(P, dtype=np.uint64))
    for layer, flt in [(1050, True), (1050, False), (3, True)]:
        cur = fam[P].copy()
        cur[layer + 1:] = 0
        got = m.prefetch_order(m.Eam(m.ModelShape(L, E), m.EamKind.iteration, counts=cur), e,
                               layer, flt)
        ol, oe, op = orc.prefetch(fam[:P], np.arange(P, dtype=np.uint64), cur, layer, flt)
        assert np.array_equal(got["layer_idx"], ol) and np.array_equal(got["expert_idx"], oe)
        assert np.array_equal(got["priority"], op)
