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
