"""CPU, world size 2 over gloo: the N>1 host logic of the P-sharded matcher.

Each rank owns `shard_range` of a global collection, computes its shard's
argmin with the ORACLE (global seqs, global index base), all-gathers the
24-byte per-probe results in the exact [n_parts][Q][3] layout the device
merge kernel consumes, and merges lexicographically on (distance, seq).  The
merged result must equal the oracle's match over the whole collection.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def merge_lexicographic(parts):
    """[N][Q] structured (index, seq, distance) -> [Q]; the k_merge rule."""
    best = parts[0].copy()
    for k in range(1, parts.shape[0]):
        m = parts[k]
        better = (m["distance"] < best["distance"]) | (
            (m["distance"] == best["distance"]) & (m["seq"] < best["seq"]))
        best[better] = m[better]
    return best


def _worker(rank, world, port, P, Q, L, E, dup, out_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    from paper_2401_14361_b200 import gen_bench_family
    from paper_2401_14361_b200._lib import MATCH_DTYPE
    from paper_2401_14361_b200.sharded import gathered_layout, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    fam = gen_bench_family(7, L, E, P + Q)
    if dup:  # cross-shard exact ties: the globally oldest seq must win
        fam[P - 5:P] = fam[0:5]
        fam[P:P + 5] = fam[0:5]
    s, e = shard_range(P, rank, world)
    idx, seq, d, found = orc.match(fam[s:e], np.arange(s, e, dtype=np.uint64), fam[P:])
    local = np.zeros(Q, MATCH_DTYPE)
    local["index"] = idx + s  # moe_eamc_set_index_base(start)
    local["seq"] = seq
    local["distance"] = d
    mine = torch.from_numpy(local.view(np.float64).reshape(Q, 3).copy())
    parts = torch.empty(gathered_layout(world, Q), dtype=torch.float64)
    dist.all_gather_into_tensor(parts, mine)
    merged = merge_lexicographic(
        parts.numpy().copy().view(MATCH_DTYPE)[..., 0].reshape(world, Q))
    if rank == 0:
        gi, gs, gd, _ = orc.match(fam[:P], np.arange(P, dtype=np.uint64), fam[P:])
        out_q.put((bool(np.array_equal(merged["index"], gi)),
                   bool(np.array_equal(merged["seq"], gs)),
                   bool(np.array_equal(merged["distance"], gd))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("P,dup", [(301, False), (400, True)])
def test_sharded_match_gloo_world2(P, dup):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, P, 24, 12, 64, dup, q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    res = q.get(timeout=10)
    assert res == (True, True, True)


def test_shard_range_partition():
    from paper_2401_14361_b200.sharded import shard_range
    for P in (1, 7, 10_000, 1 << 20):
        for N in (1, 2, 3, 8):
            rs = [shard_range(P, r, N) for r in range(N)]
            assert rs[0][0] == 0 and rs[-1][1] == P
            assert all(rs[i][1] == rs[i + 1][0] for i in range(N - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def _decide_worker(rank, world, port, P, L, E, out_q):
    """The host logic of sharded.ShardedDecider (SURVEY 8e, K4+K5) with the
    per-shard device steps restated by the ORACLE: shard distances and
    minimum -> MIN all-reduce of the double's bits -> members
    d <= d_min + 0.01 (eam.cpp:143) -> u64 rows > layer -> SUM all-reduce ->
    order.  Must equal the oracle's unsharded prefetch_priorities."""
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, Workload
    from paper_2401_14361_b200.sharded import shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    w = Workload(L, E, 2, n_groups=6, prompt_len=3, decode_len=4, batch_size=2, seed=77)
    ents = orc.request_eams(w, P)
    s, e = shard_range(P, rank, world)
    ok = True
    for r, it, layer in [(500, 1, 0), (501, 2, L // 2), (502, 3, L - 2)]:
        probe = orc.iteration_probe(w, r, it, layer)
        _, _, d = orc.match_within(ents[s:e], np.arange(s, e, dtype=np.uint64), probe, 2.0)
        # match_within returns (distance, seq) order; the members are a set
        dall = np.array([orc.distance(ents[i], probe) for i in range(s, e)])
        assert np.array_equal(np.sort(d), np.sort(dall))
        dmin = torch.tensor([np.float64(dall.min()).view(np.int64)], dtype=torch.int64)
        dist.all_reduce(dmin, op=dist.ReduceOp.MIN)
        gmin = dmin.numpy().view(np.float64)[0]
        members = dall <= gmin + 0.01
        agg = np.zeros((L, E), np.int64)
        agg[layer + 1:] = ents[s:e][members][:, layer + 1:].astype(np.int64).sum(0)
        t = torch.from_numpy(agg.reshape(-1).copy())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total = t.numpy().reshape(1, L, E).astype(np.uint64)
        for flt in (True, False):
            got = orc.prefetch(total, np.zeros(1, np.uint64), probe, layer, flt)
            want = orc.prefetch(ents, np.arange(P, dtype=np.uint64), probe, layer, flt)
            ok &= all(np.array_equal(a, b) for a, b in zip(got, want))
    flags = torch.tensor([int(ok)])
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        out_q.put(bool(flags.item()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_decide_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_decide_worker, args=(r, 2, port, 161, 10, 16, q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def _trace_worker(rank, world, port, bad_rank, out_q):
    """sharded.ShardedTracer (token-sharded K1) over gloo, the ORACLE standing
    in for each rank's device step on its clipped token range: MAX all-reduce
    of the range flag, SUM all-reduce of the partials, accumulate.  Must equal
    the oracle's Eam::record over the whole requests; with an out-of-range id
    on one rank, every rank raises and nobody's counts move."""
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, Workload
    from paper_2401_14361_b200.eamc import ModelShape
    from paper_2401_14361_b200.sharded import ShardedTracer, request_split, token_split
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    L, E, k = 12, 32, 2
    w = Workload(L, E, k, n_groups=6, prompt_len=5, decode_len=7, batch_size=3, seed=13)
    picks, offs = [], [0]
    for r in range(9):
        _, pk = orc.trace_picks(w, r)
        picks.append(pk)
        offs.append(offs[-1] + pk.shape[0])
    picks = np.concatenate(picks).astype(np.uint32)
    offs = np.array(offs, np.uint64)
    offs[4] = offs[3]  # an empty request
    T = picks.shape[0]
    if bad_rank >= 0:
        t0b, t1b, _ = token_split(T, offs, bad_rank, world)
        picks[(t0b + t1b) // 2, 3, 1] = E
    rc_all, want = orc.trace(L, E, k, picks, offs)

    def local(topk_local, local_offsets, partial, bad, stream):
        rc, part = orc.trace(L, E, k, np.ascontiguousarray(topk_local), local_offsets)
        if rc != 0:
            bad[0] = 1
        else:
            partial += torch.from_numpy(part.astype(np.int32))

    t0, t1, _ = token_split(T, offs, rank, world)
    tr = ShardedTracer(ModelShape(L, E, k), rank, world, local=local)
    base = torch.full((len(offs) - 1, L, E), 3, dtype=torch.int32)
    counts = base.clone()
    raised = False
    try:
        tr.trace(picks[t0:t1], T, offs, counts)
    except IndexError:
        raised = True
    ok = True
    if bad_rank >= 0:
        ok &= raised and torch.equal(counts, base) and rc_all != 0
    else:
        ok &= (not raised) and np.array_equal(counts.numpy().astype(np.uint64) - 3, want)
        # request-owned split: each rank traces its own requests, no collective
        r0, r1 = request_split(offs, rank, world)
        a, b = int(offs[r0]), int(offs[r1])
        rc, mine = orc.trace(L, E, k, picks[a:b], offs[r0:r1 + 1] - offs[r0])
        ok &= rc == 0 and np.array_equal(mine, want[r0:r1])
        spans = [torch.tensor([r0, r1])]
        gathered = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, spans[0])
        cov = sorted((int(g[0]), int(g[1])) for g in gathered)
        ok &= cov[0][0] == 0 and cov[-1][1] == len(offs) - 1 and all(
            cov[i][1] == cov[i + 1][0] for i in range(world - 1))
    flags = torch.tensor([int(bool(ok))])
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        out_q.put(bool(flags.item()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("bad_rank", [-1, 1])
def test_sharded_trace_gloo_world2(bad_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_trace_worker, args=(r, 2, port, bad_rank, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def test_trace_splits_partition():
    from paper_2401_14361_b200.sharded import request_split, token_split
    offs = np.array([0, 10, 10, 250, 251, 900, 1000], np.uint64)
    for N in (1, 2, 3, 8):
        rs = [request_split(offs, r, N) for r in range(N)]
        assert rs[0][0] == 0 and rs[-1][1] == 6
        assert all(rs[i][1] == rs[i + 1][0] for i in range(N - 1))
        tot = np.zeros(6, np.int64)
        for r in range(N):
            t0, t1, loc = token_split(1000, offs, r, N)
            assert np.all(np.diff(loc.astype(np.int64)) >= 0) and loc[-1] <= t1 - t0
            tot += np.diff(loc.astype(np.int64))
        assert np.array_equal(tot, np.diff(offs.astype(np.int64)))
