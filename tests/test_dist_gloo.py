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
