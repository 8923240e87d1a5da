"""P-sharded EAMC matching across ranks.

Rank r of N owns the contiguous global slot range `shard_range(P, r, N)`;
its entries carry their GLOBAL insertion numbers as seqs and report global
indices (`moe_eamc_set_index_base`).  The probe batch is replicated.  Each
rank matches against its shard, the per-rank `moe_match[Q]` results (24 B
per probe) are all-gathered (NCCL over NVLink in production) into a
[N][Q] tensor and merged on the device by `moe_match_merge_device`
(lexicographic (distance, seq) min, eam.cpp:123-124).  The exchange is O(Q)
and independent of P.
"""
from __future__ import annotations

import ctypes as C
from typing import Tuple

import numpy as np

MATCH_WORDS = 3  # moe_match = {u64 index, u64 seq, f64 distance} viewed as 3 x f64/i64


def shard_range(P_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block partition of the global slot range."""
    base, rem = divmod(P_total, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def gathered_layout(world: int, Q: int):
    """All-gather buffer the merge kernel consumes: [n_parts * Q] x 24 B, part-major
    (the concatenation all_gather_into_tensor produces on every backend)."""
    return (world * Q, MATCH_WORDS)


class ShardedMatcher:
    """Owns one rank's shard; `match_device` returns the merged global result."""

    def __init__(self, eamc, rank: int, world: int, P_total: int, group=None):
        from . import _lib
        self._lib = _lib
        self.eamc, self.rank, self.world, self.group = eamc, rank, world, group
        self.start, self.end = shard_range(P_total, rank, world)
        _lib.check(_lib.lib.moe_eamc_set_index_base(eamc._h, self.start))

    def load_shard(self, counts: np.ndarray) -> None:
        """counts = this rank's [end-start][L][E] entries; seqs = global slot numbers."""
        self.eamc.append(counts, np.arange(self.start, self.end, dtype=np.uint64))

    def match_device(self, probes, probe_bytes: int, out, parts, final, stream):
        """probes/out/parts/final are torch CUDA tensors; returns `final` ([Q] moe_match)."""
        import torch.distributed as dist
        lib, check = self._lib.lib, self._lib.check
        Q = out.shape[0]
        sp = C.c_void_p(stream.cuda_stream)
        check(lib.moe_eamc_match_device(self.eamc._h, probes.data_ptr(), probe_bytes, Q,
                                        out.data_ptr(), sp))
        if self.world == 1:
            return out
        dist.all_gather_into_tensor(parts, out, group=self.group)
        check(lib.moe_match_merge_device(parts.data_ptr(), self.world, Q, final.data_ptr(), sp))
        return final


class ShardedDecider:
    """P-sharded prefetch_priorities (SURVEY.md 8e, K4 window aggregate + K5).

    policy.cpp:88-126 over a collection sharded by P, split at its two
    reductions: each rank computes its shard's exact distances and minimum
    (`moe_eamc_window_min_device`), the minimum is MIN-all-reduced (the bits of
    a non-negative double order like the double), each rank aggregates the rows
    > current_layer of its members d <= d_min + window (eam.cpp:143) into u64
    [L][E] (`moe_eamc_window_aggregate_device`), the rows are SUM-all-reduced
    (exact integers, order-independent), and the order is computed from the sum
    (`moe_eamc_prefetch_order_device`).  The result is bit-identical to
    `prefetch_order` on the unsharded collection; the exchange is
    8 + 8*L*E bytes per rank, independent of P.
    """

    def __init__(self, eamc, group=None, stream=None):
        import torch
        from . import _lib
        self._lib, self.eamc, self.group = _lib, eamc, group
        self.dev = torch.device("cuda", eamc.device)
        # one explicit stream for the library calls and the collectives (the
        # legacy default stream would be read as "the handle's stream")
        self.stream = stream or torch.cuda.Stream(device=self.dev)
        L, E = eamc.shape.n_layers, eamc.shape.n_experts_per_layer
        self.L, self.E = L, E
        self._dmin = torch.empty(1, dtype=torch.int64, device=self.dev)
        self._agg = torch.empty(L * E, dtype=torch.int64, device=self.dev)
        self._out = torch.empty((max(L * E, 1), 2), dtype=torch.float64, device=self.dev)
        self._n = torch.zeros(1, dtype=torch.int32, device=self.dev)

    def prefetch_order(self, cur_eam_counts: np.ndarray, current_layer: int,
                       apply_floor_filter: bool = True, window: float = 0.01) -> np.ndarray:
        import torch
        import torch.distributed as dist
        lib, check = self._lib.lib, self._lib.check
        cur = np.ascontiguousarray(cur_eam_counts, np.uint64).reshape(self.L, self.E)
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        h = self.eamc._h
        with torch.cuda.stream(self.stream):
            sp = C.c_void_p(self.stream.cuda_stream)
            check(lib.moe_eamc_window_min_device(h, cur.ctypes.data, self._dmin.data_ptr(), sp))
            if world > 1:
                dist.all_reduce(self._dmin, op=dist.ReduceOp.MIN, group=self.group)
            check(lib.moe_eamc_window_aggregate_device(h, current_layer, window,
                                                       self._dmin.data_ptr(),
                                                       self._agg.data_ptr(), sp))
            if world > 1:
                dist.all_reduce(self._agg, op=dist.ReduceOp.SUM, group=self.group)
            check(lib.moe_eamc_prefetch_order_device(h, self._agg.data_ptr(), current_layer,
                                                     int(apply_floor_filter),
                                                     self._out.data_ptr(),
                                                     self._n.data_ptr(), sp))
            n = int(self._n.item())
            out = self._out[:n].cpu().numpy()
        return out.view(np.uint8).reshape(n, 16).copy().view(self._lib.CAND_DTYPE)[:, 0]
