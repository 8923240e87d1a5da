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


WIDTH_SENTINEL = 0xFFFFFFFFFFFFFFFE  # moe_match.index of a probe the device path could not
                                    # represent at its shard's storage width (moe_eamc.h)


class ShardedMatcher:
    """Owns one rank's shard; `match_device` returns the merged global result.

    `gather(parts, out)` is the exchange (default: NCCL/gloo
    all_gather_into_tensor over `group`); it is injectable so one process can
    drive several shards (tests on a single GPU)."""

    def __init__(self, eamc, rank: int, world: int, P_total: int, group=None, gather=None):
        from . import _lib
        self._lib = _lib
        self.eamc, self.rank, self.world, self.group = eamc, rank, world, group
        self.start, self.end = shard_range(P_total, rank, world)
        self._gather = gather
        _lib.check(_lib.lib.moe_eamc_set_index_base(eamc._h, self.start))

    def load_shard(self, counts: np.ndarray, seqs: np.ndarray) -> None:
        """counts = this rank's [end-start][L][E] entries in slot order; seqs =
        their GLOBAL insertion numbers (Eamc::entry_seq, or a snapshot's
        "seq" fields).  Slot order is not seq order once entries have been
        replaced (eam.cpp:164-177), and the (distance, seq) tie-break of
        eam.cpp:123-124 needs the real seqs."""
        seqs = np.ascontiguousarray(seqs, np.uint64)
        if seqs.shape != (self.end - self.start,):
            raise ValueError("load_shard: one global seq per entry of the shard")
        self.eamc.append(counts, seqs)

    def _exchange(self, parts, out):
        if self._gather is not None:
            self._gather(parts, out)
        else:
            import torch.distributed as dist
            dist.all_gather_into_tensor(parts, out, group=self.group)

    def match_device(self, probes, probe_bytes: int, out, parts, final, stream):
        """probes/out/parts/final are torch CUDA tensors; returns `final` ([Q]
        moe_match), stream-ordered on `stream` (the collective included).  A
        probe whose counts exceed some shard's storage width comes back as the
        width sentinel (index WIDTH_SENTINEL, distance NaN) -- k_merge never
        hides it behind another shard's answer; `match` resolves it."""
        import torch
        lib, check = self._lib.lib, self._lib.check
        Q = out.shape[0]
        with torch.cuda.stream(stream):
            sp = C.c_void_p(stream.cuda_stream)
            check(lib.moe_eamc_match_device(self.eamc._h, probes.data_ptr(), probe_bytes, Q,
                                            out.data_ptr(), sp))
            if self.world == 1:
                return out
            self._exchange(parts, out)
            check(lib.moe_match_merge_device(parts.data_ptr(), self.world, Q, final.data_ptr(),
                                             sp))
        return final

    def match(self, probes_u64: np.ndarray, stream=None) -> np.ndarray:
        """Host-level sharded Eamc::match over [Q][L][E] u64 probes: the device
        pass, then the width-sentinel probes redone through the synchronous
        host path (which widens this rank's shard) and merged again.  Every
        rank sees the same merged result, so every rank takes the same redo."""
        import torch
        from ._lib import MATCH_DTYPE
        probes_u64 = np.ascontiguousarray(probes_u64, np.uint64)
        Q = probes_u64.shape[0]
        dev = torch.device("cuda", self.eamc.device)
        stream = stream or torch.cuda.Stream(device=dev)
        d_pr = torch.from_numpy(probes_u64.view(np.int64)).to(dev)
        out = torch.empty((Q, MATCH_WORDS), dtype=torch.float64, device=dev)
        parts = torch.empty(gathered_layout(self.world, Q), dtype=torch.float64, device=dev)
        final = torch.empty((Q, MATCH_WORDS), dtype=torch.float64, device=dev)
        res = self.match_device(d_pr, 8, out, parts, final, stream)
        stream.synchronize()
        got = _to_matches(res)
        redo = np.nonzero(got["index"] == WIDTH_SENTINEL)[0]
        if len(redo):
            sub = np.ascontiguousarray(probes_u64[redo])
            mine = np.zeros(len(redo), MATCH_DTYPE)
            self._lib.check(self._lib.lib.moe_eamc_match(self.eamc._h, sub.ctypes.data,
                                                         len(redo), mine.ctypes.data, None))
            if self.world == 1:
                got[redo] = mine
            else:
                o2 = torch.from_numpy(mine.view(np.float64).reshape(-1, MATCH_WORDS)).to(dev)
                p2 = torch.empty(gathered_layout(self.world, len(redo)), dtype=torch.float64,
                                 device=dev)
                f2 = torch.empty_like(o2)
                with torch.cuda.stream(stream):
                    self._exchange(p2, o2)
                    self._lib.check(self._lib.lib.moe_match_merge_device(
                        p2.data_ptr(), self.world, len(redo), f2.data_ptr(),
                        C.c_void_p(stream.cuda_stream)))
                stream.synchronize()
                got[redo] = _to_matches(f2)
        return got


def _to_matches(t) -> np.ndarray:
    from ._lib import MATCH_DTYPE
    a = t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)
    return np.ascontiguousarray(a).view(np.uint8).reshape(-1, 24).copy().view(MATCH_DTYPE)[:, 0]


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
