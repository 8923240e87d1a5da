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
