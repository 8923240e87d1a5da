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


# ---------------------------------------------------------------- K1 tracing
def request_split(offsets: np.ndarray, rank: int, world: int) -> Tuple[int, int]:
    """Request-owned split of K1: rank r takes the contiguous
    requests [r0, r1) whose token ranges start in its 1/world share of the
    token stream (balanced by tokens, not by request count).  Each rank traces
    its own requests; no collective."""
    offsets = np.asarray(offsets, np.uint64)
    T0, T1 = int(offsets[0]), int(offsets[-1])
    R = len(offsets) - 1

    def cut(k):
        t = T0 + (T1 - T0) * k // world
        return int(np.searchsorted(offsets[:R], t, side="left")) if k < world else R
    return cut(rank), cut(rank + 1)


def token_split(n_tokens: int, offsets: np.ndarray, rank: int, world: int):
    """Token-sharded split of K1: rank r takes tokens [t0, t1) of the stream;
    returns (t0, t1, local_offsets) with every request's range clipped to the
    rank's tokens (requests outside it become empty), so the rank's partial
    histograms sum over ranks to Eam::record over the whole request."""
    base, rem = divmod(n_tokens, world)
    t0 = rank * base + min(rank, rem)
    t1 = t0 + base + (1 if rank < rem else 0)
    off = np.asarray(offsets, np.uint64).astype(np.int64)
    local = np.clip(off - t0, 0, t1 - t0).astype(np.uint64)
    return t0, t1, local


class ShardedTracer:
    """Token-sharded K1 (Eam::record, eam.cpp:41-52, over router top-k ids):
    each rank histograms its token range of every request it intersects into a
    zeroed partial [R][L][E] u32 (moe_eam_trace_device), the out-of-range flag
    is MAX-all-reduced and the partials SUM-all-reduced (exact, order-free
    integer sums; NCCL over NVLink in production), and the sum is added to the
    caller's counts on every rank.  All-or-nothing across ranks (eam.cpp:42-47):
    an out-of-range id on any rank raises IndexError on every rank with the
    counts untouched.  The exchange is R*L*E*4 bytes, independent of T.

    `local`/`allreduce` are injectable so one process can drive several
    ranks' device steps (single-GPU tests) and CPU tests can stand an oracle in
    for the device step."""

    def __init__(self, shape, rank: int, world: int, group=None, local=None, allreduce=None):
        self.shape, self.rank, self.world, self.group = shape, rank, world, group
        self._local = local or self._device_local
        self._allreduce = allreduce or self._dist_allreduce

    def _device_local(self, topk_local, local_offsets, partial, bad, stream):
        """This rank's device step: partial += histograms of its tokens."""
        import torch
        from . import _lib
        sh = self.shape.c()
        with torch.cuda.stream(stream):
            d_off = torch.from_numpy(np.ascontiguousarray(local_offsets).view(np.int64)).to(
                partial.device, non_blocking=False)
            _lib.check(_lib.lib.moe_eam_trace_device(
                C.byref(sh), C.c_void_p(topk_local.data_ptr()), topk_local.element_size(),
                C.c_uint64(topk_local.shape[0]), C.c_void_p(d_off.data_ptr()),
                C.c_uint64(len(local_offsets) - 1), C.c_void_p(partial.data_ptr()),
                C.c_void_p(bad.data_ptr()), C.c_void_p(stream.cuda_stream)))
        return d_off  # kept alive until the stream has used it

    def _dist_allreduce(self, t, op):
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM,
                            group=self.group)

    def trace(self, topk_local, n_tokens: int, offsets: np.ndarray, counts, stream=None):
        """topk_local: this rank's ids [t1-t0][L][k] (token_split); offsets:
        the GLOBAL request offsets; counts: [R][L][E] int32 tensor, accumulated."""
        import torch
        t0, t1, local = token_split(n_tokens, offsets, self.rank, self.world)
        if topk_local.shape[0] != t1 - t0:
            raise ValueError("trace: topk_local must hold this rank's token range")
        stream = stream or (torch.cuda.current_stream(counts.device)
                            if counts.is_cuda else None)
        if counts.is_cuda:  # inputs made on the caller's current stream
            stream.wait_stream(torch.cuda.current_stream(counts.device))
        ctx = torch.cuda.stream(stream) if counts.is_cuda else _null()
        with ctx:
            partial = torch.zeros_like(counts)
            bad = torch.zeros(1, dtype=torch.int32, device=counts.device)
        keep = self._local(topk_local, local, partial, bad, stream)
        with ctx:
            self._allreduce(bad, "max")
            if int(bad.item()):  # some rank saw an id >= E: nobody's counts move
                raise IndexError("Eam::record: expert index out of range")
            self._allreduce(partial, "sum")
            counts += partial
        del keep
        return counts


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
