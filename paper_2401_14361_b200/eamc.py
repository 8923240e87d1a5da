"""Python mirror of the reference's EAM/EAMC/policy API over libmoe_eamc.

Names, argument meaning and error behaviour follow moesim's C++ API
(proj/core/include/moesim/eam.hpp, policy.hpp, model.hpp) so that parity
tests read like the reference's own tests:

  reference (C++)                          here
  ---------------------------------------  -----------------------------------
  ModelShape / ExpertId (model.hpp:19-41)  ModelShape / ExpertId
  Eam (eam.hpp:25-56)                      Eam (host value type, u64 counts)
  eam_distance (eam.hpp:61)                eam_distance           [GPU]
  Eamc (eam.hpp:76-116)                    Eamc (device-resident) [GPU]
  prefetch_priorities (policy.hpp:87)      prefetch_priorities    [GPU]
  cache_priority (policy.hpp:93)           cache_priority         [GPU]
  select_eviction_victim (policy.hpp:105)  select_eviction_victim [GPU]
  TransferQueue (policy.hpp:55-80)         TransferQueue (host, as in the reference)
  eamc_capacity_bound (eam.hpp:121)        eamc_capacity_bound
  std::invalid_argument / out_of_range     ValueError / IndexError

`Eam` stays a host value type like the reference's (record/accumulate/set
are bookkeeping on one L x E matrix); the batched tracer that turns router
top-k ids into count matrices is `trace_requests` (GPU kernel K1).
"""
from __future__ import annotations

import ctypes as C
import os
import dataclasses
import enum
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import (CAND_DTYPE, MATCH_DTYPE, NONE, SLOT_DTYPE, CountOverflowError, CudaError,
                   TraceIngestError,
                   EamcSnapshotError, check, lib, ptr)

kEpsilon = 1e-4          # policy.hpp:22
kMaxPriority = float("inf")  # policy.hpp:26
kMatchWindow = 0.01      # policy.hpp:30


class EamKind(enum.IntEnum):
    iteration = 0
    request = 1


class Phase(enum.IntEnum):
    prefill = 0
    decode = 1


@dataclasses.dataclass(frozen=True)
class ModelShape:
    """model.hpp:19-29"""
    n_layers: int
    n_experts_per_layer: int
    top_k: int = 1

    def validate(self) -> None:  # model.cpp:13-19
        if self.n_layers < 1:
            raise ValueError("ModelShape: n_layers must be >= 1")
        if self.n_experts_per_layer < 1:
            raise ValueError("ModelShape: n_experts_per_layer must be >= 1")
        if self.top_k < 1 or self.top_k > self.n_experts_per_layer:
            raise ValueError("ModelShape: top_k must be in [1, n_experts_per_layer]")

    def total_experts(self) -> int:
        return self.n_layers * self.n_experts_per_layer

    def c(self) -> _lib.moe_shape:
        return _lib.moe_shape(self.n_layers, self.n_experts_per_layer, self.top_k)


@dataclasses.dataclass(frozen=True, order=True)
class ExpertId:
    """model.hpp:33-41 (lexicographic order is the tie-breaker everywhere)"""
    layer_idx: int = 0
    expert_idx: int = 0

    def flat(self, shape: ModelShape) -> int:
        return self.layer_idx * shape.n_experts_per_layer + self.expert_idx


@dataclasses.dataclass
class RoutingEvent:
    """model.hpp:50-54: assignments are (expert_idx, token_count) pairs."""
    layer_idx: int
    assignments: List[Tuple[int, int]]


class Eam:
    """Expert Activation Matrix (eam.hpp:25-56): L x E uint64 counts."""

    def __init__(self, shape: ModelShape, kind: EamKind = EamKind.request,
                 phase: Phase = Phase.decode, counts=None):
        shape.validate()
        self.shape = shape
        self.kind = EamKind(kind)
        self.phase = Phase(phase)
        if counts is None:
            self.counts = np.zeros((shape.n_layers, shape.n_experts_per_layer), np.uint64)
        else:
            self.counts = np.array(counts, dtype=np.uint64).reshape(
                shape.n_layers, shape.n_experts_per_layer)

    def at(self, layer: int, expert: int) -> int:
        return int(self.counts[layer, expert])

    def row_sum(self, layer: int) -> int:
        return int(self.counts[layer].sum())

    def row(self, layer: int) -> np.ndarray:
        return self.counts[layer]

    def set(self, layer: int, expert: int, count: int) -> None:  # eam.cpp:64-68
        if not (0 <= layer < self.shape.n_layers and 0 <= expert < self.shape.n_experts_per_layer):
            raise IndexError("Eam::set: index out of range")
        self.counts[layer, expert] = count

    def record(self, event: RoutingEvent) -> None:
        """eam.cpp:41-52: validate every index, then add (no partial writes)."""
        if not 0 <= event.layer_idx < self.shape.n_layers:
            raise IndexError("Eam::record: layer index out of range")
        for e, _ in event.assignments:
            if not 0 <= e < self.shape.n_experts_per_layer:
                raise IndexError("Eam::record: expert index out of range")
        for e, t in event.assignments:
            self.counts[event.layer_idx, e] += np.uint64(t)

    def accumulate(self, other: "Eam") -> None:  # eam.cpp:54-60
        if self.shape != other.shape:
            raise ValueError("Eam::accumulate: shape mismatch")
        if self.phase != other.phase:
            raise ValueError("Eam::accumulate: phase mismatch")
        self.counts += other.counts

    def reset(self) -> None:
        self.counts[:] = 0

    def copy(self) -> "Eam":
        return Eam(self.shape, self.kind, self.phase, self.counts.copy())

    def __eq__(self, other) -> bool:  # eam.hpp:49 (defaulted ==)
        return (isinstance(other, Eam) and self.shape == other.shape and self.kind == other.kind
                and self.phase == other.phase and np.array_equal(self.counts, other.counts))

    def _buf(self) -> np.ndarray:
        return np.ascontiguousarray(self.counts, np.uint64)


def eam_distance(a: Eam, b: Eam) -> float:
    """eam.cpp:91-104, evaluated on the GPU."""
    if a.shape != b.shape:
        raise ValueError("eam_distance: shape mismatch")
    out = C.c_double()
    sh = a.shape.c()
    check(lib.moe_eam_distance(C.byref(sh), ptr(a._buf()), ptr(b._buf()), C.byref(out)))
    return out.value


@dataclasses.dataclass
class EamcMatch:
    """eam.hpp:67-71"""
    index: int
    seq: int
    distance: float


class Eamc:
    """Fixed-capacity, device-resident collection (eam.hpp:76-116)."""

    def __init__(self, shape: ModelShape, phase: Phase = Phase.decode, capacity: int = 1,
                 device: int = 0, count_bytes: int = 0, _handle=None):
        self.shape = shape
        self._h = C.c_void_p()
        if _handle is not None:
            self._h = _handle
        else:
            sh = shape.c()
            check(lib.moe_eamc_create(C.byref(sh), int(phase), capacity, count_bytes, device,
                                      C.byref(self._h)))
        self.device = device

    @classmethod
    def sharded(cls, shape: ModelShape, phase: Phase = Phase.decode, capacity: int = 1,
                device_ids: Sequence[int] = (0,), count_bytes: int = 0) -> "Eamc":
        """A P-sharded collection with the unsharded Eamc semantics:
        shard s on device_ids[s] (ids may repeat), contiguous global slot ranges,
        NCCL collectives when every shard has its own GPU
        (moe_eamc_create_sharded)."""
        h = C.c_void_p()
        ids = (C.c_int * len(device_ids))(*device_ids)
        sh = shape.c()
        check(lib.moe_eamc_create_sharded(C.byref(sh), int(phase), capacity, count_bytes,
                                          len(device_ids), ids, C.byref(h)))
        return cls(shape, phase, capacity, device=device_ids[0], _handle=h)

    def shard_layout(self) -> Tuple[int, bool]:
        """(number of shards, whether NCCL carries the collectives)."""
        n, nccl = C.c_int(), C.c_int()
        check(lib.moe_eamc_shard_layout(self._h, C.byref(n), C.byref(nccl)))
        return n.value, bool(nccl.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.moe_eamc_destroy(h)
            self._h = C.c_void_p()

    def copy(self) -> "Eamc":
        """Deep copy (the reference's implicit copy constructor): same slots,
        seqs and next_seq, a new device collection."""
        h = C.c_void_p()
        check(lib.moe_eamc_clone(self._h, C.byref(h)))
        return Eamc(self.shape, device=self.device, _handle=h)

    __copy__ = copy

    def __deepcopy__(self, memo):
        return self.copy()

    # -- accessors (eam.hpp:80-87) -------------------------------------
    def _info(self):
        sh = _lib.moe_shape()
        ph = C.c_int()
        cap = C.c_uint64()
        size = C.c_uint64()
        nxt = C.c_uint64()
        cb = C.c_int()
        check(lib.moe_eamc_info(self._h, C.byref(sh), C.byref(ph), C.byref(cap), C.byref(size),
                                C.byref(nxt), C.byref(cb)))
        return sh, ph.value, cap.value, size.value, nxt.value, cb.value

    def phase(self) -> Phase:
        return Phase(self._info()[1])

    def capacity(self) -> int:
        return self._info()[2]

    def size(self) -> int:
        return self._info()[3]

    def empty(self) -> bool:
        return self.size() == 0

    def next_seq(self) -> int:
        return self._info()[4]

    def count_bytes(self) -> int:
        return self._info()[5]

    def entry(self, index: int) -> Eam:
        out = np.zeros((self.shape.n_layers, self.shape.n_experts_per_layer), np.uint64)
        seq = C.c_uint64()
        check(lib.moe_eamc_entry(self._h, index, ptr(out), C.byref(seq)))
        return Eam(self.shape, EamKind.request, self.phase(), out)

    def entry_seq(self, index: int) -> int:
        seq = C.c_uint64()
        check(lib.moe_eamc_entry(self._h, index, None, C.byref(seq)))
        return seq.value

    # -- construction ---------------------------------------------------
    def insert(self, eam: Eam) -> Optional[Eam]:
        """eam.cpp:152-178: returns the evicted entry when full."""
        if eam.shape != self.shape:
            raise ValueError("Eamc::insert: shape mismatch")
        slot = C.c_int64()
        ev = np.zeros((self.shape.n_layers, self.shape.n_experts_per_layer), np.uint64)
        check(lib.moe_eamc_insert(self._h, ptr(eam._buf()), int(eam.kind), int(eam.phase),
                                  C.byref(slot), ptr(ev)))
        if slot.value < 0:
            return None
        return Eam(self.shape, EamKind.request, self.phase(), ev)

    def build(self, counts: np.ndarray) -> np.ndarray:
        """Batched construction: n sequential inserts; returns evicted slots (-1 = appended)."""
        counts = np.ascontiguousarray(counts, np.uint64)
        n = counts.shape[0]
        slots = np.zeros(max(n, 1), np.int64)
        check(lib.moe_eamc_build(self._h, ptr(counts), n, ptr(slots)))
        return slots[:n]

    def build_clustered(self, counts: np.ndarray, iterations: int = 5):
        """Clustering construction (opt-in, parity-unpinned; moe_eamc_build_clustered):
        iteration 0 = build(counts), then k-medoids-style refinement.  Returns
        (objective per iteration, input index of every slot's EAM, iterations run)."""
        counts = np.ascontiguousarray(counts, np.uint64)
        n = counts.shape[0]
        obj = np.zeros(iterations + 1, np.float64)
        rep = np.zeros(max(self.capacity(), 1), np.uint64)
        it = C.c_uint32()
        check(lib.moe_eamc_build_clustered(self._h, ptr(counts), n, iterations, ptr(obj), ptr(rep),
                                           C.byref(it)))
        return obj, rep[:self.size()], it.value

    def build_from_traces(self, trace_path: str) -> int:
        """`moesim eamc save` minus the write (moesim_main.cpp:203-221): the request
        EAMs of this collection's phase, from a JSONL trace file, inserted in file
        order.  Returns the number inserted; raises TraceIngestError on a bad line."""
        n = C.c_uint64()
        check(lib.moe_eamc_build_from_traces(self._h, os.fsencode(trace_path), C.byref(n)))
        return n.value

    def append(self, counts: np.ndarray, seqs: np.ndarray) -> None:
        """Bulk load with caller-assigned seqs (snapshot / shard semantics)."""
        seqs = np.ascontiguousarray(seqs, np.uint64)
        counts = np.ascontiguousarray(counts)
        if counts.dtype == np.uint64:
            check(lib.moe_eamc_append(self._h, ptr(counts), ptr(seqs), len(seqs)))
        else:
            check(lib.moe_eamc_append_packed(self._h, ptr(counts), counts.dtype.itemsize,
                                             ptr(seqs), len(seqs)))

    # -- matching ---------------------------------------------------------
    def match_batch(self, probes: np.ndarray) -> np.ndarray:
        """Eamc::match over [Q][L][E] probes -> structured array (index, seq, distance)."""
        narrow = isinstance(probes, np.ndarray) and probes.dtype in (np.uint8, np.uint16,
                                                                     np.uint32)
        probes = np.ascontiguousarray(probes, probes.dtype if narrow else np.uint64)
        if probes.shape[1:] != (self.shape.n_layers, self.shape.n_experts_per_layer):
            raise ValueError("Eamc: probe shape mismatch")
        Q = probes.shape[0]
        out = np.zeros(max(Q, 1), MATCH_DTYPE)
        if narrow:  # u8/u16/u32 counts: shipped narrow (moe_eamc_match_packed)
            check(lib.moe_eamc_match_packed(self._h, ptr(probes), probes.dtype.itemsize, Q,
                                            ptr(out), None))
        else:
            check(lib.moe_eamc_match(self._h, ptr(probes), Q, ptr(out), None))
        return out[:Q]

    def match(self, probe: Eam) -> Optional[EamcMatch]:
        """eam.cpp:118-129"""
        if probe.shape != self.shape:
            raise ValueError("Eamc: probe shape mismatch")
        m = self.match_batch(probe.counts[None])[0]
        if int(m["index"]) == NONE:
            return None
        return EamcMatch(int(m["index"]), int(m["seq"]), float(m["distance"]))

    def match_within(self, probe: Eam, window: float) -> List[EamcMatch]:
        """eam.cpp:131-150"""
        if probe.shape != self.shape:
            raise ValueError("Eamc: probe shape mismatch")
        cap = max(self.size(), 1)
        out = np.zeros(cap, MATCH_DTYPE)
        n = C.c_uint64()
        check(lib.moe_eamc_match_within(self._h, ptr(probe._buf()), window, ptr(out), cap,
                                        C.byref(n)))
        return [EamcMatch(int(m["index"]), int(m["seq"]), float(m["distance"]))
                for m in out[:n.value]]

    # -- snapshots (eam.cpp:184-256) ------------------------------------
    def save(self, path: str) -> None:
        check(lib.moe_eamc_save(self._h, str(path).encode()))

    def save_binary(self, path: str) -> None:
        """The binary snapshot fast path (load() reads either format)."""
        check(lib.moe_eamc_save_binary(self._h, str(path).encode()))

    @staticmethod
    def load(path: str, expected: Optional[ModelShape] = None, device: int = 0) -> "Eamc":
        h = C.c_void_p()
        sh = expected.c() if expected is not None else None
        check(lib.moe_eamc_load(str(path).encode(), C.byref(sh) if sh is not None else None,
                                device, C.byref(h)))
        s = _lib.moe_shape()
        check(lib.moe_eamc_info(h, C.byref(s), None, None, None, None, None))
        return Eamc(ModelShape(s.n_layers, s.n_experts_per_layer, s.top_k), _handle=h,
                    device=device)


@dataclasses.dataclass
class PrefetchCandidate:
    """policy.hpp:46-50"""
    expert: ExpertId
    priority: float


def _cands(arr: np.ndarray) -> List[PrefetchCandidate]:
    return [PrefetchCandidate(ExpertId(int(c["layer_idx"]), int(c["expert_idx"])),
                              float(c["priority"])) for c in arr]


def _check_decision_probe(cur_eam: Eam, eamc: Eamc, current_layer: int) -> bool:
    """policy.cpp:90-95 validation order: current_layer against the probe's
    own shape (out_of_range), an empty collection answers {} (returns False),
    then Eamc::check_probe (eam.cpp:113-116, invalid_argument) -- which also
    keeps the C side from reading a probe of the wrong size."""
    if current_layer < 0 or current_layer >= cur_eam.shape.n_layers:
        raise IndexError("prefetch_priorities: current_layer out of range")
    if eamc.size() == 0:
        return False
    if cur_eam.shape != eamc.shape:
        raise ValueError("Eamc: probe shape mismatch")
    return True


def prefetch_priorities(cur_eam: Eam, eamc: Eamc, current_layer: int,
                        apply_floor_filter: bool = False) -> List[PrefetchCandidate]:
    """policy.cpp:88-126 (+ the engine floor filter, engine.cpp:663-668)."""
    if not _check_decision_probe(cur_eam, eamc, current_layer):
        return []
    cap = max(cur_eam.shape.total_experts(), 1)
    out = np.zeros(cap, CAND_DTYPE)
    n = C.c_uint64()
    check(lib.moe_prefetch_priorities(eamc._h, ptr(cur_eam._buf()), current_layer,
                                      int(apply_floor_filter), ptr(out), cap, C.byref(n)))
    return _cands(out[:n.value])


def prefetch_order(cur_eam: Eam, eamc: Eamc, current_layer: int,
                   apply_floor_filter: bool = True) -> np.ndarray:
    """Same as prefetch_priorities, as a structured array (layer, expert, priority)."""
    if not _check_decision_probe(cur_eam, eamc, current_layer):
        return np.zeros(0, CAND_DTYPE)
    cap = max(cur_eam.shape.total_experts(), 1)
    out = np.zeros(cap, CAND_DTYPE)
    n = C.c_uint64()
    check(lib.moe_prefetch_priorities(eamc._h, ptr(cur_eam._buf()), current_layer,
                                      int(apply_floor_filter), ptr(out), cap, C.byref(n)))
    return out[:n.value]


def cache_priority(request_eam: Eam, expert: ExpertId) -> float:
    """policy.cpp:128-141"""
    out = C.c_double()
    sh = request_eam.shape.c()
    if expert.layer_idx < 0 or expert.expert_idx < 0:
        raise IndexError("cache_priority: expert out of range")
    check(lib.moe_cache_priority(C.byref(sh), ptr(request_eam._buf()), expert.layer_idx,
                                 expert.expert_idx, C.byref(out)))
    return out.value


@dataclasses.dataclass
class SlotView:
    """policy.hpp:96-101"""
    slot: int
    occupant: ExpertId
    prefetch_protected: bool = False
    pinned: bool = False


def _slot_array(slots: Sequence[SlotView]) -> np.ndarray:
    a = np.zeros(max(len(slots), 1), SLOT_DTYPE)
    for i, s in enumerate(slots):
        a[i]["slot"] = s.slot
        a[i]["layer_idx"] = s.occupant.layer_idx
        a[i]["expert_idx"] = s.occupant.expert_idx
        a[i]["prefetch_protected"] = int(s.prefetch_protected)
        a[i]["pinned"] = int(s.pinned)
    return a


def select_eviction_victim(slots: Sequence[SlotView], request_eam: Eam) -> Optional[int]:
    """policy.cpp:143-159"""
    a = _slot_array(slots)
    v = C.c_int64()
    sh = request_eam.shape.c()
    check(lib.moe_select_eviction_victim(C.byref(sh), ptr(request_eam._buf()), ptr(a), len(slots),
                                         C.byref(v)))
    return None if v.value < 0 else int(v.value)


def decide(cur_eam: Eam, eamc: Eamc, current_layer: int, request_eam: Eam,
           slots: Sequence[SlotView]) -> Tuple[np.ndarray, Optional[int]]:
    """Fused K5+K6: floor-filtered prefetch order and eviction victim in one launch."""
    if current_layer < 0 or current_layer >= cur_eam.shape.n_layers:
        raise IndexError("prefetch_priorities: current_layer out of range")
    if cur_eam.shape != eamc.shape:
        raise ValueError("Eamc: probe shape mismatch")
    if (request_eam.shape.n_layers, request_eam.shape.n_experts_per_layer) != (
            eamc.shape.n_layers, eamc.shape.n_experts_per_layer):
        raise ValueError("decide: request EAM shape does not match the collection")
    a = _slot_array(slots)
    cap = max(cur_eam.shape.total_experts(), 1)
    out = np.zeros(cap, CAND_DTYPE)
    n = C.c_uint64()
    v = C.c_int64()
    check(lib.moe_decide(eamc._h, ptr(cur_eam._buf()), current_layer, ptr(request_eam._buf()),
                         ptr(a), len(slots), ptr(out), cap, C.byref(n), C.byref(v)))
    return out[:n.value], (None if v.value < 0 else int(v.value))


def eamc_capacity_bound(shape: ModelShape, similarity: float) -> int:
    """eam.cpp:258-268"""
    out = C.c_uint64()
    sh = shape.c()
    check(lib.moe_eamc_capacity_bound(C.byref(sh), similarity, C.byref(out)))
    return out.value


def trace_requests(shape: ModelShape, topk_idx: np.ndarray, offsets: np.ndarray,
                   counts: Optional[np.ndarray] = None) -> np.ndarray:
    """K1: router top-k ids [T][L][k] -> per-request L x E counts (accumulated into
    `counts` when given).  All-or-nothing like Eam::record (eam.cpp:41-52)."""
    topk_idx = np.ascontiguousarray(topk_idx)
    if topk_idx.dtype not in (np.uint8, np.uint16, np.uint32, np.int32):
        raise ValueError("topk_idx must be uint8/uint16/uint32/int32")
    offsets = np.ascontiguousarray(offsets, np.uint64)
    R = len(offsets) - 1
    if counts is None:
        counts = np.zeros((max(R, 0), shape.n_layers, shape.n_experts_per_layer), np.uint64)
    counts = np.ascontiguousarray(counts, np.uint64)
    sh = shape.c()
    T = topk_idx.shape[0] if topk_idx.ndim else 0
    check(lib.moe_eam_trace(C.byref(sh), ptr(topk_idx), topk_idx.dtype.itemsize, T, ptr(offsets),
                            R, ptr(counts)))
    return counts


class TransferQueue:
    """policy.cpp:43-86.  Host-side by design: a priority
    queue keyed by expert with overwrite-on-resubmit; pop order is priority
    descending, (layer, expert) ascending."""

    def __init__(self):
        self._by_expert = {}

    def submit(self, expert: ExpertId, priority: float) -> None:
        self._by_expert[expert] = priority

    def cancel(self, expert: ExpertId) -> bool:
        return self._by_expert.pop(expert, None) is not None

    def cancel_all(self) -> int:
        n = len(self._by_expert)
        self._by_expert.clear()
        return n

    def _order(self):
        return sorted(self._by_expert.items(), key=lambda kv: (-kv[1], kv[0]))

    def peek(self) -> Optional[PrefetchCandidate]:
        if not self._by_expert:
            return None
        e, p = self._order()[0]
        return PrefetchCandidate(e, p)

    def pop(self) -> Optional[PrefetchCandidate]:
        top = self.peek()
        if top is not None:
            del self._by_expert[top.expert]
        return top

    def contains(self, expert: ExpertId) -> bool:
        return expert in self._by_expert

    def priority_of(self, expert: ExpertId) -> Optional[float]:
        return self._by_expert.get(expert)

    def size(self) -> int:
        return len(self._by_expert)

    def empty(self) -> bool:
        return not self._by_expert

    def __iter__(self):
        for e, p in self._order():
            yield PrefetchCandidate(e, p)


def ingest_request_eams(trace_path: str, shape: ModelShape, phase: Phase) -> np.ndarray:
    """ingest_traces (workload.cpp:209-232) + request_level_eam
    (moesim_main.cpp:192-201) for one phase: [n][L][E] u64 in file order."""
    sh = shape.c()
    n = C.c_uint64()
    check(lib.moe_traces_request_eams(os.fsencode(trace_path), C.byref(sh), int(phase), None, 0,
                                      C.byref(n)))
    out = np.zeros((max(n.value, 1), shape.n_layers, shape.n_experts_per_layer), np.uint64)
    check(lib.moe_traces_request_eams(os.fsencode(trace_path), C.byref(sh), int(phase),
                                      ptr(out), n.value, C.byref(n)))
    return out[:n.value]


def eamc_save_from_traces(trace_path: str, shape: ModelShape, phase: Phase, capacity: int,
                          out_path: str, device: int = 0) -> "Eamc":
    """`moesim eamc save --trace T --out O` (moesim_main.cpp:203-221)."""
    e = Eamc(shape, phase, capacity, device=device)
    e.build_from_traces(trace_path)
    e.save(out_path)
    return e


class ExpertCache:
    """GPU expert-weight slots filled by chunked DMA in the engine's prefetch
    order (moe_expert_cache_*): the reference's TransferQueue,
    GpuBuffer and contention rules (engine.cpp:306-357, :429-529) over real
    cudaMemcpyAsync of host expert weights ([L][E][expert_bytes] uint8)."""

    def __init__(self, shape: ModelShape, host_weights: np.ndarray, n_slots: int,
                 chunk_bytes: int = 16 << 20, device: int = 0):
        self.shape = shape
        self.weights = np.ascontiguousarray(host_weights, np.uint8)
        L, E = shape.n_layers, shape.n_experts_per_layer
        if self.weights.ndim != 3 or self.weights.shape[:2] != (L, E):
            raise ValueError("host_weights must be [L][E][expert_bytes] uint8")
        self.expert_bytes = self.weights.shape[2]
        self._h = C.c_void_p()
        sh = shape.c()
        check(lib.moe_expert_cache_create(C.byref(sh), self.expert_bytes, n_slots, chunk_bytes,
                                          ptr(self.weights), device, C.byref(self._h)))
        self.n_slots = n_slots

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.moe_expert_cache_destroy(h)
            self._h = C.c_void_p()

    def set_request_eam(self, request_eam: "Eam") -> None:
        check(lib.moe_expert_cache_set_request_eam(self._h, ptr(request_eam._buf())))

    def submit(self, order: np.ndarray) -> None:
        """recompute_prefetch: cancel_all, then the (floor-filtered) order."""
        order = np.ascontiguousarray(order, CAND_DTYPE)
        check(lib.moe_expert_cache_submit(self._h, ptr(order), len(order)))

    def progress(self, wait_idle: bool = False) -> None:
        check(lib.moe_expert_cache_progress(self._h, int(wait_idle)))

    def acquire(self, expert: ExpertId) -> Tuple[int, bool]:
        p = C.c_void_p()
        hit = C.c_int()
        check(lib.moe_expert_cache_acquire(self._h, expert.layer_idx, expert.expert_idx,
                                           C.byref(p), C.byref(hit)))
        return p.value, bool(hit.value)

    def release(self, expert: ExpertId) -> None:
        check(lib.moe_expert_cache_release(self._h, expert.layer_idx, expert.expert_idx))

    def slot(self, i: int) -> dict:
        occ, res, prot, pri = C.c_int64(), C.c_int(), C.c_int(), C.c_double()
        check(lib.moe_expert_cache_slot(self._h, i, C.byref(occ), C.byref(res), C.byref(prot),
                                        C.byref(pri)))
        E = self.shape.n_experts_per_layer
        ex = None if occ.value < 0 else ExpertId(occ.value // E, occ.value % E)
        return {"expert": ex, "residency": res.value, "protected": bool(prot.value),
                "priority": pri.value}

    def read_slot(self, i: int) -> np.ndarray:
        out = np.zeros(self.expert_bytes, np.uint8)
        check(lib.moe_expert_cache_read_slot(self._h, i, ptr(out)))
        return out

    def stats(self) -> dict:
        s = _lib.moe_expert_cache_stats()
        check(lib.moe_expert_cache_stats_get(self._h, C.byref(s)))
        return {n: getattr(s, n) for n, _ in s._fields_}
