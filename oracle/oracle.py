"""ctypes bindings for the CPU ORACLE (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps liboracle.so -- the plain-C restatement of the reference
algorithm (eamc_oracle.c / workload_oracle.c).  `RefLib` wraps
oracle/_ref/libmoesim_ref.so -- the unmodified reference library compiled
from /root/reference sources (oracle/Makefile) behind ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module.  The product package never
does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoesim_ref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


def build_oracle() -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])
    if os.path.isdir("/root/reference/proj"):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


class _Rng(C.Structure):
    _fields_ = [("state", C.c_uint64)]


class _Workload(C.Structure):
    _fields_ = [
        ("L", C.c_uint32), ("E", C.c_uint32), ("top_k", C.c_uint32),
        ("n_groups", C.c_uint32), ("group_fidelity", C.c_double), ("reuse_skew", C.c_double),
        ("prompt_vals", C.POINTER(C.c_uint32)), ("prompt_w", C.POINTER(C.c_double)),
        ("prompt_n", C.c_uint32),
        ("decode_vals", C.POINTER(C.c_uint32)), ("decode_w", C.POINTER(C.c_double)),
        ("decode_n", C.c_uint32),
        ("batch_size", C.c_uint32), ("seed", C.c_uint64),
    ]


class Workload:
    """WorkloadSpec (workload.hpp:33-45) with constant prompt/decode lengths."""

    def __init__(self, L, E, top_k, n_groups=24, group_fidelity=0.9, reuse_skew=1.2,
                 prompt_len=4, decode_len=8, batch_size=8, seed=1001):
        self._pv = (C.c_uint32 * 1)(prompt_len)
        self._pw = (C.c_double * 1)(1.0)
        self._dv = (C.c_uint32 * 1)(decode_len)
        self._dw = (C.c_double * 1)(1.0)
        self.params = dict(L=L, E=E, top_k=top_k, n_groups=n_groups,
                           group_fidelity=group_fidelity, reuse_skew=reuse_skew,
                           prompt_len=prompt_len, decode_len=decode_len,
                           batch_size=batch_size, seed=seed)
        self.c = _Workload(L, E, top_k, n_groups, group_fidelity, reuse_skew,
                           self._pv, self._pw, 1, self._dv, self._dw, 1, batch_size, seed)


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        lib = C.CDLL(path)
        self.lib = lib
        lib.orc_rng_stream.restype = _Rng
        lib.orc_rng_stream.argtypes = [C.c_uint64, C.c_uint64]
        lib.orc_rng_next_u64.restype = C.c_uint64
        lib.orc_rng_next_u64.argtypes = [C.POINTER(_Rng)]
        lib.orc_rng_bounded.restype = C.c_uint64
        lib.orc_rng_bounded.argtypes = [C.POINTER(_Rng), C.c_uint64]
        lib.orc_rng_bernoulli.restype = C.c_int
        lib.orc_rng_bernoulli.argtypes = [C.POINTER(_Rng), C.c_double]
        lib.orc_bench_family.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, u64p]
        lib.orc_random_eam.argtypes = [C.POINTER(_Rng), C.c_uint32, C.c_uint32, u64p]
        lib.orc_eam_distance.restype = C.c_double
        lib.orc_eam_distance.argtypes = [C.c_uint32, C.c_uint32, u64p, u64p]
        lib.orc_match_batch.argtypes = [C.c_uint32, C.c_uint32, u64p, u64p, C.c_uint64, u64p,
                                        C.c_uint64, u64p, u64p, f64p, u8p]
        lib.orc_match_within.restype = C.c_uint64
        lib.orc_match_within.argtypes = [C.c_uint32, C.c_uint32, u64p, u64p, C.c_uint64, u64p,
                                         C.c_double, u64p, u64p, f64p]
        lib.orc_insert.restype = C.c_int64
        lib.orc_insert.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u64p, u64p,
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), u64p]
        lib.orc_prefetch_priorities.restype = C.c_uint64
        lib.orc_prefetch_priorities.argtypes = [C.c_uint32, C.c_uint32, u64p, u64p, C.c_uint64,
                                                u64p, C.c_uint32, C.c_int, u32p, u32p, f64p]
        lib.orc_cache_priority.restype = C.c_double
        lib.orc_cache_priority.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_uint32, C.c_uint32]
        lib.orc_select_victim.restype = C.c_int64
        lib.orc_select_victim.argtypes = [C.c_uint32, C.c_uint32, u64p, u64p, u32p, u32p, u8p,
                                          u8p, C.c_uint64]
        lib.orc_trace.restype = C.c_int
        lib.orc_trace.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u32p, C.c_uint64, u64p,
                                  C.c_uint64, u64p]
        lib.orc_capacity_bound.restype = C.c_uint64
        lib.orc_capacity_bound.argtypes = [C.c_uint32, C.c_uint32, C.c_double]
        lib.orc_generate_trace.restype = C.c_uint32
        lib.orc_generate_trace.argtypes = [C.POINTER(_Workload), C.c_uint64, C.c_void_p,
                                           C.c_void_p, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64)]
        lib.orc_request_eam.restype = C.c_uint32
        lib.orc_request_eam.argtypes = [C.POINTER(_Workload), C.c_uint64, C.c_int, u64p]
        lib.orc_iteration_probe.restype = C.c_int
        lib.orc_iteration_probe.argtypes = [C.POINTER(_Workload), C.c_uint64, C.c_uint32,
                                            C.c_uint32, u64p]

    # -- input families ---------------------------------------------------
    def bench_family(self, seed, L, E, n):
        out = np.zeros((n, L, E), np.uint64)
        self.lib.orc_bench_family(seed, L, E, n, out)
        return out

    def rng(self, seed):
        return _Rng(seed)

    def random_eam(self, rng, L, E):
        out = np.zeros((L, E), np.uint64)
        self.lib.orc_random_eam(C.byref(rng), L, E, out)
        return out

    def request_eams(self, w: Workload, n, phase=1, start=0):
        p = w.params
        out = np.zeros((n, p["L"], p["E"]), np.uint64)
        row = np.zeros((p["L"], p["E"]), np.uint64)
        for i in range(n):
            self.lib.orc_request_eam(C.byref(w.c), start + i, phase, row)
            out[i] = row
        return out

    def iteration_probe(self, w: Workload, request_index, iteration, layer):
        p = w.params
        out = np.zeros((p["L"], p["E"]), np.uint64)
        rc = self.lib.orc_iteration_probe(C.byref(w.c), request_index, iteration, layer, out)
        assert rc == 0
        return out

    def trace_picks(self, w: Workload, request_index):
        """(iteration counts [n_iter][L][E], picks [T][L][k]) for one request."""
        p = w.params
        nt, pt = C.c_uint64(), C.c_uint64()
        n_iter = self.lib.orc_generate_trace(C.byref(w.c), request_index, None, None,
                                             C.byref(nt), C.byref(pt))
        counts = np.zeros((n_iter, p["L"], p["E"]), np.uint64)
        picks = np.zeros((nt.value, p["L"], p["top_k"]), np.uint32)
        self.lib.orc_generate_trace(C.byref(w.c), request_index, counts.ctypes.data,
                                    picks.ctypes.data, C.byref(nt), C.byref(pt))
        return counts, picks

    # -- path ---------------------------------------------------------------
    def distance(self, a, b):
        a = np.ascontiguousarray(a, np.uint64)
        b = np.ascontiguousarray(b, np.uint64)
        L, E = a.shape[-2:]
        return self.lib.orc_eam_distance(L, E, a, b)

    def match(self, entries, seqs, probes):
        entries = np.ascontiguousarray(entries, np.uint64)
        probes = np.ascontiguousarray(probes, np.uint64)
        seqs = np.ascontiguousarray(seqs, np.uint64)
        L, E = probes.shape[-2:]
        Q = probes.shape[0]
        idx = np.zeros(Q, np.uint64)
        seq = np.zeros(Q, np.uint64)
        dist = np.zeros(Q, np.float64)
        found = np.zeros(Q, np.uint8)
        P = entries.shape[0] if entries.size else 0
        if P == 0:
            entries = np.zeros((1, L, E), np.uint64)
            seqs = np.zeros(1, np.uint64)
        self.lib.orc_match_batch(L, E, entries, seqs, P, probes, Q, idx, seq, dist, found)
        return idx, seq, dist, found

    def match_within(self, entries, seqs, probe, window):
        entries = np.ascontiguousarray(entries, np.uint64)
        probe = np.ascontiguousarray(probe, np.uint64)
        seqs = np.ascontiguousarray(seqs, np.uint64)
        L, E = probe.shape
        P = entries.shape[0]
        idx = np.zeros(max(P, 1), np.uint64)
        seq = np.zeros(max(P, 1), np.uint64)
        d = np.zeros(max(P, 1), np.float64)
        n = self.lib.orc_match_within(L, E, entries, seqs, P, probe, window, idx, seq, d)
        return idx[:n], seq[:n], d[:n]

    def prefetch(self, entries, seqs, cur, layer, apply_filter=True):
        entries = np.ascontiguousarray(entries, np.uint64)
        cur = np.ascontiguousarray(cur, np.uint64)
        seqs = np.ascontiguousarray(seqs, np.uint64)
        L, E = cur.shape
        P = entries.shape[0]
        cap = max(L * E, 1)
        ol = np.zeros(cap, np.uint32)
        oe = np.zeros(cap, np.uint32)
        op = np.zeros(cap, np.float64)
        if P == 0:
            entries = np.zeros((1, L, E), np.uint64)
            seqs = np.zeros(1, np.uint64)
        n = self.lib.orc_prefetch_priorities(L, E, entries, seqs, P, cur, layer,
                                             int(apply_filter), ol, oe, op)
        return ol[:n], oe[:n], op[:n]

    def cache_priority(self, req, layer, expert):
        req = np.ascontiguousarray(req, np.uint64)
        L, E = req.shape
        return self.lib.orc_cache_priority(L, E, req, layer, expert)

    def select_victim(self, req, slot, layer, expert, prot, pinned):
        req = np.ascontiguousarray(req, np.uint64)
        L, E = req.shape
        n = len(slot)
        return self.lib.orc_select_victim(
            L, E, req, np.ascontiguousarray(slot, np.uint64),
            np.ascontiguousarray(layer, np.uint32), np.ascontiguousarray(expert, np.uint32),
            np.ascontiguousarray(prot, np.uint8), np.ascontiguousarray(pinned, np.uint8), n)

    def trace(self, L, E, k, topk, offsets):
        topk = np.ascontiguousarray(topk, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        R = len(offsets) - 1
        T = topk.shape[0]
        out = np.zeros((max(R, 1), L, E), np.uint64)
        rc = self.lib.orc_trace(L, E, k, topk, T, offsets, R, out)
        return rc, out[:R]

    def capacity_bound(self, L, E, sim):
        return self.lib.orc_capacity_bound(L, E, sim)

    def insert_replay(self, L, E, capacity, eams):
        """Sequential Eamc::insert of `eams`; returns (entries, seqs, slots)."""
        cap = max(capacity, 1)
        entries = np.zeros((cap, L, E), np.uint64)
        seqs = np.zeros(cap, np.uint64)
        size = C.c_uint64(0)
        nxt = C.c_uint64(0)
        slots = np.zeros(len(eams), np.int64)
        for i, e in enumerate(eams):
            slots[i] = self.lib.orc_insert(L, E, capacity, entries, seqs, C.byref(size),
                                           C.byref(nxt), np.ascontiguousarray(e, np.uint64))
        n = size.value
        return entries[:n], seqs[:n], slots


class RefLib:
    """The reference library itself (oracle/_ref), driven through ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = C.CDLL(path)
        self.lib = lib
        lib.ref_eam_distance.restype = C.c_double
        lib.ref_eam_distance.argtypes = [C.c_uint32, C.c_uint32, u64p, u64p]
        lib.ref_eamc_new.restype = C.c_void_p
        lib.ref_eamc_new.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_uint64]
        lib.ref_eamc_free.argtypes = [C.c_void_p]
        lib.ref_eamc_size.restype = C.c_uint64
        lib.ref_eamc_size.argtypes = [C.c_void_p]
        lib.ref_eamc_insert.restype = C.c_int
        lib.ref_eamc_insert.argtypes = [C.c_void_p, u64p, C.c_int, C.c_int, C.POINTER(C.c_int64)]
        lib.ref_eamc_entry.argtypes = [C.c_void_p, C.c_uint64, u64p, C.POINTER(C.c_uint64)]
        lib.ref_eamc_match.restype = C.c_int
        lib.ref_eamc_match.argtypes = [C.c_void_p, u64p, C.c_uint64, u64p, u64p, f64p, u8p]
        lib.ref_eamc_match_mt.restype = C.c_double
        lib.ref_eamc_match_mt.argtypes = [C.c_void_p, u64p, C.c_uint64, u64p, u64p, f64p, u8p,
                                          C.c_int]
        lib.ref_eamc_match_within.restype = C.c_int64
        lib.ref_eamc_match_within.argtypes = [C.c_void_p, u64p, C.c_double, u64p, u64p, f64p,
                                              C.c_uint64]
        lib.ref_prefetch_priorities.restype = C.c_int64
        lib.ref_prefetch_priorities.argtypes = [C.c_void_p, u64p, C.c_uint32, C.c_int, u32p,
                                                u32p, f64p, C.c_uint64]
        lib.ref_cache_priority.restype = C.c_int
        lib.ref_cache_priority.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_uint32, C.c_uint32,
                                           C.POINTER(C.c_double)]
        lib.ref_select_victim.restype = C.c_int64
        lib.ref_select_victim.argtypes = [C.c_uint32, C.c_uint32, u64p, u64p, u32p, u32p, u8p,
                                          u8p, C.c_uint64]
        lib.ref_eam_record.restype = C.c_int
        lib.ref_eam_record.argtypes = [C.c_uint32, C.c_uint32, u64p, C.c_uint32, u32p, u64p,
                                       C.c_uint64]
        lib.ref_trace_mt.restype = C.c_double
        lib.ref_trace_mt.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, u8p, u64p, C.c_uint64,
                                     u64p, C.c_int]
        lib.ref_capacity_bound.restype = C.c_uint64
        lib.ref_capacity_bound.argtypes = [C.c_uint32, C.c_uint32, C.c_double]
        lib.ref_bench_match.restype = C.c_uint64
        lib.ref_bench_match.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64,
                                        C.c_uint64, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]
        lib.ref_generate_trace_counts.restype = C.c_uint32
        lib.ref_generate_trace_counts.argtypes = [
            C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_uint32,
            C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, u64p, C.c_uint32]

        lib.ref_gen_bench.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64,
                                      C.c_uint64, u64p]
        lib.ref_eamc_fill_bench.restype = C.c_int
        lib.ref_eamc_fill_bench.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]

    def trace_mt(self, L, E, k, topk_u8, offsets, n_threads):
        """Per-request EAMs from u8 router ids through the reference's Eam::record
        (RoutingEvent per layer, workload.cpp:166-181); returns (seconds, counts)."""
        topk_u8 = np.ascontiguousarray(topk_u8, np.uint8)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        R = len(offsets) - 1
        out = np.zeros((R, L, E), np.uint64)
        sec = self.lib.ref_trace_mt(L, E, k, topk_u8, offsets, R, out, n_threads)
        return sec, out

    def gen_bench(self, seed, L, E, n, skip=0):
        """bench_match's EAM stream (bench.cpp:44-54) from the reference Rng."""
        out = np.zeros((n, L, E), np.uint64)
        self.lib.ref_gen_bench(seed, L, E, skip, n, out)
        return out

    def distance(self, a, b):
        a = np.ascontiguousarray(a, np.uint64)
        b = np.ascontiguousarray(b, np.uint64)
        L, E = a.shape[-2:]
        return self.lib.ref_eam_distance(L, E, a, b)

    class Eamc:
        def __init__(self, ref, L, E, top_k, phase, capacity):
            self.ref = ref
            self.L, self.E = L, E
            self.h = ref.lib.ref_eamc_new(L, E, top_k, phase, capacity)
            self.phase = phase
            if not self.h:
                raise ValueError("invalid Eamc arguments")

        def __del__(self):
            if getattr(self, "h", None):
                self.ref.lib.ref_eamc_free(self.h)
                self.h = None

        def size(self):
            return self.ref.lib.ref_eamc_size(self.h)

        def fill_bench(self, seed, n):
            """Insert the first n EAMs of the bench stream (bench.cpp:61-62)."""
            rc = self.ref.lib.ref_eamc_fill_bench(self.h, seed, n)
            if rc:
                raise ValueError(f"ref fill error {rc}")

        def insert(self, counts, kind=1, phase=None):
            slot = C.c_int64()
            rc = self.ref.lib.ref_eamc_insert(self.h, np.ascontiguousarray(counts, np.uint64),
                                              kind, self.phase if phase is None else phase,
                                              C.byref(slot))
            if rc:
                raise ValueError(f"ref insert error {rc}")
            return slot.value

        def entries(self):
            n = self.size()
            out = np.zeros((n, self.L, self.E), np.uint64)
            seqs = np.zeros(n, np.uint64)
            s = C.c_uint64()
            row = np.zeros((self.L, self.E), np.uint64)
            for i in range(n):
                self.ref.lib.ref_eamc_entry(self.h, i, row, C.byref(s))
                out[i] = row
                seqs[i] = s.value
            return out, seqs

        def match(self, probes, threads=1):
            probes = np.ascontiguousarray(probes, np.uint64)
            Q = probes.shape[0]
            idx = np.zeros(Q, np.uint64)
            seq = np.zeros(Q, np.uint64)
            d = np.zeros(Q, np.float64)
            f = np.zeros(Q, np.uint8)
            if threads == 1:
                rc = self.ref.lib.ref_eamc_match(self.h, probes, Q, idx, seq, d, f)
                if rc:
                    raise ValueError(f"ref match error {rc}")
                return idx, seq, d, f
            secs = self.ref.lib.ref_eamc_match_mt(self.h, probes, Q, idx, seq, d, f, threads)
            return idx, seq, d, f, secs

        def match_within(self, probe, window):
            P = max(self.size(), 1)
            idx = np.zeros(P, np.uint64)
            seq = np.zeros(P, np.uint64)
            d = np.zeros(P, np.float64)
            n = self.ref.lib.ref_eamc_match_within(self.h, np.ascontiguousarray(probe, np.uint64),
                                                   window, idx, seq, d, P)
            if n < 0:
                raise ValueError(f"ref match_within error {-n}")
            return idx[:n], seq[:n], d[:n]

        def prefetch(self, cur, layer, apply_filter=True):
            cap = max(self.L * self.E, 1)
            ol = np.zeros(cap, np.uint32)
            oe = np.zeros(cap, np.uint32)
            op = np.zeros(cap, np.float64)
            n = self.ref.lib.ref_prefetch_priorities(self.h, np.ascontiguousarray(cur, np.uint64),
                                                     layer, int(apply_filter), ol, oe, op, cap)
            if n < 0:
                raise ValueError(f"ref prefetch error {-n}")
            return ol[:n], oe[:n], op[:n]

    def eamc(self, L, E, top_k=1, phase=1, capacity=1):
        return RefLib.Eamc(self, L, E, top_k, phase, capacity)

    def bench_match(self, n_entries, L, E, n_queries, seed):
        mean = C.c_double()
        med = C.c_double()
        ck = self.lib.ref_bench_match(n_entries, L, E, n_queries, seed, C.byref(mean),
                                      C.byref(med))
        return ck, mean.value, med.value

    def cache_priority(self, req, layer, expert):
        req = np.ascontiguousarray(req, np.uint64)
        L, E = req.shape
        out = C.c_double()
        rc = self.lib.ref_cache_priority(L, E, req, layer, expert, C.byref(out))
        if rc:
            raise IndexError("out of range")
        return out.value

    def select_victim(self, req, slot, layer, expert, prot, pinned):
        req = np.ascontiguousarray(req, np.uint64)
        L, E = req.shape
        return self.lib.ref_select_victim(
            L, E, req, np.ascontiguousarray(slot, np.uint64),
            np.ascontiguousarray(layer, np.uint32), np.ascontiguousarray(expert, np.uint32),
            np.ascontiguousarray(prot, np.uint8), np.ascontiguousarray(pinned, np.uint8),
            len(slot))

    def trace_counts(self, w: Workload, request_index):
        p = w.params
        n = self.lib.ref_generate_trace_counts(
            p["L"], p["E"], p["top_k"], p["n_groups"], p["group_fidelity"], p["reuse_skew"],
            p["prompt_len"], p["decode_len"], p["batch_size"], p["seed"], request_index,
            np.zeros(1, np.uint64), 0)
        out = np.zeros((n, p["L"], p["E"]), np.uint64)
        self.lib.ref_generate_trace_counts(
            p["L"], p["E"], p["top_k"], p["n_groups"], p["group_fidelity"], p["reuse_skew"],
            p["prompt_len"], p["decode_len"], p["batch_size"], p["seed"], request_index, out, n)
        return out

    def capacity_bound(self, L, E, sim):
        return self.lib.ref_capacity_bound(L, E, sim)
