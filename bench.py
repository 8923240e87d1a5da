#!/usr/bin/env python
"""bench.py -- EAM-vs-EAMC distance evals/s on B200 (BASELINE.json `metric`).

Headline workload (BASELINE.json configs[4], "SC", the configuration the
metric is quoted on): Switch-base-128 shape (L=12, E=128; SURVEY 8 fixes SC's
unstated shape to the reference benchmark's 12x128), an EAMC of P = 2^20
entries matched against a 65,536-probe batch.  Inputs are the reference
benchmark's own synthetic EAM family (bench.cpp:44-54, seed 55): the first P
EAMs of the stream are the collection, the next 65,536 the probes.  A step =
one Eamc::match pass of the probe batch over the whole collection
(eam.cpp:118-129 per probe).  At N > 1 the collection is P-sharded (rank r
owns slots [r*P/N, (r+1)*P/N)), the probes are replicated and the per-shard
argmins are merged over NCCL (all_gather + device lexicographic merge):
total work fixed, i.e. strong scaling.

The line also carries the SC streaming regime (same collection, Q = 8: the
HBM-bound case the north star's ">= 60% of HBM roofline at P >= 1M" is about)
as `roofline_streaming`, and the other SURVEY 8 rows under `rows` (SW, DS, NL,
tracing, MIX), each with the reference CPU path timed beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EAM-vs-EAMC distance evals/sec + % HBM roofline at 1/2/4/8 B200"
L, E, TOPK = 12, 128, 1
SEED = 55
SC_P, SC_Q = 1 << 20, 65536      # BASELINE configs[4]: P = 1M (2^20), 65k-query batch
STREAM_Q = 8                     # SC streaming regime (HBM-bound), same collection
SW_P, SW_Q = 10_000, 4096        # BASELINE configs[1] (a row now)
CPU_SAMPLE_Q = 64                # reference probes timed / parity-checked at SC


def sc_config(N):
    """The `config` of both arms (identical dicts, so the driver can compare)."""
    return {
        "workload": (f"SC (BASELINE configs[4]): P={SC_P} EAMs (L={L} E={E}, Switch-base-128 "
                     f"shape) sharded P/N over N={N} GPU(s), Q={SC_Q}-probe batch, "
                     "Eamc::match per probe"),
        "L": L, "E": E, "P_total": SC_P, "P_per_gpu": SC_P // N, "Q": SC_Q, "seed": SEED,
        "count_bytes": 1,
        "l2": ("inputs larger than L2 (1.61 GB u8 collection + 3.2 GB fp16 operand copy per "
               "pass) and a 256 MiB L2 flush between timed steps, outside the events"),
        "parallelism": (f"P-sharded x{N}, NCCL all_gather + device lexicographic merge"
                        if N > 1 else "single GPU"),
    }


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def ncu_traffic(key):
    """dram bytes/launch of the named kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    v = d.get(key, {})
    return v.get("dram_bytes_per_launch")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------- ours
def _events_timed(torch, stream, steps, step_fn, pre=None):
    """K device-timed steps on `stream` (CUDA events around each step)."""
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for i in range(steps):
        if pre is not None:
            pre()
        evs[i][0].record(stream)
        step_fn()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def _as_matches(t):
    """device/host moe_match[Q] tensor (Q x 3 f64 words) -> structured numpy."""
    from paper_2401_14361_b200 import _lib
    a = t.cpu().numpy() if hasattr(t, "cpu") else t
    return np.ascontiguousarray(a).view(np.uint8).reshape(-1, 24).copy().view(
        _lib.MATCH_DTYPE)[:, 0]


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2401_14361_b200 as m
    from paper_2401_14361_b200 import _lib

    rank, world, local = dist_env()
    N = world
    torch.cuda.set_device(local)
    if N > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    # One explicit stream for everything (flush, events, library kernels, NCCL):
    # torch's default stream is the legacy stream 0, which the C ABI reads as
    # "use the handle's internal stream".
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    sp = C.c_void_p(stream.cuda_stream)

    def barrier():
        if N > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if N > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- SC collection shard (P/N entries per rank) + the replicated probe batch
    P = SC_P // N
    shard = m.gen_bench_family(SEED, L, E, P, skip=rank * P, dtype=np.uint8)
    eamc = m.Eamc(m.ModelShape(L, E, TOPK), m.Phase.decode, P, device=local)
    eamc.append(shard, np.arange(rank * P, (rank + 1) * P, dtype=np.uint64))
    del shard
    _lib.check(_lib.lib.moe_eamc_set_index_base(eamc._h, rank * P))
    probes_u8 = m.gen_bench_family(SEED, L, E, SC_Q, skip=SC_P, dtype=np.uint8)
    d_probes = torch.from_numpy(probes_u8).to(dev)
    d_out = torch.empty((SC_Q, 3), dtype=torch.float64, device=dev)      # moe_match[Q]
    d_parts = torch.empty((N * SC_Q, 3), dtype=torch.float64, device=dev)
    d_final = torch.empty((SC_Q, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step_device():
        _lib.check(_lib.lib.moe_eamc_match_device(eamc._h, d_probes.data_ptr(), 1, SC_Q,
                                                  d_out.data_ptr(), sp))
        if N > 1:
            dist.all_gather_into_tensor(d_parts, d_out)
            _lib.check(_lib.lib.moe_match_merge_device(d_parts.data_ptr(), N, SC_Q,
                                                       d_final.data_ptr(), sp))
            return d_final
        return d_out

    for _ in range(args.warmup):
        step_device()
    barrier()

    # ---- timed region: K steps, L2 flushed between steps (outside the events)
    clocks = ClockSampler(local)
    time.sleep(0.05)
    barrier()
    ms_steps = _events_timed(torch, stream, args.steps, step_device, pre=flush.zero_)
    barrier()
    clk = clocks.stop()
    # Per-kernel times come from a second, identical pass with the library's
    # per-kernel events on: events between the kernels break the programmatic
    # dependent launch overlap, so that pass is not the one `value` is timed on.
    _lib.check(_lib.lib.moe_eamc_set_profiling(eamc._h, 1))
    barrier()
    ms_prof = _events_timed(torch, stream, args.steps, step_device, pre=flush.zero_)
    kms = (C.c_double * 3)()
    kcalls = (C.c_uint64 * 3)()
    _lib.check(_lib.lib.moe_eamc_kernel_times(eamc._h, kms, kcalls))
    _lib.check(_lib.lib.moe_eamc_set_profiling(eamc._h, 0))
    t_ms = max_over_ranks(sum(ms_steps))
    evals_per_step = SC_P * SC_Q
    value = evals_per_step * args.steps / (t_ms / 1e3)
    # per step: k_prep_u8, k_tc2_screen, k_refine, and the device-gated exact
    # pass k_match<1,1,1> + k_merge_partials (launched every step, exit at once
    # unless a candidate bucket overflowed); + k_merge for N > 1
    gpu_launches = args.steps * (5 + (1 if N > 1 else 0))
    res = _as_matches(step_device())  # the result of a timed-config step (parity sample)

    # ---- roofline of the dominant kernel (the screen), live CUDA events
    hbm_peak, tf_peak, peak_kind = load_peaks()
    screen_ms = kms[1] / max(kcalls[1], 1)
    ops_alg = 2.0 * L * E * P * SC_Q
    bytes_alg = P * L * E * 1 + SC_Q * L * E * 1 + 24 * SC_Q
    ach = ops_alg / (screen_ms / 1e3) / 1e12
    roofline = {
        "bound": "tensor",
        "kernel": "k_tc2_screen (tcgen05.mma.cta_group::2 kind::f16, 256x256 tiles, screen pass)",
        "achieved": ach, "peak": tf_peak, "unit": "TFLOP/s", "frac": ach / tf_peak,
        "traffic": ncu_traffic("sc_batch_screen"),
        "alg_ops_per_launch": ops_alg, "alg_bytes_per_launch": bytes_alg,
        "launch_ms": screen_ms,
        "share_of_step": screen_ms / (sum(ms_prof) / args.steps),
        "frac_of_nominal_2250": ach / 2250.0,
        "kernel_times": "per-kernel CUDA events on the launching stream, from a profiled pass of "
                        "the same K steps (ms_per_step_profiled)",
        "note": (f"peak = {peak_kind} dense bf16 cuBLAS burst (MEASURED_PEAKS.json); ops = "
                 "2*L*E*P*Q (SURVEY.md 8d), executed as one fp16 tensor-core GEMM over "
                 "unit-normalised rows (K=L*E), fp32 accumulate in TMEM, exact integer/fp64 "
                 "refine of the survivors; the 65k batch is compute-bound by construction "
                 f"(HBM view: {bytes_alg / (screen_ms / 1e3) / 1e9:.1f} GB/s of {hbm_peak:.0f})"),
    }

    # ---- e2e: the reference-facing C ABI call with HOST u64 probes (the
    # reference's Eam storage, eam.hpp:55) in pinned memory and host results
    # out, every step (host narrowing, H2D, matching, D2H inside the call)
    h_probes = torch.from_numpy(probes_u8.astype(np.uint64)).pin_memory()
    h_out = np.zeros(SC_Q, _lib.MATCH_DTYPE)
    h_parts = torch.empty((N * SC_Q, 3), dtype=torch.float64, device=dev)

    def step_e2e():
        _lib.check(_lib.lib.moe_eamc_match(eamc._h, h_probes.data_ptr(), SC_Q, h_out.ctypes.data,
                                           None))
        if N > 1:
            mine = torch.from_numpy(h_out.view(np.float64).reshape(SC_Q, 3)).to(dev)
            dist.all_gather_into_tensor(h_parts, mine)
            _lib.check(_lib.lib.moe_match_merge_device(h_parts.data_ptr(), N, SC_Q,
                                                       d_final.data_ptr(), sp))
            return _as_matches(d_final)
        return h_out

    for _ in range(2):
        step_e2e()
    barrier()
    e2e_steps = max(3, min(args.steps, 8))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        got_e2e = step_e2e()
    barrier()
    t_e2e = max_over_ranks(time.perf_counter() - t0)
    e2e_val = evals_per_step * e2e_steps / t_e2e
    e2e_same = bool(np.array_equal(got_e2e, res)) if N == 1 else None
    host_threads = int(_lib.lib.moe_host_threads())
    del h_probes

    # ---- SC streaming regime (north-star target: >= 60% HBM roofline at P >= 1M)
    streaming = None
    if not args.no_streaming:
        streaming = run_streaming(args, m, _lib, torch, dist, rank, N, dev, sp, flush, eamc,
                                  hbm_peak, peak_kind)

    # ---- the other SURVEY 8 rows (SW, prefetch decisions, construction, tracing, MIX)
    rows = None
    if N == 1 and not args.no_rows:
        del eamc  # free the SC collection before the rows allocate theirs
        torch.cuda.empty_cache()
        rows = run_rows(args, m, _lib, torch, dev, sp, stream, flush)

    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": ("synthetic: reference bench family F1 (bench.cpp:44-54, seed 55); u8 is the "
                     "count storage width (counts 1..32, lossless), distances are exact fp64"),
            "config": sc_config(N),
            "roofline": roofline,
            "e2e": {"value": e2e_val, "unit": "evals/s", "steps": e2e_steps,
                    "api": ("moe_eamc_match (host u64 probes [Q][L][E], pinned) + host results, "
                            f"u64 narrowed to the u8 storage width on {host_threads} host threads "
                            "inside the call; wall clock"),
                    "h2d_bytes_per_step": int(SC_Q * L * E * 1),
                    "d2h_bytes_per_step": int(SC_Q * 24),
                    "host_input_bytes_per_step": int(SC_Q * L * E * 8),
                    "same_result_as_device_api": e2e_same},
            "gpu_launches": gpu_launches,
            "ms_per_step_profiled": sum(ms_prof) / args.steps,
            "kernel_ms_per_step": {"prep": kms[0] / max(kcalls[0], 1), "screen": screen_ms,
                                   "refine": kms[2] / max(kcalls[2], 1)},
            "clocks": clk,
        }
        if streaming:
            out["roofline_streaming"] = streaming.pop("roofline")
            out["streaming"] = streaming
        if rows:
            out["rows"] = rows
        if N == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"], out["parity_sample"] = cpu_baseline(args, probes_u8, res)
    if N > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def run_sw_row(args, m, _lib, torch, dev, sp, stream, flush):
    """BASELINE configs[1] (SW): P=10k, Q=4096, one B200 -- device-resident
    value + roofline, e2e through the host API, reference on all host cores
    over the whole batch with a bitwise check."""
    shard = m.gen_bench_family(SEED, L, E, SW_P, dtype=np.uint8)
    probes_u8 = m.gen_bench_family(SEED, L, E, SW_Q, skip=SW_P, dtype=np.uint8)
    eamc = m.Eamc(m.ModelShape(L, E, TOPK), m.Phase.decode, SW_P, device=dev.index)
    eamc.append(shard, np.arange(SW_P, dtype=np.uint64))
    d_probes = torch.from_numpy(probes_u8).to(dev)
    d_out = torch.empty((SW_Q, 3), dtype=torch.float64, device=dev)

    def step():
        _lib.check(_lib.lib.moe_eamc_match_device(eamc._h, d_probes.data_ptr(), 1, SW_Q,
                                                  d_out.data_ptr(), sp))

    for _ in range(max(args.warmup, 5)):
        step()
    torch.cuda.synchronize()
    steps = max(args.steps, 50)
    ms = _events_timed(torch, stream, steps, step, pre=flush.zero_)
    _lib.check(_lib.lib.moe_eamc_set_profiling(eamc._h, 1))
    ms_prof = _events_timed(torch, stream, steps, step, pre=flush.zero_)
    kms = (C.c_double * 3)()
    kc = (C.c_uint64 * 3)()
    _lib.check(_lib.lib.moe_eamc_kernel_times(eamc._h, kms, kc))
    _lib.check(_lib.lib.moe_eamc_set_profiling(eamc._h, 0))
    res = _as_matches(d_out)
    hbm_peak, tf_peak, peak_kind = load_peaks()
    screen_ms = kms[1] / max(kc[1], 1)
    ops_alg = 2.0 * L * E * SW_P * SW_Q
    ach = ops_alg / (screen_ms / 1e3) / 1e12
    row = {
        "workload": (f"SW (BASELINE configs[1]): L={L} E={E} top-{TOPK}, EAMC P={SW_P}, "
                     f"Q={SW_Q} probes, device-resident u8, L2 flushed between steps"),
        "value": SW_P * SW_Q * steps / (sum(ms) / 1e3), "unit": "evals/s", "steps": steps,
        "ms_per_step": sum(ms) / steps, "ms_per_step_profiled": sum(ms_prof) / steps,
        "kernel_ms_per_step": {"prep": kms[0] / max(kc[0], 1), "screen": screen_ms,
                               "refine": kms[2] / max(kc[2], 1)},
        "roofline": {"bound": "tensor", "kernel": "k_tc2_screen", "achieved": ach,
                     "peak": tf_peak, "unit": "TFLOP/s", "frac": ach / tf_peak,
                     "traffic": ncu_traffic("sw_screen"), "launch_ms": screen_ms,
                     "alg_ops_per_launch": ops_alg,
                     "alg_bytes_per_launch": SW_P * L * E + SW_Q * L * E + 24 * SW_Q},
    }
    # e2e through the host API (u64 probes, the reference's storage type)
    h_probes = torch.from_numpy(probes_u8.astype(np.uint64)).pin_memory()
    h_out = np.zeros(SW_Q, _lib.MATCH_DTYPE)
    for _ in range(3):
        _lib.check(_lib.lib.moe_eamc_match(eamc._h, h_probes.data_ptr(), SW_Q, h_out.ctypes.data,
                                           None))
    n_e2e = 30
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        _lib.check(_lib.lib.moe_eamc_match(eamc._h, h_probes.data_ptr(), SW_Q, h_out.ctypes.data,
                                           None))
    t_e2e = (time.perf_counter() - t0) / n_e2e
    row["e2e"] = {"value": SW_P * SW_Q / t_e2e, "unit": "evals/s", "ms_per_step": t_e2e * 1e3,
                  "api": "moe_eamc_match, host u64 probes (pinned) + host results",
                  "h2d_bytes_per_step": SW_Q * L * E, "d2h_bytes_per_step": SW_Q * 24}
    ref, _ = _ref_or_none()
    if ref is not None and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        er = ref.eamc(L, E, TOPK, 1, SW_P)
        er.fill_bench(SEED, SW_P)
        pr = ref.gen_bench(SEED, L, E, SW_Q, skip=SW_P)
        idx, seq, d, f, secs = er.match(pr, threads=cores)
        row["cpu_baseline"] = {"value": SW_P * SW_Q / secs, "unit": "evals/s", "cores": cores,
                               "kind": "reference",
                               "sample": f"all {SW_Q} probes (std::thread over the const matcher)"}
        row["parity_sample"] = {
            "probes": SW_Q,
            "bitwise_equal_index_seq_distance": bool(
                np.array_equal(idx, res["index"]) and np.array_equal(seq, res["seq"]) and
                np.array_equal(d, res["distance"]))}
        row["speedup_vs_reference"] = row["value"] / row["cpu_baseline"]["value"]
        row["e2e_speedup_vs_reference"] = row["e2e"]["value"] / row["cpu_baseline"]["value"]
    return row


def _ref_or_none():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import REF_SO, Oracle, RefLib
    return (RefLib() if os.path.exists(REF_SO) else None), Oracle()


def run_rows(args, m, _lib, torch, dev, sp, stream, flush):
    """Measured lines for SURVEY 8 rows beyond the headline matcher, each with
    the reference CPU path (oracle/_ref) timed on this box beside it."""
    from concurrent.futures import ThreadPoolExecutor
    hbm_peak, _, peak_kind = load_peaks()
    ref, orc = _ref_or_none()
    cores = os.cpu_count() or 1
    out = {"sw_match": run_sw_row(args, m, _lib, torch, dev, sp, stream, flush)}

    # -- A10/A11 prefetch decisions, DS shape (L=59, E=160, top-6): one decode
    #    step = 58 prefetch_priorities calls (l = 0..57) + floor filter
    L2, E2, P2 = 59, 160, 10_000
    fam = m.gen_bench_family(SEED, L2, E2, P2 + 1, dtype=np.uint8)
    s2 = m.ModelShape(L2, E2, 6)
    e2 = m.Eamc(s2, m.Phase.decode, P2)
    e2.append(fam[:P2], np.arange(P2, dtype=np.uint64))
    base = fam[P2].astype(np.uint64)
    probes = []
    for l in range(L2 - 1):
        pr = base.copy()
        pr[l + 1:] = 0  # the engine's iteration EAM at layer l (engine.cpp:546, :587)
        probes.append(pr)
    # the engine's call (engine.cpp:658-668) through the C ABI: host u64
    # iteration EAM in, ordered candidates out, preallocated output buffer
    import ctypes as C
    cap2 = L2 * E2
    cand = np.zeros(cap2, _lib.CAND_DTYPE)
    n_c = C.c_uint64()
    probes = [np.ascontiguousarray(pr) for pr in probes]

    def decode_step():
        res = []
        for l in range(L2 - 1):
            _lib.check(_lib.lib.moe_prefetch_priorities(e2._h, probes[l].ctypes.data, l, 1,
                                                        cand.ctypes.data, cap2, C.byref(n_c)))
            res.append(cand[:n_c.value].copy())
        return res

    orders = decode_step()  # warm-up + the results compared with the reference
    # timed: the engine's 58 calls back to back (arguments prepared once, as the
    # engine holds them; no result copies in the loop)
    fn, hnd, pn = _lib.lib.moe_prefetch_priorities, e2._h, C.byref(n_c)
    pp = [pr.ctypes.data for pr in probes]
    cp = cand.ctypes.data
    t0 = time.perf_counter()
    reps = 10
    for _ in range(reps):
        for l in range(L2 - 1):
            fn(hnd, pp[l], l, 1, cp, cap2, pn)
    t_gpu = (time.perf_counter() - t0) / reps
    _lib.check(fn(hnd, pp[0], 0, 1, cp, cap2, pn))
    row = {"workload": f"DS decode step: L={L2} E={E2} top-6, EAMC P={P2} (F1), 58 "
                       "prefetch_priorities calls + floor filter, C ABI with host buffers",
           "gpu_ms_per_step": t_gpu * 1e3, "gpu_decisions_per_s": (L2 - 1) / t_gpu,
           "us_per_decision": t_gpu / (L2 - 1) * 1e6}
    if ref is not None:
        er = ref.eamc(L2, E2, 6, 1, P2)
        for x in fam[:P2]:
            er.insert(x.astype(np.uint64))
        t0 = time.perf_counter()
        with ThreadPoolExecutor(cores) as ex:
            refs = list(ex.map(lambda l: er.prefetch(probes[l], l, True), range(L2 - 1)))
        t_cpu = time.perf_counter() - t0
        same = all(np.array_equal(o["layer_idx"], r[0]) and np.array_equal(o["expert_idx"], r[1])
                   and np.array_equal(o["priority"], r[2]) for o, r in zip(orders, refs))
        row.update({"cpu_ms_per_step": t_cpu * 1e3, "cpu_cores": cores, "cpu_kind": "reference",
                    "cpu_note": "the 58 reference calls run concurrently on all host cores "
                                "(the engine makes them one after another): generous to the CPU",
                    "speedup": t_cpu / t_gpu, "parity_bitwise_order": bool(same)})
    out["prefetch_decode_step"] = row

    # -- A9/K7 EAMC construction, NL shape (L=24, E=128): insert replay at
    #    capacity P=10k (each step: argmin over P, replace in place)
    L3, E3, P3, n3, nw3 = 24, 128, 10_000, 8192, 8192
    reps3 = 3
    fam3 = m.gen_bench_family(3, L3, E3, P3 + nw3 + reps3 * n3, dtype=np.uint8)
    e3 = m.Eamc(m.ModelShape(L3, E3), m.Phase.decode, P3)
    e3.append(fam3[:P3], np.arange(P3, dtype=np.uint64))  # = P3 inserts below capacity
    steps_all = fam3[P3:].astype(np.uint64)
    e3.build(steps_all[:nw3])  # warm-up: buffers, staging memory, kernels
    # three consecutive blocks of n3 steps (wall clock: the host API includes the
    # host narrowing and the transfers); the median is reported
    ts3 = []
    for r3 in range(reps3):
        steps = steps_all[nw3 + r3 * n3:nw3 + (r3 + 1) * n3]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e3.build(steps)
        ts3.append(time.perf_counter() - t0)
    t_gpu = sorted(ts3)[reps3 // 2]
    row = {"workload": f"NL construction replay: L={L3} E={E3}, capacity P={P3}, {n3} "
                       "at-capacity Eamc::insert steps (F1), host API (moe_eamc_build, host "
                       "u64 EAMs)",
           "gpu_us_per_step": t_gpu / n3 * 1e6, "gpu_evals_per_s": n3 * P3 / t_gpu,
           "extrapolated_N100k_s": 90_000 * t_gpu / n3}
    if ref is not None:
        # the reference from the same starting collection: parity of the
        # first steps (a fresh device collection replays them) and CPU time
        er = ref.eamc(L3, E3, 1, 1, P3)
        for x in fam3[:P3]:
            er.insert(x.astype(np.uint64))
        ns = 256  # about 10 s of reference inserts; spans the first blocked-replay block
        e3p = m.Eamc(m.ModelShape(L3, E3), m.Phase.decode, P3)
        e3p.append(fam3[:P3], np.arange(P3, dtype=np.uint64))
        slots_p = e3p.build(steps_all[:ns])
        t0 = time.perf_counter()
        rs = [er.insert(x) for x in steps_all[:ns]]
        t_cpu = (time.perf_counter() - t0) / ns
        ent_ref = er.entries()
        same_ent = all(np.array_equal(e3p.entry(i).counts, ent_ref[0][i])
                       and e3p.entry_seq(i) == ent_ref[1][i] for i in range(0, P3, 97))
        row.update({"cpu_us_per_step": t_cpu * 1e6, "cpu_cores": 1, "cpu_kind": "reference",
                    "cpu_sample": f"{ns} at-capacity inserts (Eamc::insert, eam.cpp:152-178)",
                    "speedup": t_cpu / (t_gpu / n3),
                    "parity_steps": ns,
                    "parity_victims_and_entries": bool(list(slots_p[:ns]) == rs and same_ent)})
    row["roofline"] = {"bound": "latency", "achieved": n3 / t_gpu, "unit": "steps/s",
                       "peak": None, "frac": None,
                       "note": "a sequential victim chain (eam.cpp:164-177): one CTA decides "
                               "the steps of a 512-step block in order (k_replay_block); the "
                               "block's screen distances come from tcgen05 GEMMs"}
    out["construction"] = row

    # -- the step-wise construction path (one screen + refine + replace per insert;
    #    taken for single inserts, L > 64 or P > 16,384), timed at P = 20,000
    P7, n7 = 20_000, 256
    fam7 = m.gen_bench_family(5, L3, E3, P7 + 32 + n7, dtype=np.uint8)
    e7 = m.Eamc(m.ModelShape(L3, E3), m.Phase.decode, P7)
    e7.append(fam7[:P7], np.arange(P7, dtype=np.uint64))
    st7 = fam7[P7:].astype(np.uint64)
    e7.build(st7[:32])  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e7.build(st7[32:])
    t7 = time.perf_counter() - t0
    out["construction_stepwise"] = {
        "workload": f"L={L3} E={E3}, capacity P={P7} (> 16,384: the step-wise replay), {n7} "
                    "at-capacity inserts (moe_eamc_build, host u64 EAMs)",
        "gpu_us_per_step": t7 / n7 * 1e6, "gpu_evals_per_s": n7 * P7 / t7}
    del e7

    # -- north-star (3): clustering construction, NL config (configs[2]):
    #    N = 100k request EAMs (F2 grouped workload, L=24 E=128 top-2) -> P = 10k.
    #    Iteration 0 = the reference insert replay over all N (the full configs[2]
    #    construction, timed on its own); then k-medoids-style refinement
    #    (opt-in, parity-unpinned: the reference defers clustering).
    N6, P6, it6 = 100_000, 10_000, 5
    from oracle import Workload
    w6 = Workload(L3, E3, 2, seed=1001)
    with ThreadPoolExecutor(cores) as ex:
        parts6 = list(ex.map(lambda k: orc.request_eams(w6, N6 // 20, start=k * (N6 // 20)),
                             range(20)))
    eams6 = np.concatenate(parts6)
    e6 = m.Eamc(m.ModelShape(L3, E3, 2), m.Phase.decode, P6)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    obj0, _, _ = e6.build_clustered(eams6, iterations=0)
    t_replay = time.perf_counter() - t0
    e6 = m.Eamc(m.ModelShape(L3, E3, 2), m.Phase.decode, P6)
    t0 = time.perf_counter()
    obj6, rep6, ran6 = e6.build_clustered(eams6, iterations=it6)
    t_clu = time.perf_counter() - t0
    out["construction_nl_full"] = {
        "workload": f"NL configs[2]: N={N6} request EAMs (F2 grouped workload, L={L3} E={E3} "
                    f"top-2) -> P={P6} representatives",
        "replay_s": t_replay, "replay_steps": N6,
        "replay_objective": float(obj0[0]),
        "clustered_s": t_clu, "clustered_iterations": int(ran6),
        "clustered_objective": [float(x) for x in obj6[:ran6 + 1]],
        "objective_reduction": float(1.0 - obj6[ran6] / obj6[0]),
        "note": "objective = sum over the N EAMs of the distance to the nearest representative; "
                "iteration 0 is the reference construction (parity-tested); the refinement is "
                "opt-in and parity-unpinned (no reference implementation)"}
    del e6, eams6, parts6

    # -- A2/K1 tracing, DS shape: T = 1M router tokens x 59 layers x top-6 ids
    #    (u8, resident) -> R = 1000 per-request count matrices (u32), accumulated
    L4, E4, k4, T4 = 59, 160, 6, 1_000_000
    R4 = T4 // 1000
    rng = np.random.default_rng(1001)
    zipf = 1.0 / np.arange(1, E4 + 1) ** 1.2
    basei = rng.choice(E4, size=(T4, L4), p=zipf / zipf.sum()).astype(np.uint16)
    picks = ((basei[:, :, None] + np.arange(k4, dtype=np.uint16)[None, None, :]) % E4).astype(np.uint8)
    offs = np.arange(0, T4 + 1, 1000, dtype=np.uint64)
    d_picks = torch.from_numpy(picks).to(dev)
    d_offs = torch.from_numpy(offs.astype(np.int64)).to(dev)
    d_counts = torch.zeros((R4, L4, E4), dtype=torch.int32, device=dev)
    d_bad = torch.zeros(1, dtype=torch.int32, device=dev)
    s4 = m.ModelShape(L4, E4, k4)
    import ctypes as C
    sh = s4.c()

    def trace_dev():
        _lib.check(_lib.lib.moe_eam_trace_device(C.byref(sh), d_picks.data_ptr(), 1, T4,
                                                 d_offs.data_ptr(), R4, d_counts.data_ptr(),
                                                 d_bad.data_ptr(), sp))
    for _ in range(3):
        trace_dev()
    torch.cuda.synchronize()
    d_counts.zero_()
    torch.cuda.synchronize()
    n_ev = 10
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n_ev)]
    for a_, b_ in evs:
        a_.record(stream)
        trace_dev()  # the whole call: k_trace_lane + its gated rollback
        b_.record(stream)
    torch.cuda.synchronize()
    t_dev = sum(a_.elapsed_time(b_) for a_, b_ in evs) / n_ev / 1e3
    dev_counts = d_counts.cpu().numpy().astype(np.uint64) // n_ev  # n_ev accumulations
    bytes_alg = T4 * L4 * k4 * 1 + R4 * L4 * E4 * 4 + 8 * (R4 + 1)
    host_counts = m.trace_requests(s4, picks, offs)  # warm-up (buffers) + parity result
    acc = np.zeros_like(host_counts)
    reps4 = 3
    t0 = time.perf_counter()
    for _ in range(reps4):
        m.trace_requests(s4, picks, offs, counts=acc)  # accumulates, as Eam::record does
    t_e2e = (time.perf_counter() - t0) / reps4
    row = {"workload": f"DS tracing: T={T4} tokens x L={L4} x top-{k4} u8 ids, R={R4} requests",
           "gpu_ms": t_dev * 1e3, "picks_per_s": T4 * L4 * k4 / t_dev,
           "roofline": {"bound": "hbm", "kernel": "k_trace_lane (+ gated rollback), whole call",
                        "achieved": bytes_alg / t_dev / 1e9, "peak": hbm_peak,
                        "unit": "GB/s", "frac": bytes_alg / t_dev / 1e9 / hbm_peak,
                        "traffic": ncu_traffic("k_trace_lane"),
                        "alg_bytes": bytes_alg, "note": f"peak = {peak_kind} HBM; bytes = "
                        "T*L*k ids + R*L*E*4 counts + 8*(R+1) offsets (SURVEY 8d)"},
           "e2e_ms": t_e2e * 1e3,
           "e2e_api": ("moe_eam_trace (host u8 ids + host u64 counts accumulated; transfers "
                       "through pinned staging inside the call)")}
    if ref is not None:  # the reference's Eam::record on all host cores, full workload
        ncpu = os.cpu_count() or 1
        sec, ref_counts = ref.trace_mt(L4, E4, k4, picks, offs, ncpu)
        row.update({"cpu_picks_per_s": T4 * L4 * k4 / sec, "cpu_cores": ncpu,
                    "cpu_kind": "reference",
                    "cpu_sample": f"all {T4} tokens (reference Eam::record, one RoutingEvent per "
                                  "request and layer as workload.cpp:166-181; std::thread over "
                                  "requests)",
                    "speedup": (T4 * L4 * k4 / t_dev) / (T4 * L4 * k4 / sec),
                    "parity_full": bool(np.array_equal(host_counts, ref_counts)
                                        and np.array_equal(dev_counts, ref_counts))})
    else:
        ns = 20_000
        t0 = time.perf_counter()
        rc, ref_counts = orc.trace(L4, E4, k4, picks[:ns].astype(np.uint32),
                                   np.arange(0, ns + 1, 1000, dtype=np.uint64))
        t_cpu = time.perf_counter() - t0
        row.update({"cpu_picks_per_s": ns * L4 * k4 / t_cpu, "cpu_cores": 1, "cpu_kind": "port",
                    "cpu_sample": f"{ns} tokens (oracle restatement)",
                    "parity_sample": bool(rc == 0 and np.array_equal(host_counts[:ns // 1000],
                                                                     ref_counts))})
    out["tracing"] = row
    del d_picks, d_counts

    # -- real expert prefetch -- the GPU order drives chunked DMA of
    #    expert weights (16 MB chunks) into GPU expert slots
    Lx, Ex, nbx, slx = 4, 8, 32 << 20, 16
    wx = np.empty((Lx, Ex, nbx), np.uint8)
    wx[...] = 7
    sx = m.ModelShape(Lx, Ex, 2)
    cx = m.ExpertCache(sx, wx, slx, chunk_bytes=16 << 20)
    cx.set_request_eam(m.Eam(sx, counts=np.ones((Lx, Ex), np.uint64)))
    ordx = np.zeros(slx, _lib.CAND_DTYPE)
    for i in range(slx):
        ordx[i] = (i // Ex, i % Ex, 1.0 - i / 64)
    cx.submit(ordx[:2])
    cx.progress(wait_idle=True)  # warm-up: page-locking, events
    b0 = cx.stats()["bytes_moved"]
    t0 = time.perf_counter()
    cx.submit(ordx)
    cx.progress(wait_idle=True)
    t_x = time.perf_counter() - t0
    stx = cx.stats()
    out["expert_prefetch"] = {
        "workload": f"{slx} expert slots of {nbx >> 20} MB, a {slx}-candidate prefetch order, "
                    "16 MB chunks (moe_expert_cache_*: the engine's transfer rules over real "
                    "cudaMemcpyAsync from page-locked host weights)",
        "gb_per_s": (stx["bytes_moved"] - b0) / t_x / 1e9,
        "transfers": int(stx["transfers_completed"]), "ms": t_x * 1e3}
    del cx, wx

    # -- MIX matcher (configs[0] shape): P=300, Q=1000 probes, latency regime
    L5, E5, P5, Q5 = 32, 8, 300, 1000
    fam5 = m.gen_bench_family(SEED, L5, E5, P5 + Q5)
    e5 = m.Eamc(m.ModelShape(L5, E5, 2), m.Phase.decode, P5)
    e5.append(fam5[:P5], np.arange(P5, dtype=np.uint64))
    d5 = torch.from_numpy(fam5[P5:].astype(np.uint8)).to(dev)
    o5 = torch.empty((Q5, 3), dtype=torch.float64, device=dev)
    for _ in range(5):
        _lib.check(_lib.lib.moe_eamc_match_device(e5._h, d5.data_ptr(), 1, Q5, o5.data_ptr(), sp))
    torch.cuda.synchronize()
    a5, b5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a5.record(stream)
    for _ in range(50):
        _lib.check(_lib.lib.moe_eamc_match_device(e5._h, d5.data_ptr(), 1, Q5, o5.data_ptr(), sp))
    b5.record(stream)
    torch.cuda.synchronize()
    t5 = a5.elapsed_time(b5) / 50 / 1e3
    row = {"workload": f"MIX: L={L5} E={E5} top-2, EAMC P={P5}, Q={Q5} probes (F1), device API",
           "gpu_us_per_batch": t5 * 1e6, "evals_per_s": P5 * Q5 / t5,
           "us_per_query": t5 / Q5 * 1e6}
    if ref is not None:
        er = ref.eamc(L5, E5, 2, 1, P5)
        for x in fam5[:P5]:
            er.insert(x)
        idx, seq, d, f, secs = er.match(fam5[P5:], threads=cores)
        row.update({"cpu_evals_per_s": P5 * Q5 / secs, "cpu_cores": cores, "cpu_kind": "reference",
                    "speedup": (P5 * Q5 / t5) / (P5 * Q5 / secs)})
    out["mix_match"] = row

    # -- MIX prefetch decisions (configs[0]: match + prefetch priority per query):
    # prefetch_priorities + floor filter at layer l = q mod (L-1), through the C ABI
    # with host buffers, each probe an iteration EAM truncated at its layer
    pp = []
    for q in range(Q5):
        x = np.ascontiguousarray(fam5[P5 + q].astype(np.uint64))
        x[q % (L5 - 1) + 1:] = 0
        pp.append(x)
    cap5 = L5 * E5
    o5p = np.zeros(cap5, _lib.CAND_DTYPE)
    n5 = C.c_uint64()
    for q in range(20):
        _lib.check(_lib.lib.moe_prefetch_priorities(e5._h, pp[q].ctypes.data, q % (L5 - 1), 1,
                                                    o5p.ctypes.data, cap5, C.byref(n5)))
    got = []
    for q in range(64):  # the results compared with the reference
        _lib.check(_lib.lib.moe_prefetch_priorities(e5._h, pp[q].ctypes.data, q % (L5 - 1), 1,
                                                    o5p.ctypes.data, cap5, C.byref(n5)))
        got.append(o5p[:n5.value].copy())
    fn5, h5, pn5, op5 = _lib.lib.moe_prefetch_priorities, e5._h, C.byref(n5), o5p.ctypes.data
    pq = [x.ctypes.data for x in pp]
    t0 = time.perf_counter()
    for q in range(Q5):
        fn5(h5, pq[q], q % (L5 - 1), 1, op5, cap5, pn5)
    t5p = time.perf_counter() - t0
    _lib.check(fn5(h5, pq[0], 0, 1, op5, cap5, pn5))
    # the same through the opt-in persistent decision server (one resident CTA
    # for a small collection, fed through a pinned mailbox instead of a launch)
    _lib.check(_lib.lib.moe_eamc_set_decision_server(h5, 8))
    for q in range(20):
        _lib.check(fn5(h5, pq[q], q % (L5 - 1), 1, op5, cap5, pn5))
    srv_same = True
    for q in range(64):
        _lib.check(fn5(h5, pq[q], q % (L5 - 1), 1, op5, cap5, pn5))
        srv_same &= bool(np.array_equal(o5p[:n5.value], got[q]))
    t0 = time.perf_counter()
    for q in range(Q5):
        fn5(h5, pq[q], q % (L5 - 1), 1, op5, cap5, pn5)
    t5s = time.perf_counter() - t0
    _lib.check(_lib.lib.moe_eamc_set_decision_server(h5, 0))
    row = {"workload": f"MIX prefetch: L={L5} E={E5}, EAMC P={P5}, {Q5} prefetch_priorities "
                       "calls (l = q mod (L-1)) + floor filter, C ABI with host buffers",
           "us_per_decision": t5p / Q5 * 1e6, "decisions_per_s": Q5 / t5p,
           "us_per_decision_server": t5s / Q5 * 1e6,
           "server_note": "opt-in moe_eamc_set_decision_server: one resident CTA polls a pinned "
                          "mailbox (no launch per decision); results equal the launched path's",
           "server_same_orders": srv_same}
    if ref is not None:
        t0 = time.perf_counter()
        ok = True
        for q in range(64):
            rl, rx, rp = er.prefetch(pp[q], q % (L5 - 1), True)
            ok &= (np.array_equal(got[q]["layer_idx"], rl) and
                   np.array_equal(got[q]["expert_idx"], rx) and
                   np.array_equal(got[q]["priority"], rp))
        t_ref = (time.perf_counter() - t0) / 64
        row.update({"cpu_us_per_decision": t_ref * 1e6, "cpu_cores": 1, "cpu_kind": "reference",
                    "cpu_sample": "64 of the 1,000 decisions", "speedup": t_ref / (t5p / Q5),
                    "parity_bitwise_order": bool(ok)})
    out["mix_prefetch"] = row
    return out


def run_streaming(args, m, _lib, torch, dist, rank, N, dev, sp, flush, e, hbm_peak, peak_kind):
    """SC streaming regime: the headline's P = 2^20 collection (sharded P/N),
    Q = 8 probes -- the HBM-bound case (arithmetic intensity 2Q/s_c)."""
    assert sp.value, "streaming leg must run on the explicit bench stream"
    P = SC_P // N
    probes = m.gen_bench_family(SEED, L, E, STREAM_Q, skip=SC_P, dtype=np.uint8)
    d_pr = torch.from_numpy(probes).to(dev)
    d_out = torch.empty((STREAM_Q, 3), dtype=torch.float64, device=dev)
    d_parts = torch.empty((N * STREAM_Q, 3), dtype=torch.float64, device=dev)
    d_fin = torch.empty((STREAM_Q, 3), dtype=torch.float64, device=dev)

    def step():
        _lib.check(_lib.lib.moe_eamc_match_device(e._h, d_pr.data_ptr(), 1, STREAM_Q,
                                                  d_out.data_ptr(), sp))
        if N > 1:
            dist.all_gather_into_tensor(d_parts, d_out)
            _lib.check(_lib.lib.moe_match_merge_device(d_parts.data_ptr(), N, STREAM_Q,
                                                       d_fin.data_ptr(), sp))

    stream = torch.cuda.current_stream()

    def timed(steps, profile):
        if N > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if profile:
            _lib.check(_lib.lib.moe_eamc_set_profiling(e._h, 1))
        ms = _events_timed(torch, stream, steps, step, pre=flush.zero_)
        kms = (C.c_double * 3)()
        kc = (C.c_uint64 * 3)()
        if profile:
            _lib.check(_lib.lib.moe_eamc_kernel_times(e._h, kms, kc))
            _lib.check(_lib.lib.moe_eamc_set_profiling(e._h, 0))
        t = torch.tensor([sum(ms)], dtype=torch.float64, device=dev)
        if N > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), kms[1] / max(kc[1], 1)

    for _ in range(3):
        step()
    steps = 30
    t_ms, _ = timed(steps, False)   # value: no per-kernel events (PDL intact)
    _, screen_ms = timed(steps, True)
    bytes_alg = P * L * E * 1 + STREAM_Q * L * E * 1 + 24 * STREAM_Q
    ach = bytes_alg / (screen_ms / 1e3) / 1e9
    return {
        "workload": f"SC streaming: P={SC_P} (P/GPU={P}), Q={STREAM_Q}, L={L} E={E}, u8",
        "value": P * N * STREAM_Q * steps / (t_ms / 1e3), "unit": "evals/s",
        "ms_per_step": t_ms / steps, "steps": steps,
        "roofline": {"bound": "hbm",
                     "kernel": "k_tci8_screen<4> (tcgen05.mma kind::i8, block-diagonal probes)",
                     "achieved": ach,
                     "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                     "traffic": ncu_traffic("sc_screen"), "launch_ms": screen_ms,
                     "alg_bytes_per_launch": bytes_alg,
                     "note": (f"peak = {peak_kind} HBM copy bandwidth (MEASURED_PEAKS.json); "
                              "bytes = P*L*E*s_c + Q*L*E*s_q + 24*Q (SURVEY.md 8d)")},
    }


def cpu_baseline(args, probes_u8, gpu_res):
    """The reference CPU path (oracle/_ref = moesim compiled from its own
    sources) on this box's host cores, on a bounded sample of the SC workload
    (the full P = 2^20 collection, CPU_SAMPLE_Q probes spread over the batch);
    the sampled probes are also checked against the GPU result bit for bit."""
    ref, orc = _ref_or_none()
    cores = os.cpu_count() or 1
    pick = np.linspace(0, SC_Q - 1, CPU_SAMPLE_Q).astype(np.int64)
    pr = probes_u8[pick].astype(np.uint64)
    if ref is not None:
        kind = "reference"
        t0 = time.perf_counter()
        e = ref.eamc(L, E, TOPK, 1, SC_P)
        e.fill_bench(SEED, SC_P)          # bench_match's fill loop (bench.cpp:61-62)
        t_fill = time.perf_counter() - t0
        idx, seq, d, f, secs = e.match(pr, threads=cores)
        del e
    else:  # the reference was not built on this box: the C restatement, one thread
        kind, cores, t_fill = "port", 1, 0.0
        fam = orc.bench_family(SEED, L, E, SC_P)
        t0 = time.perf_counter()
        idx, seq, d, f = orc.match(fam, np.arange(SC_P, dtype=np.uint64), pr[:4])
        secs = time.perf_counter() - t0
        pick, pr = pick[:4], pr[:4]
    g = gpu_res[pick]
    ok = bool(np.array_equal(idx, g["index"]) and np.array_equal(seq, g["seq"]) and
              np.array_equal(d, g["distance"]))
    return ({"value": SC_P * len(pr) / secs, "unit": "evals/s", "cores": cores, "kind": kind,
             "sample": (f"{len(pr)} of the {SC_Q} SC probes (every {SC_Q // len(pr)}th) vs the "
                        f"full P={SC_P} collection, Eamc::match "
                        f"({'std::thread over the const matcher' if cores > 1 else 'one thread'}),"
                        f" {secs:.1f} s (+{t_fill:.1f} s collection fill, untimed)")},
            {"probes": int(len(pr)), "bitwise_equal_index_seq_distance": ok})


# --------------------------------------------------------------- reference
def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: moesim compiled
    from its sources) on this box's host cores, on our arm's config (SC:
    P = 2^20, bench family seed 55); each step is a bounded sample of the batch
    (one probe per host thread).  Inputs come from the reference's own Rng
    (ref_shim), so this arm loads nothing from the product package.  Rank 0
    only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import REF_SO, RefLib
    N = max(world, args.gpus)
    cores = os.cpu_count() or 1
    if not os.path.exists(REF_SO):
        return {"impl": "reference", "unavailable": "oracle/_ref/libmoesim_ref.so was not built"}
    ref = RefLib()
    e = ref.eamc(L, E, TOPK, 1, SC_P)
    e.fill_bench(SEED, SC_P)                      # bench.cpp:61-62
    per_step = cores
    n_pr = per_step * (args.steps + args.warmup)
    probes = ref.gen_bench(SEED, L, E, n_pr, skip=SC_P)  # bench.cpp:64-66
    for i in range(args.warmup):
        e.match(probes[i * per_step:(i + 1) * per_step], threads=cores)
    secs = 0.0
    for i in range(args.warmup, args.warmup + args.steps):
        secs += e.match(probes[i * per_step:(i + 1) * per_step], threads=cores)[4]
    val = SC_P * per_step * args.steps / secs
    return {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "evals/s", "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference bench family F1 (bench.cpp:44-54, seed 55)",
        "config": sc_config(N),
        "cpu_baseline": {"value": val, "unit": "evals/s", "cores": cores, "kind": "reference",
                         "sample": (f"{per_step} probes per step (one per host thread) x "
                                    f"{args.steps} steps vs the full P={SC_P} collection")},
        "e2e": {"value": val, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-streaming", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rows", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    out = run_reference(args) if args.impl == "reference" else run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
