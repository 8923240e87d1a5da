#!/usr/bin/env python
"""bench.py -- EAM-vs-EAMC distance evals/s on B200 (BASELINE.json `metric`).

Default workload (BASELINE.json configs[1], "SW"): Switch-Transformers-base-128
shape (L=12, E=128, top-1), an EAMC of P=10,000 entries per GPU matched
against a 4,096-probe batch.  Inputs are the reference benchmark's own
synthetic EAM family (bench.cpp:44-54, seed 55): the first P*N EAMs of the
stream are the collection (rank r owns [r*P, (r+1)*P)), the next Q are the
probes.  A step = one Eamc::match pass of the probe batch over the whole
collection; at N>1 the collection is P-sharded and the per-shard argmins are
merged over NCCL (all_gather + device lexicographic merge): weak scaling.

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
P_PER_GPU, Q = 10_000, 4096
SEED = 55
STREAM_P, STREAM_Q = 1 << 20, 8   # SC streaming regime (P >= 1M), north-star HBM target
BATCH_Q = 65536                  # SC batch regime (BASELINE configs[4]: 65k-query batch)


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

    # ---- collection shard + probes (host-generated, reference bench stream)
    P = P_PER_GPU
    shard = m.gen_bench_family(SEED, L, E, P, skip=rank * P, dtype=np.uint8)
    probes_u8 = m.gen_bench_family(SEED, L, E, Q, skip=N * P, dtype=np.uint8)
    eamc = m.Eamc(m.ModelShape(L, E, TOPK), m.Phase.decode, P, device=local)
    eamc.append(shard, np.arange(rank * P, (rank + 1) * P, dtype=np.uint64))
    _lib.check(_lib.lib.moe_eamc_set_index_base(eamc._h, rank * P))

    d_probes = torch.from_numpy(probes_u8).to(dev)
    d_out = torch.empty((Q, 3), dtype=torch.float64, device=dev)      # moe_match[Q]
    d_parts = torch.empty((N * Q, 3), dtype=torch.float64, device=dev)
    d_final = torch.empty((Q, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step_device():
        _lib.check(_lib.lib.moe_eamc_match_device(eamc._h, d_probes.data_ptr(), 1, Q,
                                                  d_out.data_ptr(), sp))
        if N > 1:
            dist.all_gather_into_tensor(d_parts, d_out)
            _lib.check(_lib.lib.moe_match_merge_device(d_parts.data_ptr(), N, Q,
                                                       d_final.data_ptr(), sp))
            return d_final
        return d_out

    # warmup
    for _ in range(args.warmup):
        step_device()
    barrier()

    # ---- timed region: K steps, L2 flushed between steps (outside the events)
    def timed(profile):
        if profile:
            _lib.check(_lib.lib.moe_eamc_set_profiling(eamc._h, 1))
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        barrier()
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            step_device()
            evs[i][1].record(stream)
        barrier()
        return [a.elapsed_time(b) for a, b in evs]

    clocks = ClockSampler(local)
    time.sleep(0.05)
    ms_steps = timed(False)
    clk = clocks.stop()
    # Per-kernel times come from a second, identical pass with the library's
    # per-kernel events on: events between the kernels break the programmatic
    # dependent launch overlap, so that pass is not the one `value` is timed on.
    ms_prof = timed(True)
    kms = (C.c_double * 3)()
    kcalls = (C.c_uint64 * 3)()
    _lib.check(_lib.lib.moe_eamc_kernel_times(eamc._h, kms, kcalls))
    _lib.check(_lib.lib.moe_eamc_set_profiling(eamc._h, 0))
    t_total = torch.tensor([sum(ms_steps)], dtype=torch.float64, device=dev)
    if N > 1:
        dist.all_reduce(t_total, op=dist.ReduceOp.MAX)
    t_ms = float(t_total.item())
    evals_per_step = P * N * Q
    value = evals_per_step * args.steps / (t_ms / 1e3)
    # per step: k_prep_u8, k_tc2_screen, k_refine, and the device-gated exact
    # pass k_match<1,1,1> + k_merge_partials (launched every step, exit at once
    # unless a candidate bucket overflowed); + k_merge for N > 1
    gpu_launches = args.steps * (5 + (1 if N > 1 else 0))

    # result of the last step, for the parity sample
    res = step_device().cpu().numpy().view(np.uint8).reshape(Q, 24).copy().view(
        _lib.MATCH_DTYPE)[:, 0]

    # ---- roofline of the dominant kernel (screen pass), live CUDA events
    hbm_peak, tf_peak, peak_kind = load_peaks()
    screen_ms = kms[1] / max(kcalls[1], 1)
    ops_alg = 2.0 * L * E * P * Q
    bytes_alg = P * L * E * 1 + Q * L * E * 1 + 24 * Q
    roofline = {
        "bound": "tensor",
        "kernel": "k_tc2_screen (tcgen05.mma.cta_group::2 kind::f16, 256x256 tiles, screen pass)",
        "achieved": ops_alg / (screen_ms / 1e3) / 1e12, "peak": tf_peak, "unit": "TFLOP/s",
        "frac": ops_alg / (screen_ms / 1e3) / 1e12 / tf_peak,
        "traffic": ncu_traffic("sw_screen"),
        "alg_ops_per_launch": ops_alg, "alg_bytes_per_launch": bytes_alg,
        "launch_ms": screen_ms,
        "share_of_step": screen_ms / (sum(ms_prof) / args.steps),
        "kernel_times": "per-kernel CUDA events on the launching stream, from a profiled pass of "
                        "the same K steps (ms_per_step_profiled)",
        "note": (f"peak = {peak_kind} dense bf16 (MEASURED_PEAKS.json); ops = 2*L*E*P*Q "
                 "(SURVEY.md 8d), executed as one fp16 tensor-core GEMM over unit-normalised "
                 "rows (K=L*E), fp32 accumulate in TMEM; the operands are the fp16 copies "
                 "(2 B/count), so ncu traffic is ~2x the u8 algorithmic bytes. HBM view: "
                 f"{bytes_alg / (screen_ms / 1e3) / 1e9:.1f} GB/s of {hbm_peak:.0f}"),
    }

    # ---- e2e: public host API, pinned u64 probes in, results out, every step
    import torch as _t
    h_probes = _t.from_numpy(probes_u8.astype(np.uint64)).pin_memory()
    h_out = np.zeros(Q, _lib.MATCH_DTYPE)
    h_parts = _t.empty((N * Q, 3), dtype=_t.float64, device=dev)

    def step_e2e():
        _lib.check(_lib.lib.moe_eamc_match(eamc._h, h_probes.data_ptr(), Q, h_out.ctypes.data,
                                           None))
        if N > 1:
            mine = _t.from_numpy(h_out.view(np.float64).reshape(Q, 3)).to(dev)
            dist.all_gather_into_tensor(h_parts, mine)
            _lib.check(_lib.lib.moe_match_merge_device(h_parts.data_ptr(), N, Q,
                                                       d_final.data_ptr(), sp))
            return d_final.cpu()
        return h_out

    for _ in range(min(args.warmup, 3)):
        step_e2e()
    barrier()
    e2e_steps = max(3, min(args.steps, 50))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_e2e()
    if N > 1:
        dist.barrier()
    t_e2e = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if N > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_val = evals_per_step * e2e_steps / float(t_e2e.item())

    # the same through moe_eamc_match_packed: host probes already narrow (u8,
    # as traced counts of this workload are), 6.3 MB per step instead of 50 MB
    h_probes8 = _t.from_numpy(probes_u8).pin_memory()

    def step_e2e_packed():
        _lib.check(_lib.lib.moe_eamc_match_packed(eamc._h, h_probes8.data_ptr(), 1, Q,
                                                  h_out.ctypes.data, None))

    for _ in range(min(args.warmup, 3)):
        step_e2e_packed()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_e2e_packed()
    e2e_packed_val = P * Q * e2e_steps / (time.perf_counter() - t0)
    host_threads = int(_lib.lib.moe_host_threads())

    # ---- the other SURVEY 8 rows (prefetch decisions, construction, tracing, MIX)
    rows = None
    if N == 1 and not args.no_rows:
        rows = run_rows(args, m, _lib, torch, dev, sp, stream)

    # ---- streaming regime (north-star target: >= 60% HBM roofline at P >= 1M)
    streaming = None
    if not args.no_streaming:
        streaming = run_streaming(args, m, _lib, torch, dist, rank, N, dev, sp, flush, hbm_peak,
                                  peak_kind)

    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic: reference bench family F1 (bench.cpp:44-54, seed 55)",
            "config": {
                "workload": (f"SW (BASELINE configs[1]): Switch-base-128 shape L={L} E={E} "
                             f"top-{TOPK}, EAMC P={P} per GPU (P_total={P * N}), Q={Q} probes"),
                "L": L, "E": E, "P_per_gpu": P, "P_total": P * N, "Q": Q, "count_bytes": 1,
                "l2": "flushed between timed steps (256 MiB write, outside the events)",
                "parallelism": (f"P-sharded x{N}, NCCL all_gather + device lexicographic merge"
                                if N > 1 else "single GPU"),
            },
            "roofline": roofline,
            "e2e": {"value": e2e_val, "unit": "evals/s", "steps": e2e_steps,
                    "api": ("moe_eamc_match (host u64 probes, pinned) + D2H results; u64 "
                            f"narrowed to u8 on {host_threads} host threads inside the call"),
                    "h2d_bytes_per_step": int(Q * L * E * 1),
                    "d2h_bytes_per_step": int(Q * 24)},
            "e2e_packed_u8": {"value": e2e_packed_val * N, "unit": "evals/s", "steps": e2e_steps,
                              "api": "moe_eamc_match_packed (host u8 probes, pinned) + D2H results "
                                     "(per-rank, scaled by N)",
                              "h2d_bytes_per_step": int(Q * L * E), "d2h_bytes_per_step": int(Q * 24)},
            "gpu_launches": gpu_launches,
            "ms_per_step_profiled": sum(ms_prof) / args.steps,
            "kernel_ms_per_step": {"prep": kms[0] / max(kcalls[0], 1), "screen": screen_ms,
                                   "refine": kms[2] / max(kcalls[2], 1)},
            "clocks": clk,
        }
        if streaming:
            out["streaming"] = streaming
        if rows:
            out["rows"] = rows
        if N == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"], out["parity_sample"] = cpu_baseline(args, probes_u8, res)
    if N > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def _ref_or_none():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import REF_SO, Oracle, RefLib
    return (RefLib() if os.path.exists(REF_SO) else None), Oracle()


def run_rows(args, m, _lib, torch, dev, sp, stream):
    """Measured lines for SURVEY 8 rows beyond the headline matcher, each with
    the reference CPU path (oracle/_ref) timed on this box beside it."""
    from concurrent.futures import ThreadPoolExecutor
    hbm_peak, _, peak_kind = load_peaks()
    ref, orc = _ref_or_none()
    cores = os.cpu_count() or 1
    out = {}

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

    orders = decode_step()
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        orders = decode_step()
    t_gpu = (time.perf_counter() - t0) / reps
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
        ns = 20
        e3p = m.Eamc(m.ModelShape(L3, E3), m.Phase.decode, P3)
        e3p.append(fam3[:P3], np.arange(P3, dtype=np.uint64))
        slots_p = e3p.build(steps_all[:ns])
        t0 = time.perf_counter()
        rs = [er.insert(x) for x in steps_all[:ns]]
        t_cpu = (time.perf_counter() - t0) / ns
        row.update({"cpu_us_per_step": t_cpu * 1e6, "cpu_cores": 1, "cpu_kind": "reference",
                    "speedup": t_cpu / (t_gpu / n3),
                    "parity_first_steps": bool(list(slots_p[:ns]) == rs)})
    out["construction"] = row

    # -- A2/K1 tracing, DS shape: T = 1M router tokens x 59 layers x top-6 ids
    #    (u8, resident) -> R = 1000 per-request count matrices
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
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(10)]
    for a, b in evs:
        a.record(stream)
        trace_dev()
        b.record(stream)
    torch.cuda.synchronize()
    t_dev = sum(a.elapsed_time(b) for a, b in evs) / len(evs) / 1e3
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
           "roofline": {"bound": "hbm", "achieved": bytes_alg / t_dev / 1e9, "peak": hbm_peak,
                        "unit": "GB/s", "frac": bytes_alg / t_dev / 1e9 / hbm_peak,
                        "alg_bytes": bytes_alg, "note": f"peak = {peak_kind} HBM"},
           "e2e_ms": t_e2e * 1e3,
           "e2e_api": ("moe_eam_trace (host u8 ids + host u64 counts accumulated; transfers "
                       "through pinned staging inside the call)")}
    ns = 20_000
    t0 = time.perf_counter()
    rc, ref_counts = orc.trace(L4, E4, k4, picks[:ns].astype(np.uint32),
                               np.arange(0, ns + 1, 1000, dtype=np.uint64))
    t_cpu = time.perf_counter() - t0
    row.update({"cpu_picks_per_s": ns * L4 * k4 / t_cpu, "cpu_cores": 1, "cpu_kind": "port",
                "cpu_sample": f"{ns} tokens (oracle restatement of workload.cpp:166-181 + "
                              "Eam::record)",
                "parity_sample": bool(rc == 0 and np.array_equal(host_counts[:ns // 1000],
                                                                 ref_counts))})
    out["tracing"] = row
    del d_picks, d_counts

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
    t0 = time.perf_counter()
    got = []
    for q in range(Q5):
        _lib.check(_lib.lib.moe_prefetch_priorities(e5._h, pp[q].ctypes.data, q % (L5 - 1), 1,
                                                    o5p.ctypes.data, cap5, C.byref(n5)))
        if q < 64:
            got.append(o5p[:n5.value].copy())
    t5p = time.perf_counter() - t0
    row = {"workload": f"MIX prefetch: L={L5} E={E5}, EAMC P={P5}, {Q5} prefetch_priorities "
                       "calls (l = q mod (L-1)) + floor filter, C ABI with host buffers",
           "us_per_decision": t5p / Q5 * 1e6, "decisions_per_s": Q5 / t5p}
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


def run_streaming(args, m, _lib, torch, dist, rank, N, dev, sp, flush, hbm_peak, peak_kind):
    assert sp.value, "streaming leg must run on the explicit bench stream"
    """SC streaming regime: P = 2^20 entries (sharded P/N), Q = 8 probes."""
    P = STREAM_P // N
    shard = m.gen_bench_family(SEED, L, E, P, skip=rank * P, dtype=np.uint8)
    probes = m.gen_bench_family(SEED, L, E, STREAM_Q, skip=STREAM_P, dtype=np.uint8)
    e = m.Eamc(m.ModelShape(L, E, TOPK), m.Phase.decode, P, device=dev.index)
    e.append(shard, np.arange(rank * P, (rank + 1) * P, dtype=np.uint64))
    del shard
    _lib.check(_lib.lib.moe_eamc_set_index_base(e._h, rank * P))
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

    def timed(step_fn, steps, profile):
        if N > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if profile:
            _lib.check(_lib.lib.moe_eamc_set_profiling(e._h, 1))
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        for i in range(steps):
            flush.zero_()
            evs[i][0].record(stream)
            step_fn()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        kms = (C.c_double * 3)()
        kc = (C.c_uint64 * 3)()
        if profile:
            _lib.check(_lib.lib.moe_eamc_kernel_times(e._h, kms, kc))
            _lib.check(_lib.lib.moe_eamc_set_profiling(e._h, 0))
        t = torch.tensor([sum(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64,
                         device=dev)
        if N > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), kms[1] / max(kc[1], 1)

    for _ in range(3):
        step()
    steps = 30
    t_ms, _ = timed(step, steps, False)   # value: no per-kernel events (PDL intact)
    _, screen_ms = timed(step, steps, True)
    bytes_alg = P * L * E * 1 + STREAM_Q * L * E * 1 + 24 * STREAM_Q
    ach = bytes_alg / (screen_ms / 1e3) / 1e9
    out = {
        "workload": f"SC streaming: P={STREAM_P} (P/GPU={P}), Q={STREAM_Q}, L={L} E={E}, u8",
        "value": P * N * STREAM_Q * steps / (t_ms / 1e3), "unit": "evals/s",
        "ms_per_step": t_ms / steps, "steps": steps,
        "roofline": {"bound": "hbm",
                     "kernel": "k_tci8_screen<4> (tcgen05.mma kind::i8, block-diagonal probes)",
                     "achieved": ach,
                     "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                     "traffic": ncu_traffic("sc_screen"), "launch_ms": screen_ms,
                     "alg_bytes_per_launch": bytes_alg,
                     "note": f"peak = {peak_kind} HBM copy bandwidth (MEASURED_PEAKS.json)"},
    }
    if args.no_batch:
        return out
    # SC batch regime (BASELINE configs[4]): the same collection, a 65,536-probe batch;
    # compute-bound by construction, so its roofline is the tensor pipe
    QB = BATCH_Q
    pb = torch.from_numpy(m.gen_bench_family(SEED, L, E, QB, skip=STREAM_P + STREAM_Q,
                                             dtype=np.uint8)).to(dev)
    b_out = torch.empty((QB, 3), dtype=torch.float64, device=dev)
    b_parts = torch.empty((N * QB, 3), dtype=torch.float64, device=dev)
    b_fin = torch.empty((QB, 3), dtype=torch.float64, device=dev)

    def bstep():
        _lib.check(_lib.lib.moe_eamc_match_device(e._h, pb.data_ptr(), 1, QB, b_out.data_ptr(),
                                                  sp))
        if N > 1:
            dist.all_gather_into_tensor(b_parts, b_out)
            _lib.check(_lib.lib.moe_match_merge_device(b_parts.data_ptr(), N, QB,
                                                       b_fin.data_ptr(), sp))

    bstep()
    bsteps = 3
    tb_ms, _ = timed(bstep, bsteps, False)
    _, bscreen_ms = timed(bstep, bsteps, True)
    ops = 2.0 * L * E * P * QB
    _, tf_peak, _ = load_peaks()
    out["batch"] = {
        "workload": f"SC batch: P={STREAM_P} (P/GPU={P}), Q={QB}, L={L} E={E}, u8",
        "value": P * N * QB * bsteps / (tb_ms / 1e3), "unit": "evals/s",
        "ms_per_step": tb_ms / bsteps, "steps": bsteps,
        "roofline": {"bound": "tensor",
                     "kernel": "k_tc2_screen (tcgen05.mma.cta_group::2 kind::f16)",
                     "achieved": ops / (bscreen_ms / 1e3) / 1e12, "peak": tf_peak,
                     "unit": "TFLOP/s", "frac": ops / (bscreen_ms / 1e3) / 1e12 / tf_peak,
                     "launch_ms": bscreen_ms, "alg_ops_per_launch": ops,
                     "frac_of_nominal_2250": ops / (bscreen_ms / 1e3) / 1e12 / 2250.0,
                     "note": ("ops = 2*L*E*P*Q (SURVEY.md 8d); peak = measured cuBLAS bf16 "
                              "8192^3 burst (MEASURED_PEAKS.json, taken under the 1000 W cap); "
                              "frac_of_nominal_2250 = against the nominal dense fp16 peak")},
    }
    return out


def cpu_baseline(args, probes_u8, gpu_res):
    """The reference CPU path (oracle/_ref = moesim compiled from its sources) on
    this box's host cores, bounded sample of the SW workload; also checks the
    sampled probes against the GPU result bit for bit."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import REF_SO, Oracle, RefLib
    import paper_2401_14361_b200 as m
    fam = m.gen_bench_family(SEED, L, E, P_PER_GPU, dtype=np.uint64)
    cores = os.cpu_count() or 1
    if os.path.exists(REF_SO):
        ref = RefLib()
        kind = "reference"
        e = ref.eamc(L, E, TOPK, 1, P_PER_GPU)
        for x in fam:
            e.insert(x)

        def run(pr):
            idx, seq, d, f, secs = e.match(pr, threads=cores)
            return idx, d, secs
    else:
        orc = Oracle()
        kind = "port"
        cores = 1

        def run(pr):
            t0 = time.perf_counter()
            idx, seq, d, f = orc.match(fam, np.arange(P_PER_GPU, dtype=np.uint64), pr)
            return idx, d, time.perf_counter() - t0
    chunk = max(cores * 2, 8)
    done, secs = 0, 0.0
    ok = True
    while done < Q and secs < args.cpu_seconds:
        pr = probes_u8[done:done + chunk].astype(np.uint64)
        idx, d, s = run(pr)
        secs += s
        ok &= bool(np.array_equal(idx, gpu_res["index"][done:done + chunk]) and
                   np.array_equal(d, gpu_res["distance"][done:done + chunk]))
        done += len(pr)
    val = P_PER_GPU * done / secs
    return ({"value": val, "unit": "evals/s", "cores": cores, "kind": kind,
             "sample": (f"{done} of {Q} SW probes vs P={P_PER_GPU} (Eamc::match, "
                        f"{'std::thread over the const matcher' if cores > 1 else 'one thread'}), "
                        f"{secs:.1f} s")},
            {"probes": done, "bitwise_equal_index_and_distance": ok})


# --------------------------------------------------------------- reference
def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref) on this box's host
    cores, on our arm's config; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import REF_SO, Oracle, RefLib
    import paper_2401_14361_b200 as m
    N = max(world, args.gpus)
    P = P_PER_GPU * N
    fam = m.gen_bench_family(SEED, L, E, P + Q, dtype=np.uint64)
    cores = os.cpu_count() or 1
    if os.path.exists(REF_SO):
        kind = "reference"
        e = RefLib().eamc(L, E, TOPK, 1, P)
        for x in fam[:P]:
            e.insert(x)

        def run(pr):
            return e.match(pr, threads=cores)[4]
    else:
        kind = "port"
        orc = Oracle()
        cores = 1

        def run(pr):
            t0 = time.perf_counter()
            orc.match(fam[:P], np.arange(P, dtype=np.uint64), pr)
            return time.perf_counter() - t0
    per_step = max(cores, 4)
    probes = fam[P:]
    for i in range(args.warmup):
        run(probes[:per_step])
    secs = 0.0
    for i in range(args.steps):
        s0 = (i * per_step) % (Q - per_step)
        secs += run(probes[s0:s0 + per_step])
    val = P * per_step * args.steps / secs
    return {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "evals/s", "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference bench family F1 (bench.cpp:44-54, seed 55)",
        "config": {"workload": (f"SW (BASELINE configs[1]): L={L} E={E} top-{TOPK}, EAMC "
                                f"P={P}, Q={Q}; each step a {per_step}-probe sample"),
                   "L": L, "E": E, "P_total": P, "Q": Q},
        "cpu_baseline": {"value": val, "unit": "evals/s", "cores": cores, "kind": kind,
                         "sample": f"{per_step} probes per step x {args.steps} steps"},
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
    ap.add_argument("--no-batch", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    out = run_reference(args) if args.impl == "reference" else run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
