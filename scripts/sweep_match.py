"""Matcher sweep on one GPU: screen-kernel time vs probe-batch size Q.

    python scripts/sweep_match.py [--P 1048576] [--qs 1,2,4,8,16,64,4096]

Prints one JSON object per (P, Q) with the per-kernel device times measured
by the library's CUDA-event instrumentation (moe_eamc_set_profiling), the
algorithmic HBM bytes / integer ops of the screen pass and their rates.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2401_14361_b200 as m
    from paper_2401_14361_b200 import _lib
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=1 << 20)
    ap.add_argument("--L", type=int, default=12)
    ap.add_argument("--E", type=int, default=128)
    ap.add_argument("--qs", default="1,2,4,8,16,64,4096")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    L, E, P = a.L, a.E, a.P
    fam = m.gen_bench_family(55, L, E, P, dtype=np.uint8)
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
    e.append(fam, np.arange(P, dtype=np.uint64))
    del fam
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sp = C.c_void_p(stream.cuda_stream)
    for Q in [int(x) for x in a.qs.split(",")]:
        pr = torch.from_numpy(m.gen_bench_family(55, L, E, Q, skip=P, dtype=np.uint8)).cuda()
        out = torch.empty((Q, 3), dtype=torch.float64, device="cuda")
        for _ in range(2):
            _lib.check(_lib.lib.moe_eamc_match_device(e._h, pr.data_ptr(), 1, Q, out.data_ptr(),
                                                      sp))
        _lib.check(_lib.lib.moe_eamc_set_profiling(e._h, 1))
        for _ in range(a.reps):
            flush.zero_()
            _lib.check(_lib.lib.moe_eamc_match_device(e._h, pr.data_ptr(), 1, Q, out.data_ptr(),
                                                      sp))
        ms = (C.c_double * 3)()
        calls = (C.c_uint64 * 3)()
        _lib.check(_lib.lib.moe_eamc_kernel_times(e._h, ms, calls))
        _lib.check(_lib.lib.moe_eamc_set_profiling(e._h, 0))
        t = [ms[i] / max(calls[i], 1) for i in range(3)]
        byt = P * L * E + Q * L * E + 24 * Q
        ops = 2.0 * L * E * P * Q
        print(json.dumps({"P": P, "Q": Q, "prep_ms": t[0], "screen_ms": t[1], "refine_ms": t[2],
                          "screen_GBps": byt / t[1] / 1e6, "screen_TOPS": ops / t[1] / 1e9,
                          "evals_per_s": P * Q / ((t[0] + t[1] + t[2]) / 1e3)}), flush=True)


if __name__ == "__main__":
    main()
