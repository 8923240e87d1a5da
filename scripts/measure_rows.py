"""Quick timing of the non-matcher rows on one GPU (development tool).

    python scripts/measure_rows.py [--rows build,trace,prefetch]

build    : NL shape (L=24, E=128) construction replay, at-capacity steps/s
trace    : DS shape (L=59, E=160, top-6) K1 tracing of T router tokens
prefetch : DS shape decode step = 58 prefetch_priorities calls (P entries)
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2401_14361_b200 as m
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="build,trace,prefetch")
    ap.add_argument("--P", type=int, default=10_000)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--tokens", type=int, default=1_000_000)
    a = ap.parse_args()
    rows = a.rows.split(",")
    if "build" in rows:
        L, E, P, n = 24, 128, a.P, a.steps
        fam = m.gen_bench_family(3, L, E, P + n)
        e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
        e.build(fam[:P])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        slots = e.build(fam[P:])
        t = time.perf_counter() - t0
        print(json.dumps({"row": "build", "L": L, "E": E, "P": P, "steps": n,
                          "us_per_step": t / n * 1e6, "steps_per_s": n / t,
                          "evals_per_s": n * P / t, "replaced": int((slots >= 0).sum())}))
    if "trace" in rows:
        L, E, k, T = 59, 160, 6, a.tokens
        R = T // 1000
        rng = np.random.default_rng(0)
        # skewed top-k ids (80% from 8 hot experts per layer), distinct within a token
        hot = rng.integers(0, E, size=(L, 8))
        picks = np.empty((T, L, k), np.uint8)
        for l in range(L):
            base = rng.random((T, 1)) < 0.8
            perm = np.argsort(rng.random((T, E)), axis=1)[:, :k]
            hotsel = np.stack([np.roll(hot[l], s)[:k] for s in range(1)], 0)[0]
            picks[:, l, :] = np.where(base, hotsel[None, :], perm)
        offs = np.arange(0, T + 1, 1000, dtype=np.uint64)
        s = m.ModelShape(L, E, k)
        m.trace_requests(s, picks[:1000], offs[:2])
        t0 = time.perf_counter()
        out = m.trace_requests(s, picks, offs)
        t = time.perf_counter() - t0
        print(json.dumps({"row": "trace(host api, incl. H2D of picks)", "T": T, "R": R,
                          "ms": t * 1e3, "picks_per_s": T * L * k / t,
                          "sum_ok": int(out.sum()) == T * L * k}))
    if "prefetch" in rows:
        L, E, P = 59, 160, a.P
        fam = m.gen_bench_family(5, L, E, P + 1)
        s = m.ModelShape(L, E, 6)
        e = m.Eamc(s, m.Phase.decode, P)
        e.build(fam[:P])
        cur = fam[P].copy()
        m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=cur), e, 3)
        t0 = time.perf_counter()
        n = 0
        for l in range(L - 1):
            probe = cur.copy()
            probe[l + 1:] = 0
            m.prefetch_order(m.Eam(s, m.EamKind.iteration, counts=probe), e, l)
            n += 1
        t = time.perf_counter() - t0
        print(json.dumps({"row": "prefetch decode step (58 calls)", "P": P, "ms_per_step": t * 1e3,
                          "ms_per_call": t / n * 1e3}))


if __name__ == "__main__":
    main()
