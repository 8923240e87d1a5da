"""Per-layer decision latency at DS (development tool): the C-ABI call
moe_prefetch_priorities for each current layer l of a decode step, min over
repetitions, to separate the output-size-dependent cost ((L-l-1)*E candidates)
from the fixed cost."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

import paper_2401_14361_b200 as m  # noqa: E402
from paper_2401_14361_b200 import _lib  # noqa: E402

L, E = 59, 160
P = int(os.environ.get("DEC_P", "10000"))
REPS = int(os.environ.get("DEC_REPS", "12"))
fam = m.gen_bench_family(55, L, E, P + 1, dtype=np.uint8)
e = m.Eamc(m.ModelShape(L, E, 2), m.Phase.decode, P)
e.append(fam[:P], np.arange(P, dtype=np.uint64))
base = fam[P].astype(np.uint64)
probes = []
for l in range(L - 1):
    pr = base.copy()
    pr[l + 1:] = 0
    probes.append(np.ascontiguousarray(pr))
cap = L * E
out = np.zeros(cap, _lib.CAND_DTYPE)
n = C.c_uint64()
best = np.full(L - 1, 1e9)
only = os.environ.get("DEC_L")  # time one layer only (MOE_DEC_TIMING=1 then prints its phases)
if only is not None:
    l = int(only)
    for rep in range(200):
        _lib.check(_lib.lib.moe_prefetch_priorities(e._h, probes[l].ctypes.data, l, 1,
                                                    out.ctypes.data, cap, C.byref(n)))
    print(f"l={l}: {n.value} candidates returned", flush=True)
    sys.exit(0)
for rep in range(REPS):
    for l in range(L - 1):
        t0 = time.perf_counter()
        _lib.check(_lib.lib.moe_prefetch_priorities(e._h, probes[l].ctypes.data, l, 1,
                                                    out.ctypes.data, cap, C.byref(n)))
        dt = time.perf_counter() - t0
        if rep >= min(2, REPS - 1):
            best[l] = min(best[l], dt)
for l in (0, 1, 10, 29, 45, 56, 57):
    print(f"l={l:2d} candidates={(L - l - 1) * E:5d}  min {best[l] * 1e6:6.1f} us")
print(f"mean of per-layer minima {best.mean() * 1e6:.1f} us")
