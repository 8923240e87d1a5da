"""MIX decision timing in the bench's call pattern (development tool): P=300
collection (L=32, E=8), 1,000 prefetch_priorities calls with unrelated probes
at layer q mod 31, launched and through the one-CTA decision server
(MOE_DEC_TIMING=1 adds the launched kernel's phase split on stderr)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

import paper_2401_14361_b200 as m  # noqa: E402
from paper_2401_14361_b200 import _lib  # noqa: E402

L, E, P, Q = 32, 8, 300, 1000
fam = m.gen_bench_family(55, L, E, P + Q, dtype=np.uint8)
e = m.Eamc(m.ModelShape(L, E, 2), m.Phase.decode, P)
e.append(fam[:P], np.arange(P, dtype=np.uint64))
pp = []
for q in range(Q):
    x = np.ascontiguousarray(fam[P + q].astype(np.uint64))
    x[q % (L - 1) + 1:] = 0
    pp.append(x)
cap = L * E
out = np.zeros(cap, _lib.CAND_DTYPE)
n = C.c_uint64()
fn, h = _lib.lib.moe_prefetch_priorities, e._h
for srv in (0, 8):
    _lib.check(_lib.lib.moe_eamc_set_decision_server(h, srv))
    for q in range(50):
        fn(h, pp[q].ctypes.data, q % (L - 1), 1, out.ctypes.data, cap, C.byref(n))
    best = 1e9
    for rep in range(3):
        t0 = time.perf_counter()
        for q in range(Q):
            fn(h, pp[q].ctypes.data, q % (L - 1), 1, out.ctypes.data, cap, C.byref(n))
        best = min(best, time.perf_counter() - t0)
    print(f"server={srv}: {best / Q * 1e6:.1f} us per decision", flush=True)
_lib.check(_lib.lib.moe_eamc_set_decision_server(h, 0))
