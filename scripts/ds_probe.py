"""DS decision-path timing: the 58 prefetch_priorities calls of one decode
step (L=59, E=160, P=10k; DS_P / DS_L / DS_E override) through the C ABI,
wall time per call (MOE_DEC_TIMING=1 adds the library's launch/completion
split on stderr)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

import paper_2401_14361_b200 as m  # noqa: E402
from paper_2401_14361_b200 import _lib  # noqa: E402

L = int(os.environ.get("DS_L", "59"))
E = int(os.environ.get("DS_E", "160"))
P = int(os.environ.get("DS_P", "10000"))
fam = m.gen_bench_family(55, L, E, P + 1, dtype=np.uint8)
SRV = int(os.environ.get("DS_SERVER", "0"))
e = m.Eamc(m.ModelShape(L, E, 2), m.Phase.decode, P)
e.append(fam[:P], np.arange(P, dtype=np.uint64))
if SRV:
    _lib.check(_lib.lib.moe_eamc_set_decision_server(e._h, SRV))
base = fam[P].astype(np.uint64)
probes = []
for l in range(L - 1):
    pr = base.copy()
    pr[l + 1:] = 0
    probes.append(np.ascontiguousarray(pr))
cap = L * E
out = np.zeros(cap, _lib.CAND_DTYPE)
n = C.c_uint64()
for _ in range(2):
    for l in range(L - 1):
        _lib.check(_lib.lib.moe_prefetch_priorities(e._h, probes[l].ctypes.data, l, 1,
                                                    out.ctypes.data, cap, C.byref(n)))
reps = int(os.environ.get("REPS", "5"))
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    for l in range(L - 1):
        _lib.check(_lib.lib.moe_prefetch_priorities(e._h, probes[l].ctypes.data, l, 1,
                                                    out.ctypes.data, cap, C.byref(n)))
    ts.append(time.perf_counter() - t0)
print(f"server={SRV} L={L} E={E} P={P}: C-ABI decode step {min(ts)*1e3:.3f} ms "
      f"({min(ts)/(L-1)*1e6:.1f} us/call)", flush=True)
