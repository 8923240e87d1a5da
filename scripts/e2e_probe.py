"""Time the host match API (pinned u64 probes -> results) on the SW workload."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_14361_b200 as m
from paper_2401_14361_b200 import _lib
L, E, P, Q = 12, 128, 10000, 4096
fam = m.gen_bench_family(55, L, E, P + Q, dtype=np.uint8)
e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
e.append(fam[:P], np.arange(P, dtype=np.uint64))
hp = torch.from_numpy(fam[P:].astype(np.uint64)).pin_memory()
out = np.zeros(Q, _lib.MATCH_DTYPE)
for _ in range(3):
    _lib.check(_lib.lib.moe_eamc_match(e._h, hp.data_ptr(), Q, out.ctypes.data, None))
t0 = time.perf_counter()
n = 30
for _ in range(n):
    _lib.check(_lib.lib.moe_eamc_match(e._h, hp.data_ptr(), Q, out.ctypes.data, None))
t = (time.perf_counter() - t0) / n
print(os.environ.get("MOE_PIPE_CHUNK", "default"), f"{t*1e3:.3f} ms/step", f"{P*Q/t:.3e} evals/s")
