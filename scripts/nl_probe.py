"""NL construction replay timing: L=24, E=128, capacity P=10k, at-capacity
Eamc::insert steps through moe_eamc_build (blocked vs stepwise replay)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_14361_b200 as m  # noqa: E402

L, E, P = 24, 128, 10_000
n = int(os.environ.get("NL_STEPS", "20000"))
fam = m.gen_bench_family(3, L, E, P + n, dtype=np.uint8)
steps = fam[P:].astype(np.uint64)
e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
e.append(fam[:P], np.arange(P, dtype=np.uint64))
e.build(steps[:600])  # warm-up (kernels, buffers)
torch.cuda.synchronize()
t0 = time.perf_counter()
slots = e.build(steps[600:])
dt = time.perf_counter() - t0
k = n - 600
print(f"{os.environ.get('MOE_REPLAY_STEPWISE', '0')=} {os.environ.get('MOE_REPLAY_BLOCK', '512')=}: "
      f"{k} steps {dt*1e3:.1f} ms = {dt/k*1e6:.2f} us/step, {k*P/dt:.3e} evals/s")
