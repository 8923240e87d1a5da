"""SW workload (L=12, E=128, P=10k, Q=4096) through the device match API, a
few calls -- the target for ncu captures of k_prep / screen / k_refine."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_14361_b200 as m  # noqa: E402
from paper_2401_14361_b200 import _lib  # noqa: E402

L, E, P, Q = 12, 128, 10000, 4096
fam = m.gen_bench_family(55, L, E, P + Q, dtype=np.uint8)
e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
e.append(fam[:P], np.arange(P, dtype=np.uint64))
dp = torch.from_numpy(fam[P:]).cuda()
out = torch.empty((Q, 3), dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
for _ in range(int(os.environ.get("N_CALLS", "3"))):
    _lib.check(_lib.lib.moe_eamc_match_device(e._h, dp.data_ptr(), 1, Q, out.data_ptr(),
                                              C.c_void_p(st.cuda_stream)))
torch.cuda.synchronize()
print("ok")
