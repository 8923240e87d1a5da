"""SW step timing (development tool): moe_eamc_match_device on L=12, E=128,
P=10k, Q=4096 device-resident u8 probes, CUDA events on the launching stream,
L2 flushed (256 MiB write) between calls outside the events; median of 100."""
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
with torch.cuda.stream(st):
    for i in range(110):
        flush.fill_(i & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        _lib.check(_lib.lib.moe_eamc_match_device(e._h, dp.data_ptr(), 1, Q, out.data_ptr(),
                                                  C.c_void_p(st.cuda_stream)))
        b.record(st)
        b.synchronize()
        if i >= 10:
            ts.append(a.elapsed_time(b))
print(f"SW step median {np.median(ts) * 1e3:.1f} us")
