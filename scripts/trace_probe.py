"""DS tracing micro-run for profiling (1M tokens x 59 layers x top-6 u8 ids;
TRACE_R requests of equal length, default 1,000)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2401_14361_b200 as m
from paper_2401_14361_b200 import _lib
L, E, k, T = 59, 160, 6, 1_000_000
R = int(os.environ.get("TRACE_R", T // 1000))
rng = np.random.default_rng(1001)
zipf = 1.0 / np.arange(1, E + 1) ** 1.2
basei = rng.choice(E, size=(T, L), p=zipf / zipf.sum()).astype(np.uint16)
picks = ((basei[:, :, None] + np.arange(k, dtype=np.uint16)[None, None, :]) % E).astype(np.uint8)
d_p = torch.from_numpy(picks).cuda()
d_o = torch.from_numpy(np.linspace(0, T, R + 1).astype(np.int64)).cuda()
d_c = torch.zeros((R, L, E), dtype=torch.int32, device="cuda")
d_b = torch.zeros(1, dtype=torch.int32, device="cuda")
sh = m.ModelShape(L, E, k).c()
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for it in range(int(os.environ.get("TRACE_ITERS", "8"))):
    ev[0].record(st)
    _lib.check(_lib.lib.moe_eam_trace_device(C.byref(sh), d_p.data_ptr(), 1, T, d_o.data_ptr(), R,
                                             d_c.data_ptr(), d_b.data_ptr(), C.c_void_p(st.cuda_stream)))
    ev[1].record(st)
    torch.cuda.synchronize()
    print("trace ms", ev[0].elapsed_time(ev[1]))
