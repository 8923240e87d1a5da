"""K1 tracing under compute-sanitizer (development tool):

    compute-sanitizer --tool memcheck python scripts/sanitize_trace.py

Small DS / SW / MIX / odd shapes through the host API (lane, own and generic
kernels), totals checked against T * L * k."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_14361_b200 as m  # noqa: E402

rng = np.random.default_rng(3)
for (L, E, k, T, R) in [(59, 160, 6, 4096, 7), (12, 128, 1, 20000, 11), (32, 8, 2, 9000, 13),
                        (7, 40, 2, 3000, 5), (7, 40, 3, 3000, 5), (59, 160, 6, 500, 200)]:
    picks = rng.integers(0, E, size=(T, L, k)).astype(np.uint8)
    offs = np.linspace(0, T, R + 1).astype(np.uint64)
    got = m.trace_requests(m.ModelShape(L, E, k), picks, offs)
    assert int(got.sum()) == T * L * k, (L, E, k)
    print(L, E, k, "ok", flush=True)
