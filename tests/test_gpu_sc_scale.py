"""SC at its own size (BASELINE configs[4]): P = 2^20 entries (12 x 128, the
reference bench family, seed 55), matched on the device with the batch
(Q = 65,536, tcgen05 f16 screen) and streaming (Q = 8, tcgen05 i8 screen)
paths; sampled probes compared bitwise with the reference library itself
(oracle/_ref: Eamc::match over the same 2^20 entries, std::thread over
probes), or with the C oracle when the reference is not built."""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

L, E, P, SEED = 12, 128, 1 << 20, 55


@pytest.fixture(scope="module")
def sc(m):
    import torch
    fam = m.gen_bench_family(SEED, L, E, P, dtype=np.uint8)
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
    e.append(fam, np.arange(P, dtype=np.uint64))
    return e, fam


def _device_match(m, e, probes):
    import ctypes as C
    import torch
    from paper_2401_14361_b200 import _lib
    st = torch.cuda.Stream()
    d = torch.from_numpy(probes).cuda()
    out = torch.empty((len(probes), 3), dtype=torch.float64, device="cuda")
    st.wait_stream(torch.cuda.current_stream())
    _lib.check(_lib.lib.moe_eamc_match_device(e._h, C.c_void_p(d.data_ptr()), 1, len(probes),
                                              C.c_void_p(out.data_ptr()),
                                              C.c_void_p(st.cuda_stream)))
    st.synchronize()
    a = out.cpu().numpy()
    return np.ascontiguousarray(a).view(np.uint8).reshape(-1, 24).copy().view(
        _lib.MATCH_DTYPE)[:, 0]


def _reference(ref, orc, fam, probes):
    if ref is not None:
        er = ref.eamc(L, E, 1, 1, P)
        er.fill_bench(SEED, P)
        idx, seq, d, f, _ = er.match(probes.astype(np.uint64), threads=os.cpu_count() or 1)
        return idx, seq, d
    idx, seq, d, _ = orc.match(fam, np.arange(P, dtype=np.uint64), probes.astype(np.uint64))
    return idx, seq, d


def test_sc_batch_and_streaming_vs_reference(m, orc, sc):
    from oracle import REF_SO, RefLib
    ref = RefLib() if os.path.exists(REF_SO) else None
    e, fam = sc
    probes = m.gen_bench_family(SEED, L, E, 65536, skip=P, dtype=np.uint8)
    got = _device_match(m, e, probes)                 # batch regime (f16 tensor-core screen)
    got8 = _device_match(m, e, probes[:8])            # streaming regime (i8 screen)
    sample = np.concatenate([np.arange(8), np.arange(8, 65536, 4093)])
    n = len(sample) if ref is not None else 12
    sample = sample[:n]
    idx, seq, d = _reference(ref, orc, fam, probes[sample])
    assert np.array_equal(got["index"][sample], idx)
    assert np.array_equal(got["seq"][sample], seq)
    assert np.array_equal(got["distance"][sample], d)
    assert np.array_equal(got8, got[:8])
