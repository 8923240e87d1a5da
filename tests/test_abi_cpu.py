"""CPU: the C-ABI library loads, exports every symbol the header declares, its
host-only pieces agree with the oracle, and it fails loudly without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, gpu_available

HEADER = os.path.join(ROOT, "include", "moe_eamc.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:moe_status|int|const char\*)\s+(moe_\w+)\(", text,
                                 re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2401_14361_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert sorted(_lib.EXPORTS) == syms
    assert _lib.lib.moe_abi_version() == 1


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2401_14361_b200", "libmoe_eamc.so")
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_gen_bench_family_matches_oracle(orc):
    from paper_2401_14361_b200 import gen_bench_family
    for seed, L, E in [(55, 12, 128), (0, 32, 8), (3, 59, 160)]:
        want = orc.bench_family(seed, L, E, 50)
        got = gen_bench_family(seed, L, E, 50)
        assert np.array_equal(got, want)
        got8 = gen_bench_family(seed, L, E, 20, skip=30, dtype=np.uint8)
        assert np.array_equal(got8.astype(np.uint64), want[30:])


def test_capacity_bound_host(golden):
    import paper_2401_14361_b200 as m
    cap = golden("traces.npz")["cap"]
    assert m.eamc_capacity_bound(m.ModelShape(12, 128, 1), 0.75) == cap[0]
    assert m.eamc_capacity_bound(m.ModelShape(12, 128, 1), 0.98) == cap[1]
    assert m.eamc_capacity_bound(m.ModelShape(1, 1, 1), 0.75) == cap[2]
    with pytest.raises(ValueError):
        m.eamc_capacity_bound(m.ModelShape(2, 2, 1), 0.9)


def test_shape_validation_host():
    import paper_2401_14361_b200 as m
    with pytest.raises(ValueError):
        m.Eam(m.ModelShape(0, 4, 1))
    with pytest.raises(ValueError):
        m.Eam(m.ModelShape(2, 2, 3))


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly():
    import paper_2401_14361_b200 as m
    with pytest.raises(m.CudaError):
        m.Eamc(m.ModelShape(2, 4, 1), m.Phase.decode, 4)
    with pytest.raises(m.CudaError):
        m.eam_distance(m.Eam(m.ModelShape(1, 2)), m.Eam(m.ModelShape(1, 2)))


def test_eam_value_type_record():
    """Eam bookkeeping semantics (test_eam.cpp:72-97)."""
    import paper_2401_14361_b200 as m
    s = m.ModelShape(2, 2, 1)
    e = m.Eam(s, m.EamKind.iteration, m.Phase.decode)
    e.record(m.RoutingEvent(0, [(1, 3)]))
    e.record(m.RoutingEvent(0, [(1, 3)]))
    assert e.at(0, 1) == 6 and e.at(0, 0) == 0
    with pytest.raises(IndexError):
        e.record(m.RoutingEvent(2, [(0, 1)]))
    with pytest.raises(IndexError):
        e.record(m.RoutingEvent(1, [(0, 1), (2, 5)]))
    assert e.row_sum(1) == 0
    r = m.Eam(s, m.EamKind.request, m.Phase.prefill)
    with pytest.raises(ValueError):
        r.accumulate(e)


def test_transfer_queue_order():
    """TransferQueue (test_policy.cpp:195-238)."""
    import paper_2401_14361_b200 as m
    E = m.ExpertId
    q = m.TransferQueue()
    q.submit(E(2, 0), 0.9)
    q.submit(E(1, 1), 0.4)
    q.submit(E(0, 5), m.kMaxPriority)
    assert q.peek().expert == E(0, 5)
    assert q.pop().expert == E(0, 5)
    q.submit(E(1, 1), 0.95)  # overwrite
    assert q.size() == 2 and q.pop().expert == E(1, 1)
    q.submit(E(3, 0), 0.9)
    assert [c.expert for c in q] == [E(2, 0), E(3, 0)]  # tie -> ExpertId asc
    assert q.cancel(E(2, 0)) and not q.cancel(E(2, 0))
    assert q.cancel_all() == 1 and q.empty()
