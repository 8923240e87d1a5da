"""Clustering construction (moe_eamc_build_clustered; north-star item 3).

OPT-IN and PARITY-UNPINNED: the reference defers clustering (PAPER.md:591,
SPEC.md:8), so there is no reference output to compare with.  What is pinned:
iteration 0 equals the reference construction (ordered Eamc::insert,
eam.cpp:152-178) bitwise; every reported objective equals the oracle's
sum_i min_p d(eam_i, rep_p) over the collection at that point; the objective
never increases; representatives are input EAMs with seq = input index; the
result is deterministic."""
import numpy as np
import pytest

from oracle import Workload

pytestmark = pytest.mark.gpu


def _objective(orc, reps, seqs, eams):
    _, _, d, _ = orc.match(reps, seqs, eams)
    return float(np.sum(d))


@pytest.mark.parametrize("L,E,N,P,src", [(6, 32, 600, 60, "bench"), (12, 64, 2000, 100, "f2"),
                                         (24, 128, 3000, 150, "f2")])
def test_clustered_construction(m, orc, L, E, N, P, src):
    if src == "bench":
        eams = m.gen_bench_family(11, L, E, N)
    else:
        eams = orc.request_eams(Workload(L, E, 2, seed=5), N)
    s = m.ModelShape(L, E, 2)
    e = m.Eamc(s, m.Phase.decode, P)
    obj, rep, it = e.build_clustered(eams, iterations=6)
    # iteration 0 = the reference construction
    ref_ent, ref_seqs, _ = orc.insert_replay(L, E, P, eams)
    assert obj[0] == pytest.approx(_objective(orc, ref_ent, ref_seqs, eams), rel=0, abs=1e-9)
    assert np.all(np.diff(obj) <= 1e-9), obj          # never increases
    print(src, L, E, N, P, "objective per iteration:", obj, "iterations run:", it)
    if src == "f2":  # grouped, skewed routing: the refinement must find something
        assert it >= 1 and obj[it] < obj[0]
    # representatives: input EAMs, seq = input index, distinct
    assert e.size() == P and len(set(rep.tolist())) == P
    got = np.stack([e.entry(i).counts for i in range(P)])
    seqs = np.array([e.entry_seq(i) for i in range(P)], np.uint64)
    assert np.array_equal(got, eams[rep.astype(np.int64)]) and np.array_equal(seqs, rep)
    assert obj[-1] == pytest.approx(_objective(orc, got, seqs, eams), rel=0, abs=1e-9)
    # deterministic
    e2 = m.Eamc(s, m.Phase.decode, P)
    obj2, rep2, it2 = e2.build_clustered(eams, iterations=6)
    assert np.array_equal(obj, obj2) and np.array_equal(rep, rep2) and it == it2


def test_clustered_zero_iterations_is_build(m, orc):
    L, E, N, P = 8, 16, 300, 40
    eams = m.gen_bench_family(3, L, E, N)
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
    obj, rep, it = e.build_clustered(eams, iterations=0)
    ref_ent, ref_seqs, _ = orc.insert_replay(L, E, P, eams)
    assert it == 0
    for i in range(P):
        assert np.array_equal(e.entry(i).counts, ref_ent[i]) and e.entry_seq(i) == ref_seqs[i]
    assert np.array_equal(rep, ref_seqs)
    with pytest.raises(ValueError):  # must start empty
        e.build_clustered(eams, iterations=1)
