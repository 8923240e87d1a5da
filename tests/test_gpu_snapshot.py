"""Snapshot I/O (Eamc::save/load, eam.cpp:184-256): the
binary fast path holds exactly what JSON v1 holds -- slot order, seqs,
next_seq, counts at every storage width -- loads back into a collection that
answers bitwise like the saved one, and rejects corrupt files with
EamcSnapshotError like the reference's loader."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _collection(m, orc, L, E, cap, n, seed, scale=1):
    fam = m.gen_bench_family(seed, L, E, n + 40).copy() * scale
    ent, seqs, _ = orc.insert_replay(L, E, cap, fam[:n])  # slot order != seq order
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, cap)
    e.append(ent, seqs)
    return e, fam[n:]


@pytest.mark.parametrize("scale,cb", [(1, 1), (300, 2), (70_000, 4)])
def test_binary_round_trip(m, orc, tmp_path, scale, cb):
    e, probes = _collection(m, orc, 6, 48, 200, 330, 5, scale)
    assert e.count_bytes() == cb
    pj, pb = tmp_path / "s.json", tmp_path / "s.bin"
    e.save(str(pj))
    e.save_binary(str(pb))
    fj, fb = m.Eamc.load(str(pj)), m.Eamc.load(str(pb))
    for f in (fj, fb):
        assert f.size() == e.size() and f.capacity() == e.capacity()
        assert f.next_seq() == e.next_seq() and f.phase() == e.phase()
        for i in range(e.size()):
            assert f.entry_seq(i) == e.entry_seq(i)
            assert np.array_equal(f.entry(i).counts, e.entry(i).counts)
        assert np.array_equal(f.match_batch(probes), e.match_batch(probes))
    assert fb.count_bytes() == cb
    # the binary snapshot re-saved as JSON is byte-identical to the original JSON
    pj2 = tmp_path / "s2.json"
    fb.save(str(pj2))
    assert pj.read_bytes() == pj2.read_bytes()
    # subsequent inserts behave identically (next_seq and slots preserved)
    inc = m.gen_bench_family(77, 6, 48, 5) * scale
    assert np.array_equal(fb.build(inc), e.build(inc))


def test_binary_empty_and_errors(m, tmp_path):
    s = m.ModelShape(3, 8)
    e = m.Eamc(s, m.Phase.prefill, 4)
    p = tmp_path / "empty.bin"
    e.save_binary(str(p))
    f = m.Eamc.load(str(p), expected=s)
    assert f.size() == 0 and f.phase() == m.Phase.prefill and f.capacity() == 4
    with pytest.raises(m.EamcSnapshotError):  # eam.cpp:252-254
        m.Eamc.load(str(p), expected=m.ModelShape(3, 9))
    raw = p.read_bytes()
    e.append(np.ones((2, 3, 8), np.uint64), np.array([4, 9], np.uint64))
    e.save_binary(str(p))
    full = p.read_bytes()
    for bad in (full[:-1], full[:40], full + b"x", b"MOEEAMCB" + b"\x02" + full[9:]):
        q = tmp_path / "bad.bin"
        q.write_bytes(bad)
        with pytest.raises(m.EamcSnapshotError):
            m.Eamc.load(str(q))
    assert len(raw) == 64


def test_binary_sharded_and_speed(m, orc, tmp_path):
    """A sharded collection's binary snapshot equals the unsharded one's; at
    P = 100k (SW shape) the binary path is timed next to JSON v1."""
    L, E, P = 12, 128, 100_000
    fam = m.gen_bench_family(55, L, E, P, dtype=np.uint8)
    seqs = np.arange(P, dtype=np.uint64)
    e = m.Eamc(m.ModelShape(L, E), m.Phase.decode, P)
    e.append(fam, seqs)
    e3 = m.Eamc.sharded(m.ModelShape(L, E), m.Phase.decode, P, [0, 0, 0])
    e3.append(fam, seqs)
    p1, p3, pj = tmp_path / "one.bin", tmp_path / "three.bin", tmp_path / "one.json"
    t0 = time.perf_counter()
    e.save_binary(str(p1))
    t_bin_save = time.perf_counter() - t0
    e3.save_binary(str(p3))
    assert p1.read_bytes() == p3.read_bytes()
    t0 = time.perf_counter()
    f = m.Eamc.load(str(p1))
    t_bin_load = time.perf_counter() - t0
    t0 = time.perf_counter()
    e.save(str(pj))
    t_json_save = time.perf_counter() - t0
    t0 = time.perf_counter()
    m.Eamc.load(str(pj))
    t_json_load = time.perf_counter() - t0
    print(f"P=100k snapshot: binary save {t_bin_save:.3f}s load {t_bin_load:.3f}s | "
          f"JSON save {t_json_save:.3f}s load {t_json_load:.3f}s")
    assert f.size() == P and f.entry_seq(P - 1) == P - 1
    assert t_bin_save < t_json_save and t_bin_load < t_json_load
