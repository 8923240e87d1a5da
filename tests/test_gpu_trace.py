"""K1 tracing (Eam::record, eam.cpp:41-52, per token as workload.cpp:166-181)
against the oracle at scale: the lane (bank-locked counters), request-owned
and generic kernels,
ragged / empty / multi-chunk requests, counts that overflow the 16-bit lane
copies within a request, the device rollback that makes a failed call
all-or-nothing (eam.cpp:42-47), concurrent calls on two streams, and shapes
whose L x E histogram exceeds one block's shared memory."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ragged_offsets(rng, T, R):
    cuts = np.sort(rng.integers(0, T + 1, size=R - 1))
    offs = np.concatenate([[0], cuts, [T]]).astype(np.uint64)
    offs[R // 2] = offs[R // 2 - 1]  # an empty request
    return offs


def _picks(rng, T, L, E, k):
    """Zipf-skewed first pick, k picks at a random stride (u32, [T][L][k])."""
    zipf = 1.0 / np.arange(1, E + 1) ** 1.2
    base = rng.choice(E, size=(T, L), p=zipf / zipf.sum()).astype(np.uint32)
    step = rng.integers(1, max(2, E // k), size=(T, L, 1)).astype(np.uint32)
    return (base[:, :, None] + step * np.arange(k, dtype=np.uint32)[None, None, :]) % E


def _oracle_trace(orc, L, E, k, picks, offs, per=100):
    """The oracle over slices of requests (bounded host memory at 1M tokens)."""
    R = len(offs) - 1
    out = np.zeros((R, L, E), np.uint64)
    for a in range(0, R, per):
        b = min(R, a + per)
        t0, t1 = int(offs[a]), int(offs[b])
        rc, got = orc.trace(L, E, k, picks[t0:t1].astype(np.uint32), offs[a:b + 1] - offs[a])
        assert rc == 0
        out[a:b] = got
    return out


def _device_trace(shape, picks_t, offs, counts_t, bad_t, stream):
    from paper_2401_14361_b200 import _lib
    import torch
    sh = shape.c()
    stream.wait_stream(torch.cuda.current_stream())  # inputs made on the current stream
    d_offs = torch.from_numpy(offs.astype(np.int64)).to(counts_t.device)
    _lib.check(_lib.lib.moe_eam_trace_device(
        C.byref(sh), C.c_void_p(picks_t.data_ptr()), picks_t.element_size(),
        C.c_uint64(picks_t.shape[0]), C.c_void_p(d_offs.data_ptr()), C.c_uint64(len(offs) - 1),
        C.c_void_p(counts_t.data_ptr()), C.c_void_p(bad_t.data_ptr()),
        C.c_void_p(stream.cuda_stream)))
    return d_offs


@pytest.mark.parametrize("L,E,k,T,R", [
    (59, 160, 6, 60_000, 37),    # DS shape, lane-copy kernel
    (12, 128, 1, 50_000, 9),     # SW shape (L*k = 12: several tokens per 16-byte chunk)
    (32, 8, 2, 80_000, 50),      # MIX shape
    (1, 256, 1, 30_000, 3),      # E = 256: every byte is a valid id
    (7, 40, 3, 41_000, 4),       # odd L, L*k = 21
    (3, 5, 5, 9_000, 5),         # k = E, strided picks: duplicate ids inside a (token, layer)
    (22, 64, 3, 30_000, 9),      # k odd, L*k even: position pairs straddle layers (lane kernel)
    (4, 256, 2, 20_000, 6),      # E = 256 on the lane kernel (no trash ids)
    (59, 160, 6, 3_000, 400),    # short requests (< 16 tokens on average): k_trace_own
])
def test_trace_ragged_vs_oracle(m, orc, L, E, k, T, R):
    rng = np.random.default_rng(L * 1000 + E)
    picks = _picks(rng, T, L, E, k)
    offs = _ragged_offsets(rng, T, R)
    offs[1] = min(int(offs[-1]), 20_000)  # one long request (spans token chunks)
    offs = np.maximum.accumulate(offs)
    rc, want = orc.trace(L, E, k, picks.astype(np.uint32), offs)
    assert rc == 0
    s = m.ModelShape(L, E, k)
    base = rng.integers(0, 1000, size=want.shape).astype(np.uint64)
    for dt in (np.uint8, np.uint16, np.uint32):
        got = m.trace_requests(s, picks.astype(dt), offs, counts=base.copy())
        assert np.array_equal(got, want + base), dt


def test_trace_lane_copy_overflow(m, orc):
    """One cell taking 3 ids per token for 100k tokens (300k > 65,535, the
    16-bit lane-copy limit within a piece): pieces and flushes must carry it."""
    L, E, k, T = 2, 4, 3, 100_000
    picks = np.zeros((T, L, k), np.uint8)
    picks[:, 1, :] = [1, 1, 3]
    offs = np.array([0, 3, T], np.uint64)
    rc, want = orc.trace(L, E, k, picks.astype(np.uint32), offs)
    assert rc == 0 and want[1, 0, 0] == 3 * (T - 3)
    got = m.trace_requests(m.ModelShape(L, E, k), picks, offs)
    assert np.array_equal(got, want)


def test_trace_ds_full_size_device(m, orc):
    """BASELINE configs[3] size: 1M tokens x 59 layers x top-6 (354M u8 ids),
    1,000 requests, through the device API into u32 counts."""
    import torch
    L, E, k, T, R = 59, 160, 6, 1_000_000, 1000
    rng = np.random.default_rng(1001)
    picks = np.concatenate([_picks(rng, T // 10, L, E, k).astype(np.uint8) for _ in range(10)])
    offs = np.arange(0, T + 1, T // R, dtype=np.uint64)
    want = _oracle_trace(orc, L, E, k, picks, offs)
    st = torch.cuda.Stream()
    d_picks = torch.from_numpy(picks).cuda()
    counts = torch.zeros((R, L, E), dtype=torch.int32, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    keep = _device_trace(m.ModelShape(L, E, k), d_picks, offs, counts, bad, st)
    st.synchronize()
    del keep
    assert int(bad.item()) == 0
    assert np.array_equal(counts.cpu().numpy().astype(np.uint64), want)


@pytest.mark.parametrize("dt", [np.uint8, np.uint16])
def test_trace_device_rollback(m, dt):
    """An out-of-range id deep inside a long request: the device call sets the
    flag and leaves the u32 counts exactly as they were (the additions made by
    every other block are rolled back)."""
    import torch
    L, E, k, T = 59, 160, 6, 200_000
    rng = np.random.default_rng(3)
    picks = _picks(rng, T, L, E, k).astype(dt)
    picks[150_001, 40, 2] = E  # bad id
    offs = np.array([0, 1000, 2000, 190_000, T], np.uint64)
    st = torch.cuda.Stream()
    d_picks = torch.from_numpy(picks).cuda()
    base = torch.from_numpy(rng.integers(0, 2**31, size=(4, L, E)).astype(np.int32)).cuda()
    counts = base.clone()
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    keep = _device_trace(m.ModelShape(L, E, k), d_picks, offs, counts, bad, st)
    st.synchronize()
    del keep
    assert int(bad.item()) == 1
    assert torch.equal(counts, base)
    # host API: IndexError and the caller's counts untouched
    hb = np.full((4, L, E), 7, np.uint64)
    with pytest.raises(IndexError):
        m.trace_requests(m.ModelShape(L, E, k), picks, offs, counts=hb)
    assert (hb == 7).all()


def test_trace_concurrent_streams(m, orc):
    """Two device calls in flight on two streams (round 1 shared one scratch
    histogram between them): both results exact."""
    import torch
    L, E, k, T = 24, 128, 2, 300_000
    rng = np.random.default_rng(11)
    sh = m.ModelShape(L, E, k)
    runs = []
    for i in range(2):
        picks = _picks(rng, T, L, E, k).astype(np.uint8)
        offs = np.linspace(0, T, 31).astype(np.uint64)
        rc, want = orc.trace(L, E, k, picks.astype(np.uint32), offs)
        runs.append((torch.from_numpy(picks).cuda(), offs, want))
    torch.cuda.synchronize()
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs, keep = [], []
    for (d_picks, offs, _), st in zip(runs, sts):
        counts = torch.zeros((len(offs) - 1, L, E), dtype=torch.int32, device="cuda")
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        keep.append(_device_trace(sh, d_picks, offs, counts, bad, st))
        outs.append((counts, bad))
    torch.cuda.synchronize()
    for (counts, bad), (_, _, want) in zip(outs, runs):
        assert int(bad.item()) == 0
        assert np.array_equal(counts.cpu().numpy().astype(np.uint64), want)


def test_trace_wide_shape(m, orc):
    """L x E = 300 x 1000 (1.2 MB of u32 histogram, beyond one block's shared
    memory; round 1 returned MOE_ERR_CUDA): layer groups split it."""
    L, E, k, T = 300, 1000, 2, 3000
    rng = np.random.default_rng(5)
    picks = rng.integers(0, E, size=(T, L, k))
    offs = np.array([0, 1000, 1001, T], np.uint64)
    rc, want = orc.trace(L, E, k, picks.astype(np.uint32), offs)
    assert rc == 0
    for dt in (np.uint16, np.uint32):
        got = m.trace_requests(m.ModelShape(L, E, k), picks.astype(dt), offs)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_tracer_device_steps(m, orc, world):
    """Token-sharded K1 (sharded.ShardedTracer) with the real device step: the
    ranks are emulated one after another on this GPU, each adding its partial
    (the SUM all-reduce's result is the sum of the partials); the total equals
    the oracle's Eam::record over the whole requests, with requests cut by the
    rank boundaries."""
    import torch
    from paper_2401_14361_b200.sharded import ShardedTracer, token_split
    L, E, k, T = 59, 160, 6, 50_000
    rng = np.random.default_rng(21)
    picks = _picks(rng, T, L, E, k).astype(np.uint8)
    offs = _ragged_offsets(rng, T, 23)
    want = _oracle_trace(orc, L, E, k, picks, offs)
    counts = torch.zeros((len(offs) - 1, L, E), dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()
    for rank in range(world):
        t0, t1, _ = token_split(T, offs, rank, world)
        tr = ShardedTracer(m.ModelShape(L, E, k), rank, world, allreduce=lambda t, op: None)
        tr.trace(torch.from_numpy(np.ascontiguousarray(picks[t0:t1])).cuda(), T, offs, counts,
                 stream=st)
    st.synchronize()
    assert np.array_equal(counts.cpu().numpy().astype(np.uint64), want)


def test_trace_unaligned_ids(m, orc):
    """A u8 id stream starting at an odd address (the lane kernel needs 2-byte
    alignment, k_trace_own 16): the generic kernel takes it, results exact."""
    import torch
    L, E, k, T = 59, 160, 6, 20_000
    rng = np.random.default_rng(8)
    picks = _picks(rng, T, L, E, k).astype(np.uint8)
    offs = np.linspace(0, T, 9).astype(np.uint64)
    rc, want = orc.trace(L, E, k, picks.astype(np.uint32), offs)
    assert rc == 0
    buf = torch.zeros(picks.size + 1, dtype=torch.uint8, device="cuda")
    buf[1:] = torch.from_numpy(picks.reshape(-1)).cuda()
    view = buf[1:].view(T, L, k)
    assert view.data_ptr() % 2 == 1
    counts = torch.zeros((len(offs) - 1, L, E), dtype=torch.int32, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.cuda.Stream()
    keep = _device_trace(m.ModelShape(L, E, k), view, offs, counts, bad, st)
    st.synchronize()
    del keep
    assert int(bad.item()) == 0
    assert np.array_equal(counts.cpu().numpy().astype(np.uint64), want)
