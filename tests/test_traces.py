"""Trace ingest: the JSONL trace format of model.hpp:103-114
read with the reference's validation (model.cpp:32-71) and folded into
request-level EAMs (moesim_main.cpp:192-201); `moesim eamc save` on the GPU
must write the reference's snapshot byte for byte.  Fixtures come from the
reference library itself (oracle/make_trace_golden.py)."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TRACE = os.path.join(GOLD, "traces_small.jsonl")


def request_eams_py(path, L, E, phase):
    """Test-side restatement of request_level_eam over the raw JSON lines."""
    out = []
    for line in open(path):
        if not line.strip():
            continue
        its = json.loads(line)["iterations"]
        if phase == 1 and len(its) < 2:
            continue
        c = np.zeros((L, E), np.uint64)
        for it in (its[:1] if phase == 0 else its[1:]):
            for layer, assigns in it:
                for e, tok in assigns:
                    c[layer, e] += tok
        out.append(c)
    return np.stack(out)


@pytest.mark.parametrize("phase", [0, 1])
def test_ingest_request_eams(host_pkg, phase):
    m = host_pkg
    bad = json.load(open(os.path.join(GOLD, "bad_traces.json")))
    L, E = bad["L"], bad["E"]
    got = m.ingest_request_eams(TRACE, m.ModelShape(L, E, bad["top_k"]), m.Phase(phase))
    want = request_eams_py(TRACE, L, E, phase)
    assert got.shape == want.shape and np.array_equal(got, want)


def test_ingest_errors_match_reference(host_pkg, tmp_path):
    m = host_pkg
    bad = json.load(open(os.path.join(GOLD, "bad_traces.json")))
    shape = m.ModelShape(bad["L"], bad["E"], bad["top_k"])
    for c in bad["cases"]:
        p = tmp_path / (c["name"] + ".jsonl")
        p.write_text(c["jsonl"])
        if c["rc"] == 0:
            m.ingest_request_eams(str(p), shape, m.Phase.decode)
            continue
        with pytest.raises(m.TraceIngestError) as ei:
            m.ingest_request_eams(str(p), shape, m.Phase.decode)
        msg = str(ei.value)
        if "bad JSON" in c["error"] or "bad trace structure" in c["error"]:
            # the reference appends nlohmann's own parser message
            head = c["error"].split(":")[0] + ":" + c["error"].split(":")[1]
            assert msg.startswith(head), (msg, c["error"])
        else:
            assert msg == c["error"], (msg, c["error"])
    with pytest.raises(m.TraceIngestError):
        m.ingest_request_eams(str(tmp_path / "missing.jsonl"), shape, m.Phase.decode)


@pytest.mark.gpu
@pytest.mark.parametrize("phase,name", [(0, "prefill"), (1, "decode")])
def test_eamc_save_matches_reference_snapshot(m, tmp_path, phase, name):
    bad = json.load(open(os.path.join(GOLD, "bad_traces.json")))
    shape = m.ModelShape(bad["L"], bad["E"], bad["top_k"])
    out = tmp_path / f"{name}.json"
    e = m.eamc_save_from_traces(TRACE, shape, m.Phase(phase), bad["capacity"], str(out))
    assert e.size() == bad["capacity"]
    assert out.read_bytes() == open(os.path.join(GOLD, f"eamc_save_{name}.json"), "rb").read()
