""".kvtr container: the package's writer reproduces the reference-written
file byte for byte (sha256 frozen by tests/golden/make_trace_golden.py; the arrays come from
oracle.synth, the bit-exact restatement of the reference generator), the reader returns the
same arrays, malformed files raise TraceFormatError, and (GPU) decoding the trace selects the
reference engine's exact sets at every (step, layer, head)."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import synth

CASE = json.loads((Path(__file__).parent / "golden" / "trace_case.json").read_text())


def _trace():
    from paper_2506_20187_b200 import trace as T
    sp = CASE["spec"]
    L, H, D, N, S = sp["n_layers"], sp["n_heads"], sp["head_dim"], sp["n_context"], sp["n_steps"]
    prof = synth.Profile(desert_rate=sp["desert_rate"], n_hot_regions=sp["n_hot_regions"],
                         score_gap=sp["score_gap"], seed=sp["seed"])
    keys = np.empty((L, H, N, D), np.float32)
    vals = np.empty_like(keys)
    qs = np.empty((S, L, H, D), np.float32)
    for l in range(L):
        for h in range(H):
            k, q, v, _ = synth.lane(prof, l, h, N, D, S, with_values=True)
            keys[l, h], vals[l, h], qs[:, l, h] = k, v, q
    return T.AttentionTrace(T.TraceHeader(L, H, D, N, S, True), keys, qs, vals)


def test_write_matches_reference_bytes_and_read_roundtrip(tmp_path):
    from paper_2506_20187_b200 import trace as T
    tr = _trace()
    p = tmp_path / "t.kvtr"
    nbytes = T.write_trace(tr, p)
    assert nbytes == tr.header.expected_nbytes()
    assert hashlib.sha256(p.read_bytes()).hexdigest() == CASE["sha256"]
    for mmap in (True, False):
        back = T.read_trace(p, mmap=mmap)
        assert back.header == tr.header
        assert np.array_equal(back.keys, tr.keys) and np.array_equal(back.values, tr.values)
        assert np.array_equal(back.queries, tr.queries)


def test_malformed_traces(tmp_path):
    from paper_2506_20187_b200 import trace as T
    p = tmp_path / "t.kvtr"
    T.write_trace(_trace(), p)
    good = p.read_bytes()
    for bad in (b"XVTR" + good[4:], good[:-4], good[:10], good[:4] + (2).to_bytes(4, "little") + good[8:],
                good[:28] + (6).to_bytes(4, "little") + good[32:]):
        q = tmp_path / "bad.kvtr"
        q.write_bytes(bad)
        with pytest.raises(T.TraceFormatError):
            T.read_trace(q)


@pytest.mark.gpu
def test_run_trace_selects_reference_sets(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_20187_b200 import trace as T
    from paper_2506_20187_b200.decode import run_trace
    p = tmp_path / "t.kvtr"
    T.write_trace(_trace(), p)
    tr = T.read_trace(p)
    res = run_trace(tr)
    for s, per_layer in enumerate(CASE["selected"]):
        for l, heads in enumerate(per_layer):
            for h, ref in enumerate(heads):
                assert res["selected"][s][l][h].tolist() == ref, (s, l, h)
