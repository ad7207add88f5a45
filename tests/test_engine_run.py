"""The decode loop and its reports against the reference engine's own
reports on the same trace (fixtures frozen by tests/golden/make_engine_golden.py).

Ablation rows without adaptive evaluation (baseline, +LKA) fetch cold records independently of
the selector, so every steps.csv / schedule.csv / ledger.csv / ablate.csv cell must match, the
f64 quality columns within 1e-9.  With IAKM the selected sets -- hence recall and desert rate
-- still match; eval_count and the selector's cold fetches follow this pipeline's rule
(runner.py docstring)."""

from __future__ import annotations

import csv
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import synth

CASE = json.loads((Path(__file__).parent / "golden" / "engine_cases.json").read_text())
FLOAT_TOL = ("output_similarity", "dropped_mass")


def _write_trace(path, sp=None):
    from paper_2506_20187_b200 import trace as T
    sp = sp or CASE["spec"]
    prof = synth.Profile(desert_rate=sp["desert_rate"], n_hot_regions=sp["n_hot_regions"],
                         score_gap=sp["score_gap"], seed=sp["seed"])
    K, Q, V = synth.trace(prof, sp["n_layers"], sp["n_heads"], sp["n_context"], sp["head_dim"], sp["n_steps"],
                          with_values=sp["has_values"])
    T.write_trace(T.AttentionTrace(T.TraceHeader(sp["n_layers"], sp["n_heads"], sp["head_dim"], sp["n_context"],
                                                 sp["n_steps"], sp["has_values"]), K, Q, V), path)


def test_run_config_echo_matches_reference(tmp_path):
    from paper_2506_20187_b200.engine import ABLATION_ROWS, RunConfig
    import dataclasses
    base = RunConfig(trace_path="x", placement_chunk=CASE["spec"]["placement_chunk"])
    for label, flags in ABLATION_ROWS:
        cfg = dataclasses.replace(base, iakm="iakm" in flags, lka="lka" in flags, dtp="dtp" in flags)
        head = json.loads(CASE["rows"][label]["summary"].splitlines()[0])
        assert cfg.echo() == head["config"], label
    with pytest.raises(ValueError):
        RunConfig(trace_path="x", importance_rate=0.0)
    with pytest.raises(ValueError):
        RunConfig(trace_path="x", placement_chunk=0)


@pytest.mark.gpu
def test_ablation_reports_match_reference(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_20187_b200 import engine as E
    tp = tmp_path / "t.kvtr"
    _write_trace(tp)
    results = E.ablate(E.RunConfig(trace_path=str(tp), placement_chunk=CASE["spec"]["placement_chunk"]),
                       tmp_path / "work")
    for label, rep in results:
        ref = CASE["rows"][label]
        od = tmp_path / ("out-" + label.replace("+", "plus-").lower())
        E.write_report(rep, od)
        with open(od / "steps.csv") as fh:
            got = list(csv.reader(fh))
        want = ref["steps"]
        assert got[0] == want[0] and len(got) == len(want)
        cols = want[0]
        exact_cols = [c for c in cols if c not in FLOAT_TOL]
        if "iakm" in dict(E.ABLATION_ROWS)[label]:
            exact_cols = ["step", "layer", "recall", "desert_rate"]
        for g, w in zip(got[1:], want[1:]):
            gr, wr = dict(zip(cols, g)), dict(zip(cols, w))
            for c in exact_cols:
                assert gr[c] == wr[c], (label, gr["step"], gr["layer"], c, gr[c], wr[c])
            for c in FLOAT_TOL:
                assert abs(float(gr[c]) - float(wr[c])) <= 1e-9, (label, c, gr[c], wr[c])
        head = json.loads((od / "summary.json-lines").read_text().splitlines()[0])
        assert head == json.loads(ref["summary"].splitlines()[0])
        if "iakm" not in dict(E.ABLATION_ROWS)[label]:
            assert (od / "schedule.csv").read_text() == ref["schedule"], label
            assert (od / "ledger.csv").read_text() == ref["ledger"], label
    E.write_ablation(results, tmp_path / "abl")
    got = (tmp_path / "abl" / "ablate.csv").read_text().splitlines()
    want = CASE["ablate"].splitlines()
    assert got[:3] == want[:3]  # header, baseline, +LKA
    for g, w in zip(got[3:], want[3:]):  # +IAKM / ALL: the same mean desert rate
        assert g.split(",")[:4] == w.split(",")[:4] and g.split(",")[5] == w.split(",")[5]
    means = {lab: np.mean([r.eval_count for r in rep.rows]) for lab, rep in results}
    assert means["+IAKM"] < means["+LKA"]  # adaptive evaluation scores fewer than every token


@pytest.mark.gpu
def test_no_values_trace_with_explicit_tier(tmp_path):
    """Second reference run: a trace without values (output_similarity / dropped_mass are nan
    in both), an explicit TierConfig and 16-token records."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_20187_b200 import engine as E
    from paper_2506_20187_b200.tiered_store import TierConfig
    c2 = CASE["case2"]
    tp = tmp_path / "t2.kvtr"
    _write_trace(tp, c2["spec"])
    cfg = E.RunConfig(trace_path=str(tp), placement_chunk=c2["spec"]["placement_chunk"],
                      tier=TierConfig(cold_dir=tmp_path / "unused", **c2["tier"]))
    for label, rep in E.ablate(cfg, tmp_path / "work"):
        ref = c2["rows"][label]
        od = tmp_path / ("out-" + label.replace("+", "plus-").lower())
        E.write_report(rep, od)
        with open(od / "steps.csv") as fh:
            got = list(csv.reader(fh))
        cols = ref["steps"][0]
        iakm = "iakm" in dict(E.ABLATION_ROWS)[label]
        check = ["step", "layer", "recall", "desert_rate", "output_similarity", "dropped_mass"] if iakm else cols
        assert len(got) == len(ref["steps"])
        for g, w in zip(got[1:], ref["steps"][1:]):
            gr, wr = dict(zip(cols, g)), dict(zip(cols, w))
            for col in check:
                assert gr[col] == wr[col], (label, gr["step"], gr["layer"], col, gr[col], wr[col])
        assert json.loads((od / "summary.json-lines").read_text().splitlines()[0]) == \
            json.loads(ref["summary"].splitlines()[0])
        if not iakm:
            assert (od / "ledger.csv").read_text() == ref["ledger"], label
            assert (od / "schedule.csv").read_text() == ref["schedule"], label
