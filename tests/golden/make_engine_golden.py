"""Freeze the reference engine's reports on a small seeded trace.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_engine_golden.py

kvtier.engine.ablate (engine.py:487-502) runs the cumulative feature ladder (baseline, +LKA,
+IAKM, ALL) over a synthetic trace (regenerated bit-identically by oracle.synth in the
tests); for every row this records steps.csv (parsed), schedule.csv, ledger.csv and the
summary records (engine.py:419-466).  tests/test_engine_run.py runs the B200 engine on the
same trace.
"""

from __future__ import annotations

import csv
import json
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
from kvtier import engine as E  # noqa: E402
from kvtier.trace import DesertProfile, TraceHeader, generate_synthetic, write_trace  # noqa: E402

OUT = Path(__file__).resolve().parent / "engine_cases.json"

SPEC = {"n_layers": 4, "n_heads": 2, "head_dim": 32, "n_context": 700, "n_steps": 3, "has_values": True,
        "desert_rate": 0.7, "n_hot_regions": 3, "score_gap": 1.0, "seed": 11, "placement_chunk": 32}


def main():
    hdr = TraceHeader(n_layers=SPEC["n_layers"], n_heads=SPEC["n_heads"], head_dim=SPEC["head_dim"],
                      n_context=SPEC["n_context"], n_steps=SPEC["n_steps"], has_values=SPEC["has_values"])
    prof = DesertProfile(desert_rate=SPEC["desert_rate"], n_hot_regions=SPEC["n_hot_regions"],
                         score_gap=SPEC["score_gap"], seed=SPEC["seed"])
    tr = generate_synthetic(prof, hdr)
    rows = {}
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "t.kvtr"
        write_trace(tr, p)
        cfg = E.RunConfig(trace_path=str(p), placement_chunk=SPEC["placement_chunk"])
        results = E.ablate(cfg, Path(td) / "work")
        for label, rep in results:
            od = Path(td) / ("out-" + label.replace("+", "plus-").lower())
            E.write_report(rep, od)
            with open(od / "steps.csv") as fh:
                steps = list(csv.reader(fh))
            rows[label] = {"steps": steps, "schedule": (od / "schedule.csv").read_text(),
                           "ledger": (od / "ledger.csv").read_text(),
                           "summary": (od / "summary.json-lines").read_text()}
        E.write_ablation(results, Path(td) / "abl")
        ablate_csv = (Path(td) / "abl" / "ablate.csv").read_text()
    # second case: no values (quality columns nan), explicit tier budget, placement chunk 16
    spec2 = dict(SPEC, has_values=False, seed=12, n_context=300, placement_chunk=16, n_steps=2)
    hdr2 = TraceHeader(n_layers=spec2["n_layers"], n_heads=spec2["n_heads"], head_dim=spec2["head_dim"],
                       n_context=spec2["n_context"], n_steps=spec2["n_steps"], has_values=False)
    tr2 = generate_synthetic(DesertProfile(seed=spec2["seed"]), hdr2)
    rec = 2 * 16 * spec2["head_dim"] * 2
    tier2 = {"hot_capacity": 2 * spec2["n_heads"] * 2 * spec2["n_context"] * spec2["head_dim"] * 2 + 6 * rec,
             "warm_capacity": 5 * rec, "early_layers_pinned": 2}
    rows2 = {}
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "t2.kvtr"
        write_trace(tr2, p)
        from kvtier.tiered_store import TierConfig
        cfg = E.RunConfig(trace_path=str(p), placement_chunk=16, tier=TierConfig(cold_dir=td, **tier2))
        for label, rep in E.ablate(cfg, Path(td) / "work"):
            od = Path(td) / ("out-" + label.replace("+", "plus-").lower())
            E.write_report(rep, od)
            with open(od / "steps.csv") as fh:
                rows2[label] = {"steps": list(csv.reader(fh)), "ledger": (od / "ledger.csv").read_text(),
                                "schedule": (od / "schedule.csv").read_text(),
                                "summary": (od / "summary.json-lines").read_text()}
    OUT.write_text(json.dumps({"spec": SPEC, "rows": rows, "ablate": ablate_csv,
                               "case2": {"spec": spec2, "tier": tier2, "rows": rows2}}))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
