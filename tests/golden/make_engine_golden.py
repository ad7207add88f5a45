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
    OUT.write_text(json.dumps({"spec": SPEC, "rows": rows, "ablate": ablate_csv}))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
