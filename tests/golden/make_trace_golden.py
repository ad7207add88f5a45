"""Freeze a reference `.kvtr` trace and the reference's exact selections on it.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_trace_golden.py

kvtier.trace.generate_synthetic + write_trace (trace.py:107-133, 270-315) write the file; its
sha256 is frozen (the arrays are regenerated bit-identically by oracle.synth in the tests, so
the file itself is not committed).  Expected selections are the reference engine's oracle
sets (engine.py:345-348: lexsort of score_tokens) with k = ceil(rate * n), rate 0.5 for the
first two layers and 0.1 after (engine.py:83-86, 312).
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
from kvtier import importance as imp  # noqa: E402
from kvtier.trace import DesertProfile, TraceHeader, generate_synthetic, write_trace  # noqa: E402

OUT = Path(__file__).resolve().parent / "trace_case.json"


def main():
    spec = {"n_layers": 3, "n_heads": 2, "head_dim": 128, "n_context": 1024, "n_steps": 2,
            "desert_rate": 0.7, "n_hot_regions": 3, "score_gap": 1.0, "seed": 7}
    hdr = TraceHeader(n_layers=spec["n_layers"], n_heads=spec["n_heads"], head_dim=spec["head_dim"],
                      n_context=spec["n_context"], n_steps=spec["n_steps"], has_values=True)
    prof = DesertProfile(desert_rate=spec["desert_rate"], n_hot_regions=spec["n_hot_regions"],
                         score_gap=spec["score_gap"], seed=spec["seed"])
    tr = generate_synthetic(prof, hdr)
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "t.kvtr"
        write_trace(tr, p)
        digest = hashlib.sha256(p.read_bytes()).hexdigest()
    n = spec["n_context"]
    sel = []
    for s in range(spec["n_steps"]):
        per_layer = []
        for l in range(spec["n_layers"]):
            k = math.ceil((0.5 if l < 2 else 0.1) * n)
            heads = []
            for h in range(spec["n_heads"]):
                scores = imp.score_tokens(tr.queries[s, l, h].astype(np.float64), tr.keys[l, h].astype(np.float64))
                order = np.lexsort((np.arange(n), -scores))
                heads.append(sorted(int(t) for t in order[:k]))
            per_layer.append(heads)
        sel.append(per_layer)
    OUT.write_text(json.dumps({"spec": spec, "sha256": digest, "selected": sel}))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
