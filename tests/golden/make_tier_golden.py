"""Freeze the reference TieredStore's residency + ledger behaviour (tiered_store.py:141-592).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_tier_golden.py

Drives kvtier.tiered_store (real cold files under a temp dir) with seeded operation
sequences -- the calls engine.run makes per (step, layer, head): open_row, load_abstracts,
cold fetches (fetch_chunk), touch, ensure_hot over runs, close_row (engine.py:307-365) --
plus a few invalid operations, and records every ledger row, the tier of every record after
each row, the byte totals and the exception type of each invalid op.  The B200 package's
`tiered_store` replays the same sequences (tests/test_tiered_store.py).
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

from kvtier import tiered_store as ts  # noqa: E402
from kvtier.trace import DesertProfile, TraceHeader, generate_synthetic  # noqa: E402

OUT = Path(__file__).resolve().parent / "tier_cases.json"


def runs(tokens):
    toks = sorted(set(int(t) for t in tokens))
    out = []
    for t in toks:
        if out and out[-1][1] == t:
            out[-1][1] = t + 1
        else:
            out.append([t, t + 1])
    return out


def case(seed, n_layers, n_heads, n_ctx, d, steps, chunk, hot_recs, warm_recs, pinned, thresh, window, k_frac):
    hdr = TraceHeader(n_layers=n_layers, n_heads=n_heads, head_dim=d, n_context=n_ctx, n_steps=steps, has_values=True)
    trace = generate_synthetic(DesertProfile(seed=seed), hdr)
    rec = ts.kv_nbytes(chunk, d)
    per_lane = ts.kv_nbytes(n_ctx, d)
    pinned_bytes = pinned * n_heads * per_lane
    cfg = dict(hot_capacity=pinned_bytes + hot_recs * rec, warm_capacity=warm_recs * rec,
               early_layers_pinned=pinned, hot_frequency_threshold=thresh, frequency_window=window)
    rng = np.random.default_rng(seed)
    ops, rows, states, errors = [], [], [], []
    with tempfile.TemporaryDirectory() as td:
        store = ts.place_initial(trace, ts.TierConfig(cold_dir=td, **cfg), chunk_size=chunk)

        def snapshot():
            return [[store._records[(l, h)][i].tier[0] for i in range(len(store._records[(l, h)]))]
                    for l in range(n_layers) for h in range(n_heads)]

        states.append({"hot": store.hot_used, "warm": store.warm_used, "tiers": snapshot()})
        k = max(1, int(k_frac * n_ctx))
        prev = {}
        for step in range(steps):
            for layer in range(n_layers):
                store.open_row(step, layer)
                ops.append(["open_row", step, layer])
                for head in range(n_heads):
                    store.load_abstracts(layer, head)
                    ops.append(["load_abstracts", layer, head])
                    # selection: keep half of the previous step's set (frequency), refresh the rest
                    old = prev.get((layer, head), [])
                    keep = list(rng.choice(old, size=len(old) // 2, replace=False)) if old else []
                    fresh = list(rng.choice(n_ctx, size=k, replace=False))
                    sel = sorted(set(int(t) for t in keep + fresh))[:k]
                    prev[(layer, head)] = sel
                    # cold fetches of a few selected cold records (what select_top_k does)
                    cold = store.cold_spans(layer, head)
                    hit = [s for s in cold if any(s[0] <= t < s[1] for t in sel)]
                    for s in hit[: int(rng.integers(0, len(hit) + 1))]:
                        store.fetch_chunk(layer, head, *s)
                        ops.append(["fetch_chunk", layer, head, s[0], s[1]])
                    store.touch(layer, head, sel)
                    ops.append(["touch", layer, head, sel])
                    rr = runs(sel)
                    store.ensure_hot(layer, head, [tuple(r) for r in rr])
                    ops.append(["ensure_hot", layer, head, rr])
                row = store.close_row()
                ops.append(["close_row"])
                rows.append([row.step, row.layer, row.abstract_bytes, row.cold_to_warm, row.warm_to_hot,
                             row.hot_to_warm, row.fetch_ops, row.cold_bytes_at_open, row.r])
                store.check_invariants()
                states.append({"hot": store.hot_used, "warm": store.warm_used, "tiers": snapshot()})
        # invalid operations: the exception type the reference raises
        probes = []
        lane = (pinned, 0)
        recs = store._records[lane]
        warmish = [r for r in recs if r.tier != ts.COLD]
        if warmish:
            probes.append(["fetch_chunk", lane[0], lane[1], warmish[0].start, warmish[0].end])
        coldr = [r for r in recs if r.tier == ts.COLD]
        if coldr:
            probes.append(["promote_hot", lane[0], lane[1], [[coldr[0].start, coldr[0].end]]])
        probes.append(["fetch_chunk", lane[0], lane[1], 5, 5])
        probes.append(["fetch_chunk", lane[0], lane[1], n_ctx + 10, n_ctx + 20])
        for p in probes:
            try:
                if p[0] == "fetch_chunk":
                    store.fetch_chunk(*p[1:])
                else:
                    store.promote_hot(p[1], p[2], [tuple(x) for x in p[3]])
                errors.append([p, None])
            except Exception as e:  # noqa: BLE001 -- the type is the fixture
                errors.append([p, type(e).__name__])
    return {"seed": seed, "n_layers": n_layers, "n_heads": n_heads, "n_ctx": n_ctx, "d": d, "chunk": chunk,
            "config": cfg, "ops": ops, "rows": rows, "states": states, "errors": errors}


def capacity_case():
    """place_initial refusing pinned layers that do not fit (tiered_store.py:569-570)."""
    hdr = TraceHeader(n_layers=2, n_heads=1, head_dim=8, n_context=64, n_steps=1, has_values=True)
    trace = generate_synthetic(DesertProfile(seed=1), hdr)
    with tempfile.TemporaryDirectory() as td:
        try:
            ts.place_initial(trace, ts.TierConfig(hot_capacity=512, warm_capacity=512, cold_dir=td,
                                                  early_layers_pinned=1), chunk_size=16)
            return None
        except Exception as e:  # noqa: BLE001
            return type(e).__name__


def main():
    cases = [
        case(1, 3, 2, 128, 16, 5, 16, hot_recs=6, warm_recs=5, pinned=1, thresh=2, window=3, k_frac=0.15),
        case(2, 4, 2, 256, 8, 6, 32, hot_recs=5, warm_recs=4, pinned=1, thresh=3, window=4, k_frac=0.1),
        case(3, 2, 3, 96, 16, 4, 8, hot_recs=9, warm_recs=7, pinned=0, thresh=2, window=2, k_frac=0.2),
        case(4, 3, 1, 200, 8, 6, 16, hot_recs=3, warm_recs=2, pinned=1, thresh=4, window=5, k_frac=0.12),
    ]
    OUT.write_text(json.dumps({"cases": cases, "pinned_overflow": capacity_case()}))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
