"""Row 12 (tiered_store.py:141-592) parity, CPU: the package's `tiered_store` replays operation
sequences frozen from the reference TieredStore (tests/golden/make_tier_golden.py) and must
reproduce every ledger row (abstract / cold->warm / warm->hot / hot->warm bytes, fetch ops,
cold bytes at open, r), the tier of every record after every row, the hot/warm byte totals
and the exception type of each invalid operation."""

from __future__ import annotations

import json
from pathlib import Path

import pytest

from paper_2506_20187_b200 import tiered_store as ts

CASES = json.loads((Path(__file__).parent / "golden" / "tier_cases.json").read_text())


def _tiers(store, n_layers, n_heads):
    return [[r.tier[0] for r in store.lane_records(l, h)] for l in range(n_layers) for h in range(n_heads)]


@pytest.mark.parametrize("ci", range(len(CASES["cases"])))
def test_replay_matches_reference_ledger(ci):
    c = CASES["cases"][ci]
    L, H = c["n_layers"], c["n_heads"]
    store = ts.place_initial(L, H, c["d"], c["n_ctx"], ts.TierConfig(**c["config"]), chunk_size=c["chunk"])
    states = iter(c["states"])
    st = next(states)
    assert (store.hot_used, store.warm_used) == (st["hot"], st["warm"])
    assert _tiers(store, L, H) == st["tiers"]
    rows = iter(c["rows"])
    for op in c["ops"]:
        name, args = op[0], op[1:]
        if name == "open_row":
            store.open_row(*args)
        elif name == "load_abstracts":
            store.load_abstracts(*args)
        elif name == "fetch_chunk":
            store.fetch_chunk(*args)
        elif name == "touch":
            store.touch(*args)
        elif name == "ensure_hot":
            store.ensure_hot(args[0], args[1], [tuple(s) for s in args[2]])
        elif name == "close_row":
            row = store.close_row()
            want = next(rows)
            got = [row.step, row.layer, row.abstract_bytes, row.cold_to_warm, row.warm_to_hot, row.hot_to_warm,
                   row.fetch_ops, row.cold_bytes_at_open, row.r]
            assert got == want, (ci, got, want)
            store.check_invariants()
            st = next(states)
            assert (store.hot_used, store.warm_used) == (st["hot"], st["warm"])
            assert _tiers(store, L, H) == st["tiers"]
    for probe, err in c["errors"]:
        name = probe[0]
        try:
            if name == "fetch_chunk":
                store.fetch_chunk(*probe[1:])
            else:
                store.promote_hot(probe[1], probe[2], [tuple(x) for x in probe[3]])
            got = None
        except Exception as e:  # noqa: BLE001
            got = type(e).__name__
        assert got == err, (probe, got, err)


def test_pinned_overflow_and_config_errors():
    with pytest.raises(getattr(ts, CASES["pinned_overflow"])):
        ts.place_initial(2, 1, 8, 64, ts.TierConfig(hot_capacity=512, warm_capacity=512, early_layers_pinned=1),
                         chunk_size=16)
    with pytest.raises(ValueError):
        ts.TierConfig(hot_capacity=0, warm_capacity=1)
    with pytest.raises(ValueError):
        ts.TieredStore(ts.TierConfig(hot_capacity=1, warm_capacity=1, early_layers_pinned=3), 2, 1, 8)


def test_ledger_csv_and_move_hook(tmp_path):
    moves = []
    store = ts.place_initial(2, 1, 8, 64, ts.TierConfig(hot_capacity=512, warm_capacity=512, early_layers_pinned=0),
                             chunk_size=16, on_move=lambda r, a, b: moves.append((r.layer, r.start, a, b)))
    store.open_row(0, 1)
    cold = store.cold_spans(1, 0)
    assert cold
    store.ensure_hot(1, 0, [cold[0]])
    row = store.close_row()
    assert row.cold_to_warm == ts.kv_nbytes(16, 8) and row.warm_to_hot == ts.kv_nbytes(16, 8)
    assert (1, cold[0][0], "cold", "warm") in moves and (1, cold[0][0], "warm", "hot") in moves
    store.write_ledger(tmp_path / "ledger.csv")
    lines = (tmp_path / "ledger.csv").read_text().splitlines()
    assert lines[0].split(",") == list(ts.LEDGER_COLUMNS) and len(lines) == 2


def test_place_initial_call_forms():
    from paper_2506_20187_b200 import tiered_store as ts
    cfg = ts.TierConfig(hot_capacity=4096, warm_capacity=4096, early_layers_pinned=0)
    a = ts.place_initial(1, 1, 8, 64, cfg, 16)
    b = ts.place_initial(1, 1, 8, 64, cfg, chunk_size=16)
    assert [r.start for r in a.lane_records(0, 0)] == [r.start for r in b.lane_records(0, 0)] == [0, 16, 32, 48]
    with pytest.raises(TypeError):
        ts.place_initial(1, 1, 8, 64, cfg, chunk=16)
    with pytest.raises(TypeError):
        ts.place_initial(1, 1, 8)
