"""Loader for the frozen reference fixtures in tests/golden/ (see make_golden.py)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from oracle import synth

GOLDEN = Path(__file__).resolve().parent / "golden"
STATES = ("candidate", "important", "desert", "pad")


def regen(gen: dict):
    """Rebuild (keys, values, queries) bit-identically from a fixture's generator spec."""
    kind = gen["kind"]
    if kind == "rand":  # make_golden.build_select_cases (a)
        rng = np.random.default_rng(gen["seed"])
        n = gen["n"]
        keys = rng.normal(size=(n, 16))
        query = rng.normal(size=16)
        vals = rng.normal(size=(n, 16))
        q2 = rng.normal(size=16)
        return keys, vals, np.stack([query, q2])
    if kind == "synth":
        prof = synth.Profile(desert_rate=gen["desert_rate"], n_hot_regions=gen["n_hot_regions"],
                             score_gap=gen["score_gap"], seed=gen["seed"])
        k, q, v, _ = synth.lane(prof, 0, 0, gen["n"], gen["d"], gen["steps"], with_values=True)
        return k, v, q
    if kind == "cfg1":
        rng = np.random.default_rng(gen["seed"])
        keys = rng.normal(size=(4096, 128)).astype(np.float32)
        vals = rng.normal(size=(4096, 128)).astype(np.float32)
        qs = rng.normal(size=(2, 128)).astype(np.float32)
        return keys, vals, qs
    raise ValueError(kind)


def select_cases():
    """List of dicts: name, keys, values, queries, k, m, steps, and per step s:
    sel{s}, eval{s}, spans{s}, mspans{s}, desert{s}, attn{s}, (dmax{s}, dmin{s})."""
    z = np.load(GOLDEN / "select_cases.npz")
    names = [str(x) for x in z["names"]]
    cases = []
    for i, name in enumerate(names):
        pre = f"{i}/"
        rec = {key[len(pre):]: z[key] for key in z.files if key.startswith(pre)}
        gen = json.loads(str(rec.pop("gen")))
        if gen is not None:
            rec["keys"], rec["values"], rec["queries"] = regen(gen)
        rec["name"] = name
        rec["k"] = int(rec["k"])
        rec["m"] = int(rec["m"])
        rec["steps"] = int(rec["steps"])
        cases.append(rec)
    return cases


def spans_to_list(a: np.ndarray):
    return [(int(s), int(e), STATES[int(c)]) for s, e, c in np.asarray(a).reshape(-1, 3)]


def load_json(name: str):
    return json.loads((GOLDEN / name).read_text())
