"""Generate golden fixtures by running the REFERENCE (kvtier, pure Python) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are frozen here as small
fixtures (npz + json).  Inputs are either stored verbatim or regenerated from seeds by
`oracle.synth` (pinned against the reference by synth_digests.json).

What is frozen, with the reference call that produced it:
  select_cases.npz   kvtier.chunk_tree.build_partition / select_top_k / merge_desert
                     (chunk_tree.py:171-379) and kvtier.engine.attention_output
                     (engine.py:145-154) on random, planted, tie and walkthrough lanes,
                     2 steps each with a persistent partition (test_chunk_tree.py:359-509).
  bounds_cases.npz   kvtier.importance.bound_chunks_batch / bound_chunk (importance.py:108-137)
  scores_cases.npz   kvtier.importance.attention_logits (importance.py:27-33)
  c01_digests.json   test_acceptance.py:50-95 (criterion 1): sha256 of the sorted selected set
                     for 1,000 seeded planted traces x 2 steps.
  synth_digests.json sha256 of generate_synthetic outputs (trace.py:270-315)
  scalars.json       chunk_cost / plan_chunk_count / ChunkPlanConfig.chunk_size_for /
                     desert_rate_on_grid / hand examples (test_importance.py, test_engine.py)
"""

from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

import kvtier  # noqa: E402
from kvtier import chunk_tree as ct  # noqa: E402
from kvtier import engine as eng  # noqa: E402
from kvtier import importance as imp  # noqa: E402
from kvtier.trace import DesertProfile, TraceHeader, generate_synthetic  # noqa: E402

OUT = Path(__file__).resolve().parent
STATE_CODE = {"candidate": 0, "important": 1, "desert": 2, "pad": 3}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def spans_arr(part) -> np.ndarray:
    return np.array([(c.start, c.end, STATE_CODE[c.state]) for c in part.leaves], dtype=np.int64)


def select_case(name, keys, values, queries, k, m, merge_between=True, gen=None):
    """Run the reference on one lane for len(queries) steps with a persistent partition.

    gen: json-able spec from which tests/golden_io.py regenerates keys/values/queries
    bit-identically (numpy default_rng or oracle.synth); inputs are stored inline otherwise.
    """
    n, d = keys.shape
    part = ct.build_partition(n, m, keys=np.asarray(keys, np.float64).copy())
    rec = {"k": np.int64(k), "m": np.int64(m), "gen": np.array(json.dumps(gen))}
    if gen is None:
        rec.update({"keys": np.asarray(keys), "values": np.asarray(values),
                    "queries": np.asarray(queries)})
    for s, q in enumerate(queries):
        r = ct.select_top_k(part, np.asarray(q, np.float64), k)
        sel = np.array(sorted(r.selected), dtype=np.int64)
        rec[f"sel{s}"] = sel
        rec[f"order{s}"] = np.array(r.important_tokens, dtype=np.int64)
        rec[f"eval{s}"] = np.int64(r.eval_count)
        rec[f"spans{s}"] = spans_arr(part)
        rec[f"desert{s}"] = np.array(r.desert_chunks, dtype=np.int64).reshape(-1, 2)
        merges = ct.merge_desert(part)
        rec[f"merges{s}"] = np.int64(merges)
        rec[f"mspans{s}"] = spans_arr(part)
        # merged desert abstracts (checked against make_abstract in test_chunk_tree.py:397-410)
        if gen is None:
            dz = [c for c in part.leaves if c.state == "desert"]
            rec[f"dmax{s}"] = np.array([c.abstract.max_key for c in dz]).reshape(-1, d)
            rec[f"dmin{s}"] = np.array([c.abstract.min_key for c in dz]).reshape(-1, d)
        if len(sel):
            rec[f"attn{s}"] = eng.attention_output(q, np.asarray(keys, np.float64)[sel],
                                                   np.asarray(values, np.float64)[sel])
        else:
            rec[f"attn{s}"] = np.zeros(d)
        if not merge_between:
            break
    rec["steps"] = np.int64(len(queries))
    return name, rec


def build_select_cases():
    cases = []
    # (a) random normal f64 lanes, test_chunk_tree.py:359-369 shapes
    for n in (1, 2, 7, 33, 64, 257, 1024):
        for seed in (0, 1, 2):
            rng = np.random.default_rng(seed)
            keys = rng.normal(size=(n, 16))
            query = rng.normal(size=16)
            vals = rng.normal(size=(n, 16))
            q2 = rng.normal(size=16)
            m = max(1, ct.next_pow2(n) // 8)
            for k in sorted({1, max(1, n // 3), n}):
                cases.append(select_case(f"rand_n{n}_s{seed}_k{k}", keys, vals, np.stack([query, q2]), k, m,
                                         gen={"kind": "rand", "n": n, "seed": seed}))
    # (b) planted traces (test_chunk_tree.py:386-396, 478-509; test_acceptance.py c01 shapes)
    for seed in range(8):
        n = 300 + 17 * seed
        tr = generate_synthetic(DesertProfile(desert_rate=0.6, seed=seed),
                                TraceHeader(1, 1, 32, n, 2, has_values=True))
        cases.append(select_case(f"plant_s{seed}", tr.keys[0, 0], tr.values[0, 0], tr.queries[:, 0, 0],
                                 math.ceil(0.1 * n), ct.next_pow2(n) // 8,
                                 gen={"kind": "synth", "desert_rate": 0.6, "n_hot_regions": 3, "score_gap": 1.0,
                                      "seed": seed, "n": n, "d": 32, "steps": 2}))
    for n in (1024, 4096):
        tr = generate_synthetic(DesertProfile(desert_rate=0.7, n_hot_regions=3, score_gap=1.0, seed=3),
                                TraceHeader(1, 1, 64, n, 4, has_values=True))
        cases.append(select_case(f"econ_n{n}", tr.keys[0, 0], tr.values[0, 0], tr.queries[:, 0, 0],
                                 math.ceil(0.1 * n), n // 64,
                                 gen={"kind": "synth", "desert_rate": 0.7, "n_hot_regions": 3, "score_gap": 1.0,
                                      "seed": 3, "n": n, "d": 64, "steps": 4}))
    # (c) ties (test_chunk_tree.py:372-383)
    cases.append(select_case("ties_ones", np.ones((16, 4)), np.arange(64.0).reshape(16, 4),
                             np.ones((2, 4)), 5, 4))
    keys2 = np.vstack([np.ones((8, 4)), np.full((8, 4), 2.0)])
    cases.append(select_case("ties_two", keys2, np.arange(64.0).reshape(16, 4), np.ones((2, 4)), 10, 4))
    # (d) walkthrough (test_chunk_tree.py:424-470)
    d = 8
    u = np.ones(d) / math.sqrt(d)
    amps = np.full(32, 0.15)
    amps[0], amps[10] = 2.2, 2.0
    amps[28:32] = [4.0, 4.1, 4.2, 4.3]
    cases.append(select_case("walkthrough", amps[:, None] * u[None, :],
                             np.random.default_rng(0).normal(size=(32, d)), np.stack([u, u]), 6, 8))
    # (e) config-1 shape: d=128, n=4096, random N(0,1) f32 KV (test_trace.py:26-31), C=64
    for seed in range(2):
        rng = np.random.default_rng(seed)
        keys = rng.normal(size=(4096, 128)).astype(np.float32)
        vals = rng.normal(size=(4096, 128)).astype(np.float32)
        qs = rng.normal(size=(2, 128)).astype(np.float32)
        cases.append(select_case(f"cfg1_s{seed}", keys, vals, qs, math.ceil(0.1 * 4096), 4096 // 64,
                                 gen={"kind": "cfg1", "seed": seed}))
    # (f) k edges (test_chunk_tree.py:399-410)
    rng = np.random.default_rng(5)
    keys = rng.normal(size=(64, 8))
    q = rng.normal(size=8)
    for k in (0, 64):
        cases.append(select_case(f"kedge_{k}", keys, rng.normal(size=(64, 8)), np.stack([q, q]), k, 8))
    # (g) merge semantics (test_chunk_tree.py:583-610)
    rng = np.random.default_rng(11)
    keys = rng.normal(size=(64, 4))
    cases.append(select_case("merge_adj", keys, keys, np.stack([rng.normal(size=4)] * 2), 3, 16))
    rng = np.random.default_rng(12)
    keys = rng.normal(size=(32, 4))
    cases.append(select_case("merge_cover", keys, keys, np.stack([rng.normal(size=4)] * 2), 1, 8))
    return cases


def save_cases(cases, path):
    flat = {"names": np.array([c[0] for c in cases])}
    for i, (_, rec) in enumerate(cases):
        for key, v in rec.items():
            flat[f"{i}/{key}"] = np.asarray(v)
    np.savez_compressed(path, **flat)


def build_bounds_cases():
    rng = np.random.default_rng(2024)
    qs, mx, mn, U, L, rows, smin, smax, dd = [], [], [], [], [], [], [], [], []
    for i in range(600):
        d = int(rng.choice([1, 4, 16, 64, 128]))
        n = int(rng.integers(1, 65))
        scale = float(rng.lognormal(0.0, 1.0))
        keys = rng.normal(scale=scale, size=(n, d))
        if rng.random() < 0.1:
            keys[:] = keys[0]
        if rng.random() < 0.5:
            keys = keys.astype(np.float32).astype(np.float64)
        q = rng.normal(scale=scale, size=d)
        if rng.random() < 0.05:
            q[:] = 0.0
        a = imp.make_abstract(keys)
        ub, lb = imp.bound_chunk(q, a)
        s = imp.attention_logits(q, keys)
        # pad to d=128 rows so they stack
        pad = lambda v: np.concatenate([v, np.zeros(128 - d)])
        qs.append(pad(q)); mx.append(pad(a.max_key)); mn.append(pad(a.min_key))
        U.append(ub); L.append(lb); rows.append(n); smin.append(s.min()); smax.append(s.max()); dd.append(d)
    np.savez_compressed(OUT / "bounds_cases.npz", q=np.array(qs), max_key=np.array(mx), min_key=np.array(mn),
                        U=np.array(U), L=np.array(L), rows=np.array(rows), smin=np.array(smin),
                        smax=np.array(smax), d=np.array(dd))


def build_scores_cases():
    rng = np.random.default_rng(7)
    out = {}
    for i, (n, d) in enumerate([(2, 4), (32, 8), (100, 64), (513, 128), (1000, 128)]):
        keys = rng.normal(size=(n, d)).astype(np.float32)
        q = rng.normal(size=d).astype(np.float32)
        out[f"{i}/keys"] = keys
        out[f"{i}/q"] = q
        out[f"{i}/logits"] = imp.attention_logits(q, keys)
        out[f"{i}/softmax"] = imp.score_tokens(q, keys, mode="softmax")
    np.savez_compressed(OUT / "scores_cases.npz", n_cases=np.int64(5), **out)


def build_c01():
    sizes = [33, 64, 100, 257, 512, 777, 1024, 2048, 3000, 4096]
    rates = [0.05, 0.10, 0.25]
    rows = []
    for seed in range(1000):
        n = sizes[seed % len(sizes)]
        hdr = TraceHeader(n_layers=1, n_heads=1, head_dim=64, n_context=n, n_steps=2)
        prof = DesertProfile(desert_rate=0.3 + 0.6 * ((seed * 7) % 10) / 10.0, n_hot_regions=1 + seed % 5,
                             seed=seed)
        tr = generate_synthetic(prof, hdr)
        keys = tr.keys[0, 0].astype(np.float64)
        k = max(1, math.ceil(rates[seed % len(rates)] * n))
        part = kvtier.build_partition(n, max(1, ct.next_pow2(n) // 64), keys=keys.copy())
        row = {"seed": seed, "n": n, "k": k, "desert_rate": prof.desert_rate,
               "n_hot_regions": prof.n_hot_regions, "m": max(1, ct.next_pow2(n) // 64), "steps": []}
        for step in range(2):
            q = tr.queries[step, 0, 0].astype(np.float64)
            res = kvtier.select_top_k(part, q, k)
            sel = np.array(sorted(res.selected), dtype=np.int64)
            brute = np.lexsort((np.arange(n), -imp.score_tokens(q, keys)))[:k]
            assert set(brute.tolist()) == res.selected
            row["steps"].append({"sha": sha(sel), "eval": res.eval_count})
        rows.append(row)
    (OUT / "c01_digests.json").write_text(json.dumps(rows))


def build_synth_digests():
    rows = []
    for (dr, nr, seed, n, d, S, Lh, H) in [(0.7, 3, 1, 1000, 64, 3, 2, 2), (0.3, 5, 7, 33, 64, 2, 1, 1),
                                           (0.9, 1, 3, 4096, 128, 2, 1, 1), (0.0, 3, 2, 100, 8, 2, 1, 1),
                                           (0.7, 3, 0, 65536, 128, 2, 1, 1)]:
        tr = generate_synthetic(DesertProfile(desert_rate=dr, n_hot_regions=nr, seed=seed),
                                TraceHeader(Lh, H, d, n, S, has_values=True))
        rows.append({"desert_rate": dr, "n_hot_regions": nr, "seed": seed, "n": n, "d": d, "steps": S,
                     "layers": Lh, "heads": H, "keys": sha(tr.keys), "queries": sha(tr.queries),
                     "values": sha(tr.values)})
    (OUT / "synth_digests.json").write_text(json.dumps(rows, indent=1))


def build_scalars():
    s = {}
    s["chunk_cost"] = [[m, n, rho, ct.chunk_cost(m, n, rho)]
                       for n in (64, 1024, 4096) for m in (1, 4, 16, 64) for rho in (0.0, 0.25, 0.5, 0.6)
                       if n % m == 0]
    s["plan_chunk_count"] = [[n, rho, lo, hi, ct.plan_chunk_count(n, rho, min_chunk_size=lo, max_chunk_size=hi)]
                             for n in (32, 256, 1000, 4096, 65536) for rho in (0.0, 0.05, 0.25, 0.45, 0.6, 0.8)
                             for lo, hi in ((8, 64), (8, 256), (1, 1024))]
    cfgs = []
    for rho in (None, (0.1, 0.3, 0.45)):
        cfg = ct.ChunkPlanConfig(rho=rho)
        for layer in (0, 1, 2, 5, 31):
            for step, nst in ((0, 256), (19, 256), (20, 256), (100, 256), (0, 1), (3, 4)):
                for nctx in (5, 100, 1024, 65536):
                    cfgs.append([None if rho is None else list(rho), layer, step, nst, nctx,
                                 cfg.chunk_size_for(layer, step, nst, nctx)])
    s["chunk_size_for"] = cfgs
    s["desert_rate_on_grid"] = [[sorted(sel), n, g, eng.desert_rate_on_grid(set(sel), n, g)]
                                for sel, n, g in (([], 64, 16), ([0, 1, 2], 64, 16), ([0, 16, 32, 48], 64, 16),
                                                  ([70], 72, 16), ([5, 6, 700, 4000], 4096, 64))]
    s["softmax_2_0"] = imp.softmax(np.array([2.0, 0.0])).tolist()
    q = np.array([math.sqrt(2.0), 0.0])
    s["attention_hand"] = eng.attention_output(q, np.array([[1.0, 0.0], [0.0, 0.0]]),
                                               np.array([[1.0, 0.0], [0.0, 1.0]])).tolist()
    a = imp.make_abstract(np.array([[1.0, 0.0], [0.0, 1.0]]))
    s["bound_hand"] = list(imp.bound_chunk(np.array([2.0, 1.0]), a))
    s["bound_neg"] = list(imp.bound_chunk(np.array([-1.0]), imp.make_abstract(np.array([[2.0], [-3.0]]))))
    s["next_pow2"] = [[n, ct.next_pow2(n)] for n in (1, 2, 3, 33, 64, 65, 4097)]
    (OUT / "scalars.json").write_text(json.dumps(s, indent=1))


if __name__ == "__main__":
    save_cases(build_select_cases(), OUT / "select_cases.npz")
    build_bounds_cases()
    build_scores_cases()
    build_scalars()
    build_synth_digests()
    build_c01()
    print("golden fixtures written to", OUT)
