"""Pin the C oracle against the reference's own outputs (frozen in tests/golden/).

CPU only.  These tests are what makes the oracle trustworthy as the checker of the CUDA
path: every set, span, eval count and value here was produced by running kvtier itself
(tests/golden/make_golden.py)."""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from oracle import synth
from tests import golden_io as G


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_synth_restatement_matches_reference_digests():
    for row in G.load_json("synth_digests.json"):
        prof = synth.Profile(desert_rate=row["desert_rate"], n_hot_regions=row["n_hot_regions"], seed=row["seed"])
        K, Q, V = synth.trace(prof, row["layers"], row["heads"], row["n"], row["d"], row["steps"], True)
        assert sha(K) == row["keys"] and sha(Q) == row["queries"] and sha(V) == row["values"], row


def test_scores_match_reference_logits(oracle_lib):
    z = np.load(G.GOLDEN / "scores_cases.npz")
    for i in range(int(z["n_cases"])):
        keys, q = z[f"{i}/keys"], z[f"{i}/q"]
        mine = oracle_lib.scores(q, keys)
        ref = z[f"{i}/logits"]
        scale = np.abs(keys.astype(np.float64)) @ np.abs(q.astype(np.float64)) / math.sqrt(q.shape[0])
        assert np.all(np.abs(mine - ref) <= 4e-16 * q.shape[0] * scale + 1e-300)


def test_hand_examples(oracle_lib):
    s = G.load_json("scalars.json")
    # importance.py hand examples (test_importance.py:27-40,120-140)
    assert oracle_lib.scores(np.ones(4), np.array([[1.0] * 4, [0.0] * 4])).tolist() == [2.0, 0.0]
    U, L = oracle_lib.bounds(np.array([2.0, 1.0]), np.array([1.0, 1.0]), np.array([0.0, 0.0]), rows=[2])
    assert abs(U[0] - s["bound_hand"][0]) <= 1e-12 and abs(L[0] - s["bound_hand"][1]) <= 1e-12
    U, L = oracle_lib.bounds(np.array([-1.0]), np.array([2.0]), np.array([-3.0]), rows=[2])
    assert abs(U[0] - s["bound_neg"][0]) <= 1e-12 and abs(L[0] - s["bound_neg"][1]) <= 1e-12
    out = oracle_lib.attention(np.array([math.sqrt(2.0), 0.0]), np.array([[1.0, 0.0], [0.0, 0.0]]),
                               np.array([[1.0, 0.0], [0.0, 1.0]]))
    np.testing.assert_allclose(out, s["attention_hand"], atol=1e-12)
    mx, mn = oracle_lib.abstract(np.array([[1.0, -2.0], [3.0, 0.5], [-1.0, 4.0]]))
    assert mx.tolist() == [3.0, 4.0] and mn.tolist() == [-1.0, -2.0]


def test_np_sum_restatement(oracle_lib):
    rng = np.random.default_rng(0)
    for _ in range(3000):
        n = int(rng.integers(1, 300))
        a = rng.normal(size=n) * 10.0 ** rng.integers(-5, 5, size=n)
        assert oracle_lib.np_sum(a) == float(a.sum())


def test_bounds_match_reference_and_are_sound(oracle_lib):
    z = np.load(G.GOLDEN / "bounds_cases.npz")
    for i in range(z["U"].shape[0]):
        d = int(z["d"][i])
        q, M, N = z["q"][i, :d], z["max_key"][i, :d], z["min_key"][i, :d]
        rows = int(z["rows"][i])
        U, L = oracle_lib.bounds(q, M, N, rows=[rows])
        A = np.sum(np.abs(q) * np.maximum(np.abs(M), np.abs(N))) / math.sqrt(d)
        tol = 64 * 2.0 ** -52 * (A + 1e-300)
        assert abs(U[0] - z["U"][i]) <= tol and abs(L[0] - z["L"][i]) <= tol, i
        # reference acceptance criterion c02 (test_acceptance.py:101-123): 1e-9 soundness
        assert L[0] <= z["smin"][i] + 1e-9 and z["smax"][i] <= U[0] + 1e-9
        if rows == 1:
            assert abs(U[0] - z["smax"][i]) <= 1e-12 and abs(L[0] - z["smin"][i]) <= 1e-12
        # reference-mode (numpy arithmetic) restatement is bit-exact
        Ur, Lr = oracle_lib.bounds_ref(q, M, N)
        assert Ur[0] == z["U"][i] and Lr[0] == z["L"][i], i


def test_select_cases_match_reference(oracle_lib):
    for c in G.select_cases():
        keys = np.asarray(c["keys"], np.float64)
        n = keys.shape[0]
        bnb = oracle_lib.BnBPartition(keys, c["m"])
        for s in range(c["steps"]):
            q = np.asarray(c["queries"][s], np.float64)
            ref_sel = c[f"sel{s}"]
            # canonical brute force == reference set
            mine = oracle_lib.select(q, keys, c["k"])
            assert np.array_equal(mine, ref_sel), (c["name"], s)
            # restated branch and bound: same set, same eval count, same leaves
            toks, ev = bnb.select(q, c["k"])
            assert sorted(toks) == ref_sel.tolist(), (c["name"], s)
            assert ev == int(c[f"eval{s}"]), (c["name"], s)
            assert bnb.leaves() == G.spans_to_list(c[f"spans{s}"]), (c["name"], s)
            assert bnb.merge() == int(c[f"merges{s}"])
            assert bnb.leaves() == G.spans_to_list(c[f"mspans{s}"]), (c["name"], s)
            # canonical partition: desert leaves == reference merged desert leaves
            # (reference leaf ends may run into the pad region: compare on [0, n))
            canon = oracle_lib.canonical_partition(ref_sel, n)
            ref_m = G.spans_to_list(c[f"mspans{s}"])
            clip = lambda L: [(a, min(b, n), st) for a, b, st in L if st == "desert"]
            assert clip(canon) == clip(ref_m), (c["name"], s)
            sel_union = {t for a, b, st in ref_m if st == "important" for t in range(a, min(b, n))}
            assert sel_union == set(ref_sel.tolist())
            if f"dmax{s}" in c:
                i_des = [i for i, x in enumerate(bnb.leaves()) if x[2] == "desert"]
                for j, i in enumerate(i_des):
                    mx, mn = bnb.leaf_abstract(i)
                    np.testing.assert_array_equal(mx, c[f"dmax{s}"][j])
                    np.testing.assert_array_equal(mn, c[f"dmin{s}"][j])
            if len(ref_sel):
                out = oracle_lib.attention(q, keys, c["values"], ref_sel)
                np.testing.assert_allclose(out, c[f"attn{s}"], rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("part", range(4))
def test_c01_selection_exactness_digests(oracle_lib, part):
    rows = G.load_json("c01_digests.json")[part::4]
    for row in rows:
        n, k = row["n"], row["k"]
        prof = synth.Profile(desert_rate=row["desert_rate"], n_hot_regions=row["n_hot_regions"], seed=row["seed"])
        keys, queries, _, _ = synth.lane(prof, 0, 0, n, 64, 2, with_values=False)
        k64 = keys.astype(np.float64)
        for s in range(2):
            sel = oracle_lib.select(queries[s], k64, k)
            assert sha(sel) == row["steps"][s]["sha"], (row["seed"], s)
