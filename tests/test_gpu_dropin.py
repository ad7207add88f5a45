"""The kvtier-compatible API on the B200 against the reference's own frozen outputs and
against the behaviour its test-suite pins (test_importance.py, test_chunk_tree.py,
test_engine.py, test_acceptance.py c01/c02), re-asserted through paper_2506_20187_b200."""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from oracle import synth  # noqa: E402
from tests import golden_io as G  # noqa: E402


@pytest.fixture(scope="module")
def kv():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_20187_b200 as kv_
    return kv_


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# -- frozen reference outputs -------------------------------------------------------------------


def test_golden_select_cases(kv):
    for c in G.select_cases():
        keys = np.asarray(c["keys"])
        n = keys.shape[0]
        part = kv.build_partition(n, c["m"], keys=keys)
        for s in range(c["steps"]):
            q = c["queries"][s]
            res = kv.select_top_k(part, q, c["k"])
            ref = c[f"sel{s}"]
            assert sorted(res.important_tokens) == ref.tolist(), (c["name"], s)
            # canonical boundaries: desert leaves == reference desert leaves after merge_desert
            ref_m = G.spans_to_list(c[f"mspans{s}"])
            clip = lambda L: [(a, min(b, n)) for a, b, st in L if st == "desert"]
            assert clip(part.leaf_spans()) == clip(ref_m), (c["name"], s)
            imp = {t for a, b, st in part.leaf_spans() if st == "important" for t in range(a, min(b, n))}
            assert imp == set(ref.tolist())
            if f"dmax{s}" in c:
                dz = [x for x in part.leaves if x.state == "desert"]
                for j, x in enumerate(dz):
                    np.testing.assert_array_equal(x.abstract.max_key, c[f"dmax{s}"][j])
                    np.testing.assert_array_equal(x.abstract.min_key, c[f"dmin{s}"][j])
            n_des = sum(1 for x in part.leaves if x.state == "desert")
            kv.merge_desert(part)  # canonical already: only pad leaves can still coalesce
            assert sum(1 for x in part.leaves if x.state == "desert") == n_des
            if len(ref):
                out = kv.attention_output(q, keys[ref], np.asarray(c["values"])[ref])
                np.testing.assert_allclose(out, c[f"attn{s}"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("part_i", range(4))
def test_c01_selection_exactness(kv, part_i):
    """test_acceptance.py:50-95 -- 1,000 seeded traces x 2 steps, persistent partition."""
    for row in G.load_json("c01_digests.json")[part_i::4]:
        n, k = row["n"], row["k"]
        prof = synth.Profile(desert_rate=row["desert_rate"], n_hot_regions=row["n_hot_regions"], seed=row["seed"])
        keys, queries, _, _ = synth.lane(prof, 0, 0, n, 64, 2, with_values=False)
        part = kv.build_partition(n, row["m"], keys=keys)
        for s in range(2):
            res = kv.select_top_k(part, queries[s], k)
            assert sha(np.array(sorted(res.important_tokens), dtype=np.int64)) == row["steps"][s]["sha"], row["seed"]


# -- importance.py behaviour (test_importance.py) --------------------------------------------------


def test_importance_hand_examples(kv):
    s = G.load_json("scalars.json")
    assert kv.attention_logits(np.ones(4), np.array([[1.0] * 4, [0.0] * 4])).tolist() == [2.0, 0.0]
    w = kv.softmax(np.array([2.0, 0.0]))
    np.testing.assert_allclose(w, s["softmax_2_0"], atol=1e-15)
    np.testing.assert_allclose(kv.softmax(np.full(4, 3.7)), 0.25, atol=1e-12)
    a = kv.make_abstract(np.array([[1.0, -2.0], [3.0, 0.5], [-1.0, 4.0]]))
    assert a.max_key.tolist() == [3.0, 4.0] and a.min_key.tolist() == [-1.0, -2.0]
    assert (a.start, a.end, a.n_tokens) == (0, 3, 3)
    assert kv.make_abstract(np.zeros((5, 64))).nbytes() == 512
    up, lo = kv.bound_chunk(np.array([2.0, 1.0]), kv.make_abstract(np.array([[1.0, 0.0], [0.0, 1.0]])))
    assert abs(up - s["bound_hand"][0]) <= 1e-12 and abs(lo - s["bound_hand"][1]) <= 1e-12
    up, lo = kv.bound_chunk(np.array([-1.0]), kv.make_abstract(np.array([[2.0], [-3.0]])))
    assert abs(up - 3.0) <= 1e-12 and abs(lo + 2.0) <= 1e-12
    with pytest.raises(ValueError):
        kv.score_tokens(np.ones(3), np.ones((4, 5)))
    with pytest.raises(ValueError):
        kv.make_abstract(np.zeros((4, 2)), 2, 2)
    with pytest.raises(ValueError):
        kv.merge_abstracts(kv.make_abstract(np.zeros((8, 2)), 0, 3), kv.make_abstract(np.zeros((8, 2)), 4, 8))
    keys = np.arange(12, dtype=float).reshape(6, 2)
    m = kv.merge_abstracts(kv.make_abstract(keys, 3, 6), kv.make_abstract(keys, 0, 3))
    w = kv.make_abstract(keys, 0, 6)
    assert (m.start, m.end) == (0, 6) and np.array_equal(m.max_key, w.max_key) and np.array_equal(m.min_key, w.min_key)


def test_singleton_bounds_exact_and_batch_matches_scalar(kv):
    rng = np.random.default_rng(1)
    for _ in range(50):
        d = int(rng.integers(1, 65))
        q = rng.normal(size=d)
        key = rng.normal(size=(1, d))
        up, lo = kv.bound_chunk(q, kv.make_abstract(key))
        ex = kv.attention_logits(q, key)[0]
        assert up == ex and lo == ex
    q = rng.normal(size=16)
    keys = rng.normal(size=(64, 16))
    ab = [kv.make_abstract(keys, s, s + 8) for s in range(0, 64, 8)]
    U, L = kv.bound_chunks_batch(q, np.stack([a.max_key for a in ab]), np.stack([a.min_key for a in ab]))
    for i, a in enumerate(ab):
        ub, lb = kv.bound_chunk(q, a)
        assert U[i] == ub and L[i] == lb
    sb = kv.bound_chunk(q, ab[0], "softmax")
    assert sb.upper == pytest.approx(math.exp(kv.bound_chunk(q, ab[0]).upper), rel=1e-12)


# -- chunk_tree.py behaviour (test_chunk_tree.py) -------------------------------------------------


def test_partition_build_and_errors(kv):
    keys = np.random.default_rng(1).normal(size=(33, 4))
    part = kv.build_partition(33, 8, keys=keys)
    spans = part.leaf_spans()
    assert part.n_pad == 64 and spans[-3:] == [(40, 48, "pad"), (48, 56, "pad"), (56, 64, "pad")]
    assert spans[4] == (32, 40, "candidate")
    with pytest.raises(ValueError):
        kv.build_partition(32, 3, keys=np.zeros((32, 2)))
    with pytest.raises(ValueError):
        kv.build_partition(32, 8)


def test_k_edges_and_tiling(kv):
    rng = np.random.default_rng(5)
    keys = rng.normal(size=(64, 8))
    q = rng.normal(size=8)
    part = kv.build_partition(64, 8, keys=keys)
    r0 = kv.select_top_k(part, q, 0)
    assert r0.important_tokens == [] and r0.eval_count >= 1
    assert all(c.state in ("desert", "pad") for c in part.leaves)
    part = kv.build_partition(64, 8, keys=keys)
    rn = kv.select_top_k(part, q, 64)
    assert sorted(rn.important_tokens) == list(range(64)) and rn.desert_chunks == []
    with pytest.raises(ValueError):
        kv.select_top_k(part, q, 65)
    rng = np.random.default_rng(9)
    keys = rng.normal(size=(256, 8))
    part = kv.build_partition(256, 8, keys=keys)
    for _ in range(5):
        qq = rng.normal(size=8)
        res = kv.select_top_k(part, qq, 25)
        assert res.selected == set(O.select(qq, keys, 25).tolist())
        kv.merge_desert(part)
        st = [c.start for c in part.leaves]
        en = [c.end for c in part.leaves]
        assert st[0] == 0 and en[-1] == part.n_pad and all(e == s for e, s in zip(en, st[1:]))


def test_cold_fetch_semantics(kv):
    class FakeStore:
        def __init__(self, keys):
            self.keys = np.asarray(keys, dtype=np.float64)
            self.calls = []

        def fetch(self, start, end):
            self.calls.append((start, end))
            return self.keys[start:end]

    rng = np.random.default_rng(10)
    u = np.ones(8) / math.sqrt(8)
    amps = rng.uniform(0.0, 0.2, size=64)
    amps[40:48] = 3.0 + rng.uniform(0, 0.1, size=8)
    keys = amps[:, None] * u[None, :]
    abstracts = [kv.make_abstract(keys, s, s + 8) for s in range(32, 64, 8)]
    part = kv.build_partition(64, 8, keys=keys.copy(), abstracts=abstracts)
    store = FakeStore(keys)
    res = kv.select_top_k(part, u, 8, store=store)
    assert res.selected == set(range(40, 48)) and store.calls == [(40, 48)] and res.fetch_set == [(40, 48)]
    keys = np.array([[0.1], [5.0], [0.2], [0.3]])
    part = kv.build_partition(4, 4, keys=keys.copy(), abstracts=[kv.make_abstract(keys, 1, 2)])
    store = FakeStore(keys)
    res = kv.select_top_k(part, np.array([1.0]), 1, store=store)
    assert res.selected == {1} and store.calls == [(1, 2)]
    keys = np.full((8, 2), 1.0)
    part = kv.build_partition(8, 4, keys=keys.copy(), abstracts=[kv.make_abstract(keys, s, s + 2) for s in range(0, 8, 2)])
    with pytest.raises(RuntimeError):
        kv.select_top_k(part, np.ones(2), 3)


def test_economy_on_desert_traces(kv):
    """test_chunk_tree.py:485-509 and test_acceptance.py c03 economy bounds."""
    for n in (1024, 4096):
        keys, queries, _, _ = synth.lane(synth.Profile(0.7, 3, 1.0, 0), 0, 0, n, 64, 4, with_values=False)
        part = kv.build_partition(n, n // 64, keys=keys)
        k = math.ceil(0.1 * n)
        res = kv.select_top_k(part, queries[0], k)
        assert res.selected == set(O.select(queries[0], keys, k).tolist())
        assert res.eval_count <= 0.6 * n
    n = 4096
    keys, queries, _, _ = synth.lane(synth.Profile(0.7, 3, 1.0, 3), 0, 0, n, 64, 4, with_values=False)
    part = kv.build_partition(n, n // 64, keys=keys)
    counts = []
    for s in range(4):
        res = kv.select_top_k(part, queries[s], math.ceil(0.1 * n))
        assert res.selected == set(O.select(queries[s], keys, math.ceil(0.1 * n)).tolist())
        counts.append(res.eval_count)
        kv.merge_desert(part)
    assert np.mean(counts) <= 0.35 * n, counts
    assert counts[-1] < counts[0], counts


def test_dump_format(kv):
    import re
    rng = np.random.default_rng(13)
    keys = rng.normal(size=(33, 4))
    part = kv.build_partition(33, 8, keys=keys)
    kv.select_top_k(part, rng.normal(size=4), 5)
    lines = kv.dump_partition(part).strip().splitlines()
    pat = re.compile(r"^\d+ \d+ (candidate|important|desert|pad) (-?[\d.e+-]+|nan|-?inf) (-?[\d.e+-]+|nan|-?inf) (hot|warm|cold)$")
    assert len(lines) == len(part.leaves) and all(pat.match(x) for x in lines) and lines[0].startswith("0 ")


# -- engine.py behaviour (test_engine.py) ------------------------------------------------------------


def test_attention_output_examples(kv):
    q = np.array([math.sqrt(2.0), 0.0])
    out = kv.attention_output(q, np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([[1.0, 0.0], [0.0, 1.0]]))
    w = math.e / (math.e + 1.0)
    np.testing.assert_allclose(out, [w, 1.0 - w], atol=1e-12)
    rng = np.random.default_rng(0)
    q, K, V = rng.normal(size=8), rng.normal(size=(24, 8)), rng.normal(size=(24, 8))
    np.testing.assert_allclose(kv.attention_output(q, K, V), O.attention(q, K, V), rtol=1e-12, atol=1e-14)
    with pytest.raises(ValueError):
        kv.attention_output(q, K, None)
    with pytest.raises(ValueError):
        kv.attention_output(q, K, V[:-1])
    assert kv.desert_rate_on_grid({0, 1, 2}, 64, 16) == 0.75
    assert kv.token_runs([5, 1, 2, 3, 9]) == [(1, 4), (5, 6), (9, 10)]
