"""Tiered values on the GPU (host_tier.py, csrc/tier.cu): V served from an HBM hot tier over
pinned host memory.

* The attention outputs equal the fully resident decoder's bit for bit (same codes, same K7
  arithmetic, only the row addressing differs), with both the INT4 and the raw-bf16 share of
  the theta split (raw rows are quantised on the way into the pool with the K8 codec).
* The device's residency policy is the reference store's: replaying the same selections
  through TieredStore (the restatement of tiered_store.py:224-372 whose ledger is pinned to
  the reference's, tests/test_tiered_store.py) gives the same warm_to_hot / hot_to_warm bytes
  in every (step, layer) row and the same hot set at the end, with evictions in play.  The
  device serves a layer's lanes together, so the replay touches every lane of the layer
  before the ensure_hot calls (engine.py:342-343 interleaves them lane by lane; with a hot
  budget tight enough to evict a record that a later lane of the same layer still needs, the
  lane-serial loop re-fetches it within the layer, which the batched step does not)
  (random keys, a fresh query per step, 8-token records, a hot budget below the records the
  run touches)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import workload as W

pytestmark = pytest.mark.gpu

L_, H, N, D, CREC = 3, 4, 8192, 128, 8


def _workload(steps, data="random", seed=3):
    """N(0,1)-like keys and a fresh query per step (workload.py "random"): the selection, and
    with 8-token records the touched records, change from step to step."""
    from paper_2506_20187_b200 import ops
    kv = []
    qs = np.empty((steps, L_, H, D), np.float32)
    g = W.gen_args(None, D, data)
    for l in range(L_):
        p = W.lane_params(seed, l, np.arange(H), N, D, data)
        K = torch.empty((H, N, D), dtype=torch.bfloat16, device="cuda")
        V = torch.empty_like(K)
        ops.synth_layer(K, V, p, N, g)
        kv.append((K, V))
        qs[:, l] = W.queries(seed, steps, l, np.arange(H), 1, p["u"], 0, D, data)
    return kv, torch.from_numpy(qs).cuda()


def _decoders(kv, hot_records, keep_raw=False):
    from paper_2506_20187_b200 import ops
    from paper_2506_20187_b200.decode import SparseDecoder
    from paper_2506_20187_b200.host_tier import TieredDecoder
    kw = dict(importance_rate=0.1, early_layer_rate=0.1)
    res = SparseDecoder(L_, 1, H, D, N, dtype=ops.I4, **kw)
    tie = TieredDecoder(L_, 1, H, D, N, hot_records, crec=CREC, keep_raw=keep_raw, **kw)
    for l, (K, V) in enumerate(kv):
        res.load_layer(l, K, V)
        tie.load_layer(l, K, V)
    res.set_length(N)
    tie.set_length(N)
    return res, tie


def _replay_store(hot_records):
    from paper_2506_20187_b200.tiered_store import HOT, WARM, TierConfig, kv_nbytes, place_initial
    rb = kv_nbytes(CREC, D)
    cfg = TierConfig(hot_capacity=hot_records * rb, warm_capacity=10 ** 15, early_layers_pinned=0)
    st = place_initial(L_, H, D, N, cfg, CREC)
    for recs in st.lanes.values():  # the device pool starts empty: every record warm
        for r in recs:
            r.tier = WARM
    st.used = {HOT: 0, WARM: sum(r.nbytes for recs in st.lanes.values() for r in recs)}
    return st


def _runs(sel):
    runs, s = [], None
    for i, t in enumerate(sel):
        if s is None:
            s, p = t, t
        elif t == p + 1:
            p = t
        else:
            runs.append((s, p + 1))
            s, p = t, t
    if s is not None:
        runs.append((s, p + 1))
    return runs


def _selection_records(res, Q):
    """Per step, the set of (layer, lane, record) the resident decoder's selections touch."""
    out = []
    for s in range(Q.shape[0]):
        res.step(Q[s])
        recs = set()
        for l in range(L_):
            b = res._buffers()[l]
            n_sel, sel = b["n_sel"].cpu().numpy(), b["sel_tok"].cpu().numpy()
            for h in range(H):
                recs.update((l, h, int(t) // CREC) for t in sel[h, :n_sel[h]])
        out.append(recs)
    return out


@pytest.mark.parametrize("keep_raw", [False, True])
def test_tiered_outputs_equal_resident_and_ledger_equals_reference_store(keep_raw):
    steps = 6
    kv, Q = _workload(steps)
    res, _ = _decoders(kv, 1)
    ws = _selection_records(res, Q)
    peak, union = max(len(w) for w in ws), len(set().union(*ws))
    assert union > peak, "the drift must change the touched records between steps"
    hot = peak + (union - peak) // 3  # every step fits, the run does not: evictions
    del res
    res, tie = _decoders(kv, hot, keep_raw)
    if keep_raw:
        tie.set_theta([0.5, 0.0, 1.0])  # INT4 / raw shares of every layer's misses
    st = _replay_store(hot)
    evictions = 0
    for s in range(steps):
        o_res = res.step(Q[s]).clone()
        o_tie = tie.step(Q[s]).clone()
        torch.cuda.synchronize()
        assert torch.equal(o_res, o_tie), f"step {s}: tiered attention differs from resident"
        rows = tie.ledger_rows()
        for l in range(L_):
            b = tie._buffers()[l]
            n_sel = b["n_sel"].cpu().numpy()
            sel = b["sel_tok"].cpu().numpy()
            st.open_row(s, l)
            toks = [sorted(int(t) for t in sel[h, :n_sel[h]]) for h in range(H)]
            for h in range(H):  # the layer's lanes are touched together (see the module doc)
                st.touch(l, h, toks[h])
            for h in range(H):
                st.ensure_hot(l, h, _runs(toks[h]))
            row = st.close_row()
            assert rows[l]["warm_to_hot"] == row.warm_to_hot, (s, l)
            assert rows[l]["hot_to_warm"] == row.hot_to_warm, (s, l)
            evictions += row.hot_to_warm
    assert evictions > 0, "the run must exercise evictions"
    hot_ref = {(r.layer, r.head, r.start // CREC) for recs in st.lanes.values() for r in recs if r.tier == "hot"}
    assert tie.tier.hot_records() == hot_ref


def test_capacity_error_when_a_step_does_not_fit():
    from paper_2506_20187_b200.tiered_store import CapacityError
    kv, Q = _workload(1)
    _, tie = _decoders(kv, 40)
    tie.step(Q[0])
    with pytest.raises(CapacityError):
        tie.ledger_rows()


@pytest.mark.parametrize("d,kvg", [(256, 1), (128, 2)])
def test_tiered_other_shapes_match_resident(d, kvg):
    """d = 256 records and GQA (query lanes i / g share KV lane i / g's hot records): the
    paged attention over the hot tier matches the resident decoder (bit for bit without GQA;
    within 1e-5 with it)."""
    from paper_2506_20187_b200 import ops
    from paper_2506_20187_b200.decode import SparseDecoder
    from paper_2506_20187_b200.host_tier import TieredDecoder
    Lx, H, n = 2, 4, 4096
    Hkv = H // kvg
    kw = dict(importance_rate=0.1, early_layer_rate=0.1, n_kv_heads=Hkv)
    res = SparseDecoder(Lx, 1, H, d, n, dtype=ops.I4, **kw)
    tie = TieredDecoder(Lx, 1, H, d, n, 4000, crec=8, **kw)
    g = torch.Generator(device="cuda").manual_seed(7)
    for l in range(Lx):
        K = torch.randn((Hkv, n, d), device="cuda", generator=g).to(torch.bfloat16)
        V = torch.randn((Hkv, n, d), device="cuda", generator=g).to(torch.bfloat16)
        res.load_layer(l, K, V)
        tie.load_layer(l, K, V)
    res.set_length(n)
    tie.set_length(n)
    for s in range(3):
        q = torch.randn((Lx, H, d), device="cuda", generator=g)
        a, b = res.step(q).clone(), tie.step(q).clone()
        torch.cuda.synchronize()
        tie.ledger_rows()
        if kvg == 1:
            assert torch.equal(a, b), s
        else:
            err = ((a - b).norm(dim=-1) / a.norm(dim=-1)).max().item()
            assert err <= 1e-5, (s, err)
