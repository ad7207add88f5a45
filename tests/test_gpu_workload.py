"""The bench workload on the GPU: the counter-hash generator (csrc/synth.cu) equals its host
restatement (oracle ora_synth_lane) bit for bit, and SparseDecoder at config-3 shape
(B = 8 x 32 heads = 256 lanes, 64K tokens, INT4 KV, layers 0-1 at rate 0.5 / C = 8 with the
adaptive switch to C = 64 bounds, layer 2 at rate 0.1 / C = 64) selects the oracle's exact
sets and attends within tolerance on sampled lanes."""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import workload as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    oracle.build()
    return oracle


@pytest.mark.parametrize("data", ["planted", "random"])
def test_generator_device_equals_host(O, data):
    from paper_2506_20187_b200 import ops
    n, d, lanes = 3000, 128, 5
    p = W.lane_params(7, 3, np.arange(100, 100 + lanes), n, d, data)
    g = W.gen_args(None, d, data)
    K = torch.empty((lanes, n + 8, d), dtype=torch.bfloat16, device="cuda")
    V = torch.empty_like(K)
    ops.synth_layer(K, V, p, n, g)
    torch.cuda.synchronize()
    for i in range(lanes):
        kh, vh = O.synth_lane(n, d, p["seed"][i], p["u"][i], p["regions"][i], g)
        np.testing.assert_array_equal(K[i, :n].float().cpu().numpy(), kh)
        np.testing.assert_array_equal(V[i, :n].float().cpu().numpy(), vh)


def test_generator_planted_shape(O):
    """Scores separate: every hot token outranks every desert token (the planted model)."""
    n, d = 8192, 128
    p = W.lane_params(0, 5, [3], n, d, "planted")
    kh, _ = O.synth_lane(n, d, p["seed"][0], p["u"][0], p["regions"][0], W.gen_args(None, d, "planted"), values=False)
    q = W.queries(0, 1, 5, [3], 1, p["u"], 3, d)[0, 0]
    s = kh.astype(np.float64) @ q.astype(np.float64)
    hot = np.zeros(n, bool)
    for a, b in p["regions"][0]:
        hot[a:b] = True
    assert hot.sum() == math.ceil(0.3 * n)
    assert s[hot].min() > s[~hot].max()


def test_decoder_config3_shape_matches_oracle(O):
    from paper_2506_20187_b200 import ops
    from paper_2506_20187_b200.decode import SparseDecoder
    L, B, H, d, n = 3, 8, 32, 128, 65536
    lanes = B * H
    dec = SparseDecoder(L, B, H, d, n, dtype=ops.I4, device="cuda")
    g = W.gen_args(None, d, "planted")
    kb = torch.empty((lanes, n, d), dtype=torch.bfloat16, device="cuda")
    vb = torch.empty_like(kb)
    params = []
    for l in range(L):
        p = W.lane_params(11, l, np.arange(lanes), n, d, "planted")
        params.append(p)
        ops.synth_layer(kb, vb, p, n, g)
        dec.load_layer(l, kb, vb)
    del kb, vb
    torch.cuda.empty_cache()
    dec.set_length(n)
    Q = np.stack([W.queries(11, 2, l, np.arange(lanes), 1, params[l]["u"], 0, d) for l in range(L)], axis=1)
    dec.step(torch.from_numpy(Q[0]).cuda())
    torch.cuda.synchronize()
    coarse = dec.adapt_bound_granularity()
    assert coarse[0] and coarse[1] and not coarse[2]  # rate-0.5 layers prune nothing on C = 8
    out = dec.step(torch.from_numpy(Q[1]).cuda())
    torch.cuda.synchronize()
    bufs = dec._buffers()
    for l in range(L):
        k = dec.k_for(l)
        assert k == math.ceil((0.5 if l < 2 else 0.1) * n)
        sel = bufs[l]["sel_tok"][:, :k].cpu().numpy()
        o = out[l].cpu().numpy()
        for i in (0, 37, 128, 255):
            rk = dec.K.data[l, i, :n].cpu().numpy()
            rv = dec.V.data[l, i, :n].cpu().numpy()
            Kh, Vh = O.synth_lane(n, d, params[l]["seed"][i], params[l]["u"][i], params[l]["regions"][i], g)
            assert np.array_equal(rk, O.i4_quant(Kh)) and np.array_equal(rv, O.i4_quant(Vh))
            Kd, Vd = O.i4_dequant(rk, d), O.i4_dequant(rv, d)
            ref = O.select(Q[1, l, i], Kd, k)
            assert np.array_equal(np.sort(sel[i].astype(np.int64)), ref), (l, i)
            att = O.attention(Q[1, l, i], Kd, Vd, ref)
            assert np.linalg.norm(o[i] - att) / np.linalg.norm(att) <= 2e-3, (l, i)


@pytest.mark.parametrize("dtype", ["int4", "bf16"])
def test_selection_hints_across_steps_stay_exact(O, dtype):
    """The selector's per-lane hint (the previous step's k-th estimate, kvt_layer_args.sel_hint)
    is state carried across steps: repeated queries take the hinted bucket, changed ones miss it
    and fall back to the histogram.  Every step selects the oracle's exact set either way."""
    from paper_2506_20187_b200 import ops
    from paper_2506_20187_b200.decode import SparseDecoder
    L_, H, n, d = 2, 8, 16384, 128
    dt = ops.I4 if dtype == "int4" else torch.bfloat16
    dec = SparseDecoder(L_, 1, H, d, n, dtype=dt, importance_rate=0.1, early_layer_rate=0.1)
    g = W.gen_args(None, d, "planted")
    ps, Kd = [], []
    for l in range(L_):
        p = W.lane_params(5, l, np.arange(H), n, d, "planted")
        ps.append(p)
        K = torch.empty((H, n, d), dtype=torch.bfloat16, device="cuda")
        V = torch.empty_like(K)
        ops.synth_layer(K, V, p, n, g)
        dec.load_layer(l, K, V)
        if dtype == "int4":
            Kd.append(np.stack([O.i4_dequant(dec.K.data[l, i, :n].cpu().numpy(), d) for i in range(H)]))
        else:
            Kd.append(dec.K[l, :, :n].float().cpu().numpy())
    dec.set_length(n)
    planted = np.stack([W.queries(5, 1, l, np.arange(H), 1, ps[l]["u"], 0, d, "planted")[0] for l in range(L_)])
    rng = np.random.default_rng(1)
    steps = [planted, planted, planted + 0.3 * rng.standard_normal(planted.shape).astype(np.float32),
             rng.standard_normal(planted.shape).astype(np.float32), planted]
    for s, qh in enumerate(steps):
        dec.step(torch.from_numpy(qh).cuda())
        torch.cuda.synchronize()
        for l in range(L_):
            b = dec._buffers()[l]
            k = dec.k_for(l)
            sel = b["sel_tok"][:, :k].cpu().numpy()
            for i in range(H):
                ref = O.select(qh[l, i], Kd[l][i], k)
                assert np.array_equal(np.sort(sel[i].astype(np.int64)), ref), (dtype, s, l, i)
