"""INT4 KV compression (K8) and the INT4 paths of K1/K4/K5/K7 against the C oracle.

The reference has no quantizer (parity of the codes is against the codec defined in
oracle/kvt_oracle.c, itself checked against an independent numpy formulation in
tests/test_host_cpu.py); selection, logits and attention on the dequantised values are
held to the same bar as bf16: bit-exact sets/dots, attention within 1e-2."""

from __future__ import annotations

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from oracle import synth  # noqa: E402


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_20187_b200 import ops as _ops
    return _ops


@pytest.mark.parametrize("src_dt", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("d", [32, 96, 128, 256])
def test_kv_quant_codes_bitexact(ops, src_dt, d):
    rng = np.random.default_rng(d)
    lanes, n = 3, 777
    x = (rng.normal(size=(lanes, n, d)) * rng.choice([0.01, 1.0, 30.0], size=(lanes, 1, 1))).astype(np.float32)
    x[0, 5] = 0.0          # constant group -> scale 0
    x[1, 7, :32] = 3.25    # constant group with nonzero value
    x[2, 9, :32] = 1000.0 + rng.normal(size=32) * 1e-3   # narrow range at large magnitude
    x[2, 10, :32] = rng.normal(size=32) * 1e-6            # fp16-subnormal scales
    x[0, 11, :32] = 3e-41                                 # f32 subnormal inputs
    if src_dt != torch.float16:
        x[1, 12, :32] = rng.normal(size=32) * 1e5         # beyond the fp16 range: clamped
        x[1, 13, 0] = -9e4
    xt = torch.from_numpy(x).to(src_dt).cuda()
    dst = ops.I4KV.empty(lanes, n + 5, d, xt.device)
    ops.kv_quant(xt, dst, 0, n)
    got = dst.data[:, :n].cpu().numpy()
    xs = xt.float().cpu().numpy()
    for i in range(lanes):
        ref = O.i4_quant(xs[i])
        assert np.array_equal(got[i], ref), i
    # outward rounding: every dequantised value lies within half a step of its (clamped) input
    deq = np.stack([O.i4_dequant(got[i], d) for i in range(lanes)])
    scale = got[..., d // 2:].copy().view(np.float16).reshape(lanes, n, d // 32, 2)[..., 0].astype(np.float64)
    step = np.repeat(scale, 32, axis=-1)
    xc = np.clip(xs, -65504, 65504).astype(np.float64)
    assert np.all(np.abs(deq - xc) <= 0.5 * step * (1 + 1e-6) + 1e-6 * np.abs(xc) + 1e-30)


def _i4_lanes(ops, kind, lanes, n, d, seed):
    if kind == "random":
        rng = np.random.default_rng(seed)
        K = rng.normal(size=(lanes, n, d)).astype(np.float32)
        V = rng.normal(size=(lanes, n, d)).astype(np.float32)
        Q = rng.normal(size=(lanes, d)).astype(np.float32)
    else:
        K = np.empty((lanes, n, d), np.float32)
        V = np.empty_like(K)
        Q = np.empty((lanes, d), np.float32)
        for i in range(lanes):
            k, q, v, _ = synth.lane(synth.Profile(0.7, 3, 1.0, seed), 0, i, n, d, 1)
            K[i], V[i], Q[i] = k, v, q[0]
    kt = ops.I4KV.empty(lanes, n, d, "cuda")
    vt = ops.I4KV.empty(lanes, n, d, "cuda")
    ops.kv_quant(torch.from_numpy(K).to(torch.bfloat16).cuda(), kt)
    ops.kv_quant(torch.from_numpy(V).to(torch.bfloat16).cuda(), vt)
    Kd = np.stack([O.i4_dequant(kt.data[i].cpu().numpy(), d) for i in range(lanes)]).astype(np.float64)
    Vd = np.stack([O.i4_dequant(vt.data[i].cpu().numpy(), d) for i in range(lanes)]).astype(np.float64)
    return kt, vt, Kd, Vd, Q


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("kind", ["random", "planted"])
@pytest.mark.parametrize("n,C,rate", [(4096, 64, 0.1), (2000, 8, 0.5), (65536, 64, 0.1)])
def test_int4_select_attend_matches_oracle(ops, kind, n, C, rate, exact):
    lanes, d = (3 if n <= 4096 else 2), 128
    kt, vt, Kd, Vd, Q = _i4_lanes(ops, kind, lanes, n, d, seed=n)
    k = math.ceil(rate * n)
    qt = torch.from_numpy(Q).cuda()
    amax, amin = ops.abstract_build(kt, n, C)
    m = ops.n_grid_leaves(n, C)
    for i in range(lanes):
        mx = np.stack([Kd[i, c * C:(c + 1) * C].max(0) for c in range(m)])
        assert np.array_equal(amax[i, :m].double().cpu().numpy(), mx)
    ws = ops.LayerWorkspace(lanes, n, m, d, qt.device)
    out = {"sel_tok": torch.empty((lanes, k), dtype=torch.int32, device="cuda"),
           "sel_score": torch.empty((lanes, k), dtype=torch.float64, device="cuda"),
           "n_sel": torch.empty(lanes, dtype=torch.int32, device="cuda"),
           "run_start": torch.empty((lanes, k), dtype=torch.int32, device="cuda"),
           "run_len": torch.empty((lanes, k), dtype=torch.int32, device="cuda"),
           "n_runs": torch.empty(lanes, dtype=torch.int32, device="cuda"),
           "out": torch.empty((lanes, d), dtype=torch.float32, device="cuda"),
           "evals": torch.empty(lanes, dtype=torch.int64, device="cuda")}
    ops.select_attend(qt, kt, vt, amax, amin, n, k, C, ws, out, exact_scores=exact)
    torch.cuda.synchronize()
    logits = ops.token_scores(qt.double(), kt, n).cpu().numpy()
    for i in range(lanes):
        dd = O.dots(Q[i], Kd[i])
        ref = O.topk(dd, k)
        assert np.array_equal(out["sel_tok"][i].cpu().numpy().astype(np.int64), ref)
        if exact:
            assert np.array_equal(out["sel_score"][i].cpu().numpy(), dd[ref])
        else:
            A = np.abs(Q[i]).astype(np.float64) @ np.abs(Kd[i]).max(0)
            assert np.all(np.abs(out["sel_score"][i].cpu().numpy() - dd[ref]) <= 1e-6 * A)
        assert np.array_equal(logits[i], O.scores(Q[i], Kd[i]))
        att = O.attention(Q[i], Kd[i], Vd[i], ref)
        err = np.linalg.norm(out["out"][i].cpu().numpy() - att) / np.linalg.norm(att)
        assert err <= 1e-2, err


@pytest.mark.parametrize("qkind", ["normal", "wide", "f64"])
@pytest.mark.parametrize("kind", ["random", "planted"])
@pytest.mark.parametrize("d,C", [(128, 64), (128, 8), (256, 64)])
def test_i4mma_estimates_within_bound(ops, kind, qkind, d, C):
    """K4 on the integer tensor cores: every candidate's estimate lies within the per-lane
    bound err[:, 3] of its canonical f64 dot, the candidate list equals the CUDA-core f32
    path's, and the bound is tight enough to keep the re-scoring band narrow."""
    lanes, n = 5, 3000
    kt, vt, Kd, Vd, Q = _i4_lanes(ops, kind, lanes, n, d, seed=d + C)
    rng = np.random.default_rng(7)
    if qkind == "wide":  # dims spanning 10 decades: exercises the digit residual
        Q = (Q * 10.0 ** rng.uniform(-8, 2, size=Q.shape)).astype(np.float32)
    Q[lanes - 1] = 0.0   # a zero query: every estimate exact
    qt = torch.from_numpy(Q).cuda()
    if qkind == "f64":
        qt = qt.double()
    k = math.ceil(0.1 * n)
    amax, amin = ops.abstract_build(kt, n, C)
    U, Lo, A = ops.chunk_bounds(qt, amax, amin, n, C, want_A=True)
    plan = ops.select_plan(U, Lo, n, k, C, A=A, d=d)
    cs32, ct32 = ops.cand_score_f32(qt, kt, plan, n)
    cs, ct = ops.cand_score_i4mma(qt, kt, plan, n)
    torch.cuda.synchronize()
    nc = plan["n_cand"].cpu().numpy()
    err = plan["err"].cpu().numpy()
    for i in range(lanes):
        m = int(nc[i])
        toks = ct[i, :m].cpu().numpy()
        assert np.array_equal(toks, ct32[i, :m].cpu().numpy())
        dd = O.dots(Q[i].astype(np.float64) if qkind == "f64" else Q[i], Kd[i])
        est = cs[i, :m].double().cpu().numpy()
        e = err[i, 3]
        gap = np.abs(est - dd[toks]).max() if m else 0.0
        assert gap <= e, (i, gap, e)
        if i == lanes - 1:
            assert gap == 0.0
        else:
            Amax = np.abs(Q[i]).astype(np.float64) @ np.abs(Kd[i]).max(0)
            assert 0 < e <= 2e-5 * Amax, (e, Amax)
            # the f32 MMA epilogue adds ~11 u per group: within a small factor of the CUDA-core
            # f32 bound (both keep the re-scored band a few ulps wide)
            assert e <= 8 * err[i, 0]


@pytest.mark.parametrize("d", [32, 96, 128, 256])
def test_kv_dequant_bitexact(ops, d):
    """kvt_kv_dequant == the oracle's fmaf(code, scale, min) (f32 exactly; bf16/f16 = RN of it)."""
    from paper_2506_20187_b200.tier import kv_dequant
    rng = np.random.default_rng(100 + d)
    lanes, n = 3, 533
    x = (rng.normal(size=(lanes, n, d)) * 3.0).astype(np.float32)
    rec = ops.I4KV.empty(lanes, n, d, "cuda")
    ops.kv_quant(torch.from_numpy(x).cuda(), rec, 0, n)
    ref = np.stack([O.i4_dequant(rec.data[i].cpu().numpy(), d) for i in range(lanes)])
    for dt in (torch.float32, torch.bfloat16, torch.float16):
        out = torch.full((lanes, n, d), 7.0, dtype=dt, device="cuda")
        kv_dequant(rec, out, 5, n - 3)
        got = out.float().cpu().numpy()
        want = torch.from_numpy(ref).to(dt).float().numpy()
        assert np.array_equal(got[:, 5:n - 3], want[:, 5:n - 3]), dt
        assert np.all(got[:, :5] == 7.0) and np.all(got[:, n - 3:] == 7.0), dt


def test_codec_reciprocal_exhaustive(ops):
    """The codec's fast reciprocal equals fl32(1/s) for every positive finite fp16 scale."""
    from paper_2506_20187_b200 import _lib as L
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    L.check(L.kvt_i4_recip_check(bad.data_ptr(), torch.cuda.current_stream().cuda_stream), "recip_check")
    assert int(bad.item()) == 0


@pytest.mark.parametrize("dt", ["int4", "bf16"])
@pytest.mark.parametrize("kind", ["random", "planted"])
@pytest.mark.parametrize("Hkv", [1, 2, 8])
def test_gqa_kv_sharing_matches_oracle(ops, dt, kind, Hkv):
    """Config 4 layout (GQA): query lanes b*H + h read KV lane b*Hkv + h // g.  Each query lane's
    selection is the oracle top-k of ITS query against the shared keys (the reference
    replicates the KV head per query head, adapters.py:121-136 -- identical results).
    Hkv = H is the plain multi-layer decoder (one workspace shared by layers of different C)."""
    from paper_2506_20187_b200.decode import SparseDecoder
    B, H, d, n, L = 2, 8, 128, 4096, 3
    g = H // Hkv
    rng = np.random.default_rng(11)
    if kind == "random":
        K = rng.normal(size=(B * Hkv, n, d)).astype(np.float32)
        V = rng.normal(size=(B * Hkv, n, d)).astype(np.float32)
        Q = rng.normal(size=(B * H, d)).astype(np.float32)
    else:
        K = np.empty((B * Hkv, n, d), np.float32)
        V = np.empty_like(K)
        Q = np.empty((B * H, d), np.float32)
        for j in range(B * Hkv):
            k, q, v, _ = synth.lane(synth.Profile(0.7, 3, 1.0, 5), 0, j, n, d, 1)
            K[j], V[j] = k, v
            for h in range(g):  # query heads of a group: same planted direction, own noise
                Q[j * g + h] = q[0] * (1.0 + 0.1 * h) + rng.normal(size=d).astype(np.float32) * 0.05
    dec = SparseDecoder(L, B, H, d, n, dtype=ops.I4 if dt == "int4" else torch.bfloat16, device="cuda",
                        n_kv_heads=Hkv)
    kt = torch.from_numpy(K).to(torch.bfloat16).cuda()
    vt = torch.from_numpy(V).to(torch.bfloat16).cuda()
    for l in range(L):
        dec.load_layer(l, kt, vt)
    dec.set_length(n)
    q = torch.from_numpy(Q).cuda()[None].expand(L, -1, -1).contiguous()
    out = dec.step(q)
    torch.cuda.synchronize()
    if dt == "int4":
        Kd = np.stack([O.i4_dequant(dec.K.data[0, j].cpu().numpy(), d) for j in range(B * Hkv)]).astype(np.float64)
        Vd = np.stack([O.i4_dequant(dec.V.data[0, j].cpu().numpy(), d) for j in range(B * Hkv)]).astype(np.float64)
    else:
        Kd, Vd = kt.double().cpu().numpy(), vt.double().cpu().numpy()
    for l in (0, 2):
        bufs = dec._buffers()[l]
        k = dec.k_for(l)
        for i in range(B * H):
            j = i // g
            ref = O.topk(O.dots(Q[i], Kd[j]), k)
            got = bufs["sel_tok"][i, :k].cpu().numpy().astype(np.int64)
            assert np.array_equal(got, ref), (dt, kind, l, i)
            att = O.attention(Q[i], Kd[j], Vd[j], ref)
            err = np.linalg.norm(out[l, i].cpu().numpy() - att) / np.linalg.norm(att)
            assert err <= 1e-2, (dt, kind, l, i, err)


@pytest.mark.parametrize("g", [2, 4])
@pytest.mark.parametrize("overlap", ["same", "mixed", "disjoint"])
@pytest.mark.parametrize("k", [700, 2200])
def test_gqa_union_attention_matches_oracle(ops, g, overlap, k):
    """The GQA union kernels (attn_gqa.cu: a union plan per 2048-token window, then one pass over
    the group's union with P.V on the tensor cores, the heads as MMA rows) against the f64 oracle
    over the same selections, with identical, partly shared and disjoint per-head selections
    across several token windows."""
    n_kv, d, n = 3, 128, 9000
    rng = np.random.default_rng(7 + g)
    V = torch.from_numpy(rng.normal(size=(n_kv, n, d)).astype(np.float32)).cuda()
    vi = ops.I4KV.empty(n_kv, n, d, "cuda")
    ops.kv_quant(V, vi)
    Vd = np.stack([O.i4_dequant(vi.data[j].cpu().numpy(), d) for j in range(n_kv)]).astype(np.float64)
    sel = np.zeros((n_kv * g, k), np.int32)
    for j in range(n_kv):
        base = np.sort(rng.choice(n, size=k, replace=False))
        for h in range(g):
            if overlap == "same":
                s_ = base
            elif overlap == "disjoint":
                s_ = np.sort(rng.choice(np.arange(h, n, g), size=k, replace=False))
            else:
                s_ = np.sort(np.unique(np.concatenate([base[: k // 2], rng.choice(n, size=k, replace=False)]))[:k])
                if len(s_) < k:
                    s_ = base
            sel[j * g + h] = s_
    score = (rng.normal(size=(n_kv * g, k)) * 30.0).astype(np.float64)
    st = torch.from_numpy(sel).cuda()
    ss = torch.from_numpy(score).cuda()
    ns = torch.full((n_kv * g,), k, dtype=torch.int32, device="cuda")
    out = ops.sparse_decode_attn_gqa(vi, st, ss, ns, g, n).cpu().numpy()
    scale = 1.0 / np.sqrt(d)
    for i in range(n_kv * g):
        w = np.exp((score[i] - score[i].max()) * scale)
        ref = (w[:, None] * Vd[i // g][sel[i]]).sum(0) / w.sum()
        err = np.linalg.norm(out[i] - ref) / np.linalg.norm(ref)
        assert err <= 2e-5, (g, overlap, i, err)


@pytest.mark.parametrize("d", [128, 256])
@pytest.mark.parametrize("g", [2, 3, 4, 6, 8])
def test_gqa_shared_bounds_equal_replicated(ops, g, d):
    """Group-shared K3 (one abstract read per KV lane for its g query lanes; even groups take the
    paired-head kernel, odd ones the per-head loop) gives bit-identical U, L, A to the
    single-head kernel over replicated abstracts (the reference's per-head replication,
    adapters.py:121-136)."""
    n_kv, n, C = 5, 3000, 64
    rng = np.random.default_rng(g)
    K = torch.from_numpy(rng.normal(size=(n_kv, n, d)).astype(np.float32)).to(torch.bfloat16).cuda()
    q = torch.from_numpy(rng.normal(size=(n_kv * g, d)).astype(np.float32)).cuda()
    amax, amin = ops.abstract_build(K, n, C, abs_dtype=torch.bfloat16)
    mag = ops.lane_abs_mag(amax, amin, ops.n_grid_leaves(n, C))
    with ops.kv_group(g):
        U1, L1, A1 = ops.chunk_bounds_fast(q, amax, amin, n, C, mag)
    rep = lambda t: t.repeat_interleave(g, dim=0).contiguous()
    U0, L0, A0 = ops.chunk_bounds_fast(q, rep(amax), rep(amin), n, C, rep(mag))
    torch.cuda.synchronize()
    assert torch.equal(U1, U0) and torch.equal(L1, L0) and torch.equal(A1, A0)


@pytest.mark.parametrize("dt", ["int4", "bf16"])
def test_adaptive_bound_granularity_keeps_the_selection(ops, dt):
    """Switching a C = 8 layer's pruning to the C = 64 abstracts changes only how much is
    pruned: the selected sets and the attention outputs are identical."""
    from paper_2506_20187_b200.decode import SparseDecoder
    B, H, d, n, L = 1, 4, 128, 4096, 3
    rng = np.random.default_rng(3)
    K = torch.from_numpy(rng.normal(size=(B * H, n, d)).astype(np.float32)).to(torch.bfloat16).cuda()
    dec = SparseDecoder(L, B, H, d, n, dtype=ops.I4 if dt == "int4" else torch.bfloat16, device="cuda")
    for l in range(L):
        dec.load_layer(l, K, K)
    dec.set_length(n)
    q = torch.from_numpy(rng.normal(size=(L, B * H, d)).astype(np.float32)).cuda()
    out0 = dec.step(q).clone()
    sel0 = [dec._buffers()[l]["sel_tok"].clone() for l in range(L)]
    flags = dec.adapt_bound_granularity(threshold=0.0)  # force the coarse grid where one exists
    assert flags[:2] == [True, True] and not flags[2]
    out1 = dec.step(q)
    torch.cuda.synchronize()
    for l in range(L):
        assert torch.equal(dec._buffers()[l]["sel_tok"], sel0[l]), l
    assert torch.equal(out0, out1)


@pytest.mark.parametrize("dt", ["int4", "bf16"])
def test_decoder_head_dim_256(ops, dt):
    """d = 256 through the decode path (fast bounds G = 2, INT4 MMA scoring R = 2, 256-wide
    attention formats): every layer's selection equals the oracle and attention is within 1e-2."""
    from paper_2506_20187_b200.decode import SparseDecoder
    B, H, d, n, L = 1, 4, 256, 2048, 3
    rng = np.random.default_rng(9)
    K = rng.normal(size=(B * H, n, d)).astype(np.float32)
    V = rng.normal(size=(B * H, n, d)).astype(np.float32)
    Q = rng.normal(size=(L, B * H, d)).astype(np.float32)
    dec = SparseDecoder(L, B, H, d, n, dtype=ops.I4 if dt == "int4" else torch.bfloat16, device="cuda")
    kt = torch.from_numpy(K).to(torch.bfloat16).cuda()
    vt = torch.from_numpy(V).to(torch.bfloat16).cuda()
    for l in range(L):
        dec.load_layer(l, kt, vt)
    dec.set_length(n)
    out = dec.step(torch.from_numpy(Q).cuda())
    torch.cuda.synchronize()
    for l in range(L):
        if dt == "int4":
            Kd = np.stack([O.i4_dequant(dec.K.data[l, j].cpu().numpy(), d) for j in range(B * H)]).astype(np.float64)
            Vd = np.stack([O.i4_dequant(dec.V.data[l, j].cpu().numpy(), d) for j in range(B * H)]).astype(np.float64)
        else:
            Kd, Vd = kt.double().cpu().numpy(), vt.double().cpu().numpy()
        k = dec.k_for(l)
        for i in range(B * H):
            ref = O.topk(O.dots(Q[l, i], Kd[i]), k)
            got = dec._buffers()[l]["sel_tok"][i, :k].cpu().numpy().astype(np.int64)
            assert np.array_equal(got, ref), (dt, l, i)
            att = O.attention(Q[l, i], Kd[i], Vd[i], ref)
            assert np.linalg.norm(out[l, i].cpu().numpy() - att) / np.linalg.norm(att) <= 1e-2


@pytest.mark.parametrize("dt", ["int4", "bf16"])
def test_decoder_append_odd_context_matches_oracle(ops, dt):
    """Decode while appending: an odd context (not a multiple of 8 or 64), one appended token per
    step (tail-chunk abstracts, |key| maxima and coarse abstracts refreshed), the adaptive
    coarse grid switched on midway.  Every step's selection equals the oracle top-k over the
    current context and attention is within 1e-2."""
    from paper_2506_20187_b200.decode import SparseDecoder
    B, H, d, n0, L, steps = 1, 2, 128, 1001, 3, 4
    rng = np.random.default_rng(21)
    cap = n0 + steps
    K = rng.normal(size=(B * H, cap, d)).astype(np.float32)
    V = rng.normal(size=(B * H, cap, d)).astype(np.float32)
    K[:, -2:] *= 3.0  # appended tokens with large keys: they must enter the selection
    dec = SparseDecoder(L, B, H, d, cap, dtype=ops.I4 if dt == "int4" else torch.bfloat16, device="cuda")
    kt = torch.from_numpy(K).to(torch.bfloat16).cuda()
    vt = torch.from_numpy(V).to(torch.bfloat16).cuda()
    for l in range(L):
        dec.load_layer(l, kt[:, :n0], vt[:, :n0])
    dec.set_length(n0)
    for s in range(steps):
        q = torch.from_numpy(rng.normal(size=(L, B * H, d)).astype(np.float32)).cuda()
        out = dec.step(q)
        torch.cuda.synchronize()
        n = dec.n
        for l in range(L):
            if dt == "int4":
                Kd = np.stack([O.i4_dequant(dec.K.data[l, j, :n].cpu().numpy(), d) for j in range(B * H)]).astype(np.float64)
                Vd = np.stack([O.i4_dequant(dec.V.data[l, j, :n].cpu().numpy(), d) for j in range(B * H)]).astype(np.float64)
            else:
                Kd, Vd = kt[:, :n].double().cpu().numpy(), vt[:, :n].double().cpu().numpy()
            k = dec.k_for(l)
            for i in range(B * H):
                qi = q[l, i].cpu().numpy()
                ref = O.topk(O.dots(qi, Kd[i]), k)
                got = dec._buffers()[l]["sel_tok"][i, :k].cpu().numpy().astype(np.int64)
                assert np.array_equal(got, ref), (dt, s, l, i)
                att = O.attention(qi, Kd[i], Vd[i], ref)
                assert np.linalg.norm(out[l, i].cpu().numpy() - att) / np.linalg.norm(att) <= 1e-2
        if s == 1:
            dec.adapt_bound_granularity(threshold=0.0)
        if s < steps - 1:
            kn = kt[:, n:n + 1].permute(1, 0, 2).expand(L, -1, -1).contiguous()
            vn = vt[:, n:n + 1].permute(1, 0, 2).expand(L, -1, -1).contiguous()
            dec.append(kn, vn)


def test_int4_select3_many_lanes(ops):
    """INT4 keys (many exact score ties from the 4-bit codes) through the many-lane selector at
    64K: sets bit-exact against the canonical scores of the dequantised keys."""
    lanes, n, d, C = 38, 65536, 128, 64
    k = math.ceil(0.1 * n)
    kt, vt, Kd, Vd, Q = _i4_lanes(ops, "random", lanes, n, d, seed=9)
    del Vd
    qt = torch.from_numpy(Q).cuda()
    amax, amin = ops.abstract_build(kt, n, C)
    ws = ops.LayerWorkspace(lanes, n, ops.n_grid_leaves(n, C), d, qt.device)
    out = {"sel_tok": torch.empty((lanes, k), dtype=torch.int32, device="cuda"),
           "sel_score": torch.empty((lanes, k), dtype=torch.float64, device="cuda"),
           "n_sel": torch.empty(lanes, dtype=torch.int32, device="cuda"),
           "out": torch.empty((lanes, d), dtype=torch.float32, device="cuda")}
    ops.select_attend(qt, kt, vt, amax, amin, n, k, C, ws, out)
    s = ops.token_scores(qt.double(), torch.from_numpy(Kd).cuda(), n)
    ref = torch.sort(torch.sort(-s, dim=1, stable=True).indices[:, :k], dim=1).values
    bad = (out["sel_tok"].long() != ref).any(1).nonzero().flatten().tolist()
    assert not bad, bad[:5]
    for i in (0, lanes - 1):
        assert np.array_equal(out["sel_tok"][i].cpu().numpy().astype(np.int64), O.topk(O.dots(Q[i], Kd[i]), k))


def test_gqa_union_long_selections_multiwindow_ranges(ops):
    """Long, near-uniform-weight selections (rate 0.5, small score spread) over many KV lanes, so
    each P.V range spans several windows: the centred code split keeps the tensor-core sums
    free of cancellation (the uncentred one drifted to ~2e-3 here)."""
    g, n_kv, d, n, k = 4, 40, 128, 65536, 32768
    rng = np.random.default_rng(11)
    V = torch.from_numpy(rng.normal(size=(n_kv, n, d)).astype(np.float32)).cuda()
    vi = ops.I4KV.empty(n_kv, n, d, "cuda")
    ops.kv_quant(V, vi)
    sel = np.zeros((n_kv * g, k), np.int32)
    for j in range(n_kv):
        base = np.sort(rng.choice(n, size=k, replace=False))
        for h in range(g):
            sel[j * g + h] = base
    score = (rng.normal(size=(n_kv * g, k)) * 0.3 + 20.0).astype(np.float64)
    st, ss = torch.from_numpy(sel).cuda(), torch.from_numpy(score).cuda()
    ns = torch.full((n_kv * g,), k, dtype=torch.int32, device="cuda")
    out = ops.sparse_decode_attn_gqa(vi, st, ss, ns, g, n).cpu().numpy()
    scale = 1.0 / np.sqrt(d)
    for j in (0, 17, n_kv - 1):
        Vd = O.i4_dequant(vi.data[j].cpu().numpy(), d).astype(np.float64)
        for h in range(g):
            i = j * g + h
            w = np.exp((score[i] - score[i].max()) * scale)
            ref = (w[:, None] * Vd[sel[i]]).sum(0) / w.sum()
            err = np.linalg.norm(out[i] - ref) / np.linalg.norm(ref)
            assert err <= 2e-5, (j, h, err)


def test_fused_append_equals_per_layer_path(ops):
    """kvt_kv_append (one launch per decode step: INT4 records of every layer and lane, the tail
    chunk of every bf16 abstract grid, absmag) equals the per-layer path bit for bit, across a
    chunk boundary and with an intermediate grid from adapt_chunking."""
    from paper_2506_20187_b200.decode import SparseDecoder
    L_, H, d, n0 = 3, 4, 128, 1000
    a = SparseDecoder(L_, 1, H, d, n0 + 80, dtype=ops.I4, importance_rate=0.1, early_layer_rate=0.5)
    b = SparseDecoder(L_, 1, H, d, n0 + 80, dtype=ops.I4, importance_rate=0.1, early_layer_rate=0.5)
    g = torch.Generator(device="cuda").manual_seed(3)
    for l in range(L_):
        K = torch.randn((H, n0, d), device="cuda", generator=g).to(torch.bfloat16)
        V = torch.randn((H, n0, d), device="cuda", generator=g).to(torch.bfloat16)
        a.load_layer(l, K, V)
        b.load_layer(l, K, V)
    a.set_length(n0)
    b.set_length(n0)
    for dec in (a, b):  # an intermediate grid (C = 16) on layer 0
        dec._ensure_grid(0, 16)
    for s in range(70):  # crosses the 64- and 16-token chunk boundaries
        kn = (torch.randn((L_, H, d), device="cuda", generator=g) * 3).to(torch.bfloat16)
        vn = torch.randn((L_, H, d), device="cuda", generator=g).to(torch.bfloat16)
        a.append(kn, vn, fused=True)
        b.append(kn, vn, fused=False)
    torch.cuda.synchronize()
    n = n0 + 70
    assert torch.equal(a.K.data[:, :, :n], b.K.data[:, :, :n]) and torch.equal(a.V.data[:, :, :n], b.V.data[:, :, :n])
    for l in range(L_):
        m = ops.n_grid_leaves(n, a.C[l])
        assert torch.equal(a.amax[l][:, :m], b.amax[l][:, :m]) and torch.equal(a.amin[l][:, :m], b.amin[l][:, :m])
        assert torch.equal(a.absmag[l], b.absmag[l])
        if a.amax_c[l] is not None:
            mc = ops.n_grid_leaves(n, a.coarse_C)
            assert torch.equal(a.amax_c[l][:, :mc], b.amax_c[l][:, :mc])
    mx_a, mn_a = a._mid[(0, 16)]
    mx_b, mn_b = b._mid[(0, 16)]
    m16 = ops.n_grid_leaves(n, 16)
    assert torch.equal(mx_a[:, :m16], mx_b[:, :m16]) and torch.equal(mn_a[:, :m16], mn_b[:, :m16])
