"""Kernel-level parity on the B200: every C-ABI stage against the C oracle.

Bar (BASELINE.json north_star): logits, bounds, abstracts, selected sets, runs and
partitions bit-exact; attention within 2e-3 relative (f32 values) / 1e-2 (bf16)."""

from __future__ import annotations

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from oracle import synth  # noqa: E402

DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16, "f64": torch.float64}


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_20187_b200 import ops as _ops
    return _ops


def _keys(rng, lanes, n, d, dt):
    k = rng.normal(size=(lanes, n, d)).astype(np.float32)
    t = torch.from_numpy(k).to(DT[dt]).cuda()
    return t, t.double().cpu().numpy()


@pytest.mark.parametrize("dt", ["f32", "bf16", "f16", "f64"])
@pytest.mark.parametrize("d", [1, 4, 16, 64, 100, 128, 256])
def test_token_scores_bitexact(ops, dt, d):
    rng = np.random.default_rng(d)
    lanes, n = 3, 301
    kt, kh = _keys(rng, lanes, n, d, dt)
    q = rng.normal(size=(lanes, d))
    qt = torch.from_numpy(q).cuda()
    got = ops.token_scores(qt, kt, n).cpu().numpy()
    for i in range(lanes):
        ref = O.scores(q[i], kh[i])
        assert np.array_equal(got[i], ref), (dt, d, i)


@pytest.mark.parametrize("dt", ["f32", "bf16", "f64"])
@pytest.mark.parametrize("d,C", [(4, 1), (16, 8), (64, 64), (128, 64), (128, 8), (100, 7)])
def test_abstracts_and_bounds_bitexact(ops, dt, d, C):
    rng = np.random.default_rng(7 * d + C)
    lanes, n = 2, 517
    kt, kh = _keys(rng, lanes, n, d, dt)
    q = rng.normal(size=(lanes, d)) * rng.choice([0.1, 1.0, 10.0])
    q[:, 0] = 0.0
    amax, amin = ops.abstract_build(kt, n, C)
    U, L = ops.chunk_bounds(torch.from_numpy(q).cuda(), amax, amin, n, C, scaled=True)
    Ur_raw, Lr_raw = ops.chunk_bounds(torch.from_numpy(q).cuda(), amax, amin, n, C)
    m = ops.n_grid_leaves(n, C)
    for i in range(lanes):
        mx = np.stack([kh[i, c * C:(c + 1) * C].max(0) for c in range(m)])
        mn = np.stack([kh[i, c * C:(c + 1) * C].min(0) for c in range(m)])
        assert np.array_equal(amax[i, :m].double().cpu().numpy(), mx)
        assert np.array_equal(amin[i, :m].double().cpu().numpy(), mn)
        rows = [min(C, n - c * C) for c in range(m)]
        Ur, Lr = O.bounds(q[i], mx, mn, rows)
        assert np.array_equal(U[i, :m].cpu().numpy(), Ur)
        assert np.array_equal(L[i, :m].cpu().numpy(), Lr)
        s = O.scores(q[i], kh[i])
        for c in range(m):
            seg = s[c * C:(c + 1) * C]
            assert Lr[c] <= seg.min() and seg.max() <= Ur[c]  # sound for canonical logits
        Ur2, Lr2 = O.bounds(q[i], mx, mn, rows, scaled=False)
        assert np.array_equal(Ur_raw[i, :m].cpu().numpy(), Ur2)
        assert np.array_equal(Lr_raw[i, :m].cpu().numpy(), Lr2)
        dd = O.dots(q[i], kh[i])
        for c in range(m):
            seg = dd[c * C:(c + 1) * C]
            assert Lr2[c] <= seg.min() and seg.max() <= Ur2[c]  # sound for raw canonical dots


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_bf16_abstracts_outward_and_bounds_bitexact(ops, dt):
    """bf16 abstracts round max up / min down; bounds over them are bit-exact vs the oracle
    fed the same rounded abstracts, and sound for every canonical dot."""
    rng = np.random.default_rng(11)
    lanes, n, d, C = 3, 1000, 128, 64
    kt, kh = _keys(rng, lanes, n, d, dt)
    q = rng.normal(size=(lanes, d))
    amax, amin = ops.abstract_build(kt, n, C, abs_dtype=torch.bfloat16)
    U, L = ops.chunk_bounds(torch.from_numpy(q).cuda(), amax, amin, n, C)
    m = ops.n_grid_leaves(n, C)
    for i in range(lanes):
        mx = np.stack([kh[i, c * C:(c + 1) * C].max(0) for c in range(m)])
        mn = np.stack([kh[i, c * C:(c + 1) * C].min(0) for c in range(m)])
        bmx = amax[i, :m].double().cpu().numpy()
        bmn = amin[i, :m].double().cpu().numpy()
        assert np.all(bmx >= mx) and np.all(bmn <= mn)
        rt = lambda a: torch.from_numpy(a).float().to(torch.bfloat16).double().numpy()
        assert np.all(bmx <= np.nextafter(rt(mx) + np.abs(rt(mx)) * 2 ** -7, np.inf))
        rows = [min(C, n - c * C) for c in range(m)]
        Ur, Lr = O.bounds(q[i], bmx, bmn, rows, scaled=False)
        assert np.array_equal(U[i, :m].cpu().numpy(), Ur) and np.array_equal(L[i, :m].cpu().numpy(), Lr)
        dd = O.dots(q[i], kh[i])
        for c in range(m):
            seg = dd[c * C:(c + 1) * C]
            assert Lr[c] <= seg.min() and seg.max() <= Ur[c]


def test_bound_soundness_c02(ops):
    """test_acceptance.py:101-123 criterion 2, on canonical logits (no tolerance)."""
    rng = np.random.default_rng(2024)
    d, lanes, C = 64, 64, 64
    for rep in range(25):
        scale = float(rng.lognormal(0.0, 1.0))
        k = rng.normal(scale=scale, size=(lanes, C, d))
        k[rng.random(lanes) < 0.1] = k[:1, :1]
        q = rng.normal(scale=scale, size=(lanes, d))
        q[rng.random(lanes) < 0.05] = 0.0
        kt = torch.from_numpy(k).cuda()
        amax, amin = ops.abstract_build(kt, C, C)
        U, L = ops.chunk_bounds(torch.from_numpy(q).cuda(), amax, amin, C, C, scaled=True)
        s = ops.token_scores(torch.from_numpy(q).cuda(), kt, C).cpu().numpy()
        assert np.all(L[:, 0].cpu().numpy() <= s.min(1))
        assert np.all(s.max(1) <= U[:, 0].cpu().numpy())


def _lane_data(kind, lanes, n, d, seed):
    if kind == "random":
        rng = np.random.default_rng(seed)
        return (rng.normal(size=(lanes, n, d)).astype(np.float32), rng.normal(size=(lanes, n, d)).astype(np.float32),
                rng.normal(size=(lanes, d)).astype(np.float32))
    if kind == "ties":
        rng = np.random.default_rng(seed)
        K = np.ones((lanes, n, d), np.float32)
        K[:, ::7] = 2.0
        return K, rng.normal(size=(lanes, n, d)).astype(np.float32), np.ones((lanes, d), np.float32)
    if kind == "neartie":
        # many keys whose dots differ by a few f64 ulps only: the f32 estimates tie, the
        # canonical f64 dots do not -> exercises the band re-scoring
        rng = np.random.default_rng(seed)
        K = rng.normal(size=(lanes, n, d)).astype(np.float32)
        Q = np.ones((lanes, d), np.float32)
        base = np.full(d, 0.25, np.float32)
        K[:, : n // 3] = base
        K[:, : n // 3, 0] += (np.arange(n // 3) % 97 * 2.0 ** -20).astype(np.float32)
        return K, rng.normal(size=(lanes, n, d)).astype(np.float32), Q
    K = np.empty((lanes, n, d), np.float32)
    V = np.empty_like(K)
    Q = np.empty((lanes, d), np.float32)
    for i in range(lanes):
        k, q, v, _ = synth.lane(synth.Profile(desert_rate=0.7, seed=seed), 0, i, n, d, 1)
        K[i], V[i], Q[i] = k, v, q[0]
    return K, V, Q


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("kind", ["random", "planted", "ties", "neartie"])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("n,C,rate", [(4096, 64, 0.10), (1000, 8, 0.5), (65536, 64, 0.10), (33, 4, 0.1)])
def test_fused_select_attend_matches_oracle(ops, kind, dt, n, C, rate, exact):
    lanes, d = (4 if n <= 4096 else 2), 128
    K, V, Q = _lane_data(kind, lanes, n, d, seed=n + C)
    k = math.ceil(rate * n)
    kt = torch.from_numpy(K).to(DT[dt]).cuda()
    vt = torch.from_numpy(V).to(DT[dt]).cuda()
    qt = torch.from_numpy(Q).cuda()
    amax, amin = ops.abstract_build(kt, n, C)
    ws = ops.LayerWorkspace(lanes, n, ops.n_grid_leaves(n, C), d, kt.device)
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
    Kh = kt.double().cpu().numpy()
    Vh = vt.double().cpu().numpy()
    tol = 2e-3 if dt == "f32" else 1e-2
    for i in range(lanes):
        s = O.dots(Q[i], Kh[i])
        ref = O.topk(s, k)
        got = out["sel_tok"][i].cpu().numpy().astype(np.int64)
        assert np.array_equal(got, ref), (kind, dt, n, i)
        if exact:
            assert np.array_equal(out["sel_score"][i].cpu().numpy(), s[ref])
        else:  # f32 estimates for the sure tokens, canonical for the band
            A = np.abs(Q[i]).astype(np.float64) @ np.abs(Kh[i]).max(0)
            assert np.all(np.abs(out["sel_score"][i].cpu().numpy() - s[ref]) <= 1e-6 * A)
        runs = O.runs(ref)
        nr = int(out["n_runs"][i])
        assert nr == len(runs)
        rs = out["run_start"][i, :nr].cpu().numpy()
        rl = out["run_len"][i, :nr].cpu().numpy()
        assert [(int(a), int(a + b)) for a, b in zip(rs, rl)] == runs
        att = O.attention(Q[i], Kh[i], Vh[i], ref)
        err = np.linalg.norm(out["out"][i].cpu().numpy() - att) / np.linalg.norm(att)
        assert err <= tol, err
        assert int(out["evals"][i]) >= ops.n_grid_leaves(n, C) + k


def test_select_plan_prunes_planted(ops):
    n, d, C = 65536, 128, 64
    K, V, Q = _lane_data("planted", 2, n, d, seed=3)
    kt = torch.from_numpy(K).cuda()
    amax, amin = ops.abstract_build(kt, n, C)
    U, L = ops.chunk_bounds(torch.from_numpy(Q).cuda(), amax, amin, n, C)
    plan = ops.select_plan(U, L, n, math.ceil(0.1 * n), C)
    frac = plan["n_cand"].cpu().numpy() / n
    assert np.all(frac < 0.45), frac  # ~30% hot + boundary chunks


def test_runs_partition(ops):
    rng = np.random.default_rng(0)
    n = 5000
    for trial in range(20):
        k = int(rng.integers(0, 300))
        sel = np.sort(rng.choice(n, size=k, replace=False)) if k else np.zeros(0, np.int64)
        st = torch.from_numpy(sel.astype(np.int32))[None].cuda()
        ns = torch.tensor([k], dtype=torch.int32).cuda()
        r = ops.runs_scan(st if k else torch.zeros((1, 0), dtype=torch.int32, device="cuda"), ns, n)
        npart = int(r["n_part"][0])
        ps = r["part_start"][0, :npart].cpu().numpy()
        pst = r["part_state"][0, :npart].cpu().numpy()
        pe = np.append(ps[1:], n)
        got = [(int(a), int(b), "important" if c == 1 else "desert") for a, b, c in zip(ps, pe, pst)]
        ref = [x for x in O.canonical_partition(sel, n) if x[2] != "pad"]
        assert got == ref


@pytest.mark.parametrize("C,n", [(8, 65536), (8, 1003), (4, 517), (64, 4096), (0, 3000)])
def test_select_plan_items_merge_candidate_runs(ops, C, n):
    """Items tile exactly the candidate tokens in ascending order (out_pos = stream index),
    hold <= 64 tokens, and are cut only at run starts and multiples of 64."""
    rng = np.random.default_rng(C * 7 + n)
    lanes = 3
    if C:
        nl = ops.n_grid_leaves(n, C)
        starts = [np.arange(nl) * C for _ in range(lanes)]
        ls = nleaves = None
    else:  # explicit partition with random leaf sizes
        starts = []
        for _ in range(lanes):
            cuts = np.sort(rng.choice(np.arange(1, n), size=400, replace=False))
            starts.append(np.concatenate([[0], cuts]))
        nl = max(len(s) for s in starts)
        ls = torch.zeros((lanes, nl), dtype=torch.int32)
        for i, s in enumerate(starts):
            ls[i, :len(s)] = torch.from_numpy(s.astype(np.int32))
        ls = ls.cuda()
        nleaves = torch.tensor([len(s) for s in starts], dtype=torch.int32, device="cuda")
    U = torch.from_numpy(rng.normal(size=(lanes, nl))).cuda()
    Lo = U - 1.0
    k = max(1, n // 3)
    plan = ops.select_plan(U, Lo, n, k, C, leaf_start=ls, n_leaves=nleaves, want_cand_leaf=True)
    for i in range(lanes):
        st = starts[i]
        ends = np.append(st[1:], n)
        cl = plan["cand_leaf"][i, :len(st)].cpu().numpy().astype(bool)
        cand_tok = np.concatenate([np.arange(a, b) for a, b, c in zip(st, ends, cl) if c] or [np.zeros(0, int)])
        ni = int(plan["n_items"][i])
        it = plan["items"][i, :ni].cpu().numpy()
        assert int(plan["n_cand"][i]) == len(cand_tok)
        toks = np.concatenate([np.arange(t, t + c) for t, c, _ in it] or [np.zeros(0, int)])
        assert np.array_equal(toks, cand_tok)
        assert np.all(it[:, 1] >= 1) and np.all(it[:, 1] <= 64)
        assert np.array_equal(it[:, 2], np.concatenate([[0], np.cumsum(it[:-1, 1])]) if ni else it[:, 2])
        # maximal: an item boundary inside a run only at multiples of 64
        for a, b in zip(it[:-1], it[1:]):
            if a[0] + a[1] == b[0]:
                assert b[0] % 64 == 0


@pytest.mark.parametrize("kind", ["random", "planted"])
@pytest.mark.parametrize("d,C,n", [(128, 64, 4096), (128, 8, 1003), (256, 64, 2049)])
def test_chunk_bounds_fast_sound_and_tight(ops, kind, d, C, n):
    """Directed-rounding f32 bounds enclose the canonical f64 bounds of the same bf16 abstracts
    (hence every dot of the chunk) and stay within ~1e-6 relative of them; A_lane bounds A."""
    lanes = 3
    K, V, Q = _lane_data(kind, lanes, n, d, seed=d + C)
    kt = torch.from_numpy(K).to(torch.bfloat16).cuda()
    qt = torch.from_numpy(Q).cuda()
    amax, amin = ops.abstract_build(kt, n, C, abs_dtype=torch.bfloat16)
    m = ops.n_grid_leaves(n, C)
    mag = ops.lane_abs_mag(amax, amin, m)
    Uf, Lf, Af = ops.chunk_bounds_fast(qt, amax, amin, n, C, mag)
    Uc, Lc, Ac = ops.chunk_bounds(qt, amax, amin, n, C, want_A=True)
    Uf, Lf, Af, Uc, Lc, Ac = (x[:, :m].cpu().numpy() for x in (Uf, Lf, Af, Uc, Lc, Ac))
    # canonical bounds carry their own widening slack; compare against the exact abstract sums
    mx = amax[:, :m].double().cpu().numpy()
    mn = amin[:, :m].double().cpu().numpy()
    q = Q.astype(np.float64)[:, None, :]
    Ux = np.where(q >= 0, q * mx, q * mn).sum(-1)
    Lx = np.where(q >= 0, q * mn, q * mx).sum(-1)
    Ax = (np.abs(q) * np.maximum(np.abs(mx), np.abs(mn))).sum(-1)
    assert np.all(Uf >= Ux) and np.all(Lf <= Lx)
    assert np.all(Uf - Ux <= 1e-5 * Ax + 1e-30) and np.all(Lx - Lf <= 1e-5 * Ax + 1e-30)
    assert np.all(Af >= Ax.max(1, keepdims=True) * (1 - 1e-12))
    # every canonical dot of the chunk (bf16 keys) lies inside
    dots = np.einsum("lnd,ld->ln", kt.double().cpu().numpy(), Q.astype(np.float64))
    for i in range(lanes):
        for c in range(m):
            seg = dots[i, c * C:min(n, (c + 1) * C)]
            assert seg.max() <= Uf[i, c] and seg.min() >= Lf[i, c]


@pytest.mark.parametrize("kind", ["ties", "neartie", "planted"])
def test_select3_many_lanes_matches_oracle(ops, kind):
    """The many-lane selector (CTA per lane, used from 37 lanes up; the decode step runs it at
    256 lanes) at 64K with exact and near ties: sets bit-exact, ties to the lowest index.
    Reference: the canonical K4 scores (bit-exact vs the oracle, test_token_scores_bitexact)
    ordered by (score desc, index asc); three lanes re-checked against the C oracle itself."""
    lanes, n, d, C = 38, 65536, 128, 64
    k = math.ceil(0.1 * n)
    K, V, Q = _lane_data(kind, lanes, n, d, seed=77)
    kt = torch.from_numpy(K).bfloat16().cuda()
    del K
    vt = torch.from_numpy(V).bfloat16().cuda()
    del V
    qt = torch.from_numpy(Q).cuda()
    amax, amin = ops.abstract_build(kt, n, C)
    ws = ops.LayerWorkspace(lanes, n, ops.n_grid_leaves(n, C), d, kt.device)
    out = {"sel_tok": torch.empty((lanes, k), dtype=torch.int32, device="cuda"),
           "sel_score": torch.empty((lanes, k), dtype=torch.float64, device="cuda"),
           "n_sel": torch.empty(lanes, dtype=torch.int32, device="cuda"),
           "out": torch.empty((lanes, d), dtype=torch.float32, device="cuda")}
    ops.select_attend(qt, kt, vt, amax, amin, n, k, C, ws, out)
    s = ops.token_scores(qt.double(), kt, n)
    ref = torch.sort(torch.sort(-s, dim=1, stable=True).indices[:, :k], dim=1).values
    got = out["sel_tok"].long()
    bad = (got != ref).any(1).nonzero().flatten().tolist()
    assert not bad, (kind, bad[:5])
    Kh = kt.double().cpu().numpy()
    for i in (0, lanes // 2, lanes - 1):
        assert np.array_equal(got[i].cpu().numpy(), O.topk(O.dots(Q[i], Kh[i]), k)), i


def test_k2_abstract_merge_segments_and_coarsening():
    """K2 (kvt_abstract_merge): explicit segments equal numpy's max / min of the rows (f64,
    bit-exact); uniform coarsening of bf16 outward-rounded C = 8 abstracts equals building the
    C = 64 grid from the keys directly (rounding up commutes with max), tail chunk included."""
    import torch
    from paper_2506_20187_b200 import ops
    g = torch.Generator().manual_seed(5)
    rows = torch.randn((37, 128), generator=g, dtype=torch.float64)
    rows2 = rows - torch.rand((37, 128), generator=g, dtype=torch.float64)
    segs = [(0, 1), (1, 9), (9, 10), (10, 37)]
    mx, mn = ops.abstract_merge(rows.cuda(), rows2.cuda(), seg_begin=[a for a, _ in segs], seg_end=[b for _, b in segs])
    for i, (a, b) in enumerate(segs):
        assert torch.equal(mx[i].cpu(), rows[a:b].max(0).values)
        assert torch.equal(mn[i].cpu(), rows2[a:b].min(0).values)
    lanes, n, d = 3, 64 * 20 + 24, 128
    K = torch.randn((lanes, n, d), generator=g).to(torch.bfloat16).cuda()
    f8 = ops.abstract_build(K, n, 8, abs_dtype=torch.bfloat16)
    f64 = ops.abstract_build(K, n, 64, abs_dtype=torch.bfloat16)
    c = ops.abstract_merge(f8[0], f8[1], factor=8, m_in=ops.n_grid_leaves(n, 8))
    assert torch.equal(c[0], f64[0]) and torch.equal(c[1], f64[1])


def test_live_chunks_counts_distinct_chunks_of_the_selection():
    """kvt_live_chunks (the skew input of SparseDecoder.adapt_chunking): chunks of size 2^lg
    holding a selected token, from the runs, equal numpy's count of distinct t >> lg."""
    import torch
    from paper_2506_20187_b200 import _lib as L, ops
    rng = np.random.default_rng(9)
    lanes, n = 5, 70000
    sels = [np.sort(rng.choice(n, size=s, replace=False)) for s in (1, 7, 700, 7000, 35000)]
    kmax = max(len(x) for x in sels)
    st = torch.zeros((lanes, kmax), dtype=torch.int32)
    for i, x in enumerate(sels):
        st[i, :len(x)] = torch.from_numpy(x.astype(np.int32))
    ns = torch.tensor([len(x) for x in sels], dtype=torch.int32)
    r = ops.runs_scan(st.cuda(), ns.cuda(), n)
    out = torch.empty((lanes, 4), dtype=torch.int64, device="cuda")
    L.check(L.kvt_live_chunks(r["run_start"].data_ptr(), r["run_len"].data_ptr(), r["n_runs"].data_ptr(),
                              r["run_start"].stride(0), lanes, 3, 4, out.data_ptr(), ops._stream()), "live_chunks")
    got = out.cpu().numpy()
    for i, x in enumerate(sels):
        for j, lg in enumerate(range(3, 7)):
            assert got[i, j] == len(np.unique(x >> lg)), (i, lg)


def test_select_plan_staged_and_global_paths_agree(ops):
    """The plan stages U and A in shared memory next to the keys when a lane's leaves fit
    (<= 4096); the same partition with a wider leaf stride takes the global-memory path.  Items,
    counts, evaluations and the error record must be identical."""
    rng = np.random.default_rng(5)
    lanes, n = 4, 20000
    starts = []
    for _ in range(lanes):
        cuts = np.sort(rng.choice(np.arange(1, n), size=1500, replace=False))
        starts.append(np.concatenate([[0], cuts]).astype(np.int32))
    nl = max(len(s) for s in starts)
    U = rng.normal(size=(lanes, nl))
    Lo = U - np.abs(rng.normal(size=(lanes, nl)))
    A = np.abs(rng.normal(size=(lanes, nl))) + 1.0
    nleaves = torch.tensor([len(s) for s in starts], dtype=torch.int32, device="cuda")
    outs = []
    for stride in (nl, 5000):  # <= 4096 leaves per lane: staged; 5000: global loads
        ls = torch.zeros((lanes, stride), dtype=torch.int32)
        pad = lambda x: torch.from_numpy(np.pad(x, ((0, 0), (0, stride - nl)))).cuda()
        for i, s in enumerate(starts):
            ls[i, :len(s)] = torch.from_numpy(s)
        plan = ops.select_plan(pad(U), pad(Lo), n, n // 10, 0, leaf_start=ls.cuda(), n_leaves=nleaves,
                               A=pad(A), d=128)
        torch.cuda.synchronize()
        outs.append(plan)
    a, b = outs
    for key in ("n_items", "n_cand", "evals", "err"):
        assert torch.equal(a[key], b[key]), key
    for i in range(lanes):
        ni = int(a["n_items"][i])
        assert torch.equal(a["items"][i, :ni], b["items"][i, :ni]), i
