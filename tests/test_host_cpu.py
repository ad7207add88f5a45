"""CPU-only checks: the C ABI library loads and exports every declared symbol; host-side
logic (chunk plan, cost model, grid metrics) equals the reference's frozen values."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from tests import golden_io as G

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "kvtier_b200.h").read_text()
    return re.findall(r"KVT_API\s+[\w\s\*]+?\b(kvt_\w+)\s*\(", text)


def test_library_exports_every_header_symbol():
    from paper_2506_20187_b200 import _lib
    names = declared_symbols()
    assert len(names) >= 15
    for nm in names:
        assert hasattr(_lib.handle(), nm), nm
    assert set(names) == set(_lib.EXPORTED)
    assert _lib.kvt_version() == 100
    assert _lib.kvt_status_string(-2).decode() == "k out of range"


def test_abi_rejects_bad_arguments_without_gpu():
    """Argument validation happens before any CUDA call, so it is testable on CPU."""
    from paper_2506_20187_b200 import _lib as L
    assert L.kvt_select_plan(1, 10, 4, None, None, 0, 1, 1, 3, 11, 1, 1, 1, 1, None, None, None) == L.ERR_K
    assert L.kvt_chunk_bounds(None, 0, 1, 4, 10, 4, None, None, 0, None, None, 0, 0, None, None, None, 0, 0, None) == L.ERR_ARG
    assert L.kvt_topk_select(1, 1, 1, 1, 1, -1, 1, 1, 1, 1, None) == L.ERR_K
    with pytest.raises(ValueError):
        L.check(L.ERR_K, "x")
    with pytest.raises(RuntimeError):
        L.check(L.ERR_COLD, "x")


def test_chunk_plan_matches_reference_values():
    from paper_2506_20187_b200 import chunk_tree as ct
    s = G.load_json("scalars.json")
    for m, n, rho, v in s["chunk_cost"]:
        assert ct.chunk_cost(m, n, rho) == pytest.approx(v, abs=1e-12)
    for n, rho, lo, hi, v in s["plan_chunk_count"]:
        assert ct.plan_chunk_count(n, rho, min_chunk_size=lo, max_chunk_size=hi) == v
    for rho, layer, step, nst, nctx, v in s["chunk_size_for"]:
        cfg = ct.ChunkPlanConfig(rho=None if rho is None else tuple(rho))
        assert cfg.chunk_size_for(layer, step, nst, nctx) == v
    for n, v in s["next_pow2"]:
        assert ct.next_pow2(n) == v
    with pytest.raises(ValueError):
        ct.chunk_cost(16, 1024, 1.0)
    with pytest.raises(ValueError):
        ct.plan_chunk_count(1024, 1.5)
    with pytest.raises(ValueError):
        ct.ChunkPlanConfig(default_chunk_size=48)
    with pytest.raises(ValueError):
        ct.ChunkPlanConfig(early_chunk_size=128, default_chunk_size=64)


def test_grid_metrics_match_reference_values():
    from paper_2506_20187_b200.engine import desert_rate_on_grid
    for sel, n, g, v in G.load_json("scalars.json")["desert_rate_on_grid"]:
        assert desert_rate_on_grid(set(sel), n, g) == v


def test_shard_blocks_cover_disjointly():
    from paper_2506_20187_b200.shard import lane_block, token_block
    for n in (1, 7, 32, 256, 1000):
        for w in (1, 2, 4, 8):
            blocks = [lane_block(n, w, r) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            toks = [token_block(n * 64 + 3, w, r) for r in range(w)]
            assert toks[0][0] == 0 and toks[-1][1] == n * 64 + 3
            assert all(a[1] == b[0] and (a[1] % 64 == 0 or a[1] == n * 64 + 3) for a, b in zip(toks, toks[1:]))


def test_int4_codec_oracle_matches_numpy_definition():
    """The C oracle's INT4 codec equals an independent numpy statement of DESIGN.md sec. 2."""
    import numpy as np
    from oracle import oracle as O
    rng = np.random.default_rng(0)
    x = (rng.normal(size=(500, 128)) * rng.choice([0.001, 1.0, 100.0], size=(500, 1))).astype(np.float32)
    x[3] = 1.5
    rec = O.i4_quant(x)
    g = x.reshape(500, 4, 32)
    lo, hi = g.min(2), g.max(2)

    def h_dir(v, up):  # fp16 rounded toward +inf (up) or -inf, from float32 v
        h = v.astype(np.float16)
        bad = (h.astype(np.float32) < v) if up else (h.astype(np.float32) > v)
        return np.where(bad, np.nextafter(h, np.float16(np.inf if up else -np.inf)), h)

    def f32_up(exact64):  # fl_ru of a value known exactly in f64
        r = exact64.astype(np.float32)
        return np.where(r.astype(np.float64) < exact64, np.nextafter(r, np.float32(np.inf)), r)

    mh = h_dir(lo, False)
    m = mh.astype(np.float32)
    diff = f32_up(hi.astype(np.float64) - m.astype(np.float64))  # exact in f64 for these ranges
    sh = h_dir(f32_up(diff.astype(np.float64) * np.float64(np.float32(0.0666666701436042785645))), True)
    s = sh.astype(np.float32)
    assert np.all(15 * s.astype(np.float64) >= hi.astype(np.float64) - m) and np.all(m <= lo)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = (np.float32(1) / s).astype(np.float32)
        # fl32(x - m) * inv is exact in f64 (24 x 24 bits); np.rint = RN_int, ties to even
        qv = (g - m[..., None]).astype(np.float32).astype(np.float64) * inv[..., None].astype(np.float64)
    assert np.all(np.where(s[..., None] == 0, 0, qv) <= 15.5)
    c = np.where(s[..., None] == 0, 0, np.rint(qv)).astype(np.uint8).reshape(500, 128)
    assert np.array_equal(rec[:, :64], (c[:, 0::2] | (c[:, 1::2] << 4)).astype(np.uint8))
    assert np.array_equal(rec[:, 64:], np.stack([sh, mh], -1).reshape(500, 8).view(np.uint8))
    deq = O.i4_dequant(rec, 128)
    ref = (c.astype(np.float32).reshape(500, 4, 32) * s[..., None] + m[..., None]).reshape(500, 128)
    assert np.abs(deq - ref).max() <= 1e-6 * np.abs(ref).max()
