"""Small end-to-end runs of every decode-path kernel, for compute-sanitizer (memcheck,
racecheck, synccheck):  compute-sanitizer --tool racecheck python tools/sanitize.py"""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2506_20187_b200 import ops, tier  # noqa: E402
from paper_2506_20187_b200.decode import SparseDecoder  # noqa: E402

torch.manual_seed(0)
for dt in (ops.I4, torch.bfloat16):
    dec = SparseDecoder(3, 1, 4, 128, 2048, dtype=dt, device="cuda")
    k = torch.randn((dec.lanes, 2048, 128), device="cuda", dtype=torch.bfloat16)
    v = torch.randn_like(k)
    for l in range(3):
        dec.load_layer(l, k, v)
    dec.set_length(2048)
    q = torch.randn((3, dec.lanes, 128), device="cuda")
    out = dec.step(q)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
# few lanes, long context
kt = torch.randn((2, 16384, 128), device="cuda", dtype=torch.bfloat16)
amax, amin = ops.abstract_build(kt, 16384, 64)
ws = ops.LayerWorkspace(2, 16384, ops.n_grid_leaves(16384, 64), 128, kt.device)
kk = math.ceil(0.1 * 16384)
o = {"sel_tok": torch.empty((2, kk), dtype=torch.int32, device="cuda"),
     "sel_score": torch.empty((2, kk), dtype=torch.float64, device="cuda"),
     "n_sel": torch.empty(2, dtype=torch.int32, device="cuda"),
     "run_start": torch.empty((2, kk), dtype=torch.int32, device="cuda"),
     "run_len": torch.empty((2, kk), dtype=torch.int32, device="cuda"),
     "n_runs": torch.empty(2, dtype=torch.int32, device="cuda"),
     "out": torch.empty((2, 128), dtype=torch.float32, device="cuda")}
ops.select_attend(torch.randn((2, 128), device="cuda"), kt, kt, amax, amin, 16384, kk, 64, ws, o)
torch.cuda.synchronize()
# many lanes (>= 37: the CTA-per-lane select3 path the decode step uses), random keys (every
# token a candidate) and all-equal keys (one tie bucket larger than the list: the fallback)
for dt in (ops.I4, torch.bfloat16):
    for kind in ("random", "ties"):
        dec = SparseDecoder(3, 10, 4, 128, 8192, dtype=dt, device="cuda")
        k = torch.randn((dec.lanes, 8192, 128), device="cuda", dtype=torch.bfloat16)
        if kind == "ties":
            k = torch.ones_like(k)
        v = torch.randn_like(k)
        for l in range(3):
            dec.load_layer(l, k, v)
        dec.set_length(8192)
        out = dec.step(torch.randn((3, dec.lanes, 128), device="cuda"))
        torch.cuda.synchronize()
        assert torch.isfinite(out).all()
# codec round trip + attention helpers
x = torch.randn((4, 777, 128), device="cuda", dtype=torch.bfloat16)
rec = ops.I4KV.empty(4, 777, 128, "cuda")
ops.kv_quant(x, rec)
y = torch.empty_like(x)
tier.kv_dequant(rec, y)
parts = torch.randn((3, 4, 130), device="cuda", dtype=torch.float64)
parts[:, :, 1] = parts[:, :, 1].abs()
ops.lse_merge(parts, 0.1)
torch.cuda.synchronize()
# round 2: GQA union attention (plan + pv), K2 merges, live chunks, the hot tier with evictions
from paper_2506_20187_b200 import _lib as L  # noqa: E402
from paper_2506_20187_b200.host_tier import TieredDecoder  # noqa: E402
dec = SparseDecoder(3, 2, 8, 128, 9000, dtype=ops.I4, device="cuda", n_kv_heads=2)
k = torch.randn((dec.kv_lanes, 9000, 128), device="cuda", dtype=torch.bfloat16)
v = torch.randn_like(k)
for l in range(3):
    dec.load_layer(l, k, v)
dec.set_length(9000)
out = dec.step(torch.randn((3, dec.lanes, 128), device="cuda"))
dec.adapt_chunking()
out = dec.step(torch.randn((3, dec.lanes, 128), device="cuda"))
torch.cuda.synchronize()
assert torch.isfinite(out).all()
ops.abstract_merge(dec.amax[0], dec.amin[0], seg_lane=[0, 1, 1], seg_begin=[0, 3, 9], seg_end=[5, 9, 10])
td = TieredDecoder(3, 1, 4, 128, 8192, 9000, crec=8, keep_raw=True, importance_rate=0.1, early_layer_rate=0.1)
k = torch.randn((4, 8192, 128), device="cuda", dtype=torch.bfloat16)
for l in range(3):
    td.load_layer(l, k, torch.randn_like(k))
td.set_length(8192)
td.set_theta([0.5, 0.0, 1.0])
for s in range(3):
    out = td.step(torch.randn((3, 4, 128), device="cuda"))
    torch.cuda.synchronize()
    td.ledger_rows()
assert torch.isfinite(out).all()
print("sanitize run ok")
