"""Band statistics of the exact top-k select (select3): per layer, the number of candidates
whose f32 estimate lies within 2E of the k-th estimate T (re-scored canonically in f64), for
the bench workload.  Development tool.   python tools/band_stats.py [--dtype int4] [--layers 4]"""
import argparse, math, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch
import bench
from paper_2506_20187_b200 import ops
from paper_2506_20187_b200.decode import SparseDecoder

p = argparse.ArgumentParser()
p.add_argument("--dtype", default="int4")
p.add_argument("--batch", type=int, default=2)
p.add_argument("--ctx", type=int, default=65536)
p.add_argument("--layers", type=int, default=3)
p.add_argument("--data", default="planted")
a = p.parse_args()
dev = torch.device("cuda")
dt = {"bf16": torch.bfloat16, "int4": ops.I4}[a.dtype]
L = a.layers
dec = SparseDecoder(L, a.batch, 32, 128, a.ctx, dtype=dt, device=dev)
gen = torch.Generator(device=dev); gen.manual_seed(0)
rng = np.random.default_rng(0)
u = torch.empty((L, dec.lanes, 128), device=dev)
kb = torch.empty((dec.lanes, a.ctx, 128), dtype=torch.bfloat16, device=dev); vb = torch.empty_like(kb)
for l in range(L):
    bench.fill_layer(torch, kb, vb, a.ctx, 128, a.data, rng, gen, u[l])
    if a.dtype == "int4":
        dec.load_layer(l, kb, vb)
    else:
        dec.K[l].copy_(kb); dec.V[l].copy_(vb)
dec.set_length(a.ctx)
Q = bench.make_queries(torch, u, 1, a.data, gen)[0]
for l in range(L):
    C, n, k = dec.C[l], dec.n, dec.k_for(l)
    U, Lo, A = ops.chunk_bounds_fast(Q[l], dec.amax[l], dec.amin[l], n, C, dec.absmag[l])
    plan = ops.select_plan(U, Lo, n, k, C, A=A, d=128)
    if a.dtype == "int4":
        cs, ct = ops.cand_score_i4mma(Q[l], dec.K[l], plan, n)
    else:
        cs, ct = ops.cand_score_f32(Q[l], dec.K[l], plan, n)
    err = plan["err"].cpu().numpy(); nc = plan["n_cand"].cpu().numpy()
    bands, widths = [], []
    for i in range(dec.lanes):
        s = cs[i, :nc[i]].double().cpu().numpy()
        E = err[i, 3] if err[i, 3] > 0 else err[i, 0]
        T = np.sort(s)[::-1][k - 1]
        bands.append(int(np.sum(np.abs(s - T) <= 2 * E)))
        widths.append(E / max(abs(T), 1e-30))
    print(f"layer {l}: C={C} k={k} n_cand mean {nc.mean():.0f}  band mean {np.mean(bands):.1f} max {max(bands)}  E/|T| {np.median(widths):.2e}")
