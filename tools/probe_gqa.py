"""Probe (not product code): GQA union path vs per-query-lane path at config-4 lane shape."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import workload as W
from paper_2506_20187_b200 import ops
from paper_2506_20187_b200.decode import SparseDecoder

B, H, Hkv, d, n = int(sys.argv[1]) if len(sys.argv) > 1 else 2, 32, 8, 128, 131072
g = H // Hkv
L = 3
dec = SparseDecoder(L, B, H, d, n, dtype=ops.I4, device="cuda", n_kv_heads=Hkv)
kv_ids = np.arange(B * Hkv)
kb = torch.empty((B * Hkv, n, d), dtype=torch.bfloat16, device="cuda")
vb = torch.empty_like(kb)
gen = W.gen_args(None, d, "planted")
params = []
for l in range(L):
    p = W.lane_params(0, l, kv_ids, n, d, "planted")
    params.append(p)
    ops.synth_layer(kb, vb, p, n, gen)
    dec.load_layer(l, kb, vb)
dec.set_length(n)
l = 2
q = torch.from_numpy(W.queries(0, 1, l, np.arange(B * H), g, params[l]["u"], 0, d, "planted")[0]).cuda()
k = dec.k_for(l)
C, amax, amin = dec.grid(l)

def ev():
    return torch.cuda.Event(enable_timing=True)

def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record(); e1.synchronize()
    return r, e0.elapsed_time(e1) / reps * 1e3

with ops.kv_group(g):
    (U, Lo, A), tb = timed(lambda: ops.chunk_bounds_fast(q, amax, amin, n, C, dec.absmag[l]))
    print("bounds us", round(tb, 1))
    for grp in (1, g):
        plan, tp = timed(lambda: ops.select_plan(U, Lo, n, k, C, A=A, d=d, group=grp))
        with ops.cand_group(grp):
            def sc():
                plan["err"][:, 3] = 0
                return ops.cand_score_i4mma(q, dec.K[l], plan, n)
            (cs, ct), ts = timed(sc)
            (st, ss, ns, runs), tsel = timed(lambda: ops.topk_select_band(cs, ct, plan, k, q, dec.K[l]))
        torch.cuda.synchronize()
        nc = plan["n_cand"].cpu().numpy()
        err = plan["err"].cpu().numpy()
        print(f"grp {grp}: plan {tp:.1f} us score {ts:.1f} us select {tsel:.1f} us  n_cand mean {nc.mean():.0f} "
              f"min {nc.min()} max {nc.max()}  E(+3) mean {err[:,3].mean():.3e} max {err[:,3].max():.3e}  "
              f"E(+0) {err[:,0].mean():.3e} tau {err[:4,1]} umax {err[:4,2]}")
        sel = st[:, :k].cpu().numpy()
        if grp == 1:
            sel1 = np.sort(sel, axis=1)
        else:
            print("sets equal:", np.array_equal(np.sort(sel, axis=1), sel1))
