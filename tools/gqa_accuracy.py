import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2506_20187_b200 import ops
from oracle import oracle as O
O.build()
for (n, k, spread, seed, n_kv) in [(9000, 2200, 30.0, 1, 2), (131072, 13107, 0.3, 3, 2), (131072, 13107, 0.3, 3, 40), (131072, 13107, 30.0, 6, 40), (65536, 6554, 0.3, 7, 96)]:
    g, d = 4, 128
    rng = np.random.default_rng(seed)
    V = torch.from_numpy(rng.normal(size=(n_kv, n, d)).astype(np.float32)).cuda()
    vi = ops.I4KV.empty(n_kv, n, d, "cuda"); ops.kv_quant(V, vi)
    Vd = np.stack([O.i4_dequant(vi.data[j].cpu().numpy(), d) for j in range(n_kv)]).astype(np.float64)
    sel = np.zeros((n_kv * g, k), np.int32)
    for j in range(n_kv):
        base = np.sort(rng.choice(n, size=k, replace=False))
        for h in range(g): sel[j * g + h] = base
    score = (rng.normal(size=(n_kv * g, k)) * spread + 20).astype(np.float64)
    st, ss = torch.from_numpy(sel).cuda(), torch.from_numpy(score).cuda()
    ns = torch.full((n_kv * g,), k, dtype=torch.int32, device="cuda")
    out = ops.sparse_decode_attn_gqa(vi, st, ss, ns, g, n).cpu().numpy()
    with ops.kv_group(g):
        out2 = ops.sparse_decode_attn(vi, st, ss, ns).cpu().numpy()
    scale = 1.0 / np.sqrt(d)
    e1 = e2 = 0
    for i in range(n_kv * g):
        w = np.exp((score[i] - score[i].max()) * scale)
        ref = (w[:, None] * Vd[i // g][sel[i]]).sum(0) / w.sum()
        e1 = max(e1, np.linalg.norm(out[i] - ref) / np.linalg.norm(ref))
        e2 = max(e2, np.linalg.norm(out2[i] - ref) / np.linalg.norm(ref))
    print(n, k, spread, n_kv, "union", e1, "per-lane", e2, flush=True)
