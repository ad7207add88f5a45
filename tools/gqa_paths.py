"""Union vs per-lane GQA attention inside SparseDecoder (same selections): per-lane relative
difference of the two outputs, by layer.  Development check."""
import os, sys
import numpy as np, torch
sys.path.insert(0, '.')
import workload as W
from paper_2506_20187_b200 import ops
from paper_2506_20187_b200.decode import SparseDecoder
L_, n, d = 3, int(sys.argv[1]) if len(sys.argv) > 1 else 16384, 128
B, H, Hkv = (int(x) for x in (sys.argv[2:5] if len(sys.argv) > 4 else (2, 8, 2)))
dec = SparseDecoder(L_, B, H, d, n, dtype=ops.I4, n_kv_heads=Hkv)
kvl = B * Hkv
g = W.gen_args(None, d, "planted")
qs = []
for l in range(L_):
    p = W.lane_params(0, l, np.arange(kvl), n, d, "planted")
    K = torch.empty((kvl, n, d), dtype=torch.bfloat16, device="cuda"); V = torch.empty_like(K)
    ops.synth_layer(K, V, p, n, g)
    dec.load_layer(l, K, V)
    qs.append(W.queries(0, 1, l, np.arange(B * H), H // Hkv, p["u"], 0, d, "planted")[0])
dec.set_length(n)
q = torch.from_numpy(np.stack(qs)).cuda()
os.environ["KVT_GQA_UNION"] = "0"
o0 = dec.step(q).clone()
os.environ["KVT_GQA_UNION"] = "1"
o1 = dec.step(q).clone()
for l in range(L_):
    r = ((o1[l] - o0[l]).norm(dim=1) / o0[l].norm(dim=1)).cpu().numpy()
    print("layer", l, "k", dec.k_for(l), "max rel diff", r.max(), "argmax lane", r.argmax(), "median", np.median(r))
