import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2506_20187_b200 import ops
from paper_2506_20187_b200.decode import SparseDecoder
B, H, d, n, L = 2, 8, 128, 4096, 3
rng = np.random.default_rng(11)
K = torch.from_numpy(rng.normal(size=(B * H, n, d)).astype(np.float32)).to(torch.bfloat16).cuda()
Q = torch.from_numpy(rng.normal(size=(L, B * H, d)).astype(np.float32)).cuda()
dec = SparseDecoder(L, B, H, d, n, dtype=torch.bfloat16, device="cuda")
for l in range(L): dec.load_layer(l, K, K)
dec.set_length(n)
out = dec.step(Q); torch.cuda.synchronize()
per = [dec.layer(l, Q[l])["out"].clone() for l in range(L)]; torch.cuda.synchronize()
for l in range(L):
    print("layer", l, "step vs layer() max|diff|", float((out[l] - per[l]).abs().max()))
# layer 2 alone twice
a = dec.layer(2, Q[2])["out"].clone(); b = dec.layer(2, Q[2])["out"].clone(); torch.cuda.synchronize()
print("layer2 repeat diff", float((a - b).abs().max()))
# direct attention on layer-2 selection
bufs = dec._buffers()[2]
o2 = ops.sparse_decode_attn(dec.V[2], bufs["sel_tok"], bufs["sel_score"], bufs["n_sel"]); torch.cuda.synchronize()
print("layer2 vs standalone attn", float((o2 - a).abs().max()), "splits-1", float((ops.sparse_decode_attn(dec.V[2], bufs["sel_tok"], bufs["sel_score"], bufs["n_sel"], splits=1) - o2).abs().max()))
