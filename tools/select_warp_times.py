import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2506_20187_b200 import _lib as L, ops
from paper_2506_20187_b200.decode import SparseDecoder
args = bench.parse([]); dev = torch.device("cuda:0")
sp = bench.shard_plan(args.batch, bench.N_HEADS, args.kv_heads, 1, 0, args.scaling)
dec, params, _ = bench.build_decoder(args, sp, dev, torch, ops, SparseDecoder)
Q = torch.from_numpy(bench.make_queries(args, sp, params, 4)).to(dev)
for s in range(3): dec.step(Q[s])
dec.adapt_bound_granularity(); dec.step(Q[3]); torch.cuda.synchronize()
buf = torch.zeros(dec.lanes * 8 + 64 * 16 + 64, dtype=torch.int64, device=dev)
L.check(L.kvt_debug_select_phases(buf.data_ptr()), "p"); dec.layer(2, Q[3][2]); torch.cuda.synchronize(); L.kvt_debug_select_phases(None)
b = buf.cpu().numpy()
ph = b[:dec.lanes * 8].reshape(dec.lanes, 8).astype(np.float64)
wt = b[dec.lanes * 8: dec.lanes * 8 + 64 * 16].reshape(64, 16).astype(np.float64)
for c in range(0, 64, 9):
    t5 = ph[c, 5]
    print("cta", c, "compaction per-warp end (us after phase-5 start):", np.round((wt[c] - t5) / 1e3, 1), "phase6", round((ph[c, 6] - t5) / 1e3, 1))
