"""Phase timing of the K5 selector (select3.cu s3_mark points) on the bench's config-3
workload: builds the decoder exactly as bench.py does, runs warm-up steps, then re-runs the
chosen layers with the phase buffer set and prints per-phase CTA-mean durations (us) and the
launch span.  Development tool.   python tools/select_phases.py [bench args] --layers-probe 0,2"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_20187_b200 import _lib as L, ops  # noqa: E402
from paper_2506_20187_b200.decode import SparseDecoder  # noqa: E402

argv = sys.argv[1:]
NEXTQ = '--next-query' in argv
if NEXTQ:
    argv.remove('--next-query')
probe = [0, 2]
if "--layers-probe" in argv:
    i = argv.index("--layers-probe")
    probe = [int(x) for x in argv[i + 1].split(",")]
    del argv[i:i + 2]
args = bench.parse(argv)
dev = torch.device("cuda:0")
torch.cuda.set_device(0)
sp = bench.shard_plan(args.batch, bench.N_HEADS, args.kv_heads, 1, 0, args.scaling)
dec, params, _ = bench.build_decoder(args, sp, dev, torch, ops, SparseDecoder)
Q = torch.from_numpy(bench.make_queries(args, sp, params, 5)).to(dev)
for s in range(3):
    dec.step(Q[s])
dec.adapt_bound_granularity()
dec.step(Q[3])
torch.cuda.synchronize()
buf = torch.zeros((dec.lanes, 8), dtype=torch.int64, device=dev)
names = ["hist", "find_bin", "merged_pass", "list+band_sel", "band_rescore", "compaction", "runs"]
for l in probe:
    buf.zero_()
    L.check(L.kvt_debug_select_phases(buf.data_ptr()), "phases")
    dec.layer(l, Q[4 if '--next-query' in sys.argv[0:0] or NEXTQ else 3][l])
    torch.cuda.synchronize()
    L.check(L.kvt_debug_select_phases(None), "phases")
    t = buf.cpu().numpy().astype(np.float64)
    ok = t[:, 0] > 0
    t = t[ok]
    print(f"  hist ran in {(t[:, 1] > 0).sum()} of {len(t)} CTAs (the rest took the hinted bucket)")
    t0 = t[:, 0].min()
    print(f"layer {l}: CTAs {ok.sum()}  span {(t[:, 7].max() - t0) / 1e3:.1f} us  start spread {(t[:, 0].max() - t0) / 1e3:.1f} us")
    for p in range(1, 8):
        v = t[:, p] - t[:, p - 1]
        v = v[(t[:, p] > 0) & (t[:, p - 1] > 0)]
        if len(v):
            print(f"  {names[p - 1]:14s} mean {v.mean() / 1e3:7.2f} us  max {v.max() / 1e3:7.2f}")
    nc = dec._buffers()[l]
