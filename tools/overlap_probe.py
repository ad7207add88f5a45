"""Would two lane halves on two streams overlap one half's latency-bound kernels (plan, select)
with the other's streaming kernels?  Config 3 split into two B = 4 decoders (lanes 0-127 and
128-255, each its own CUDA graph); the two graphs replayed back to back on one stream vs on two
streams.  Development probe: python tools/overlap_probe.py [--steps N]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_20187_b200 import ops  # noqa: E402
from paper_2506_20187_b200.decode import SparseDecoder  # noqa: E402

steps = 20
args = bench.parse(["--batch", "8"])
dev = torch.device("cuda:0")
torch.cuda.set_device(0)
halves = []
for r in range(2):
    sp = bench.shard_plan(8, bench.N_HEADS, args.kv_heads, 2, r, "strong")
    dec, params, _ = bench.build_decoder(args, sp, dev, torch, ops, SparseDecoder)
    Q = torch.from_numpy(bench.make_queries(args, sp, params, 4)).to(dev)
    st = torch.cuda.Stream(device=dev)
    qs = torch.empty_like(Q[0]); out = torch.empty(qs.shape, device=dev, dtype=torch.float32)
    with torch.cuda.stream(st):
        for s in range(3):
            qs.copy_(Q[s]); dec.step(qs, out)
        st.synchronize()
        dec.adapt_bound_granularity()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            dec.step(qs, out)
        g.replay()
        st.synchronize()
    halves.append((dec, g, st))
    print(f"half {r}: lanes {dec.lanes}", flush=True)

def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
    for _ in range(steps):
        fn()
    for _, _, st in halves:
        torch.cuda.current_stream().wait_stream(st)
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps

s0 = halves[0][2]
def seq():
    with torch.cuda.stream(s0):
        halves[0][1].replay(); halves[1][1].replay()
def one():
    with torch.cuda.stream(s0):
        halves[0][1].replay()
def conc():
    cur = torch.cuda.current_stream()
    for _, g, st in halves:
        st.wait_stream(cur)
        with torch.cuda.stream(st):
            g.replay()
for _ in range(2):
    print(f"one half alone {timed(one):.3f} ms/step; halves back to back {timed(seq):.3f}; "
          f"halves on two streams {timed(conc):.3f}", flush=True)
