"""Per-kernel microbenchmarks on B200 (CUDA events on the launching stream, inputs >> L2).

    python tools/microbench.py quant [--lanes 256 --n 65536]

Prints one JSON line per kernel: device ms per launch and algorithmic GB/s
against the measured HBM peak in MEASURED_PEAKS.json.  Development tool; bench.py is the
contract.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2506_20187_b200 import ops, tier  # noqa: E402


def peak():
    p = ROOT / "MEASURED_PEAKS.json"
    return float(json.loads(p.read_text())["hbm_gbs"]) if p.exists() else 6650.0


def timeit(fn, reps=10, warm=2):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def report(name, ms, nbytes, **kw):
    gbs = nbytes / (ms / 1e3) / 1e9
    print(json.dumps({"kernel": name, "ms": round(ms, 4), "algo_bytes": nbytes, "gbs": round(gbs, 1),
                      "frac": round(gbs / peak(), 3), **kw}), flush=True)


def quant(a):
    d = 128
    for dt in (torch.bfloat16, torch.float32):
        lanes = a.lanes if dt == torch.bfloat16 else a.lanes // 2
        x = torch.randn((lanes, a.n, d), device="cuda", dtype=dt)
        dst = ops.I4KV.empty(lanes, a.n, d, x.device)
        ms = timeit(lambda: ops.kv_quant(x, dst, 0, a.n))
        nb = lanes * a.n * (d * x.element_size() + ops.row_bytes_i4(d))
        report(f"kv_quant[{dt}]", ms, nb, lanes=lanes, n=a.n)
        del x, dst
        torch.cuda.empty_cache()
    # decode-time append: one token per lane
    x = torch.randn((a.lanes, 1, d), device="cuda", dtype=torch.bfloat16)
    dst = ops.I4KV.empty(a.lanes, 1, d, x.device)
    ms = timeit(lambda: ops.kv_quant(x, dst, 0, 1), reps=100)
    report("kv_quant[append 1 token]", ms, a.lanes * (d * 2 + ops.row_bytes_i4(d)), lanes=a.lanes)


def dequant(a):
    d = 128
    src = ops.I4KV.empty(a.lanes, a.n, d, "cuda")
    src.data.random_(0, 255)
    src.data.view(torch.float16)[..., d // 4:] = 0.01  # finite (scale, min) pairs
    out = torch.empty((a.lanes, a.n, d), dtype=torch.bfloat16, device="cuda")
    ms = timeit(lambda: tier.kv_dequant(src, out))
    report("kv_dequant[bf16]", ms, a.lanes * a.n * (d * 2 + ops.row_bytes_i4(d)), lanes=a.lanes, n=a.n)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("which", nargs="+")
    p.add_argument("--lanes", type=int, default=256)
    p.add_argument("--n", type=int, default=65536)
    a = p.parse_args()
    for w in a.which:
        globals()[w](a)



def _planted_sel(lanes, n, k, dev, seed=0):
    """Sorted selected sets like the planted workload: k tokens inside 3 hot regions (30% of n)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    hot = torch.cat([torch.arange(int(n * a), int(n * a) + n // 10) for a in (0.1, 0.45, 0.8)])
    sel = torch.stack([torch.sort(hot[torch.randperm(hot.numel(), generator=g)[:k]]).values for _ in range(lanes)])
    return sel.to(torch.int32).to(dev)


def attn(a):
    from paper_2506_20187_b200 import _lib as Lb
    d = 128
    for fmt in ("int4", "bf16"):
        lanes = a.lanes if fmt == "int4" else a.lanes // 2
        if fmt == "int4":
            V = ops.I4KV.empty(lanes, a.n, d, "cuda")
            V.data.random_(0, 255)
            V.data.view(torch.float16)[..., d // 4:] = 0.01
            rb = ops.row_bytes_i4(d)
        else:
            V = torch.randn((lanes, a.n, d), device="cuda", dtype=torch.bfloat16)
            rb = 2 * d
        for k in (a.n // 10, a.n // 2):
            st = _planted_sel(lanes, a.n, k, "cuda") if k < a.n // 2 else \
                torch.sort(torch.randperm(a.n, device="cuda")[:k]).values.to(torch.int32).expand(lanes, k).contiguous()
            ss = torch.randn((lanes, k), dtype=torch.float64, device="cuda")
            ns = torch.full((lanes,), k, dtype=torch.int32, device="cuda")
            res = {}
            for sp in [0, 2, 3, 4, 6, 7, 8, 10, 12, 16, 24, 32, 48, 64]:
                if sp and (k + sp - 1) // sp > 4096:
                    continue
                ms = timeit(lambda: ops.sparse_decode_attn(V, st, ss, ns, splits=sp), reps=20)
                res[sp] = round(ms * 1e3, 1)
            best = min((v, s) for s, v in res.items() if s)
            report(f"attn[{fmt}] k={k} best splits={best[1]}", best[0] / 1e3, lanes * k * (rb + 12), lanes=lanes,
                   us_by_splits=res)


if __name__ == "__main__":
    main()
