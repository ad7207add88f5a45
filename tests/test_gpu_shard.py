"""Config 5 (sequence sharding) on the GPU kernels: every rank owns a token
shard of every lane, selects exactly with the global threshold exchange and contributes a
partial softmax state merged by kvt_lse_merge.  Ranks are emulated by threads on one GPU
with barrier-based all-reduce / all-gather (the torch.distributed wrappers are exercised
under gloo in tests/test_dist_gloo.py).  The union of the shards' selections must be the
oracle's global top-k (bit-exact, ties to the lowest token) and the merged attention must
match attention_output over it (engine.py:145-154) within the bf16 bar."""

from __future__ import annotations

import math
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from oracle import synth  # noqa: E402


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_20187_b200 import ops as _ops
    return _ops


class _Comm:
    """In-process collectives for `world` threads (sum / stack in rank order)."""

    def __init__(self, world):
        self.world = world
        self.slots = [None] * world
        self.bar = threading.Barrier(world)

    def _exchange(self, rank, t, combine):
        torch.cuda.synchronize()
        self.slots[rank] = t.clone()
        self.bar.wait()
        res = combine([s for s in self.slots])
        self.bar.wait()
        return res

    def fns(self, rank):
        return (lambda t: self._exchange(rank, t, lambda xs: torch.stack(xs).sum(0)),
                lambda t: self._exchange(rank, t, lambda xs: torch.stack(xs)))


def _data(kind, lanes, n, d, seed):
    rng = np.random.default_rng(seed)
    if kind == "planted":
        K = np.empty((lanes, n, d), np.float32)
        V = np.empty_like(K)
        Q = np.empty((lanes, d), np.float32)
        for i in range(lanes):
            k, q, v, _ = synth.lane(synth.Profile(0.7, 3, 1.0, seed), 0, i, n, d, 1)
            K[i], V[i], Q[i] = k, v, q[0]
        return K, V, Q
    K = rng.normal(size=(lanes, n, d)).astype(np.float32)
    V = rng.normal(size=(lanes, n, d)).astype(np.float32)
    Q = rng.normal(size=(lanes, d)).astype(np.float32)
    if kind == "ties":  # identical key rows across the shard boundary: exact score ties
        K[:, ::7] = K[:, :1]
        Q = np.abs(Q)
    return K, V, Q


@pytest.mark.parametrize("kind", ["random", "planted", "ties"])
@pytest.mark.parametrize("world,n,rate", [(2, 4096, 0.1), (4, 4096, 0.5), (3, 1000, 0.1)])
def test_seq_shard_matches_unsharded(ops, kind, world, n, rate):
    from paper_2506_20187_b200.shard import seq_shard_select_attend, token_block
    lanes, d, C = 4, 128, 64
    k = math.ceil(rate * n)
    K, V, Q = _data(kind, lanes, n, d, seed=world * 10 + n)
    kt = torch.from_numpy(K).to(torch.bfloat16).cuda()
    vt = torch.from_numpy(V).to(torch.bfloat16).cuda()
    qt = torch.from_numpy(Q).cuda()
    comm = _Comm(world)
    results = [None] * world
    errors = []

    def run(rank):
        try:
            torch.cuda.set_device(0)
            t0, t1 = token_block(n, world, rank)
            ar, ag = comm.fns(rank)
            out, sel = seq_shard_select_attend(qt, kt[:, t0:t1].contiguous(), vt[:, t0:t1].contiguous(), t1 - t0,
                                               C, k, rank, ar, ag)
            torch.cuda.synchronize()
            results[rank] = (out.cpu().numpy(), [s.cpu().numpy().astype(np.int64) + t0 for s in sel])
        except BaseException as e:  # surface thread failures in the test
            errors.append(e)
            comm.bar.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    Kh, Vh = kt.double().cpu().numpy(), vt.double().cpu().numpy()
    for i in range(lanes):
        union = np.sort(np.concatenate([results[r][1][i] for r in range(world)]))
        ref = O.topk(O.dots(Q[i], Kh[i]), k)
        assert np.array_equal(union, ref), (kind, i)
        att = O.attention(Q[i], Kh[i], Vh[i], ref)
        for r in range(world):  # every rank ends with the same merged output
            err = np.linalg.norm(results[r][0][i] - att) / np.linalg.norm(att)
            assert err <= 1e-2, (kind, i, r, err)


def test_lse_merge_kernel_matches_torch(ops):
    """kvt_lse_merge == the log-sum-exp combine of normalised partials (f64)."""
    rng = np.random.default_rng(5)
    P, lanes, d = 5, 7, 64
    m = rng.normal(size=(P, lanes)) * 20
    l = rng.uniform(0.5, 3.0, size=(P, lanes))
    l[1, 2] = 0.0  # an empty shard
    o = rng.normal(size=(P, lanes, d))
    parts = torch.from_numpy(np.concatenate([m[..., None], l[..., None], o], -1)).cuda()
    scale = 0.125
    out, out64 = ops.lse_merge(parts, scale, want_f64=True)
    M = np.where(l > 0, m, -np.inf).max(0)
    w = np.where(l > 0, np.exp((m - M) * scale) * l, 0.0)
    ref = (w[..., None] * o).sum(0) / w.sum(0)[..., None]
    assert np.allclose(out64.cpu().numpy(), ref, rtol=1e-12, atol=1e-12)


def test_nccl_allgather_merge_single_rank():
    """kvt_lse_allgather_merge (NCCL bound at run time) on a one-rank communicator: the
    gathered part merges back to the rank's own output, and the merge kernel equals the torch
    log-sum-exp formula on a multi-part input."""
    import torch
    from paper_2506_20187_b200 import ops
    from paper_2506_20187_b200.shard import NcclLseMerge, lse_merge
    g = torch.Generator().manual_seed(4)
    n, d = 37, 128
    o = torch.randn((n, d), generator=g, dtype=torch.float64).cuda()
    m = torch.randn(n, generator=g, dtype=torch.float64).cuda()
    l = torch.rand(n, generator=g, dtype=torch.float64).cuda() + 0.5
    nm = NcclLseMerge(0, 1)
    try:
        out = nm.merge(m, l, o, 0.1)
        torch.cuda.synchronize()
        assert torch.allclose(out, o, rtol=1e-12, atol=1e-12)
    finally:
        nm.close()
    P = 3
    parts = torch.randn((P, n, d + 2), generator=g, dtype=torch.float64).cuda()
    parts[:, :, 1] = parts[:, :, 1].abs() + 0.1
    got = ops.lse_merge(parts, 0.1)
    # torch restatement: o_p normalised -> un-normalised sums l_p o_p at scale-adjusted maxima
    mm = parts[:, :, 0] * 0.1
    ref = lse_merge(mm, parts[:, :, 1], parts[:, :, 2:] * parts[:, :, 1:2])
    assert torch.allclose(got.double(), ref, rtol=1e-5, atol=1e-6)
