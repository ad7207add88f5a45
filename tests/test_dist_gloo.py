"""World-size-2 gloo runs of the multi-GPU host logic (CPU): batch x head sharding needs no
collective and reproduces the single-process result; the sequence-sharded LSE merge
(all-gather + log-sum-exp combine) equals softmax attention over the union."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _partial_state(q, K, V, idx):
    """(m, l, o) of softmax attention over rows idx -- what K7 emits per split."""
    if len(idx) == 0:
        return -np.inf, 0.0, np.zeros(K.shape[1])
    s = O.scores(q, K[idx])
    m = s.max()
    w = np.exp(s - m)
    return m, w.sum(), w @ V[idx]


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_20187_b200.shard import allgather_lse_merge, lane_block, max_over_ranks, token_block
    rng = np.random.default_rng(0)
    lanes, n, d, k = 6, 512, 16, 51
    K = rng.normal(size=(lanes, n, d))
    V = rng.normal(size=(lanes, n, d))
    Q = rng.normal(size=(lanes, d))
    # --- sequence sharding: global exact top-k, per-rank partial softmax, LSE merge ---
    t0, t1 = token_block(n, world, rank)
    ms, ls, os_ = [], [], []
    for i in range(lanes):
        sel = O.select(Q[i], K[i], k)             # global threshold (exact set)
        mine = sel[(sel >= t0) & (sel < t1)]      # this rank's slice of the selected set
        m, l, o = _partial_state(Q[i], K[i], V[i], mine)
        ms.append(m); ls.append(l); os_.append(o)
    out = allgather_lse_merge(torch.tensor(ms), torch.tensor(ls), torch.tensor(np.stack(os_)))
    ref = np.stack([O.attention(Q[i], K[i], V[i], O.select(Q[i], K[i], k)) for i in range(lanes)])
    err_seq = float(np.abs(out.numpy() - ref).max())
    # --- batch x head sharding: disjoint lanes, results gathered only for checking ---
    a, b = lane_block(lanes, world, rank)
    local = torch.tensor(np.stack([O.attention(Q[i], K[i], V[i], O.select(Q[i], K[i], k)) for i in range(a, b)]
                                  or [np.zeros(d)])[: b - a])
    sizes = [None] * world
    dist.all_gather_object(sizes, (a, b, local.numpy()))
    full = np.concatenate([x[2] for x in sorted(sizes, key=lambda x: x[0])])
    err_lane = float(np.abs(full - ref).max())
    t = max_over_ranks(float(rank + 1))
    # --- exact global top-k threshold exchange over sequence shards (incl. heavy ties) ---
    from paper_2506_20187_b200.shard import global_topk_mask
    ok_topk = True
    for trial in range(4):
        rng2 = np.random.default_rng(100 + trial)
        full_scores = rng2.normal(size=1000)
        if trial >= 2:
            full_scores = np.round(full_scores, 1)  # many exact ties across shard boundaries
        t0, t1 = token_block(1000, world, rank, align=1)
        for kk in (1, 37, 500, 1000):
            m = global_topk_mask(torch.tensor(full_scores[t0:t1]), kk).numpy()
            got = np.nonzero(m)[0] + t0
            gathered = [None] * world
            dist.all_gather_object(gathered, got.tolist())
            allsel = sorted(x for g in gathered for x in g)
            ref = O.topk(full_scores, kk).tolist()
            ok_topk &= allsel == ref
    # --- the batched per-lane threshold exchange used by the GPU config-5 path ---
    from paper_2506_20187_b200.shard import _ord_keys, radix_threshold
    rng3 = np.random.default_rng(7)
    scores = np.round(rng3.normal(size=(5, 600)), 2)  # ties
    t0, t1 = token_block(600, world, rank, align=1)
    keys = _ord_keys(torch.tensor(scores[:, t0:t1]))
    kv = torch.tensor([1, 60, 300, 599, 600])

    def allreduce(x):
        dist.all_reduce(x)
        return x

    T, take = radix_threshold(keys, torch.ones_like(keys, dtype=torch.bool), kv, allreduce)
    for i in range(5):
        kth_score = scores[i, O.topk(scores[i], int(kv[i]))].min()  # O.topk: the set, token order
        ok_topk &= int(T[i]) == int(_ord_keys(torch.tensor([kth_score]))[0])
        n_gt = int((scores[i] > kth_score).sum())
        ok_topk &= int(take[i]) == int(kv[i]) - n_gt
    if rank == 0:
        ret.put((err_seq, err_lane, t, ok_topk))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharding(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    err_seq, err_lane, t, ok_topk = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err_seq < 1e-12 and err_lane == 0.0 and t == float(world)
    assert ok_topk
