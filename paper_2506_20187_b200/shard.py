"""Multi-GPU partitioning of the hot path.

* batch x head sharding: lanes (b, h) are independent trees, so each
  rank owns a disjoint, contiguous block of lanes and needs NO collective on the data path.
* sequence sharding (config 5): each rank owns a contiguous token range of every lane and
  produces a partial softmax state (m, l, o[d]) over its slice of the selected set; the
  states are merged exactly with a log-sum-exp combine after an all-gather.  This is the
  only collective in the design, and it moves (d + 2) floats per lane per rank.

Everything here is device-agnostic torch so the same code runs under NCCL on the GPUs and
under gloo in the CPU tests (tests/test_dist_gloo.py).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def lane_block(n_lanes: int, world: int, rank: int) -> tuple[int, int]:
    """[start, end) of the lanes owned by `rank` (balanced contiguous blocks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_lanes, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def batch_block(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Batch rows owned by `rank`; a row keeps all its heads together (no TP)."""
    return lane_block(batch, world, rank)


def token_block(n: int, world: int, rank: int, align: int = 64) -> tuple[int, int]:
    """Contiguous token range of `rank` for sequence sharding, aligned to chunk boundaries."""
    chunks = (n + align - 1) // align
    a, b = lane_block(chunks, world, rank)
    return min(n, a * align), min(n, b * align)


def lse_merge(m: torch.Tensor, l: torch.Tensor, o: torch.Tensor) -> torch.Tensor:
    """Combine partial softmax states.  m, l: [P, lanes]; o: [P, lanes, d] holding
    sum_i exp(s_i - m_p) v_i.  Returns softmax-weighted outputs [lanes, d]; parts with
    l == 0 (no selected token) are ignored."""
    valid = l > 0
    mm = torch.where(valid, m, torch.full_like(m, -torch.inf))
    M = mm.max(dim=0).values
    w = torch.where(valid, torch.exp(mm - M[None]), torch.zeros_like(m))
    den = (w * l).sum(dim=0)
    num = (w[..., None] * o).sum(dim=0)
    return num / den.clamp_min(torch.finfo(num.dtype).tiny)[..., None]


def allgather_lse_merge(m: torch.Tensor, l: torch.Tensor, o: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather every rank's (m, l, o) for its token shard and merge (NCCL on GPUs)."""
    world = dist.get_world_size(group)
    packed = torch.cat([m[..., None], l[..., None], o], dim=-1).contiguous()  # [lanes, d+2]
    parts = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed, group=group)
    out = torch.stack(parts)
    return lse_merge(out[..., 0], out[..., 1], out[..., 2:])


class NcclLseMerge:
    """The sequence-sharded path's only collective through the library (kvt_lse_allgather_merge:
    NCCL all-gather of each rank's (m, l, o) + the log-sum-exp merge kernel, one stream-ordered
    call).  The NCCL unique id goes from rank 0 to the others over torch.distributed (any
    backend); with world == 1 no process group is needed."""

    def __init__(self, rank: int = 0, world: int = 1, group=None):
        import ctypes
        from . import _lib as L
        if not L.kvt_nccl_available():
            raise RuntimeError("libnccl.so.2 could not be loaded")
        self.L, self.rank, self.world = L, rank, world
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            L.check(L.kvt_nccl_unique_id(uid), "nccl_unique_id")
        if world > 1:
            obj = [bytes(uid) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            ctypes.memmove(uid, obj[0], 128)
        self.comm = ctypes.c_void_p()
        L.check(L.kvt_nccl_comm_init(ctypes.byref(self.comm), world, rank, uid), "nccl_comm_init")

    def merge(self, m: torch.Tensor, l: torch.Tensor, o: torch.Tensor, logit_scale: float) -> torch.Tensor:
        """m, l: [lanes] f64 (kvt_attn_lse of this rank's shard); o: [lanes, d] this rank's
        normalised output -> merged output f64 [lanes, d] on every rank."""
        from . import ops
        part = torch.cat([m[:, None], l[:, None], o.double()], dim=1).contiguous()
        n, d = o.shape
        gather = torch.empty((self.world, n, d + 2), dtype=torch.float64, device=o.device)
        out = torch.empty((n, d), dtype=torch.float64, device=o.device)
        self.L.check(self.L.kvt_lse_allgather_merge(self.comm, self.world, part.data_ptr(), n, d, float(logit_scale),
                                                    gather.data_ptr(), None, out.data_ptr(), ops._stream()),
                     "lse_allgather_merge")
        return out

    def close(self) -> None:
        if self.comm:
            self.L.check(self.L.kvt_nccl_comm_destroy(self.comm), "nccl_comm_destroy")
            self.comm = None


_MIN64 = -(2 ** 63)


def _ord_keys(scores: torch.Tensor) -> torch.Tensor:
    """Bit patterns (held in int64) of the unsigned orderable keys of float64 scores:
    larger score -> larger unsigned key; -0 == +0."""
    s = torch.where(scores == 0, torch.zeros_like(scores), scores)
    b = s.view(torch.int64)
    return torch.where(b < 0, ~b, b | torch.tensor(_MIN64, dtype=torch.int64, device=b.device))


def global_topk_mask(scores: torch.Tensor, k: int, group=None) -> torch.Tensor:
    """Exact top-k across a sequence-sharded lane.

    Every rank holds the canonical scores of its contiguous token shard (rank order = token
    order).  An 8-round radix select over the 64-bit orderable keys, each round an
    all-reduce of a 256-bin histogram (the "global threshold exchange"), finds the exact
    k-th key T; ties at T go to the lowest token indices, i.e. to lower ranks first (one
    all-gather of the per-rank tie counts).  Returns this rank's boolean selection mask.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    keys = _ord_keys(scores.double())
    dev = keys.device
    prefix = torch.zeros((), dtype=torch.int64, device=dev)
    mask = torch.zeros((), dtype=torch.int64, device=dev)
    remaining = int(k)
    for shift in range(56, -8, -8):
        sel = (keys & mask) == prefix
        digits = ((keys >> shift) & 0xFF)[sel]
        hist = torch.bincount(digits, minlength=256).to(torch.int64)
        dist.all_reduce(hist, group=group)
        h = hist.flip(0).cumsum(0)  # counts from the top digit down
        idx = int(torch.searchsorted(h, torch.tensor(remaining, device=dev)).item())
        b = 255 - idx
        above = int(h[idx - 1].item()) if idx > 0 else 0
        prefix = prefix | (torch.tensor(b, dtype=torch.int64, device=dev) << shift)
        mask = mask | (torch.tensor(0xFF, dtype=torch.int64, device=dev) << shift)
        remaining -= above
    # unsigned comparison through the sign flip; ties share the key `prefix`
    flip = torch.tensor(_MIN64, dtype=torch.int64, device=dev)
    gt = (keys ^ flip) > (prefix ^ flip)
    eq = keys == prefix
    eq_counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(eq_counts, eq.sum().reshape(1), group=group)
    before = int(sum(int(c.item()) for c in eq_counts[:rank]))
    take = max(0, min(int(eq.sum().item()), remaining - before))
    eq_rank = torch.cumsum(eq.to(torch.int64), 0) - 1
    return gt | (eq & (eq_rank < take))


# ---- config 5 on the GPU: exact sequence-sharded select + attend ------------------------------


def radix_threshold(keys: torch.Tensor, valid: torch.Tensor, k: torch.Tensor, allreduce) -> tuple:
    """Per-lane exact k-th largest of the orderable int64 keys [lanes, m] (valid mask) across
    shards: 8 rounds, each one all-reduce of a [lanes, 256] digit histogram (the "global
    threshold exchange").  Returns (T keys [lanes], remaining ties to take at T [lanes])."""
    lanes = keys.shape[0]
    dev = keys.device
    prefix = torch.zeros(lanes, dtype=torch.int64, device=dev)
    mask = torch.zeros(lanes, dtype=torch.int64, device=dev)
    remaining = k.to(torch.int64).clone()
    ar = torch.arange(256, device=dev)
    for shift in range(56, -8, -8):
        sel = valid & ((keys & mask[:, None]) == prefix[:, None])
        digits = (keys >> shift) & 0xFF
        hist = torch.zeros((lanes, 256), dtype=torch.int64, device=dev)
        hist.scatter_add_(1, digits, sel.to(torch.int64))
        hist = allreduce(hist)
        h = hist.flip(1).cumsum(1)  # counts from the top digit down
        idx = torch.searchsorted(h, remaining[:, None]).squeeze(1).clamp_max(255)
        b = 255 - idx
        above = torch.where(idx > 0, h.gather(1, (idx - 1).clamp_min(0)[:, None]).squeeze(1), torch.zeros_like(idx))
        prefix = prefix | (b << shift)
        mask = mask | (torch.full_like(mask, 0xFF) << shift)
        remaining = remaining - above
    del ar
    return prefix, remaining


def seq_shard_select_attend(q: torch.Tensor, keys, values, n_local: int, C: int, k: int, shard_rank: int,
                            allreduce, allgather, decoder_bufs=None):
    """One layer of config 5 on this rank's token shard (GPU kernels + two small collectives).

    1. exact local top-min(k, n_local) of every lane with the fused kernels (canonical scores):
       every token of the global top-k is in its own shard's top-k, so this loses nothing;
    2. the global k-th score by `radix_threshold` over those candidates (ties at T go to the
       lowest tokens, i.e. to lower shard ranks first: one all-gather of per-rank tie counts);
    3. K7 over this rank's globally selected subset -> (m, l, o) per lane;
    4. all-gather of (m, l, o) and the log-sum-exp merge kernel (kvt_lse_merge).
    Returns (attention output f32 [lanes, d], this rank's selected local token ids as a list
    of int32 tensors).  `allreduce(t)` sums over ranks, `allgather(t)` stacks rank tensors in
    rank order (torch.distributed wrappers on real ranks; emulated in single-GPU tests)."""
    from . import ops
    lanes, d = q.shape
    kk = min(k, n_local)
    amax, amin = ops.abstract_build(keys, n_local, C, abs_dtype=torch.bfloat16)
    ws = ops.LayerWorkspace(lanes, n_local, ops.n_grid_leaves(n_local, C), d, q.device)
    out = {"sel_tok": torch.empty((lanes, max(kk, 1)), dtype=torch.int32, device=q.device),
           "sel_score": torch.empty((lanes, max(kk, 1)), dtype=torch.float64, device=q.device),
           "n_sel": torch.empty(lanes, dtype=torch.int32, device=q.device),
           "out": torch.empty((lanes, d), dtype=torch.float32, device=q.device)}
    ops.select_attend(q, keys, values, amax, amin, n_local, kk, C, ws, out, exact_scores=True)
    sc = out["sel_score"][:, :kk]
    keys64 = _ord_keys(sc)
    valid = torch.ones_like(keys64, dtype=torch.bool)
    T, take = radix_threshold(keys64, valid, torch.full((lanes,), k, device=q.device), allreduce)
    flip = torch.tensor(_MIN64, dtype=torch.int64, device=q.device)
    gt = (keys64 ^ flip) > (T ^ flip)[:, None]
    eq = keys64 == T[:, None]
    eq_all = allgather(eq.sum(1))  # [world, lanes]
    before = eq_all[:shard_rank].sum(0) if shard_rank > 0 else torch.zeros(lanes, dtype=torch.int64, device=q.device)
    my_take = (take - before).clamp(min=0)
    eq_rank = torch.cumsum(eq.to(torch.int64), 1) - 1
    mine = gt | (eq & (eq_rank < my_take[:, None]))
    # compact this rank's subset (token order is preserved: sel_tok is ascending)
    n_mine = mine.sum(1).to(torch.int32)
    order = torch.argsort((~mine).to(torch.int8), dim=1, stable=True)
    st = torch.gather(out["sel_tok"][:, :kk], 1, order).contiguous()
    ss = torch.gather(sc, 1, order).contiguous()
    o, lse = ops.sparse_decode_attn(values, st, ss, n_mine, want_lse=True)
    part = torch.cat([lse, o.double()], dim=1)  # [lanes, d + 2]
    parts = allgather(part)  # [world, lanes, d + 2]
    res = ops.lse_merge(parts, 1.0 / (d ** 0.5))
    return res, [st[i, :int(n_mine[i])] for i in range(lanes)]


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (multi-GPU timing is the slowest rank)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
