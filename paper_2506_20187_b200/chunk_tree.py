"""Drop-in for kvtier.chunk_tree (chunk_tree.py:1-387): sizing model, partitions, exact
top-k selection on the B200, desert merging.

Host-side scalar logic (next_pow2, chunk_cost, plan_chunk_count, ChunkPlanConfig) mirrors
the reference semantics.  `select_top_k` keeps the reference's contract -- the exact
top-k set by logit, ties to the lower index, cold chunks fetched through `store` only when
they can hold a selected token, `RuntimeError` for a cold chunk without a store -- but
evaluates it the GPU way instead of a serial heap:

  level A  K3 bounds of every live leaf; plan: tau = k-th largest lower bound (row
           weighted); leaves with U < tau are pruned, and so are leaves that >= k tokens
           rank before under the tie-break (L_i == U_j, i before j; _dominance_prune);
  level B  surviving leaves wider than the base grid are re-bounded per base chunk
           (abstracts built once at build_partition) and pruned again;
  cold     candidate regions inside abstract-only leaves are fetched via ChunkSource;
  K4/K5    candidate tokens get canonical f64 logits, a cluster radix select takes the
           top k (score desc, index asc).

After selection the partition is the canonical one the reference reaches after
select_top_k + merge_desert: maximal runs of selected tokens (IMPORTANT) and their
complement (DESERT, exact merged abstracts), plus the original PAD tail.  `important_tokens`
is returned in rank order (score desc, index asc) -- the order the reference's heap confirms
singletons in; a chunk it confirms whole is appended in index order there, so the two orders
can differ inside such a chunk (its tests compare sets).  eval_count = bounds evaluated + tokens exactly scored.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Protocol

import numpy as np
import torch

from . import ops
from .importance import ChunkAbstract, device, merge_abstracts, to_device

# -- chunk-count cost model (chunk_tree.py:34-123) ------------------------------------------------


def next_pow2(n: int) -> int:
    if n < 1:
        raise ValueError("n must be >= 1")
    return 1 << (n - 1).bit_length()


def _check_rho(rho: float) -> None:
    if not 0.0 <= rho < 1.0:
        raise ValueError(f"rho must be in [0, 1), got {rho}")


def chunk_cost(m: int, n: int, rho: float) -> float:
    """A(m) = m * sum_{i<L} (2 rho)^i, L = max(1, log2(n/m)) (chunk_tree.py:40-54)."""
    _check_rho(rho)
    if m < 1 or n < 1 or n % m != 0:
        raise ValueError(f"m={m} must divide n={n}")
    levels = max(1, int(math.log2(n // m)))
    r = 2.0 * rho
    if r == 1.0:
        return float(m * levels)
    return m * (1.0 - r ** levels) / (1.0 - r)


def plan_chunk_count(n: int, rho: float, *, min_chunk_size: int = 8, max_chunk_size: int = 64) -> int:
    """argmin_m A(m) over powers of two (ties -> fewer chunks), size clamped (chunk_tree.py:62-83)."""
    _check_rho(rho)
    if min_chunk_size > max_chunk_size:
        raise ValueError("min_chunk_size must be <= max_chunk_size")
    n_eff = next_pow2(n)
    best_m, best = 1, math.inf
    m = 1
    while m <= n_eff:
        c = chunk_cost(m, n_eff, rho)
        if c < best - 1e-12:
            best_m, best = m, c
        m *= 2
    size = min(max(n_eff // best_m, min_chunk_size), max_chunk_size, n_eff)
    return n_eff // size


@dataclass
class ChunkPlanConfig:
    """Per-layer / per-step initial chunk size (chunk_tree.py:86-123)."""

    default_chunk_size: int = 64
    early_chunk_size: int = 8
    early_layers: int = 2
    early_steps_fraction: float = 0.075
    rho: tuple[float, ...] | None = None

    def __post_init__(self):
        for name in ("default_chunk_size", "early_chunk_size"):
            v = getattr(self, name)
            if v < 1 or v & (v - 1):
                raise ValueError(f"{name} must be a positive power of two, got {v}")
        if self.early_chunk_size > self.default_chunk_size:
            raise ValueError("early_chunk_size must be <= default_chunk_size")
        if self.early_layers < 0:
            raise ValueError("early_layers must be >= 0")
        if not 0.0 <= self.early_steps_fraction <= 1.0:
            raise ValueError("early_steps_fraction must be in [0, 1]")

    def early_step_count(self, n_steps: int) -> int:
        return math.ceil(self.early_steps_fraction * n_steps)

    def chunk_size_for(self, layer: int, step: int, n_steps: int, n_context: int) -> int:
        if layer < self.early_layers or step < self.early_step_count(n_steps):
            return min(self.early_chunk_size, next_pow2(n_context))
        if self.rho is not None:
            rho = self.rho[layer % len(self.rho)]
            m = plan_chunk_count(n_context, rho, min_chunk_size=self.early_chunk_size,
                                 max_chunk_size=self.default_chunk_size)
            return next_pow2(n_context) // m
        return min(self.default_chunk_size, next_pow2(n_context))


# -- partition structure (chunk_tree.py:127-168) -------------------------------------------------

CANDIDATE = "candidate"
IMPORTANT = "important"
DESERT = "desert"
PAD = "pad"


@dataclass
class ChunkNode:
    start: int
    end: int
    abstract: ChunkAbstract | None = None
    upper: float = math.nan
    lower: float = math.nan
    state: str = CANDIDATE
    residency: str = "warm"
    abstract_only: bool = False
    children: tuple = ()

    @property
    def size(self) -> int:
        return self.end - self.start


@dataclass
class Partition:
    leaves: list[ChunkNode]
    n_real: int
    n_pad: int
    keys: np.ndarray | None = None  # host copy [n_real, d]
    # device state (not part of the reference type)
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    def real_leaves(self) -> list[ChunkNode]:
        return [c for c in self.leaves if c.state != PAD]

    def leaf_spans(self) -> list[tuple[int, int, str]]:
        return [(c.start, c.end, c.state) for c in self.leaves]


class ChunkSource(Protocol):
    """Cold-tier hook: make keys for [start, end) resident and return them (chunk_tree.py:165-168)."""

    def fetch(self, start: int, end: int) -> np.ndarray: ...


def _keys_dtype(keys: np.ndarray) -> torch.dtype:
    return torch.float32 if keys.dtype == np.float32 else torch.float64


def build_partition(n: int, m: int, keys: np.ndarray | None = None,
                    abstracts: list[ChunkAbstract] | None = None) -> Partition:
    """m uniform leaves over [0, next_pow2(n)), trailing pads (chunk_tree.py:171-210).
    Abstracts of resident leaves are built on the GPU (K1)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    n_pad = next_pow2(n)
    if m < 1 or n_pad % m != 0:
        raise ValueError(f"m={m} must be a power-of-two divisor of padded n={n_pad}")
    size = n_pad // m
    host_keys = None
    if keys is not None:
        k = np.asarray(keys)
        if k.ndim != 2 or k.shape[0] != n:
            raise ValueError(f"keys rows {k.shape[0] if k.ndim else None} != n {n}")
        host_keys = np.array(k, dtype=np.float32 if k.dtype == np.float32 else np.float64, copy=True)
    by_start = {a.start: a for a in abstracts or []}
    n_real_leaves = (n + size - 1) // size
    cold = [s in by_start and by_start[s].end == min(s + size, n) for s in range(0, n_real_leaves * size, size)]
    if host_keys is None and not all(cold):
        first = next(i for i, c in enumerate(cold) if not c)
        raise ValueError(f"no keys and no abstract covering chunk [{first * size}, {first * size + size})")
    dev: dict = {"base_size": size}
    base_max = base_min = None
    if host_keys is not None:
        kd = to_device(host_keys)
        dev["keys"] = kd[None]
        bmax, bmin = ops.abstract_build(dev["keys"], n, size)
        base_max, base_min = bmax[0].double(), bmin[0].double()
    d = host_keys.shape[1] if host_keys is not None else abstracts[0].max_key.shape[0]
    if base_max is None:
        base_max = torch.empty((n_real_leaves, d), dtype=torch.float64, device=device())
        base_min = torch.empty_like(base_max)
    leaves: list[ChunkNode] = []
    for i, start in enumerate(range(0, n_pad, size)):
        end = start + size
        if start >= n:
            leaves.append(ChunkNode(start=start, end=end, state=PAD))
            continue
        if cold[i]:
            a = by_start[start]
            base_max[i] = torch.as_tensor(a.max_key, dtype=torch.float64)
            base_min[i] = torch.as_tensor(a.min_key, dtype=torch.float64)
            leaves.append(ChunkNode(start=start, end=end, abstract=a, abstract_only=True, residency="cold"))
        else:
            leaves.append(ChunkNode(start=start, end=end))  # abstract materialised lazily below
    dev["base_max"], dev["base_min"] = base_max, base_min
    hm, hn = base_max.cpu().numpy(), base_min.cpu().numpy()
    for i, c in enumerate(leaves):
        if c.state != PAD and c.abstract is None:
            c.abstract = ChunkAbstract(start=c.start, end=c.end, max_key=hm[i].copy(), min_key=hn[i].copy())
    dev["cold"] = [(c.start, min(c.end, n)) for c in leaves if c.abstract_only]
    return Partition(leaves=leaves, n_real=n, n_pad=n_pad, keys=host_keys, _dev=dev)


# -- selection (chunk_tree.py:216-338) ------------------------------------------------------------


@dataclass
class SelectionResult:
    k: int
    important_tokens: list[int]
    eval_count: int
    fetch_set: list[tuple[int, int]] = field(default_factory=list)
    desert_chunks: list[tuple[int, int]] = field(default_factory=list)

    @property
    def selected(self) -> set[int]:
        return set(self.important_tokens)


def _dominance_prune(U: torch.Tensor, L: torch.Tensor, starts: np.ndarray, n: int, k: int) -> torch.Tensor:
    """Tie-aware pruning under the reference's order (score desc, index asc; chunk_tree.py:233-338).

    The tokens of leaf i rank strictly before every token of leaf j when L_i > U_j, or when
    L_i == U_j and leaf i lies before leaf j (equal scores go to the lower index).  Leaf j can
    hold no selected token once such leaves cover >= k tokens.  This is the rule the heap
    applies implicitly -- it never pops j before the budget fills -- and it subsumes the plan's
    tau rule (U_j < k-th largest L).  It matters where bounds tie exactly: chunks of identical
    rows have U == L (exact, no widening), e.g. the flat chunks of the walkthrough
    (test_chunk_tree.py:214-228).  Returns U with -inf at the pruned leaves; on device."""
    m = len(starts)
    if k <= 0 or m < 2:
        return U
    dev = U.device
    u, lo = U[0, :m], L[0, :m]
    st = torch.from_numpy(np.asarray(starts, dtype=np.int64)).to(dev)
    size = torch.diff(st, append=torch.tensor([n], dtype=torch.int64, device=dev)).to(torch.float64)
    cnt = torch.empty(m, dtype=torch.float64, device=dev)
    blk = max(1, (1 << 24) // m)
    for j0 in range(0, m, blk):
        j1 = min(m, j0 + blk)
        uj, sj = u[j0:j1, None], st[j0:j1, None]
        before = (lo[None, :] > uj) | ((lo[None, :] == uj) & (st[None, :] < sj))
        cnt[j0:j1] = (before.to(torch.float64) * size[None, :]).sum(dim=1)
    out = U.clone()
    out[0, :m] = torch.where(cnt >= k, torch.full_like(u, -math.inf), u)
    return out


def _bounds_plan(q, amax, amin, starts: np.ndarray, n: int, k: int):
    dev = q.device
    ls = torch.from_numpy(np.ascontiguousarray(starts, dtype=np.int32))[None].to(dev)
    nl = torch.tensor([len(starts)], dtype=torch.int32, device=dev)
    U, L = ops.chunk_bounds(q[None], amax[None], amin[None], n, 0, ls, nl)
    plan = ops.select_plan(_dominance_prune(U, L, starts, n, k), L, n, k, 0, ls, nl, want_cand_leaf=True)
    return U, L, plan


def _overlaps(spans, a: int, b: int) -> list[tuple[int, int]]:
    return [s for s in spans if s[0] < b and a < s[1]]


def select_top_k(partition: Partition, query: np.ndarray, k: int, store: ChunkSource | None = None) -> SelectionResult:
    """Exact top-k tokens by logit, ties broken by lower index (chunk_tree.py:233-338)."""
    n = partition.n_real
    if k < 0 or k > n:
        raise ValueError(f"k must be in [0, {n}], got {k}")
    dev = partition._dev
    q = to_device(query, torch.float64)
    live = partition.real_leaves()
    for c in live:
        c.state = CANDIDATE
    result = SelectionResult(k=k, important_tokens=[], eval_count=0)

    # ---- level A: leaves of the current partition ----
    starts_a = np.array([c.start for c in live], dtype=np.int64)
    ends_a = np.array([min(c.end, n) for c in live], dtype=np.int64)
    amax_a = to_device(np.stack([c.abstract.max_key for c in live]), torch.float64)
    amin_a = to_device(np.stack([c.abstract.min_key for c in live]), torch.float64)
    U, L, plan = _bounds_plan(q, amax_a, amin_a, starts_a, n, k)
    result.eval_count += len(live)
    cand_a = plan["cand_leaf"][0, :len(live)].cpu().numpy().astype(bool)
    # the pipeline prunes on raw dots; the leaf attributes keep kvtier's logit scale
    sd = math.sqrt(q.shape[0])
    Uh, Lh = U[0, :len(live)].cpu().numpy(), L[0, :len(live)].cpu().numpy()
    for c, u, l in zip(live, Uh, Lh):
        c.upper, c.lower = float(u) / sd, float(l) / sd

    # ---- level B: refine wide candidate leaves on the base grid ----
    bs = dev["base_size"]
    unit_s, unit_src = [], []  # src >= 0: base chunk row; src < 0: -(leaf index) - 1
    refined = 0
    for i, c in enumerate(live):
        s, e = int(starts_a[i]), int(ends_a[i])
        if cand_a[i] and k > 0 and (e - 1) // bs > s // bs:
            for b in range(s // bs, (e - 1) // bs + 1):
                unit_s.append(max(s, b * bs))
                unit_src.append(b)
                refined += 1
        else:
            unit_s.append(s)
            unit_src.append(-i - 1)
    if refined:
        src = np.array(unit_src)
        is_base = src >= 0
        idx_base = torch.from_numpy(np.where(is_base, src, 0)).to(q.device)
        idx_leaf = torch.from_numpy(np.where(is_base, 0, -src - 1)).to(q.device)
        mask = torch.from_numpy(is_base)[:, None].to(q.device)
        amax_b = torch.where(mask, dev["base_max"][idx_base], amax_a[idx_leaf])
        amin_b = torch.where(mask, dev["base_min"][idx_base], amin_a[idx_leaf])
        starts_b = np.array(unit_s, dtype=np.int64)
        U, L, plan = _bounds_plan(q, amax_b.contiguous(), amin_b.contiguous(), starts_b, n, k)
        result.eval_count += refined
        starts_u = starts_b
    else:
        starts_u = starts_a
    ends_u = np.append(starts_u[1:], n)
    cand_u = plan["cand_leaf"][0, :len(starts_u)].cpu().numpy().astype(bool)

    # ---- cold tier: fetch cold records that can hold a selected token ----
    cold = dev.get("cold", [])
    if cold:
        need = []
        for s, e, cflag in zip(starts_u, ends_u, cand_u):
            if cflag:
                for span in _overlaps(cold, int(s), int(e)):
                    if span not in need:
                        need.append(span)
        for s, e in sorted(need):
            if store is None:
                raise RuntimeError(f"chunk [{s},{e}) is cold but no store was given")
            block = store.fetch(s, e)
            if partition.keys is None:
                raise RuntimeError("partition has no key storage to fetch into")
            partition.keys[s:e] = block
            dev["keys"][0, s:e] = to_device(np.asarray(block), dev["keys"].dtype)
            cold.remove((s, e))
            result.fetch_set.append((s, e))
            for c in live:
                if c.start < e and s < min(c.end, n):
                    c.residency = "warm"
                    if not _overlaps(cold, c.start, min(c.end, n)):
                        c.abstract_only = False
    if "keys" not in dev:
        raise RuntimeError("partition has no key storage to fetch into")

    # ---- K4 + K5: exact top-k ----
    cs, ct = ops.cand_score(q[None], dev["keys"], plan, n)
    n_cand = int(plan["n_cand"][0].item())
    result.eval_count += n_cand
    sel_tok, sel_score, n_sel = ops.topk_select(cs, ct, plan["n_cand"], k)
    sel = sel_tok[0, :k].cpu().numpy().astype(np.int64)
    sc = sel_score[0, :k].cpu().numpy()
    # rank order (score desc, index asc): the order the reference's heap confirms singletons in
    result.important_tokens = [int(t) for t in sel[np.lexsort((sel, -sc))]]

    # ---- canonical partition: selected runs + complement runs (K6) ----
    _rebuild(partition, sel_tok, sel_score, n_sel, k)
    result.desert_chunks = [(c.start, min(c.end, n)) for c in partition.leaves if c.state == DESERT]
    return result


def _rebuild(partition: Partition, sel_tok, sel_score, n_sel, k: int) -> None:
    n = partition.n_real
    dev = partition._dev
    runs = ops.runs_scan(sel_tok.contiguous(), n_sel, n, want_partition=True)
    npart = int(runs["n_part"][0].item())
    pstart = runs["part_start"][0, :npart].cpu().numpy().astype(np.int64)
    pstate = runs["part_state"][0, :npart].cpu().numpy()
    pend = np.append(pstart[1:], n)
    pads = [c for c in partition.leaves if c.state == PAD]
    real_end = pads[0].start if pads else partition.n_pad
    # per-leaf score bounds of important runs: exact extremes of their logits
    nr = int(runs["n_runs"][0].item())
    rlen = runs["run_len"][0, :nr].cpu().numpy().astype(np.int64)
    sc = sel_score[0].cpu().numpy() / math.sqrt(dev["base_max"].shape[1])  # raw dots -> logits
    run_hi, run_lo, pos = [], [], 0
    for ln in rlen:
        seg = sc[pos:pos + ln]
        run_hi.append(float(seg.max()))
        run_lo.append(float(seg.min()))
        pos += ln
    # exact abstracts: resident pieces from keys (K1 spans), cold spans from stored abstracts,
    # then one K2 segment per leaf over its pieces (in leaf order)
    cold = dev.get("cold", [])
    pieces_s, pieces_e, rows, seg_b, seg_e = [], [], [], [], []
    bs = dev["base_size"]
    for li, (s, e) in enumerate(zip(pstart, pend)):
        pos = int(s)
        seg_b.append(len(rows))
        for cs_, ce_ in sorted(_overlaps(cold, int(s), int(e))):
            if cs_ > pos:
                rows.append(("span", len(pieces_s)))
                pieces_s.append(pos); pieces_e.append(cs_)
            rows.append(("base", cs_ // bs))  # whole cold record: its stored (base) abstract
            pos = ce_
        if pos < e:
            rows.append(("span", len(pieces_s)))
            pieces_s.append(pos); pieces_e.append(int(e))
        seg_e.append(len(rows))
    gdev = dev["base_max"].device
    if pieces_s:
        pmx, pmn = ops.abstract_spans(dev["keys"], torch.zeros(len(pieces_s), dtype=torch.int32),
                                      torch.tensor(pieces_s, dtype=torch.int32), torch.tensor(pieces_e, dtype=torch.int32))
        pmx, pmn = pmx.double(), pmn.double()
    else:
        pmx = pmn = torch.empty((0, dev["base_max"].shape[1]), dtype=torch.float64, device=gdev)
    ns = pmx.shape[0]
    idx = torch.tensor([i if kind == "span" else ns + i for kind, i in rows], dtype=torch.int64, device=gdev)
    src_mx = torch.cat([pmx, dev["base_max"].double()]).index_select(0, idx)
    src_mn = torch.cat([pmn, dev["base_min"].double()]).index_select(0, idx)
    amax, amin = ops.abstract_merge(src_mx, src_mn, seg_begin=seg_b, seg_end=seg_e)
    hmx, hmn = amax.cpu().numpy(), amin.cpu().numpy()
    leaves: list[ChunkNode] = []
    r = 0
    for li in range(npart):
        s, e = int(pstart[li]), int(pend[li])
        end = real_end if li == npart - 1 else e
        is_cold = any(True for _ in _overlaps(cold, s, e))
        node = ChunkNode(start=s, end=end,
                         abstract=ChunkAbstract(start=s, end=end, max_key=hmx[li], min_key=hmn[li]),
                         residency="cold" if is_cold else "warm", abstract_only=is_cold)
        if pstate[li] == 1:
            node.state = IMPORTANT
            node.upper, node.lower = run_hi[r], run_lo[r]
            r += 1
        else:
            node.state = DESERT
        leaves.append(node)
    partition.leaves = leaves + pads


# -- desert merging (chunk_tree.py:344-379) --------------------------------------------------------


def merge_desert(partition: Partition) -> int:
    """Coalesce adjacent desert leaves (and adjacent pad leaves); returns merges done."""
    merged: list[ChunkNode] = []
    count = 0
    for node in partition.leaves:
        prev = merged[-1] if merged else None
        if prev is not None and node.state == prev.state and prev.state in (DESERT, PAD) and prev.end == node.start:
            fused = ChunkNode(
                start=prev.start, end=node.end,
                abstract=merge_abstracts(prev.abstract, node.abstract) if prev.state == DESERT else None,
                state=prev.state,
                residency="cold" if "cold" in (prev.residency, node.residency) else prev.residency,
                abstract_only=prev.abstract_only or node.abstract_only,
            )
            merged[-1] = fused
            count += 1
        else:
            merged.append(node)
    partition.leaves = merged
    return count


def dump_partition(partition: Partition) -> str:
    """One leaf per line: 'start end state upper lower residency' (chunk_tree.py:382-387)."""
    lines = [f"{c.start} {c.end} {c.state} {c.upper:.9g} {c.lower:.9g} {c.residency}" for c in partition.leaves]
    return "\n".join(lines) + ("\n" if lines else "")
