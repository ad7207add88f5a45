"""Hot / warm / cold residency and the transfer ledger of the decode path.

Restates the policy of the reference `kvtier.tiered_store` (`tiered_store.py:141-592`) --
same public names, byte accounting, placement, eviction order and errors -- over B200
memory instead of files:

  hot   HBM (where K7 reads),
  warm  pinned host memory (the `tier.HostTier` staging area, streamed to HBM by
        cudaMemcpyAsync on a side stream, optionally INT4-compressed),
  cold  the slower host tier (in the reference: per-lane record files).

Only bookkeeping happens here; the bytes move through optional hooks (`on_move(record,
src_tier, dst_tier)`) so the same object drives real transfers on the GPU box and runs as
pure host logic in the CPU tests.  Parity: `tests/test_tiered_store.py` replays operation
sequences frozen from the reference (`tests/golden/make_tier_golden.py`) and compares every
ledger row, every record's tier after every row, and the error types.

Accounting (`tiered_store.py:53-60`): a record of n tokens costs 2 * n * d * 2 bytes (fp16
K + V), a chunk summary 2 * d * 4 bytes.  Ledger r = (abstract + cold->warm bytes) / bytes
cold at row open (`tiered_store.py:131-136`).
"""

from __future__ import annotations

import csv
from collections import deque
from dataclasses import dataclass
from pathlib import Path
from typing import Callable, Iterable, Sequence

import numpy as np

from . import cold_files as CF
from .cold_files import ColdStoreError  # (tiered_store.py:71-72)  noqa: F401

HOT, WARM, COLD = "hot", "warm", "cold"
LEDGER_COLUMNS = ("step", "layer", "abstract_bytes", "cold_to_warm", "warm_to_hot", "hot_to_warm", "r")


def kv_nbytes(n_tokens: int, head_dim: int) -> int:
    """fp16 keys + values of n_tokens rows (tiered_store.py:53-55)."""
    return 4 * n_tokens * head_dim


def abstract_nbytes(head_dim: int) -> int:
    """One chunk summary: f32 max and min key vectors (tiered_store.py:58-60)."""
    return 8 * head_dim


class CapacityError(RuntimeError):
    """The hot + warm budgets cannot hold what may not go cold (tiered_store.py:63-64)."""


class ResidencyError(RuntimeError):
    """An operation's tier precondition does not hold (tiered_store.py:67-68)."""




@dataclass(frozen=True)
class TierConfig:
    """Budgets and policy knobs (tiered_store.py:75-94); `cold_dir` is accepted for API
    compatibility -- the cold tier here is host memory."""

    hot_capacity: int
    warm_capacity: int
    cold_dir: str | Path | None = None
    bandwidth_hot_warm: float = 8.0
    bandwidth_warm_cold: float = 2.0
    early_layers_pinned: int = 2
    hot_frequency_threshold: int = 4
    frequency_window: int = 16

    def __post_init__(self) -> None:
        checks = ((min(self.hot_capacity, self.warm_capacity) > 0, "budgets"),
                  (min(self.bandwidth_hot_warm, self.bandwidth_warm_cold) > 0, "link rates"),
                  (self.early_layers_pinned >= 0, "pinned layer count"),
                  (min(self.hot_frequency_threshold, self.frequency_window) >= 1, "frequency policy"))
        for ok, what in checks:
            if not ok:
                raise ValueError(f"TierConfig: invalid {what}")


@dataclass(eq=False)
class ChunkRecord:
    """One placement unit: a token span of one (layer, head) lane."""

    layer: int
    head: int
    start: int
    end: int
    nbytes: int
    tier: str
    pinned: bool
    access_count: int = 0
    offset: int = 0  # payload offset in the lane's KVCF file (file-backed stores)
    last_touch: int = -1

    @property
    def n_tokens(self) -> int:
        return self.end - self.start

    @property
    def replica_on_cold(self) -> bool:  # every non-pinned record is written through
        return not self.pinned

    def order_key(self):  # eviction order: least recently touched, then position
        return (self.last_touch, self.start, self.layer, self.head)


@dataclass
class LedgerRow:
    step: int
    layer: int
    abstract_bytes: int = 0
    cold_to_warm: int = 0
    warm_to_hot: int = 0
    hot_to_warm: int = 0
    fetch_ops: int = 0
    cold_bytes_at_open: int = 0

    @property
    def r(self) -> float:
        return 0.0 if self.cold_bytes_at_open == 0 else \
            (self.abstract_bytes + self.cold_to_warm) / self.cold_bytes_at_open


class TieredStore:
    """Residency manager: per-lane record lists (sorted by start), byte totals per tier, a
    per-token touch log for the frequency exemption and the open ledger row."""

    def __init__(self, config: TierConfig, n_layers: int, n_heads: int, head_dim: int,
                 on_move: Callable[[ChunkRecord, str, str], None] | None = None):
        if config.early_layers_pinned > n_layers:
            raise ValueError(f"{config.early_layers_pinned} pinned layers but only {n_layers} layers")
        self.config = config
        self.n_layers, self.n_heads, self.head_dim = n_layers, n_heads, head_dim
        self.on_move = on_move
        self.lanes: dict[tuple[int, int], list[ChunkRecord]] = {}
        self.used = {HOT: 0, WARM: 0}
        self.step = 0
        self.row: LedgerRow | None = None
        self.touch_log: dict[tuple[int, int], dict[int, deque]] = {}
        self.ledger_rows: list[LedgerRow] = []
        # file-backed cold tier (place_initial(trace, ...) with a cold_dir): KVCF/KVAB files
        self.cold_dir: Path | None = None

    # -- views ------------------------------------------------------------------------------
    @property
    def hot_used(self) -> int:
        return self.used[HOT]

    @property
    def warm_used(self) -> int:
        return self.used[WARM]

    def lane_records(self, layer: int, head: int) -> list[ChunkRecord]:
        return self.lanes[(layer, head)]

    def cold_spans(self, layer: int, head: int) -> list[tuple[int, int]]:
        return [(r.start, r.end) for r in self.lanes[(layer, head)] if r.tier == COLD]

    def cold_resident_bytes(self, layer: int) -> int:
        return sum(r.nbytes for h in range(self.n_heads) for r in self.lanes.get((layer, h), ()) if r.tier == COLD)

    def _all(self):
        for recs in self.lanes.values():
            yield from recs

    def _move(self, rec: ChunkRecord, dst: str) -> None:
        src = rec.tier
        if src in self.used:
            self.used[src] -= rec.nbytes
        if dst in self.used:
            self.used[dst] += rec.nbytes
        rec.tier = dst
        if self.on_move is not None:
            self.on_move(rec, src, dst)

    # -- ledger (tiered_store.py:188-220) ----------------------------------------------------
    def open_row(self, step: int, layer: int) -> LedgerRow:
        if self.row is not None:
            raise RuntimeError("open_row: a ledger row is already open")
        self.step = step
        self.row = LedgerRow(step=step, layer=layer, cold_bytes_at_open=self.cold_resident_bytes(layer))
        return self.row

    def close_row(self) -> LedgerRow:
        if self.row is None:
            raise RuntimeError("close_row without open_row")
        row, self.row = self.row, None
        self.ledger_rows.append(row)
        return row

    def transmission_ratio(self, layer: int, step: int | None = None) -> float:
        for row in reversed(self.ledger_rows):
            if row.layer == layer and (step is None or row.step == step):
                return row.r
        raise KeyError((layer, step))

    def write_ledger(self, path: str | Path) -> None:
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(LEDGER_COLUMNS)
            for r in self.ledger_rows:
                w.writerow([r.step, r.layer, r.abstract_bytes, r.cold_to_warm, r.warm_to_hot, r.hot_to_warm, str(r.r)])

    def _count(self, field: str, nbytes: int) -> None:
        if self.row is not None:
            setattr(self.row, field, getattr(self.row, field) + nbytes)

    # -- frequency (tiered_store.py:224-248) -------------------------------------------------
    def touch(self, layer: int, head: int, tokens: Iterable[int]) -> None:
        toks = sorted({int(t) for t in tokens})
        log = self.touch_log.setdefault((layer, head), {})
        for t in toks:
            q = log.setdefault(t, deque())
            if not q or q[-1] != self.step:
                q.append(self.step)
        if not toks:
            return
        # records covering any touched token (tokens and records both sorted by start)
        i = 0
        for rec in self.lanes[(layer, head)]:
            while i < len(toks) and toks[i] < rec.start:
                i += 1
            if i < len(toks) and toks[i] < rec.end:
                rec.access_count += 1
                rec.last_touch = self.step

    def frequency_exempt(self, layer: int, head: int, start: int, end: int) -> bool:
        log = self.touch_log.get((layer, head))
        if not log:
            return False
        horizon = self.step - self.config.frequency_window
        for t in range(start, end):
            q = log.get(t)
            if q is None:
                continue
            while q and q[0] <= horizon:
                q.popleft()
            if len(q) >= self.config.hot_frequency_threshold:
                return True
        return False

    # -- movement (tiered_store.py:250-372) --------------------------------------------------
    def _covering(self, layer: int, head: int, start: int, end: int) -> list[ChunkRecord]:
        hit = [r for r in self.lanes[(layer, head)] if r.start < end and start < r.end] if end > start else []
        if not hit:
            raise ValueError(f"lane ({layer}, {head}): no record covers tokens {start}..{end}")
        return hit

    def fetch_chunk(self, layer: int, head: int, start: int, end: int) -> list[ChunkRecord]:
        """Cold -> warm for every record covering [start, end) (whole records).  Returns the
        records; their payload is moved by the on_move hook."""
        hit = self._covering(layer, head, start, end)
        bad = [r for r in hit if r.tier != COLD]
        if bad:
            raise ResidencyError(f"lane ({layer}, {head}): fetch needs cold records, "
                                 f"got {[(r.start, r.tier) for r in bad]}")
        payload = []
        for rec in sorted(hit, key=lambda r: r.start):
            if self.cold_dir is not None:
                payload.append(CF.read_record(self.data_path(layer, head), rec.offset, rec.n_tokens, self.head_dim))
            self._move(rec, WARM)
            rec.last_touch = self.step
            rec.access_count += 1
            self._count("cold_to_warm", rec.nbytes)
            if self.row is not None:
                self.row.fetch_ops += 1
        self._evict_warm({id(r) for r in hit})
        if self.cold_dir is None:
            return hit
        # file-backed: the reference's return value, widened f32 (keys, values)
        return (np.concatenate([k for k, _ in payload]).astype(np.float32),
                np.concatenate([v for _, v in payload]).astype(np.float32))

    def promote_hot(self, layer: int, head: int, spans: Iterable[tuple[int, int]]) -> int:
        moved = 0
        keep: set[int] = set()
        for start, end in spans:
            for rec in self._covering(layer, head, start, end):
                if rec.tier == COLD:
                    raise ResidencyError(f"lane ({layer}, {head}): record at {rec.start} is cold; "
                                         "promote_hot needs it fetched")
                rec.last_touch = self.step
                keep.add(id(rec))
                if rec.tier == WARM:
                    self._move(rec, HOT)
                    moved += rec.nbytes
                    self._count("warm_to_hot", rec.nbytes)
        self._evict_hot(keep)
        self._evict_warm(keep)
        return moved

    def ensure_hot(self, layer: int, head: int, spans: Iterable[tuple[int, int]]) -> int:
        """Every record covering `spans` makes the trip to hot, one at a time (fetch if cold,
        then promote), so the warm tier never has to hold the whole working set."""
        order: list[ChunkRecord] = []
        seen: set[int] = set()
        for start, end in spans:
            for rec in self._covering(layer, head, start, end):
                if id(rec) not in seen:
                    seen.add(id(rec))
                    order.append(rec)
        moved = 0
        for rec in order:
            if rec.tier == COLD:
                self.fetch_chunk(layer, head, rec.start, rec.end)
            moved += self.promote_hot(layer, head, [(rec.start, rec.end)])
        return moved

    def _evict_hot(self, keep: set[int]) -> None:
        while self.used[HOT] > self.config.hot_capacity:
            pool = [r for r in self._all() if r.tier == HOT and id(r) not in keep]
            cand = [r for r in pool if not r.pinned] or pool  # pinned data may sit warm
            if not cand:
                raise CapacityError(f"hot budget {self.config.hot_capacity} B below this step's working set")
            victim = min(cand, key=ChunkRecord.order_key)
            self._move(victim, WARM)
            self._count("hot_to_warm", victim.nbytes)

    def _evict_warm(self, keep: set[int]) -> None:
        while self.used[WARM] > self.config.warm_capacity:
            pool = [r for r in self._all() if r.tier == WARM and id(r) not in keep and not r.pinned]
            cand = [r for r in pool if not self.frequency_exempt(r.layer, r.head, r.start, r.end)] or pool
            if not cand:
                raise CapacityError(f"warm budget {self.config.warm_capacity} B below this step's working set")
            self._move(min(cand, key=ChunkRecord.order_key), COLD)  # replica exists: no write

    def load_abstracts(self, layer: int, head: int):
        """Bill one summary per currently-cold record of the lane.  In-memory store: the
        decoder keeps every lane's abstracts resident in HBM, nothing moves, the cold spans
        are returned.  File-backed store: the lane's KVAB file is read and validated and the
        cold records' summaries are returned as ChunkAbstracts (tiered_store.py:390-408),
        ColdStoreError if one is missing."""
        spans = self.cold_spans(layer, head)
        if self.cold_dir is None:
            self._count("abstract_bytes", len(spans) * abstract_nbytes(self.head_dim))
            return spans
        if not spans:
            return []
        lane = CF.read_abstract_file(self.abstract_path(layer, head), self.head_dim)
        every = {(a.start, a.end): a for a in lane.as_chunk_abstracts()}  # validates each record
        missing = [sp for sp in spans if sp not in every]
        if missing:
            raise ColdStoreError(f"no summary record for cold chunk [{missing[0][0]}, {missing[0][1]}) in "
                                 f"{self.abstract_path(layer, head)}")
        self._count("abstract_bytes", len(spans) * abstract_nbytes(self.head_dim))
        return [every[sp] for sp in spans]

    def data_path(self, layer: int, head: int) -> Path:
        return CF.data_path(self.cold_dir, layer, head)

    def abstract_path(self, layer: int, head: int) -> Path:
        return CF.abstract_path(self.cold_dir, layer, head)

    # -- integrity (tiered_store.py:412-435) -------------------------------------------------
    def check_invariants(self) -> None:
        tot = {HOT: 0, WARM: 0}
        problems = []
        for lane, recs in self.lanes.items():
            problems += [f"{lane}: gap at {a.end}" for a, b in zip(recs, recs[1:]) if a.end != b.start]
            for r in recs:
                tot[r.tier] = tot.get(r.tier, 0) + r.nbytes
                if r.pinned and r.tier == COLD:
                    problems.append(f"{lane}: pinned record {r.start} is cold")
        tot.pop(COLD, None)
        if set(tot) != {HOT, WARM}:
            problems.append(f"unknown tiers {set(tot) - {HOT, WARM}}")
        if tot != self.used:
            problems.append(f"byte totals {self.used} != records {tot}")
        if tot.get(HOT, 0) > self.config.hot_capacity or tot.get(WARM, 0) > self.config.warm_capacity:
            problems.append("over budget")
        if problems:
            raise AssertionError("; ".join(problems))


def place_initial(*args, chunk_size: int = 64, spans_by_lane: dict | None = None,
                  on_move: Callable[[ChunkRecord, str, str], None] | None = None, **kw) -> TieredStore:
    """Initial residency (tiered_store.py:510-592): pinned early layers first, then the most
    recent tokens of every lane claim hot, then warm; the rest starts cold.  Pinned layers
    must fit in hot + warm.

    Two call forms:
      place_initial(trace, config, chunk_size=64, *, spans_by_lane=None)   -- the reference's;
          with config.cold_dir set, every non-pinned lane is written through to its KVCF/KVAB
          pair (byte-identical to the reference's files) and fetch_chunk / load_abstracts
          read them back;
      place_initial(n_layers, n_heads, head_dim, n_context, config, chunk_size=64, ...)
          -- bookkeeping only (the decoder holds the bytes in HBM / pinned host memory)."""
    trace = None
    if args and hasattr(args[0], "header"):
        if len(args) > 3:
            raise TypeError("place_initial(trace, config, chunk_size=64, *, spans_by_lane=None)")
        trace, config = args[0], (args[1] if len(args) > 1 else kw.pop("config", None))
        if len(args) > 2:
            chunk_size = args[2]
        h = trace.header
        n_layers, n_heads, head_dim, n_context = h.n_layers, h.n_heads, h.head_dim, h.n_context
    else:
        if len(args) not in (5, 6):
            raise TypeError("place_initial(n_layers, n_heads, head_dim, n_context, config, chunk_size=64, ...)")
        n_layers, n_heads, head_dim, n_context, config = args[:5]
        if len(args) > 5:
            chunk_size = args[5]
    if kw or config is None:
        raise TypeError(f"place_initial: unexpected arguments {sorted(kw)}" if kw else "place_initial: missing config")
    store = TieredStore(config, n_layers, n_heads, head_dim, on_move)
    files = trace is not None and config.cold_dir is not None
    if files:
        store.cold_dir = Path(config.cold_dir)
        store.cold_dir.mkdir(parents=True, exist_ok=True)
    every: list[ChunkRecord] = []
    for layer in range(n_layers):
        pinned = layer < config.early_layers_pinned
        for head in range(n_heads):
            spans = (spans_by_lane[(layer, head)] if spans_by_lane is not None else
                     [(s, min(s + chunk_size, n_context)) for s in range(0, n_context, chunk_size)])
            offs = [0] * len(spans)
            if files and not pinned:
                offs = CF.write_lane_files(store.data_path(layer, head), store.abstract_path(layer, head), spans,
                                           trace.keys[layer, head],
                                           None if trace.values is None else trace.values[layer, head], head_dim)
            recs = sorted((ChunkRecord(layer, head, s, e, kv_nbytes(e - s, head_dim), COLD, pinned, offset=o)
                           for (s, e), o in zip(spans, offs)), key=lambda r: r.start)
            store.lanes[(layer, head)] = recs
            every.extend(recs)
    if sum(r.nbytes for r in every if r.pinned) > config.hot_capacity + config.warm_capacity:
        raise CapacityError("the pinned early layers need more than hot + warm")
    room = {HOT: config.hot_capacity, WARM: config.warm_capacity}
    for rec in sorted(every, key=lambda r: (not r.pinned, -r.start, r.layer, r.head)):
        for tier in (HOT, WARM):
            if rec.nbytes <= room[tier]:
                room[tier] -= rec.nbytes
                rec.tier = tier
                break
        else:
            if rec.pinned:
                raise CapacityError(f"no room left for pinned record {rec.start} of layer {rec.layer}")
    store.used = {HOT: config.hot_capacity - room[HOT], WARM: config.warm_capacity - room[WARM]}
    store.check_invariants()
    return store
