"""Tiered values for the batched decoder: an HBM hot tier of V records over a pinned-host warm
tier, moved by the GPU itself (north-star item 5).

The reference keeps every record's bytes in a tier and moves whole placement records with
TieredStore.touch / ensure_hot / promote_hot, evicting the least recently touched record,
ordered (last_touch, start, layer, head) (tiered_store.py:224-372), once per lane from
engine.py:342-343; pipeline.py:79-103 sizes the compressed share theta of the warm -> hot
bytes so the transfer hides behind compute.  Here:

* the WARM tier is pinned host memory holding every V record of every layer (INT4 records,
  plus, optionally, the raw bf16 rows for the uncompressed share of the theta split);
* the HOT tier is a pool of record slots in HBM, shared by all layers and lanes (the
  reference's single hot budget), addressed through a record table;
* per (step, layer), after the selection, kvt_tier_layer touches the records the selected
  runs overlap, evicts exactly the records the reference would (LRU by (stamp, start, layer,
  lane), on the device: no host round trip), copies the misses host -> HBM over the host link
  (INT4 as stored, or raw bf16 quantised on the way) and counts the ledger row;
* K7 reads V through the table (kvt_sparse_decode_attn_paged).

TieredDecoder.step pipelines the layers on two streams: the tier work of layer l runs on a
side stream while the main stream selects layer l + 1, and layer l's attention waits for its
records (event join).  The step's queries are all known up front (the trace-driven
engine.run and bench.py), which is what makes that overlap legal.  K and the abstracts stay
resident: every step scores ~35 % of the tokens against K, while V is read only at the ~10 %
selected ones.
"""

from __future__ import annotations

import ctypes
import math

import torch

from . import _lib as L
from . import ops
from .decode import SparseDecoder
from .tier import PipelineParams, solve_theta
from .tiered_store import CapacityError, kv_nbytes


def theta_for_rows(rows: list[dict], params: PipelineParams, crec: int, d: int) -> list[float]:
    """DTP controller (pipeline.py:79-103): per layer, the smallest compressed share theta that
    hides the layer's warm -> hot transfer behind its compute, with the raw volume taken from
    the previous step's ledger row (promotions x raw bf16 record bytes)."""
    raw_rec = crec * d * 2
    return [solve_theta(r["promotions"] * raw_rec, params).theta for r in rows]


class HotTier:
    """HBM hot tier (pool + record table + LRU state) over pinned host V records."""

    def __init__(self, n_layers: int, kv_lanes: int, n_cap: int, d: int, n_slots: int, crec: int = 64,
                 device=None, keep_raw: bool = False):
        if d not in (128, 256):
            raise ValueError("the hot tier holds INT4 records of d = 128 or 256")
        self.L, self.kv_lanes, self.n_cap, self.d, self.crec = n_layers, kv_lanes, n_cap, d, crec
        self.n_rec = -(-n_cap // crec)
        if self.n_rec * n_layers * kv_lanes > (1 << 26):
            raise ValueError("more than 2^26 records: the eviction key field is 26 bits")
        self.n_slots = int(n_slots)
        if not 0 < self.n_slots < 2 ** 31:
            raise ValueError("n_slots out of range")
        dev = torch.device(device or "cuda")
        self.device = dev
        self.rb = ops.row_bytes_i4(d)
        i32, i64 = torch.int32, torch.int64
        self.table = torch.full((n_layers, kv_lanes, self.n_rec), -1, dtype=i32, device=dev)
        self.owner = torch.full((self.n_slots,), -1, dtype=i64, device=dev)
        self.stamp = torch.full((self.n_slots,), -1, dtype=i32, device=dev)
        self.free_stack = torch.arange(self.n_slots, dtype=i32, device=dev)
        self.free_top = torch.tensor([self.n_slots], dtype=i32, device=dev)
        self.miss_cap = kv_lanes * self.n_rec
        self.miss = torch.empty(self.miss_cap, dtype=i64, device=dev)
        self.victims = torch.empty(self.miss_cap, dtype=i32, device=dev)
        self.slot_of_miss = torch.empty(self.miss_cap, dtype=i32, device=dev)
        self.ctl = torch.zeros(L.kvt_tier_ctl_bytes(), dtype=torch.uint8, device=dev)
        self.pool = torch.empty((self.n_slots, crec, self.rb), dtype=torch.uint8, device=dev)
        self.step_dev = torch.zeros(1, dtype=i32, device=dev)
        self.theta = torch.ones(n_layers, dtype=torch.float32, device=dev)
        self.ledger = torch.zeros((n_layers, 4), dtype=i64, device=dev)
        # warm tier: pinned host rows, [L][kv_lanes][N][row]
        self.host_i4 = torch.empty((n_layers, kv_lanes, n_cap, self.rb), dtype=torch.uint8, pin_memory=True)
        self.host_raw = (torch.empty((n_layers, kv_lanes, n_cap, d), dtype=torch.bfloat16, pin_memory=True)
                         if keep_raw else None)
        self.ledger_rec_bytes = kv_nbytes(crec, d)  # the reference's byte model (K + V fp16)
        self.phys_rec_bytes = crec * self.rb        # what actually crosses the link (INT4)

    # -- warm tier contents ---------------------------------------------------------------------

    def write_layer(self, layer: int, v: torch.Tensor, t0: int = 0) -> None:
        """Rows [t0, t0 + T) of one layer's values ([kv_lanes, T, d] on the device) -> the
        pinned host tier (INT4 via K8 on the device; raw bf16 too when kept)."""
        T = v.shape[1]
        tmp = ops.I4KV.empty(self.kv_lanes, T, self.d, v.device)
        ops.kv_quant(v, tmp)
        self.host_i4[layer, :, t0:t0 + T].copy_(tmp.data)
        if self.host_raw is not None:
            self.host_raw[layer, :, t0:t0 + T].copy_(v.to(torch.bfloat16))

    # -- per (step, layer) ----------------------------------------------------------------------

    def layer(self, layer: int, bufs: dict, n_lanes: int, kv_group: int = 1) -> None:
        """kvt_tier_layer on the current stream: touch / evict / fetch for layer `layer`'s runs."""
        a = L.KvtTierArgs()
        a.n_lanes, a.kv_group, a.d, a.crec = n_lanes, kv_group, self.d, self.crec
        a.step = self.step_dev.data_ptr()
        a.run_start, a.run_len, a.n_runs = (bufs["run_start"].data_ptr(), bufs["run_len"].data_ptr(),
                                            bufs["n_runs"].data_ptr())
        a.run_stride = bufs["run_start"].stride(0)
        a.table = self.table.data_ptr()
        a.table_base = layer * self.kv_lanes * self.n_rec
        a.table_stride, a.n_lk = self.n_rec, self.L * self.kv_lanes
        a.stamp, a.owner, a.n_slots = self.stamp.data_ptr(), self.owner.data_ptr(), self.n_slots
        a.free_stack, a.free_top = self.free_stack.data_ptr(), self.free_top.data_ptr()
        a.victims, a.slot_of_miss = self.victims.data_ptr(), self.slot_of_miss.data_ptr()
        a.miss, a.miss_cap = self.miss.data_ptr(), self.miss_cap
        a.ctl, a.pool = self.ctl.data_ptr(), self.pool.data_ptr()
        a.host_i4 = self.host_i4[layer].data_ptr()
        a.host_raw = None if self.host_raw is None else self.host_raw[layer].data_ptr()
        a.host_lane_tokens, a.n_tok = self.n_cap, self.n_cap
        a.theta = self.theta[layer:layer + 1].data_ptr()
        a.ledger_rec_bytes = self.ledger_rec_bytes
        a.ledger_row = self.ledger[layer].data_ptr()
        L.check(L.kvt_tier_layer(a, ops._stream()), "tier_layer")

    def attend(self, layer: int, bufs: dict, out: torch.Tensor, ws: ops.LayerWorkspace, kv_group: int = 1) -> None:
        """K7 over the hot tier for layer `layer` (every selected record is hot after layer())."""
        n_lanes = bufs["sel_tok"].shape[0]
        old = L.kvt_set_kv_group(kv_group)
        try:
            L.check(L.kvt_sparse_decode_attn_paged(
                self.pool.data_ptr(), self.table[layer].data_ptr(), self.n_rec, self.crec, n_lanes, self.d,
                bufs["sel_tok"].data_ptr(), bufs["sel_score"].data_ptr(), bufs["n_sel"].data_ptr(),
                bufs["sel_tok"].stride(0), 1.0 / math.sqrt(self.d), 0, ws.buf.data_ptr(), out.data_ptr(), None,
                ops._stream()), "sparse_decode_attn_paged")
        finally:
            L.kvt_set_kv_group(old)

    def reset(self) -> None:
        """Every record back to warm only (empty pool); the step counter is kept."""
        self.table.fill_(-1)
        self.owner.fill_(-1)
        self.stamp.fill_(-1)
        torch.arange(self.n_slots, dtype=torch.int32, device=self.device, out=self.free_stack)
        self.free_top.fill_(self.n_slots)

    def last_call(self) -> dict:
        """State of the last kvt_tier_layer call (synchronises; diagnostics)."""
        buf = (ctypes.c_longlong * 4)()
        L.check(L.kvt_tier_read_ctl(self.ctl.data_ptr(), buf, ops._stream()), "tier_read_ctl")
        return {"misses": buf[0], "evictions": buf[1], "need": buf[2], "victims": buf[3]}

    def hot_records(self) -> set[tuple[int, int, int]]:
        """(layer, kv lane, record) of every hot record (host copy; synchronises)."""
        own = self.owner.cpu()
        out = set()
        for i in own[own >= 0].tolist():
            lk, rec = divmod(i, self.n_rec)
            layer, lane = divmod(lk, self.kv_lanes)
            out.add((layer, lane, rec))
        return out


class TieredDecoder(SparseDecoder):
    """SparseDecoder whose values live in a HotTier: K, abstracts and the selection as before,
    V records served from an HBM pool of `hot_records` slots backed by pinned host memory."""

    def __init__(self, n_layers: int, batch: int, n_heads: int, head_dim: int, n_cap: int, hot_records: int,
                 dtype=ops.I4, crec: int = 64, keep_raw: bool = False, device=None, **kw):
        super().__init__(n_layers, batch, n_heads, head_dim, n_cap, dtype=dtype, device=device, values="tiered", **kw)
        self.tier = HotTier(n_layers, self.kv_lanes, n_cap, head_dim, hot_records, crec, self.device, keep_raw)
        self.side = torch.cuda.Stream(device=self.device)
        self.ev_sel = [torch.cuda.Event() for _ in range(n_layers)]
        self.ev_tier = [torch.cuda.Event() for _ in range(n_layers)]
        self.steps_done = 0

    def load_layer(self, layer: int, k: torch.Tensor, v: torch.Tensor, t0: int = 0) -> None:
        super().load_layer(layer, k, v, t0)
        self.tier.write_layer(layer, v, t0)

    def append(self, k_new: torch.Tensor, v_new: torch.Tensor) -> None:
        raise NotImplementedError("tiered values: append rows with load_layer(layer, k, v, t0) + set_length")

    def set_theta(self, theta) -> None:
        """Per-layer compressed share of the misses (tier.solve_theta); needs keep_raw for < 1."""
        th = torch.as_tensor(theta, dtype=torch.float32).reshape(-1).expand(self.L)
        if (th < 1).any() and self.tier.host_raw is None:
            raise ValueError("theta < 1 needs the raw host copy (keep_raw=True)")
        self.tier.theta.copy_(th)

    def plan_theta(self, params: PipelineParams, rows: list[dict] | None = None) -> list[float]:
        """Set every layer's theta from the last step's ledger rows (theta_for_rows) and return it.
        Without the raw host copy every transfer is INT4 already (theta = 1)."""
        if self.tier.host_raw is None:
            th = [1.0] * self.L
        else:
            th = theta_for_rows(rows if rows is not None else self.ledger_rows(), params, self.tier.crec, self.d)
        self.set_theta(th)
        return th

    def step(self, q: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """All layers of one decode step; q: [L, lanes, d] -> [L, lanes, d] f32.  Layer l's
        tier work (side stream) overlaps layer l + 1's selection (main stream)."""
        if out is None:
            out = torch.empty((self.L, self.lanes, self.d), dtype=torch.float32, device=self.device)
        bufs = self._buffers()
        main = torch.cuda.current_stream(self.device)
        self.tier.ledger.zero_()
        for l in range(self.L):
            self.layer(l, q[l], attend=False)
            self.ev_sel[l].record(main)
            with torch.cuda.stream(self.side):
                self.side.wait_event(self.ev_sel[l])
                self.tier.layer(l, bufs[l], self.lanes, self.kv_group)
                self.ev_tier[l].record(self.side)
            if l > 0:
                main.wait_event(self.ev_tier[l - 1])
                self.tier.attend(l - 1, bufs[l - 1], out[l - 1], self._ws, self.kv_group)
        main.wait_event(self.ev_tier[self.L - 1])
        self.tier.attend(self.L - 1, bufs[self.L - 1], out[self.L - 1], self._ws, self.kv_group)
        self.tier.step_dev.add_(1)
        self.steps_done += 1
        return out

    def ledger_rows(self) -> list[dict]:
        """This step's ledger rows (after step(); synchronises): per layer warm_to_hot /
        hot_to_warm bytes in the reference's byte model, promotions, and the physical INT4
        bytes that crossed the host link."""
        lg = self.tier.ledger.cpu().tolist()
        rows = []
        for l, (w2h, h2w, ops_, st) in enumerate(lg):
            if st == -1:
                raise CapacityError(f"hot tier smaller than the working set of layer {l}")
            rows.append({"layer": l, "warm_to_hot": w2h, "hot_to_warm": h2w, "promotions": ops_,
                         "link_bytes": ops_ * self.tier.phys_rec_bytes})
        return rows
