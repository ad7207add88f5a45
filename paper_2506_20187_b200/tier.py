"""Host-tier streaming and the DTP compression split (north-star item 5; SURVEY §8(a) rows
12-13, §8(f) ranks 1-2).

Two parts:

* The latency model and theta solver of the reference (`pipeline.py:35-225`), restated as
  host arithmetic with the same names and semantics: for one layer with hot-link volume d,
  hiding requires  overhead + (d(1-theta) + d theta ratio)/bw <= compute + d theta/rate,
  linear in theta; `solve_theta` returns the smallest feasible theta; `build_schedule` lays
  out none / prefetch / dtp steps.  Here the parameters are MEASURED on the box
  (`HostTier.calibrate`): bw = pinned H2D copy rate, rate = K8 dequantisation rate,
  ratio = INT4 record bytes / bf16 row bytes (0.3125 at d = 128), compute = the layer's
  select + attend time.

* `HostTier`: KV chunks that live in pinned host memory (the "warm" tier of
  `tiered_store.py`), streamed to HBM on a side stream with `cudaMemcpyAsync`, split by
  theta: a theta fraction of the chunks crosses PCIe as INT4 records and is expanded on the
  device by `kvt_kv_dequant`, the rest as bf16 rows.  An event orders the transfer before
  the consuming layer's kernels, so transfer overlaps the previous layer's scoring.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple, Sequence

import torch

from . import _lib as L
from . import ops

MODES = ("none", "prefetch", "dtp")


@dataclass(frozen=True)
class PipelineParams:
    """pipeline.py:35-57."""

    compute_ms: float = 3.125
    overhead_ms: float = 0.0
    bw_hot_warm: float = 8.0
    bw_warm_cold: float = 2.0
    compress_ratio: float = 0.25
    decompress_rate: float = 32.0
    eval_ms_per_op: float = 1e-3

    def __post_init__(self) -> None:
        if self.compute_ms <= 0:
            raise ValueError("compute_ms must be positive")
        if self.overhead_ms < 0:
            raise ValueError("overhead_ms must be >= 0")
        if self.bw_hot_warm <= 0 or self.bw_warm_cold <= 0:
            raise ValueError("bandwidths must be positive")
        if not 0 < self.compress_ratio <= 1:
            raise ValueError("compress_ratio must be in (0, 1]")
        if self.decompress_rate <= 0:
            raise ValueError("decompress_rate must be positive")
        if self.eval_ms_per_op < 0:
            raise ValueError("eval_ms_per_op must be >= 0")


@dataclass(frozen=True)
class LayerLoad:
    """pipeline.py:60-70: bytes a layer moves this step, plus its evaluation time."""

    d_cold: float = 0.0
    d_warm: float = 0.0
    eval_ms: float = 0.0

    def __post_init__(self) -> None:
        if self.d_cold < 0 or self.d_warm < 0 or self.eval_ms < 0:
            raise ValueError("loads must be non-negative")


class ThetaSolution(NamedTuple):
    theta: float
    feasible: bool
    residual_ms: float


def solve_theta(d_bytes: float, params: PipelineParams, extra_overhead_ms: float = 0.0) -> ThetaSolution:
    """Smallest compressed fraction hiding the transfer inside compute (pipeline.py:79-103)."""
    if d_bytes < 0:
        raise ValueError("transfer volume must be >= 0")
    lead = params.overhead_ms + extra_overhead_ms
    gap = lead + d_bytes / params.bw_hot_warm - params.compute_ms
    if gap <= 0:
        return ThetaSolution(0.0, True, 0.0)
    if d_bytes == 0 or params.compress_ratio == 1.0:
        return ThetaSolution(0.0, False, gap)
    gain = d_bytes * (1.0 - params.compress_ratio) / params.bw_hot_warm + d_bytes / params.decompress_rate
    theta = gap / gain
    if theta > 1.0:
        return ThetaSolution(1.0, False, gap - gain)
    return ThetaSolution(theta, True, 0.0)


@dataclass(frozen=True)
class LayerTiming:
    layer: int
    eval: tuple[float, float]
    cold: tuple[float, float]
    warm: tuple[float, float]
    decompress: tuple[float, float]
    compute: tuple[float, float]
    theta: float
    idle_ms: float

    @property
    def gpu_end(self) -> float:
        return self.compute[1]

    eval_ms = property(lambda self: self.eval[1] - self.eval[0])
    cold_ms = property(lambda self: self.cold[1] - self.cold[0])
    warm_ms = property(lambda self: self.warm[1] - self.warm[0])
    decompress_ms = property(lambda self: self.decompress[1] - self.decompress[0])
    compute_ms = property(lambda self: self.compute[1] - self.compute[0])


@dataclass(frozen=True)
class StepSchedule:
    mode: str
    layers: tuple[LayerTiming, ...]
    total_ms: float

    @property
    def idle_ms(self) -> float:
        return sum(t.idle_ms for t in self.layers)

    def layer_latencies(self) -> list[float]:
        out, prev = [], 0.0
        for t in self.layers:
            out.append(t.gpu_end - prev)
            prev = t.gpu_end
        return out


def _durations(load: LayerLoad, p: PipelineParams, theta: float):
    ev = load.eval_ms + p.overhead_ms
    cold = load.d_cold / p.bw_warm_cold if load.d_cold else 0.0
    warm = load.d_warm * (1.0 - theta * (1.0 - p.compress_ratio)) / p.bw_hot_warm if load.d_warm else 0.0
    dec = load.d_warm * theta / p.decompress_rate if theta else 0.0
    return ev, cold, warm, dec


def build_schedule(loads: Sequence[LayerLoad], params: PipelineParams, mode: str) -> StepSchedule:
    """One step's intervals under none / prefetch / dtp (pipeline.py:172-225)."""
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}; expected one of {MODES}")
    if not loads:
        raise ValueError("need at least one layer load")
    out = []
    lane_free = gpu_free = 0.0
    for li, load in enumerate(loads):
        if mode == "none":
            lane_free = gpu_free
        if mode == "dtp":
            _, cold0, _, _ = _durations(load, params, 0.0)
            th = solve_theta(load.d_warm, params, extra_overhead_ms=load.eval_ms + cold0).theta
            thetas = sorted({0.0, th})
        else:
            thetas = [0.0]
        best = None
        for th in thetas:
            ev, cold, warm, dec = _durations(load, params, th)
            lane_end = lane_free + ev + cold + warm
            gpu_start = max(gpu_free, lane_end)
            gpu_end = gpu_start + dec + params.compute_ms
            key = (gpu_end, lane_end, th)
            if best is None or key < best[0]:
                best = (key, th, ev, cold, warm, dec, lane_end, gpu_start, gpu_end)
        _, th, ev, cold, warm, dec, lane_end, gpu_start, gpu_end = best
        t_ev = (lane_free, lane_free + ev)
        t_cold = (t_ev[1], t_ev[1] + cold)
        t_warm = (t_cold[1], t_cold[1] + warm)
        t_dec = (gpu_start, gpu_start + dec)
        out.append(LayerTiming(li, t_ev, t_cold, t_warm, t_dec, (t_dec[1], t_dec[1] + params.compute_ms), th,
                               gpu_start - gpu_free))
        lane_free, gpu_free = lane_end, gpu_end
    return StepSchedule(mode=mode, layers=tuple(out), total_ms=gpu_free)


SCHEDULE_COLUMNS = ("step", "layer", "mode", "eval_ms", "cold_ms", "warm_ms", "compute_ms", "decompress_ms",
                    "theta", "idle_ms")


def schedule_rows(step: int, schedule: StepSchedule) -> list[list]:
    """schedule.csv rows (pipeline.py:244-276)."""
    return [[step, t.layer, schedule.mode] + [str(v) for v in (t.eval_ms, t.cold_ms, t.warm_ms, t.compute_ms,
                                                                 t.decompress_ms, t.theta, t.idle_ms)]
            for t in schedule.layers]


def compare_modes(loads: Sequence[LayerLoad], params: PipelineParams) -> dict[str, float]:
    return {m: build_schedule(loads, params, m).total_ms for m in MODES}


# ------------------------------------------------------------------------------------------------
# pinned host tier
# ------------------------------------------------------------------------------------------------


def kv_dequant(src: "ops.I4KV", dst: torch.Tensor, t_begin: int = 0, t_end: int | None = None) -> torch.Tensor:
    """Expand INT4 records rows [t_begin, t_end) into bf16/f32/f16 rows of dst (kvt_kv_dequant)."""
    ls_d, d = ops._lanes(dst)
    t_end = src.shape[1] if t_end is None else t_end
    L.check(L.kvt_kv_dequant(src.data_ptr(), src.stride(0), src.shape[0], t_begin, t_end, d, dst.data_ptr(),
                             ops.dtype_code(dst), ls_d, ops._stream()), "kv_dequant")
    return dst


class HostTier:
    """Chunks of one layer's KV held in pinned host memory, streamed into an HBM cache.

    host_raw: bf16 [lanes, N, d] pinned; host_i4: INT4 records [lanes, N, rb] pinned (built
    once with K8 on the device and copied down).  `stream(ranges, theta)` copies the token
    ranges [(s, e), ...] of every lane into `dst` (bf16 [lanes, N_cap, d] in HBM) on the
    tier's side stream and returns the CUDA event the consumer must wait on.
    """

    def __init__(self, keys_bf16: torch.Tensor, device=None):
        if keys_bf16.dtype != torch.bfloat16 or keys_bf16.dim() != 3:
            raise ValueError("HostTier holds bf16 [lanes, N, d] rows")
        dev = torch.device(device or "cuda")
        self.lanes, self.n, self.d = keys_bf16.shape
        self.host_raw = keys_bf16.cpu().pin_memory()
        tmp = ops.I4KV.empty(self.lanes, self.n, self.d, dev)
        ops.kv_quant(keys_bf16.to(dev), tmp)
        self.host_i4 = tmp.data.cpu().pin_memory()
        self.rb = ops.row_bytes_i4(self.d)
        self.stream_ = torch.cuda.Stream(device=dev)
        self.stage = None
        self.device = dev

    def _stage(self, rows: int) -> "ops.I4KV":
        if self.stage is None or self.stage.shape[1] < rows:
            self.stage = ops.I4KV.empty(self.lanes, rows, self.d, self.device)
        return self.stage

    def stream(self, dst: torch.Tensor, ranges: list[tuple[int, int]], theta: float) -> torch.cuda.Event:
        """Copy `ranges` of every lane into dst; the first ceil(theta * chunks) ranges go as
        INT4 records (+ on-device dequant), the rest as bf16.  Returns the completion event."""
        n_comp = int(math.ceil(theta * len(ranges) - 1e-12))
        ev = torch.cuda.Event()
        # the side stream must not overwrite dst (or the stage) while the consumer stream still
        # reads them: it starts after the consumer's queued work
        self.stream_.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream_):
            comp = ranges[:n_comp]
            if comp:
                rows = sum(e - s for s, e in comp)
                st = self._stage(rows)
                pos = 0
                for s, e in comp:
                    # per lane: [s, e) of one lane is contiguous in the pinned [lanes, N, row]
                    # buffer, so every copy is a true async DMA (a [:, s:e] slice is strided and
                    # would be staged through pageable memory)
                    for ln in range(self.lanes):
                        st.data[ln, pos:pos + e - s].copy_(self.host_i4[ln, s:e], non_blocking=True)
                    pos += e - s
                pos = 0
                for s, e in comp:
                    kv_dequant(ops.I4KV(st.data[:, pos:pos + e - s], self.d), dst[:, s:e])
                    pos += e - s
            for s, e in ranges[n_comp:]:
                for ln in range(self.lanes):
                    dst[ln, s:e].copy_(self.host_raw[ln, s:e], non_blocking=True)
            ev.record(self.stream_)
        dst.record_stream(self.stream_)
        return ev

    def calibrate(self, dst: torch.Tensor, chunk: int = 64, n_chunks: int = 256) -> dict:
        """Measure H2D bf16 rate, INT4 H2D + dequant rate on this box -> PipelineParams fields
        (bytes per ms, as the reference's model uses)."""
        n_chunks = min(n_chunks, self.n // chunk)
        ranges = [(i * chunk, (i + 1) * chunk) for i in range(n_chunks)]
        raw_bytes = self.lanes * n_chunks * chunk * self.d * 2
        out = {}
        for name, th in (("raw", 0.0), ("int4", 1.0)):
            self.stream(dst, ranges, th).synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.stream_)
            self.stream(dst, ranges, th)
            e1.record(self.stream_)
            e1.synchronize()
            out[name] = e0.elapsed_time(e1)
        bw = raw_bytes / out["raw"]                      # bytes per ms over the host link
        eff = raw_bytes / out["int4"]                    # original bytes per ms, compressed path
        ratio = self.rb / (2.0 * self.d)
        # compressed path time = ratio*raw/bw + raw/rate  ->  rate
        t_dec = out["int4"] - ratio * raw_bytes / bw
        rate = raw_bytes / t_dec if t_dec > 0 else float("inf")
        return {"bw_hot_warm": bw, "compress_ratio": ratio, "decompress_rate": rate,
                "raw_ms": out["raw"], "int4_ms": out["int4"], "bytes": raw_bytes, "int4_effective": eff}
