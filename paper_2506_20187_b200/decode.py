"""Batched decode-step API: a resident KV cache with per-layer chunk abstracts and the
fused per-layer select + sparse-attend pipeline (the body of engine.run's lane loop,
engine.py:307-357, for every (batch row, head) lane of a layer at once).

Layout in HBM:
  K, V       [L][B*H][N_cap][d]   key/value rows, lanes contiguous (bf16 by default)
  amax/amin  per layer [B*H][ceil(N_cap/C_l)][d] bf16 chunk abstracts rounded outward
             (importance.py:56-87 summaries; exact f32 on request)
  absmag     per layer [B*H][d] f32 max |key| over the lane's chunks (bf16 abstracts only):
             enables the directed-rounding f32 bounds (bounds_fast.cu) in select_attend
  coarse     layers whose plan chunk C_l is finer than default_chunk_size also keep C = 64
             abstracts; adapt_bound_granularity() switches a layer's pruning to them when its
             observed candidate fraction shows the fine bounds prune nothing (layers 0-1 at
             rate 0.5).  The selected set is exact either way; only bound bytes change.
  C_l        ChunkPlanConfig: early layers use early_chunk_size, the rest default_chunk_size
             (chunk_tree.py:111-123, steady state after the early steps)
  k_l        ceil(rate_l * n), rate 0.5 for layers < early_layers else 0.1 (engine.py:83-86,312)
"""

from __future__ import annotations

import math
import os

import torch

from . import ops
from .chunk_tree import ChunkPlanConfig


class SparseDecoder:
    def __init__(self, n_layers: int, batch: int, n_heads: int, head_dim: int, n_cap: int,
                 dtype: torch.dtype = torch.bfloat16, plan: ChunkPlanConfig | None = None,
                 importance_rate: float = 0.10, early_layer_rate: float = 0.50, device=None,
                 abstract_dtype: torch.dtype = torch.bfloat16, n_kv_heads: int | None = None,
                 values: str = "resident"):
        if not torch.cuda.is_available():
            raise RuntimeError("SparseDecoder needs a CUDA device (B200, sm_100a)")
        self.L, self.B, self.H, self.d = n_layers, batch, n_heads, head_dim
        self.lanes = batch * n_heads  # query lanes
        self.Hkv = n_kv_heads or n_heads
        if n_heads % self.Hkv:
            raise ValueError("n_heads must be a multiple of n_kv_heads")
        self.kv_group = n_heads // self.Hkv  # GQA: query heads per KV head (adjacent)
        self.kv_lanes = batch * self.Hkv
        self.n_cap = n_cap
        self.dtype = dtype
        self.plan = plan or ChunkPlanConfig()
        self.rates = [early_layer_rate if l < self.plan.early_layers else importance_rate for l in range(n_layers)]
        self.C = [self.plan.early_chunk_size if l < self.plan.early_layers else self.plan.default_chunk_size
                  for l in range(n_layers)]
        self.device = torch.device(device or "cuda")
        if values not in ("resident", "tiered"):
            raise ValueError("values must be 'resident' or 'tiered'")
        # values="tiered": V lives in a host_tier.HotTier (HBM hot records over pinned host
        # memory); the decoder keeps K and the abstracts and runs the selection only
        if dtype == ops.I4:  # INT4 records (K8), 0.3125x of bf16 at d = 128
            self.K = ops.I4KV(torch.empty((n_layers, self.kv_lanes, n_cap, ops.row_bytes_i4(head_dim)),
                                          dtype=torch.uint8, device=self.device), head_dim)
            self.V = ops.I4KV(torch.empty_like(self.K.data), head_dim) if values == "resident" else None
        else:
            self.K = torch.empty((n_layers, self.kv_lanes, n_cap, head_dim), dtype=dtype, device=self.device)
            self.V = torch.empty_like(self.K) if values == "resident" else None
        # bf16 abstracts rounded outward (max up, min down): half the bound-pass bytes, still sound
        adt = abstract_dtype if abstract_dtype is not None else ops.abs_dtype_for(dtype)
        self.amax = [torch.empty((self.kv_lanes, ops.n_grid_leaves(n_cap, C), head_dim), dtype=adt,
                                 device=self.device) for C in self.C]
        self.amin = [torch.empty_like(a) for a in self.amax]
        self.absmag = ([torch.zeros((self.kv_lanes, head_dim), dtype=torch.float32, device=self.device)
                        for _ in range(n_layers)] if adt == torch.bfloat16 else None)
        if self.kv_group > 1 and self.absmag is None:
            raise ValueError("GQA sharing needs bf16 abstracts (the decode-path bounds)")
        self.coarse_C = self.plan.default_chunk_size
        self.amax_c = [torch.empty((self.kv_lanes, ops.n_grid_leaves(n_cap, self.coarse_C), head_dim), dtype=adt,
                                   device=self.device) if C < self.coarse_C and self.absmag is not None else None
                       for C in self.C]
        self.amin_c = [None if a is None else torch.empty_like(a) for a in self.amax_c]
        self.use_coarse = [False] * n_layers
        self.grid_C = list(self.C)      # chunk size each layer prunes on (adapt_chunking)
        self._mid = {}                  # (layer, C) -> intermediate-grid abstracts (K2 from the fine grid)
        self.rho_measured = [None] * n_layers
        self.n = 0
        self._ws = None
        self._bufs = None

    # -- cache maintenance ------------------------------------------------------------------------

    def set_length(self, n: int) -> None:
        """Declare K/V[:, :, :n] filled (prefill) and (re)build every chunk abstract (K1)."""
        if n > self.n_cap:
            raise ValueError("n exceeds cache capacity")
        self.n = n
        for l in range(self.L):
            ops.abstract_build(self.K[l], n, self.C[l], self.amax[l], self.amin[l])
            if self.absmag is not None:
                ops.lane_abs_mag(self.amax[l], self.amin[l], ops.n_grid_leaves(n, self.C[l]), out=self.absmag[l])
            if self.amax_c[l] is not None:  # K2: the coarse grid from the fine one, keys not re-read
                ops.abstract_merge(self.amax[l], self.amin[l], factor=self.coarse_C // self.C[l],
                                   m_in=ops.n_grid_leaves(n, self.C[l]), out=(self.amax_c[l], self.amin_c[l]))
        for (l, C), (mx, mn) in self._mid.items():
            ops.abstract_merge(self.amax[l], self.amin[l], factor=C // self.C[l],
                               m_in=ops.n_grid_leaves(n, self.C[l]), out=(mx, mn))
        self._bufs = None

    def load_layer(self, layer: int, k: torch.Tensor, v: torch.Tensor, t0: int = 0) -> None:
        """Write rows [t0, t0 + T) of one layer from [kv_lanes, T, d] tensors (quantising for INT4)."""
        T = k.shape[1]
        if self.dtype == ops.I4:
            ops.kv_quant(k, ops.I4KV(self.K.data[layer, :, t0:t0 + T], self.d))
            if self.V is not None:
                ops.kv_quant(v, ops.I4KV(self.V.data[layer, :, t0:t0 + T], self.d))
        else:
            self.K[layer, :, t0:t0 + T] = k.to(self.dtype)
            if self.V is not None:
                self.V[layer, :, t0:t0 + T] = v.to(self.dtype)

    def _append_tables(self):
        """Device tables of kvt_kv_append: every bf16 abstract grid (fine, coarse, intermediate)
        and the per-layer absmag pointers; rebuilt when the set of grids changes."""
        key = tuple(sorted(self._mid))
        if getattr(self, "_app_key", None) == key:
            return self._app_grids, self._app_n, self._app_mag
        import numpy as np
        rows = []
        for l in range(self.L):
            grids = [(self.amax[l], self.amin[l], self.C[l])]
            if self.amax_c[l] is not None:
                grids.append((self.amax_c[l], self.amin_c[l], self.coarse_C))
            grids += [(mx, mn, C) for (ll, C), (mx, mn) in self._mid.items() if ll == l]
            rows += [(mx.data_ptr(), mn.data_ptr(), mx.stride(0), C, l) for mx, mn, C in grids]
        dt = np.dtype([("amax", "<u8"), ("amin", "<u8"), ("ls", "<i8"), ("C", "<i4"), ("layer", "<i4")])
        tab = np.array(rows, dtype=dt)
        self._app_grids = torch.from_numpy(tab.view(np.uint8).copy()).to(self.device)
        self._app_n = len(rows)
        self._app_mag = torch.tensor([a.data_ptr() for a in self.absmag], dtype=torch.int64, device=self.device)
        self._app_key = key
        return self._app_grids, self._app_n, self._app_mag

    def append(self, k_new: torch.Tensor, v_new: torch.Tensor, fused: bool = True) -> None:
        """Append one token per KV lane ([L, kv_lanes, d]) and refresh the tail chunk abstracts.
        INT4 KV with bf16 abstracts at d = 128: one kvt_kv_append launch for every layer and
        lane (quantise + abstract / absmag refresh); otherwise per-layer launches."""
        if self.n >= self.n_cap:
            raise ValueError("cache full")
        if (fused and self.dtype == ops.I4 and self.absmag is not None and self.d == 128 and self.V is not None
                and k_new.dtype in (torch.bfloat16, torch.float32) and v_new.dtype == k_new.dtype):
            k_new, v_new = k_new.contiguous(), v_new.contiguous()
            grids, ng, mag = self._append_tables()
            ops.L.check(ops.L.kvt_kv_append(
                k_new.data_ptr(), v_new.data_ptr(), ops.dtype_code(k_new), k_new.stride(0), k_new.stride(1), self.L,
                self.kv_lanes, self.d, self.n, self.K.data.data_ptr(), self.V.data.data_ptr(), self.K.data.stride(0),
                self.K.data.stride(1), grids.data_ptr(), ng, mag.data_ptr(), ops._stream()), "kv_append")
            self.n += 1
            self._bufs = None
            return
        for l in range(self.L):
            self.load_layer(l, k_new[l][:, None, :].contiguous(), v_new[l][:, None, :].contiguous(), self.n)
        self.n += 1
        for l in range(self.L):
            c = (self.n - 1) // self.C[l]
            ops.abstract_build(self.K[l], self.n, self.C[l], self.amax[l], self.amin[l], c, c + 1)
            if self.absmag is not None:  # the refreshed tail chunk can only raise the maxima
                tail = torch.maximum(self.amax[l][:, c].float().abs(), self.amin[l][:, c].float().abs())
                torch.maximum(self.absmag[l], tail, out=self.absmag[l])
            if self.amax_c[l] is not None:
                cc = (self.n - 1) // self.coarse_C
                ops.abstract_build(self.K[l], self.n, self.coarse_C, self.amax_c[l], self.amin_c[l], cc, cc + 1)
        for (l, C), (mx, mn) in self._mid.items():  # the tail chunk of every intermediate grid (K2)
            f = C // self.C[l]
            cc = (self.n - 1) // C
            m_in = ops.n_grid_leaves(self.n, self.C[l])
            lanes = torch.arange(self.kv_lanes, dtype=torch.int32)
            tmx, tmn = ops.abstract_merge(self.amax[l], self.amin[l], seg_lane=lanes,
                                          seg_begin=torch.full_like(lanes, cc * f),
                                          seg_end=torch.full_like(lanes, min(m_in, cc * f + f)))
            mx[:, cc] = tmx
            mn[:, cc] = tmn
        self._bufs = None

    def grid(self, l: int):
        """(C, amax, amin) the layer's pruning runs on: the plan chunk, or the size adapt_chunking
        chose (intermediate sizes are K2 merges of the fine abstracts)."""
        C = self.grid_C[l]
        if C == self.C[l]:
            return C, self.amax[l], self.amin[l]
        if C == self.coarse_C and self.amax_c[l] is not None:
            return C, self.amax_c[l], self.amin_c[l]
        mx, mn = self._mid[(l, C)]
        return C, mx, mn

    def _ensure_grid(self, l: int, C: int) -> None:
        if C in (self.C[l], self.coarse_C) or (l, C) in self._mid:
            return
        mx = torch.empty((self.kv_lanes, ops.n_grid_leaves(self.n_cap, C), self.d), dtype=self.amax[l].dtype,
                         device=self.device)
        mn = torch.empty_like(mx)
        ops.abstract_merge(self.amax[l], self.amin[l], factor=C // self.C[l], m_in=ops.n_grid_leaves(self.n, self.C[l]),
                           out=(mx, mn))
        self._mid[(l, C)] = (mx, mn)

    def adapt_chunking(self, margin: float = 0.1) -> list[int]:
        """Adaptive chunk sizing from the last step's selection (outside graph capture: it reads
        the step's counters).  For every layer whose plan chunk is finer than default_chunk_size
        (chunk_tree.py:111-123: early layers at 8), the live chunks of its selected runs at every
        size C = C_l .. 64 (kvt_live_chunks: the skew of the layer's attention weights) give the
        expected candidate tokens of each grid, infl * live(C) * C, with infl measured on the
        current grid; the layer prunes on the grid with the fewest bound + candidate bytes
        (switching only for a > margin gain).  The reference's importance density rho (the
        fraction of a live chunk's halves that stay live, averaged over the levels) is recorded
        in rho_measured.  Returns the chunk size per layer."""
        bufs = self._buffers()
        sA = self.amax[0].element_size()
        rowK = ops.row_bytes_i4(self.d) if self.dtype == ops.I4 else self.d * self.K.element_size()
        for l in range(self.L):
            if self.amax_c[l] is None:
                continue
            sizes = []
            c = self.C[l]
            while c <= self.coarse_C:
                sizes.append(c)
                c *= 2
            b = bufs[l]
            live = torch.empty((self.lanes, len(sizes)), dtype=torch.int64, device=self.device)
            L_ = ops.L
            L_.check(L_.kvt_live_chunks(b["run_start"].data_ptr(), b["run_len"].data_ptr(), b["n_runs"].data_ptr(),
                                        b["run_start"].stride(0), self.lanes, int(math.log2(sizes[0])), len(sizes),
                                        live.data_ptr(), ops._stream()), "live_chunks")
            lv = live.double().sum(0).cpu().tolist()
            cur = self.grid_C[l]
            m_cur = ops.n_grid_leaves(self.n, cur)
            n_cand = max(b["evals"].double().mean().item() - m_cur, 1.0) * self.lanes
            infl = n_cand / max(lv[sizes.index(cur)] * cur, 1.0)
            cost = {C: self.lanes * ops.n_grid_leaves(self.n, C) * (2 * self.d * sA + 24) + infl * lv[j] * C * rowK
                    for j, C in enumerate(sizes)}
            best = min(cost, key=cost.get)
            if best != cur and cost[best] < (1.0 - margin) * cost[cur]:
                self._ensure_grid(l, best)
                self.grid_C[l] = best
            dens = [lv[j] / (2.0 * lv[j + 1]) for j in range(len(sizes) - 1) if lv[j + 1] > 0]
            self.rho_measured[l] = sum(dens) / len(dens) if dens else None
        self.use_coarse = [self.grid_C[l] != self.C[l] for l in range(self.L)]
        return list(self.grid_C)

    def adapt_bound_granularity(self, threshold: float = 0.9) -> list[bool]:
        """Compatibility wrapper of adapt_chunking: True for the layers that no longer prune on
        their plan chunk."""
        self.adapt_chunking()
        return list(self.use_coarse)

    def k_for(self, layer: int) -> int:
        return math.ceil(self.rates[layer] * self.n)

    # -- the hot path -------------------------------------------------------------------------------

    def _buffers(self):
        if self._bufs is not None:
            return self._bufs
        dev, lanes, d = self.device, self.lanes, self.d
        bufs = []
        hints = getattr(self, "_hints", None)
        if hints is None:  # per-lane selector state survives buffer rebuilds (n changes on append)
            hints = self._hints = [torch.full((lanes,), float("nan"), dtype=torch.float32, device=dev)
                                   for _ in range(self.L)]
        for l in range(self.L):
            k = self.k_for(l)
            bufs.append({
                "sel_tok": torch.empty((lanes, max(k, 1)), dtype=torch.int32, device=dev),
                "sel_score": torch.empty((lanes, max(k, 1)), dtype=torch.float64, device=dev),
                "n_sel": torch.empty(lanes, dtype=torch.int32, device=dev),
                "run_start": torch.empty((lanes, max(k, 1)), dtype=torch.int32, device=dev),
                "run_len": torch.empty((lanes, max(k, 1)), dtype=torch.int32, device=dev),
                "n_runs": torch.empty(lanes, dtype=torch.int32, device=dev),
                "out": torch.empty((lanes, d), dtype=torch.float32, device=dev),
                "evals": torch.empty(lanes, dtype=torch.int64, device=dev),
                # the previous step's k-th estimate per lane (state across steps; NaN = none)
                "sel_hint": hints[l],
            })
        maxl = max(ops.n_grid_leaves(self.n_cap, C) for C in self.C)
        if self._ws is None or self._ws.key != (lanes, self.n_cap, maxl, d):
            self._ws = ops.LayerWorkspace(lanes, self.n_cap, maxl, d, dev)
        self._bufs = bufs
        return bufs

    def layer(self, l: int, q: torch.Tensor, attend: bool = True) -> dict:
        """Select + attend for layer l; q: [lanes, d] (f32 or f64).  Returns the layer buffers.
        attend=False (or tiered values): the selection only (sel_tok, runs, ...)."""
        bufs = self._buffers()
        C, amax, amin = self.grid(l)
        if attend and self.V is not None:
            o, v = bufs[l], self.V[l]
        else:  # no attention: values alias the keys (same lane stride), no output buffer
            o, v = {kk: vv for kk, vv in bufs[l].items() if kk != "out"}, self.K[l]
        ops.select_attend(q, self.K[l], v, amax, amin, self.n, self.k_for(l), C,
                          self._ws, o, abs_mag=None if self.absmag is None else self.absmag[l],
                          kv_group=self.kv_group)
        return bufs[l]

    def step(self, q: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """All layers for one decode step; q: [L, lanes, d] -> attention outputs [L, lanes, d] f32."""
        if self.V is None:
            raise RuntimeError("tiered values: use host_tier.TieredDecoder.step")
        if out is None:
            out = torch.empty((self.L, self.lanes, self.d), dtype=torch.float32, device=self.device)
        bufs = self._buffers()
        for l in range(self.L):  # attention outputs land directly in out[l]
            C, amax, amin = self.grid(l)
            ops.select_attend(q[l], self.K[l], self.V[l], amax, amin, self.n, self.k_for(l),
                              C, self._ws, {**bufs[l], "out": out[l]},
                              abs_mag=None if self.absmag is None else self.absmag[l], kv_group=self.kv_group)
        return out

    # -- accounting ---------------------------------------------------------------------------------

    def algorithmic_bytes(self, n_cand: list[list[int]], layers: list[int] | None = None) -> dict:
        """Per-kernel algorithmic HBM bytes for one step (SURVEY.md sec. 8(d) formulas), or for the
        given layers only.  n_cand[l][lane] = candidate tokens of that lane at layer l."""
        sK = self.K.element_size()
        sA = self.amax[0].element_size()
        d = self.d
        out = {"bounds": 0, "score": 0, "select": 0, "attn": 0, "plan": 0, "runs": 0}
        for l in (range(self.L) if layers is None else layers):
            m = ops.n_grid_leaves(self.n, self.grid(l)[0])
            k = self.k_for(l)
            nc = sum(n_cand[l])
            # abstracts once per KV lane (GQA query lanes of a group share them), q + U, L, A per lane
            out["bounds"] += self.kv_lanes * m * 2 * d * sA + self.lanes * (d * 8 + m * 24)
            out["plan"] += self.lanes * m * 24 + nc // 64 * 12
            if self.kv_group > 1 and self.dtype == ops.I4:
                # GQA union: each KV lane's candidate records are read once for its g heads
                # (n_cand of every query lane is the union), one f32 estimate per head
                out["score"] += nc // self.kv_group * (d * sK + 4) + nc * 4
            else:
                out["score"] += nc * (d * sK + 8)                                  # f32 estimate + token
            out["select"] += nc * 8 + self.lanes * k * 12
            out["runs"] += self.lanes * k * 4 * 3
            if self.kv_group > 1 and self.dtype == ops.I4 and os.environ.get("KVT_GQA_UNION", "0") == "1":
                # GQA union K7: a V row once per KV lane for its g heads; counted at the smallest
                # possible union (k rows per KV lane), so the fraction is never inflated by g
                out["attn"] += self.kv_lanes * k * d * sK + self.lanes * (k * 12 + d * 4)
            else:
                out["attn"] += self.lanes * k * (d * sK + 4 + 8) + self.lanes * d * 4
        return out


def run_trace(trace, dtype=torch.float32, importance_rate: float = 0.10, early_layer_rate: float = 0.50,
              plan: ChunkPlanConfig | None = None, device=None) -> dict:
    """Decode every step of a `.kvtr` trace on the GPU (the selection + attention of
    engine.run's lane loop, engine.py:307-357; every (layer, head) is one lane, B = 1).
    f32 keys keep the canonical scores identical to the reference's f64 arithmetic on the
    trace's f32 inputs.  Returns {"selected": [step][layer][head] sorted token arrays,
    "out": f32 [steps, layers, heads, d] attention outputs (zeros when the trace has no values)}."""
    import numpy as np
    h = trace.header
    dev = torch.device(device or "cuda")
    dec = SparseDecoder(h.n_layers, 1, h.n_heads, h.head_dim, h.n_context, dtype=dtype, plan=plan,
                        importance_rate=importance_rate, early_layer_rate=early_layer_rate, device=dev)
    for l in range(h.n_layers):
        k = torch.from_numpy(np.array(trace.keys[l], dtype=np.float32)).to(dev)  # copy: mmap is read-only
        v = torch.from_numpy(np.array(trace.values[l], dtype=np.float32)).to(dev) if trace.values is not None \
            else torch.zeros_like(k)
        dec.load_layer(l, k, v)
    dec.set_length(h.n_context)
    selected, outs = [], []
    for s in range(h.n_steps):
        q = torch.from_numpy(np.array(trace.queries[s], dtype=np.float32)).to(dev)
        outs.append(dec.step(q).clone())
        bufs = dec._buffers()
        selected.append([[bufs[l]["sel_tok"][i, :dec.k_for(l)].cpu().numpy().astype(np.int64)
                          for i in range(h.n_heads)] for l in range(h.n_layers)])
    out = torch.stack(outs)
    if trace.values is None:
        out.zero_()
    return {"selected": selected, "out": out}
