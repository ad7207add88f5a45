"""Torch-level wrappers of the C ABI (device tensors in, device tensors out).

Every function launches on torch's current CUDA stream and checks the returned
kvt_status.  Lanes are the leading dimension: keys/values are [n_lanes, N_cap, d] with
contiguous rows (lane stride = tensor.stride(0)), queries are [n_lanes, d].
"""

from __future__ import annotations

import functools
import math

import torch

from . import _lib as L

ITEM_TOKENS = 64
_DT = {torch.float32: L.F32, torch.float64: L.F64, torch.bfloat16: L.BF16, torch.float16: L.F16}
I4 = "int4"


class I4KV:
    """INT4-compressed KV rows (kvt_kv_quant records): `data` is uint8 [n_lanes, N_cap, d/2 + d/8]
    (lane stride in bytes), `d` the logical head dim.  Dequantised value fmaf(code, scale, min)."""

    def __init__(self, data: torch.Tensor, d: int):
        if data.dtype != torch.uint8 or data.dim() < 3 or data.shape[-1] != row_bytes_i4(d):
            raise ValueError("I4KV data must be uint8 [..., n_lanes, N_cap, d/2 + d/8]")
        self.data, self.d = data, d
        self.dtype = I4

    @classmethod
    def empty(cls, n_lanes: int, n_cap: int, d: int, device) -> "I4KV":
        return cls(torch.empty((n_lanes, n_cap, row_bytes_i4(d)), dtype=torch.uint8, device=device), d)

    @property
    def shape(self):
        return tuple(self.data.shape[:-1]) + (self.d,)

    @property
    def device(self):
        return self.data.device

    @property
    def is_cuda(self):
        return self.data.is_cuda

    def data_ptr(self):
        return self.data.data_ptr()

    def stride(self, i):
        return self.data.stride(i)

    def __getitem__(self, idx):
        return I4KV(self.data[idx], self.d)

    def element_size(self):
        return row_bytes_i4(self.d) / self.d


def row_bytes_i4(d: int) -> int:
    return d // 2 + (d // 32) * 4


def dtype_code(t) -> int:
    if isinstance(t, I4KV):
        return L.I4
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}") from None


def abs_dtype_for(key_dtype) -> torch.dtype:
    """Abstract storage dtype: f64 for f64 keys, f32 otherwise (importance.py:75-77 wire f32)."""
    return torch.float64 if key_dtype == torch.float64 else torch.float32


class kv_group:
    """GQA scope for the standalone decode-path wrappers (kvt_set_kv_group): inside
    `with ops.kv_group(g):` query lane i reads key/value/abstract lane i // g."""

    def __init__(self, g: int):
        self.g = max(int(g), 1)

    def __enter__(self):
        self.old = L.kvt_set_kv_group(self.g)
        return self

    def __exit__(self, *exc):
        L.kvt_set_kv_group(self.old)


class cand_group:
    """GQA union candidates for the standalone wrappers (kvt_set_cand_group): inside
    `with ops.cand_group(g):` cand_score_i4mma scores the per-KV-lane union items of
    select_plan(..., group=g) for all g query lanes, and topk_select_band reads the shared
    token-id row of each group."""

    def __init__(self, g: int):
        self.g = max(int(g), 1)

    def __enter__(self):
        self.old = L.kvt_set_cand_group(self.g)
        return self

    def __exit__(self, *exc):
        L.kvt_set_cand_group(self.old)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _on_device(fn):
    """Device guard: run the wrapper with its first CUDA operand's device current, so the ABI
    launches on that device and on torch's current stream *of that device* (the library
    launches on cudaGetDevice's device)."""
    @functools.wraps(fn)
    def wrapper(*args, **kw):
        dev = None
        for a in list(args) + list(kw.values()):
            if isinstance(a, (torch.Tensor, I4KV)) and a.is_cuda:
                dev = a.device
                break
        if dev is None or dev.index is None or dev.index == torch.cuda.current_device():
            return fn(*args, **kw)
        with torch.cuda.device(dev):
            return fn(*args, **kw)
    return wrapper


def _p(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def _nz(t: torch.Tensor) -> torch.Tensor:
    """Never hand a NULL pointer to the ABI for an empty (k = 0) operand."""
    if t.numel() == 0:
        return torch.zeros(1, dtype=t.dtype, device=t.device)
    return t.contiguous()


def require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("paper_2506_20187_b200 runs on CUDA (sm_100a) only; got a CPU tensor")


def _lanes(t) -> tuple[int, int]:
    """(lane_stride, d) of a [n_lanes, N, d] tensor with contiguous rows (bytes for I4KV)."""
    if isinstance(t, I4KV):
        if t.data.stride(2) != 1 or t.data.stride(1) != t.data.shape[2]:
            raise ValueError("I4KV rows must be contiguous")
        return t.data.stride(0), t.d
    if t.dim() != 3 or t.stride(2) != 1 or t.stride(1) != t.shape[2]:
        raise ValueError(f"expected [n_lanes, N, d] with contiguous rows, got shape {tuple(t.shape)} strides {t.stride()}")
    return t.stride(0), t.shape[2]


def n_grid_leaves(n: int, C: int) -> int:
    return (n + C - 1) // C


# -- K8 ----------------------------------------------------------------------------------------


@_on_device
def kv_quant(src: torch.Tensor, dst: I4KV, t_begin: int = 0, t_end: int | None = None) -> I4KV:
    """INT4-compress rows [t_begin, t_end) of every lane of src [n_lanes, N, d] into dst (K8)."""
    require_cuda(src)
    ls, d = _lanes(src)
    t_end = src.shape[1] if t_end is None else t_end
    if dst.d != d or dst.shape[0] != src.shape[0] or dst.shape[1] < t_end:
        raise ValueError("kv_quant: destination shape mismatch")
    L.check(L.kvt_kv_quant(src.data_ptr(), dtype_code(src), src.shape[0], ls, t_begin, t_end, d, dst.data_ptr(),
                           dst.stride(0), _stream()), "kv_quant")
    return dst


# -- K1 ----------------------------------------------------------------------------------------


@_on_device
def abstract_build(keys, n: int, C: int, amax: torch.Tensor | None = None,
                   amin: torch.Tensor | None = None, c_begin: int = 0, c_end: int | None = None,
                   abs_dtype: torch.dtype | None = None):
    """Uniform-grid chunk abstracts (importance.py:80-87) -> (amax, amin) [n_lanes, m_cap, d].
    abs_dtype: exact f32/f64 (default) or torch.bfloat16 (rounded outward, half the bytes)."""
    require_cuda(keys)
    ls, d = _lanes(keys)
    nl = keys.shape[0]
    m = n_grid_leaves(n, C)
    c_end = m if c_end is None else c_end
    if amax is not None:
        abs_dtype = amax.dtype
    adt = abs_dtype or abs_dtype_for(keys.dtype)
    if amax is None:
        amax = torch.empty((nl, m, d), dtype=adt, device=keys.device)
        amin = torch.empty_like(amax)
    if amin.dtype != adt or amax.stride(2) != 1:
        raise ValueError("abstract buffers must be contiguous rows of the abstract dtype")
    L.check(L.kvt_abstract_build(keys.data_ptr(), dtype_code(keys), nl, ls, n, d, C, c_begin, c_end,
                                 amax.data_ptr(), amin.data_ptr(), dtype_code(amax), amax.stride(0), _stream()),
            "abstract_build")
    return amax, amin


@_on_device
def abstract_spans(keys: torch.Tensor, lane_of: torch.Tensor, starts: torch.Tensor, ends: torch.Tensor):
    """Exact abstracts of arbitrary spans -> (amax, amin) [S, d]."""
    require_cuda(keys)
    ls, d = _lanes(keys)
    S = starts.numel()
    adt = abs_dtype_for(keys.dtype)
    amax = torch.empty((S, d), dtype=adt, device=keys.device)
    amin = torch.empty_like(amax)
    if S:
        lane_of = lane_of.to(device=keys.device, dtype=torch.int32).contiguous()
        starts = starts.to(device=keys.device, dtype=torch.int32).contiguous()
        ends = ends.to(device=keys.device, dtype=torch.int32).contiguous()
        L.check(L.kvt_abstract_spans(keys.data_ptr(), dtype_code(keys), ls, d, S, lane_of.data_ptr(),
                                     starts.data_ptr(), ends.data_ptr(), amax.data_ptr(), amin.data_ptr(),
                                     _stream()), "abstract_spans")
    return amax, amin


@_on_device
def abstract_merge(amax: torch.Tensor, amin: torch.Tensor, seg_lane=None, seg_begin=None, seg_end=None,
                   factor: int = 0, m_in: int = 0, out: tuple | None = None):
    """K2 (kvt_abstract_merge): element-wise max / min over segments of consecutive chunk
    abstracts.  amax/amin: [lanes, m, d] (or [m, d] = one lane).  Explicit segments
    (seg_lane, seg_begin, seg_end int sequences) -> [S, d]; or uniform coarsening by `factor`
    over the first m_in chunks -> [lanes, ceil(m_in / factor), d] (or into `out`)."""
    require_cuda(amax, amin)
    a3 = amax if amax.dim() == 3 else amax[None]
    b3 = amin if amin.dim() == 3 else amin[None]
    if a3.shape != b3.shape or a3.dtype != b3.dtype or a3.stride(2) != 1 or a3.stride(1) != a3.shape[2] \
            or b3.stride() != a3.stride():
        raise ValueError("abstract_merge: amax / amin must be matching [lanes, m, d] row-major tensors")
    nl, _, d = a3.shape
    dev = a3.device
    if seg_begin is not None:
        sb = torch.as_tensor(seg_begin, dtype=torch.int32).to(dev).contiguous()
        se = torch.as_tensor(seg_end, dtype=torch.int32).to(dev).contiguous()
        sl = (torch.zeros_like(sb) if seg_lane is None else
              torch.as_tensor(seg_lane, dtype=torch.int32).to(dev).contiguous())
        S = sb.numel()
        omx = torch.empty((S, d), dtype=a3.dtype, device=dev) if out is None else out[0]
        omn = torch.empty_like(omx) if out is None else out[1]
        if S:
            L.check(L.kvt_abstract_merge(a3.data_ptr(), b3.data_ptr(), dtype_code(a3), a3.stride(0), d, S,
                                         sl.data_ptr(), sb.data_ptr(), se.data_ptr(), 0, 0, 0, omx.data_ptr(),
                                         omn.data_ptr(), 0, _stream()), "abstract_merge")
        return omx, omn
    if factor < 1 or m_in < 1:
        raise ValueError("abstract_merge: give segments or factor >= 1 and m_in >= 1")
    m_out = -(-m_in // factor)
    if out is None:
        omx = torch.empty((nl, m_out, d), dtype=a3.dtype, device=dev)
        omn = torch.empty_like(omx)
    else:
        omx, omn = out
    L.check(L.kvt_abstract_merge(a3.data_ptr(), b3.data_ptr(), dtype_code(a3), a3.stride(0), d, nl * m_out, None,
                                 None, None, factor, m_in, m_out, omx.data_ptr(), omn.data_ptr(), omx.stride(0),
                                 _stream()), "abstract_merge")
    return omx, omn


# -- K3 ----------------------------------------------------------------------------------------


@_on_device
def chunk_bounds(q: torch.Tensor, amax: torch.Tensor, amin: torch.Tensor, n: int, C: int = 0,
                 leaf_start: torch.Tensor | None = None, n_leaves: torch.Tensor | None = None,
                 scaled: bool = False, want_A: bool = False):
    """Sound canonical (U, L) per leaf (importance.py:108-137) -> float64 [n_lanes, max_leaves].
    scaled=False: bounds on raw dots (pipeline); scaled=True: on logits dot/sqrt(d) (API)."""
    require_cuda(q, amax, amin)
    nl, d = q.shape
    if leaf_start is not None:
        lstride = leaf_start.shape[1]
        maxl = lstride
    else:
        lstride = 0
        maxl = n_grid_leaves(n, C)
    U = torch.empty((nl, max(maxl, 1)), dtype=torch.float64, device=q.device)
    Lo = torch.empty_like(U)
    A = torch.empty_like(U) if want_A else None
    L.check(L.kvt_chunk_bounds(q.data_ptr(), dtype_code(q), nl, d, n, C, _p(leaf_start), _p(n_leaves), lstride,
                               amax.data_ptr(), amin.data_ptr(), dtype_code(amax), amax.stride(0), U.data_ptr(),
                               Lo.data_ptr(), _p(A), U.stride(0), int(scaled), _stream()), "chunk_bounds")
    return (U, Lo, A) if want_A else (U, Lo)


# -- K4 ----------------------------------------------------------------------------------------


@_on_device
def token_scores(q: torch.Tensor, keys: torch.Tensor, n: int | None = None) -> torch.Tensor:
    """Canonical f64 logits of all tokens (importance.py:27-33) -> [n_lanes, n]."""
    require_cuda(q, keys)
    ls, d = _lanes(keys)
    nl = keys.shape[0]
    n = keys.shape[1] if n is None else n
    if q.shape != (nl, d):
        raise ValueError(f"shape mismatch: keys {tuple(keys.shape)} vs query {tuple(q.shape)}")
    out = torch.empty((nl, max(n, 1)), dtype=torch.float64, device=q.device)
    L.check(L.kvt_token_scores(q.data_ptr(), dtype_code(q), keys.data_ptr(), dtype_code(keys), nl, ls, n, d,
                               out.data_ptr(), out.stride(0), _stream()), "token_scores")
    return out[:, :n]


@_on_device
def select_plan(U: torch.Tensor, Lo: torch.Tensor, n: int, k: int, C: int = 0,
                leaf_start: torch.Tensor | None = None, n_leaves: torch.Tensor | None = None,
                want_cand_leaf: bool = False, A: torch.Tensor | None = None, d: int = 0, group: int = 1):
    """tau + candidate items -> dict(items, n_items, n_cand, cand_leaf, evals[, err]).
    With A (from chunk_bounds(want_A=True)) and d, also the f32 scoring error bound err.
    group = g > 1 (GQA union, kvt_select_plan_group): items / n_items per KV lane (the union of
    its g query lanes' candidates); n_cand, evals, err per query lane."""
    nl = U.shape[0]
    maxl = leaf_start.shape[1] if leaf_start is not None else n_grid_leaves(n, C)
    item_cap = (n + ITEM_TOKENS - 1) // ITEM_TOKENS + maxl
    dev = U.device
    items = torch.empty((nl, item_cap, 3), dtype=torch.int32, device=dev)
    n_items = torch.empty(nl, dtype=torch.int32, device=dev)
    n_cand = torch.empty(nl, dtype=torch.int32, device=dev)
    evals = torch.empty(nl, dtype=torch.int64, device=dev)
    cand_leaf = torch.zeros((nl, max(maxl, 1)), dtype=torch.int8, device=dev) if want_cand_leaf else None
    lstride = leaf_start.shape[1] if leaf_start is not None else maxl
    err = torch.empty((nl, 4), dtype=torch.float64, device=dev) if A is not None else None
    L.check(L.kvt_select_plan_group(nl, n, C, _p(leaf_start), _p(n_leaves), lstride, U.data_ptr(), Lo.data_ptr(),
                                    U.stride(0), k, items.data_ptr(), item_cap, n_items.data_ptr(),
                                    n_cand.data_ptr(), _p(cand_leaf), evals.data_ptr(), _p(A), _p(err), d,
                                    max(int(group), 1), _stream()), "select_plan")
    return {"items": items, "n_items": n_items, "n_cand": n_cand, "cand_leaf": cand_leaf, "evals": evals,
            "item_cap": item_cap, "err": err}


@_on_device
def cand_score(q: torch.Tensor, keys: torch.Tensor, plan: dict, n: int, blocks_per_lane: int = 0):
    """Raw canonical dots of candidate tokens -> (cand_score f64 [n_lanes, n], cand_tok i32)."""
    require_cuda(q, keys)
    ls, d = _lanes(keys)
    nl = keys.shape[0]
    cs = torch.empty((nl, max(n, 1)), dtype=torch.float64, device=q.device)
    ct = torch.empty((nl, max(n, 1)), dtype=torch.int32, device=q.device)
    if blocks_per_lane <= 0:
        blocks_per_lane = max(1, min((plan["item_cap"] + 7) // 8, (148 * 8 + nl - 1) // nl))
    L.check(L.kvt_cand_score(q.data_ptr(), dtype_code(q), keys.data_ptr(), dtype_code(keys), nl, ls, d,
                             plan["items"].data_ptr(), plan["item_cap"], plan["n_items"].data_ptr(), cs.data_ptr(),
                             ct.data_ptr(), cs.stride(0), blocks_per_lane, _stream()), "cand_score")
    return cs, ct


@_on_device
def cand_score_f32(q: torch.Tensor, keys, plan: dict, n: int):
    """Fast f32 estimates of the candidate dots (|err| <= plan["err"]) -> (cs32 f32, cand_tok i32)."""
    require_cuda(q, keys)
    ls, d = _lanes(keys)
    nl = q.shape[0]
    cs = torch.empty((nl, max(n, 1)), dtype=torch.float32, device=q.device)
    ct = torch.empty((nl, max(n, 1)), dtype=torch.int32, device=q.device)
    L.check(L.kvt_cand_score_f32(q.data_ptr(), dtype_code(q), keys.data_ptr(), dtype_code(keys), nl, ls, d,
                                 plan["items"].data_ptr(), plan["item_cap"], plan["n_items"].data_ptr(), cs.data_ptr(),
                                 ct.data_ptr(), cs.stride(0), _stream()), "cand_score_f32")
    return cs, ct


@_on_device
def cand_score_i4mma(q: torch.Tensor, keys: "I4KV", plan: dict, n: int):
    """INT4 keys: estimates with exact int32 inner products on the tensor cores.  Also max-es
    the per-lane bound on |estimate - canonical dot| into plan["err"][:, 3] (used as E by
    topk_select_band) -> (cs32 f32, cand_tok i32)."""
    require_cuda(q, keys)
    ls, d = _lanes(keys)
    nl = q.shape[0]
    cs = torch.empty((nl, max(n, 1)), dtype=torch.float32, device=q.device)
    ct = torch.empty((nl, max(n, 1)), dtype=torch.int32, device=q.device)
    ws = torch.empty(max(int(L.kvt_i4_qprep_bytes(nl, d)), 16), dtype=torch.uint8, device=q.device)
    L.check(L.kvt_cand_score_i4mma(q.data_ptr(), dtype_code(q), keys.data_ptr(), nl, ls, d, plan["items"].data_ptr(),
                                   plan["item_cap"], plan["n_items"].data_ptr(), cs.data_ptr(), ct.data_ptr(),
                                   cs.stride(0), plan["err"].data_ptr(), ws.data_ptr(), _stream()), "cand_score_i4mma")
    return cs, ct


@_on_device
def topk_select_band(cs32: torch.Tensor, ct: torch.Tensor, plan: dict, k: int, q: torch.Tensor, keys,
                     want_runs: bool = True):
    """Exact canonical top-k from f32 estimates (band re-scoring) -> (sel_tok, sel_score, n_sel[, runs])."""
    ls, d = _lanes(keys)
    nl = cs32.shape[0]
    dev = cs32.device
    st = torch.empty((nl, max(k, 1)), dtype=torch.int32, device=dev)
    ss = torch.empty((nl, max(k, 1)), dtype=torch.float64, device=dev)
    ns = torch.empty(nl, dtype=torch.int32, device=dev)
    scratch = plan.get("scratch")
    if scratch is None or scratch.shape != cs32.shape:
        scratch = plan["scratch"] = torch.empty(cs32.shape, dtype=torch.float64, device=dev)
    runs = None
    if want_runs:
        runs = {"run_start": torch.empty((nl, max(k, 1)), dtype=torch.int32, device=dev),
                "run_len": torch.empty((nl, max(k, 1)), dtype=torch.int32, device=dev),
                "n_runs": torch.empty(nl, dtype=torch.int32, device=dev)}
    L.check(L.kvt_topk_select_band(cs32.data_ptr(), ct.data_ptr(), plan["n_cand"].data_ptr(), cs32.stride(0),
                                   plan["err"].data_ptr(), nl, k, q.data_ptr(), dtype_code(q), keys.data_ptr(),
                                   dtype_code(keys), ls, d, scratch.data_ptr(), st.data_ptr(), ss.data_ptr(),
                                   st.stride(0), ns.data_ptr(),
                                   _p(runs["run_start"]) if runs else None, _p(runs["run_len"]) if runs else None,
                                   st.stride(0), _p(runs["n_runs"]) if runs else None, _stream()), "topk_select_band")
    if want_runs:
        return st[:, :k], ss[:, :k], ns, runs
    return st[:, :k], ss[:, :k], ns


@_on_device
def topk_select(cs: torch.Tensor, ct: torch.Tensor, n_cand: torch.Tensor, k: int, want_runs: bool = False):
    """Exact top-k (score desc, token asc) -> (sel_tok i32 [n_lanes,k] ascending, sel_score f64, n_sel)
    [+ dict(run_start, run_len, n_runs) from the fused run scan]."""
    nl = cs.shape[0]
    dev = cs.device
    st = torch.empty((nl, max(k, 1)), dtype=torch.int32, device=dev)
    ss = torch.empty((nl, max(k, 1)), dtype=torch.float64, device=dev)
    ns = torch.empty(nl, dtype=torch.int32, device=dev)
    runs = None
    if want_runs:
        runs = {"run_start": torch.empty((nl, max(k, 1)), dtype=torch.int32, device=dev),
                "run_len": torch.empty((nl, max(k, 1)), dtype=torch.int32, device=dev),
                "n_runs": torch.empty(nl, dtype=torch.int32, device=dev)}
    L.check(L.kvt_topk_select_runs(cs.data_ptr(), ct.data_ptr(), n_cand.data_ptr(), cs.stride(0), nl, k,
                                   st.data_ptr(), ss.data_ptr(), st.stride(0), ns.data_ptr(),
                                   _p(runs["run_start"]) if runs else None, _p(runs["run_len"]) if runs else None,
                                   st.stride(0), _p(runs["n_runs"]) if runs else None, _stream()), "topk_select")
    if want_runs:
        return st[:, :k], ss[:, :k], ns, runs
    return st[:, :k], ss[:, :k], ns


@_on_device
def runs_scan(sel_tok: torch.Tensor, n_sel: torch.Tensor, n: int, want_partition: bool = True):
    """Selected runs (+ canonical partition) -> dict."""
    nl = sel_tok.shape[0]
    k = sel_tok.shape[1]
    dev = sel_tok.device
    st = _nz(sel_tok)
    sstride = sel_tok.shape[1] if k > 0 else 1
    rs = torch.empty((nl, max(k, 1)), dtype=torch.int32, device=dev)
    rl = torch.empty_like(rs)
    nr = torch.empty(nl, dtype=torch.int32, device=dev)
    ps = pst = npart = None
    pcap = 2 * k + 2
    if want_partition:
        ps = torch.empty((nl, pcap), dtype=torch.int32, device=dev)
        pst = torch.empty((nl, pcap), dtype=torch.int8, device=dev)
        npart = torch.empty(nl, dtype=torch.int32, device=dev)
    L.check(L.kvt_runs_scan(st.data_ptr(), n_sel.data_ptr(), sstride, nl, n, rs.data_ptr(), rl.data_ptr(),
                            rs.stride(0), nr.data_ptr(), _p(ps), _p(pst), pcap, _p(npart), _stream()), "runs_scan")
    return {"run_start": rs, "run_len": rl, "n_runs": nr, "part_start": ps, "part_state": pst, "n_part": npart}


@_on_device
def sparse_decode_attn(values: torch.Tensor, sel_tok: torch.Tensor, sel_score: torch.Tensor, n_sel: torch.Tensor,
                       splits: int = 0, want_f64: bool = False, logit_scale: float | None = None,
                       want_lse: bool = False):
    """softmax(sel_score * logit_scale) @ V[sel] (engine.py:145-154) -> out f32 [n_lanes, d] (and f64).
    logit_scale defaults to 1/sqrt(d) (sel_score = raw dots from K4/K5); pass 1.0 for logits.
    want_lse: also return the lanes' merged softmax state (m, l) f64 [n_lanes, 2] (kvt_attn_lse)."""
    require_cuda(values)
    ls, d = _lanes(values)
    nl = n_sel.shape[0]
    k = sel_tok.shape[1]
    # splits <= 0: chosen by kvt_sparse_decode_attn (wave-aware); the workspace holds 64
    ws = torch.zeros(max(1, L.kvt_attn_workspace_bytes(nl, d, 64 if splits <= 0 else splits)), dtype=torch.uint8,
                     device=values.device)
    out = torch.empty((nl, d), dtype=torch.float32, device=values.device)
    out64 = torch.empty((nl, d), dtype=torch.float64, device=values.device) if want_f64 else None
    st = _nz(sel_tok)
    ss = _nz(sel_score)
    sstride = sel_tok.shape[1] if k > 0 else 1
    if logit_scale is None:
        logit_scale = 1.0 / math.sqrt(d)
    L.check(L.kvt_sparse_decode_attn(values.data_ptr(), dtype_code(values), nl, ls, d, st.data_ptr(), ss.data_ptr(),
                                     n_sel.data_ptr(), sstride, float(logit_scale), splits, ws.data_ptr(),
                                     out.data_ptr(), _p(out64), _stream()), "sparse_decode_attn")
    res = (out, out64) if want_f64 else (out,)
    if want_lse:
        lse = torch.empty((nl, 2), dtype=torch.float64, device=values.device)
        L.check(L.kvt_attn_lse(ws.data_ptr(), nl, lse.data_ptr(), _stream()), "attn_lse")
        res = res + (lse,)
    return res if len(res) > 1 else res[0]


@_on_device
def lse_merge(parts: torch.Tensor, logit_scale: float, want_f64: bool = False):
    """Merge shard partials parts [P, n_lanes, d + 2] f64 = (m, l, o normalised) (kvt_lse_merge)."""
    require_cuda(parts)
    P, nl, d2 = parts.shape
    parts = parts.contiguous().double()
    out = torch.empty((nl, d2 - 2), dtype=torch.float32, device=parts.device)
    out64 = torch.empty((nl, d2 - 2), dtype=torch.float64, device=parts.device) if want_f64 else None
    L.check(L.kvt_lse_merge(parts.data_ptr(), P, nl, d2 - 2, float(logit_scale), out.data_ptr(), _p(out64),
                            _stream()), "lse_merge")
    return (out, out64) if want_f64 else out


# -- fused per-layer pipeline ---------------------------------------------------------------------


class LayerWorkspace:
    """Caller-owned scratch for kvt_select_attend, sized once for (n_lanes, n_cap, leaves, d)."""

    def __init__(self, n_lanes: int, n_cap: int, max_leaves: int, d: int, device):
        self.bytes = int(L.kvt_layer_workspace_bytes(n_lanes, n_cap, max_leaves, d))
        self.buf = torch.zeros(self.bytes, dtype=torch.uint8, device=device)  # attn tickets start at 0
        self.key = (n_lanes, n_cap, max_leaves, d)


@_on_device
def select_attend(q: torch.Tensor, keys, values, amax: torch.Tensor, amin: torch.Tensor,
                  n: int, k: int, C: int, ws: LayerWorkspace, out: dict, attn_splits: int = 0,
                  score_blocks: int = 0, exact_scores: bool = False, abs_mag: torch.Tensor | None = None,
                  kv_group: int = 1) -> None:
    """One layer, all lanes: K3 -> plan -> K4 -> K5 -> K6 -> K7 into the caller's `out` buffers
    (sel_tok, sel_score, n_sel, run_start, run_len, n_runs, out, evals).
    abs_mag ([n_lanes, d] f32 max |key| per lane, see lane_abs_mag): directed-rounding f32
    bounds for bf16 abstracts instead of the canonical f64 ones (same selected set).
    kv_group (GQA): q has kv_group lanes per lane of keys/values/abstracts/abs_mag."""
    ls, d = _lanes(keys)
    if q.shape[0] != keys.shape[0] * max(kv_group, 1):
        raise ValueError("q must have kv_group lanes per key lane")
    a = L.KvtLayerArgs()
    a.n_lanes, a.n, a.k, a.d, a.C = q.shape[0], n, k, d, C
    a.key_dtype, a.v_dtype, a.q_dtype, a.abs_dtype = dtype_code(keys), dtype_code(values), dtype_code(q), dtype_code(amax)
    a.q, a.keys, a.values, a.lane_stride = q.data_ptr(), keys.data_ptr(), values.data_ptr(), ls
    if values.stride(0) != ls:
        raise ValueError("keys and values must share the lane stride")
    a.amax, a.amin, a.abs_lane_stride = amax.data_ptr(), amin.data_ptr(), amax.stride(0)
    a.leaf_start, a.n_leaves, a.leaf_stride = None, None, 0
    a.sel_tok, a.sel_score, a.n_sel = out["sel_tok"].data_ptr(), out["sel_score"].data_ptr(), out["n_sel"].data_ptr()
    a.run_start = _p(out.get("run_start"))
    a.run_len = _p(out.get("run_len"))
    a.n_runs = _p(out.get("n_runs"))
    a.out = _p(out.get("out"))
    a.evals = _p(out.get("evals"))
    a.attn_splits, a.score_blocks, a.exact_scores = attn_splits, score_blocks, int(exact_scores)
    a.abs_mag = _p(abs_mag)
    a.kv_group = max(kv_group, 1)
    a.sel_hint = _p(out.get("sel_hint"))
    L.check(L.kvt_select_attend(a, ws.buf.data_ptr(), ws.bytes, _stream()), "select_attend")


@_on_device
def sparse_decode_attn_gqa(values, sel_tok: torch.Tensor, sel_score: torch.Tensor, n_sel: torch.Tensor, kv_group: int,
                           n_ctx: int, want_f64: bool = False, ws: torch.Tensor | None = None,
                           scratch: torch.Tensor | None = None, out: torch.Tensor | None = None):
    """GQA union K7 (kvt_sparse_decode_attn_gqa): INT4 values [n_kv, N, rb], query lanes i / g
    share KV lane i / g -> out f32 [n_lanes, d] (and f64).  ws (zeroed once; the kernels leave
    it zeroed), scratch and out may be passed in to reuse them across calls."""
    require_cuda(values)
    ls, d = _lanes(values)
    nl = n_sel.shape[0]
    dev = values.device
    if ws is None:
        ws = torch.zeros(L.kvt_attn_workspace_bytes(nl, d, 64), dtype=torch.uint8, device=dev)
    sb = L.kvt_attn_gqa_scratch_bytes(nl, kv_group, n_ctx)
    if scratch is None:
        scratch = torch.empty(max(sb, 1), dtype=torch.uint8, device=dev)
    elif scratch.numel() < sb:
        raise ValueError(f"scratch holds {scratch.numel()} bytes, the GQA union needs {sb}")
    if out is None:
        out = torch.empty((nl, d), dtype=torch.float32, device=dev)
    out64 = torch.empty((nl, d), dtype=torch.float64, device=dev) if want_f64 else None
    L.check(L.kvt_sparse_decode_attn_gqa(values.data_ptr(), nl, ls, d, kv_group, n_ctx, sel_tok.data_ptr(),
                                         sel_score.data_ptr(), n_sel.data_ptr(), sel_tok.shape[1],
                                         1.0 / math.sqrt(d), ws.data_ptr(), scratch.data_ptr(), sb, out.data_ptr(),
                                         _p(out64), _stream()), "sparse_decode_attn_gqa")
    return (out, out64) if want_f64 else out


def lane_abs_mag(amax: torch.Tensor, amin: torch.Tensor, m: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """Per-lane max |key| over chunks [0, m) from the (outward-rounded) abstracts -> f32 [n_lanes, d]
    (the abs_mag operand of select_attend / kvt_chunk_bounds_fast)."""
    mag = torch.maximum(amax[:, :m].float().abs().amax(dim=1), amin[:, :m].float().abs().amax(dim=1))
    if out is None:
        return mag.contiguous()
    out.copy_(mag)
    return out


@_on_device
def chunk_bounds_fast(q: torch.Tensor, amax: torch.Tensor, amin: torch.Tensor, n: int, C: int,
                      abs_mag: torch.Tensor):
    """Sound f32 directed-rounding (U, L, A_lane) over bf16 abstracts (kvt_chunk_bounds_fast)."""
    require_cuda(q, amax, amin, abs_mag)
    nl, d = q.shape
    m = n_grid_leaves(n, C)
    U = torch.empty((nl, max(m, 1)), dtype=torch.float64, device=q.device)
    Lo = torch.empty_like(U)
    A = torch.empty_like(U)
    L.check(L.kvt_chunk_bounds_fast(q.contiguous().data_ptr(), nl, d, n, C, amax.data_ptr(), amin.data_ptr(),
                                    amax.stride(0), abs_mag.data_ptr(), U.data_ptr(), Lo.data_ptr(), A.data_ptr(),
                                    U.stride(0), _stream()), "chunk_bounds_fast")
    return U, Lo, A


def sqrt_d(d: int) -> float:
    return math.sqrt(d)


# -- synthetic workload (bench / tests; not on the decode path) ------------------------------------


@_on_device
def synth_layer(keys: torch.Tensor | None, values: torch.Tensor | None, params: dict, n: int, gen: dict) -> None:
    """Fill rows [0, n) of bf16 keys / values [n_lanes, N_cap, d] with the counter-hash synthetic
    workload (kvt_synth_layer).  params: per-lane {"seed" u32, "u" f32 [lanes, d], "regions" i32
    [lanes, R, 2]} (workload.lane_params); gen: workload.gen_args."""
    t = keys if keys is not None else values
    require_cuda(t)
    if t.dtype != torch.bfloat16:
        raise ValueError("synth_layer writes bf16 rows")
    ls, d = _lanes(t)
    nl = t.shape[0]
    if keys is not None and values is not None and (values.shape != keys.shape or values.stride(0) != ls):
        raise ValueError("keys and values must share shape and lane stride")
    dev = t.device
    seed = torch.from_numpy(params["seed"].astype("uint32").view("int32")).to(dev)
    u = torch.from_numpy(params["u"]).to(device=dev, dtype=torch.float32).contiguous()
    reg = torch.from_numpy(params["regions"]).to(device=dev, dtype=torch.int32).contiguous()
    if seed.numel() != nl or u.shape != (nl, d):
        raise ValueError("synth_layer: params do not match the lanes")
    L.check(L.kvt_synth_layer(_p(keys), _p(values), nl, ls, n, d, seed.data_ptr(), u.data_ptr(), reg.data_ptr(),
                              reg.shape[1], float(gen["desert_base"]), float(gen["desert_span"]),
                              float(gen["hot_base"]), float(gen["hot_span"]), float(gen["noise_scale"]),
                              int(gen["planted"]), _stream()), "synth_layer")
