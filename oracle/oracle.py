"""ctypes front-end for the C oracle (oracle/kvt_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker for the CUDA path and the bench CPU baseline.
Importable from tests/, __graft_entry__.smoke() and bench.py; never from the product
package (paper_2506_20187_b200/), which must fail loudly instead of falling back here.

Every function widens its inputs to float64 (exact for f32/bf16/f16 data), exactly as the
reference does (`np.asarray(..., dtype=np.float64)`, importance.py:29-30,82,115).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"

_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_ip = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)

# state codes used by kvt_oracle.c (match chunk_tree.py:127-130 names)
STATES = ("candidate", "important", "desert", "pad")


def build(force: bool = False) -> Path:
    src = _HERE / "kvt_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.ora_dot.restype = ctypes.c_double
        L.ora_dot.argtypes = [_dp, _dp, ctypes.c_int]
        L.ora_scores.argtypes = [_dp, _dp, _i64, ctypes.c_int, _dp]
        L.ora_dots.argtypes = [_dp, _dp, _i64, ctypes.c_int, _dp]
        L.ora_bounds2.argtypes = [_dp, _dp, _dp, _i64, ctypes.c_int, _ip, _dp, _dp, ctypes.c_int]
        L.ora_abstract.argtypes = [_dp, ctypes.c_int, _i64, _i64, _dp, _dp]
        L.ora_bound_slack_factor.restype = ctypes.c_double
        L.ora_bound_slack_factor.argtypes = [ctypes.c_int]
        L.ora_bounds.argtypes = [_dp, _dp, _dp, _i64, ctypes.c_int, _ip, _dp, _dp]
        L.ora_np_sum.restype = ctypes.c_double
        L.ora_np_sum.argtypes = [_dp, _i64]
        L.ora_bounds_ref.argtypes = [_dp, _dp, _dp, _i64, ctypes.c_int, _dp, _dp]
        L.ora_i4_record_bytes.restype = ctypes.c_int
        L.ora_i4_record_bytes.argtypes = [ctypes.c_int]
        L.ora_i4_quant.argtypes = [_fp, _i64, ctypes.c_int, ctypes.c_void_p]
        L.ora_i4_dequant.argtypes = [ctypes.c_void_p, _i64, ctypes.c_int, _fp]
        L.ora_synth_lane.argtypes = [_fp, _fp, _i64, ctypes.c_int, ctypes.c_uint32, _fp, _i32p, ctypes.c_int,
                                     ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                     ctypes.c_int]
        L.ora_topk.restype = _i64
        L.ora_topk.argtypes = [_dp, _i64, _i64, _ip]
        L.ora_runs.restype = _i64
        L.ora_runs.argtypes = [_ip, _i64, _ip, _ip]
        L.ora_attention.argtypes = [_dp, _dp, _dp, _ip, _i64, ctypes.c_int, _dp]
        L.ora_part_new.restype = ctypes.c_void_p
        L.ora_part_new.argtypes = [_dp, _i64, ctypes.c_int, _i64]
        L.ora_part_free.argtypes = [ctypes.c_void_p]
        L.ora_part_select.restype = _i64
        L.ora_part_select.argtypes = [ctypes.c_void_p, _dp, _i64, _ip]
        L.ora_part_merge.restype = _i64
        L.ora_part_merge.argtypes = [ctypes.c_void_p]
        L.ora_part_n_leaves.restype = _i64
        L.ora_part_n_leaves.argtypes = [ctypes.c_void_p]
        L.ora_part_leaves.argtypes = [ctypes.c_void_p, _ip, _ip, _i32p]
        L.ora_part_leaf_abstract.argtypes = [ctypes.c_void_p, _i64, _dp, _dp]
        L.ora_bench_lanes.restype = ctypes.c_double
        L.ora_bench_lanes.argtypes = [_i64, _i64, ctypes.c_int, _i64, _i64, ctypes.c_int,
                                      ctypes.c_int, _fp, _fp, _fp, ctypes.c_int, _dp, _ip,
                                      ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), _dp]
        _lib = L
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


# -- importance.py restatements ------------------------------------------------------------


def scores(query, keys) -> np.ndarray:
    """Canonical-order fl(k.q)/fl(sqrt(d)) per key row (importance.py:27-33)."""
    q, k = _f64(query), _f64(keys)
    if k.ndim != 2 or q.ndim != 1 or k.shape[1] != q.shape[0]:
        raise ValueError(f"shape mismatch: keys {k.shape} vs query {q.shape}")
    out = np.empty(k.shape[0], dtype=np.float64)
    lib().ora_scores(_p(q), _p(k), k.shape[0], q.shape[0], _p(out))
    return out


def dots(query, keys) -> np.ndarray:
    """Raw canonical dots q.k (the B200 pipeline's selection key; logits = dots / sqrt d)."""
    q, k = _f64(query), _f64(keys)
    if k.ndim != 2 or q.ndim != 1 or k.shape[1] != q.shape[0]:
        raise ValueError(f"shape mismatch: keys {k.shape} vs query {q.shape}")
    out = np.empty(k.shape[0], dtype=np.float64)
    lib().ora_dots(_p(q), _p(k), k.shape[0], q.shape[0], _p(out))
    return out


def abstract(keys, start: int = 0, end: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """(max_key, min_key) of keys[start:end) (importance.py:80-87)."""
    k = _f64(keys)
    end = k.shape[0] if end is None else end
    if end <= start:
        raise ValueError(f"empty chunk [{start}, {end})")
    d = k.shape[1]
    mx, mn = np.empty(d), np.empty(d)
    lib().ora_abstract(_p(k), d, start, end, _p(mx), _p(mn))
    return mx, mn


def bounds(query, max_keys, min_keys, rows=None, scaled: bool = True) -> tuple[np.ndarray, np.ndarray]:
    """Sound canonical (U, L) per abstract row (importance.py:108-137); scaled=False gives the
    raw (unscaled) bounds the B200 pipeline prunes with."""
    q, M, N = _f64(query), _f64(max_keys), _f64(min_keys)
    if M.ndim == 1:
        M, N = M[None, :], N[None, :]
    m, d = M.shape
    U, L = np.empty(m), np.empty(m)
    r = None if rows is None else np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    lib().ora_bounds2(_p(q), _p(M), _p(N), m, d, None if r is None else _p(r, _ip), _p(U), _p(L), int(scaled))
    return U, L


def bounds_ref(query, max_keys, min_keys) -> tuple[np.ndarray, np.ndarray]:
    """(U, L) with numpy's own arithmetic (no soundness widening) -- the reference's values."""
    q, M, N = _f64(query), _f64(max_keys), _f64(min_keys)
    if M.ndim == 1:
        M, N = M[None, :], N[None, :]
    m, d = M.shape
    U, L = np.empty(m), np.empty(m)
    lib().ora_bounds_ref(_p(q), _p(M), _p(N), m, d, _p(U), _p(L))
    return U, L


def np_sum(a) -> float:
    x = _f64(a)
    return lib().ora_np_sum(_p(x), x.shape[0])


def slack_factor(d: int) -> float:
    return lib().ora_bound_slack_factor(d)


def i4_record_bytes(d: int) -> int:
    return lib().ora_i4_record_bytes(d)


def i4_quant(x) -> np.ndarray:
    """INT4 records [n, d/2 + d/8] (uint8) of f32 rows x [n, d] (DESIGN.md sec. 2 codec)."""
    X = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    n, d = X.shape
    if d % 32:
        raise ValueError("d must be a multiple of 32")
    rec = np.zeros((n, i4_record_bytes(d)), dtype=np.uint8)
    lib().ora_i4_quant(_p(X, _fp), n, d, rec.ctypes.data_as(ctypes.c_void_p))
    return rec


def i4_dequant(rec, d: int) -> np.ndarray:
    R = np.ascontiguousarray(np.asarray(rec, dtype=np.uint8))
    n = R.shape[0]
    x = np.empty((n, d), dtype=np.float32)
    lib().ora_i4_dequant(R.ctypes.data_as(ctypes.c_void_p), n, d, _p(x, _fp))
    return x


def synth_lane(n: int, d: int, seed: int, u, regions, g: dict, keys: bool = True, values: bool = True):
    """Host regeneration of one synthetic lane (csrc/synth.cu recipe) -> (K, V) f32 [n, d]
    holding the bf16 values the GPU generator writes (None where not requested).
    g: workload.gen_args(...)."""
    K = np.empty((n, d), np.float32) if keys else None
    V = np.empty((n, d), np.float32) if values else None
    uu = np.ascontiguousarray(np.asarray(u, dtype=np.float32).reshape(d))
    rr = np.ascontiguousarray(np.asarray(regions, dtype=np.int32).reshape(-1, 2))
    lib().ora_synth_lane(None if K is None else _p(K, _fp), None if V is None else _p(V, _fp), n, d,
                         int(seed) & 0xFFFFFFFF, _p(uu, _fp), rr.ctypes.data_as(_i32p), rr.shape[0],
                         g["desert_base"], g["desert_span"], g["hot_base"], g["hot_span"], g["noise_scale"],
                         g["planted"])
    return K, V


def topk(score_vec, k: int) -> np.ndarray:
    """k indices, ascending, of the top-k by (score desc, index asc)."""
    s = _f64(score_vec)
    out = np.empty(max(k, 1), dtype=np.int64)
    lib().ora_topk(_p(s), s.shape[0], k, _p(out, _ip))
    return out[:k].copy()


def select(query, keys, k: int) -> np.ndarray:
    """Brute-force exact top-k by canonical dot (score desc, index asc), ascending indices."""
    return topk(dots(query, keys), k)


def runs(sel) -> list[tuple[int, int]]:
    s = np.ascontiguousarray(np.asarray(sorted(sel), dtype=np.int64))
    k = s.shape[0]
    a, b = np.empty(max(k, 1), np.int64), np.empty(max(k, 1), np.int64)
    r = lib().ora_runs(_p(s, _ip), k, _p(a, _ip), _p(b, _ip))
    return [(int(a[i]), int(b[i])) for i in range(r)]


def canonical_partition(sel, n: int) -> list[tuple[int, int, str]]:
    """Selected runs + complement (desert) runs + trailing pad, tiling [0, next_pow2(n))."""
    n_pad = 1 << max(0, (n - 1).bit_length())
    out, pos = [], 0
    for s, e in runs(sel):
        if s > pos:
            out.append((pos, s, "desert"))
        out.append((s, e, "important"))
        pos = e
    if pos < n:
        out.append((pos, n, "desert"))
    if n < n_pad:
        out.append((n, n_pad, "pad"))
    return out


def attention(query, keys, values, idx=None) -> np.ndarray:
    """softmax(canonical logits) @ V over rows idx (engine.py:145-154)."""
    q, K, V = _f64(query), _f64(keys), _f64(values)
    if idx is None:
        idx = np.arange(K.shape[0])
    ii = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    out = np.empty(q.shape[0])
    lib().ora_attention(_p(q), _p(K), _p(V), _p(ii, _ip), ii.shape[0], q.shape[0], _p(out))
    return out


# -- chunk_tree.py restatement (branch and bound) -----------------------------------------


class BnBPartition:
    """C restatement of build_partition/select_top_k/merge_desert (chunk_tree.py:171-379)."""

    def __init__(self, keys, m: int):
        self.keys = _f64(keys)
        self.n, self.d = self.keys.shape
        self._h = lib().ora_part_new(_p(self.keys), self.n, self.d, m)
        if not self._h:
            raise ValueError(f"m={m} must be a power-of-two divisor of padded n")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().ora_part_free(h)
            self._h = None

    def select(self, query, k: int) -> tuple[list[int], int]:
        q = _f64(query)
        out = np.empty(max(k, 1), dtype=np.int64)
        ev = lib().ora_part_select(self._h, _p(q), k, _p(out, _ip))
        if ev < 0:
            raise ValueError(f"k must be in [0, {self.n}], got {k}")
        return [int(t) for t in out[:k]], int(ev)

    def merge(self) -> int:
        return int(lib().ora_part_merge(self._h))

    def leaves(self) -> list[tuple[int, int, str]]:
        nl = lib().ora_part_n_leaves(self._h)
        a, b = np.empty(nl, np.int64), np.empty(nl, np.int64)
        st = np.empty(nl, np.int32)
        lib().ora_part_leaves(self._h, _p(a, _ip), _p(b, _ip), st.ctypes.data_as(_i32p))
        return [(int(a[i]), int(b[i]), STATES[int(st[i])]) for i in range(nl)]

    def leaf_abstract(self, i: int) -> tuple[np.ndarray, np.ndarray]:
        mx, mn = np.empty(self.d), np.empty(self.d)
        lib().ora_part_leaf_abstract(self._h, i, _p(mx), _p(mn))
        return mx, mn


def bench_lanes(keys: np.ndarray, values: np.ndarray, queries: np.ndarray, k: int, m: int,
                nthreads: int, merge: bool = False, want_out: bool = False):
    """Time the reference algorithm (B&B select + attention) over independent lanes.

    keys/values: f32 [lanes, n, d]; queries: f32 [steps, lanes, d].  Returns a dict with
    wall seconds for the timed phase, evals [steps, lanes] and optional outputs.
    """
    K = np.ascontiguousarray(keys, dtype=np.float32)
    V = np.ascontiguousarray(values, dtype=np.float32)
    Q = np.ascontiguousarray(queries, dtype=np.float32)
    lanes, n, d = K.shape
    steps = Q.shape[0]
    evals = np.zeros((steps, lanes), dtype=np.int64)
    out = np.zeros((steps, lanes, d)) if want_out else None
    mx = ctypes.c_double(0.0)
    sm = ctypes.c_double(0.0)
    ls = np.zeros((steps, lanes))
    wall = lib().ora_bench_lanes(lanes, n, d, m, k, steps, int(merge), _p(K, _fp), _p(V, _fp),
                                 _p(Q, _fp), nthreads, None if out is None else _p(out),
                                 _p(evals, _ip), ctypes.byref(mx), ctypes.byref(sm), _p(ls))
    # step-synchronous wall estimate: lanes run round-robin on threads, so a step's critical
    # path is the busiest thread's sum of its lane-step times
    t = min(nthreads, lanes) if lanes else 1
    step_wall = np.array([max(ls[s, i::t].sum() for i in range(t)) for s in range(steps)]) if lanes else np.zeros(steps)
    return {"wall_s": wall, "max_thread_s": mx.value, "sum_thread_s": sm.value,
            "lane_step_s": sm.value / max(1, lanes * steps), "lane_step_times": ls, "step_wall_s": step_wall,
            "evals": evals, "out": out, "lanes": lanes, "steps": steps, "threads": nthreads}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def next_pow2(n: int) -> int:
    return 1 << max(0, (n - 1).bit_length())


def k_for(rate: float, n: int) -> int:
    """engine.py:312  k = ceil(rate * n)."""
    return math.ceil(rate * n)
