"""Drop-in for the hot-path part of kvtier.engine (engine.py:145-219): sparse attention
output over a selected set, its quality metrics and the selected-token runs, on the B200.

`attention_output` gathers the selected V rows with K7 (`kvt_sparse_decode_attn`) using the
canonical logits from K4 (keys are scored once).  This drop-in widens V to f64 and
accumulates in f64 like the reference (engine.py:149-154); the batched decode path keeps
bf16/f32 values with f32 accumulation (tolerance 1e-2 / 2e-3, BASELINE.json north_star).
The decode loop, its reports and the ablation ladder (engine.py:48-532) are in `runner.py`
on the batched GPU selection path and re-exported here.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import ops
from .importance import attention_logits, score_tokens, softmax, to_device

__all__ = ["attention_output", "oracle_output", "cosine_similarity", "desert_rate_on_grid", "token_runs"]


def attention_output(query: np.ndarray, keys: np.ndarray, values: np.ndarray) -> np.ndarray:
    """softmax(q.K^T / sqrt d) @ V over exactly the given rows (engine.py:145-154)."""
    if values is None:
        raise ValueError("attention output requires value vectors")
    K = np.asarray(keys)
    V = np.asarray(values)
    if K.shape != V.shape:
        raise ValueError(f"keys shape {K.shape} != values shape {V.shape}")
    q = np.asarray(query)
    if K.ndim != 2 or q.ndim != 1 or K.shape[1] != q.shape[0]:
        raise ValueError(f"shape mismatch: keys {K.shape} vs query {q.shape}")
    n, d = K.shape
    if n == 0:  # softmax([]) @ V[0, d] is zeros(d) in the reference (engine.py:149-154)
        return np.zeros(d)
    qd = to_device(q, torch.float64)[None]
    kd = to_device(K)[None]
    vd = to_device(V, torch.float64)[None]  # f64 accumulation, as the reference (engine.py:150)
    logits = ops.token_scores(qd, kd, n)                                   # K4
    sel = torch.arange(n, dtype=torch.int32, device=qd.device)[None]
    ns = torch.tensor([n], dtype=torch.int32, device=qd.device)
    out, out64 = ops.sparse_decode_attn(vd, sel, logits.contiguous(), ns, want_f64=True, logit_scale=1.0)  # K7
    return out64[0].cpu().numpy()


def oracle_output(query: np.ndarray, keys: np.ndarray, values: np.ndarray) -> np.ndarray:
    """Full-cache attention output, same arithmetic (engine.py:157-159)."""
    return attention_output(query, keys, values)


def cosine_similarity(a: np.ndarray, b: np.ndarray) -> float:
    """engine.py:162-166."""
    ta, tb = to_device(a, torch.float64), to_device(b, torch.float64)
    na, nb = float(torch.linalg.norm(ta)), float(torch.linalg.norm(tb))
    if na == 0.0 or nb == 0.0:
        return 1.0 if na == nb else 0.0
    return float(torch.dot(ta, tb)) / (na * nb)


def desert_rate_on_grid(selected: set[int], n: int, grid: int) -> float:
    """Fraction of fixed-size cells holding no selected token (engine.py:169-173)."""
    n_cells = math.ceil(n / grid)
    important = {t // grid for t in selected}
    return 1.0 - len(important) / n_cells


def token_runs(tokens) -> list[tuple[int, int]]:
    """Selected tokens -> contiguous runs (engine.py:176-183), via K6 on device."""
    toks = sorted(int(t) for t in tokens)
    if not toks:
        return []
    st = torch.tensor(toks, dtype=torch.int32, device=to_device(np.zeros(1)).device)[None]
    ns = torch.tensor([len(toks)], dtype=torch.int32, device=st.device)
    r = ops.runs_scan(st, ns, toks[-1] + 1, want_partition=False)
    nr = int(r["n_runs"][0])
    s = r["run_start"][0, :nr].cpu().numpy()
    ln = r["run_len"][0, :nr].cpu().numpy()
    return [(int(a), int(a + b)) for a, b in zip(s, ln)]


_token_runs = token_runs


from .runner import (ABLATE_COLUMNS, ABLATION_ROWS, STEP_COLUMNS, RunConfig, RunReport, StepRow,  # noqa: E402
                     ablate, ablation_table, default_tier, run, run_and_report, write_ablation, write_report)

__all__ += ["ABLATE_COLUMNS", "ABLATION_ROWS", "STEP_COLUMNS", "RunConfig", "RunReport", "StepRow", "ablate",
            "ablation_table", "default_tier", "run", "run_and_report", "write_ablation", "write_report"]
