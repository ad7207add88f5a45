"""Synthetic decode workload shared by bench.py's two arms and the tests (not product code).

The planted-desert model of the reference generator (`kvtier.trace.generate_synthetic`,
trace.py:270-315): per (layer, KV lane) hot regions placed like `_place_regions`
(trace.py:225-238, multinomial gaps between 3 runs, 30 % of the tokens hot), a unit
direction u, keys a_t*u + noise (desert a ~ U(-0.25, 0.25), hot a = 1.27 + U(0, 0.5)),
queries gain*u (gain ~ U(1, 2)) and N(0,1)-like values.  The per-lane scalars (regions, u,
query gains, a 32-bit lane seed) are drawn here on the host with numpy; the per-token
arrays are a counter hash of the lane seed (paper_2506_20187_b200/csrc/synth.cu on the GPU,
oracle/kvt_oracle.c `ora_synth_lane` on the host -- bit-identical), so both bench arms and
the parity check see the same tensors.  `data="random"`: N(0,1)-like keys and queries.

Pure numpy: importable by the reference arm without loading the CUDA library.
"""

from __future__ import annotations

import math

import numpy as np

DESERT_AMP = 0.25            # trace.py:215
HOT_SPAN = 0.5               # trace.py:216
PLANT_MARGIN = 0.02          # trace.py:217
SCORE_GAP = 1.0              # DesertProfile default score_gap
DESERT_RATE = 0.7
N_REGIONS = 3
F32 = np.float32
DESERT_BASE, DESERT_SPAN = F32(-DESERT_AMP), F32(2 * DESERT_AMP)
HOT_BASE, HOT_SPAN_F = F32(DESERT_AMP + SCORE_GAP + PLANT_MARGIN), F32(HOT_SPAN)


def noise_scale(d: int) -> np.float32:
    return F32(0.05 / math.sqrt(d))  # trace.py:286


def mix32(x):
    """lowbias32 on uint32 (numpy arrays or ints); synth.cu synth_mix."""
    x = np.asarray(x, dtype=np.uint32)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint32(16))
        x = (x * np.uint32(0x7FEB352D)).astype(np.uint32)
        x = x ^ (x >> np.uint32(15))
        x = (x * np.uint32(0x846CA68B)).astype(np.uint32)
        x = x ^ (x >> np.uint32(16))
    return x


def lane_seed(seed: int, layer: int, kv_lane) -> np.ndarray:
    """32-bit seed of (run seed, layer, global KV lane)."""
    s = mix32(np.uint32(seed & 0xFFFFFFFF) ^ np.uint32(0x2545F491))
    s = mix32(s ^ np.uint32(layer & 0xFFFFFFFF))
    return mix32(s ^ np.asarray(kv_lane, dtype=np.uint32))


def place_regions(rng: np.random.Generator, n: int, desert_rate: float = DESERT_RATE,
                  n_regions: int = N_REGIONS) -> list[tuple[int, int]]:
    """_plan_lane + _place_regions (trace.py:225-267): r contiguous hot runs >= 1 token apart."""
    n_hot = math.ceil((1.0 - desert_rate) * n)
    if n_hot == 0:
        return []
    r = min(n_regions, n_hot, n - n_hot + 1)
    base, extra = divmod(n_hot, r)
    sizes = [base + (1 if i < extra else 0) for i in range(r)]
    slack = n - n_hot - (r - 1)
    gaps = rng.multinomial(slack, [1.0 / (r + 1)] * (r + 1)) if slack > 0 else [0] * (r + 1)
    out, pos = [], int(gaps[0])
    for i, s in enumerate(sizes):
        out.append((pos, pos + s))
        pos += s + (1 + int(gaps[i + 1]) if i < r - 1 else 0)
    return out


def lane_params(seed: int, layer: int, kv_lanes, n: int, d: int, data: str = "planted") -> dict:
    """Per-KV-lane generator inputs for one layer: seed u32 [lanes], u f32 [lanes, d],
    regions i32 [lanes, 3, 2] (zero-length when random)."""
    kv_lanes = np.asarray(kv_lanes, dtype=np.int64)
    m = kv_lanes.shape[0]
    u = np.zeros((m, d), F32)
    reg = np.zeros((m, N_REGIONS, 2), np.int32)
    if data == "planted":
        for i, g in enumerate(kv_lanes):
            rng = np.random.default_rng([seed, layer, int(g)])
            rr = place_regions(rng, n)  # regions first, then u: the reference's draw order
            for r, (s, e) in enumerate(rr):
                reg[i, r] = (s, e)
            v = rng.normal(size=d)
            u[i] = (v / np.linalg.norm(v)).astype(F32)
    elif data != "random":
        raise ValueError(f"unknown data {data!r}")
    return {"seed": lane_seed(seed, layer, kv_lanes), "u": u, "regions": reg}


def queries(seed: int, steps: int, layer: int, q_lanes, kv_group: int, u_kv: np.ndarray, kv_lane0: int,
            d: int, data: str = "planted") -> np.ndarray:
    """f32 [steps, lanes, d] queries of one layer for global query lanes q_lanes.  Planted:
    gain*u of the lane's KV head (trace.py:309-310), gain ~ U(1, 2) per step; random: N(0,1).
    u_kv holds the directions of global KV lanes kv_lane0, kv_lane0 + 1, ..."""
    q_lanes = np.asarray(q_lanes, dtype=np.int64)
    out = np.empty((steps, q_lanes.shape[0], d), F32)
    for i, g in enumerate(q_lanes):
        rng = np.random.default_rng([seed, layer, int(g), 1])
        if data == "planted":
            gains = rng.uniform(1.0, 2.0, size=steps)
            uk = u_kv[int(g) // kv_group - kv_lane0].astype(np.float64)
            out[:, i] = (gains[:, None] * uk[None, :]).astype(F32)
        else:
            out[:, i] = rng.normal(size=(steps, d)).astype(F32)
    return out


def gen_args(p: dict, d: int, data: str) -> dict:
    """Scalar arguments of kvt_synth_layer / ora_synth_lane for these lane params."""
    return {"desert_base": DESERT_BASE, "desert_span": DESERT_SPAN, "hot_base": HOT_BASE,
            "hot_span": HOT_SPAN_F, "noise_scale": noise_scale(d), "planted": int(data == "planted"),
            "n_regions": N_REGIONS}
