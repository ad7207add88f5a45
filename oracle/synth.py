"""Planted-desert synthetic lanes: a restatement of the reference input generator.

TEST INFRASTRUCTURE ONLY (input generator for parity fixtures and the bench's CPU sample).

Follows `kvtier.trace.generate_synthetic` (trace.py:270-315) with its helpers
`_split_region_sizes` (:220-222), `_place_regions` (:225-238), `_lane_rng` (:252-253) and
`_plan_lane` (:256-267).  The draw order on the per-lane generator
`np.random.default_rng([seed, layer, head])` is what makes a lane bit-identical to the
reference's: (multinomial gaps) -> u ~ N(0,1)^d -> desert amps U(-0.25, 0.25)^n ->
hot amps U(0, 0.5)^n_hot -> noise N(0, (0.05/sqrt d)^2)^{n x d} -> step gains U(1, 2)^S
-> values N(0,1)^{n x d}.  tests/test_oracle_golden.py checks byte equality against the
reference here and against committed digests on the GPU box.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DESERT_AMP = 0.25   # trace.py:215
HOT_SPAN = 0.5      # trace.py:216
PLANT_MARGIN = 0.02  # trace.py:217


@dataclass(frozen=True)
class Profile:
    """Mirror of DesertProfile (trace.py:70-104)."""

    desert_rate: float = 0.7
    n_hot_regions: int = 3
    score_gap: float = 1.0
    seed: int = 0
    per_layer_density: tuple[float, ...] | None = None


def _region_sizes(n_hot: int, r: int) -> list[int]:
    q, rem = divmod(n_hot, r)
    return [q + 1 if i < rem else q for i in range(r)]


def _regions(rng: np.random.Generator, n: int, sizes: list[int]) -> list[tuple[int, int]]:
    r = len(sizes)
    free = n - sum(sizes) - (r - 1)
    if free > 0:
        gaps = rng.multinomial(free, [1.0 / (r + 1)] * (r + 1))
    else:
        gaps = [0] * (r + 1)
    out, pos = [], int(gaps[0])
    for i, sz in enumerate(sizes):
        out.append((pos, pos + sz))
        pos += sz + (1 + int(gaps[i + 1]) if i < r - 1 else 0)
    return out


def _plan(rng, prof: Profile, n: int, layer: int):
    if prof.per_layer_density is not None:
        frac = prof.per_layer_density[layer % len(prof.per_layer_density)]
    else:
        frac = 1.0 - prof.desert_rate
    n_hot = math.ceil(frac * n)
    if n_hot == 0:
        return [], 0
    r = min(prof.n_hot_regions, n_hot, n - n_hot + 1)
    return _regions(rng, n, _region_sizes(n_hot, r)), n_hot


def lane(prof: Profile, layer: int, head: int, n: int, d: int, n_steps: int,
         with_values: bool = True):
    """One (layer, head) lane: keys f32 [n,d], queries f32 [n_steps,d], values f32 or None,
    and the planted hot regions."""
    rng = np.random.default_rng([prof.seed, layer, head])
    regions, n_hot = _plan(rng, prof, n, layer)
    u = rng.normal(size=d)
    u /= np.linalg.norm(u)
    amps = rng.uniform(-DESERT_AMP, DESERT_AMP, size=n)
    if n_hot:
        hot = (DESERT_AMP + prof.score_gap + PLANT_MARGIN) + rng.uniform(0.0, HOT_SPAN, size=n_hot)
        pos = 0
        for s, e in regions:
            amps[s:e] = hot[pos:pos + (e - s)]
            pos += e - s
    noise = rng.normal(scale=0.05 / math.sqrt(d), size=(n, d))
    noise -= np.outer(noise @ u, u)
    keys = (amps[:, None] * u[None, :] + noise).astype(np.float32)
    gains = rng.uniform(1.0, 2.0, size=n_steps)
    queries = (gains[:, None] * u[None, :]).astype(np.float32)
    values = rng.normal(size=(n, d)).astype(np.float32) if with_values else None
    return keys, queries, values, regions


def trace(prof: Profile, n_layers: int, n_heads: int, n: int, d: int, n_steps: int,
          with_values: bool = False):
    """Whole trace in the reference layout: keys [L,H,N,D], queries [S,L,H,D], values."""
    K = np.empty((n_layers, n_heads, n, d), np.float32)
    Q = np.empty((n_steps, n_layers, n_heads, d), np.float32)
    V = np.empty((n_layers, n_heads, n, d), np.float32) if with_values else None
    for l in range(n_layers):
        for h in range(n_heads):
            k, q, v, _ = lane(prof, l, h, n, d, n_steps, with_values)
            K[l, h] = k
            Q[:, l, h] = q
            if with_values:
                V[l, h] = v
    return K, Q, V
