"""kvtier's own hot-path test expectations, run through module aliasing (INTEGRATION.md
Option A): `import kvtier.importance` etc. resolve to this package's drop-in modules, so the
test bodies read exactly like the reference's (`/root/reference/pkg/tests/test_importance.py`,
`test_chunk_tree.py`, `test_engine.py`; each test cites the line it restates).  The
reference tree is not read at run time (it does not exist on the GPU box).

Aliases: kvtier.importance / chunk_tree / engine -> paper_2506_20187_b200.importance /
chunk_tree / engine; kvtier.pipeline -> .tier; kvtier.tiered_store -> .tiered_store;
kvtier.trace -> this package's .kvtr reader/writer plus `generate_synthetic` /
`DesertProfile` from oracle/synth.py (the reference generator restated byte-identically,
tests/test_oracle_golden.py pins it).  Every test here needs the GPU (the drop-in has no CPU
path) and is marked `gpu`.
"""

from __future__ import annotations

import sys
import types

import pytest


def pytest_collection_modifyitems(config, items):
    for it in items:
        if "ref_suite" in str(it.fspath):
            it.add_marker(pytest.mark.gpu)


def _install_aliases():
    if "kvtier" in sys.modules and getattr(sys.modules["kvtier"], "__b200_alias__", False):
        return
    import numpy as np

    from oracle import synth
    from paper_2506_20187_b200 import chunk_tree, engine, importance, tier, tiered_store
    from paper_2506_20187_b200 import trace as ptrace

    tr = types.ModuleType("kvtier.trace")
    for name in dir(ptrace):
        if not name.startswith("__"):
            setattr(tr, name, getattr(ptrace, name))

    def DesertProfile(desert_rate=0.7, n_hot_regions=3, score_gap=1.0, seed=0, per_layer_density=None):
        return synth.Profile(desert_rate, n_hot_regions, score_gap, seed,
                             None if per_layer_density is None else tuple(per_layer_density))

    def generate_synthetic(profile, header):
        K, Q, V = synth.trace(profile, header.n_layers, header.n_heads, header.n_context, header.head_dim,
                              header.n_steps, with_values=header.has_values)
        return ptrace.AttentionTrace(header=header, keys=K, queries=Q, values=V)

    tr.DesertProfile = DesertProfile
    tr.generate_synthetic = generate_synthetic
    pkg = types.ModuleType("kvtier")
    pkg.__b200_alias__ = True
    pkg.__path__ = []
    mods = {"importance": importance, "chunk_tree": chunk_tree, "engine": engine, "pipeline": tier,
            "tiered_store": tiered_store, "trace": tr}
    sys.modules["kvtier"] = pkg
    for k, m in mods.items():
        sys.modules[f"kvtier.{k}"] = m
        setattr(pkg, k, m)
    del np


def pytest_configure(config):
    try:
        import torch
        if not torch.cuda.is_available():
            return
        _install_aliases()
    except ImportError:
        return


def pytest_ignore_collect(collection_path, config):
    # without a GPU the aliased modules cannot be imported: skip collecting the suite's files
    try:
        import torch
        gpu = torch.cuda.is_available()
    except ImportError:
        gpu = False
    if not gpu and collection_path.name.startswith("test_") and "ref_suite" in str(collection_path):
        return True
    return None
