"""Freeze the reference's cold-tier files and what its store reads back from them.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_coldfile_golden.py

kvtier.tiered_store.place_initial(trace, TierConfig(cold_dir=...)) writes one KVCF record
file and one KVAB summary file per non-pinned lane (tiered_store.py:442-480, 510-592).  For
seeded synthetic traces (regenerated bit-identically by oracle.synth in the tests) this
records the sha256 of every file, the bytes load_abstracts / fetch_chunk return
(tiered_store.py:260-289, 376-408), and the exception type each corrupted file raises.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
from kvtier import tiered_store as ts  # noqa: E402
from kvtier.trace import DesertProfile, TraceHeader, generate_synthetic  # noqa: E402

OUT = Path(__file__).resolve().parent / "coldfile_cases.json"

CASES = [
    # odd context (last record partial), values present
    {"n_layers": 3, "n_heads": 2, "head_dim": 16, "n_context": 200, "n_steps": 1, "has_values": True,
     "seed": 3, "chunk": 32, "pinned": 1, "spans": None},
    # no values (zero value planes), irregular spans
    {"n_layers": 2, "n_heads": 2, "head_dim": 8, "n_context": 96, "n_steps": 1, "has_values": False,
     "seed": 5, "chunk": 16, "pinned": 0, "spans": [[0, 10], [10, 50], [50, 51], [51, 96]]},
]

# (file kind, corruption) -> applied to lane (last layer, head 0)
CORRUPTIONS = ["abs_missing", "abs_truncated", "abs_bad_magic", "abs_head_dim", "abs_min_gt_max",
               "abs_nan", "abs_span_renamed", "kv_missing", "kv_truncated"]


def h(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def corrupt(kind: str, kv: Path, ab: Path, d: int, cold_offset: int) -> None:
    """cold_offset: payload offset of the lane's last cold record (kv_truncated cuts inside it)."""
    if kind == "abs_missing":
        ab.unlink()
    elif kind == "abs_truncated":
        ab.write_bytes(ab.read_bytes()[:-4])
    elif kind == "abs_bad_magic":
        ab.write_bytes(b"KVXX" + ab.read_bytes()[4:])
    elif kind == "abs_head_dim":
        b = bytearray(ab.read_bytes())
        b[12:16] = (d + 1).to_bytes(4, "little")
        ab.write_bytes(bytes(b))
    elif kind in ("abs_min_gt_max", "abs_nan"):
        b = bytearray(ab.read_bytes())
        rec = 8 + 8 * d
        off = 16 + rec + 8 + 4 * d            # record 1, min_key[0]
        val = np.float32(1e30) if kind == "abs_min_gt_max" else np.float32(np.nan)
        b[off:off + 4] = val.tobytes()
        ab.write_bytes(bytes(b))
    elif kind == "abs_span_renamed":
        b = bytearray(ab.read_bytes())
        b[16:20] = (7777).to_bytes(4, "little")   # record 0's start no longer matches
        ab.write_bytes(bytes(b))
    elif kind == "kv_missing":
        kv.unlink()
    elif kind == "kv_truncated":
        kv.write_bytes(kv.read_bytes()[:cold_offset + 10])


def build(c, td):
    hdr = TraceHeader(n_layers=c["n_layers"], n_heads=c["n_heads"], head_dim=c["head_dim"],
                      n_context=c["n_context"], n_steps=c["n_steps"], has_values=c["has_values"])
    trace = generate_synthetic(DesertProfile(seed=c["seed"]), hdr)
    per_lane = ts.kv_nbytes(c["n_context"], c["head_dim"])
    widest = max(e - s for s, e in c["spans"]) if c["spans"] else c["chunk"]
    rec = ts.kv_nbytes(widest, c["head_dim"])
    cfg = ts.TierConfig(hot_capacity=c["pinned"] * c["n_heads"] * per_lane + 2 * rec, warm_capacity=2 * rec,
                        cold_dir=td, early_layers_pinned=c["pinned"])
    spans = None
    if c["spans"] is not None:
        spans = {(l, hd): [tuple(s) for s in c["spans"]] for l in range(c["n_layers"]) for hd in range(c["n_heads"])}
    store = ts.place_initial(trace, cfg, chunk_size=c["chunk"], spans_by_lane=spans)
    return store, cfg


def run_case(c):
    out = {"spec": c}
    with tempfile.TemporaryDirectory() as td:
        store, cfg = build(c, td)
        out["files"] = {p.name: h(p.read_bytes()) for p in sorted(Path(td).iterdir())}
        out["config"] = {"hot_capacity": cfg.hot_capacity, "warm_capacity": cfg.warm_capacity}
        reads = []
        store.open_row(0, c["n_layers"] - 1)
        for hd in range(c["n_heads"]):
            layer = c["n_layers"] - 1
            ab = store.load_abstracts(layer, hd)
            blob = b"".join(np.array([a.start, a.end], np.int64).tobytes() + a.max_key.tobytes() + a.min_key.tobytes()
                            for a in ab)
            cold = store.cold_spans(layer, hd)
            fetched = []
            for s in cold[:2]:
                k, v = store.fetch_chunk(layer, hd, *s)
                fetched.append([list(s), h(k.astype(np.float32).tobytes() + v.astype(np.float32).tobytes())])
            reads.append({"n_abstracts": len(ab), "abstracts": h(blob), "fetched": fetched})
        row = store.close_row()
        out["reads"] = reads
        out["row"] = [row.abstract_bytes, row.cold_to_warm, row.warm_to_hot, row.hot_to_warm]
    errs = {}
    for kind in CORRUPTIONS:
        with tempfile.TemporaryDirectory() as td:
            store, _ = build(c, td)
            layer = c["n_layers"] - 1
            kv, ab = store._data_path(layer, 0), store._abstract_path(layer, 0)
            last_cold = [r for r in store._records[(layer, 0)] if r.tier == ts.COLD][-1]
            corrupt(kind, kv, ab, c["head_dim"], last_cold.offset)
            try:
                if kind.startswith("abs"):
                    store.load_abstracts(layer, 0)
                else:
                    s = store.cold_spans(layer, 0)[-1]
                    store.fetch_chunk(layer, 0, *s)
                errs[kind] = None
            except Exception as e:  # noqa: BLE001 -- the type is the fixture
                errs[kind] = type(e).__name__
    out["errors"] = errs
    return out


def main():
    OUT.write_text(json.dumps([run_case(c) for c in CASES], indent=1))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
