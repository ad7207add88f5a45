"""Cold-tier files: the reference's per-lane record file (`KVCF`) and
chunk-summary file (`KVAB`), written byte-identically and read with the same validation and
errors (`tiered_store.py:43-47,442-507,376-408`), plus the uploads that put their contents
in HBM for the decode kernels.

Per (layer, head) lane, under the store's cold directory (`tiered_store.py:185-189`):

  layer{L:03d}_head{H:03d}.kv    KVCF data file
      16-byte header  b"KVCF", u32 version (1), u32 n_records, u32 head_dim
      n_records x 16-byte table entries (u32 start, u32 end, u64 payload offset)
      payloads, in table order: keys f16 [end-start][d], then values f16 [end-start][d]
      (zeros when the trace has no values)
  layer{L:03d}_head{H:03d}.abs   KVAB summary file
      16-byte header  b"KVAB", u32 version (1), u32 n_records, u32 head_dim
      n_records x (u32 start, u32 end, max_key f32 [d], min_key f32 [d])

All little-endian.  The summary's extrema are exact element-wise max/min of the f32 trace
keys; `abstracts_from_device` takes them from K1 (`kvt_abstract_spans`, bit-exact) instead
of recomputing them on the host.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np

DATA_MAGIC, ABSTRACT_MAGIC, FILE_VERSION = b"KVCF", b"KVAB", 1
FILE_HEADER = struct.Struct("<4sIII")      # magic, version, n_records, head_dim
TABLE_ENTRY = struct.Struct("<IIQ")        # start, end, payload offset
SPAN = struct.Struct("<II")


class ColdStoreError(RuntimeError):
    """A cold-tier file is missing, truncated or holds a corrupt record (tiered_store.py:71-72)."""


def data_path(cold_dir: str | Path, layer: int, head: int) -> Path:
    return Path(cold_dir) / f"layer{layer:03d}_head{head:03d}.kv"


def abstract_path(cold_dir: str | Path, layer: int, head: int) -> Path:
    return Path(cold_dir) / f"layer{layer:03d}_head{head:03d}.abs"


def write_lane_files(data_file: str | Path, abstract_file: str | Path, spans: Sequence[tuple[int, int]],
                     keys: np.ndarray, values: np.ndarray | None, head_dim: int,
                     abstracts: tuple[np.ndarray, np.ndarray] | None = None) -> list[int]:
    """Write one lane's KVCF + KVAB pair (tiered_store.py:446-480); returns each record's
    payload offset.  `abstracts` = precomputed (max, min) f32 [len(spans), d] (e.g. from K1);
    default: host max/min over `keys`."""
    spans = [(int(s), int(e)) for s, e in spans]
    rec_bytes = [2 * (e - s) * head_dim * 2 for s, e in spans]
    first = FILE_HEADER.size + len(spans) * TABLE_ENTRY.size
    offsets = (first + np.concatenate([[0], np.cumsum(rec_bytes[:-1], dtype=np.int64)])).tolist() if spans else []
    with open(data_file, "wb") as fh:
        fh.write(FILE_HEADER.pack(DATA_MAGIC, FILE_VERSION, len(spans), head_dim))
        fh.write(b"".join(TABLE_ENTRY.pack(s, e, off) for (s, e), off in zip(spans, offsets)))
        for s, e in spans:
            fh.write(np.ascontiguousarray(keys[s:e], dtype=np.float16).tobytes())
            fh.write(np.zeros((e - s, head_dim), np.float16).tobytes() if values is None
                     else np.ascontiguousarray(values[s:e], dtype=np.float16).tobytes())
    if abstracts is None:
        amax = np.stack([keys[s:e].max(axis=0) for s, e in spans]).astype(np.float32) if spans else None
        amin = np.stack([keys[s:e].min(axis=0) for s, e in spans]).astype(np.float32) if spans else None
    else:
        amax, amin = (np.asarray(a, dtype=np.float32) for a in abstracts)
    with open(abstract_file, "wb") as fh:
        fh.write(FILE_HEADER.pack(ABSTRACT_MAGIC, FILE_VERSION, len(spans), head_dim))
        for i, (s, e) in enumerate(spans):
            fh.write(SPAN.pack(s, e) + amax[i].tobytes() + amin[i].tobytes())
    return [int(o) for o in offsets]


@dataclass
class LaneAbstracts:
    """A parsed KVAB file: spans int64 [n, 2] and the f32 extrema [n, d]."""

    spans: np.ndarray
    max_key: np.ndarray
    min_key: np.ndarray

    def as_chunk_abstracts(self, rows=None) -> list:
        """The reference's return type (list of f64 ChunkAbstract, tiered_store.py:505)."""
        from .importance import ChunkAbstract
        rows = range(len(self.spans)) if rows is None else rows
        return [ChunkAbstract(int(self.spans[i, 0]), int(self.spans[i, 1]),
                              self.max_key[i].astype(np.float64), self.min_key[i].astype(np.float64))
                for i in rows]


def read_abstract_file(path: str | Path, head_dim: int) -> LaneAbstracts:
    """Parse and validate a KVAB file (tiered_store.py:483-507): same checks, same errors --
    missing, shorter than the header, bad magic/version, head_dim mismatch, size not implied
    by n_records, non-finite extrema or min > max."""
    path = Path(path)
    if not path.is_file():
        raise ColdStoreError(f"missing summary file {path}")
    raw = path.read_bytes()
    if len(raw) < FILE_HEADER.size:
        raise ColdStoreError(f"summary file {path} shorter than its header")
    magic, version, n, d = FILE_HEADER.unpack_from(raw)
    if magic != ABSTRACT_MAGIC or version != FILE_VERSION:
        raise ColdStoreError(f"summary file {path} has a bad magic/version")
    if d != head_dim:
        raise ColdStoreError(f"summary file {path} head_dim {d} != expected {head_dim}")
    rec = SPAN.size + 8 * head_dim
    if len(raw) != FILE_HEADER.size + n * rec:
        raise ColdStoreError(f"summary file {path} has {len(raw)} bytes, expected {FILE_HEADER.size + n * rec}")
    body = np.frombuffer(raw, np.uint8, n * rec, FILE_HEADER.size).reshape(n, rec)
    spans = body[:, :SPAN.size].copy().view("<u4").astype(np.int64)
    ext = body[:, SPAN.size:].copy().view("<f4").reshape(n, 2, head_dim)
    amax, amin = ext[:, 0], ext[:, 1]
    bad = ~(np.isfinite(amax).all(1) & np.isfinite(amin).all(1)) | (amin > amax).any(1)
    if bad.any():
        i = int(np.flatnonzero(bad)[0])
        raise ColdStoreError(f"corrupt summary record for chunk [{spans[i, 0]}, {spans[i, 1]}) in {path}")
    return LaneAbstracts(spans, np.ascontiguousarray(amax), np.ascontiguousarray(amin))


def read_record(path: str | Path, offset: int, n_tokens: int, head_dim: int) -> tuple[np.ndarray, np.ndarray]:
    """One record's fp16 (keys, values) [n_tokens, d] (tiered_store.py:376-388; the
    file-backed `TieredStore.fetch_chunk` widens them to f32 as the reference does)."""
    path = Path(path)
    if not path.is_file():
        raise ColdStoreError(f"missing cold data file {path}")
    plane = n_tokens * head_dim * 2
    with open(path, "rb") as fh:
        fh.seek(offset)
        raw = fh.read(2 * plane)
    if len(raw) != 2 * plane:
        raise ColdStoreError(f"truncated record at offset {offset} ({n_tokens} tokens) in {path}")
    kv = np.frombuffer(raw, np.float16).reshape(2, n_tokens, head_dim)
    return kv[0], kv[1]


def read_table(path: str | Path) -> tuple[int, np.ndarray]:
    """A KVCF file's (head_dim, table int64 [n, 3] = start, end, offset), validated against
    the file size."""
    path = Path(path)
    if not path.is_file():
        raise ColdStoreError(f"missing cold data file {path}")
    size = path.stat().st_size
    with open(path, "rb") as fh:
        head = fh.read(FILE_HEADER.size)
        if len(head) < FILE_HEADER.size:
            raise ColdStoreError(f"data file {path} shorter than its header")
        magic, version, n, d = FILE_HEADER.unpack(head)
        if magic != DATA_MAGIC or version != FILE_VERSION:
            raise ColdStoreError(f"data file {path} has a bad magic/version")
        raw = fh.read(n * TABLE_ENTRY.size)
    if len(raw) != n * TABLE_ENTRY.size:
        raise ColdStoreError(f"data file {path}: truncated record table")
    t = np.frombuffer(raw, np.dtype([("s", "<u4"), ("e", "<u4"), ("o", "<u8")]))
    table = np.stack([t["s"].astype(np.int64), t["e"].astype(np.int64), t["o"].astype(np.int64)], 1)
    if n and int((table[:, 2] + 4 * (table[:, 1] - table[:, 0]) * d).max()) > size:
        raise ColdStoreError(f"data file {path}: a record runs past the end of the file")
    return d, table


# -- HBM uploads -----------------------------------------------------------------------------

def abstracts_from_device(keys, spans: Sequence[tuple[int, int]]) -> tuple[np.ndarray, np.ndarray]:
    """K1 (`kvt_abstract_spans`) over one lane's device keys [n, d] f32 -> the KVAB extrema
    (f32 [len(spans), d]); exact, so the file is byte-identical to the host writer's."""
    import torch
    from . import ops
    st = torch.tensor([s for s, _ in spans], dtype=torch.int32)
    en = torch.tensor([e for _, e in spans], dtype=torch.int32)
    amax, amin = ops.abstract_spans(keys.unsqueeze(0), torch.zeros_like(st), st, en)
    return amax.float().cpu().numpy(), amin.float().cpu().numpy()


def upload_abstracts(lane: LaneAbstracts, rows, amax_dst, amin_dst, slots) -> None:
    """Copy summary rows `rows` of a parsed KVAB file into abstract tensors [m, d] at leaf
    slots `slots`.  Destinations must be f32 or f64 (exact); a bf16 abstract has to be
    rounded outward, which only K1 does."""
    import torch
    if amax_dst.dtype not in (torch.float32, torch.float64) or amin_dst.dtype != amax_dst.dtype:
        raise TypeError(f"abstract destinations must be f32/f64, got {amax_dst.dtype}/{amin_dst.dtype}")
    rows = np.asarray(rows, np.int64)
    if rows.size == 0:
        return
    dev = amax_dst.device
    idx = torch.as_tensor(np.asarray(slots, np.int64), device=dev)
    amax_dst.index_copy_(0, idx, torch.from_numpy(lane.max_key[rows]).pin_memory().to(dev, non_blocking=True).to(amax_dst.dtype))
    amin_dst.index_copy_(0, idx, torch.from_numpy(lane.min_key[rows]).pin_memory().to(dev, non_blocking=True).to(amin_dst.dtype))


def upload_records(path: str | Path, records: Sequence[tuple[int, int, int]], head_dim: int, k_dst, v_dst) -> int:
    """Cold -> HBM for records (start, end, offset) of one lane: each payload is read from the
    KVCF file straight into one pinned staging buffer, copied to the device in one
    cudaMemcpyAsync and scattered into k_dst / v_dst [n_cap, d] at the records' token rows
    (fp16 -> destination dtype on the device).  Returns the payload bytes moved."""
    import torch
    records = sorted((int(s), int(e), int(o)) for s, e, o in records)
    if not records:
        return 0
    n_tok = sum(e - s for s, e, _ in records)
    stage = torch.empty((2 * n_tok, head_dim), dtype=torch.float16, pin_memory=True)
    buf = stage.numpy().view(np.uint8).reshape(-1)
    pos = 0
    with open(path, "rb") as fh:
        for s, e, off in records:
            nb = 2 * (e - s) * head_dim * 2
            fh.seek(off)
            if fh.readinto(memoryview(buf[pos:pos + nb])) != nb:
                raise ColdStoreError(f"truncated record [{s}, {e}) in {path}")
            pos += nb
    dev = stage.to(k_dst.device, non_blocking=True)
    r = 0
    for s, e, _ in records:
        n = e - s
        k_dst[s:e].copy_(dev[r:r + n])
        v_dst[s:e].copy_(dev[r + n:r + 2 * n])
        r += 2 * n
    return 4 * n_tok * head_dim
