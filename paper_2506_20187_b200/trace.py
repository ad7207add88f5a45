"""`.kvtr` attention traces: the reference's binary container
(`trace.py:1-200`), read memory-mapped so large traces stream into the decoder without a
full host copy, and written byte-identically.

Container (`trace.py:7-13`), little-endian:
    32-byte header  b"KVTR", then 7 x u32: version, n_layers, n_heads, head_dim, n_context,
                    n_steps, flags (bit 0: values present)
    keys     f32 [n_layers][n_heads][n_context][head_dim]
    values   f32 (same shape, only with flag bit 0)
    queries  f32 [n_steps][n_layers][n_heads][head_dim]
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

MAGIC, VERSION, FLAG_HAS_VALUES = b"KVTR", 1, 0x1
_HDR = struct.Struct("<4s7I")
HEADER_BYTES = _HDR.size


class TraceFormatError(ValueError):
    """The bytes are not a well-formed trace (trace.py:35-36)."""


@dataclass(frozen=True)
class TraceHeader:
    n_layers: int
    n_heads: int
    head_dim: int
    n_context: int
    n_steps: int
    has_values: bool = False

    def keys_shape(self) -> tuple[int, int, int, int]:
        return (self.n_layers, self.n_heads, self.n_context, self.head_dim)

    def queries_shape(self) -> tuple[int, int, int, int]:
        return (self.n_steps, self.n_layers, self.n_heads, self.head_dim)

    def expected_nbytes(self) -> int:
        kv = int(np.prod(self.keys_shape())) * (2 if self.has_values else 1)
        return HEADER_BYTES + 4 * (kv + int(np.prod(self.queries_shape())))


@dataclass
class AttentionTrace:
    header: TraceHeader
    keys: np.ndarray            # f32 [L][H][N][D]
    queries: np.ndarray         # f32 [S][L][H][D]
    values: np.ndarray | None = None


def _header(blob) -> TraceHeader:
    if len(blob) < HEADER_BYTES:
        raise TraceFormatError(f"{len(blob)} bytes: shorter than the {HEADER_BYTES}-byte header")
    magic, version, L, H, D, N, S, flags = _HDR.unpack_from(blob)
    if magic != MAGIC:
        raise TraceFormatError(f"not a trace (magic {magic!r})")
    if version != VERSION:
        raise TraceFormatError(f"trace version {version} (supported: {VERSION})")
    if flags & ~FLAG_HAS_VALUES:
        raise TraceFormatError(f"unknown flag bits {flags & ~FLAG_HAS_VALUES:#x}")
    return TraceHeader(L, H, D, N, S, bool(flags & FLAG_HAS_VALUES))


def read_trace(path: str | Path, mmap: bool = True) -> AttentionTrace:
    """Parse a .kvtr file (trace.py:156-177).  mmap=True maps the file read-only, so keys and
    values are paged in as the decoder copies each layer to the GPU."""
    path = Path(path)
    raw = np.memmap(path, dtype=np.uint8, mode="r") if mmap else np.frombuffer(path.read_bytes(), dtype=np.uint8)
    h = _header(bytes(raw[:HEADER_BYTES]))
    if raw.size != h.expected_nbytes():
        raise TraceFormatError(f"{path.name}: {raw.size} bytes, the header implies {h.expected_nbytes()}")
    f32 = raw[HEADER_BYTES:].view("<f4")
    nk, nq = int(np.prod(h.keys_shape())), int(np.prod(h.queries_shape()))
    keys = f32[:nk].reshape(h.keys_shape())
    values = f32[nk:2 * nk].reshape(h.keys_shape()) if h.has_values else None
    off = nk * (2 if h.has_values else 1)
    queries = f32[off:off + nq].reshape(h.queries_shape())
    return AttentionTrace(h, keys, queries, values)


def write_trace(trace: AttentionTrace, path: str | Path) -> int:
    """Serialize (trace.py:107-133); byte-identical to the reference writer."""
    h = trace.header
    parts = [np.ascontiguousarray(trace.keys, dtype="<f4")]
    if h.has_values:
        if trace.values is None:
            raise TraceFormatError("the header declares values but there are none")
        parts.append(np.ascontiguousarray(trace.values, dtype="<f4"))
    parts.append(np.ascontiguousarray(trace.queries, dtype="<f4"))
    shapes = [h.keys_shape()] * (len(parts) - 1) + [h.queries_shape()]
    for a, shp in zip(parts, shapes):
        if a.shape != shp:
            raise TraceFormatError(f"array shape {a.shape} does not match the header's {shp}")
    blob = _HDR.pack(MAGIC, VERSION, h.n_layers, h.n_heads, h.head_dim, h.n_context, h.n_steps,
                     FLAG_HAS_VALUES if h.has_values else 0) + b"".join(a.tobytes() for a in parts)
    Path(path).write_bytes(blob)
    return len(blob)
