"""Matrix files of the reference's cli module:
the MCAM binary format, CSV, and cmd_attn_import's validation.

MCAM (bit-exact, little-endian): 4-byte magic "MCAM", u32 version == 1, u64
rows, u64 cols, then rows*cols IEEE-754 float64, row-major. Readers reject a
bad magic / version, a payload whose length does not match the header (the
message names expected vs actual bytes), and non-finite entries
(FormatError, carrying the byte offset); attention imports also reject
negative entries (DomainError) and renormalise rows whose sums miss 1 by more
than 1e-6 (with a warning).
"""
from __future__ import annotations

import struct
import warnings

import numpy as np

MAGIC = b"MCAM"
VERSION = 1
HEADER = struct.Struct("<4sIQQ")   # 24 bytes


class FormatError(ValueError):
    """Malformed matrix file; `offset` is the byte offset of the problem."""

    def __init__(self, msg: str, offset: int):
        super().__init__(f"{msg} (byte offset {offset})")
        self.offset = offset


class DomainError(ValueError):
    """An attention entry outside [0, 1] (negative)."""


def encode_mcam(m) -> bytes:
    a = np.ascontiguousarray(np.asarray(m, dtype="<f8"))
    if a.ndim != 2:
        raise ValueError("MCAM holds a 2-D matrix")
    return HEADER.pack(MAGIC, VERSION, a.shape[0], a.shape[1]) + a.tobytes()


def decode_mcam(buf: bytes) -> np.ndarray:
    if len(buf) < HEADER.size:
        raise FormatError(f"truncated header: expected {HEADER.size} bytes, got {len(buf)}", len(buf))
    magic, version, rows, cols = HEADER.unpack_from(buf)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r} (expected b'MCAM')", 0)
    if version != VERSION:
        raise FormatError(f"unsupported version {version} (expected 1)", 4)
    want = HEADER.size + rows * cols * 8
    if len(buf) != want:
        kind = "truncated" if len(buf) < want else "oversized"
        raise FormatError(f"{kind} payload: expected {want} bytes for {rows} x {cols}, got {len(buf)}",
                          min(len(buf), want))
    a = np.frombuffer(buf, dtype="<f8", offset=HEADER.size).reshape(rows, cols).astype(np.float64)
    bad = np.flatnonzero(~np.isfinite(a))
    if bad.size:
        raise FormatError(f"non-finite entry at ({bad[0] // cols}, {bad[0] % cols})", HEADER.size + 8 * int(bad[0]))
    return a


def write_mcam(path: str, m) -> None:
    with open(path, "wb") as f:
        f.write(encode_mcam(m))


def read_mcam(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        return decode_mcam(f.read())


def read_csv(path: str) -> np.ndarray:
    """Comma-separated rows of reals ("1,0\\n0,1" is I2); ragged rows and
    unparsable or non-finite fields raise FormatError at their byte offset."""
    with open(path, "rb") as f:
        text = f.read()
    rows, off = [], 0
    for line in text.split(b"\n"):
        raw = line.rstrip(b"\r")
        if raw.strip():
            vals, pos = [], off
            for field in raw.split(b","):
                try:
                    v = float(field)
                except ValueError:
                    raise FormatError(f"not a number: {field.decode(errors='replace')!r}", pos) from None
                if not np.isfinite(v):
                    raise FormatError(f"non-finite entry {field.decode()!r}", pos)
                vals.append(v)
                pos += len(field) + 1
            if rows and len(vals) != len(rows[0]):
                raise FormatError(f"ragged row: {len(vals)} fields, expected {len(rows[0])}", off)
            rows.append(vals)
        off += len(line) + 1
    if not rows:
        raise FormatError("empty matrix", 0)
    return np.array(rows, dtype=np.float64)


def attn_import(path: str, fmt: str = "mcam", tol: float = 1e-6) -> np.ndarray:
    """cmd_attn_import: a validated attention matrix."""
    if fmt not in ("mcam", "csv"):
        raise ValueError(f"unknown format {fmt!r} (mcam or csv)")
    a = read_mcam(path) if fmt == "mcam" else read_csv(path)
    neg = np.flatnonzero(a < 0)
    if neg.size:
        r, c = divmod(int(neg[0]), a.shape[1])
        raise DomainError(f"negative attention entry {float(a[r, c])!r} at ({r}, {c})")
    s = a.sum(axis=1)
    off = np.flatnonzero(np.abs(s - 1.0) > tol)
    if off.size:
        if np.any(s <= 0):
            raise DomainError(f"attention row {int(np.flatnonzero(s <= 0)[0])} sums to 0")
        warnings.warn(f"{off.size} attention rows do not sum to 1 within {tol:g}; renormalised", stacklevel=2)
        a = a / s[:, None]
    return a
