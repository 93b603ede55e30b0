"""Compact storage for the bench-scale golden fixtures (test infrastructure).

Range grids of full-size frames are mostly noise in the low mantissa bits, so
they are stored as a packed validity bitmask plus the finite values,
byte-shuffled (all first bytes, then all second bytes, ...) and
lzma-compressed -- lossless, about 5-6 bytes per valid cell instead of 8 per
cell.  Large reference outputs that must be bit-exact but are not needed
cell by cell (neighbour slots, fp64 normals) are pinned by SHA-256 digests of
their canonical bytes; labels are stored as arrays (they compress well and
show where a mismatch is).
"""

from __future__ import annotations

import hashlib
import lzma

import numpy as np


def pack_ranges(ranges: np.ndarray) -> dict:
    r = np.ascontiguousarray(ranges, dtype=np.float64)
    fin = ~np.isnan(r)
    vals = r[fin]
    shuf = vals.view(np.uint8).reshape(-1, 8).T.copy()  # byte planes
    blob = lzma.compress(shuf.tobytes(), preset=9)
    return {"r_shape": np.array(r.shape, np.int64), "r_fin": np.packbits(fin.ravel()),
            "r_blob": np.frombuffer(blob, np.uint8)}


def unpack_ranges(d: dict) -> np.ndarray:
    shape = tuple(int(v) for v in d["r_shape"])
    n = int(np.prod(shape))
    fin = np.unpackbits(d["r_fin"])[:n].astype(bool)
    raw = np.frombuffer(lzma.decompress(d["r_blob"].tobytes()), np.uint8)
    vals = raw.reshape(8, -1).T.copy().view(np.float64).ravel()
    out = np.full(n, np.nan)
    out[fin] = vals
    return out.reshape(shape)


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype.str).encode())
    h.update(str(a.shape).encode())
    h.update(a.tobytes())
    return h.hexdigest()


def normals_digest(values: np.ndarray, mask: np.ndarray, dtype=np.float64) -> str:
    """Digest of (mask, normals of the masked nodes) in `dtype` (absent rows
    excluded, so NaN payloads do not matter)."""
    m = np.asarray(mask, bool)
    v = np.asarray(values)[m].astype(dtype)
    return digest(np.packbits(m)) + digest(v)


def near_threshold_edges(neighbors, values, mask, thr, eps=1e-4):
    """|E_near|: forward edges (slots N0..N2) between nodes
    with normals where some component's |dn_c| is within eps of T_c."""
    nb = np.asarray(neighbors)[:, :3]
    v = np.asarray(values, np.float64)
    m = np.asarray(mask, bool)
    p = np.repeat(np.arange(nb.shape[0]), 3)
    q = nb.ravel()
    ok = (q >= 0)
    p, q = p[ok], q[ok]
    ok = m[p] & m[q]
    p, q = p[ok], q[ok]
    d = np.abs(v[p] - v[q])
    near = (np.abs(d - np.asarray(thr, np.float64)[None, :]) < eps).any(axis=1)
    return int(near.sum()), int(p.size)
