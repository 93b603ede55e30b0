"""CPU oracle for the lidarseg hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain NumPy restatement of the reference package's per-scan
pipeline (``/root/reference/pkg/src/lidarseg``).  It exists so that the CUDA
path in ``paper_2005_02704_b200`` can be checked for parity on identical
inputs.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` leg may import it; the product path never
does (it fails loudly when its CUDA library is missing).

Pinning: every function below is checked against golden vectors produced by
running the *reference itself* (``tests/golden/make_golden.py`` imports the
reference read-only in the build container and stores inputs + outputs as
``tests/golden/*.npz``); see ``tests/test_oracle_golden.py``.  ``bin_points``
has no reference counterpart; it is pinned by round-trip and
known-answer tests instead.

Arithmetic order matters: the GPU kernels reproduce these exact IEEE fp64
operation sequences (no FMA contraction), so the restatement spells each one
out rather than leaning on library helpers whose association could change.
"""

from __future__ import annotations

import numpy as np

TWO_PI = 2.0 * np.pi
MIN_ACCUM = 1e-12  # reference normals.py:22
# Forward/backward slot displacements (dring, dpos); reference mesh.py:27.
SLOTS = ((1, 0), (1, 1), (0, 1), (-1, 0), (-1, -1), (0, -1))


# ---------------------------------------------------------------- data model
def ray_tables(elevations: np.ndarray, steps: int):
    """cos/sin of ring elevations and of the full azimuth table.

    Follows reference scan.py:119-121 (phi = 2*pi*j/S evaluated as
    ``(2*pi*j)/S``) and scan.py:130-139 (dir = (ct*cp, ct*sp, st)).
    """
    theta = np.asarray(elevations, dtype=np.float64)
    phi = 2.0 * np.pi * np.arange(steps) / steps
    return np.cos(theta), np.sin(theta), np.cos(phi), np.sin(phi)


def ray_directions(elevations, steps):
    """(R, S, 3) unit beam directions, reference scan.py:130-139."""
    ct, st, cp, sp = ray_tables(elevations, steps)
    out = np.empty((ct.size, steps, 3))
    out[:, :, 0] = ct[:, None] * cp[None, :]
    out[:, :, 1] = ct[:, None] * sp[None, :]
    out[:, :, 2] = st[:, None]
    return out


def valid_mask(ranges, r_min, r_max):
    """Reference scan.py:177-182: finite and inside [r_min, r_max] inclusive."""
    r = np.asarray(ranges)
    with np.errstate(invalid="ignore"):
        return np.isfinite(r) & (r >= r_min) & (r <= r_max)


def subsample_steps(steps: int, interval: int) -> np.ndarray:
    """Reference scan.py:215-225: kept steps {0, k, 2k, ...} <= S-1."""
    interval = int(interval)
    if not (1 <= interval <= steps - 1):
        raise ValueError(f"interval {interval} not in [1, {steps - 1}]")
    return np.arange(0, steps, interval, dtype=np.int64)


# ---------------------------------------------------------------- binning
def bin_points(xyz, ring, rings, steps, r_min, r_max):
    """Scatter float32 points into an (R, S) float64 range grid.

    New op (no reference function; inverse of reference scan.py:192-195).
    Definition:
      r    = sqrt((x*x + y*y) + z*z) in fp64 from the f32 inputs
      phi  = atan2(y, x) in fp64, + 2*pi when negative
      step = rint((phi * S) / (2*pi)) mod S      (round half to even)
      cell = ring * S + step
    Points whose r is non-finite or outside [r_min, r_max], or whose ring is
    outside [0, R), are not binned.  On a collision the smallest r wins (the
    lowest point index among equal r, which yields the same value).  Cells
    that receive nothing are NaN.  Returns (ranges, cell) where cell[p] is the
    cell of point p or -1 when it was not binned.
    """
    xyz = np.asarray(xyz, dtype=np.float32).reshape(-1, 3)
    ring = np.asarray(ring, dtype=np.int64).reshape(-1)
    x = xyz[:, 0].astype(np.float64)
    y = xyz[:, 1].astype(np.float64)
    z = xyz[:, 2].astype(np.float64)
    r = np.sqrt((x * x + y * y) + z * z)
    phi = np.arctan2(y, x)
    phi = np.where(phi < 0.0, phi + TWO_PI, phi)
    step = np.rint((phi * steps) / TWO_PI).astype(np.int64) % steps
    ok = np.isfinite(r) & (r >= r_min) & (r <= r_max) & (ring >= 0) & (ring < rings)
    cell = np.where(ok, ring * steps + step, -1)
    flat = np.full(rings * steps, np.inf)
    np.minimum.at(flat, cell[ok], r[ok])
    flat[np.isinf(flat)] = np.nan
    return flat.reshape(rings, steps), cell.astype(np.int32)


# ---------------------------------------------------------------- mesh
def node_positions_grid(ranges, elevations, kept):
    """(R, S', 3) positions dir*r at kept steps; reference normals.py:42-46."""
    dirs = ray_directions(elevations, ranges.shape[1])[:, kept]
    return dirs * np.asarray(ranges)[:, kept, None]


def _norm3(v):
    """Row norms with numpy's association sqrt((x*x + y*y) + z*z)."""
    s = v * v
    return np.sqrt((s[..., 0] + s[..., 1]) + s[..., 2])


def build_mesh(ranges, elevations, interval, r_min, r_max, max_edge_length=None):
    """Reference mesh.py:83-136 restated.

    Returns dict with kept_steps (S',), node_ids (R, S') i32 (-1 absent),
    neighbors (N, 6) i32 slots N0..N5, node_rings (N,) i32, node_steps (N,) i64.
    """
    ranges = np.asarray(ranges, dtype=np.float64)
    R, S = ranges.shape
    kept = subsample_steps(S, interval)
    valid = valid_mask(ranges, r_min, r_max)[:, kept]
    Sk = kept.size
    ids = np.full((R, Sk), -1, dtype=np.int32)
    n = int(valid.sum())
    ids[valid] = np.arange(n, dtype=np.int32)
    grid_nb = np.full((R, Sk, 6), -1, dtype=np.int32)
    for s, (dr, dp) in enumerate(SLOTS):
        cols = (np.arange(Sk) + dp) % Sk          # kept-position wrap
        shifted = ids[:, cols]
        if dr == 1:
            grid_nb[:-1, :, s] = shifted[1:]
        elif dr == -1:
            grid_nb[1:, :, s] = shifted[:-1]
        else:
            grid_nb[:, :, s] = shifted
    grid_nb[~valid] = -1
    if Sk == 2:  # reference mesh.py:96-101: drop a slot repeating an earlier one
        for s in range(1, 6):
            cur = grid_nb[:, :, s]
            dup = (cur >= 0) & (cur[..., None] == grid_nb[:, :, :s]).any(axis=-1)
            cur[dup] = -1
    neighbors = grid_nb[valid]
    node_rings, node_pos = np.nonzero(valid)
    if max_edge_length is not None and n:
        pts = node_positions_grid(ranges, elevations, kept)[valid]
        other = np.where(neighbors >= 0, neighbors, 0)
        d = _norm3(pts[other] - pts[:, None, :])
        neighbors = np.where((neighbors >= 0) & (d <= max_edge_length), neighbors, -1).astype(np.int32)
    return {
        "kept_steps": kept,
        "node_ids": ids,
        "neighbors": neighbors.astype(np.int32),
        "node_rings": node_rings.astype(np.int32),
        "node_steps": kept[node_pos].astype(np.int64),
        "rings": R,
        "full_steps": S,
        "interval": int(interval),
    }


def mesh_triangles(node_ids):
    """Reference mesh.py:173-189: all type-A (p, down, diag) faces in row-major
    order, then all type-B (p, diag, right) faces."""
    ids = np.asarray(node_ids)
    down = np.full_like(ids, -1)
    down[:-1] = ids[1:]
    diag = np.concatenate([down[:, 1:], down[:, :1]], axis=1)
    right = np.concatenate([ids[:, 1:], ids[:, :1]], axis=1)
    faces = []
    for a, b, c in ((ids, down, diag), (ids, diag, right)):
        a, b, c = a.ravel(), b.ravel(), c.ravel()
        ok = (a >= 0) & (b >= 0) & (c >= 0)
        faces.append(np.stack([a[ok], b[ok], c[ok]], axis=1))
    return np.concatenate(faces, axis=0).astype(np.int32)


# ---------------------------------------------------------------- normals
def _cross(a, b):
    """np.cross operation order: a1*b2 - a2*b1, a2*b0 - a0*b2, a0*b1 - a1*b0."""
    return np.stack([a[:, 1] * b[:, 2] - a[:, 2] * b[:, 1],
                     a[:, 2] * b[:, 0] - a[:, 0] * b[:, 2],
                     a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]], axis=1)


def estimate_normals(ranges, elevations, mesh):
    """Reference normals.py:94-145 restated with the same fp64 op order.

    Per node: existing slots in N0..N5 order (count c); pairs (0,1) if c == 2,
    else (k, k+1 mod c); w = 1/(|Va|+|Vb|) (0 when the sum is 0);
    mean = (sum w*(Va x Vb)) / (sum w); present iff c>=2, wsum>0 and
    |mean| >= 1e-12; unit = mean/|mean|, negated when unit.pos > 0.
    """
    nb = mesh["neighbors"]
    n = nb.shape[0]
    if n == 0:
        return np.zeros((0, 3)), np.zeros(0, dtype=bool)
    pos = node_positions_grid(ranges, elevations, mesh["kept_steps"])[mesh["node_ids"] >= 0]
    exists = nb >= 0
    counts = exists.sum(axis=1)
    node_of, slot_of = np.nonzero(exists)
    ent = np.arange(node_of.size)
    start = np.concatenate([[0], np.cumsum(counts)])
    k_in = ent - start[node_of]
    last = k_in == counts[node_of] - 1
    succ = np.where(last, start[node_of], ent + 1)
    c = counts[node_of]
    keep = (c >= 3) | ((c == 2) & (k_in == 0))
    a_idx, b_idx = ent[keep], succ[keep]
    owner = node_of[a_idx]
    q = pos[nb[node_of, slot_of]]
    va = q[a_idx] - pos[owner]
    vb = q[b_idx] - pos[owner]
    cr = _cross(va, vb)
    length = _norm3(va) + _norm3(vb)
    with np.errstate(divide="ignore"):
        w = np.where(length > 0.0, 1.0 / length, 0.0)
    # bincount accumulates sequentially in pair order starting from 0.0
    wsum = np.bincount(owner, weights=w, minlength=n)
    acc = np.stack([np.bincount(owner, weights=w * cr[:, j], minlength=n) for j in range(3)], axis=1)
    with np.errstate(invalid="ignore", divide="ignore"):
        mean = acc / wsum[:, None]
        mag = _norm3(mean)
        unit = mean / mag[:, None]
    mask = (counts >= 2) & (wsum > 0.0) & (mag >= MIN_ACCUM)
    u0 = np.nan_to_num(unit)
    dot = (u0[:, 0] * pos[:, 0] + u0[:, 2] * pos[:, 2]) + u0[:, 1] * pos[:, 1]
    unit[dot > 0.0] *= -1.0
    values = np.full((n, 3), np.nan)
    values[mask] = unit[mask]
    return values, mask


# ---------------------------------------------------------------- segmentation
def pass_table(neighbors, values, mask, thresholds):
    """Reference segment.py:54-61: directed-edge threshold test (strict)."""
    nb = np.asarray(neighbors)
    safe = np.where(nb >= 0, nb, 0)
    ok = (nb >= 0) & mask[safe] & mask[:, None]
    with np.errstate(invalid="ignore"):
        diff = np.abs(values[safe] - values[:, None, :])
        return ok & np.all(diff < np.asarray(thresholds, dtype=np.float64), axis=-1)


def segment_nodes(neighbors, values, mask, thresholds):
    """Reference segment.py:63-84 restated: row-major seeds, stack DFS in slot
    order.  Returns per-node labels (0 for nodes without a normal)."""
    nb = np.asarray(neighbors)
    n = nb.shape[0]
    lab = [0] * n
    if n == 0:
        return np.zeros(0, dtype=np.int32)
    passes = pass_table(nb, values, mask, thresholds).tolist()
    nbl = nb.tolist()
    has = np.asarray(mask).tolist()
    cur = 0
    for seed in range(n):
        if lab[seed] or not has[seed]:
            continue
        cur += 1
        lab[seed] = cur
        todo = [seed]
        while todo:
            p = todo.pop()
            row, ok = nbl[p], passes[p]
            for s in range(6):
                q = row[s]
                if q >= 0 and ok[s] and lab[q] == 0:
                    lab[q] = cur
                    todo.append(q)
    return np.asarray(lab, dtype=np.int32)


def segment(mesh, values, mask, thresholds):
    """Dense (R, S) label grid, labels at node cells; reference segment.py:86-88."""
    lab = segment_nodes(mesh["neighbors"], values, mask, thresholds)
    dense = np.zeros((mesh["rings"], mesh["full_steps"]), dtype=np.int32)
    dense[mesh["node_rings"], mesh["node_steps"]] = lab
    return dense


def nearest_donor_steps(donors, targets, width):
    """Reference segment.py:91-106: nearest donor under cyclic step distance;
    ties go to the smaller actual step index."""
    donors = np.asarray(donors)
    targets = np.asarray(targets)
    ext = np.concatenate([donors - width, donors, donors + width])
    at = np.searchsorted(ext, targets)
    lo, hi = ext[at - 1], ext[at]
    dl, dr = targets - lo, hi - targets
    ls, rs = lo % width, hi % width
    return np.where(dl < dr, ls, np.where(dr < dl, rs, np.minimum(ls, rs)))


def backfill(valid, labels):
    """Reference segment.py:109-124 (reads the pre-backfill row; no cascade)."""
    labels = np.asarray(labels)
    out = labels.copy()
    width = labels.shape[1]
    for i in range(labels.shape[0]):
        row = labels[i]
        donors = np.flatnonzero(row > 0)
        targets = np.flatnonzero(valid[i] & (row == 0))
        if donors.size and targets.size:
            out[i, targets] = row[nearest_donor_steps(donors, targets, width)]
    return out


def prune_small(labels, min_segment_size):
    """Reference segment.py:127-160."""
    labels = np.asarray(labels)
    if min_segment_size <= 0:
        return labels.copy()
    counts = np.bincount(labels.ravel())
    small = np.zeros(counts.size, dtype=bool)
    small[1:] = counts[1:] < min_segment_size
    if counts.size <= 1 or not small.any():
        return labels.copy()
    out = labels.copy()
    gone = small[labels]
    width = labels.shape[1]
    for i in range(labels.shape[0]):
        targets = np.flatnonzero(gone[i])
        if targets.size == 0:
            continue
        row = labels[i]
        donors = np.flatnonzero((row > 0) & ~gone[i])
        if donors.size == 0:
            out[i, targets] = 0
        else:
            out[i, targets] = row[nearest_donor_steps(donors, targets, width)]
    keep = np.unique(out)
    keep = keep[keep > 0]
    remap = np.zeros(counts.size, dtype=np.int32)
    remap[keep] = np.arange(1, keep.size + 1, dtype=np.int32)
    return remap[out]


# ---------------------------------------------------------------- pipeline
def run_pipeline(ranges, elevations, interval, r_min, r_max,
                 thresholds=(0.2, 0.2, 0.2), min_segment_size=10):
    """Reference pipeline.py:47-70: mesh -> normals -> segment -> backfill -> prune.

    Returns dict(mesh, normals, mask, node_labels (dense, pre-completion), labels).
    """
    mesh = build_mesh(ranges, elevations, interval, r_min, r_max)
    values, mask = estimate_normals(ranges, elevations, mesh)
    node_dense = segment(mesh, values, mask, thresholds)
    labels = backfill(valid_mask(ranges, r_min, r_max), node_dense)
    labels = prune_small(labels, min_segment_size)
    return {"mesh": mesh, "normals": values, "mask": mask,
            "node_labels": node_dense, "labels": labels}


def run_from_points(xyz, ring, elevations, steps, interval, r_min, r_max,
                    thresholds=(0.2, 0.2, 0.2), min_segment_size=10):
    """bin_points followed by run_pipeline (the full hot path, one frame)."""
    ranges, cell = bin_points(xyz, ring, len(elevations), steps, r_min, r_max)
    out = run_pipeline(ranges, elevations, interval, r_min, r_max, thresholds, min_segment_size)
    out["ranges"] = ranges
    out["cell"] = cell
    return out


# ---------------------------------------------------------------- evaluation
def extract_edges(labels):
    """Reference evaluate.py:40-55: labelled cells with a differently labelled
    (nonzero) 4-neighbour; azimuth wraps, rings clamp."""
    lab = np.asarray(labels)
    pos = lab > 0
    edge = np.zeros(lab.shape, dtype=bool)
    for sh in (1, -1):
        nb = np.roll(lab, sh, axis=1)
        edge |= pos & (nb > 0) & (nb != lab)
    up = lab[:-1]
    edge[1:] |= pos[1:] & (up > 0) & (up != lab[1:])
    dn = lab[1:]
    edge[:-1] |= pos[:-1] & (dn > 0) & (dn != lab[:-1])
    return edge


def dilate_chebyshev(mask, radius):
    """Reference evaluate.py:58-70: (2r+1)^2 square, azimuth wraps, rings clamp."""
    mask = np.asarray(mask, dtype=bool)
    if radius == 0:
        return mask.copy()
    v = mask.copy()
    for d in range(1, radius + 1):
        v[d:] |= mask[:-d]
        v[:-d] |= mask[d:]
    out = v.copy()
    for d in range(1, radius + 1):
        out |= np.roll(v, d, axis=1) | np.roll(v, -d, axis=1)
    return out


def edge_counts(pred, truth, radius):
    """(n_pred, n_truth, pred edges matched, truth edges matched)."""
    pe, te = extract_edges(pred), extract_edges(truth)
    return (int(pe.sum()), int(te.sum()), int((pe & dilate_chebyshev(te, radius)).sum()),
            int((te & dilate_chebyshev(pe, radius)).sum()))


def edge_prf(pred, truth, radius):
    """Reference evaluate.py:73-94 -> (precision, recall, f1)."""
    n_p, n_t, m_p, m_t = edge_counts(pred, truth, radius)
    if n_p == 0 and n_t == 0:
        return 1.0, 1.0, 1.0
    p = m_p / n_p if n_p else 0.0
    r = m_t / n_t if n_t else 0.0
    f = 2.0 * p * r / (p + r) if p > 0.0 and r > 0.0 else 0.0
    return p, r, f
