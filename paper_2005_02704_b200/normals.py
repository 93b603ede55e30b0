"""Per-node normals, mirroring reference pkg/src/lidarseg/normals.py.

``estimate_normals`` runs on the GPU (C ABI lseg_estimate_normals) with fp64
arithmetic in the reference's operation order; the scalar helpers
(``normal_from_neighbors``, ``point_normal``) are host conveniences kept for
API compatibility (reference normals.py:49-91).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .mesh import Mesh
from .scan import GridIndex, ScanGrid, device_tables

_MIN_ACCUM = 1e-12


@dataclass(frozen=True)
class NormalMap:
    """Unit normal per mesh node; NaN rows where no normal exists."""

    values: np.ndarray  # (N, 3)
    mask: np.ndarray    # (N,)

    @property
    def n_nodes(self) -> int:
        return int(self.mask.size)

    def normal(self, node_id: int):
        if not self.mask[node_id]:
            return None
        return self.values[node_id]


def node_positions(grid: ScanGrid, mesh: Mesh) -> np.ndarray:
    """Cartesian node positions (N, 3), reference normals.py:42-46."""
    dirs = grid.config.ray_directions()[:, mesh.kept_steps]
    pts = dirs * grid.ranges[:, mesh.kept_steps, None]
    return pts[mesh.node_ids >= 0]


def normal_from_neighbors(position, neighbor_positions):
    """Scalar estimator (host), reference normals.py:49-81 semantics."""
    p = np.asarray(position, dtype=float)
    vs = [np.asarray(q, dtype=float) - p for q in neighbor_positions]
    if len(vs) < 2:
        return None
    pairs = [(0, 1)] if len(vs) == 2 else [(k, (k + 1) % len(vs)) for k in range(len(vs))]
    acc = np.zeros(3)
    wsum = 0.0
    for a, b in pairs:
        length = float(np.linalg.norm(vs[a]) + np.linalg.norm(vs[b]))
        if length <= 0.0:
            continue
        w = 1.0 / length
        acc += w * np.cross(vs[a], vs[b])
        wsum += w
    if wsum <= 0.0:
        return None
    mean = acc / wsum
    mag = float(np.linalg.norm(mean))
    if mag < _MIN_ACCUM:
        return None
    n = mean / mag
    return -n if float(n @ p) > 0.0 else n


def point_normal(grid: ScanGrid, mesh: Mesh, node: GridIndex):
    nid = mesh.node_at(int(node[0]), int(node[1]))
    if nid < 0:
        raise ValueError(f"({node[0]}, {node[1]}) is not a mesh node")
    pos = node_positions(grid, mesh)
    return normal_from_neighbors(pos[nid], [pos[q] for q in mesh.neighbors[nid] if q >= 0])


def estimate_normals_device(grid: ScanGrid, mesh: Mesh, want64: bool = True, want32: bool = False):
    """Run the normal kernel; returns device (n64 | None, n32 | None, mask u8)."""
    L = _lib.lib()
    d = mesh.device()
    dev = d["node_ids"].device
    cap = mesh.rings * mesh.kept_steps.size
    _, sn = device_tables(grid.config, dev)
    ranges = grid.device_ranges(dev)
    n64 = torch.empty((1, cap, 3), dtype=torch.float64, device=dev) if want64 else None
    n32 = torch.empty((1, cap, 3), dtype=torch.float32, device=dev) if want32 else None
    mask = torch.zeros((1, cap), dtype=torch.uint8, device=dev)
    _lib.check(L.lseg_estimate_normals(sn, 1, mesh.interval, _lib.ptr(ranges), _lib.ptr(d["node_ids"]),
                                       _lib.ptr(d["neighbors"]), _lib.ptr(d["n_nodes"]), _lib.ptr(n64),
                                       _lib.ptr(n32), _lib.ptr(mask), _lib.stream_ptr()))
    return n64, n32, mask


def estimate_normals(grid: ScanGrid, mesh: Mesh) -> NormalMap:
    """GPU estimate_normals (reference normals.py:94-145); fp64 values."""
    n = mesh.n_nodes
    if n == 0:
        return NormalMap(values=np.zeros((0, 3)), mask=np.zeros(0, dtype=bool))
    n64, _, mask = estimate_normals_device(grid, mesh)
    m = mask[0, :n].bool().cpu().numpy()
    vals = n64[0, :n].cpu().numpy()
    vals[~m] = np.nan
    return NormalMap(values=vals, mask=m)


def normals_to_grid(mesh: Mesh, normals: NormalMap) -> np.ndarray:
    out = np.full((mesh.rings, mesh.full_steps, 3), np.nan)
    ok = normals.mask
    out[mesh.node_rings[ok], mesh.node_steps[ok]] = normals.values[ok]
    return out
