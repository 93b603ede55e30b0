"""Cylindrical 6-neighbour mesh, mirroring reference pkg/src/lidarseg/mesh.py.

``build_mesh`` / ``mesh_triangles`` run on the GPU (C ABI lseg_build_mesh /
lseg_mesh_triangles); the Mesh dataclass and its helpers are the reference's
host-side view (mesh.py:30-80) so callers see identical objects.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import cached_property

import numpy as np
import torch

from . import _lib
from .scan import ScanGrid, device_tables, subsample_steps

SLOTS = ((1, 0), (1, 1), (0, 1), (-1, 0), (-1, -1), (0, -1))  # reference mesh.py:27


@dataclass(frozen=True)
class Mesh:
    """Neighbour topology of the sub-sampled grid (node ids row-major over
    (ring, kept position); ``neighbors`` slots N0..N5, -1 absent)."""

    rings: int
    full_steps: int
    interval: int
    kept_steps: np.ndarray
    node_rings: np.ndarray
    node_steps: np.ndarray
    node_ids: np.ndarray
    neighbors: np.ndarray
    _dev: dict | None = field(default=None, repr=False, compare=False)

    @property
    def n_nodes(self) -> int:
        return int(self.node_rings.size)

    @cached_property
    def degrees(self) -> np.ndarray:
        return (self.neighbors >= 0).sum(axis=1)

    def node_at(self, ring: int, step: int) -> int:
        pos = np.searchsorted(self.kept_steps, step)
        if pos >= self.kept_steps.size or self.kept_steps[pos] != step:
            return -1
        return int(self.node_ids[ring, pos])

    def neighbor_cells(self, ring: int, step: int) -> list[tuple[int, int]]:
        nid = self.node_at(ring, step)
        if nid < 0:
            raise ValueError(f"({ring}, {step}) is not a mesh node")
        return [(int(self.node_rings[q]), int(self.node_steps[q])) for q in self.neighbors[nid] if q >= 0]

    def edges(self) -> np.ndarray:
        src = np.repeat(np.arange(self.n_nodes), 6)
        dst = self.neighbors.reshape(-1)
        ok = dst >= 0
        pairs = np.stack([src[ok], dst[ok]], axis=1)
        pairs.sort(axis=1)
        return np.unique(pairs, axis=0)

    # ---- device views (frame axis of 1) used to chain ops without re-upload
    def device(self, device=None) -> dict:
        if self._dev is not None:
            return self._dev
        dev = torch.device(device or "cuda")
        Sk = self.kept_steps.size
        cap = self.rings * Sk
        nb = torch.full((1, cap, 6), -1, dtype=torch.int32)
        nb[0, : self.n_nodes] = torch.from_numpy(np.ascontiguousarray(self.neighbors, dtype=np.int32))
        d = {"node_ids": torch.from_numpy(np.ascontiguousarray(self.node_ids, np.int32)).to(dev).view(1, self.rings, Sk),
             "neighbors": nb.to(dev),
             "n_nodes": torch.tensor([self.n_nodes], dtype=torch.int32, device=dev)}
        object.__setattr__(self, "_dev", d)
        return d


def build_mesh(grid: ScanGrid, interval: int, max_edge_length: float | None = None, _device_ranges=None) -> Mesh:
    """GPU build_mesh (reference mesh.py:105-136)."""
    kept = subsample_steps(grid.config, interval)  # ValueError contract
    L = _lib.lib()
    cfg = grid.config
    R, S, Sk = cfg.rings, cfg.azimuth_steps, kept.size
    cap = R * Sk
    dev = torch.device("cuda")
    _, sn = device_tables(cfg, dev)
    ranges = grid.device_ranges(dev) if _device_ranges is None else _device_ranges
    node_ids = torch.empty((1, R, Sk), dtype=torch.int32, device=dev)
    nbrs = torch.empty((1, cap, 6), dtype=torch.int32, device=dev)
    node_rings = torch.empty((1, cap), dtype=torch.int32, device=dev)
    node_steps = torch.empty((1, cap), dtype=torch.int32, device=dev)
    n_nodes = torch.empty(1, dtype=torch.int32, device=dev)
    wsb = _lib.workspace_bytes(1, R, S, interval)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    me = float("nan") if max_edge_length is None else float(max_edge_length)
    _lib.check(L.lseg_build_mesh(sn, 1, int(interval), me, _lib.ptr(ranges), _lib.ptr(node_ids), _lib.ptr(nbrs),
                                 _lib.ptr(node_rings), _lib.ptr(node_steps), _lib.ptr(n_nodes), _lib.ptr(ws), wsb,
                                 _lib.stream_ptr()))
    n = int(n_nodes.item())
    return Mesh(rings=R, full_steps=S, interval=int(interval), kept_steps=kept,
                node_rings=node_rings[0, :n].cpu().numpy(),
                node_steps=node_steps[0, :n].cpu().numpy().astype(np.int64),
                node_ids=node_ids[0].cpu().numpy(), neighbors=nbrs[0, :n].cpu().numpy(),
                _dev={"node_ids": node_ids, "neighbors": nbrs, "n_nodes": n_nodes})


class MeshBuilder:
    """Incremental mesh construction, one kept azimuth column at a time
    (reference mesh.py:139-170; streaming contract SPEC.md:200; SURVEY.md
    §8(f) F2).

    Columns arrive in sweep order while the sensor spins.  Each
    ``add_column`` uploads the column and launches one small kernel
    (lseg_mb_column) that records the column's valid cells and their per-ring
    ranks and emits every slot of the PREVIOUS column -- all of its
    neighbours exist once the next column is in.  ``finish()`` closes the
    wrap (columns 0 and S'-1), scans the per-ring counts (O(R)) and resolves
    the emitted (ring, rank) references to the reference's row-major node
    ids in one parallel pass (lseg_mb_finish).  The result equals
    ``build_mesh`` on the assembled grid.
    """

    def __init__(self, grid_config, interval: int):
        self.config = grid_config
        self.interval = int(interval)
        self.kept = subsample_steps(grid_config, interval)
        self._n = 0
        self._L = _lib.lib()
        R, Sk = grid_config.rings, self.kept.size
        dev = torch.device("cuda")
        self._col = torch.empty((Sk, R), dtype=torch.float64, device=dev)  # one slot per column: no reuse race
        self._runcnt = torch.zeros(R, dtype=torch.int32, device=dev)
        self._colrank = torch.empty((R, Sk), dtype=torch.int32, device=dev)
        self._slots = torch.empty((R, Sk, 6), dtype=torch.int32, device=dev)
        self._host = torch.empty((Sk, R), dtype=torch.float64).pin_memory()

    def add_column(self, ranges) -> None:
        """Feed the range column for the next kept azimuth step."""
        col = np.asarray(ranges, dtype=float).reshape(-1)
        R = self.config.rings
        if col.size != R:
            raise ValueError(f"column length {col.size} != ring count {R}")
        if self._n >= self.kept.size:
            raise ValueError("all kept columns already supplied")
        j = self._n
        self._host[j].copy_(torch.from_numpy(col))
        self._col[j].copy_(self._host[j], non_blocking=True)
        _lib.check(self._L.lseg_mb_column(R, int(self.kept.size), j, float(self.config.r_min),
                                          float(self.config.r_max), _lib.ptr(self._col[j]), _lib.ptr(self._runcnt),
                                          _lib.ptr(self._colrank), _lib.ptr(self._slots), _lib.stream_ptr()))
        self._n += 1

    def finish(self) -> Mesh:
        Sk = self.kept.size
        if self._n != Sk:
            raise ValueError(f"expected {Sk} kept columns, got {self._n}")
        R, S = self.config.rings, self.config.azimuth_steps
        dev = self._runcnt.device
        node_ids = torch.empty((1, R, Sk), dtype=torch.int32, device=dev)
        nbrs = torch.empty((1, R * Sk, 6), dtype=torch.int32, device=dev)
        rowoff = torch.empty(R, dtype=torch.int32, device=dev)
        n_nodes = torch.empty(1, dtype=torch.int32, device=dev)
        _lib.check(self._L.lseg_mb_finish(R, int(Sk), _lib.ptr(self._runcnt), _lib.ptr(self._colrank),
                                          _lib.ptr(self._slots), _lib.ptr(rowoff), _lib.ptr(node_ids),
                                          _lib.ptr(nbrs), _lib.ptr(n_nodes), _lib.stream_ptr()))
        ids = node_ids[0].cpu().numpy()
        rr, pos = np.nonzero(ids >= 0)
        n = int(rr.size)
        return Mesh(rings=R, full_steps=S, interval=self.interval, kept_steps=self.kept,
                    node_rings=rr.astype(np.int32), node_steps=self.kept[pos].astype(np.int64), node_ids=ids,
                    neighbors=nbrs[0, :n].cpu().numpy(),
                    _dev={"node_ids": node_ids, "neighbors": nbrs, "n_nodes": n_nodes})


def mesh_triangles(mesh: Mesh) -> np.ndarray:
    """GPU mesh_triangles (reference mesh.py:173-189): (F, 3) node ids."""
    L = _lib.lib()
    d = mesh.device()
    R, Sk = mesh.rings, mesh.kept_steps.size
    dev = d["node_ids"].device
    tris = torch.empty((1, 2 * R * Sk, 3), dtype=torch.int32, device=dev)
    nt = torch.empty(1, dtype=torch.int32, device=dev)
    _lib.check(L.lseg_mesh_triangles(1, R, Sk, _lib.ptr(d["node_ids"]), _lib.ptr(tris), _lib.ptr(nt),
                                     _lib.stream_ptr()))
    return tris[0, : int(nt.item())].cpu().numpy()
