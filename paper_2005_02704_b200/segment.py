"""Segmentation + label completion, mirroring reference pkg/src/lidarseg/segment.py.

``segment`` is GPU union-find connected-component labelling (C ABI
lseg_segment) whose label ids equal the reference DFS's first-touch numbering
(label = 1 + rank of the component's minimum node id);
``backfill`` / ``prune_small`` are per-ring nearest-donor kernels (C ABI
lseg_backfill / lseg_prune_small).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .mesh import Mesh
from .normals import NormalMap
from .scan import ScanGrid, device_tables


@dataclass(frozen=True)
class SegmenterConfig:
    """Component-difference thresholds and the pruning floor (segment.py:22-40)."""

    threshold_i: float = 0.2
    threshold_j: float = 0.2
    threshold_k: float = 0.2
    min_segment_size: int = 10

    def __post_init__(self):
        for t in (self.threshold_i, self.threshold_j, self.threshold_k):
            if not (0.0 < t <= 2.0):
                raise ValueError("thresholds must be in (0, 2]")
        if self.min_segment_size < 0:
            raise ValueError("min_segment_size must be >= 0")

    @property
    def thresholds(self) -> np.ndarray:
        return np.array([self.threshold_i, self.threshold_j, self.threshold_k])


def segment_device(mesh: Mesh, n64, mask, cfg: SegmenterConfig):
    """Device labels (1, R, S) i32 and n_labels (1,) from device normals."""
    L = _lib.lib()
    d = mesh.device()
    dev = d["node_ids"].device
    R, S = mesh.rings, mesh.full_steps
    labels = torch.empty((1, R, S), dtype=torch.int32, device=dev)
    nl = torch.empty(1, dtype=torch.int32, device=dev)
    wsb = _lib.workspace_bytes(1, R, S, mesh.interval)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _lib.check(L.lseg_segment(1, R, S, mesh.interval, _lib.ptr(d["node_ids"]), _lib.ptr(d["neighbors"]),
                              _lib.ptr(d["n_nodes"]), _lib.ptr(n64), _lib.ptr(mask),
                              _lib.thresholds_arg(cfg.thresholds), _lib.ptr(labels), _lib.ptr(nl), _lib.ptr(ws),
                              wsb, _lib.stream_ptr()))
    return labels, nl


def segment(mesh: Mesh, normals: NormalMap, cfg: SegmenterConfig) -> np.ndarray:
    """GPU segment (reference segment.py:43-88): dense (R, S) labels."""
    _lib.lib()
    d = mesh.device()
    dev = d["node_ids"].device
    cap = mesh.rings * mesh.kept_steps.size
    n = mesh.n_nodes
    n64 = torch.zeros((1, cap, 3), dtype=torch.float64)
    mask = torch.zeros((1, cap), dtype=torch.uint8)
    if n:
        n64[0, :n] = torch.from_numpy(np.ascontiguousarray(normals.values, dtype=np.float64))
        mask[0, :n] = torch.from_numpy(np.asarray(normals.mask, dtype=np.uint8))
    labels, _ = segment_device(mesh, n64.to(dev), mask.to(dev), cfg)
    return labels[0].cpu().numpy()


def backfill_device(config, ranges_dev, labels_dev):
    L = _lib.lib()
    _, sn = device_tables(config, ranges_dev.device)
    out = torch.empty_like(labels_dev)
    F = labels_dev.shape[0] if labels_dev.dim() == 3 else 1
    _lib.check(L.lseg_backfill(sn, F, _lib.ptr(ranges_dev), _lib.ptr(labels_dev), _lib.ptr(out), _lib.stream_ptr()))
    return out


def backfill(grid: ScanGrid, labels: np.ndarray) -> np.ndarray:
    """GPU backfill (reference segment.py:109-124)."""
    lab = np.asarray(labels)
    dev = torch.device("cuda")
    _lib.lib()
    t = torch.from_numpy(np.ascontiguousarray(lab, dtype=np.int32)).to(dev)
    out = backfill_device(grid.config, grid.device_ranges(dev), t)
    return out.cpu().numpy().astype(lab.dtype, copy=False)


def prune_small_device(labels_dev, min_segment_size: int, label_bound: int):
    """labels_dev (F, R, S) or (R, S) i32 on device; returns pruned copy."""
    L = _lib.lib()
    lab3 = labels_dev if labels_dev.dim() == 3 else labels_dev.unsqueeze(0)
    F, R, S = lab3.shape
    out = torch.empty_like(lab3)
    wsb = int(L.lseg_workspace_bytes(F, R, max(S, 2), 1, int(label_bound)))
    ws = torch.empty(wsb, dtype=torch.uint8, device=lab3.device)
    _lib.check(L.lseg_prune_small(F, R, S, _lib.ptr(lab3), int(min_segment_size), int(label_bound), _lib.ptr(out),
                                  _lib.ptr(ws), wsb, _lib.stream_ptr()))
    return out if labels_dev.dim() == 3 else out[0]


def prune_small(labels: np.ndarray, min_segment_size: int) -> np.ndarray:
    """GPU prune_small (reference segment.py:127-160)."""
    lab = np.asarray(labels)
    if min_segment_size <= 0:
        return lab.copy()
    if lab.ndim != 2:
        raise ValueError("labels must be a 2-D (rings, steps) grid")
    if lab.size and lab.min() < 0:
        raise ValueError("labels must be non-negative")
    bound = int(lab.max()) + 1 if lab.size else 1
    if bound <= 1:
        return lab.copy()
    _lib.lib()
    t = torch.from_numpy(np.ascontiguousarray(lab, dtype=np.int32)).to("cuda")
    return prune_small_device(t, min_segment_size, bound).cpu().numpy()
