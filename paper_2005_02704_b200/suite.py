"""Scenes x intervals accuracy suite, batched on the GPU (the computation of
the reference CLI's ``suite`` command, cli.py:99-120, without its files):
every scene is scanned by the GPU simulator (simulate.py), all scans of one
interval go through the pipeline as one batch (BatchPipeline.run_grid), and
the edge precision / recall / F1 against the simulator's truth labels
(reference evaluate.py:73-94, the paper's Table-2 metric) is computed for
the whole batch at once (evaluate.edge_prf_batch)."""

from __future__ import annotations

import numpy as np
import torch

from .evaluate import edge_prf_batch
from .pipeline import BatchPipeline, PipelineConfig
from .scan import SensorConfig
from .simulate import Scene, apply_scan, cast_grid_batch


def scan_scenes(scenes: list[Scene], sensor: SensorConfig, device=None):
    """Device tensors (ranges (F, R, S) with NaN = INVALID, truth labels
    (F, R, S)); scan f equals the reference's scan_scene(scenes[f], sensor)
    (same noise stream, simulate.py:404-421)."""
    dev = torch.device(device or "cuda")
    rs, ls = [], []
    for sc in scenes:
        t, ids = cast_grid_batch(sc, sensor, device=dev)
        noise = None
        if sensor.noise_sigma > 0.0:
            nz = np.random.default_rng(sc.seed).normal(0.0, sensor.noise_sigma,
                                                      size=(sensor.rings, sensor.azimuth_steps))
            noise = torch.from_numpy(nz).to(dev)
        r, lab = apply_scan(t, ids, sensor, noise)
        rs.append(r[0])
        ls.append(lab[0])
    return torch.stack(rs), torch.stack(ls)


def run_suite(scenes: list[Scene], cfg: PipelineConfig, names=None, normals: str = "exact", device=None):
    """One row per (scene, interval): scene, interval, precision, recall, f1
    (the fields of the reference's report_dict, io.py:440-448, without timings)."""
    dev = torch.device(device or "cuda")
    names = names or [f"scene{i}" for i in range(len(scenes))]
    ranges, truth = scan_scenes(scenes, cfg.sensor, dev)
    rows = []
    for interval in cfg.intervals:
        bp = BatchPipeline(cfg.sensor, interval, cfg.segmenter, frames=len(scenes), device=dev, normals=normals)
        labels = bp.run_grid(ranges)
        prf = edge_prf_batch(labels, truth, cfg.eval.dilation_radius).cpu().numpy()
        for f, name in enumerate(names):
            rows.append({"scene": name, "interval": int(interval), "precision": float(prf[f, 0]),
                         "recall": float(prf[f, 1]), "f1": float(prf[f, 2])})
    return rows
