"""Golden bytes for the file formats, produced by the
REFERENCE writers in this container:

    python tests/golden/make_golden_io.py [/root/reference/pkg/src]

One small simulated scan is pushed through the reference pipeline; the
inputs (grid, labels, mesh, normals) and every writer's text are stored so
the tests can check byte identity and parser round trips.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main(ref_src="/root/reference/pkg/src"):
    sys.dont_write_bytecode = True
    sys.path.insert(0, ref_src)
    import lidarseg as L
    from lidarseg import io as lio

    scene = L.generate_scene(7, crowding=0.3)
    scene = L.Scene(primitives=scene.primitives + (
        L.Plane(point=(6.0, -4.0, -1.0), normal=(0.0, 0.3, 1.0), surface_id=900, extent=(3.0, 2.0)),), seed=42)
    cfg = L.SensorConfig.uniform(rings=8, top_deg=5.0, bottom_deg=-25.0, azimuth_steps=96, r_min=0.5, r_max=60.0,
                                 noise_sigma=0.03)
    grid = L.scan_scene(scene, cfg)
    pcfg = L.PipelineConfig(sensor=cfg, interval=2, intervals=(1, 2, 7),
                            segmenter=L.SegmenterConfig(0.25, 0.3, 0.15, min_segment_size=4),
                            eval=L.EvalConfig(dilation_radius=1))
    res = L.run_pipeline(grid, pcfg)
    mesh, nm = res.mesh, res.normals
    rep = L.EvalReport(precision=0.5, recall=0.25, f1=1.0 / 3.0, timings_ms={"mesh": 1.5, "total": 2.25})
    rows = [lio.report_dict("a", 1, rep), lio.report_dict("b", 7, L.EvalReport(0.1, 0.2, 0.3))]
    texts = {
        "scan": lio.write_scan_text(grid),
        "scan_nolabels": lio.write_scan_text(L.ScanGrid(config=cfg, ranges=grid.ranges)),
        "scene": lio.write_scene_text(scene),
        "config": lio.write_config_text(pcfg),
        "config_default": lio.write_config_text(L.PipelineConfig()),
        "labels": lio.write_labels_text(grid, res.labels),
        "ply": lio.write_labeled_ply(grid, res.labels),
        "mesh_ply": lio.write_mesh_ply(grid, mesh),
        "adjacency": lio.write_mesh_adjacency(mesh),
        "normals": lio.write_normals_text(mesh, nm),
        "report": lio.write_report_json("a", 1, rep),
        "summary": lio.write_summary_csv(rows),
    }
    np.savez_compressed(os.path.join(HERE, "io0.npz"), elev=cfg.ring_elevations, steps=96, r_min=0.5, r_max=60.0,
                        sigma=0.03, ranges=grid.ranges, truth=grid.truth_labels, labels=res.labels,
                        interval=2, kept=mesh.kept_steps, node_ids=mesh.node_ids, neighbors=mesh.neighbors,
                        node_rings=mesh.node_rings, node_steps=mesh.node_steps, nvals=nm.values, nmask=nm.mask,
                        **{"text_" + k: np.array(v) for k, v in texts.items()})
    print("wrote io0.npz", {k: len(v) for k, v in texts.items()})


if __name__ == "__main__":
    main(*sys.argv[1:])
