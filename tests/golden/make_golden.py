"""Generate golden vectors by running the REFERENCE lidarseg package.

Run in the build container only (the reference is not on the GPU box):

    python tests/golden/make_golden.py [/root/reference/pkg/src]

It imports the reference read-only, runs its own public functions
(build_mesh, mesh_triangles, estimate_normals, segment, backfill,
prune_small, run_pipeline) on seeded inputs, and stores inputs + outputs in
``tests/golden/*.npz``.  The oracle (``oracle/lidarseg_oracle.py``) and the CUDA
path are both checked against these files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main(ref_src="/root/reference/pkg/src"):
    sys.dont_write_bytecode = True
    sys.path.insert(0, ref_src)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import lidarseg as L  # the reference
    import lidarseg_oracle as O
    from paper_2005_02704_b200 import synth

    out = {}

    def pipe_case(name, ranges, elev, steps, interval, r_min, r_max, thr=(0.2, 0.2, 0.2), mseg=10,
                  xyz=None, ring=None, max_edge=None):
        cfg = L.SensorConfig(ring_elevations=elev, azimuth_steps=steps, r_min=r_min, r_max=r_max)
        grid = L.ScanGrid(config=cfg, ranges=ranges)
        mesh = L.build_mesh(grid, interval, max_edge_length=max_edge)
        nm = L.estimate_normals(grid, mesh)
        scfg = L.SegmenterConfig(*thr, min_segment_size=mseg)
        node_dense = L.segment(mesh, nm, scfg)
        filled = L.backfill(grid, node_dense)
        labels = L.prune_small(filled, mseg)
        if max_edge is None:
            pcfg = L.PipelineConfig(sensor=cfg, interval=interval, segmenter=scfg)
            res = L.run_pipeline(grid, pcfg)
            assert np.array_equal(res.labels, labels)
        d = dict(elev=np.asarray(elev, np.float64), steps=steps, interval=interval, r_min=r_min,
                 r_max=r_max, thr=np.asarray(thr, np.float64), mseg=mseg, ranges=np.asarray(ranges),
                 max_edge=-1.0 if max_edge is None else float(max_edge),
                 kept=mesh.kept_steps, node_ids=mesh.node_ids, neighbors=mesh.neighbors,
                 node_rings=mesh.node_rings, node_steps=mesh.node_steps,
                 triangles=L.mesh_triangles(mesh).astype(np.int32),
                 normals=nm.values, nmask=nm.mask, node_dense=node_dense, filled=filled,
                 labels=labels)
        if xyz is not None:
            d["xyz"] = np.asarray(xyz, np.float32)
            d["ring"] = np.asarray(ring, np.int32)
        out[name] = d

    # --- full VLP-16-shape frame from points (BASELINE configs[0]), k = 1 and 5
    shape = synth.CONFIGS["vlp16"]
    xyz, ring, _ = synth.make_batch(shape, frames=1, seed=11)
    xyz, ring = xyz.numpy(), ring.numpy()
    ranges, _ = O.bin_points(xyz, ring, shape.rings, shape.steps, shape.r_min, shape.r_max)
    for k in (1, 5):
        pipe_case(f"vlp16_k{k}", ranges, shape.elevations, shape.steps, k, shape.r_min, shape.r_max,
                  xyz=xyz, ring=ring)

    # --- small grids in the style of the reference conftest (random_smooth_grid)
    rng = np.random.default_rng(1234)
    for i, (R, S, k, keep) in enumerate([(6, 16, 1, 0.9), (8, 16, 1, 0.75), (7, 18, 2, 0.85),
                                         (5, 23, 3, 0.8), (4, 10, 5, 1.0), (4, 11, 6, 0.9),
                                         (9, 40, 7, 0.7), (3, 2048, 5, 0.95)]):
        elev = np.radians(np.linspace(10.0, -30.0, R))
        rr = 5.0 + rng.uniform(-0.5, 0.5, size=(R, S))
        rr[rng.random((R, S)) > keep] = np.nan
        thr = tuple(rng.uniform(0.05, 0.6, size=3))
        pipe_case(f"small{i}", rr, elev, S, k, 0.5, 100.0, thr=thr, mseg=int(rng.integers(0, 6)))
    # max_edge_length (reference mesh.py:122-126), outlier cell like test_mesh.py:116-131
    elev = np.radians(np.linspace(10.0, -30.0, 5))
    rr = 5.0 + rng.uniform(-0.3, 0.3, size=(5, 24))
    rr[2, 7] = 50.0
    rr[3, 11] = np.nan
    pipe_case("maxedge", rr, elev, 24, 1, 0.5, 100.0, max_edge=2.0)

    # --- segment() on prescribed random normal maps (test_segment.py:30-53 style)
    for i in range(4):
        R, S = 8, 16
        elev = np.radians(np.linspace(10.0, -30.0, R))
        rr = 5.0 + rng.uniform(-0.5, 0.5, size=(R, S))
        rr[rng.random((R, S)) > 0.8] = np.nan
        cfg = L.SensorConfig(ring_elevations=elev, azimuth_steps=S)
        grid = L.ScanGrid(config=cfg, ranges=rr)
        mesh = L.build_mesh(grid, 1)
        vals = rng.normal(size=(mesh.n_nodes, 3))
        vals /= np.linalg.norm(vals, axis=1, keepdims=True)
        mask = rng.random(mesh.n_nodes) >= 0.15
        vals[~mask] = np.nan
        thr = tuple(rng.uniform(0.2, 1.2, size=3))
        dense = L.segment(mesh, L.NormalMap(values=vals, mask=mask), L.SegmenterConfig(*thr))
        out[f"seg{i}"] = dict(elev=elev, steps=S, ranges=rr, values=vals, mask=mask,
                              thr=np.asarray(thr), node_dense=dense, neighbors=mesh.neighbors,
                              node_ids=mesh.node_ids)

    # --- backfill / prune on random label grids
    for i in range(4):
        R, S = 5, 37
        elev = np.radians(np.linspace(10.0, -30.0, R))
        rr = 5.0 + rng.uniform(-0.5, 0.5, size=(R, S))
        rr[rng.random((R, S)) > 0.8] = np.nan
        lab = rng.integers(0, 9, size=(R, S)).astype(np.int32)
        lab[rng.random((R, S)) < 0.6] = 0
        lab[2] = 0  # a ring without donors
        cfg = L.SensorConfig(ring_elevations=elev, azimuth_steps=S)
        grid = L.ScanGrid(config=cfg, ranges=rr)
        filled = L.backfill(grid, lab)
        m = int(rng.integers(0, 8))
        out[f"fill{i}"] = dict(elev=elev, steps=S, ranges=rr, labels_in=lab, filled=filled,
                               mseg=m, pruned=L.prune_small(filled, m))

    # --- edge evaluator (reference evaluate.py:40-94) on pipeline labels vs truth-like grids
    for i, (R, S, r) in enumerate([(16, 180, 2), (8, 37, 1), (5, 12, 0), (6, 64, 3)]):
        pred = rng.integers(0, 6, size=(R, S)).astype(np.int32)
        pred[rng.random((R, S)) < 0.2] = 0
        truth = np.repeat(rng.integers(0, 4, size=(R, 1 + S // 8)), 8, axis=1)[:, :S].astype(np.int32)
        rep = L.edge_prf(pred, truth, L.EvalConfig(dilation_radius=r))
        out[f"edges{i}"] = dict(pred=pred, truth=truth, radius=r, pe=L.extract_edges(pred),
                                te=L.extract_edges(truth), dil=L.dilate_chebyshev(L.extract_edges(truth), r),
                                prf=np.array([rep.precision, rep.recall, rep.f1]))
    g = out["vlp16_k1"]
    cfg = L.SensorConfig(ring_elevations=g["elev"], azimuth_steps=int(g["steps"]))
    rep = L.edge_prf(g["labels"], out["vlp16_k5"]["labels"], L.EvalConfig())
    out["edges_vlp"] = dict(pred=g["labels"], truth=out["vlp16_k5"]["labels"], radius=2,
                            prf=np.array([rep.precision, rep.recall, rep.f1]))

    for name, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(f"wrote {len(out)} golden files to {HERE}")


if __name__ == "__main__":
    main(*sys.argv[1:])
