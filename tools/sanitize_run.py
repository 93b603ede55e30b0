"""Small runs of every library entry point, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck) on a GPU box:

    compute-sanitizer --tool racecheck --kernel-name regex:k_ python tools/sanitize_run.py

Exercises: the batched pipeline (point input: ring-major and generic
binning, k = 1 / 5, exact and certified normals, segment() output), the
single-scan run_pipeline, the single ops (build_mesh, estimate_normals,
segment, backfill, prune_small, triangles), the streaming MeshBuilder, the
edge evaluator and the scan simulator.  Labels are checked against a second
run (determinism), not against the oracle (tests/ do that)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_02704_b200 as L  # noqa: E402
from paper_2005_02704_b200 import synth  # noqa: E402


def cfg_of(shape):
    return L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                          r_max=shape.r_max)


def batch(name, frames, k, normals="exact", generic=False, node_labels=False):
    shape = synth.CONFIGS[name]
    xyz, ring, off = synth.make_batch(shape, frames=frames, seed=5, device="cuda")
    if generic:  # reversed point order inside each frame: not ring-major -> generic binning
        parts = [torch.flip(torch.arange(int(off[f]), int(off[f + 1]), device="cuda"), [0]) for f in range(frames)]
        idx = torch.cat(parts)
        xyz, ring = xyz[idx].contiguous(), ring[idx].contiguous()
    bp = L.BatchPipeline(cfg_of(shape), k, frames=frames, normals=normals, keep_node_labels=node_labels)
    a = bp.run(xyz, ring, off).clone()
    b = bp.run(xyz, ring, off).clone()
    torch.cuda.synchronize()
    assert torch.equal(a, b), (name, k, normals)
    print("batch", name, frames, k, normals, "generic" if generic else "", "ok", flush=True)


def single(name):
    shape = synth.CONFIGS[name]
    xyz, ring, off = synth.make_batch(shape, frames=1, seed=6, device="cuda")
    cfg = cfg_of(shape)
    grid = L.bin_points(xyz, ring, cfg)
    res = L.run_pipeline(grid, L.PipelineConfig(interval=1))
    mesh = L.build_mesh(grid, 1)
    nm = L.estimate_normals(grid, mesh)
    lab = L.segment(mesh, nm, L.SegmenterConfig())
    lab = L.backfill(grid, lab)
    lab = L.prune_small(lab, 10)
    L.mesh_triangles(mesh)
    assert np.array_equal(np.asarray(lab), np.asarray(res.labels))
    b = L.MeshBuilder(grid.config, 1)
    for c in range(grid.config.azimuth_steps):
        b.add_column(grid.ranges[:, c])
    m2 = b.finish()
    assert np.array_equal(np.asarray(m2.neighbors), np.asarray(mesh.neighbors))
    print("single", name, "ok", flush=True)


def main():
    single("vlp16")
    batch("vlp16", 3, 1)
    batch("hdl64", 2, 1)
    batch("hdl64", 2, 5)
    batch("hdl64", 2, 1, normals="certified")
    batch("hdl64", 1, 1, node_labels=True)
    batch("vlp16", 2, 1, generic=True)
    batch("stress", 1, 1)
    # scan simulator + batched pipeline from grids + edge evaluator
    rows = L.run_suite(L.generate_suite(2005, 2), L.PipelineConfig(intervals=(1, 5)))
    print("suite", len(rows), "rows ok", flush=True)
    print("all ok", flush=True)


if __name__ == "__main__":
    main()
