"""Golden vectors for the scan simulator, produced by
running the REFERENCE simulator in this container:

    python tests/golden/make_golden_sim.py [/root/reference/pkg/src]

For a few generated scenes (reference scenes.generate_scene) it stores the
scene as packed primitive records, the reference's cast_grid (t, ids),
scan_scene (noisy ranges, truth labels) and scene_normals.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
STRIDE = 24


def pack_reference(prim) -> np.ndarray:
    """Same record layout as paper_2005_02704_b200/simulate.py:_record, from a
    reference primitive (duck-typed by class name)."""
    import lidarseg.simulate as S
    r = np.zeros(STRIDE)
    ids = list(prim.surface_ids)
    r[1:1 + len(ids)] = ids
    kind = type(prim).__name__
    if kind == "Plane":
        r[7:10], r[10:13] = prim.point, prim.normal
        if prim.extent is not None:
            u, v = S._plane_axes(prim.normal)
            r[13:16] = 1.0, prim.extent[0], prim.extent[1]
            r[16:19], r[19:22] = u, v
    elif kind == "Sphere":
        r[0] = 1
        r[7:10], r[10] = prim.center, prim.radius
    elif kind == "Cylinder":
        r[0] = 2
        r[7:10], r[10:13], r[13], r[14] = prim.base, prim.axis, prim.radius, prim.height
    elif kind == "Box":
        r[0] = 3
        r[7:10], r[10:13], r[13:22] = prim.center, prim.half_extents, prim.rotation.reshape(-1)
    else:
        r[0] = 4
        r[7:10], r[10:13] = prim.apex, prim.axis
        r[13] = np.cos(prim.half_angle) ** 2
        r[14] = prim.height
        r[15] = prim.height * np.tan(prim.half_angle)
        r[16], r[17] = np.cos(prim.half_angle), np.sin(prim.half_angle)
    return r


def main(ref_src="/root/reference/pkg/src"):
    sys.dont_write_bytecode = True
    sys.path.insert(0, ref_src)
    import lidarseg as L

    cases = [  # (scene seed, crowding, rings, steps, top, bottom, noise sigma)
        (5, 0.0, 16, 360, 15.0, -15.0, 0.0),
        (17, 0.3, 24, 480, 10.0, -30.0, 0.05),
        (101, 0.6, 32, 512, 2.0, -24.9, 0.02),
        (2024, 0.9, 12, 300, 20.0, -20.0, 0.1),
    ]
    for i, (seed, crowd, R, S, top, bot, sigma) in enumerate(cases):
        scene = L.generate_scene(seed, crowding=crowd)
        if i == 3:  # add a finite tilted plane (ramp) and an overhead patch
            extra = (L.Plane(point=(6.0, -4.0, -1.0), normal=(0.0, 0.3, 1.0), surface_id=900, extent=(3.0, 2.0)),
                     L.Plane(point=(0.0, 0.0, 4.0), normal=(0.0, 0.0, -1.0), surface_id=901, extent=(5.0, 5.0)))
            scene = L.Scene(primitives=scene.primitives + extra, seed=scene.seed)
        cfg = L.SensorConfig.uniform(rings=R, top_deg=top, bottom_deg=bot, azimuth_steps=S, r_min=0.5,
                                     r_max=100.0, noise_sigma=sigma)
        t, ids = L.cast_grid(scene, cfg)
        grid = L.scan_scene(scene, cfg)
        nrm = L.scene_normals(scene, grid)
        # suite: the pipeline on the reference's own scan + edge P/R/F1 vs truth
        pcfg = L.PipelineConfig(sensor=cfg, intervals=(1, 5))
        suite = {}
        prf = []
        for k in (1, 5):
            res = L.run_pipeline(grid, pcfg, interval=k)
            rep = L.edge_prf(res.labels, grid.truth_labels, pcfg.eval)
            suite[f"suite_labels_k{k}"] = res.labels
            prf.append([rep.precision, rep.recall, rep.f1])
        np.savez_compressed(os.path.join(HERE, f"sim{i}.npz"), seed=seed, crowding=crowd, rings=R, steps=S,
                            top=top, bottom=bot, sigma=sigma, elev=cfg.ring_elevations,
                            records=np.stack([pack_reference(p) for p in scene.primitives]),
                            t=t, ids=ids, ranges=grid.ranges, labels=grid.truth_labels, normals=nrm,
                            suite_prf=np.array(prf), **suite)
    print(f"wrote {len(cases)} simulator golden files to {HERE}")


if __name__ == "__main__":
    main(*sys.argv[1:])
