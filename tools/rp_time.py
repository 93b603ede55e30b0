"""Where the host-to-host run_pipeline time goes (HDL-64 scan): wall time of
the call vs its parts, timed around each step."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_02704_b200 as L  # noqa: E402
from paper_2005_02704_b200 import synth  # noqa: E402

shape = synth.CONFIGS["hdl64"]
xyz, ring, off = synth.make_batch(shape, frames=1, seed=77, device="cuda")
cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min, r_max=shape.r_max)
bp = L.BatchPipeline(cfg, 1, frames=1)
bp.run(xyz, ring, off)
grid = L.ScanGrid(config=cfg, ranges=bp.ranges[0].cpu().numpy())
pcfg = L.PipelineConfig(sensor=cfg, interval=1)
for _ in range(5):
    L.run_pipeline(grid, pcfg)
ts = []
for _ in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.run_pipeline(grid, pcfg)
    ts.append(time.perf_counter() - t0)
print("run_pipeline median us", np.median(ts) * 1e6)
import cProfile, pstats  # noqa: E402,E401
pr = cProfile.Profile()
pr.enable()
for _ in range(30):
    L.run_pipeline(grid, pcfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
