"""One HDL-64 frame through BatchPipeline (for ncu launch lists of the latency path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_02704_b200 as L
from paper_2005_02704_b200 import synth
name = sys.argv[1] if len(sys.argv) > 1 else "hdl64"
shape = synth.CONFIGS[name]
xyz, ring, off = synth.make_batch(shape, frames=1, seed=77, device="cpu")
xyz, ring, off = xyz.cuda(), ring.cuda(), off.cuda()
cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min, r_max=shape.r_max)
bp = L.BatchPipeline(cfg, 1, frames=1)
for _ in range(3):
    bp.run(xyz, ring, off)
torch.cuda.synchronize()
print("ok", int(bp.n_labels[0]))
