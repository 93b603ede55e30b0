"""k_tile phase breakdown (needs a library built with LSEG_PHASES=1, LSEG_LIB_PATH)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_02704_b200 as L
from paper_2005_02704_b200 import synth, _lib
shape = synth.CONFIGS["hdl64_batch"]
xyz, ring, off = synth.make_batch(shape, frames=128, seed=2005, device="cuda")
cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min, r_max=shape.r_max)
bp = L.BatchPipeline(cfg, 1, frames=128)
lib = _lib.load()
f = lib.lseg_debug_tile_phases; f.argtypes = [C.POINTER(C.c_double)]
out = (C.c_double * 8)()
bp.run(xyz, ring, off); torch.cuda.synchronize(); f(out)
for _ in range(3): bp.run(xyz, ring, off)
torch.cuda.synchronize(); f(out)
if os.environ.get("CERT", "1") == "1":
    names = ["X1+D2", "A halo", "L lists", "B normals", "X0 exact", "D dec+out"]
    tot = sum(out[0:6])
    for i in range(0, 6): print(f"{names[i]:12s} {100*out[i]/tot:5.1f}%")
else:
    names = ["", "A halo", "B1 lists", "B2 normals", "C outputs", "D masks"]
    tot = sum(out[1:6])
    for i in range(1, 6): print(f"{names[i]:12s} {100*out[i]/tot:5.1f}%")
print("tile_cc label-propagation rounds per tile: %.2f" % (out[6] / max(out[7], 1)))
