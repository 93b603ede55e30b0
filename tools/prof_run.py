"""Minimal driver for ncu: runs the batched pipeline `--iters` times on frames
generated on the CPU (so the only CUDA kernels in the process are ours plus a
few copies).  Usage under gpurun:

    python tools/prof_run.py --config hdl64_batch --frames 32 --iters 3 &&
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/prof_run.py ...
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="hdl64_batch")
    ap.add_argument("--frames", type=int, default=32)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--interval", type=int, default=1)
    a = ap.parse_args()
    import paper_2005_02704_b200 as L
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS[a.config]
    xyz, ring, off = synth.make_batch(shape, frames=a.frames, seed=2005, device="cpu")
    xyz, ring, off = xyz.cuda(), ring.cuda(), off.cuda()
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    bp = L.BatchPipeline(cfg, a.interval, frames=a.frames)
    for _ in range(a.iters):
        bp.run(xyz, ring, off)
    torch.cuda.synchronize()
    print(f"ok: {a.frames} frames, {int(xyz.shape[0])} points, {int(bp.n_nodes.sum())} nodes")


if __name__ == "__main__":
    main()
