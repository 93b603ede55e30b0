"""Multi-rank frame sharding on CPU with gloo (world_size 2): every frame is
owned exactly once, and the reduced totals equal a single-process run."""

import os
import socket

import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_02704_b200 import dist as D


def test_shard_covers_every_frame_once():
    for F in (0, 1, 7, 512, 513):
        for G in (1, 2, 4, 8):
            owned = []
            for r in range(G):
                a, n = D.shard(F, G, r)
                assert n >= 0
                owned += list(range(a, a + n))
            assert owned == list(range(F))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, frames, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import lidarseg_oracle as O
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS["vlp16"]
    first, n = D.shard(frames, world, rank)
    pts = segs = 0
    if n:
        xyz, ring, off = synth.make_batch(shape, frames=n, seed=3, first_frame=first)
        for f in range(n):
            a, b = int(off[f]), int(off[f + 1])
            res = O.run_from_points(xyz[a:b].numpy(), ring[a:b].numpy(), shape.elevations, shape.steps, 5,
                                    shape.r_min, shape.r_max)
            pts += b - a
            segs += int(res["labels"].max())
    tot = D.reduce_run(pts, n, segs, elapsed_ms=10.0 * (rank + 1))
    out[rank] = (tot["points"], tot["frames"], tot["segments"], tot["elapsed_ms"])
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_totals_match_single_process():
    frames = 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), frames, out), nprocs=2, join=True)
    single = {}
    _worker_single = None  # noqa: F841
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import lidarseg_oracle as O
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS["vlp16"]
    xyz, ring, off = synth.make_batch(shape, frames=frames, seed=3)
    pts = segs = 0
    for f in range(frames):
        a, b = int(off[f]), int(off[f + 1])
        res = O.run_from_points(xyz[a:b].numpy(), ring[a:b].numpy(), shape.elevations, shape.steps, 5,
                                shape.r_min, shape.r_max)
        pts += b - a
        segs += int(res["labels"].max())
    single = (pts, frames, segs)
    assert out[0] == out[1]
    assert out[0][:3] == single
    assert out[0][3] == 20.0  # max over ranks
