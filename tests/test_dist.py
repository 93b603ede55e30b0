"""Multi-rank frame sharding on CPU with gloo (world_size 2), through the
exact functions bench.py runs per rank (dist.rank_batch for the rank's frames,
dist.reduce_run for the run's single collective): every frame of the batch
is owned exactly once, each rank's frames are the batch's frames, and the
reduced totals equal a single-process run."""

import os
import socket

import pytest
import torch
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
            assert max(D.shard(F, G, r)[1] for r in range(G)) == -(-F // G)


def test_rank_frames_strong_and_weak():
    assert [D.rank_frames(512, 8, r) for r in range(8)] == [(64 * r, 64) for r in range(8)]
    assert [D.rank_frames(512, 2, r, "weak") for r in range(2)] == [(0, 512), (512, 512)]
    with pytest.raises(ValueError):
        D.rank_frames(4, 2, 0, "bogus")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, frames, scaling, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS["vlp16"]
    first, n, xyz, ring, off = D.rank_batch(shape, frames, world, rank, scaling, seed=3)
    # stand-in for the per-frame work: points and a per-frame checksum of the
    # rank's own inputs (the GPU pipeline itself is covered by the -m gpu tests)
    sums = [float(xyz[int(off[f]):int(off[f + 1])].double().sum()) for f in range(n)]
    tot = D.reduce_run(int(xyz.shape[0]), n, len(sums), elapsed_ms=10.0 * (rank + 1))
    out[rank] = {"first": first, "n": n, "points": int(xyz.shape[0]), "sums": sums,
                 "tot": (tot["points"], tot["frames"], tot["segments"], tot["elapsed_ms"])}
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling,frames", [("strong", 5), ("weak", 2)])
def test_two_rank_gloo_partition_and_totals(scaling, frames):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), frames, scaling, out), nprocs=2, join=True)
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS["vlp16"]
    total = frames if scaling == "strong" else 2 * frames
    xyz, ring, off = synth.make_batch(shape, frames=total, seed=3)
    want_sums = [float(xyz[int(off[f]):int(off[f + 1])].double().sum()) for f in range(total)]
    r0, r1 = out[0], out[1]
    if scaling == "strong":
        assert (r0["first"], r0["n"], r1["first"], r1["n"]) == (0, 3, 3, 2)
    else:
        assert (r0["first"], r0["n"], r1["first"], r1["n"]) == (0, frames, frames, frames)
    # each frame owned once, and each rank's frames are exactly the batch's frames
    assert r0["sums"] + r1["sums"] == want_sums
    assert r0["tot"] == r1["tot"] == (int(xyz.shape[0]), total, total, 20.0)  # sums; max elapsed over ranks
