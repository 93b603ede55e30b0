"""Frame sharding across GPUs of one node.

Frames are independent (reference cli.py:107-118 runs scans one by one), so
the batch is split into contiguous blocks of ceil(F/G) frames, one per rank
(`shard`), with no data-path collective; the only collective is one tiny
all-reduce at the end of a run carrying (points, frames, segments, elapsed).
`rank_batch` + `reduce_run` are exactly what bench.py runs per rank; the
world-size-2 gloo test (tests/test_dist.py) calls the same two functions.
Works with NCCL (GPU tensors) and gloo (CPU tensors).
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(total_frames: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [first, first + count) of frames owned by `rank`
    (ceil(F/G) per rank, the last ranks possibly shorter or empty)."""
    per = -(-total_frames // world)
    first = min(rank * per, total_frames)
    return first, min(per, total_frames - first)


def rank_frames(total_frames: int, world: int, rank: int, scaling: str = "strong") -> tuple[int, int]:
    """Frames [first, first + count) this rank processes.  "strong": the one
    batch of `total_frames` split by `shard` (BASELINE configs[3]: 512 frames
    over 1/2/4/8 GPUs); "weak": `total_frames` per rank, rank r taking the
    frames that follow rank r-1's."""
    if scaling == "strong":
        return shard(total_frames, world, rank)
    if scaling == "weak":
        return rank * total_frames, total_frames
    raise ValueError("scaling must be 'strong' or 'weak'")


def rank_batch(shape, total_frames: int, world: int, rank: int, scaling: str = "strong", seed: int = 0,
               device="cpu"):
    """This rank's frames of the synthetic batch, generated directly where
    they are processed: (first, count, xyz (P,3) f32, ring (P,) i32,
    offsets (count+1,) i64).  A rank with no frames gets empty tensors."""
    from . import synth
    first, count = rank_frames(total_frames, world, rank, scaling)
    if count == 0:
        return (first, 0, torch.empty((0, 3), dtype=torch.float32, device=device),
                torch.empty(0, dtype=torch.int32, device=device), torch.zeros(1, dtype=torch.int64, device=device))
    xyz, ring, off = synth.make_batch(shape, frames=count, seed=seed, device=device, first_frame=first)
    return first, count, xyz, ring, off


def reduce_run(points: int, frames: int, segments: int, elapsed_ms: float, device=None) -> dict:
    """The run's single collective: sums of points / frames / segments and the
    max elapsed time over ranks (CUDA-event milliseconds)."""
    dev = torch.device(device) if device is not None else torch.device("cpu")
    sums = torch.tensor([float(points), float(frames), float(segments)], dtype=torch.float64, device=dev)
    mx = torch.tensor([float(elapsed_ms)], dtype=torch.float64, device=dev)
    if dist.is_available() and dist.is_initialized():
        # pack max into the same collective: max(t) = -min(-t) is not a sum,
        # so two calls on 4 scalars -- still latency-only (~10 us on NVLink)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    s = sums.tolist()
    return {"points": int(s[0]), "frames": int(s[1]), "segments": int(s[2]), "elapsed_ms": float(mx.item())}
