"""Frame sharding across GPUs of one node.

Frames are independent, so each rank processes its own contiguous block of
frames with no data-path collective; the only collective is one tiny
all-reduce at the end of a run carrying (points, frames, segments, elapsed).
Works with NCCL (GPU tensors) and gloo (CPU tensors, used by the tests).
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


def reduce_run(points: int, frames: int, segments: int, elapsed_ms: float, device=None) -> dict:
    """The run's single collective: sums of points / frames / segments and the
    max elapsed time over ranks (CUDA-event milliseconds)."""
    dev = torch.device(device) if device is not None else torch.device("cpu")
    sums = torch.tensor([float(points), float(frames), float(segments)], dtype=torch.float64, device=dev)
    mx = torch.tensor([float(elapsed_ms)], dtype=torch.float64, device=dev)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        # pack max into the same collective: max(t) = -min(-t) is not a sum,
        # so two calls on 4 scalars -- still latency-only (~10 us on NVLink)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    s = sums.tolist()
    return {"points": int(s[0]), "frames": int(s[1]), "segments": int(s[2]), "elapsed_ms": float(mx.item())}
