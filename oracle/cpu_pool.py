"""CPU-baseline worker pool for bench.py -- TEST/BENCH INFRASTRUCTURE ONLY.

Runs the oracle port of the reference CPU path (lidarseg_oracle.run_from_points,
the same arithmetic as reference pipeline.py:47-70 preceded by the binning
restatement) over frames in a multiprocessing pool.  Kept in its own module
(numpy only) so "spawn" workers start without importing torch or CUDA.
"""

from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def _init():
    for var in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[var] = "1"


def run_frame(args):
    import lidarseg_oracle as oracle
    xyz, ring, elev, steps, interval, rmin, rmax = args
    oracle.run_from_points(xyz, ring, elev, steps, interval, rmin, rmax)
    return xyz.shape[0]


def timed_pool(jobs, workers: int, rounds: int = 1, warmup: int = 1, ctx: str = "spawn"):
    """Points/s of `rounds` passes of `jobs` over a pool of `workers`
    processes, after `warmup` untimed passes: (points_per_s, seconds)."""
    import multiprocessing as mp
    with mp.get_context(ctx).Pool(workers, initializer=_init) as pool:
        for _ in range(warmup):
            pool.map(run_frame, jobs)
        t0 = time.perf_counter()
        pts = 0
        for _ in range(rounds):
            pts += sum(pool.map(run_frame, jobs))
        dt = time.perf_counter() - t0
    return pts / dt, dt
