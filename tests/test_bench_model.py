"""bench.py's byte model is SURVEY.md §8(d)'s (CPU): the pipeline's
algorithmic bytes B = 16 P + 8 C + 36 N + 4 C, each kernel's share
(binning 16 P + 8 C, tile 8 C' + 36 N, pruning 4 C), and the committed ncu
DRAM bytes it reports next to them are the 512-frame bench workload's."""

import json
import os

from conftest import ROOT


def test_byte_model_matches_survey():
    import bench
    P, C, Ck, N = 63_199_739, 512 * 64 * 2048, 512 * 64 * 2048, 61_583_503
    assert bench.pipeline_bytes(P, C, N) == 16 * P + 8 * C + 36 * N + 4 * C
    alg = bench.alg_stage_bytes(P, C, Ck, N)
    assert alg == {"bin_rows": 16 * P + 8 * C, "tile": 8 * Ck + 36 * N, "prune_apply": 4 * C}
    # the kernels' shares cover B, plus the tile's re-read of the kept cells
    assert sum(alg.values()) == bench.pipeline_bytes(P, C, N) + 8 * Ck
    des = bench.design_stage_bytes(P, C, Ck, N, 1)
    assert all(des[k] >= alg.get(k, 0) for k in des)


def test_committed_traffic_is_the_bench_workload():
    import bench
    with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
        t = json.load(fh)
    for k in (1, 5):
        e = bench.committed_traffic("tile", 512, k)
        assert e is not None and e["frames"] == 512 and e["interval"] == k
        assert e["dram_bytes_per_launch"] == e["dram_read"] + e["dram_write"]
        assert os.path.exists(os.path.join(ROOT, e["source"]))
    assert bench.committed_traffic("tile", 128, 1) is None  # another workload: not reported
    assert all(v["frames"] == 512 for key, v in t.items() if not key.startswith("_"))
