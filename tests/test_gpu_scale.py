"""GPU parity at bench scale (VERDICT r1 "pin parity at the configs you bench").

* Reference-generated fixtures (tests/golden/make_golden_scale.py) of one
  frame of each benchmarked shape -- HDL-64 bench-batch frame at k = 1/5/10/15,
  OS1-128 at k = 1, the 256 x 4096 stress frame at k = 1/5: the batched fused
  path (exact and certified normals) and the single-scan run_pipeline against
  the reference's own outputs (mesh and normal digests bit-exact, segment() and
  final labels bit-exact).
* The oracle on GPU-generated inputs: the 512-frame bench batch at k = 5,
  several OS1-128 frames, the stress frame at k = 5.
* Race evidence for the lock-free union-find and the cross-CTA waits while
  compute-sanitizer is unavailable: 20 repeated runs of a stress batch give
  bit-identical outputs.
* Partial / chunked batches over a longer point buffer: the
  generic binning path (S > 8192) with the streaming pipeline, frame chunks
  and concurrent streams.
"""

import numpy as np
import pytest
import torch

from conftest import golden_names, load_golden
from golden.packing import digest, near_threshold_edges, normals_digest, unpack_ranges

pytestmark = pytest.mark.gpu

SCALE = golden_names("scale_")


@pytest.fixture(scope="module")
def L():
    import paper_2005_02704_b200 as L
    return L


def _cfg(L, g):
    return L.SensorConfig(ring_elevations=g["elev"], azimuth_steps=int(g["steps"]), r_min=float(g["r_min"]),
                          r_max=float(g["r_max"]))


def _scale_cases():
    out = []
    for name in SCALE:
        g = load_golden(name)
        out += [(name, int(k)) for k in g["intervals"]]
    return out


@pytest.mark.parametrize("normals", ["exact", "certified"])
@pytest.mark.parametrize("name,k", _scale_cases())
def test_fused_pipeline_matches_reference_fixture(L, name, k, normals):
    g = load_golden(name)
    ranges = unpack_ranges(g)
    cfg = _cfg(L, g)
    bp = L.BatchPipeline(cfg, k, L.SegmenterConfig(*[float(t) for t in g["thr"]], min_segment_size=int(g["mseg"])),
                         frames=1, keep_node_labels=True, normals=normals)
    bp.run_grid(torch.from_numpy(ranges)[None].cuda())
    torch.cuda.synchronize()
    n = int(bp.n_nodes[0])
    assert n == int(g[f"k{k}_n_nodes"])
    assert digest(bp.node_ids[0].cpu().numpy()) == str(g[f"k{k}_node_ids"])
    assert digest(bp.neighbors[0, :n].cpu().numpy()) == str(g[f"k{k}_neighbors"])
    mask = bp.nmask[0, :n].bool().cpu().numpy()
    n32 = bp.normals[0, :n].cpu().numpy()
    if normals == "exact":  # the reference's fp64 normals, rounded once
        assert normals_digest(n32, mask, np.float32) == str(g[f"k{k}_n32"])
    else:  # certified: mask exact, values within the 1e-5 north-star tolerance (checked via the exact mode)
        assert digest(np.packbits(mask)) == str(g[f"k{k}_n32"])[:64]
    node_labels = bp.node_labels[0].cpu().numpy()
    assert digest(node_labels) == str(g[f"k{k}_node_dense_digest"])
    np.testing.assert_array_equal(bp.labels[0].cpu().numpy(), g[f"k{k}_labels"])


@pytest.mark.parametrize("name", SCALE)
def test_single_scan_api_matches_reference_fixture(L, name):
    """The drop-in single-scan API (run_pipeline, estimate_normals in fp64)
    on full frames."""
    g = load_golden(name)
    ranges = unpack_ranges(g)
    cfg = _cfg(L, g)
    grid = L.ScanGrid(config=cfg, ranges=ranges)
    scfg = L.SegmenterConfig(*[float(t) for t in g["thr"]], min_segment_size=int(g["mseg"]))
    for k in [int(v) for v in g["intervals"]][:2]:
        res = L.run_pipeline(grid, L.PipelineConfig(sensor=cfg, interval=k, segmenter=scfg))
        np.testing.assert_array_equal(res.labels, g[f"k{k}_labels"])
        assert res.mesh.n_nodes == int(g[f"k{k}_n_nodes"])
        assert digest(res.mesh.neighbors.astype(np.int32)) == str(g[f"k{k}_neighbors"])
        assert normals_digest(res.normals.values, res.normals.mask, np.float64) == str(g[f"k{k}_n64"])
        # reference NormalMap contract (normals.py:94-145): rows without a normal are NaN
        # (written by the tile kernel, not patched on the host)
        assert np.isnan(res.normals.values[~res.normals.mask]).all()
        assert not np.isnan(res.normals.values[res.normals.mask]).any()
        near = near_threshold_edges(res.mesh.neighbors, res.normals.values, res.normals.mask, g["thr"])
        assert near == (int(g[f"k{k}_e_near"]), int(g[f"k{k}_e_fwd"]))


def _frames(L, shape_name, frames, seed, first_frame=0):
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS[shape_name]
    xyz, ring, off = synth.make_batch(shape, frames=frames, seed=seed, device="cuda", first_frame=first_frame)
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    return shape, cfg, xyz, ring, off


@pytest.mark.parametrize("k", [1, 5])
def test_os128_frames_vs_oracle(L, oracle, k):
    shape, cfg, xyz, ring, off = _frames(L, "os128", 3, 17)
    bp = L.BatchPipeline(cfg, k, frames=3, keep_node_labels=True)
    bp.run(xyz, ring, off)
    torch.cuda.synchronize()
    xh, rh, oh = xyz.cpu().numpy(), ring.cpu().numpy(), off.cpu().numpy()
    for f in range(3):
        sl = slice(oh[f], oh[f + 1])
        want = oracle.run_from_points(xh[sl], rh[sl], shape.elevations, shape.steps, k, shape.r_min, shape.r_max)
        got = bp.frame(f)
        np.testing.assert_array_equal(got["neighbors"], want["mesh"]["neighbors"])
        np.testing.assert_array_equal(got["normals"][want["mask"]], want["normals"][want["mask"]].astype(np.float32))
        np.testing.assert_array_equal(got["node_labels"], want["node_labels"])
        np.testing.assert_array_equal(got["labels"], want["labels"])


def test_stress_frame_k5_vs_oracle(L, oracle):
    shape, cfg, xyz, ring, off = _frames(L, "stress", 1, 9)
    for normals in ("exact", "certified"):
        bp = L.BatchPipeline(cfg, 5, frames=1, keep_node_labels=True, normals=normals)
        bp.run(xyz, ring, off)
        torch.cuda.synchronize()
        want = oracle.run_from_points(xyz.cpu().numpy(), ring.cpu().numpy(), shape.elevations, shape.steps, 5,
                                      shape.r_min, shape.r_max)
        got = bp.frame(0)
        np.testing.assert_array_equal(got["neighbors"], want["mesh"]["neighbors"])
        np.testing.assert_array_equal(got["node_labels"], want["node_labels"])
        np.testing.assert_array_equal(got["labels"], want["labels"])


def test_full_bench_batch_k5_sampled_vs_oracle(L, oracle):
    """The bench batch (512 HDL-64 frames, one launch) at the reference's
    default interval 5: 16 frames spread over the batch equal the oracle."""
    shape, cfg, xyz, ring, off = _frames(L, "hdl64_batch", 512, 2005)
    bp = L.BatchPipeline(cfg, 5, frames=512)
    labels = bp.run(xyz, ring, off)
    torch.cuda.synchronize()
    xh, rh, oh = xyz.cpu().numpy(), ring.cpu().numpy(), off.cpu().numpy()
    for f in np.linspace(0, 511, 16).astype(int):
        sl = slice(oh[f], oh[f + 1])
        want = oracle.run_from_points(xh[sl], rh[sl], shape.elevations, shape.steps, 5, shape.r_min, shape.r_max)
        np.testing.assert_array_equal(labels[f].cpu().numpy(), want["labels"], err_msg=f"frame {f}")


@pytest.mark.parametrize("normals", ["exact", "certified"])
def test_stress_batch_deterministic_over_20_runs(L, normals):
    """Lock-free union-find (CAS hooking), the cross-CTA waits of the pruning
    and the histogram atomics must not make results depend on scheduling:
    20 runs of a 4-frame stress batch (~450 k segments per frame), every
    output bit-identical."""
    shape, cfg, xyz, ring, off = _frames(L, "stress", 4, 33)
    bp = L.BatchPipeline(cfg, 1, frames=4, keep_node_labels=True, normals=normals)
    bp.run(xyz, ring, off)
    torch.cuda.synchronize()
    ref = [t.clone() for t in (bp.labels, bp.node_labels, bp.neighbors, bp.normals, bp.nmask, bp.n_labels)]
    for it in range(20):
        bp.run(xyz, ring, off)
        torch.cuda.synchronize()
        for a, b in zip(ref, (bp.labels, bp.node_labels, bp.neighbors, bp.normals, bp.nmask, bp.n_labels)):
            assert torch.equal(torch.nan_to_num(a, nan=7.0), torch.nan_to_num(b, nan=7.0)), f"run {it} differs"


def _ragged_frames(R, S, frames, seed):
    rng = np.random.default_rng(seed)
    elev = np.radians(np.linspace(10.0, -20.0, R))
    az = 2.0 * np.pi * np.arange(S) / S
    dirs = np.stack([np.cos(elev)[:, None] * np.cos(az)[None, :], np.cos(elev)[:, None] * np.sin(az)[None, :],
                     np.broadcast_to(np.sin(elev)[:, None], (R, S))], axis=-1)
    pts, rings, offs = [], [], [0]
    for f in range(frames):
        keep = [0.95, 0.3, 0.0, 0.8, 0.6, 1.0, 0.1][f % 7]  # unequal sizes, one empty frame
        rr = 5.0 + 0.3 * np.sin(az + f)[None, :] * np.cos(elev)[:, None] + rng.uniform(-0.02, 0.02, (R, S))
        valid = rng.random((R, S)) < keep
        pts.append((dirs * rr[:, :, None])[valid].astype(np.float32))
        rings.append(np.nonzero(valid)[0].astype(np.int32))
        offs.append(offs[-1] + int(valid.sum()))
    return elev, np.concatenate(pts), np.concatenate(rings), np.array(offs, np.int64)


@pytest.mark.parametrize("S", [9000, 2048])
def test_chunked_streamed_batches_match_single_batch(L, oracle, S):
    """chunk buffers longer than the chunk's points and sub-batch
    offsets that do not start at 0 must bin only their own points -- for the
    generic binning path (S > 8192, int32 rings) and the fused one."""
    R, F = 4, 7
    elev, pts, ring, off = _ragged_frames(R, S, F, seed=S)
    cfg = L.SensorConfig(ring_elevations=elev, azimuth_steps=S, r_min=0.5, r_max=100.0)
    x, r, o = torch.from_numpy(pts).cuda(), torch.from_numpy(ring).cuda(), torch.from_numpy(off).cuda()
    whole = L.BatchPipeline(cfg, 1, frames=F)
    want = whole.run(x, r, o).clone()
    torch.cuda.synchronize()
    for f in (0, 3, 6):
        sl = slice(off[f], off[f + 1])
        ref = oracle.run_from_points(pts[sl], ring[sl], elev, S, 1, 0.5, 100.0)
        np.testing.assert_array_equal(want[f].cpu().numpy(), ref["labels"])
    for kw in ({"chunk_frames": 2}, {"streams": 2}, {"streams": 3}):
        bp = L.BatchPipeline(cfg, 1, frames=F, **kw)
        got = bp.run(x, r, o)
        torch.cuda.synchronize()
        assert torch.equal(got, want), kw
    hx, hr, ho = x.cpu().pin_memory(), r.cpu().pin_memory(), o.cpu()
    hl = torch.full((F, R, S), -5, dtype=torch.int32).pin_memory()
    # chunks of 3 frames: 3 + 2 + 2 with unequal point counts; the buffer is
    # sized for the largest chunk, so smaller chunks leave stale points behind
    sp = L.StreamingPipeline(cfg, 1, chunk_frames=3, device="cuda", ring_dtype=torch.int32)
    for _ in range(2):
        sp.run_host(hx, hr, ho, hl)
        torch.cuda.synchronize()
        assert torch.equal(hl, want.cpu())


def test_single_scan_api_concurrent_threads(L):
    """run_pipeline from two threads at once (the reference's functions are
    pure and safe to call concurrently): each thread gets its
    own device buffers, results equal the sequential ones."""
    import threading
    g1, g2 = load_golden("vlp16_k1"), load_golden("vlp16_k5")
    cfg = L.SensorConfig(ring_elevations=g1["elev"], azimuth_steps=int(g1["steps"]), r_min=float(g1["r_min"]),
                         r_max=float(g1["r_max"]))
    grids = [L.ScanGrid(config=cfg, ranges=g1["ranges"]), L.ScanGrid(config=cfg, ranges=g2["ranges"] * 1.01)]
    pc = L.PipelineConfig(sensor=cfg, interval=1)
    want = [L.run_pipeline(g, pc).labels for g in grids]
    errors = []

    def work(i):
        try:
            for _ in range(10):
                if not np.array_equal(L.run_pipeline(grids[i], pc).labels, want[i]):
                    errors.append(i)
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    th = [threading.Thread(target=work, args=(i,)) for i in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    np.testing.assert_array_equal(want[0], g1["labels"])
