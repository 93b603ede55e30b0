"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden vectors.  Bit-exact for indices / labels; normals compared
in fp64 (expected bit-exact, asserted to 1e-12) and in fp32 to 1e-5."""

import numpy as np
import pytest
import torch

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

PIPE = golden_names("vlp16") + golden_names("small") + golden_names("maxedge")


@pytest.fixture(scope="module")
def L():
    import paper_2005_02704_b200 as L
    return L


def sensor(L, g):
    return L.SensorConfig(ring_elevations=g["elev"], azimuth_steps=int(g["steps"]), r_min=float(g["r_min"]),
                          r_max=float(g["r_max"]))


@pytest.mark.parametrize("name", PIPE)
def test_ops_match_golden(L, name):
    g = load_golden(name)
    cfg = sensor(L, g)
    grid = L.ScanGrid(config=cfg, ranges=g["ranges"])
    me = None if float(g["max_edge"]) < 0 else float(g["max_edge"])
    mesh = L.build_mesh(grid, int(g["interval"]), max_edge_length=me)
    np.testing.assert_array_equal(mesh.kept_steps, g["kept"])
    np.testing.assert_array_equal(mesh.node_ids, g["node_ids"])
    np.testing.assert_array_equal(mesh.neighbors, g["neighbors"])
    np.testing.assert_array_equal(mesh.node_rings, g["node_rings"])
    np.testing.assert_array_equal(mesh.node_steps, g["node_steps"])
    np.testing.assert_array_equal(L.mesh_triangles(mesh), g["triangles"])
    nm = L.estimate_normals(grid, mesh)
    np.testing.assert_array_equal(nm.mask, g["nmask"])
    m = nm.mask
    np.testing.assert_allclose(nm.values[m], g["normals"][m], rtol=0, atol=1e-12)
    exact = np.mean(nm.values[m] == g["normals"][m]) if m.any() else 1.0
    assert exact == 1.0, f"fp64 normals not bit-exact: {exact:.6f}"
    scfg = L.SegmenterConfig(*[float(t) for t in g["thr"]], min_segment_size=int(g["mseg"]))
    dense = L.segment(mesh, nm, scfg)
    np.testing.assert_array_equal(dense, g["node_dense"])
    filled = L.backfill(grid, dense)
    np.testing.assert_array_equal(filled, g["filled"])
    np.testing.assert_array_equal(L.prune_small(filled, int(g["mseg"])), g["labels"])
    if me is None:
        res = L.run_pipeline(grid, L.PipelineConfig(sensor=cfg, interval=int(g["interval"]), segmenter=scfg))
        np.testing.assert_array_equal(res.labels, g["labels"])
        assert set(res.timings_ms) == {"mesh", "normals", "segment", "backfill", "total"}


@pytest.mark.parametrize("name", golden_names("seg"))
def test_segment_prescribed_normals(L, name):
    g = load_golden(name)
    cfg = L.SensorConfig(ring_elevations=g["elev"], azimuth_steps=int(g["steps"]))
    grid = L.ScanGrid(config=cfg, ranges=g["ranges"])
    mesh = L.build_mesh(grid, 1)
    np.testing.assert_array_equal(mesh.neighbors, g["neighbors"])
    nm = L.NormalMap(values=g["values"], mask=g["mask"])
    dense = L.segment(mesh, nm, L.SegmenterConfig(*[float(t) for t in g["thr"]]))
    np.testing.assert_array_equal(dense, g["node_dense"])


@pytest.mark.parametrize("name", golden_names("fill"))
def test_backfill_prune_golden(L, name):
    g = load_golden(name)
    cfg = L.SensorConfig(ring_elevations=g["elev"], azimuth_steps=int(g["steps"]))
    grid = L.ScanGrid(config=cfg, ranges=g["ranges"])
    filled = L.backfill(grid, g["labels_in"])
    np.testing.assert_array_equal(filled, g["filled"])
    np.testing.assert_array_equal(L.prune_small(filled, int(g["mseg"])), g["pruned"])


@pytest.mark.parametrize("name", golden_names("vlp16"))
def test_bin_points_golden(L, name):
    g = load_golden(name)
    grid = L.bin_points(g["xyz"], g["ring"], sensor(L, g))
    np.testing.assert_array_equal(grid.ranges, g["ranges"])


def _run_batch(L, shape_name, frames, k, seed=5, normals="exact"):
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS[shape_name]
    xyz, ring, off = synth.make_batch(shape, frames=frames, seed=seed, device="cuda")
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    bp = L.BatchPipeline(cfg, k, frames=frames, keep_node_labels=True, normals=normals)
    bp.run(xyz, ring, off)
    torch.cuda.synchronize()
    return shape, cfg, bp, xyz.cpu().numpy(), ring.cpu().numpy(), off.cpu().numpy()


@pytest.mark.parametrize("normals", ["certified", "exact"])
@pytest.mark.parametrize("shape_name,frames,k", [("vlp16", 3, 1), ("vlp16", 2, 5), ("hdl64", 2, 1),
                                                  ("hdl64", 2, 5), ("os128", 1, 1), ("os128", 1, 5)])
def test_batch_pipeline_vs_oracle(L, oracle, shape_name, frames, k, normals):
    shape, cfg, bp, xyz, ring, off = _run_batch(L, shape_name, frames, k, normals=normals)
    for f in range(frames):
        sl = slice(off[f], off[f + 1])
        want = oracle.run_from_points(xyz[sl], ring[sl], shape.elevations, shape.steps, k, shape.r_min,
                                      shape.r_max)
        got = bp.frame(f)
        np.testing.assert_array_equal(got["ranges"], want["ranges"])
        np.testing.assert_array_equal(got["node_ids"], want["mesh"]["node_ids"])
        np.testing.assert_array_equal(got["neighbors"], want["mesh"]["neighbors"])
        np.testing.assert_array_equal(got["mask"], want["mask"])
        m = want["mask"]
        # normals within 1e-5 per component (fp32); the exact
        # mode is additionally the exact rounding of the reference's fp64 values
        np.testing.assert_allclose(got["normals"][m], want["normals"][m], rtol=0, atol=1e-5)
        if normals == "exact":
            np.testing.assert_array_equal(got["normals"][m], want["normals"][m].astype(np.float32))
        # labels are bit-exact in both modes (undecided edges take the exact path)
        np.testing.assert_array_equal(got["node_labels"], want["node_labels"])
        np.testing.assert_array_equal(got["labels"], want["labels"])


@pytest.mark.parametrize("normals", ["certified", "exact"])
def test_stress_frame_vs_oracle(L, oracle, normals):
    shape, cfg, bp, xyz, ring, off = _run_batch(L, "stress", 1, 1, seed=9, normals=normals)
    want = oracle.run_from_points(xyz, ring, shape.elevations, shape.steps, 1, shape.r_min, shape.r_max)
    got = bp.frame(0)
    np.testing.assert_array_equal(got["neighbors"], want["mesh"]["neighbors"])
    np.testing.assert_array_equal(got["node_labels"], want["node_labels"])
    np.testing.assert_array_equal(got["labels"], want["labels"])


def test_determinism_and_empty_frames(L):
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS["hdl64"]
    xyz, ring, off = synth.make_batch(shape, frames=2, seed=1, device="cuda")
    # frame 1 empty, frame 2 = frame 1 of the batch, frame 0 = frame 0
    n0 = int(off[1])
    off3 = torch.tensor([0, n0, n0, int(off[2])], dtype=torch.int64, device="cuda")
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    bp = L.BatchPipeline(cfg, 1, frames=3)
    a = bp.run(xyz, ring, off3).clone()
    b = bp.run(xyz, ring, off3).clone()
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert int(bp.n_nodes[1]) == 0 and int(bp.n_labels[1]) == 0
    assert int(a[1].abs().sum()) == 0
    bp1 = L.BatchPipeline(cfg, 1, frames=1)
    bp1.run(xyz[n0:], ring[n0:], torch.tensor([0, int(off[2]) - n0], dtype=torch.int64, device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(bp1.labels[0], a[2])


def test_value_errors(L):
    cfg = L.SensorConfig.uniform(rings=4, azimuth_steps=8)
    grid = L.ScanGrid(config=cfg, ranges=np.full((4, 8), 5.0))
    with pytest.raises(ValueError):
        L.build_mesh(grid, 0)
    with pytest.raises(ValueError):
        L.build_mesh(grid, 8)
    with pytest.raises(ValueError):
        L.SegmenterConfig(threshold_i=0.0)


def test_unsorted_points_take_generic_binning(L):
    """Shuffled (non ring-major) input and out-of-range ring ids give the same
    result as ring-major input (k_bin_rows flags the frame, k_bin_atomic bins it)."""
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS["vlp16"]
    xyz, ring, off = synth.make_batch(shape, frames=2, seed=4, device="cuda")
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    bp = L.BatchPipeline(cfg, 1, frames=2)
    want = bp.run(xyz, ring, off).clone()
    want_r = bp.ranges.clone()
    n0 = int(off[1])
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    perm = torch.randperm(int(off[2]) - n0, device="cuda", generator=g) + n0
    idx = torch.cat([torch.arange(n0, device="cuda"), perm])
    xs, rs = xyz[idx].contiguous(), ring[idx].contiguous()
    # extra points with invalid ring ids in frame 1 must be ignored
    xs = torch.cat([xs, torch.ones((3, 3), device="cuda")])
    rs = torch.cat([rs, torch.tensor([-1, shape.rings, 99], dtype=torch.int32, device="cuda")])
    off2 = torch.tensor([0, n0, xs.shape[0]], dtype=torch.int64, device="cuda")
    got = bp.run(xs, rs, off2)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    assert torch.equal(torch.nan_to_num(bp.ranges, nan=-1.0), torch.nan_to_num(want_r, nan=-1.0))


def test_unsorted_points_k5(L, oracle):
    """Generic binning path at k = 5 (full-resolution valid bits come from the
    atomic path), checked against the oracle."""
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS["vlp16"]
    xyz, ring, off = synth.make_batch(shape, frames=1, seed=8, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    perm = torch.randperm(xyz.shape[0], device="cuda", generator=g)
    xs, rs = xyz[perm].contiguous(), ring[perm].contiguous()
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    bp = L.BatchPipeline(cfg, 5, frames=1)
    bp.run(xs, rs, off)
    torch.cuda.synchronize()
    want = oracle.run_from_points(xyz.cpu().numpy(), ring.cpu().numpy(), shape.elevations, shape.steps, 5,
                                  shape.r_min, shape.r_max)
    np.testing.assert_array_equal(bp.frame(0)["labels"], want["labels"])


@pytest.mark.parametrize("name", golden_names("edges"))
def test_edge_evaluator_golden(L, name):
    g = load_golden(name)
    r = int(g["radius"])
    if "pe" in g:
        np.testing.assert_array_equal(L.extract_edges(g["pred"]), g["pe"])
        np.testing.assert_array_equal(L.extract_edges(g["truth"]), g["te"])
        np.testing.assert_array_equal(L.dilate_chebyshev(g["te"], r), g["dil"])
    rep = L.edge_prf(g["pred"], g["truth"], L.EvalConfig(dilation_radius=r))
    np.testing.assert_array_equal([rep.precision, rep.recall, rep.f1], g["prf"])


def test_edge_prf_batch_matches_oracle(L, oracle):
    """Batched device scoring of pipeline labels against a second labelling."""
    shape, cfg, bp, xyz, ring, off = _run_batch(L, "hdl64", 3, 1, seed=6)
    other = L.BatchPipeline(cfg, 5, frames=3)
    other.run(torch.from_numpy(xyz).cuda(), torch.from_numpy(ring).cuda(), torch.from_numpy(off).cuda())
    prf = L.edge_prf_batch(bp.labels, other.labels, 2).cpu().numpy()
    for f in range(3):
        want = oracle.edge_prf(bp.labels[f].cpu().numpy(), other.labels[f].cpu().numpy(), 2)
        np.testing.assert_allclose(prf[f], want, rtol=1e-12)


def test_byte_ring_ids_match_int32(L):
    """lseg_run_pipeline_r8 (one-byte ring ids) == lseg_run_pipeline."""
    from paper_2005_02704_b200 import synth
    for name in ("vlp16", "hdl64"):
        shape = synth.CONFIGS[name]
        xyz, ring, off = synth.make_batch(shape, frames=2, seed=12, device="cuda")
        cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                             r_max=shape.r_max)
        a = L.BatchPipeline(cfg, 1, frames=2)
        b = L.BatchPipeline(cfg, 1, frames=2)
        la = a.run(xyz, ring, off).clone()
        lb = b.run(xyz, ring.to(torch.uint8), off).clone()
        torch.cuda.synchronize()
        assert torch.equal(la, lb)
        for f in range(2):
            n = int(a.n_nodes[f])
            assert n == int(b.n_nodes[f])
            assert torch.equal(a.neighbors[f, :n], b.neighbors[f, :n])


def test_ring_segment_input_matches_ring_ids(L):
    """Ring-major points + per-frame ring segment table
    (LSEG_PIPE_RING_SEGMENTS) == per-point ring ids, incl. an empty frame."""
    from paper_2005_02704_b200 import synth
    for name, k in (("vlp16", 1), ("hdl64", 5)):
        shape = synth.CONFIGS[name]
        xyz, ring, off = synth.make_batch(shape, frames=2, seed=14, device="cuda")
        n0 = int(off[1])
        off3 = torch.tensor([0, n0, n0, int(off[2])], dtype=torch.int64, device="cuda")
        cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                             r_max=shape.r_max)
        a = L.BatchPipeline(cfg, k, frames=3)
        b = L.BatchPipeline(cfg, k, frames=3)
        la = a.run(xyz, ring, off3).clone()
        seg = L.ring_segments(ring, off3, shape.rings)
        lb = b.run(xyz, seg, off3).clone()
        torch.cuda.synchronize()
        assert torch.equal(la, lb)
        assert torch.equal(a.n_nodes, b.n_nodes)


def test_streaming_pipeline_host_to_host(L):
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS["hdl64"]
    xyz, ring, off = synth.make_batch(shape, frames=5, seed=13, device="cuda")
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    ref = L.BatchPipeline(cfg, 1, frames=5)
    want = ref.run(xyz, ring, off).cpu()
    hx, hr, ho = xyz.cpu().pin_memory(), ring.to(torch.uint8).cpu().pin_memory(), off.cpu()
    hl = torch.empty((5, shape.rings, shape.steps), dtype=torch.int32).pin_memory()
    sp = L.StreamingPipeline(cfg, 1, chunk_frames=2, device="cuda", ring_dtype=torch.uint8)
    sp.run_host(hx, hr, ho, hl)
    torch.cuda.synchronize()
    assert torch.equal(hl, want)
    # ring-segment input form
    hs = L.ring_segments(ring.cpu(), ho, shape.rings).pin_memory()
    hl2 = torch.zeros_like(hl).pin_memory()
    sp2 = L.StreamingPipeline(cfg, 1, chunk_frames=2, device="cuda", ring_dtype="segments")
    sp2.run_host(hx, hs, ho, hl2)
    torch.cuda.synchronize()
    assert torch.equal(hl2, want)
    # the whole result on the host (labels + mesh + normals), int32 rings,
    # 3 chunks of unequal size (2, 2, 1 frames)
    cap = ref.cap
    full = {"n_nodes_h": torch.zeros(5, dtype=torch.int32).pin_memory(),
            "neighbors_h": torch.zeros((5, cap, 6), dtype=torch.int32).pin_memory(),
            "normals_h": torch.zeros((5, cap, 3), dtype=torch.float32).pin_memory(),
            "mask_h": torch.zeros((5, cap), dtype=torch.uint8).pin_memory()}
    hl3 = torch.zeros_like(hl).pin_memory()
    sp3 = L.StreamingPipeline(cfg, 1, chunk_frames=2, device="cuda", ring_dtype=torch.int32)
    sp3.run_host(hx, ring.cpu().pin_memory(), ho, hl3, **full)
    torch.cuda.synchronize()
    assert torch.equal(hl3, want)
    assert torch.equal(full["n_nodes_h"], ref.n_nodes.cpu())
    for f in range(5):
        n = int(ref.n_nodes[f])
        assert torch.equal(full["neighbors_h"][f, :n], ref.neighbors[f, :n].cpu())
        assert torch.equal(full["mask_h"][f, :n], ref.nmask[f, :n].cpu())
        assert torch.equal(full["normals_h"][f, :n].view(torch.int32), ref.normals[f, :n].cpu().view(torch.int32))


@pytest.mark.parametrize("shape_name,frames,seed", [("hdl64", 4, 21), ("stress", 1, 22), ("vlp16", 8, 23)])
def test_certified_normal_bounds_hold(L, oracle, shape_name, frames, seed):
    """The certified fp32 normals obey their per-node error bound against the
    reference's exact fp64 normals (the bound is what makes the fp32 edge
    decisions safe), and stay within the 1e-5 output tolerance."""
    import ctypes as C
    from paper_2005_02704_b200 import _lib, synth
    shape = synth.CONFIGS[shape_name]
    xyz, ring, off = synth.make_batch(shape, frames=frames, seed=seed, device="cuda")
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    bp = L.BatchPipeline(cfg, 1, frames=frames, normals="certified")
    err = torch.full((frames, bp.cap), -2.0, dtype=torch.float32, device="cuda")
    lib = _lib.lib()
    lib.lseg_debug_cert_err.argtypes = [C.c_void_p]
    lib.lseg_debug_cert_err(_lib.ptr(err))
    bp.run(xyz, ring, off)
    torch.cuda.synchronize()
    xyz_h, ring_h, off_h = xyz.cpu().numpy(), ring.cpu().numpy(), off.cpu().numpy()
    n_exact = n_tot = 0
    worst = 0.0
    reasons = {}
    for f in range(frames):
        sl = slice(off_h[f], off_h[f + 1])
        want = oracle.run_from_points(xyz_h[sl], ring_h[sl], shape.elevations, shape.steps, 1, shape.r_min,
                                      shape.r_max)
        got = bp.frame(f)
        m = want["mask"]
        e = err[f, :m.size].cpu().numpy()
        d = np.abs(got["normals"][m].astype(np.float64) - want["normals"][m]).max(axis=1)
        em = e[m]
        assert (em != -1).all() and (em != -2).all()
        cert = em > 0
        assert (d[cert] <= em[cert]).all(), "certified bound violated"
        # nodes that took the exact path carry the exact fp32 rounding
        assert (d[~cert] <= 6e-8).all()
        assert d.max() <= 1e-5
        worst = max(worst, float((d[cert] / em[cert]).max()) if cert.any() else 0.0)
        n_exact += int((~cert).sum())
        n_tot += int(m.sum())
        for code in range(1, 7):
            reasons[code] = reasons.get(code, 0) + int((em == -10.0 - code).sum())
    print(f"certified: worst error/bound {worst:.3g}, exact fallbacks {n_exact}/{n_tot}, by reason {reasons}")
    assert n_exact < 0.05 * n_tot, f"exact fallbacks {n_exact}/{n_tot}"


def _grid_points(rng, R, S, top, bottom, base=5.0, noise=0.3, keep=0.9, planar=True):
    """Ring-major f32 points of a random smooth range grid (plus dropouts)."""
    elev = np.radians(np.linspace(top, bottom, R))
    az = 2.0 * np.pi * np.arange(S) / S
    if planar:
        rr = base + noise * np.sin(az)[None, :] * np.cos(elev)[:, None] + rng.uniform(-0.02, 0.02, size=(R, S))
    else:
        rr = base + rng.uniform(-noise, noise, size=(R, S))
    valid = rng.random((R, S)) < keep
    dirs = np.stack([np.cos(elev)[:, None] * np.cos(az)[None, :], np.cos(elev)[:, None] * np.sin(az)[None, :],
                     np.broadcast_to(np.sin(elev)[:, None], (R, S))], axis=-1)
    pts = (dirs * rr[:, :, None])[valid].astype(np.float32)
    ring = np.nonzero(valid)[0].astype(np.int32)
    return elev, pts, ring


@pytest.mark.parametrize("R,S,k,mseg,keep", [
    (2, 16, 1, 0, 1.0),        # minimum rings, tiny grid
    (3, 10, 9, 2, 0.9),        # k = S - 1: S' = 2, slot N5 dropped (mesh.py:96-101)
    (5, 40, 7, 3, 0.8),        # S mod k != 0 (wrap gap)
    (4, 9000, 1, 10, 0.95),    # S > 8192: generic binning path (no fused rows)
    (6, 64, 1, 10 ** 6, 0.9),  # everything small: all labels dissolve to 0
    (7, 130, 2, 1, 0.0),       # no valid point at all
    (16, 1800, 3, 5, 0.5),     # sparse, fragmented
    (3, 40, 6, 2, 0.9),        # backfill tie across the wrap gap (cell 38: 2 steps to 36 and to 0)
    (4, 50, 4, 2, 0.95),       # interior ties (j = k / 2 -> left donor) and a wrap tie (cell 49)
])
def test_edge_shapes_vs_oracle(L, oracle, R, S, k, mseg, keep):
    """Edge cases of the batched path (the reference's own tests cover them
    for the single-scan API): tiny / degenerate grids, S' = 2, wrap gaps,
    the generic binning path, total pruning, empty frames, fragmentation."""
    rng = np.random.default_rng(R * 1000 + S + k)
    elev, pts, ring = _grid_points(rng, R, S, 10.0, -20.0, keep=keep, planar=(R % 2 == 0))
    off = np.array([0, pts.shape[0]], dtype=np.int64)
    cfg = L.SensorConfig(ring_elevations=elev, azimuth_steps=S, r_min=0.5, r_max=100.0)
    for normals in ("exact", "certified"):
        bp = L.BatchPipeline(cfg, k, L.SegmenterConfig(min_segment_size=mseg), frames=1, keep_node_labels=True,
                             normals=normals)
        bp.run(torch.from_numpy(pts).cuda(), torch.from_numpy(ring).cuda(), torch.from_numpy(off).cuda())
        torch.cuda.synchronize()
        want = oracle.run_from_points(pts, ring, elev, S, k, 0.5, 100.0, min_segment_size=mseg)
        got = bp.frame(0)
        np.testing.assert_array_equal(np.nan_to_num(got["ranges"], nan=-1.0), np.nan_to_num(want["ranges"], nan=-1.0))
        np.testing.assert_array_equal(got["node_ids"], want["mesh"]["node_ids"])
        np.testing.assert_array_equal(got["neighbors"], want["mesh"]["neighbors"])
        np.testing.assert_array_equal(got["mask"], want["mask"])
        np.testing.assert_array_equal(got["node_labels"], want["node_labels"])
        np.testing.assert_array_equal(got["labels"], want["labels"])


def test_cuda_graph_capture_replays_exactly(L):
    """BatchPipeline.capture: one CUDA graph per scan (the latency path);
    replaying it after refilling the inputs in place gives the eager result."""
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS["vlp16"]
    x0, r0, o0 = synth.make_batch(shape, frames=1, seed=30, device="cuda")
    x1, r1, o1 = synth.make_batch(shape, frames=1, seed=31, device="cuda")
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    n = max(int(x0.shape[0]), int(x1.shape[0]))
    xb = torch.zeros((n, 3), dtype=torch.float32, device="cuda")
    rb = torch.zeros(n, dtype=torch.int32, device="cuda")
    ob = torch.zeros(2, dtype=torch.int64, device="cuda")
    eager = L.BatchPipeline(cfg, 1, frames=1)
    for normals in ("exact", "certified"):
        bp = L.BatchPipeline(cfg, 1, frames=1, normals=normals)
        xb[: x0.shape[0]], rb[: r0.shape[0]], ob.copy_(o0)
        g = bp.capture(xb, rb, ob)
        for x, r, o in ((x1, r1, o1), (x0, r0, o0)):
            xb[: x.shape[0]].copy_(x)
            rb[: r.shape[0]].copy_(r)
            ob.copy_(o)
            g.replay()
            want = eager.run(x, r, o)
            torch.cuda.synchronize()
            assert torch.equal(bp.labels, want)


def test_full_bench_batch_sampled_vs_oracle(L, oracle):
    """The bench workload at its full size (512 HDL-64 frames, one batch):
    four sampled frames equal the oracle exactly, and every frame satisfies
    the size-independent invariants -- final labels are exactly 1..n_final
    (compacted, no gaps), every labelled cell is a valid cell, and a ring
    with any label has all its valid cells labelled (backfill)."""
    from paper_2005_02704_b200 import synth
    shape = synth.CONFIGS["hdl64_batch"]
    F = shape.frames
    xyz, ring, off = synth.make_batch(shape, frames=F, seed=2005, device="cuda")
    cfg = L.SensorConfig(ring_elevations=shape.elevations, azimuth_steps=shape.steps, r_min=shape.r_min,
                         r_max=shape.r_max)
    bp = L.BatchPipeline(cfg, 1, frames=F)
    labels = bp.run(xyz, ring, off)
    torch.cuda.synchronize()
    # invariants on every frame (device-side)
    valid = torch.isfinite(bp.ranges) & (bp.ranges >= shape.r_min) & (bp.ranges <= shape.r_max)
    assert not bool(((labels > 0) & ~valid).any())
    mx = labels.amax(dim=(1, 2))
    for f in range(F):
        present = torch.zeros(int(mx[f]) + 1, dtype=torch.bool, device="cuda")
        present[labels[f].reshape(-1).long()] = True
        assert bool(present[1:].all()), f"frame {f}: label ids not compact"
    ring_has = (labels > 0).any(dim=2, keepdim=True)
    assert not bool((ring_has & valid & (labels == 0)).any())
    # four sampled frames against the oracle
    xh, rh, oh = xyz.cpu().numpy(), ring.cpu().numpy(), off.cpu().numpy()
    for f in (0, 137, 300, F - 1):
        sl = slice(oh[f], oh[f + 1])
        want = oracle.run_from_points(xh[sl], rh[sl], shape.elevations, shape.steps, 1, shape.r_min, shape.r_max)
        np.testing.assert_array_equal(labels[f].cpu().numpy(), want["labels"])
