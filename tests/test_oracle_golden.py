"""Pin the CPU oracle to golden vectors produced by the reference itself.

Everything is required to be bit-exact, including fp64 normals: the oracle
restates the reference's arithmetic in the same IEEE operation order.
"""

import numpy as np
import pytest

from conftest import golden_names, load_golden

PIPE = golden_names("vlp16") + golden_names("small") + golden_names("maxedge")


@pytest.mark.parametrize("name", PIPE)
def test_pipeline_matches_reference(oracle, name):
    g = load_golden(name)
    me = None if float(g["max_edge"]) < 0 else float(g["max_edge"])
    mesh = oracle.build_mesh(g["ranges"], g["elev"], int(g["interval"]), float(g["r_min"]),
                             float(g["r_max"]), max_edge_length=me)
    np.testing.assert_array_equal(mesh["kept_steps"], g["kept"])
    np.testing.assert_array_equal(mesh["node_ids"], g["node_ids"])
    np.testing.assert_array_equal(mesh["neighbors"], g["neighbors"])
    np.testing.assert_array_equal(mesh["node_rings"], g["node_rings"])
    np.testing.assert_array_equal(mesh["node_steps"], g["node_steps"])
    np.testing.assert_array_equal(oracle.mesh_triangles(mesh["node_ids"]), g["triangles"])
    vals, mask = oracle.estimate_normals(g["ranges"], g["elev"], mesh)
    np.testing.assert_array_equal(mask, g["nmask"])
    np.testing.assert_array_equal(vals[mask], g["normals"][mask])  # bit-exact fp64
    dense = oracle.segment(mesh, vals, mask, g["thr"])
    np.testing.assert_array_equal(dense, g["node_dense"])
    valid = oracle.valid_mask(g["ranges"], float(g["r_min"]), float(g["r_max"]))
    filled = oracle.backfill(valid, dense)
    np.testing.assert_array_equal(filled, g["filled"])
    np.testing.assert_array_equal(oracle.prune_small(filled, int(g["mseg"])), g["labels"])


@pytest.mark.parametrize("name", golden_names("vlp16"))
def test_run_from_points(oracle, name):
    g = load_golden(name)
    out = oracle.run_from_points(g["xyz"], g["ring"], g["elev"], int(g["steps"]), int(g["interval"]),
                                 float(g["r_min"]), float(g["r_max"]))
    np.testing.assert_array_equal(out["ranges"], g["ranges"])
    np.testing.assert_array_equal(out["labels"], g["labels"])


@pytest.mark.parametrize("name", golden_names("seg"))
def test_segment_prescribed_normals(oracle, name):
    g = load_golden(name)
    R, S = g["ranges"].shape
    mesh = oracle.build_mesh(g["ranges"], g["elev"], 1, 0.5, 100.0)
    np.testing.assert_array_equal(mesh["neighbors"], g["neighbors"])
    dense = oracle.segment(mesh, g["values"], g["mask"], g["thr"])
    np.testing.assert_array_equal(dense, g["node_dense"])


@pytest.mark.parametrize("name", golden_names("fill"))
def test_backfill_prune(oracle, name):
    g = load_golden(name)
    valid = oracle.valid_mask(g["ranges"], 0.5, 100.0)
    filled = oracle.backfill(valid, g["labels_in"])
    np.testing.assert_array_equal(filled, g["filled"])
    np.testing.assert_array_equal(oracle.prune_small(filled, int(g["mseg"])), g["pruned"])


def test_bin_round_trip(oracle):
    """grid -> valid_points (f32) -> bin_points recovers the valid mask exactly
    and r to float32 precision (SURVEY.md §8(c) binning pins)."""
    rng = np.random.default_rng(0)
    R, S = 16, 1800
    elev = np.radians(np.arange(15, -16, -2, dtype=np.float64))
    rr = rng.uniform(0.6, 99.0, size=(R, S))
    rr[rng.random((R, S)) < 0.1] = np.nan
    dirs = oracle.ray_directions(elev, S)
    valid = oracle.valid_mask(rr, 0.5, 100.0)
    pts = (dirs * rr[:, :, None])[valid].astype(np.float32)
    ring = np.nonzero(valid)[0].astype(np.int32)
    got, cell = oracle.bin_points(pts, ring, R, S, 0.5, 100.0)
    np.testing.assert_array_equal(np.isfinite(got), valid)
    np.testing.assert_allclose(got[valid], rr[valid], rtol=2e-7)
    np.testing.assert_array_equal(cell, np.flatnonzero(valid))


def test_bin_collision_and_ring_convention(oracle):
    # two points in one cell: the smaller range wins; ring 0 is the top row
    xyz = np.array([[2.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 3.0, 0.0], [0.0, 0.0, 0.2],
                    [200.0, 0.0, 0.0]], np.float32)
    ring = np.array([0, 0, 1, 1, 1], np.int32)
    got, cell = oracle.bin_points(xyz, ring, 2, 8, 0.5, 100.0)
    assert got[0, 0] == 1.0
    assert got[1, 2] == 3.0
    assert cell.tolist() == [0, 0, 10, -1, -1]  # r=0.2 < r_min, r=200 > r_max
    assert np.isnan(got).sum() == 14


@pytest.mark.parametrize("name", golden_names("edges"))
def test_edge_evaluator(oracle, name):
    g = load_golden(name)
    r = int(g["radius"])
    if "pe" in g:
        np.testing.assert_array_equal(oracle.extract_edges(g["pred"]), g["pe"])
        np.testing.assert_array_equal(oracle.extract_edges(g["truth"]), g["te"])
        np.testing.assert_array_equal(oracle.dilate_chebyshev(g["te"], r), g["dil"])
    np.testing.assert_allclose(oracle.edge_prf(g["pred"], g["truth"], r), g["prf"], rtol=0, atol=0)


SCALE = golden_names("scale_")


@pytest.mark.parametrize("name", SCALE)
def test_oracle_matches_reference_at_bench_scale(oracle, name):
    """The oracle against reference outputs on full bench-shape frames
    (HDL-64 batch frame at k = 1/5/10/15, OS1-128, the 256 x 4096 stress
    frame): mesh, fp64 normals (digest, bit-exact), segment() labels and
    final labels."""
    from golden.packing import digest, near_threshold_edges, normals_digest, unpack_ranges
    g = load_golden(name)
    ranges = unpack_ranges(g)
    for k in [int(v) for v in g["intervals"]]:
        mesh = oracle.build_mesh(ranges, g["elev"], k, float(g["r_min"]), float(g["r_max"]))
        assert mesh["neighbors"].shape[0] == int(g[f"k{k}_n_nodes"])
        assert digest(mesh["node_ids"].astype(np.int32)) == str(g[f"k{k}_node_ids"])
        assert digest(mesh["neighbors"].astype(np.int32)) == str(g[f"k{k}_neighbors"])
        vals, mask = oracle.estimate_normals(ranges, g["elev"], mesh)
        assert normals_digest(vals, mask, np.float64) == str(g[f"k{k}_n64"])
        dense = oracle.segment(mesh, vals, mask, g["thr"])
        assert digest(dense.astype(np.int32)) == str(g[f"k{k}_node_dense_digest"])
        valid = oracle.valid_mask(ranges, float(g["r_min"]), float(g["r_max"]))
        labels = oracle.prune_small(oracle.backfill(valid, dense), int(g["mseg"]))
        np.testing.assert_array_equal(labels, g[f"k{k}_labels"])
        assert near_threshold_edges(mesh["neighbors"], vals, mask, g["thr"]) == (int(g[f"k{k}_e_near"]),
                                                                                 int(g[f"k{k}_e_fwd"]))


def test_range_packing_roundtrip():
    from golden.packing import pack_ranges, unpack_ranges
    rng = np.random.default_rng(0)
    r = rng.uniform(0.5, 120.0, size=(7, 33))
    r[rng.random(r.shape) < 0.3] = np.nan
    back = unpack_ranges(pack_ranges(r))
    np.testing.assert_array_equal(np.isnan(back), np.isnan(r))
    np.testing.assert_array_equal(back[~np.isnan(r)], r[~np.isnan(r)])
