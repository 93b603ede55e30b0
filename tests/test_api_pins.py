"""Known-answer pins of the reference's hot-path behaviour, exercised through
the GPU implementation's public API (SURVEY.md §4 lists the reference tests
these restate: mesh join rules and invariants, normal estimator rules,
segmentation / backfill / prune rules).  Written from the documented
behaviour, not copied; every assertion runs the CUDA path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2005_02704_b200 as L
    return L


def sensor(L, R=4, S=8, top=10.0, bottom=-30.0, r_max=100.0):
    return L.SensorConfig.uniform(rings=R, top_deg=top, bottom_deg=bottom, azimuth_steps=S, r_max=r_max)


def const_grid(L, R=4, S=8, value=5.0, **kw):
    return L.ScanGrid(config=sensor(L, R, S, **kw), ranges=np.full((R, S), value))


def mask_grid(L, mask, value=5.0):
    mask = np.asarray(mask, bool)
    return L.ScanGrid(config=sensor(L, *mask.shape), ranges=np.where(mask, value, np.nan))


def cells(mesh):
    out = set()
    for a, b in mesh.edges():
        pa = (int(mesh.node_rings[a]), int(mesh.node_steps[a]))
        pb = (int(mesh.node_rings[b]), int(mesh.node_steps[b]))
        out.add(tuple(sorted((pa, pb))))
    return out


# ---------------------------------------------------------------- mesh
def test_slot_order_interior_top_bottom(L):
    m = L.build_mesh(const_grid(L), 1)
    # interior node: below, below-right, right, above, above-left, left
    assert m.neighbor_cells(2, 5) == [(3, 5), (3, 6), (2, 6), (1, 5), (1, 4), (2, 4)]
    # top ring has no slots above, bottom ring none below
    assert m.neighbor_cells(0, 5) == [(1, 5), (1, 6), (0, 6), (0, 4)]
    assert m.neighbor_cells(3, 5) == [(3, 6), (2, 5), (2, 4), (3, 4)]


def test_azimuth_wrap_both_ways(L):
    m = L.build_mesh(const_grid(L), 1)
    assert {(2, 0), (3, 0), (3, 7)} <= set(m.neighbor_cells(2, 7))
    assert (2, 7) in m.neighbor_cells(2, 0)
    m5 = L.build_mesh(const_grid(L, 3, 1800), 5)  # sub-sampled wrap: 1795 -> 0
    assert {(1, 0), (2, 0), (2, 1795), (1, 1790)} <= set(m5.neighbor_cells(1, 1795))


def test_only_main_diagonal(L):
    e = cells(L.build_mesh(const_grid(L), 1))
    for i in range(3):
        for j in range(8):
            assert tuple(sorted(((i, j), (i + 1, (j + 1) % 8)))) in e
            assert tuple(sorted(((i, j), (i + 1, (j - 1) % 8)))) not in e


@pytest.mark.parametrize("R,S,k", [(4, 8, 1), (3, 12, 2), (5, 9, 3), (2, 6, 1), (6, 20, 7)])
def test_full_grid_edge_and_triangle_counts(L, R, S, k):
    g = const_grid(L, R, S)
    m = L.build_mesh(g, k)
    Sk = len(L.subsample_steps(g.config, k))
    assert m.edges().shape[0] == (3 * (R - 1) + 1) * Sk
    assert L.mesh_triangles(m).shape == (2 * (R - 1) * Sk, 3)


def test_random_masks_symmetric_simple(L):
    rng = np.random.default_rng(11)
    for _ in range(25):
        R, S = int(rng.integers(2, 9)), int(rng.integers(3, 17))
        mask = rng.random((R, S)) < rng.uniform(0.3, 1.0)
        m = L.build_mesh(mask_grid(L, mask), 1)
        assert m.n_nodes == mask.sum()
        d = set()
        for a in range(m.n_nodes):
            row = m.neighbors[a][m.neighbors[a] >= 0].tolist()
            assert len(set(row)) == len(row) and a not in row
            d |= {(a, b) for b in row}
        assert all((b, a) in d for a, b in d)


def test_removing_a_cell_removes_its_six_edges(L):
    full = cells(L.build_mesh(const_grid(L, 5, 10), 1))
    mask = np.ones((5, 10), bool)
    mask[2, 4] = False
    cut = cells(L.build_mesh(mask_grid(L, mask), 1))
    gone = full - cut
    assert cut <= full and len(gone) == 6 and all((2, 4) in e for e in gone)


def test_two_kept_columns_are_deduplicated(L):
    m = L.build_mesh(const_grid(L, 4, 10), 5)
    assert m.kept_steps.tolist() == [0, 5]
    for a in range(m.n_nodes):
        row = m.neighbors[a][m.neighbors[a] >= 0].tolist()
        assert len(set(row)) == len(row)


def test_max_edge_length_drops_long_edges_symmetrically(L):
    g = const_grid(L, 3, 8)
    r = np.array(g.ranges)
    r[1, 3] = 50.0
    g = L.ScanGrid(config=g.config, ranges=r)
    free = L.build_mesh(g, 1)
    cut = L.build_mesh(g, 1, max_edge_length=10.0)
    assert (free.neighbors[free.node_at(1, 3)] >= 0).sum() == 6
    assert (cut.neighbors[cut.node_at(1, 3)] >= 0).sum() == 0
    d = {(a, int(b)) for a in range(cut.n_nodes) for b in cut.neighbors[a] if b >= 0}
    assert all((b, a) in d for a, b in d)


def test_all_invalid_grid(L):
    m = L.build_mesh(mask_grid(L, np.zeros((4, 8), bool)), 1)
    assert m.n_nodes == 0 and m.edges().shape == (0, 2)
    assert L.estimate_normals(mask_grid(L, np.zeros((4, 8), bool)), m).n_nodes == 0


# ---------------------------------------------------------------- normals
def ref_normal(p, nbrs):
    """Independent restatement of the estimator (weighted circular fan)."""
    v = [np.asarray(q, float) - p for q in nbrs]
    if len(v) < 2:
        return None
    pairs = [(0, 1)] if len(v) == 2 else [(i, (i + 1) % len(v)) for i in range(len(v))]
    acc, ws = np.zeros(3), 0.0
    for a, b in pairs:
        w = 1.0 / (np.linalg.norm(v[a]) + np.linalg.norm(v[b]))
        acc += w * np.cross(v[a], v[b])
        ws += w
    mean = acc / ws
    if np.linalg.norm(mean) < 1e-12:
        return None
    n = mean / np.linalg.norm(mean)
    return -n if n @ p > 0 else n


def test_normals_match_independent_formula(L):
    rng = np.random.default_rng(5)
    cfg = sensor(L, 7, 18)
    r = 5.0 + rng.uniform(-0.5, 0.5, (7, 18))
    r[rng.random((7, 18)) > 0.85] = np.nan
    g = L.ScanGrid(config=cfg, ranges=r)
    m = L.build_mesh(g, 1)
    nm = L.estimate_normals(g, m)
    pos = L.node_positions(g, m)
    checked = 0
    for a in range(m.n_nodes):
        want = ref_normal(pos[a], [pos[q] for q in m.neighbors[a] if q >= 0])
        if want is None:
            assert not nm.mask[a]
        else:
            assert nm.mask[a]
            np.testing.assert_allclose(nm.values[a], want, atol=1e-9)
            checked += 1
    assert checked > 50


def test_normals_unit_and_facing_sensor(L):
    rng = np.random.default_rng(9)
    cfg = sensor(L, 8, 24)
    r = 5.0 + rng.uniform(-0.5, 0.5, (8, 24))
    r[rng.random((8, 24)) > 0.9] = np.nan
    g = L.ScanGrid(config=cfg, ranges=r)
    m = L.build_mesh(g, 1)
    nm = L.estimate_normals(g, m)
    ok = nm.mask
    np.testing.assert_allclose(np.linalg.norm(nm.values[ok], axis=1), 1.0, atol=1e-6)
    assert np.all(np.einsum("ij,ij->i", nm.values[ok], L.node_positions(g, m)[ok]) <= 1e-12)


def test_two_cell_islands_have_no_normal(L):
    mask = np.zeros((4, 8), bool)
    mask[1, 2] = mask[1, 3] = True
    g = mask_grid(L, mask)
    m = L.build_mesh(g, 1)
    assert m.n_nodes == 2 and not L.estimate_normals(g, m).mask.any()


def test_scale_invariance(L):
    rng = np.random.default_rng(3)
    cfg = sensor(L, 6, 20, r_max=1000.0)
    r = 5.0 + rng.uniform(-0.5, 0.5, (6, 20))
    a = L.ScanGrid(config=cfg, ranges=r)
    b = L.ScanGrid(config=cfg, ranges=r * 7.5)
    na = L.estimate_normals(a, L.build_mesh(a, 1))
    nb = L.estimate_normals(b, L.build_mesh(b, 1))
    np.testing.assert_array_equal(na.mask, nb.mask)
    np.testing.assert_allclose(na.values[na.mask], nb.values[nb.mask], atol=1e-6)


def test_ground_plane_normals_point_up(L):
    # analytic ranges of the plane z = -1 below the sensor
    cfg = sensor(L, 16, 90, top=-5.0, bottom=-40.0)
    r = 1.0 / np.sin(-cfg.ring_elevations)[:, None] * np.ones((16, 90))
    g = L.ScanGrid(config=cfg, ranges=r)
    nm = L.estimate_normals(g, L.build_mesh(g, 1))
    up = nm.values[nm.mask] @ np.array([0.0, 0.0, 1.0])
    assert np.mean(np.degrees(np.arccos(np.clip(up, -1, 1))) < 2.0) >= 0.99


# ---------------------------------------------------------------- segmentation
def normal_map(L, vals, absent=()):
    vals = np.asarray(vals, float).copy()
    vals /= np.linalg.norm(vals, axis=1, keepdims=True)
    mask = np.ones(len(vals), bool)
    for a in absent:
        mask[a] = False
        vals[a] = np.nan
    return L.NormalMap(values=vals, mask=mask)


def test_uniform_normals_one_segment(L):
    g = mask_grid(L, np.ones((4, 8), bool))
    m = L.build_mesh(g, 1)
    d = L.segment(m, normal_map(L, np.tile([0.0, 0.0, 1.0], (m.n_nodes, 1))), L.SegmenterConfig())
    assert np.all(d[m.node_rings, m.node_steps] == 1)


def test_threshold_is_strict_and_componentwise(L):
    g = mask_grid(L, np.ones((2, 4), bool))
    m = L.build_mesh(g, 1)
    v = np.tile([0.0, 0.0, 1.0], (m.n_nodes, 1))
    v[m.node_steps >= 2] = [0.2, 0.0, 1.0]  # |di| == 0.2 exactly: must not join
    nm = L.NormalMap(values=v, mask=np.ones(m.n_nodes, bool))
    lab = L.segment(m, nm, L.SegmenterConfig(threshold_i=0.2))[m.node_rings, m.node_steps]
    assert len(np.unique(lab)) == 2
    v[m.node_steps >= 2] = [0.1, 0.1, 1.1]  # strictly inside on every component
    nm = L.NormalMap(values=v, mask=np.ones(m.n_nodes, bool))
    assert len(np.unique(L.segment(m, nm, L.SegmenterConfig())[m.node_rings, m.node_steps])) == 1


def test_labels_first_touch_and_absent_zero(L):
    rng = np.random.default_rng(1)
    cfg = sensor(L, 6, 12)
    r = 5.0 + rng.uniform(-0.5, 0.5, (6, 12))
    r[rng.random((6, 12)) > 0.8] = np.nan
    g = L.ScanGrid(config=cfg, ranges=r)
    m = L.build_mesh(g, 1)
    vals = rng.normal(size=(m.n_nodes, 3))
    absent = np.nonzero(rng.random(m.n_nodes) < 0.2)[0]
    nm = normal_map(L, vals, absent)
    lab = L.segment(m, nm, L.SegmenterConfig(0.5, 0.5, 0.5))[m.node_rings, m.node_steps]
    assert np.all((lab == 0) == ~nm.mask)
    present = lab[lab > 0]
    u = np.unique(present)
    assert u.tolist() == list(range(1, u.size + 1))
    firsts = [int(np.argmax(lab == v)) for v in u]
    assert firsts == sorted(firsts)


def test_more_permissive_thresholds_never_add_segments(L):
    rng = np.random.default_rng(3)
    g = L.ScanGrid(config=sensor(L, 8, 16), ranges=5.0 + rng.uniform(-0.5, 0.5, (8, 16)))
    m = L.build_mesh(g, 1)
    nm = normal_map(L, rng.normal(size=(m.n_nodes, 3)))
    counts = [L.segment(m, nm, L.SegmenterConfig(t, t, t))[m.node_rings, m.node_steps].max()
              for t in (0.1, 0.3, 0.6, 1.0, 2.0)]
    assert all(a >= b for a, b in zip(counts, counts[1:]))


def test_backfill_rules(L):
    g = L.ScanGrid(config=sensor(L, 2, 10), ranges=np.full((2, 10), 5.0))
    lab = np.zeros((2, 10), np.int32)
    lab[0, 0], lab[0, 5] = 1, 2
    out = L.backfill(g, lab)
    assert out[0, 3] == 2 and out[0, 2] == 1 and out[0, 9] == 1  # nearest, wrap
    assert np.all(out[1] == 0)  # a ring without donors stays 0
    lab = np.zeros((2, 10), np.int32)
    lab[0, 0], lab[0, 4] = 1, 2
    assert L.backfill(g, lab)[0, 2] == 1  # tie -> smaller step
    lab = np.zeros((2, 10), np.int32)
    lab[0, 2], lab[0, 8] = 7, 9
    assert L.backfill(g, lab)[0, 0] == 7  # tie across the wrap -> smaller actual step (2, not 8)
    r = np.full((2, 6), 5.0)
    r[0, 1] = r[0, 4] = np.nan
    g2 = L.ScanGrid(config=sensor(L, 2, 6), ranges=r)
    lab = np.zeros((2, 6), np.int32)
    lab[0, 0] = 3
    out = L.backfill(g2, lab)
    assert out[0, 1] == 0 and out[0, 4] == 0 and out[0, 2] == 3 and out[0, 5] == 3


def test_prune_rules(L):
    lab = np.zeros((2, 30), np.int32)
    lab[:, :25] = 1
    lab[0, 25:28] = 2
    out = L.prune_small(lab, 10)
    assert np.all(out[0, 25:28] == 1) and set(np.unique(out)) == {0, 1}
    assert np.all(L.prune_small(np.array([[1, 1, 2], [3, 2, 2]], np.int32), 10) == 0)
    lab = np.zeros((2, 12), np.int32)
    lab[0, :3] = 1
    lab[1, :] = 2
    out = L.prune_small(lab, 5)
    assert np.all(out[0] == 0) and np.all(out[1] == 1)  # no donor -> 0; compaction 2 -> 1
    lab = np.zeros((1, 40), np.int32)
    lab[0, :10], lab[0, 10:12], lab[0, 12:25], lab[0, 25:40] = 1, 2, 3, 4
    out = L.prune_small(lab, 5)
    assert out[0, 0] == 1 and out[0, 13] == 2 and out[0, 30] == 3
    np.testing.assert_array_equal(L.prune_small(lab, 0), lab)


# ---------------------------------------------------------------- streaming builder (F2)
@pytest.mark.parametrize("k", [1, 3])
def test_streaming_builder_equals_batch(L, k):
    rng = np.random.default_rng(42)
    g = mask_grid(L, rng.random((6, 12)) < 0.8)
    batch = L.build_mesh(g, k)
    b = L.MeshBuilder(g.config, k)
    for step in L.subsample_steps(g.config, k):
        b.add_column(np.asarray(g.ranges)[:, step])
    m = b.finish()
    np.testing.assert_array_equal(batch.neighbors, m.neighbors)
    np.testing.assert_array_equal(batch.node_ids, m.node_ids)


def test_streaming_builder_contract(L):
    g = const_grid(L)
    b = L.MeshBuilder(g.config, 1)
    b.add_column(np.full(4, 5.0))
    with pytest.raises(ValueError):
        b.finish()
    with pytest.raises(ValueError):
        b.add_column(np.full(3, 5.0))
