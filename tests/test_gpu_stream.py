"""F2 streaming mesh builder (reference MeshBuilder, mesh.py:139-170) on the
GPU against the REFERENCE's own build_mesh outputs: the golden grids (VLP-16
frames at k = 1 / 5, small grids incl. S' = 2 and S mod k != 0) and the
bench-scale fixtures (HDL-64, OS1-128, stress), fed one kept column at a
time in sweep order."""

import numpy as np
import pytest

from conftest import golden_names, load_golden
from golden.packing import digest, unpack_ranges

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2005_02704_b200 as L
    return L


def _stream(L, cfg, ranges, k):
    b = L.MeshBuilder(cfg, k)
    for step in L.subsample_steps(cfg, k):
        b.add_column(ranges[:, step])
    return b.finish()


@pytest.mark.parametrize("name", golden_names("vlp16") + golden_names("small"))
def test_streaming_builder_matches_reference_golden(L, name):
    g = load_golden(name)
    cfg = L.SensorConfig(ring_elevations=g["elev"], azimuth_steps=int(g["steps"]), r_min=float(g["r_min"]),
                         r_max=float(g["r_max"]))
    m = _stream(L, cfg, g["ranges"], int(g["interval"]))
    np.testing.assert_array_equal(m.node_ids, g["node_ids"])
    np.testing.assert_array_equal(m.neighbors, g["neighbors"])
    np.testing.assert_array_equal(m.node_rings, g["node_rings"])
    np.testing.assert_array_equal(m.node_steps, g["node_steps"])
    np.testing.assert_array_equal(L.mesh_triangles(m), g["triangles"])


@pytest.mark.parametrize("name", golden_names("scale_"))
def test_streaming_builder_matches_reference_at_scale(L, name):
    g = load_golden(name)
    cfg = L.SensorConfig(ring_elevations=g["elev"], azimuth_steps=int(g["steps"]), r_min=float(g["r_min"]),
                         r_max=float(g["r_max"]))
    ranges = unpack_ranges(g)
    for k in [int(v) for v in g["intervals"]][:2]:
        m = _stream(L, cfg, ranges, k)
        assert m.n_nodes == int(g[f"k{k}_n_nodes"])
        assert digest(m.node_ids.astype(np.int32)) == str(g[f"k{k}_node_ids"])
        assert digest(m.neighbors.astype(np.int32)) == str(g[f"k{k}_neighbors"])


def test_streaming_builder_reusable_state(L):
    """Two builders interleaved (two sensors) do not share state, and a
    builder rejects extra columns."""
    g = load_golden("small3")
    cfg = L.SensorConfig(ring_elevations=g["elev"], azimuth_steps=int(g["steps"]), r_min=float(g["r_min"]),
                         r_max=float(g["r_max"]))
    k = int(g["interval"])
    a, b = L.MeshBuilder(cfg, k), L.MeshBuilder(cfg, k)
    steps = L.subsample_steps(cfg, k)
    other = np.where(np.isnan(g["ranges"]), 5.0, np.nan)
    for s in steps:
        a.add_column(g["ranges"][:, s])
        b.add_column(other[:, s])
    with pytest.raises(ValueError):
        a.add_column(g["ranges"][:, 0])
    np.testing.assert_array_equal(a.finish().neighbors, g["neighbors"])
    want_b = L.build_mesh(L.ScanGrid(config=cfg, ranges=other), k)
    np.testing.assert_array_equal(b.finish().neighbors, want_b.neighbors)
