"""File formats against the reference writers: every
writer must reproduce the reference's bytes exactly (tests/golden/io0.npz,
made by make_golden_io.py), parsers must round-trip, and the native repr
formatter must equal Python's repr(float) on edge cases."""


import numpy as np
import pytest

from conftest import load_golden


@pytest.fixture(scope="module")
def g():
    return load_golden("io0")


@pytest.fixture(scope="module")
def L():
    import paper_2005_02704_b200 as L
    return L


def _grid(L, g, labels=True):
    cfg = L.SensorConfig(ring_elevations=g["elev"], azimuth_steps=int(g["steps"]), r_min=float(g["r_min"]),
                         r_max=float(g["r_max"]), noise_sigma=float(g["sigma"]))
    return L.ScanGrid(config=cfg, ranges=g["ranges"], truth_labels=g["truth"] if labels else None)


def _mesh(L, g):
    return L.Mesh(rings=int(g["elev"].size), full_steps=int(g["steps"]), interval=int(g["interval"]),
                  kept_steps=g["kept"], node_rings=g["node_rings"], node_steps=g["node_steps"], node_ids=g["node_ids"],
                  neighbors=g["neighbors"])


def _text(g, k):
    return str(g["text_" + k])


def test_repr_formatter_matches_python(L):
    rng = np.random.default_rng(3)
    v = np.concatenate([rng.normal(size=20000) * 10.0 ** rng.integers(-320, 300, size=20000),
                        [0.0, -0.0, np.nan, np.inf, -np.inf, 5e-324, 1.7976931348623157e308, 1e16, 1e15,
                         9999999999999998.0, 1e-4, 1e-5, 0.1, 2.5, 123456789.0, -1e-300]])
    got = L.io.format_rows(v[:, None], [0]).split("\n")[:-1]
    assert got == [repr(float(x)) for x in v]
    ints = np.array([[0, -7, 2 ** 40, 123456]], dtype=np.float64)
    assert L.io.format_rows(ints, [1, 1, 1, 1]) == "0 -7 1099511627776 123456\n"


def test_scan_writer_and_parser(L, g):
    grid = _grid(L, g)
    assert L.io.write_scan_text(grid) == _text(g, "scan")
    assert L.io.write_scan_text(_grid(L, g, labels=False)) == _text(g, "scan_nolabels")
    back = L.io.parse_scan_text(_text(g, "scan"))
    np.testing.assert_array_equal(np.isnan(back.ranges), np.isnan(grid.ranges))
    np.testing.assert_array_equal(back.ranges[~np.isnan(back.ranges)], grid.ranges[~np.isnan(grid.ranges)])
    np.testing.assert_array_equal(back.truth_labels, grid.truth_labels)
    np.testing.assert_array_equal(back.config.ring_elevations, np.radians(np.degrees(grid.config.ring_elevations)))
    with pytest.raises(ValueError):
        L.io.parse_scan_text("LSEGX 1 2 0.5 1.0\n")


def test_scene_and_config_round_trip(L, g):
    # the scene of make_golden_io.py, built with this package's generator
    sc = L.generate_scene(7, crowding=0.3)
    sc = L.Scene(primitives=sc.primitives + (L.Plane(point=(6.0, -4.0, -1.0), normal=(0.0, 0.3, 1.0),
                                                     surface_id=900, extent=(3.0, 2.0)),), seed=42)
    assert L.io.write_scene_text(sc) == _text(g, "scene")
    back = L.io.parse_scene_text(_text(g, "scene"))
    assert back.seed == 42 and back.surface_ids == sc.surface_ids
    for a, b in zip(back.primitives, sc.primitives):  # parse re-normalises axes: equal to ~1 ulp
        for k, v in vars(a).items():
            np.testing.assert_allclose(np.asarray(v, float), np.asarray(vars(b)[k], float), rtol=1e-15, atol=1e-16)
    cfg = L.io.parse_config_text(_text(g, "config"))
    assert L.io.write_config_text(cfg) == _text(g, "config")
    assert L.io.write_config_text(L.PipelineConfig()) == _text(g, "config_default")
    assert cfg.interval == 2 and cfg.intervals == (1, 2, 7) and cfg.eval.dilation_radius == 1
    assert cfg.segmenter.min_segment_size == 4
    with pytest.raises(ValueError):
        L.io.parse_config_text("[sensor]\n")
    with pytest.raises(ValueError):
        L.io.parse_scene_text("LSCENE1\nteapot id 3\n")


def test_labels_ply_normals_adjacency_reports(L, g):
    grid = _grid(L, g)
    assert L.io.write_labels_text(grid, g["labels"]) == _text(g, "labels")
    np.testing.assert_array_equal(L.io.parse_labels_text(_text(g, "labels")), g["labels"])
    assert L.io.write_labeled_ply(grid, g["labels"]) == _text(g, "ply")
    mesh = _mesh(L, g)
    nm = L.NormalMap(values=g["nvals"], mask=g["nmask"])
    assert L.io.write_normals_text(mesh, nm) == _text(g, "normals")
    assert L.io.write_mesh_adjacency(mesh) == _text(g, "adjacency")
    rep = L.EvalReport(precision=0.5, recall=0.25, f1=1.0 / 3.0, timings_ms={"mesh": 1.5, "total": 2.25})
    assert L.io.write_report_json("a", 1, rep) == _text(g, "report")
    rows = [L.io.report_dict("a", 1, rep), L.io.report_dict("b", 7, L.EvalReport(0.1, 0.2, 0.3))]
    assert L.io.write_summary_csv(rows) == _text(g, "summary")
    assert L.io.label_color(0) == (128, 128, 128)


def test_load_labels_from_files(L, g, tmp_path):
    p = tmp_path / "x.lsegl"
    p.write_text(_text(g, "labels"))
    np.testing.assert_array_equal(L.io.load_labels(p), g["labels"])
    s = tmp_path / "x.lseg"
    s.write_text(_text(g, "scan"))
    np.testing.assert_array_equal(L.io.load_labels(s), g["truth"])
    s2 = tmp_path / "y.lseg"
    s2.write_text(_text(g, "scan_nolabels"))
    with pytest.raises(ValueError):
        L.io.load_labels(s2)


@pytest.mark.gpu
def test_mesh_ply(L, g):
    assert L.io.write_mesh_ply(_grid(L, g), _mesh(L, g)) == _text(g, "mesh_ply")
