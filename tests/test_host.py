"""CPU-side tests: the C-ABI library loads and exports every declared symbol,
the host data model keeps the reference's ValueError contract, the synthetic
scan generator honours BASELINE.json's shapes."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lidarseg_b200.h")).read()
    return sorted(set(re.findall(r"\b(lseg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2005_02704_b200 import _build, _lib
    _build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 11
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)
    L = _lib.load()
    assert L.lseg_version().startswith(b"lidarseg_b200")
    assert _lib.kept_count(2048, 5) == 410 and _lib.kept_count(1800, 5) == 360
    assert _lib.kept_count(10, 10) == -1 and _lib.kept_count(10, 0) == -1
    assert _lib.workspace_bytes(4, 64, 2048, 1) > 4 * 64 * 2048 * 24


def test_ops_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2005_02704_b200 as L
    from paper_2005_02704_b200._lib import LidarSegError
    cfg = L.SensorConfig.uniform(rings=4, azimuth_steps=8)
    grid = L.ScanGrid(config=cfg, ranges=np.full((4, 8), 5.0))
    with pytest.raises(LidarSegError):
        L.build_mesh(grid, 1)


def test_sensor_and_grid_contract():
    import paper_2005_02704_b200 as L
    with pytest.raises(ValueError):
        L.SensorConfig(ring_elevations=[0.1])
    with pytest.raises(ValueError):
        L.SensorConfig(ring_elevations=[0.1, 0.2])
    with pytest.raises(ValueError):
        L.SensorConfig(ring_elevations=[0.2, 0.1], azimuth_steps=2)
    with pytest.raises(ValueError):
        L.SensorConfig(ring_elevations=[0.2, 0.1], r_min=5, r_max=1)
    cfg = L.SensorConfig.uniform(rings=4, azimuth_steps=8)
    with pytest.raises(ValueError):
        L.ScanGrid(config=cfg, ranges=np.zeros((3, 8)))
    g = L.ScanGrid(config=cfg, ranges=np.array([[5.0, np.nan, 0.1, 200.0] * 2] * 4))
    assert g.valid_mask[0].tolist() == [True, False, False, False] * 2
    assert L.subsample_steps(cfg, 3).tolist() == [0, 3, 6]
    with pytest.raises(ValueError):
        L.subsample_steps(cfg, 8)
    p = L.polar_to_cartesian(cfg, (0, 0), 5.0)
    assert p.y == 0.0 and p.x > 0
    with pytest.raises(ValueError):
        L.polar_to_cartesian(cfg, (0, 9), 5.0)
    assert L.valid_point(g, (0, 0)) and not L.valid_point(g, (0, 1))


def test_angle_tables_match_reference_expressions(oracle):
    import paper_2005_02704_b200 as L
    cfg = L.SensorConfig.uniform(rings=64, top_deg=2.0, bottom_deg=-24.9, azimuth_steps=2048)
    for a, b in zip(cfg.angle_tables(), oracle.ray_tables(cfg.ring_elevations, 2048)):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(cfg.ray_directions(), oracle.ray_directions(cfg.ring_elevations, 2048))


def test_synth_shapes():
    from paper_2005_02704_b200 import synth
    for name in ("vlp16", "hdl64"):
        s = synth.CONFIGS[name]
        xyz, ring, off = synth.make_batch(s, frames=1, seed=2)
        P = xyz.shape[0]
        assert off.tolist() == [0, P]
        assert 0.6 * s.rings * s.steps < P < s.rings * s.steps
        r = ring.numpy()
        assert np.all(np.diff(r) >= 0) and r.min() >= 0 and r.max() < s.rings  # ring-major
    assert synth.CONFIGS["hdl64_batch"].frames == 512 and synth.CONFIGS["stress"].steps == 4096
