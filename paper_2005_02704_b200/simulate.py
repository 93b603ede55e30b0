"""Scan simulator on the GPU (reference simulate.py).

Same primitives, validation and public functions as the reference
(``Plane``, ``Sphere``, ``Cylinder``, ``Box``, ``Cone``, ``Scene``,
``rotation_rpy``, ``ray_intersect``, ``cast_grid``, ``scan_scene``,
``scene_normals``); the ray casting itself runs in ``lseg_cast_grid`` /
``lseg_cast_rays`` (csrc/lseg_sim.cu), one thread per beam, and scenes are
passed to the library as packed records (``_pack``).  ``cast_grid_batch``
adds what the reference lacks: many frames with per-frame sensor poses in one
launch, results left on the device (the bench's input generator).

The range noise of ``scan_scene`` is drawn exactly as the reference draws it
(numpy ``default_rng(seed).normal`` over the row-major grid), so noisy scans
reproduce the reference's streams.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .scan import ScanGrid, SensorConfig, device_tables

_EPS = 1e-12
PRIM_STRIDE = 24  # include/lidarseg_b200.h LSEG_PRIM_STRIDE


def _unit(v) -> np.ndarray:
    v = np.asarray(v, dtype=float).reshape(3)
    n = float(np.linalg.norm(v))
    if n < _EPS:
        raise ValueError("zero-length direction vector")
    return v / n


def _as_vec3(v) -> np.ndarray:
    out = np.asarray(v, dtype=float).reshape(3)
    if not np.all(np.isfinite(out)):
        raise ValueError("vector components must be finite")
    return out


def _plane_axes(normal: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Deterministic in-plane frame of a finite plane (reference simulate.py:40-45)."""
    a = np.array([1.0, 0.0, 0.0]) if abs(normal[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    u = _unit(np.cross(normal, a))
    return u, np.cross(normal, u)


def rotation_rpy(roll: float = 0.0, pitch: float = 0.0, yaw: float = 0.0) -> np.ndarray:
    """Rz(yaw) @ Ry(pitch) @ Rx(roll) (reference simulate.py:48-56)."""
    cr, sr = np.cos(roll), np.sin(roll)
    cp, sp = np.cos(pitch), np.sin(pitch)
    cy, sy = np.cos(yaw), np.sin(yaw)
    rx = np.array([[1, 0, 0], [0, cr, -sr], [0, sr, cr]])
    ry = np.array([[cp, 0, sp], [0, 1, 0], [-sp, 0, cp]])
    rz = np.array([[cy, -sy, 0], [sy, cy, 0], [0, 0, 1]])
    return rz @ ry @ rx


@dataclass(frozen=True)
class Plane:
    """Plane through ``point`` with unit ``normal``; optionally a rectangle of
    half-sizes ``extent`` in the deterministic in-plane frame."""

    point: np.ndarray
    normal: np.ndarray
    surface_id: int
    extent: tuple[float, float] | None = None

    def __post_init__(self):
        object.__setattr__(self, "point", _as_vec3(self.point))
        object.__setattr__(self, "normal", _unit(self.normal))
        if self.extent is not None:
            hx, hy = float(self.extent[0]), float(self.extent[1])
            if hx <= 0 or hy <= 0:
                raise ValueError("plane extent half-sizes must be > 0")
            object.__setattr__(self, "extent", (hx, hy))

    @property
    def surface_ids(self) -> tuple[int, ...]:
        return (self.surface_id,)


@dataclass(frozen=True)
class Sphere:
    center: np.ndarray
    radius: float
    surface_id: int

    def __post_init__(self):
        object.__setattr__(self, "center", _as_vec3(self.center))
        if self.radius <= 0:
            raise ValueError("sphere radius must be > 0")

    @property
    def surface_ids(self) -> tuple[int, ...]:
        return (self.surface_id,)


@dataclass(frozen=True)
class Cylinder:
    """Finite cylinder from ``base`` along unit ``axis`` for ``height``;
    faces 0 side, 1 bottom cap, 2 top cap."""

    base: np.ndarray
    axis: np.ndarray
    radius: float
    height: float
    surface_ids: tuple[int, int, int]

    def __post_init__(self):
        object.__setattr__(self, "base", _as_vec3(self.base))
        object.__setattr__(self, "axis", _unit(self.axis))
        if self.radius <= 0 or self.height <= 0:
            raise ValueError("cylinder radius and height must be > 0")
        object.__setattr__(self, "surface_ids", tuple(int(i) for i in self.surface_ids))
        if len(self.surface_ids) != 3:
            raise ValueError("cylinder needs 3 surface ids (side, bottom, top)")


@dataclass(frozen=True)
class Box:
    """Oriented box (``rotation`` maps box frame to world); faces 0..5 are
    (+x, -x, +y, -y, +z, -z) in the box frame."""

    center: np.ndarray
    half_extents: np.ndarray
    surface_ids: tuple[int, ...]
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))

    def __post_init__(self):
        object.__setattr__(self, "center", _as_vec3(self.center))
        he = _as_vec3(self.half_extents)
        if np.any(he <= 0):
            raise ValueError("box half extents must be > 0")
        object.__setattr__(self, "half_extents", he)
        rot = np.asarray(self.rotation, dtype=float).reshape(3, 3)
        if not np.allclose(rot @ rot.T, np.eye(3), atol=1e-9):
            raise ValueError("box rotation must be orthonormal")
        object.__setattr__(self, "rotation", rot)
        object.__setattr__(self, "surface_ids", tuple(int(i) for i in self.surface_ids))
        if len(self.surface_ids) != 6:
            raise ValueError("box needs 6 surface ids")


@dataclass(frozen=True)
class Cone:
    """Finite cone: ``apex``, unit ``axis`` toward the base, half-angle in
    (0, pi/2), base cap at ``height``; faces 0 lateral, 1 base."""

    apex: np.ndarray
    axis: np.ndarray
    half_angle: float
    height: float
    surface_ids: tuple[int, int]

    def __post_init__(self):
        object.__setattr__(self, "apex", _as_vec3(self.apex))
        object.__setattr__(self, "axis", _unit(self.axis))
        if not (0.0 < self.half_angle < np.pi / 2):
            raise ValueError("cone half_angle must be in (0, pi/2)")
        if self.height <= 0:
            raise ValueError("cone height must be > 0")
        object.__setattr__(self, "surface_ids", tuple(int(i) for i in self.surface_ids))
        if len(self.surface_ids) != 2:
            raise ValueError("cone needs 2 surface ids (lateral, base)")


Primitive = Plane | Sphere | Cylinder | Box | Cone


@dataclass(frozen=True)
class Scene:
    """Ordered primitives plus the seed of the scan noise stream."""

    primitives: tuple
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "primitives", tuple(self.primitives))
        ids = [i for p in self.primitives for i in p.surface_ids]
        if any(i <= 0 for i in ids):
            raise ValueError("surface ids must be positive")
        if len(set(ids)) != len(ids):
            raise ValueError("surface ids must be unique scene-wide")

    @property
    def surface_ids(self) -> tuple[int, ...]:
        return tuple(i for p in self.primitives for i in p.surface_ids)


def _record(prim) -> np.ndarray:
    r = np.zeros(PRIM_STRIDE)
    ids = list(prim.surface_ids)
    r[1:1 + len(ids)] = ids
    if isinstance(prim, Plane):
        r[0] = 0
        r[7:10], r[10:13] = prim.point, prim.normal
        if prim.extent is not None:
            u, v = _plane_axes(prim.normal)
            r[13], r[14], r[15] = 1.0, prim.extent[0], prim.extent[1]
            r[16:19], r[19:22] = u, v
    elif isinstance(prim, Sphere):
        r[0] = 1
        r[7:10], r[10] = prim.center, prim.radius
    elif isinstance(prim, Cylinder):
        r[0] = 2
        r[7:10], r[10:13], r[13], r[14] = prim.base, prim.axis, prim.radius, prim.height
    elif isinstance(prim, Box):
        r[0] = 3
        r[7:10], r[10:13], r[13:22] = prim.center, prim.half_extents, prim.rotation.reshape(-1)
    elif isinstance(prim, Cone):
        r[0] = 4
        r[7:10], r[10:13] = prim.apex, prim.axis
        r[13] = np.cos(prim.half_angle) ** 2  # simulate.py:315
        r[14] = prim.height
        r[15] = prim.height * np.tan(prim.half_angle)  # :344
        r[16], r[17] = np.cos(prim.half_angle), np.sin(prim.half_angle)  # :360
    else:
        raise ValueError(f"unknown primitive {type(prim).__name__}")
    return r


def _pack(scene_or_prims, device) -> torch.Tensor:
    prims = scene_or_prims.primitives if isinstance(scene_or_prims, Scene) else tuple(scene_or_prims)
    arr = np.stack([_record(p) for p in prims]) if prims else np.zeros((1, PRIM_STRIDE))
    return torch.from_numpy(arr).to(device), len(prims)


def ray_intersect(prim, origin, direction) -> tuple[float, int] | None:
    """Smallest t > 0 where origin + t*direction hits ``prim`` and the id of
    the face hit, or None (reference simulate.py:364-380)."""
    origin = _as_vec3(origin)
    direction = np.asarray(direction, dtype=float).reshape(3)
    if abs(float(np.linalg.norm(direction)) - 1.0) > 1e-9:
        raise ValueError("ray direction must be unit length")
    t, ids = cast_rays([prim], origin[None, :], direction[None, :])
    if not np.isfinite(t[0]):
        return None
    return float(t[0]), int(ids[0])


def cast_rays(prims, origins, dirs, device=None):
    """Nearest hit of each ray among ``prims`` (first primitive wins ties)."""
    dev = torch.device(device or "cuda")
    L = _lib.lib()
    rec, n = _pack(prims, dev)
    o = torch.from_numpy(np.ascontiguousarray(origins, dtype=np.float64)).to(dev)
    d = torch.from_numpy(np.ascontiguousarray(dirs, dtype=np.float64)).to(dev)
    m = int(o.shape[0])
    t = torch.empty(m, dtype=torch.float64, device=dev)
    ids = torch.empty(m, dtype=torch.int32, device=dev)
    _lib.check(L.lseg_cast_rays(_lib.ptr(rec), n, m, _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), _lib.ptr(ids),
                                _lib.stream_ptr()))
    return t.cpu().numpy(), ids.cpu().numpy()


def cast_grid_batch(scene: Scene, config: SensorConfig, poses=None, frames: int = 1, device=None):
    """Device-resident noiseless cast of ``frames`` scans: (t, ids) tensors of
    shape (frames, rings, steps).  ``poses`` (frames, 12): beam rotation
    (row-major 3x3) and sensor origin per frame, or None (origin-centred)."""
    dev = torch.device(device or "cuda")
    L = _lib.lib()
    _, sn = device_tables(config, dev)
    rec, n = _pack(scene, dev)
    P = None
    if poses is not None:
        P = torch.as_tensor(np.asarray(poses, dtype=np.float64) if not torch.is_tensor(poses) else poses,
                            dtype=torch.float64).to(dev).contiguous()
        frames = int(P.shape[0])
    t = torch.empty((frames, config.rings, config.azimuth_steps), dtype=torch.float64, device=dev)
    ids = torch.empty((frames, config.rings, config.azimuth_steps), dtype=torch.int32, device=dev)
    _lib.check(L.lseg_cast_grid(sn, frames, _lib.ptr(rec), n, _lib.ptr(P), _lib.ptr(t), _lib.ptr(ids),
                                _lib.stream_ptr()))
    return t, ids


def cast_grid(scene: Scene, config: SensorConfig) -> tuple[np.ndarray, np.ndarray]:
    """Noiseless cast of every beam: (true ranges, surface ids); +inf / 0 where
    nothing is hit, no range window (reference simulate.py:383-401)."""
    t, ids = cast_grid_batch(scene, config)
    return t[0].cpu().numpy(), ids[0].cpu().numpy()


def apply_scan(t: torch.Tensor, ids: torch.Tensor, config: SensorConfig, noise: torch.Tensor | None = None):
    """Noise + range window on device tensors: (ranges with NaN, labels)."""
    L = _lib.lib()
    ranges = torch.empty_like(t)
    labels = torch.empty_like(ids)
    _lib.check(L.lseg_apply_scan(int(t.numel()), float(config.r_min), float(config.r_max), _lib.ptr(t),
                                 _lib.ptr(ids), _lib.ptr(noise), _lib.ptr(ranges), _lib.ptr(labels),
                                 _lib.stream_ptr()))
    return ranges, labels


def scan_scene(scene: Scene, config: SensorConfig, seed: int | None = None) -> ScanGrid:
    """One revolution: nearest hit per beam + Gaussian range noise drawn from
    ``default_rng(seed or scene.seed)`` over the row-major grid; returns that
    leave [r_min, r_max] become INVALID and lose their label (reference
    simulate.py:404-421)."""
    t, ids = cast_grid_batch(scene, config)
    noise = None
    if config.noise_sigma > 0.0:
        rng = np.random.default_rng(scene.seed if seed is None else seed)
        nz = rng.normal(0.0, config.noise_sigma, size=(config.rings, config.azimuth_steps))
        noise = torch.from_numpy(nz).to(t.device)
    ranges, labels = apply_scan(t, ids, config, noise)
    return ScanGrid(config=config, ranges=ranges[0].cpu().numpy(), truth_labels=labels[0].cpu().numpy())


def scene_normals(scene: Scene, grid: ScanGrid) -> np.ndarray:
    """Analytic surface normal per labelled cell, oriented toward the sensor;
    NaN rows for label 0; shape (rings, steps, 3) (reference simulate.py:424-448)."""
    if grid.truth_labels is None:
        raise ValueError("grid has no truth labels")
    dev = torch.device("cuda")
    L = _lib.lib()
    _, sn = device_tables(grid.config, dev)
    rec, n = _pack(scene, dev)
    r = grid.device_ranges(dev)
    lab = torch.from_numpy(np.array(grid.truth_labels, dtype=np.int32)).to(dev)
    out = torch.empty((grid.rings, grid.steps, 3), dtype=torch.float64, device=dev)
    _lib.check(L.lseg_scene_normals(sn, _lib.ptr(rec), n, _lib.ptr(r), _lib.ptr(lab), _lib.ptr(out),
                                    _lib.stream_ptr()))
    return out.cpu().numpy()
