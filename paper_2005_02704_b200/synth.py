"""Seeded synthetic spinning-Lidar scans with BASELINE.json's shapes.

Input generation is not the hot path (SURVEY.md §2 marks the reference
simulator out of scope); this is a vectorised torch ray-caster so that the
benchmark batches (512 HDL-64 frames, 64 x 1M-point stress frames) can be
produced on the device in seconds.  Primitive semantics follow the reference
simulator's analytic intersections (reference simulate.py:59-341): first hit
along the ray from the sensor origin, additive N(0, sigma) range noise along
the ray (simulate.py:414-417), then an i.i.d. dropout mask (new, BASELINE.json).

Output per frame: float32 xyz (P, 3) and int32 ring (P,) in ring-major firing
order (ring 0 = top beam, then azimuth step), dropped / missed returns removed.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch


@dataclass(frozen=True)
class ScanShape:
    """Sensor geometry + scene recipe of one BASELINE.json config."""

    name: str
    elevations_deg: tuple            # ring 0 = top, strictly decreasing
    steps: int
    r_max: float
    noise_sigma: float
    dropout: float
    r_min: float = 0.5
    boxes: int = 4
    box_side: tuple = (0.5, 4.0)
    box_centre: tuple = (5.0, 25.0)
    cylinders: int = 2
    cyl_radius: tuple = (0.2, 0.6)
    ramps: int = 0
    wall_x: float | None = None      # infinite wall x = wall_x
    wall_ring: float | None = None   # vertical cylinder around the sensor
    overhead: bool = False           # 10 x 10 m plane patch at z = +4
    frames: int = 1
    pose_step: tuple = (0.0, 0.0)    # (+x metres, yaw degrees) per frame
    extra: dict = field(default_factory=dict)

    @property
    def rings(self) -> int:
        return len(self.elevations_deg)

    @property
    def elevations(self) -> np.ndarray:
        return np.radians(np.asarray(self.elevations_deg, dtype=np.float64))


def _lin(a, b, n):
    return tuple(float(v) for v in np.linspace(a, b, n))


CONFIGS = {
    # configs[0]: VLP-16, CPU-runnable oracle case
    "vlp16": ScanShape("vlp16", tuple(float(v) for v in range(15, -16, -2)), 1800, 100.0, 0.01, 0.03,
                       boxes=4, cylinders=2, wall_x=30.0),
    # configs[1]: HDL-64E single scan
    "hdl64": ScanShape("hdl64", _lin(2.0, -24.9, 64), 2048, 120.0, 0.02, 0.05,
                       boxes=20, cylinders=10, ramps=2, wall_ring=40.0),
    # configs[2]: OS1-128
    "os128": ScanShape("os128", _lin(22.5, -22.5, 128), 2048, 120.0, 0.02, 0.05,
                       boxes=40, cylinders=20, ramps=4, wall_ring=40.0, overhead=True),
    # configs[3]: 512 HDL-64 frames, +1 m x and +0.5 deg yaw per frame
    "hdl64_batch": ScanShape("hdl64_batch", _lin(2.0, -24.9, 64), 2048, 120.0, 0.02, 0.05,
                             boxes=20, cylinders=10, ramps=2, wall_ring=40.0, frames=512,
                             pose_step=(1.0, 0.5)),
    # configs[4]: stress, 64 x (256 x 4096); the enclosing wall ring (as in
    # the HDL / OS configs) gives the upper beams a return, so ~0.8 of the
    # 1.05 M beams survive the 20 % dropout (~0.84 M points per frame)
    "stress": ScanShape("stress", _lin(30.0, -30.0, 256), 4096, 120.0, 0.05, 0.20,
                        boxes=200, box_side=(0.1, 1.0), box_centre=(3.0, 25.0),
                        cylinders=50, wall_ring=40.0, frames=64),
}


def make_scene(shape: ScanShape, seed: int) -> dict:
    """Seeded primitive parameters (numpy default_rng, like the reference)."""
    rng = np.random.default_rng(seed)
    sc: dict = {}
    n = shape.boxes
    side = rng.uniform(*shape.box_side, size=(n, 3))
    dist = rng.uniform(*shape.box_centre, size=n)
    ang = rng.uniform(0.0, 2.0 * np.pi, size=n)
    cz = -1.8 + side[:, 2] / 2.0 + rng.uniform(0.0, 0.5, size=n)
    centre = np.stack([dist * np.cos(ang), dist * np.sin(ang), cz], axis=1)
    sc["box_lo"] = centre - side / 2.0
    sc["box_hi"] = centre + side / 2.0
    m = shape.cylinders
    cr = rng.uniform(*shape.cyl_radius, size=m)
    cd = rng.uniform(*shape.box_centre, size=m)
    ca = rng.uniform(0.0, 2.0 * np.pi, size=m)
    sc["cyl"] = np.stack([cd * np.cos(ca), cd * np.sin(ca), cr, np.full(m, -1.8),
                          -1.8 + rng.uniform(1.0, 4.0, size=m)], axis=1)
    ramps = []
    for _ in range(shape.ramps):
        slope = np.radians(rng.uniform(5.0, 15.0))
        yaw = rng.uniform(0.0, 2.0 * np.pi)
        d = rng.uniform(8.0, 25.0)
        c = np.array([d * np.cos(yaw), d * np.sin(yaw), -1.8 + 0.5 * np.tan(slope) * 3.0])
        u = np.array([np.cos(yaw) * np.cos(slope), np.sin(yaw) * np.cos(slope), np.sin(slope)])
        v = np.array([-np.sin(yaw), np.cos(yaw), 0.0])
        ramps.append(np.concatenate([c, u, v, [3.0, 2.0]]))  # half-extents along u, v
    if shape.overhead:
        ramps.append(np.array([8.0, 0.0, 4.0, 1, 0, 0, 0, 1, 0, 5.0, 5.0], dtype=np.float64))
    sc["patch"] = np.array(ramps, dtype=np.float64).reshape(-1, 11)
    return sc


def _hit_boxes(o, d, lo, hi, best):
    if lo.shape[0] == 0:
        return best
    inv = 1.0 / torch.where(d.abs() < 1e-12, torch.full_like(d, 1e-12), d)
    for b in range(lo.shape[0]):
        t1 = (lo[b] - o) * inv
        t2 = (hi[b] - o) * inv
        tmin = torch.minimum(t1, t2).amax(dim=1)
        tmax = torch.maximum(t1, t2).amin(dim=1)
        t = torch.where(tmin > 1e-6, tmin, tmax)
        ok = (tmax >= tmin) & (t > 1e-6)
        best = torch.where(ok & (t < best), t, best)
    return best


def _hit_cylinders(o, d, cyl, best, inside=False):
    for c in range(cyl.shape[0]):
        cx, cy, r, z0, z1 = (cyl[c, j] for j in range(5))
        ox, oy = o[:, 0] - cx, o[:, 1] - cy
        a = d[:, 0] ** 2 + d[:, 1] ** 2
        bq = 2.0 * (ox * d[:, 0] + oy * d[:, 1])
        cq = ox * ox + oy * oy - r * r
        disc = bq * bq - 4.0 * a * cq
        sq = torch.sqrt(disc.clamp_min(0.0))
        a2 = (2.0 * a).clamp_min(1e-30)
        t = (-bq + sq) / a2 if inside else (-bq - sq) / a2
        z = o[:, 2] + t * d[:, 2]
        ok = (disc >= 0) & (t > 1e-6) & (z >= z0) & (z <= z1)
        best = torch.where(ok & (t < best), t, best)
    return best


def _hit_patches(o, d, patch, best):
    for p in range(patch.shape[0]):
        c, u, v, hu, hv = patch[p, 0:3], patch[p, 3:6], patch[p, 6:9], patch[p, 9], patch[p, 10]
        nrm = torch.linalg.cross(u, v)
        den = d @ nrm
        t = ((c - o) @ nrm) / torch.where(den.abs() < 1e-12, torch.full_like(den, 1e-12), den)
        q = o + t[:, None] * d - c
        ok = (t > 1e-6) & ((q @ u).abs() <= hu) & ((q @ v).abs() <= hv)
        best = torch.where(ok & (t < best), t, best)
    return best


def cast_frame(shape: ScanShape, scene: dict, frame: int, seed: int, device="cpu"):
    """Ray-cast one frame; returns float32 xyz (P,3) and int32 ring (P,) tensors."""
    dev = torch.device(device)
    f64 = dict(dtype=torch.float64, device=dev)
    R, S = shape.rings, shape.steps
    theta = torch.tensor(shape.elevations, **f64)
    phi = 2.0 * math.pi * torch.arange(S, **f64) / S
    ct, st = torch.cos(theta)[:, None], torch.sin(theta)[:, None]
    ds = torch.stack([(ct * torch.cos(phi)[None]).expand(R, S),
                      (ct * torch.sin(phi)[None]).expand(R, S),
                      st.expand(R, S)], dim=-1).reshape(-1, 3)
    # the object field repeats every 60 m along the sensor path so that every
    # frame of a long batch still sees the scene (consecutive frames overlap)
    tx, yaw_deg = (shape.pose_step[0] * frame) % 60.0, shape.pose_step[1] * frame
    yaw = math.radians(yaw_deg)
    rz = torch.tensor([[math.cos(yaw), -math.sin(yaw), 0.0],
                       [math.sin(yaw), math.cos(yaw), 0.0], [0.0, 0.0, 1.0]], **f64)
    d = ds @ rz.T
    o = torch.tensor([tx, 0.0, 0.0], **f64).expand_as(d)
    best = torch.full((R * S,), float("inf"), **f64)
    # ground plane z = -1.8 (reference Plane, simulate.py:59-98)
    tg = (-1.8 - o[:, 2]) / torch.where(d[:, 2] < -1e-12, d[:, 2], torch.full_like(d[:, 2], -1e-12))
    best = torch.where((d[:, 2] < -1e-12) & (tg > 0) & (tg < best), tg, best)
    if shape.wall_x is not None:
        tw = (shape.wall_x - o[:, 0]) / torch.where(d[:, 0] > 1e-12, d[:, 0], torch.full_like(d[:, 0], 1e-12))
        best = torch.where((d[:, 0] > 1e-12) & (tw > 0) & (tw < best), tw, best)
    t = lambda a: torch.as_tensor(a, **f64)
    best = _hit_boxes(o, d, t(scene["box_lo"]), t(scene["box_hi"]), best)
    best = _hit_cylinders(o, d, t(scene["cyl"]), best)
    if shape.wall_ring is not None:
        ring_cyl = torch.tensor([[tx, 0.0, shape.wall_ring, -50.0, 50.0]], **f64)
        best = _hit_cylinders(o, d, ring_cyl, best, inside=True)
    best = _hit_patches(o, d, t(scene["patch"]), best)
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed) * 1_000_003 + frame)
    noise = torch.randn(R * S, generator=gen, **f64) * shape.noise_sigma
    keep = torch.rand(R * S, generator=gen, **f64) >= shape.dropout
    r = best + noise
    keep &= torch.isfinite(best) & (best <= shape.r_max) & (r > 0)
    xyz = (ds * r[:, None])[keep].to(torch.float32)
    ring = torch.arange(R, device=dev, dtype=torch.int32).repeat_interleave(S)[keep]
    return xyz.contiguous(), ring.contiguous()


def make_batch(shape: ScanShape | str, frames: int | None = None, seed: int = 0, device="cpu",
               scene_seed: int | None = None, first_frame: int = 0):
    """Frames [first_frame, first_frame + frames) of one config: returns
    xyz (P,3) f32, ring (P,) i32, offsets (F+1,) i64."""
    if isinstance(shape, str):
        shape = CONFIGS[shape]
    frames = shape.frames if frames is None else int(frames)
    scene = make_scene(shape, seed if scene_seed is None else scene_seed)
    xs, rs, offs = [], [], [0]
    for f in range(first_frame, first_frame + frames):
        x, r = cast_frame(shape, scene, f, seed, device)
        xs.append(x)
        rs.append(r)
        offs.append(offs[-1] + x.shape[0])
    off = torch.tensor(offs, dtype=torch.int64, device=device)
    return torch.cat(xs), torch.cat(rs), off
