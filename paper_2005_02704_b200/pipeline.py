"""End-to-end hot path, mirroring reference pkg/src/lidarseg/pipeline.py.

* ``run_pipeline(scan, cfg, interval=None)`` — the reference's single-scan
  entry point (pipeline.py:47-70): one upload, one fused C-ABI call
  (lseg_run_scans), one download; stage timings from CUDA events.
* ``bin_points(xyz, ring, config)`` — the new binning op.
* ``BatchPipeline`` — the batched, device-resident form of the whole path
  (points -> labels for F frames in one C-ABI call, lseg_run_pipeline); this
  is what the benchmark measures.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .mesh import Mesh
from .normals import NormalMap
from .scan import ScanGrid, SensorConfig, device_tables, subsample_steps
from .evaluate import EvalConfig
from .segment import SegmenterConfig


@dataclass(frozen=True)
class BaselineConfig:
    """Parameters of the reference's region-growing comparison baseline
    (reference baseline.py:21-35).  Only the configuration is mirrored (it is
    part of the LSEGCFG1 format); the baseline algorithm itself is off the
    hot path and not built."""

    k_neighbors: int = 30
    angle_threshold: float = float(np.radians(3.0))
    curvature_threshold: float = 0.05
    min_cluster_size: int = 50

    def __post_init__(self):
        if self.k_neighbors < 3:
            raise ValueError("k_neighbors must be >= 3")
        if not (0.0 < self.angle_threshold < np.pi / 2):
            raise ValueError("angle_threshold must be in (0, pi/2) radians")
        if self.min_cluster_size < 0:
            raise ValueError("min_cluster_size must be >= 0")


@dataclass(frozen=True)
class PipelineConfig:
    sensor: SensorConfig = field(default_factory=SensorConfig.default)
    interval: int = 5
    intervals: tuple = (5, 10, 15)
    segmenter: SegmenterConfig = field(default_factory=SegmenterConfig)
    eval: EvalConfig = field(default_factory=EvalConfig)
    baseline: BaselineConfig = field(default_factory=BaselineConfig)

    def __post_init__(self):
        if self.interval < 1:
            raise ValueError("interval must be >= 1")
        if not self.intervals or any(i < 1 for i in self.intervals):
            raise ValueError("intervals must be positive")
        object.__setattr__(self, "intervals", tuple(int(i) for i in self.intervals))


@dataclass(frozen=True)
class PipelineResult:
    labels: np.ndarray
    normals: NormalMap
    mesh: Mesh
    timings_ms: dict


def bin_points(xyz, ring, config: SensorConfig) -> ScanGrid:
    """Scatter f32 points (P,3) + ring ids (P,) into a ScanGrid (GPU, lseg_bin_points)."""
    L = _lib.lib()
    dev = torch.device("cuda")
    x = torch.as_tensor(np.ascontiguousarray(xyz, dtype=np.float32)).reshape(-1, 3).to(dev)
    r = torch.as_tensor(np.ascontiguousarray(ring, dtype=np.int32)).reshape(-1).to(dev)
    if x.shape[0] != r.shape[0]:
        raise ValueError("xyz and ring lengths differ")
    _, sn = device_tables(config, dev)
    off = torch.tensor([0, x.shape[0]], dtype=torch.int64, device=dev)
    ranges = torch.empty((1, config.rings, config.azimuth_steps), dtype=torch.float64, device=dev)
    _lib.check(L.lseg_bin_points(sn, 1, _lib.ptr(x), _lib.ptr(r), _lib.ptr(off), x.shape[0], _lib.ptr(ranges),
                                 None, _lib.stream_ptr()))
    out = ranges[0].cpu().numpy()
    out[np.isnan(out)] = np.nan  # canonical NaN
    return ScanGrid(config=config, ranges=out)


_STAGE_OF = {"valid_bits": "mesh", "frame_scan": "mesh", "tile": "normals", "tile_cc": "segment",
             "merge": "segment", "labels_backfill": "backfill", "prune_apply": "backfill"}


def run_pipeline(scan: ScanGrid, cfg: PipelineConfig, interval: int | None = None) -> PipelineResult:
    """GPU run_pipeline (reference pipeline.py:47-70): ONE upload of the range
    grid, ONE fused C-ABI call (lseg_run_scans: valid bits -> mesh + fp64
    normals + pass masks -> components -> backfill -> prune, no host sync in
    between), ONE download of mesh, normals and labels.  The reference's
    stage timings come from the library's per-kernel CUDA events: mesh = node
    numbering, normals = the tile kernel (which also emits the mesh slots),
    segment = tile components + border merge, backfill = labels + backfill +
    pruning."""
    interval = cfg.interval if interval is None else int(interval)
    kept = subsample_steps(scan.config, interval)  # ValueError contract
    L = _lib.lib()
    conf = scan.config
    R, S, Sk = conf.rings, conf.azimuth_steps, kept.size
    cap = R * Sk
    dev = torch.device("cuda")
    _, sn = device_tables(conf, dev)
    seg = cfg.segmenter
    key = (torch.cuda.current_device(), R, S, interval)
    cache = _SCAN_BUFS.__dict__.setdefault("bufs", {})  # per thread: concurrent callers never share buffers
    bufs = cache.get(key)
    if bufs is None:
        wsb = _lib.workspace_bytes(1, R, S, interval)
        bufs = {"ws": torch.empty(wsb, dtype=torch.uint8, device=dev), "wsb": wsb,
                "ranges": torch.empty((1, R, S), dtype=torch.float64, device=dev),
                "ranges_h": torch.empty((1, R, S), dtype=torch.float64, pin_memory=True),
                "node_ids": torch.empty((1, R, Sk), dtype=torch.int32, device=dev),
                "neighbors": torch.empty((1, cap, 6), dtype=torch.int32, device=dev),
                "n64": torch.empty((1, cap, 3), dtype=torch.float64, device=dev),
                "nmask": torch.empty((1, cap), dtype=torch.uint8, device=dev),
                "cells": torch.empty((1, cap, 2), dtype=torch.int32, device=dev),
                "labels": torch.empty((1, R, S), dtype=torch.int32, device=dev),
                "counts": torch.empty((1, 2), dtype=torch.int32, device=dev)}
        cache.clear()  # keep one shape's buffers
        cache[key] = bufs
    b = bufs
    # staged through a cached pinned buffer: one host memcpy, one async H2D
    np.copyto(b["ranges_h"].numpy()[0], scan.ranges, casting="same_kind")
    b["ranges"].copy_(b["ranges_h"], non_blocking=True)
    _lib.profile_begin()
    _lib.check(L.lseg_run_scans(sn, 1, interval, _lib.thresholds_arg(seg.thresholds), int(seg.min_segment_size),
                                _lib.ptr(b["ranges"]), _lib.ptr(b["node_ids"]), _lib.ptr(b["neighbors"]),
                                _lib.ptr(b["n64"]), _lib.ptr(b["nmask"]), _lib.ptr(b["cells"]), None,
                                _lib.ptr(b["labels"]),
                                _lib.ptr(b["counts"][0, :1]), _lib.ptr(b["counts"][0, 1:]), _lib.ptr(b["ws"]), b["wsb"],
                                _lib.stream_ptr()))
    # every output downloaded asynchronously into fresh pinned host tensors
    # (torch's caching host allocator: no pinning cost per call), one
    # synchronisation; the returned arrays are views of those tensors
    pin = lambda t: torch.empty(t.shape[1:], dtype=t.dtype, pin_memory=True).copy_(t[0], non_blocking=True)
    h = {k: pin(b[k]) for k in ("counts", "node_ids", "labels", "neighbors", "n64", "nmask", "cells")}
    stages = _lib.profile_end()  # synchronises on the last event (after the copies were enqueued)
    torch.cuda.current_stream().synchronize()
    n = int(h["counts"][0])
    node_ids = h["node_ids"].numpy()
    labels = h["labels"].numpy()
    nb = h["neighbors"].numpy()[:n]
    m = h["nmask"].numpy()[:n].view(np.bool_)
    vals = h["n64"].numpy()[:n]  # NaN rows where the mask is False: written by the tile kernel
    cells = h["cells"].numpy()[:n]
    mesh = Mesh(rings=R, full_steps=S, interval=interval, kept_steps=kept, node_rings=cells[:, 0],
                node_steps=cells[:, 1].astype(np.int64), node_ids=node_ids, neighbors=nb)
    timings = {"mesh": 0.0, "normals": 0.0, "segment": 0.0, "backfill": 0.0}
    for name, (ms, _) in stages.items():
        if name in _STAGE_OF:
            timings[_STAGE_OF[name]] += ms
    timings["total"] = sum(timings.values())
    return PipelineResult(labels=labels, normals=NormalMap(values=vals, mask=m), mesh=mesh, timings_ms=timings)


_SCAN_BUFS = threading.local()


class BatchPipeline:
    """Device-resident batched hot path: F frames of points -> labels.

    Buffers are allocated once for (frames, points capacity); ``run`` takes
    device tensors xyz (P,3) f32, ring (P,) i32, offsets (F+1,) i64 and
    enqueues ONE C-ABI call (lseg_run_pipeline) on the current stream.
    """

    def __init__(self, config: SensorConfig, interval: int, segmenter: SegmenterConfig | None = None,
                 frames: int = 1, device=None, keep_node_labels: bool = False, streams: int = 1,
                 chunk_frames: int | None = None, normals: str = "exact", keep_node_ids: bool = True):
        self.L = _lib.lib()
        if normals not in ("certified", "exact"):
            raise ValueError("normals must be 'certified' or 'exact'")
        # "exact": fp64 normals in the reference's operation order, rounded to
        # fp32; "certified": fp32 normals with a rigorous error bound, exact
        # fp64 only where a decision or the output tolerance needs it (labels
        # identical in both modes)
        self.normals_mode = normals
        self.config = config
        self.interval = int(interval)
        subsample_steps(config, interval)
        self.seg = segmenter or SegmenterConfig()
        self.frames = int(frames)
        self.device = torch.device(device or "cuda")
        R, S = config.rings, config.azimuth_steps
        self.Sk = _lib.kept_count(S, interval)
        self.cap = R * self.Sk
        F, dev = self.frames, self.device
        _, self.sn = device_tables(config, dev)
        self.thr = _lib.thresholds_arg(self.seg.thresholds)
        self.ranges = torch.empty((F, R, S), dtype=torch.float64, device=dev)
        # node ids (F,R,S') are optional: derivable from the valid bits, and
        # 4 B per kept cell of HBM writes the batched path does not need
        self.node_ids = torch.empty((F, R, self.Sk), dtype=torch.int32, device=dev) if keep_node_ids else None
        self.neighbors = torch.empty((F, self.cap, 6), dtype=torch.int32, device=dev)
        self.normals = torch.empty((F, self.cap, 3), dtype=torch.float32, device=dev)
        self.nmask = torch.empty((F, self.cap), dtype=torch.uint8, device=dev)
        self.node_labels = torch.empty((F, R, S), dtype=torch.int32, device=dev) if keep_node_labels else None
        self.labels = torch.empty((F, R, S), dtype=torch.int32, device=dev)
        self.n_nodes = torch.empty(F, dtype=torch.int32, device=dev)
        self.n_labels = torch.empty(F, dtype=torch.int32, device=dev)
        # frames are independent: with streams > 1 the batch is cut into that
        # many chunks, each enqueued on its own stream (own workspace) so the
        # latency-bound kernels of one chunk overlap those of another
        self.nstreams = max(1, min(int(streams), F))
        per = -(-F // self.nstreams)
        if chunk_frames:  # sequential chunks on one stream (L2-sized intermediates)
            per = max(1, min(int(chunk_frames), F))
            self.nstreams = 1
        self.chunks = [(f0, min(F, f0 + per)) for f0 in range(0, F, per)]
        self.ws_bytes = _lib.workspace_bytes(per, R, S, interval)
        self.ws = [torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev) for _ in self.chunks]
        self.streams = ([torch.cuda.Stream(dev) for _ in self.chunks] if len(self.chunks) > 1 and not chunk_frames
                        else None)

    def _call(self, f0, f1, ws, xyz, ring, offsets):
        P = int(xyz.shape[0])
        sl = lambda t: None if t is None else t[f0:f1]
        flags = _lib.PIPE_CERT_NORMALS if self.normals_mode == "certified" else 0
        if ring.dtype == torch.uint8:
            flags |= _lib.PIPE_RING_U8
        elif ring.dtype == torch.int64 and ring.dim() == 2:
            if tuple(ring.shape) != (self.frames, self.config.rings + 1) or not ring.is_contiguous():
                raise ValueError("ring segment table must be (frames, rings + 1) int64, contiguous")
            flags |= _lib.PIPE_RING_SEGMENTS
            ring = ring[f0:]
        elif ring.dtype != torch.int32:
            raise ValueError("ring ids must be int32 / uint8, or an int64 (frames, rings + 1) segment table")
        _lib.check(self.L.lseg_run_pipeline_ex(
            self.sn, f1 - f0, self.interval, self.thr, int(self.seg.min_segment_size), flags, _lib.ptr(xyz),
            _lib.ptr(ring), _lib.ptr(offsets[f0:]), P, _lib.ptr(sl(self.ranges)), _lib.ptr(sl(self.node_ids)),
            _lib.ptr(sl(self.neighbors)), _lib.ptr(sl(self.normals)), _lib.ptr(sl(self.nmask)),
            _lib.ptr(sl(self.node_labels)), _lib.ptr(sl(self.labels)), _lib.ptr(sl(self.n_nodes)),
            _lib.ptr(sl(self.n_labels)), _lib.ptr(ws), self.ws_bytes, _lib.stream_ptr()))

    def run(self, xyz, ring, offsets):
        if self.streams is None:
            for (f0, f1), ws in zip(self.chunks, self.ws):
                self._call(f0, f1, ws, xyz, ring, offsets)
            return self.labels
        cur = torch.cuda.current_stream(self.device)
        for (f0, f1), ws, st in zip(self.chunks, self.ws, self.streams):
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                self._call(f0, f1, ws, xyz, ring, offsets)
        for st in self.streams:
            cur.wait_stream(st)
        return self.labels

    def run_grid(self, ranges: torch.Tensor) -> torch.Tensor:
        """The batch from range grids (F, R, S) f64 (NaN = INVALID) instead of
        points -- the batched form of the reference's run_pipeline(scan)
        (lseg_run_pipeline_grid).  ``self.ranges`` is not touched."""
        F = int(ranges.shape[0])
        if F > self.frames or tuple(ranges.shape[1:]) != (self.config.rings, self.config.azimuth_steps):
            raise ValueError("ranges must be (frames <= capacity, rings, azimuth_steps)")
        ranges = ranges.to(device=self.device, dtype=torch.float64).contiguous()
        flags = _lib.PIPE_CERT_NORMALS if self.normals_mode == "certified" else 0
        for (f0, f1), ws in zip(self.chunks, self.ws):  # one workspace per chunk, sequential
            f1 = min(f1, F)
            if f0 >= f1:
                break
            sl = lambda t: None if t is None else t[f0:f1]
            _lib.check(self.L.lseg_run_pipeline_grid(
                self.sn, f1 - f0, self.interval, self.thr, int(self.seg.min_segment_size), flags,
                _lib.ptr(ranges[f0:f1]), _lib.ptr(sl(self.node_ids)), _lib.ptr(sl(self.neighbors)),
                _lib.ptr(sl(self.normals)), _lib.ptr(sl(self.nmask)), _lib.ptr(sl(self.node_labels)),
                _lib.ptr(sl(self.labels)), _lib.ptr(sl(self.n_nodes)), _lib.ptr(sl(self.n_labels)), _lib.ptr(ws),
                self.ws_bytes, _lib.stream_ptr()))
        return self.labels[:F]

    def capture(self, xyz, ring, offsets) -> "torch.cuda.CUDAGraph":
        """Capture ``run`` on these (fixed) input buffers as one CUDA graph --
        the latency path for single live scans: replaying
        it costs one graph launch instead of ~15 kernel launches + memsets.
        Refill the same input tensors in place, then ``graph.replay()``."""
        self.run(xyz, ring, offsets)  # warm-up: kernel attributes, module load
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(xyz, ring, offsets)
        return g

    def frame(self, f: int) -> dict:
        """Host copies of frame f's outputs (reference-shaped)."""
        n = int(self.n_nodes[f].item())
        m = self.nmask[f, :n].bool().cpu().numpy()
        out = {"ranges": self.ranges[f].cpu().numpy(),
               "node_ids": None if self.node_ids is None else self.node_ids[f].cpu().numpy(),
               "neighbors": self.neighbors[f, :n].cpu().numpy(), "normals": self.normals[f, :n].cpu().numpy(),
               "mask": m, "labels": self.labels[f].cpu().numpy(), "n_labels": int(self.n_labels[f].item())}
        if self.node_labels is not None:
            out["node_labels"] = self.node_labels[f].cpu().numpy()
        return out


def ring_segments(ring, offsets, rings: int):
    """(F, rings + 1) int64 table of absolute point offsets of each ring of
    ring-major frames (the LSEG_PIPE_RING_SEGMENTS input form): ring i of
    frame f holds points [seg[f, i], seg[f, i + 1])."""
    r = torch.as_tensor(ring)
    off = torch.as_tensor(offsets, dtype=torch.int64, device=r.device)
    F = int(off.numel()) - 1
    out = torch.empty((F, rings + 1), dtype=torch.int64, device=r.device)
    q = torch.arange(rings + 1, dtype=r.dtype if r.dtype != torch.uint8 else torch.int32, device=r.device)
    for f in range(F):
        p0, p1 = int(off[f]), int(off[f + 1])
        rf = r[p0:p1].to(q.dtype)
        out[f] = torch.searchsorted(rf, q) + p0
    return out


def host_ring_segments(ring_h, offsets_h, rings: int, f0: int, f1: int):
    """(f1-f0, rings+1) int64 segment table of frames [f0, f1) of ring-major
    host points from their int32 ring ids: one binary search per ring
    boundary per frame on the host (the per-point ring ids stay on the host)."""
    r = ring_h.numpy() if isinstance(ring_h, torch.Tensor) else np.asarray(ring_h)
    o = offsets_h.numpy() if isinstance(offsets_h, torch.Tensor) else np.asarray(offsets_h)
    q = np.arange(rings + 1, dtype=r.dtype)
    out = np.empty((f1 - f0, rings + 1), dtype=np.int64)
    for f in range(f0, f1):
        a, b = int(o[f]), int(o[f + 1])
        out[f - f0] = np.searchsorted(r[a:b], q) + a
    return torch.from_numpy(out)


class StreamingPipeline:
    """Host-to-host batched hot path with copy/compute overlap.

    The batch is cut into chunks of ``chunk_frames``; for each chunk the
    points are copied host->device on one stream, the pipeline runs on a
    second, and the label grid is copied device->host on a third, double
    buffered, so PCIe traffic in both directions overlaps the kernels.
    Host buffers should be pinned (``torch.Tensor.pin_memory()``).
    """

    def __init__(self, config: SensorConfig, interval: int, segmenter: SegmenterConfig | None = None,
                 chunk_frames: int = 64, max_chunk_points: int | None = None, device=None,
                 ring_dtype=torch.int32, normals: str = "exact"):
        self.device = torch.device(device or "cuda")
        self.cf = int(chunk_frames)
        self.taper_min = max(1, self.cf // 8)
        R, S = config.rings, config.azimuth_steps
        self.maxp = int(max_chunk_points or self.cf * R * S)
        self.bps = [BatchPipeline(config, interval, segmenter, frames=self.cf, device=self.device, normals=normals,
                                  keep_node_ids=False) for _ in range(2)]
        self.xyz = [torch.empty((self.maxp, 3), dtype=torch.float32, device=self.device) for _ in range(2)]
        # "segments": the caller passes the (F, R+1) ring segment table of
        # ring-major points; "segments_from_ids": the caller passes int32 ring
        # ids and each chunk's table is computed on the host inside run_host
        # (binary searches of the ring boundaries, ring-major input assumed)
        self.ids_to_segments = ring_dtype == "segments_from_ids"
        self.segments = ring_dtype in ("segments", "segments_from_ids")
        self.R = R
        self.ring = [torch.empty((self.cf, R + 1), dtype=torch.int64, device=self.device) if self.segments
                     else torch.empty(self.maxp, dtype=ring_dtype, device=self.device) for _ in range(2)]
        self.off = [torch.empty(self.cf + 1, dtype=torch.int64, device=self.device) for _ in range(2)]
        self.s_in, self.s_run, self.s_out = (torch.cuda.Stream(self.device) for _ in range(3))
        self.freed = [torch.cuda.Event() for _ in range(2)]     # d2h of the chunk that used buffer b done
        self.loaded = [torch.cuda.Event() for _ in range(2)]
        self.computed = [torch.cuda.Event() for _ in range(2)]

    def run_host(self, xyz_h, ring_h, offsets_h, labels_h, n_nodes_h=None, neighbors_h=None, normals_h=None,
                 mask_h=None):
        """xyz_h (P,3) f32, ring_h (P,) i32 / u8 (with ring_dtype="segments",
        the (F, R+1) i64 table of ``ring_segments``; with "segments_from_ids",
        (P,) i32 ring ids converted per chunk on the host), offsets_h (F+1,) i64 host
        tensors (pinned); labels_h (F,R,S) i32 pinned output.  Enqueues everything and
        returns; synchronise on the current stream to wait.

        The rest of the reference's PipelineResult (pipeline.py:39-44) per
        frame, when the optional pinned outputs are given: n_nodes_h (F,) i32,
        neighbors_h (F, R*S', 6) i32 (Mesh.neighbors, rows [0, n_nodes) valid),
        normals_h (F, R*S', 3) f32 and mask_h (F, R*S') u8 (NormalMap values /
        mask; NaN where absent).  Whole node-capacity rows are copied so the
        stream never waits on a node count."""
        F = offsets_h.numel() - 1
        extra = [(h, name) for h, name in ((n_nodes_h, "n_nodes"), (neighbors_h, "neighbors"),
                                           (normals_h, "normals"), (mask_h, "nmask")) if h is not None]
        offs = offsets_h.tolist()
        cur = torch.cuda.current_stream(self.device)
        start = torch.cuda.Event()
        start.record(cur)
        for s in (self.s_in, self.s_run, self.s_out):
            s.wait_event(start)
        # chunk boundaries: full chunks, then a geometric taper (1/2, 1/4, ...)
        # so the pipeline drain -- the last chunk's kernels + label copy,
        # which nothing overlaps -- is short
        bounds = [0]
        while bounds[-1] < F:
            left = F - bounds[-1]
            step = self.cf if left > 2 * self.cf else max(self.taper_min, min(self.cf, (left + 1) // 2))
            bounds.append(min(F, bounds[-1] + step))
        for ci in range(len(bounds) - 1):
            b = ci % 2
            f0, f1 = bounds[ci], bounds[ci + 1]
            nf = f1 - f0
            p0, p1 = offs[f0], offs[f1]
            if p1 - p0 > self.maxp:
                raise ValueError("chunk has more points than max_chunk_points")
            bp = self.bps[b]
            with torch.cuda.stream(self.s_in):
                if ci >= 2:
                    self.s_in.wait_event(self.freed[b])
                self.xyz[b][: p1 - p0].copy_(xyz_h[p0:p1], non_blocking=True)
                loc = offsets_h[f0:f1 + 1] - p0
                if self.segments:  # chunk-relative segment table, empty frames as padding
                    if self.ids_to_segments:
                        seg = host_ring_segments(ring_h, offsets_h, self.R, f0, f1) - p0
                    else:
                        seg = ring_h[f0:f1] - p0
                    if nf < self.cf:
                        seg = torch.cat([seg, seg.new_full((self.cf - nf, self.R + 1), int(loc[-1]))])
                    self.ring[b].copy_(seg, non_blocking=True)
                else:
                    self.ring[b][: p1 - p0].copy_(ring_h[p0:p1], non_blocking=True)
                if nf < self.cf:  # pad the last chunk with empty frames
                    loc = torch.cat([loc, loc[-1:].expand(self.cf - nf)])
                self.off[b].copy_(loc, non_blocking=True)
                self.loaded[b].record(self.s_in)
            with torch.cuda.stream(self.s_run):
                self.s_run.wait_event(self.loaded[b])
                bp.run(self.xyz[b], self.ring[b], self.off[b])
                self.computed[b].record(self.s_run)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.computed[b])
                labels_h[f0:f1].copy_(bp.labels[:nf], non_blocking=True)
                for h, name in extra:
                    h[f0:f1].copy_(getattr(bp, name)[:nf], non_blocking=True)
                self.freed[b].record(self.s_out)
        cur.wait_stream(self.s_out)
        cur.wait_stream(self.s_run)
        cur.wait_stream(self.s_in)
        return labels_h
