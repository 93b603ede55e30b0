"""lidarseg on B200: the per-scan hot path of arXiv 2005.02704 as sm_100a CUDA.

Mirrors the reference package's public API for that path (reference
pkg/src/lidarseg/__init__.py:21-35): data model, ``build_mesh``,
``mesh_triangles``, ``estimate_normals``, ``segment``, ``backfill``,
``prune_small``, ``run_pipeline``; adds ``bin_points`` and the batched
``BatchPipeline``.  Beyond the hot path: the edge
evaluator, the streaming ``MeshBuilder`` and the scan simulator
(``cast_grid``, ``scan_scene``, ``scene_normals``, ``generate_scene``).  Every compute op runs through liblidarseg_b200.so (C ABI,
include/lidarseg_b200.h); there is no CPU fallback.
"""

from .evaluate import (EvalConfig, EvalReport, StageStats, bench, dilate_chebyshev, edge_prf, edge_prf_batch,
                       extract_edges, time_total)
from .mesh import Mesh, MeshBuilder, build_mesh, mesh_triangles
from .normals import NormalMap, estimate_normals, node_positions, normal_from_neighbors, normals_to_grid, point_normal
from .pipeline import BaselineConfig, BatchPipeline, PipelineConfig, PipelineResult, StreamingPipeline, bin_points, ring_segments, run_pipeline
from .scan import (INVALID, GridIndex, Point3, ScanGrid, SensorConfig, polar_to_cartesian, subsample_steps,
                   valid_point)
from .scenes import generate_scene, generate_suite
from .suite import run_suite, scan_scenes
from . import io
from .segment import SegmenterConfig, backfill, prune_small, segment
from .simulate import (Box, Cone, Cylinder, Plane, Scene, Sphere, cast_grid, cast_grid_batch, ray_intersect,
                       rotation_rpy, scan_scene, scene_normals)

__version__ = "0.1.0"
