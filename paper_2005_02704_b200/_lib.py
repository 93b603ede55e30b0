"""ctypes binding of liblidarseg_b200.so (the C ABI in include/lidarseg_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every op raises.  Buffers are torch CUDA tensors passed as
raw device pointers together with the current torch stream.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LSEG_LIB_PATH") or os.path.join(PKG, "liblidarseg_b200.so")


class LidarSegError(RuntimeError):
    """Raised when the CUDA library reports an error (non-ValueError codes)."""


class lseg_sensor(C.Structure):
    _fields_ = [("rings", C.c_int32), ("steps", C.c_int32), ("r_min", C.c_double), ("r_max", C.c_double),
                ("cos_el", C.c_void_p), ("sin_el", C.c_void_p), ("cos_az", C.c_void_p),
                ("sin_az", C.c_void_p)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_SIGS = {
    "lseg_last_error": (C.c_char_p, []),
    "lseg_version": (C.c_char_p, []),
    "lseg_profile_begin": (C.c_int, []),
    "lseg_profile_end": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_double), C.POINTER(_I32), _I32,
                                   C.POINTER(_I32)]),
    "lseg_kept_count": (_I32, [_I32, _I32]),
    "lseg_workspace_bytes": (C.c_size_t, [_I32, _I32, _I32, _I32, _I64]),
    "lseg_bin_points": (C.c_int, [C.POINTER(lseg_sensor), _I32, _P, _P, _P, _I64, _P, _P, _P]),
    "lseg_build_mesh": (C.c_int, [C.POINTER(lseg_sensor), _I32, _I32, C.c_double, _P, _P, _P, _P, _P, _P, _P,
                                  C.c_size_t, _P]),
    "lseg_mesh_triangles": (C.c_int, [_I32, _I32, _I32, _P, _P, _P, _P]),
    "lseg_estimate_normals": (C.c_int, [C.POINTER(lseg_sensor), _I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lseg_segment": (C.c_int, [_I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, C.POINTER(C.c_double), _P, _P, _P,
                               C.c_size_t, _P]),
    "lseg_backfill": (C.c_int, [C.POINTER(lseg_sensor), _I32, _P, _P, _P, _P]),
    "lseg_prune_small": (C.c_int, [_I32, _I32, _I32, _P, _I32, _I64, _P, _P, C.c_size_t, _P]),
    "lseg_run_pipeline_r8": (C.c_int, [C.POINTER(lseg_sensor), _I32, _I32, C.POINTER(C.c_double), _I32, _P, _P, _P,
                                       _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "lseg_eval_workspace_bytes": (C.c_size_t, [_I32, _I32, _I32]),
    "lseg_edge_counts": (C.c_int, [_I32, _I32, _I32, _P, _P, _I32, _P, _P, C.c_size_t, _P]),
    "lseg_extract_edges": (C.c_int, [_I32, _I32, _I32, _P, _P, _P, C.c_size_t, _P]),
    "lseg_dilate_chebyshev": (C.c_int, [_I32, _I32, _I32, _P, _I32, _P, _P, C.c_size_t, _P]),
    "lseg_run_pipeline": (C.c_int, [C.POINTER(lseg_sensor), _I32, _I32, C.POINTER(C.c_double), _I32, _P, _P, _P,
                                    _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "lseg_run_pipeline_grid": (C.c_int, [C.POINTER(lseg_sensor), _I32, _I32, C.POINTER(C.c_double), _I32, C.c_uint32,
                                         _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "lseg_run_scans": (C.c_int, [C.POINTER(lseg_sensor), _I32, _I32, C.POINTER(C.c_double), _I32, _P, _P, _P, _P,
                                 _P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "lseg_mb_column": (C.c_int, [_I32, _I32, _I32, C.c_double, C.c_double, _P, _P, _P, _P, _P]),
    "lseg_mb_finish": (C.c_int, [_I32, _I32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lseg_format_rows": (C.c_int64, [C.c_int64, _I32, _P, _P, _P, C.c_int64, _I32]),
    "lseg_cast_grid": (C.c_int, [C.POINTER(lseg_sensor), _I32, _P, _I32, _P, _P, _P, _P]),
    "lseg_cast_rays": (C.c_int, [_P, _I32, _I64, _P, _P, _P, _P, _P]),
    "lseg_apply_scan": (C.c_int, [_I64, C.c_double, C.c_double, _P, _P, _P, _P, _P, _P]),
    "lseg_scene_normals": (C.c_int, [C.POINTER(lseg_sensor), _P, _I32, _P, _P, _P, _P]),
    "lseg_run_pipeline_ex": (C.c_int, [C.POINTER(lseg_sensor), _I32, _I32, C.POINTER(C.c_double), _I32, C.c_uint32,
                                       _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
}
PIPE_CERT_NORMALS = 1  # include/lidarseg_b200.h LSEG_PIPE_CERT_NORMALS
PIPE_RING_U8 = 2
PIPE_RING_SEGMENTS = 4
EXPORTS = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load the shared library (no device needed) and declare signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LidarSegError(f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    """The library, with a CUDA device required (no CPU fallback exists)."""
    if not torch.cuda.is_available():
        raise LidarSegError("lidarseg_b200 needs a CUDA device (B200); no CPU fallback exists")
    return load()


def check(rc: int):
    if rc == 0:
        return
    msg = load().lseg_last_error().decode()
    if rc == -1:
        raise ValueError(msg)
    raise LidarSegError(f"lidarseg_b200 error {rc}: {msg}")


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def stream_ptr():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def thresholds_arg(thr):
    arr = (C.c_double * 3)(*[float(v) for v in thr])
    return arr


def kept_count(steps: int, interval: int) -> int:
    return int(load().lseg_kept_count(int(steps), int(interval)))


def workspace_bytes(frames, rings, steps, interval, label_bound=0) -> int:
    return int(load().lseg_workspace_bytes(int(frames), int(rings), int(steps), int(interval), int(label_bound)))


def profile_begin():
    check(lib().lseg_profile_begin())


def profile_end(max_stages: int = 64) -> dict:
    """{stage: (total_ms, launches)} for stages enqueued since profile_begin()."""
    buf = C.create_string_buffer(4096)
    ms = (C.c_double * max_stages)()
    cnt = (_I32 * max_stages)()
    n = _I32(0)
    check(lib().lseg_profile_end(buf, 4096, ms, cnt, max_stages, C.byref(n)))
    names = buf.value.decode().split(",") if n.value else []
    return {nm: (ms[i], cnt[i]) for i, nm in enumerate(names)}
