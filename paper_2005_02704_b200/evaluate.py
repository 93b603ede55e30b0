"""Edge-based precision / recall / F1, mirroring reference evaluate.py:20-94.

``extract_edges``, ``dilate_chebyshev`` and ``edge_prf`` keep the reference's
signatures and semantics; the counting runs on the GPU (C ABI
lseg_edge_counts / lseg_extract_edges / lseg_dilate_chebyshev) and
``edge_prf_batch`` scores whole frame batches on the device.  ``bench`` /
``StageStats`` / ``time_total`` are the reference's timing helpers (host).
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from statistics import mean, median

import numpy as np
import torch

from . import _lib


@dataclass(frozen=True)
class EvalConfig:
    dilation_radius: int = 2

    def __post_init__(self):
        if self.dilation_radius < 0:
            raise ValueError("dilation_radius must be >= 0")


@dataclass(frozen=True)
class EvalReport:
    precision: float
    recall: float
    f1: float
    timings_ms: dict | None = None


def _dev_grid(a, dtype):
    t = torch.as_tensor(np.ascontiguousarray(a), dtype=dtype)
    if t.dim() == 2:
        t = t.unsqueeze(0)
    return t.to("cuda")


def _ws(F, R, S):
    n = int(_lib.load().lseg_eval_workspace_bytes(F, R, S))
    return torch.empty(max(n, 1), dtype=torch.uint8, device="cuda"), n


def extract_edges(labels) -> np.ndarray:
    """Edge cells of a label grid (reference evaluate.py:40-55), GPU."""
    L = _lib.lib()
    lab = _dev_grid(labels, torch.int32)
    F, R, S = lab.shape
    out = torch.empty((F, R, S), dtype=torch.uint8, device="cuda")
    ws, n = _ws(F, R, S)
    _lib.check(L.lseg_extract_edges(F, R, S, _lib.ptr(lab), _lib.ptr(out), _lib.ptr(ws), n, _lib.stream_ptr()))
    res = out.bool().cpu().numpy()
    return res[0] if np.asarray(labels).ndim == 2 else res


def dilate_chebyshev(mask, radius: int) -> np.ndarray:
    """Binary dilation with a (2r+1)^2 square (reference evaluate.py:58-70), GPU."""
    if radius < 0:
        raise ValueError("dilation_radius must be >= 0")
    L = _lib.lib()
    m = _dev_grid(np.asarray(mask, dtype=np.uint8), torch.uint8)
    F, R, S = m.shape
    out = torch.empty((F, R, S), dtype=torch.uint8, device="cuda")
    ws, n = _ws(F, R, S)
    _lib.check(L.lseg_dilate_chebyshev(F, R, S, _lib.ptr(m), int(radius), _lib.ptr(out), _lib.ptr(ws), n,
                                       _lib.stream_ptr()))
    res = out.bool().cpu().numpy()
    return res[0] if np.asarray(mask).ndim == 2 else res


def edge_counts_device(pred, truth, radius: int):
    """(F, 4) int32 device counts for device label batches (F, R, S)."""
    L = _lib.lib()
    F, R, S = pred.shape
    counts = torch.empty((F, 4), dtype=torch.int32, device=pred.device)
    ws, n = _ws(F, R, S)
    _lib.check(L.lseg_edge_counts(F, R, S, _lib.ptr(pred), _lib.ptr(truth), int(radius), _lib.ptr(counts),
                                  _lib.ptr(ws), n, _lib.stream_ptr()))
    return counts


def _prf(n_p, n_t, m_p, m_t):
    if n_p == 0 and n_t == 0:
        return 1.0, 1.0, 1.0
    p = m_p / n_p if n_p else 0.0
    r = m_t / n_t if n_t else 0.0
    f = 2.0 * p * r / (p + r) if p > 0.0 and r > 0.0 else 0.0
    return float(p), float(r), float(f)


def edge_prf(pred_labels, truth_labels, cfg: EvalConfig) -> EvalReport:
    """Edge precision / recall / F1 with dilated matching (reference evaluate.py:73-94)."""
    pred = np.asarray(pred_labels)
    truth = np.asarray(truth_labels)
    if pred.shape != truth.shape:
        raise ValueError(f"label grids differ in shape: {pred.shape} vs {truth.shape}")
    c = edge_counts_device(_dev_grid(pred, torch.int32), _dev_grid(truth, torch.int32),
                           cfg.dilation_radius)[0].tolist()
    p, r, f = _prf(*c)
    return EvalReport(precision=p, recall=r, f1=f)


def edge_prf_batch(pred, truth, radius: int = 2) -> torch.Tensor:
    """(F, 3) precision / recall / F1 for device label batches (F, R, S)."""
    c = edge_counts_device(pred, truth, radius).double()
    n_p, n_t, m_p, m_t = c.unbind(1)
    p = torch.where(n_p > 0, m_p / n_p.clamp_min(1), torch.zeros_like(n_p))
    r = torch.where(n_t > 0, m_t / n_t.clamp_min(1), torch.zeros_like(n_t))
    f = torch.where((p > 0) & (r > 0), 2 * p * r / (p + r).clamp_min(1e-300), torch.zeros_like(p))
    both_empty = (n_p == 0) & (n_t == 0)
    one = torch.ones_like(p)
    return torch.stack([torch.where(both_empty, one, p), torch.where(both_empty, one, r),
                        torch.where(both_empty, one, f)], dim=1)


@dataclass(frozen=True)
class StageStats:
    min: float
    median: float
    mean: float
    max: float
    samples: tuple

    @classmethod
    def of(cls, samples) -> "StageStats":
        s = tuple(float(x) for x in samples)
        return cls(min=min(s), median=median(s), mean=mean(s), max=max(s), samples=s)


def bench(pipeline, repetitions: int) -> dict:
    """One discarded warm-up plus `repetitions` timed runs (reference evaluate.py:113-121)."""
    if repetitions < 3:
        raise ValueError("repetitions must be >= 3")
    pipeline()
    runs = [dict(pipeline()) for _ in range(repetitions)]
    return {stage: StageStats.of([run[stage] for run in runs]) for stage in runs[0].keys()}


def time_total(fn):
    def run():
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return {"total": (time.perf_counter() - t0) * 1e3}
    return run
