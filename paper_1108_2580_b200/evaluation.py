"""RMSE, name-for-name with the reference (pkg/src/multicf/evaluation.py:11-18).

``rmse`` is the host metric on numpy arrays; ``device_rmse`` fuses
predict + clip + squared error on the GPU (mcf_predict_sse)."""
from __future__ import annotations

import numpy as np

from .errors import MetricError, ShapeError


def rmse(pred, truth) -> float:
    pred = np.asarray(pred, dtype=np.float64)
    truth = np.asarray(truth, dtype=np.float64)
    if pred.shape != truth.shape:
        raise ShapeError(f"prediction length {pred.shape} != truth length {truth.shape}")
    if pred.size == 0:
        raise MetricError("rmse undefined on empty input")
    return float(np.sqrt(np.mean((pred - truth) ** 2)))


def device_rmse(engine, users, items, truth, clip=(0.0, 100.0)) -> float:
    """sqrt(mean((clip(q.p) - truth)^2)) over device tensors."""
    if users.numel() == 0:
        raise MetricError("rmse undefined on empty input")
    return float(engine.rmse(users, items, truth, clip).item())
