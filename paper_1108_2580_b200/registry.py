"""Kind -> trainer / predictor dispatch for the device path, mirroring the
reference's registry (pkg/src/multicf/registry.py:44-89) for the kinds this
path serves: ``als``, ``wals`` (factor.train) and ``mfitr``
(mfitr.train_mfitr, the ALS-MFITR solver)."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import factor
from .data import Dataset
from .errors import ConfigError

DEVICE_KINDS = ("als", "wals", "mfitr")
ALL_KINDS = ("knn", "time-knn", "als", "wals", "sgd", "svdpp", "time-svd", "time-svdpp",
             "mfitr", "time-mfitr")


def default_hyper(kind: str):
    if kind in ("als", "wals"):
        return factor.default_hyper(kind)
    if kind == "mfitr":
        from . import mfitr
        return mfitr.default_mfitr_hyper(kind)
    if kind in ALL_KINDS:
        raise ConfigError(f"{kind!r} is outside the device ALS/MFITR path")
    raise ConfigError(f"unknown model kind {kind!r}")


@dataclass
class TrainedModel:
    kind: str
    model: object
    context: Dataset | None = None
    report: list = field(default_factory=list)

    def predict(self, users, items, times=None, context=None) -> np.ndarray:
        """Unclipped batch predictions (registry.py:54-63)."""
        if self.kind == "mfitr":
            from . import mfitr
            return mfitr.predict_batch(self.model, users, items, times)
        return factor.predict_batch(self.model, users, items, times)


def train_model(kind: str, train: Dataset, hyper=None, seed: int = 0,
                validation: Dataset | None = None, taxonomy=None, binner=None, threads: int = 1,
                weights: np.ndarray | None = None, **device_opts) -> TrainedModel:
    if kind not in ALL_KINDS:
        raise ConfigError(f"unknown model kind {kind!r}")
    if hyper is None:
        hyper = default_hyper(kind)
    if kind == "mfitr":
        from . import mfitr
        if taxonomy is None:
            raise ConfigError(f"{kind} requires a taxonomy")
        n_items = max(train.num_items, taxonomy.num_nodes)
        model, report = mfitr.train_mfitr(kind, train, validation, taxonomy, hyper,
                                          threads=threads, seed=seed, num_items=n_items,
                                          **device_opts)
        return TrainedModel(kind, model, context=train, report=report)
    if kind not in ("als", "wals"):
        default_hyper(kind)
    model, report = factor.train(kind, train, validation, hyper, threads=threads, seed=seed,
                                 weights=weights, **device_opts)
    return TrainedModel(kind, model, context=train, report=report)
