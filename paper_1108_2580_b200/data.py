"""Rating containers for the drop-in API.

Mirrors the parts of the reference's ``multicf.data`` that sit on the ALS /
MFITR path (reference: pkg/src/multicf/data.py:19-35 ScoreScale,
data.py:75-160 Dataset).  Records stay in file order on the host; the
device layout (CSR by user, CSC by item) is built from them by
``device.DeviceRatings`` with the reference's stable in-row order
(factor.py:502, data.py:136).

Differences, all additive: ``times`` may be omitted (the ALS path never
reads it) and ``compact=True`` keeps int32 ids / float32 scores so that a
full-size split (262 M ratings) fits in host memory twice over.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, ParseError, RangeError


@dataclass(frozen=True)
class ScoreScale:
    """Closed score interval; predictions are clipped to it on emission and
    in RMSE (reference data.py:19-35, factor.py:616)."""

    lo: float = 0.0
    hi: float = 100.0

    def __post_init__(self):
        if not self.lo < self.hi:
            raise ConfigError(f"score scale requires lo < hi, got [{self.lo}, {self.hi}]")

    def clip(self, x):
        return np.clip(x, self.lo, self.hi)

    def contains(self, x) -> bool:
        return self.lo <= x <= self.hi


DEFAULT_SCALE = ScoreScale(0.0, 100.0)


@dataclass
class Dataset:
    """One split of (user, item, score[, time]) records in file order."""

    users: np.ndarray
    items: np.ndarray
    scores: np.ndarray
    times: np.ndarray
    split: str = "train"
    num_users: int = 0
    num_items: int = 0
    scale: ScoreScale = DEFAULT_SCALE
    _user_csr: tuple | None = field(default=None, repr=False, compare=False)

    @classmethod
    def from_arrays(cls, users, items, scores, times=None, split="train",
                    scale: ScoreScale = DEFAULT_SCALE,
                    num_users: int | None = None, num_items: int | None = None,
                    compact: bool = False) -> "Dataset":
        """Validate and wrap parallel arrays (reference data.py:97-119):
        equal lengths, ids in [0, num_users) x [0, num_items), counts default
        to max id + 1."""
        it, ft = (np.int32, np.float32) if compact else (np.int64, np.float64)
        users = np.ascontiguousarray(users, dtype=it)
        items = np.ascontiguousarray(items, dtype=it)
        scores = np.ascontiguousarray(scores, dtype=ft)
        n = users.size
        times = (np.zeros(n, dtype=np.int64) if times is None
                 else np.ascontiguousarray(times, dtype=np.int64))
        if not (items.size == n and scores.size == n and times.size == n):
            raise ConfigError("rating arrays must have equal length")
        nu = int(users.max()) + 1 if n else 0
        ni = int(items.max()) + 1 if n else 0
        num_users = nu if num_users is None else int(num_users)
        num_items = ni if num_items is None else int(num_items)
        if n and (int(users.min()) < 0 or nu > num_users):
            raise RangeError("user id outside [0, num_users)")
        if n and (int(items.min()) < 0 or ni > num_items):
            raise RangeError("item id outside [0, num_items)")
        return cls(users, items, scores, times, split, num_users, num_items, scale)

    def __len__(self) -> int:
        return int(self.users.size)

    def by_user(self):
        """(order, ptr): record indices grouped by user, file order inside a
        user (reference data.py:132-142)."""
        if self._user_csr is None:
            order = np.argsort(self.users, kind="stable").astype(np.int64)
            ptr = np.zeros(self.num_users + 1, dtype=np.int64)
            np.cumsum(np.bincount(self.users, minlength=self.num_users), out=ptr[1:])
            self._user_csr = (order, ptr)
        return self._user_csr

    def global_mean(self) -> float:
        return float(np.mean(self.scores, dtype=np.float64)) if len(self) else 0.0

    def degrees(self, side: str) -> np.ndarray:
        keys, n = ((self.users, self.num_users) if side == "users"
                   else (self.items, self.num_items))
        return np.bincount(keys, minlength=n).astype(np.int64)


def load_ratings(path, split: str = "train", scale: ScoreScale = DEFAULT_SCALE,
                 compact: bool = False) -> Dataset:
    """Parse `user<TAB>item<TAB>score<TAB>time` lines; blank and '#' lines are
    skipped; non-numeric fields, negative ids and scores outside the scale
    raise (reference data.py:163-191)."""
    users, items, scores, times = [], [], [], []
    with open(path, "r", encoding="utf-8") as fh:
        for line_no, line in enumerate(fh, start=1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split("\t")
            if len(parts) != 4:
                raise ParseError(path, line_no,
                                 f"expected 4 tab-separated fields, got {len(parts)}")
            try:
                u, i, sc, t = int(parts[0]), int(parts[1]), float(parts[2]), int(parts[3])
            except ValueError as exc:
                raise ParseError(path, line_no, f"non-numeric field: {exc}") from None
            if u < 0 or i < 0:
                raise ParseError(path, line_no, "negative id")
            if not scale.contains(sc):
                raise RangeError(f"{path}:{line_no}: score {sc} outside scale "
                                 f"[{scale.lo}, {scale.hi}]")
            users.append(u)
            items.append(i)
            scores.append(sc)
            times.append(t)
    return Dataset.from_arrays(users, items, scores, times, split=split, scale=scale,
                               compact=compact)
