"""B200-native ALS / MFITR sweep of arXiv 1108.2580's collaborative-filtering
ensemble: a drop-in for the reference package's ALS / wALS / MFITR fit and
predict entry points (``factor``, ``mfitr``, ``registry``), backed by the
sm_100a kernels of ``libmcf.so`` (C-ABI: include/mcf.h)."""

__version__ = "0.1.0"

from .data import DEFAULT_SCALE, Dataset, ScoreScale  # noqa: F401
from .errors import (ConfigError, DeviceError, EngineError, ShapeError,  # noqa: F401
                     SingularSystemError)
