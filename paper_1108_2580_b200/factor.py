"""Drop-in ALS / wALS entry points, backed by the sm_100a kernels.

Same names, signatures, return types and error behaviour as the reference's
``multicf.factor`` ALS section (reference pkg/src/multicf/factor.py:29-69
HyperParams/default_hyper, :126-166 init_model, :222-242 predict_batch,
:493-555 als_half_step/als_objective/als_iteration, :561-618 train).
Additive keyword-only options:

* ``reg``: ``"plain"`` (reference semantics: lam * I) or ``"weighted"``
  (lam * n_r * I, ALS-WR -- BASELINE's "weighted-lambda");
* ``init``: ``(P0, Q0)`` initial factors instead of the reference's uniform
  draw (BASELINE initialises N(0, 0.1));
* ``device``: the CUDA device; ``as_torch``: keep the fitted factors as
  device tensors instead of numpy float64 copies;
* ``devices``: ``N > 1`` fits with the rows of each half-step sharded over N
  GPUs -- the device form of the reference's ``threads`` (parallel.py:134-145,
  factor.py:528-534): one process per GPU (``torchrun --nproc-per-node N``)
  and every rank calls ``train(..., devices=N)`` on the same data (SPMD);
  results are identical to one GPU (G-invariance) and returned on every rank.

``threads`` is accepted and ignored (the device decides the parallelism).
There is no CPU fallback: without libmcf.so or a GPU these raise DeviceError.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np
import torch

from .data import DEFAULT_SCALE, Dataset, ScoreScale
from .device import AlsEngine, DeviceRatings, cuda_device
from .errors import ConfigError, DivergenceError, ShapeError

ALS_KINDS = ("als", "wals")
SGD_KINDS = ("sgd", "svdpp", "time-svd", "time-svdpp")
FACTOR_KINDS = SGD_KINDS + ALS_KINDS
INIT_AMPLITUDE = 0.005


@dataclass
class HyperParams:
    gamma: float = 5e-4
    decay: float = 0.95
    lam: float = 1e-4
    lam1: float = 1e-5
    lam2: float = 1e-4
    lam3: float = 3e-4
    iters: int = 50
    D: int = 50
    D_t: int = 8

    def __post_init__(self):
        if self.gamma <= 0:
            raise ConfigError("gamma must be > 0")
        if not 0 < self.decay <= 1:
            raise ConfigError("decay must be in (0, 1]")
        if min(self.lam, self.lam1, self.lam2, self.lam3) < 0:
            raise ConfigError("regularisation weights must be >= 0")
        if self.iters < 0:
            raise ConfigError("iters must be >= 0")
        if self.D < 1 or self.D_t < 1:
            raise ConfigError("factor dimensions must be >= 1")


def default_hyper(kind: str) -> HyperParams:
    """Reference ALS defaults: lam=1, D=120, 50 iterations (factor.py:67-68)."""
    if kind in ALS_KINDS:
        return HyperParams(gamma=1.0, decay=1.0, lam=1.0, iters=50, D=120)
    if kind in SGD_KINDS:
        raise ConfigError(f"{kind!r} is an SGD model: not part of the device ALS path")
    raise ConfigError(f"unknown factor model kind {kind!r}")


@dataclass
class FactorModel:
    """ALS model state (mu = 0, no biases, factors p/q), reference
    factor.py:72-123 restricted to the ALS kinds."""

    kind: str
    mu: float
    b_u: np.ndarray
    b_i: np.ndarray
    p: np.ndarray
    q: np.ndarray
    D: int
    seed: int
    scale: ScoreScale = DEFAULT_SCALE
    epochs_done: int = 0
    engine: AlsEngine | None = field(default=None, repr=False, compare=False)

    @property
    def num_users(self) -> int:
        return int(self.b_u.size)

    @property
    def num_items(self) -> int:
        return int(self.b_i.size)

    def check_finite(self, epoch: int) -> None:
        for name in ("p", "q"):
            arr = getattr(self, name)
            if isinstance(arr, torch.Tensor):
                ok = bool(torch.isfinite(arr).all())
            else:
                ok = bool(np.isfinite(arr).all())
            if not ok:
                raise DivergenceError(epoch, f"non-finite {name} after epoch {epoch}")

    def copy(self) -> "FactorModel":
        return dataclasses.replace(self, b_u=self.b_u.copy(), b_i=self.b_i.copy(),
                                   p=self.p.clone() if isinstance(self.p, torch.Tensor) else self.p.copy(),
                                   q=self.q.clone() if isinstance(self.q, torch.Tensor) else self.q.copy(),
                                   engine=None)


def init_model(kind: str, train: Dataset, hyper: HyperParams, seed: int, binner=None,
               num_users: int | None = None, num_items: int | None = None) -> FactorModel:
    """Reference initialisation: q then p ~ U(+-0.005/sqrt(D)) from
    default_rng([seed, 1]), biases and mu zero (factor.py:126-166)."""
    if kind not in ALS_KINDS:
        default_hyper(kind)  # raises with the right message
    U = num_users if num_users is not None else train.num_users
    I = num_items if num_items is not None else train.num_items
    rng = np.random.default_rng([seed, 1])
    amp = INIT_AMPLITUDE / np.sqrt(hyper.D)
    q = rng.uniform(-amp, amp, (I, hyper.D))
    p = rng.uniform(-amp, amp, (U, hyper.D))
    return FactorModel(kind, 0.0, np.zeros(U), np.zeros(I), p, q, hyper.D, seed, train.scale)


# ---------------------------------------------------------------------------
# device plumbing

def _ratings_for(train: Dataset, device, keep_perm: bool, num_users=None,
                 num_items=None) -> DeviceRatings:
    """Resident layouts, cached on the Dataset object (the reference rebuilds
    its CSR every half-step, factor.py:522; the device keeps it)."""
    dev = cuda_device(device)
    U = num_users if num_users is not None else train.num_users
    I = num_items if num_items is not None else train.num_items
    cache = train.__dict__.setdefault("_device_cache", {})
    key = (str(dev), U, I)
    r = cache.get(key)
    if r is None or (keep_perm and r.by_user.perm is None):
        r = DeviceRatings(train.users, train.items, train.scores, U, I, dev, keep_perm)
        cache[key] = r
    return r


def _engine_for(model: FactorModel, train: Dataset, device, keep_perm: bool) -> AlsEngine:
    """The model's engine over the resident layouts (factors NOT uploaded)."""
    r = _ratings_for(train, device, keep_perm, model.num_users, model.num_items)
    eng = model.engine
    if eng is None or eng.r is not r:
        eng = AlsEngine(r, model.D)
        model.engine = eng
    return eng


def _host(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else x


def _lam_pair(lam: float, reg: str):
    if reg == "plain":
        return float(lam), 0.0
    if reg == "weighted":
        return 0.0, float(lam)
    raise ConfigError(f"reg must be 'plain' or 'weighted', got {reg!r}")


def _sync_host(model: FactorModel, sides=("users", "items")):
    P, Q = model.engine.factors()
    if "users" in sides:
        model.p = P.double().cpu().numpy()
    if "items" in sides:
        model.q = Q.double().cpu().numpy()


# ---------------------------------------------------------------------------
# ALS

def als_half_step(model: FactorModel, train: Dataset, side: str, lam: float,
                  weights: np.ndarray | None = None, threads: int = 1, *, reg: str = "plain",
                  device=None) -> FactorModel:
    """Exactly solve one side's regularised normal equations (factor.py:512-538).

    Raises ConfigError on negative weights or a bad side, ShapeError on a
    weight-length mismatch, SingularSystemError (minimum failing row) when
    a row's system is not positive definite."""
    if side not in ("users", "items"):
        raise ConfigError(f"side must be 'users' or 'items', got {side!r}")
    if weights is not None:
        weights = np.asarray(weights, dtype=np.float64)
        if np.any(weights < 0):
            raise ConfigError("observation weights must be >= 0")
        if weights.size != len(train):
            raise ShapeError(f"expected {len(train)} weights, got {weights.size}")
    lam_c, lam_n = _lam_pair(lam, reg)
    eng = _engine_for(model, train, device, keep_perm=weights is not None)
    eng.set_factors(_host(model.p), _host(model.q))
    eng.set_weights(weights)
    eng.half_step(side, lam_c, lam_n)
    try:
        eng.check()
    finally:
        _sync_host(model, (side,))
    return model


def als_iteration(model: FactorModel, train: Dataset, lam: float,
                  weights: np.ndarray | None = None, threads: int = 1, *, reg: str = "plain",
                  device=None) -> FactorModel:
    """Items half-step, then users (factor.py:550-555)."""
    als_half_step(model, train, "items", lam, weights, threads, reg=reg, device=device)
    als_half_step(model, train, "users", lam, weights, threads, reg=reg, device=device)
    return model


def als_objective(model: FactorModel, data: Dataset, lam: float,
                  weights: np.ndarray | None = None) -> float:
    """sum w (r - q.p)^2 + lam (|P|^2 + |Q|^2) (factor.py:541-547), float64
    on the host (a metric, not the hot path)."""
    P, Q = _host(model.p), _host(model.q)
    pred = np.einsum("nd,nd->n", Q[data.items], P[data.users])
    w = np.ones(len(data)) if weights is None else np.asarray(weights, dtype=np.float64)
    err = float((w * (np.asarray(data.scores, np.float64) - pred) ** 2).sum())
    return err + lam * float((P ** 2).sum() + (Q ** 2).sum())


def predict_batch(model: FactorModel, users, items, times=None, context=None,
                  device=None) -> np.ndarray:
    """q_i . p_u with the reference's cold-start rule (unknown ids keep only
    the known terms, all zero for ALS); unclipped (factor.py:222-242)."""
    dev = cuda_device(device if device is not None else
                      (model.engine.device if model.engine is not None else None))
    u = torch.as_tensor(np.asarray(users, dtype=np.int64).astype(np.int32), device=dev)
    i = torch.as_tensor(np.asarray(items, dtype=np.int64).astype(np.int32), device=dev)
    eng = model.engine
    if eng is None:
        eng = _standalone_engine(model, dev)
    pred, _ = eng.predict(u, i, mu=model.mu)
    return pred.double().cpu().numpy()


def _standalone_engine(model: FactorModel, dev) -> AlsEngine:
    """Engine over an empty split, for prediction from host factors."""
    empty = np.zeros(0, np.int32)
    r = DeviceRatings(empty, empty, np.zeros(0, np.float32), model.num_users, model.num_items, dev)
    eng = AlsEngine(r, model.D)
    eng.set_factors(_host(model.p), _host(model.q))
    model.engine = eng
    return eng


# ---------------------------------------------------------------------------
# training driver

@dataclass
class EpochStats:
    epoch: int
    gamma: float
    objective: float
    valid_rmse: float


def sharded_world(devices) -> int:
    """World size of a devices= request: 1 (single GPU) or N > 1, which needs
    an initialised torch.distributed group of exactly N ranks (one process
    per GPU)."""
    if devices is None:
        return 1
    n = len(devices) if isinstance(devices, (list, tuple)) else int(devices)
    if n <= 1:
        return 1
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() != n:
        raise ConfigError(
            f"devices={n}: the sharded fit runs one process per GPU -- launch {n} ranks "
            f"(torchrun --nproc-per-node {n}), init_process_group('nccl'), and call "
            f"train(..., devices={n}) on every rank")
    return n


def train(kind: str, train_data: Dataset, validation: Dataset | None, hyper: HyperParams,
          threads: int = 1, seed: int = 0, binner=None, weights: np.ndarray | None = None,
          num_users: int | None = None, num_items: int | None = None, *, reg: str | None = None,
          init=None, device=None, as_torch: bool = False, objective: bool = True,
          devices=None, collective: str = "nccl") -> tuple[FactorModel, list[EpochStats]]:
    """hyper.iters ALS sweeps from a seeded (or given) initialisation; one
    EpochStats row per sweep with the training objective and the clipped
    validation RMSE (factor.py:595-618).  Factors, layouts and the
    validation split stay resident on the GPU for the whole run; one host
    synchronisation per sweep reads the metrics."""
    if kind not in ALS_KINDS:
        default_hyper(kind)
    hyper = dataclasses.replace(hyper)
    reg = reg or "plain"
    if weights is not None:
        weights = np.asarray(weights, dtype=np.float64)
        if np.any(weights < 0):
            raise ConfigError("observation weights must be >= 0")
        if weights.size != len(train_data):
            raise ShapeError(f"expected {len(train_data)} weights, got {weights.size}")
    if init is not None:
        # given factors replace the seeded draw (no host RNG pass over U+I rows)
        P0, Q0 = init
        U = num_users if num_users is not None else train_data.num_users
        I = num_items if num_items is not None else train_data.num_items
        if tuple(P0.shape) != (U, hyper.D) or tuple(Q0.shape) != (I, hyper.D):
            raise ShapeError(f"init factors must be ({U}, {hyper.D}) and ({I}, {hyper.D})")
        model = FactorModel(kind, 0.0, np.zeros(U), np.zeros(I), P0, Q0, hyper.D, seed,
                            train_data.scale)
    else:
        model = init_model(kind, train_data, hyper, seed, num_users=num_users,
                           num_items=num_items)
    world = sharded_world(devices)
    if world > 1:
        if weights is not None:
            raise ConfigError("per-observation weights are not supported by the sharded fit")
        return _train_sharded(model, train_data, validation, hyper, reg, init, device, as_torch,
                              objective, collective)
    eng = _engine_for(model, train_data, device, keep_perm=weights is not None)
    if init is not None:
        # uploaded as given (fp32 stays fp32; a pinned source copies asynchronously)
        eng.set_factors(P0, Q0)
    else:
        eng.set_factors(model.p, model.q)
    eng.set_weights(weights)
    lam_c, lam_n = _lam_pair(hyper.lam, reg)
    dev = eng.device
    vu = vi = vs = None
    if validation is not None and len(validation):
        vu = torch.as_tensor(validation.users.astype(np.int32), device=dev)
        vi = torch.as_tensor(validation.items.astype(np.int32), device=dev)
        vs = torch.as_tensor(validation.scores.astype(np.float32), device=dev)
    report: list[EpochStats] = []
    fused = objective and eng.fused_objective
    obj_buf = torch.zeros(4, dtype=torch.float64, device=dev) if fused else None
    for ep in range(hyper.iters):
        eng.sweep(lam_c, lam_n, obj_buf)
        model.epochs_done += 1
        obj = None
        if fused:
            obj = eng.sweep_objective(obj_buf)      # computed in the solve epilogue
        elif objective:
            obj = eng.objective(hyper.lam, reg)
        rm = eng.rmse(vu, vi, vs, (train_data.scale.lo, train_data.scale.hi)) if vu is not None else None
        obj_v, rm_v = eng.check_with(obj, rm)     # one host sync per sweep
        report.append(EpochStats(ep, hyper.gamma,
                                 float(obj_v) if obj_v is not None else float("nan"),
                                 float(rm_v) if rm_v is not None else float("nan")))
    if as_torch:
        model.p, model.q = eng.factors()
    else:
        _sync_host(model)
    return model, report


def _train_sharded(model: FactorModel, train_data: Dataset, validation, hyper: HyperParams,
                   reg: str, init, device, as_torch: bool, objective: bool, collective: str):
    """train() with rows sharded over the ranks of the default process group
    (parallel.ShardedAls): each rank solves its nnz-balanced row ranges and the
    solved rows are all-gathered after every half-step.  Per sweep, the
    objective terms are summed over ranks and failures reduced to the minimum
    global row (one host synchronisation); the held-out RMSE is evaluated on
    every rank from the replicated factors."""
    import torch.distributed as dist

    from .parallel import ShardedAls
    dev = cuda_device(device if device is not None else
                      torch.device("cuda", torch.cuda.current_device()))
    lam_c, lam_n = _lam_pair(hyper.lam, reg)
    U, I, D = model.num_users, model.num_items, model.D
    run = ShardedAls(train_data.users, train_data.items, train_data.scores, U, I, D,
                     device=dev, collective=collective)
    P0, Q0 = (init if init is not None else (model.p, model.q))
    run.set_factors(P0, Q0)
    ev = _standalone_engine_for(U, I, D, dev)
    vu = vi = vs = None
    if validation is not None and len(validation):
        vu = torch.as_tensor(validation.users.astype(np.int32), device=dev)
        vi = torch.as_tensor(validation.items.astype(np.int32), device=dev)
        vs = torch.as_tensor(validation.scores.astype(np.float32), device=dev)
    fused = objective and D <= 20
    obj_buf = torch.zeros(4, dtype=torch.float64, device=dev) if fused else None
    report: list[EpochStats] = []
    for ep in range(hyper.iters):
        run.sweep(lam_c, lam_n, obj_buf)
        model.epochs_done += 1
        terms = torch.zeros(1, dtype=torch.float64, device=dev)
        if fused:
            terms = obj_buf[2:3] + obj_buf[3:4] + obj_buf[1:2]   # my rows' share
        elif objective:
            terms = _sharded_objective(run, ev, hyper.lam, reg)
        dist.all_reduce(terms)
        run.check()                                            # all-reduce MIN of failures
        rm = None
        if vu is not None:
            _, sse = ev.predict(vu, vi, vs, want_pred=False, P=run.P, Q=run.Q,
                                clip=(train_data.scale.lo, train_data.scale.hi))
            rm = torch.sqrt(sse / vu.numel())
        vals = torch.cat([terms, rm if rm is not None else terms]).tolist()
        report.append(EpochStats(ep, hyper.gamma, float(vals[0]) if objective else float("nan"),
                                 float(vals[1]) if rm is not None else float("nan")))
    P, Q = run.factors()
    ev.set_factors(P, Q)
    model.engine = ev
    if as_torch:
        model.p, model.q = ev.factors()
    else:
        model.p, model.q = P.double().cpu().numpy(), Q.double().cpu().numpy()
    return model, report


def _standalone_engine_for(U: int, I: int, D: int, dev) -> AlsEngine:
    empty = np.zeros(0, np.int32)
    return AlsEngine(DeviceRatings(empty, empty, np.zeros(0, np.float32), U, I, dev), D)


def _sharded_objective(run, ev: AlsEngine, lam: float, reg: str) -> torch.Tensor:
    """This rank's share of the objective: the data term over its users'
    ratings and the regulariser of its own rows (D > 20, no fused epilogue)."""
    lay_u, lay_i = run.local["users"], run.local["items"]
    ulo, uhi = run.umap.range(run.rank)
    ilo, ihi = run.imap.range(run.rank)
    rows = ulo + torch.repeat_interleave(
        torch.arange(lay_u.n_rows, device=run.device, dtype=torch.int32), lay_u.degrees())
    _, sse = ev.predict(rows.to(torch.int32), lay_u.idx, lay_u.val, want_pred=False, P=run.P,
                        Q=run.Q, clip=(-3.0e38, 3.0e38))
    wu = lay_u.ptr if reg == "weighted" else None
    wi = lay_i.ptr if reg == "weighted" else None
    reg_t = ev.sq_norms(run.P[ulo:uhi], wu) + ev.sq_norms(run.Q[ilo:ihi], wi)
    return sse + lam * reg_t
