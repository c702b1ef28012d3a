"""MFITR (matrix factorisation with item-taxonomy regularisation) on device.

Drop-in names from the reference's ``multicf.mfitr`` (reference
pkg/src/multicf/mfitr.py:29-59 MfitrHyper, :62-89 edge weights, :92-149
model/init, :181-197 predict_batch, :219-242 graph_penalty/loss_mfitr,
:347-371 train_mfitr).

The reference trains MFITR only by SGD (mfitr.py:323-336).  This path is
the ALS-MFITR solver recommended by SURVEY.md §8(a): block-coordinate
descent on ``loss_mfitr`` (time terms off) with

* the item half-step solved layer by layer -- tracks, albums, artists, then
  every other item -- each layer's rows exactly:
      (sum_u p_u p_u^T + lam2 n_i I + tau S_i I) q_i = sum_u (r - mu) p_u + tau T_i
  with tau = lam3 + lam4 and S_i = sum w_e, T_i = sum w_e q_other over the
  item's taxonomy edges (mcf_taxonomy_terms on the current Q).  No edge joins
  two items of one layer (track < album < artist layering,
  taxonomy.py:102-103), so each layer solve zeroes grad_mfitr on its rows;
* the user half-step with the same per-observation lam2 (lam2 n_u I);
* minimum scope: mu = train mean fixed, user/item/artist biases and the
  artist factors q_a frozen at 0 (the (D+1)-augmented bias blocks are the
  next step).  gamma / decay are unused by this solver.
"""
from __future__ import annotations

import dataclasses
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr
from .data import Dataset
from .device import AlsEngine, cuda_device, stream_ptr
from .errors import ConfigError, DivergenceError
from .factor import EpochStats, FactorModel, _host, _ratings_for
from .taxonomy import TaxonomyGraph

MFITR_KINDS = ("mfitr", "time-mfitr")


@dataclass
class MfitrHyper:
    gamma: float = 8e-5
    decay: float = 0.95
    lam1: float = 1e-5
    lam2: float = 1e-4
    lam3: float = 1e-3
    lam4: float = 1e-3
    lam5: float = 1e-3
    iters: int = 50
    D: int = 50
    D_t: int = 8

    def __post_init__(self):
        if self.gamma <= 0:
            raise ConfigError("gamma must be > 0")
        if not 0 < self.decay <= 1:
            raise ConfigError("decay must be in (0, 1]")
        if min(self.lam1, self.lam2, self.lam3, self.lam4, self.lam5) < 0:
            raise ConfigError("regularisation weights must be >= 0")
        if self.iters < 0:
            raise ConfigError("iters must be >= 0")
        if self.D < 1 or self.D_t < 1:
            raise ConfigError("factor dimensions must be >= 1")


def default_mfitr_hyper(kind: str = "mfitr") -> MfitrHyper:
    if kind not in MFITR_KINDS:
        raise ConfigError(f"unknown taxonomy model kind {kind!r}")
    if kind == "time-mfitr":
        raise ConfigError("time-mfitr is outside the device path (no time terms)")
    return MfitrHyper()


@dataclass
class TaxonomyEdgeWeights:
    edge_child: np.ndarray
    edge_parent: np.ndarray
    w: np.ndarray

    def weight(self, i: int, j: int) -> float:
        hit = np.flatnonzero((self.edge_child == i) & (self.edge_parent == j))
        if hit.size == 0:
            raise KeyError(f"({i}, {j}) is not a taxonomy edge")
        return float(self.w[hit[0]])


def edge_weights(graph: TaxonomyGraph, train: Dataset, means=None, device=None,
                 num_items: int | None = None) -> TaxonomyEdgeWeights:
    """max(0, adjusted cosine) per taxonomy edge, computed on device and
    bit-identical to the reference (mcf_edge_weights; mfitr.py:78-89)."""
    if means is not None:
        raise ConfigError("custom user means are not supported on the device path")
    n_items = num_items if num_items is not None else max(train.num_items, graph.num_nodes)
    r = _ratings_for(train, device, False, train.num_users, n_items)
    dev = r.device
    E = graph.num_edges
    w = torch.zeros(E, dtype=torch.float64, device=dev)
    if E:
        ec = torch.as_tensor(graph.edge_child.astype(np.int32), device=dev)
        ep = torch.as_tensor(graph.edge_parent.astype(np.int32), device=dev)
        lay = r.by_user
        L = _lib.lib()
        ws = torch.empty(int(L.mcf_edge_weights_workspace_bytes(lay.nnz, r.num_users, n_items)),
                         dtype=torch.uint8, device=dev)
        check(L.mcf_edge_weights(ptr(lay.ptr), ptr(lay.idx), ptr(lay.val), r.num_users, n_items,
                                 ptr(ec), ptr(ep), E, ptr(w), ptr(ws), ws.numel(),
                                 stream_ptr(dev)), "mcf_edge_weights")
    return TaxonomyEdgeWeights(graph.edge_child, graph.edge_parent, w.cpu().numpy())


@dataclass
class MfitrModel:
    base: FactorModel
    b_a: np.ndarray
    q_a: np.ndarray
    artist_of_item: np.ndarray = field(repr=False)

    @property
    def kind(self) -> str:
        return "mfitr"

    @property
    def mu(self) -> float:
        return self.base.mu

    @property
    def scale(self):
        return self.base.scale

    @property
    def num_users(self) -> int:
        return self.base.num_users

    @property
    def num_items(self) -> int:
        return self.base.num_items

    def check_finite(self, epoch: int) -> None:
        self.base.check_finite(epoch)
        for name, arr in (("b_a", self.b_a), ("q_a", self.q_a)):
            if not np.isfinite(_host(arr)).all():
                raise DivergenceError(epoch, f"non-finite {name} after epoch {epoch}")


def init_mfitr(kind: str, train: Dataset, graph: TaxonomyGraph, hyper: MfitrHyper, seed: int,
               binner=None, num_users: int | None = None,
               num_items: int | None = None) -> MfitrModel:
    """Reference draw order (mfitr.py:133-149, factor.py:144-147): q then p
    ~ U(+-0.005/sqrt(D)) from default_rng([seed, 1]), mu = train mean,
    q_a ~ U from default_rng([seed, 3]); biases zero."""
    if kind not in MFITR_KINDS:
        raise ConfigError(f"unknown taxonomy model kind {kind!r}")
    U = num_users if num_users is not None else train.num_users
    I = num_items if num_items is not None else max(train.num_items, graph.num_nodes)
    D = hyper.D
    rng = np.random.default_rng([seed, 1])
    amp = 0.005 / np.sqrt(D)
    q = rng.uniform(-amp, amp, (I, D))
    p = rng.uniform(-amp, amp, (U, D))
    base = FactorModel("mfitr", train.global_mean(), np.zeros(U), np.zeros(I), p, q, D, seed,
                       train.scale)
    q_a = np.random.default_rng([seed, 3]).uniform(-amp, amp, (I, D))
    return MfitrModel(base, np.zeros(I), q_a, graph.artist_array(I))


def predict_batch(model: MfitrModel, users, items, times=None, device=None) -> np.ndarray:
    """mu + b_u + b_i + b_a + (q_i + q_a[art(i)]) . p_u, cold-start rules of
    the reference (mfitr.py:181-197, _kernels.py:344-375); unclipped."""
    base = model.base
    eng = base.engine
    dev = cuda_device(device if device is not None else (eng.device if eng else None))
    if eng is None:
        z = np.zeros(0, np.int32)
        from .device import DeviceRatings
        r = DeviceRatings(z, z, np.zeros(0, np.float32), base.num_users, base.num_items, dev)
        eng = AlsEngine(r, base.D)
        eng.set_factors(_host(base.p), _host(base.q))
        base.engine = eng
    D, ld = base.D, eng.ld
    f32 = lambda a: torch.as_tensor(np.asarray(_host(a), np.float32), device=dev)  # noqa: E731
    qa = torch.zeros(base.num_items, ld, dtype=torch.float32, device=dev)
    qa[:, :D] = f32(model.q_a)
    u = torch.as_tensor(np.asarray(users, np.int64).astype(np.int32), device=dev)
    i = torch.as_tensor(np.asarray(items, np.int64).astype(np.int32), device=dev)
    art = torch.as_tensor(model.artist_of_item.astype(np.int32), device=dev)
    pred, _ = eng.predict(u, i, mu=base.mu, b_u=f32(base.b_u), b_i=f32(base.b_i), art=art,
                          b_a=f32(model.b_a), Q_a=qa)
    return pred.double().cpu().numpy()


class MfitrSolver:
    """Device state of one ALS-MFITR fit: engine, incident-edge CSR, edge
    weights, layer row lists, S/T buffers."""

    def __init__(self, engine: AlsEngine, graph: TaxonomyGraph, w: np.ndarray, hyper: MfitrHyper,
                 mu: float):
        dev = engine.device
        self.eng, self.hyper, self.mu = engine, hyper, float(mu)
        I = engine.r.num_items
        inc_ptr, inc_edge, inc_other = graph.incident_edges(I)
        self.inc_ptr = torch.as_tensor(inc_ptr, device=dev)
        self.inc_edge = torch.as_tensor(inc_edge.astype(np.int32), device=dev)
        self.inc_other = torch.as_tensor(inc_other.astype(np.int32), device=dev)
        self.w = torch.as_tensor(np.asarray(w, np.float32), device=dev)
        self.w64 = torch.as_tensor(np.asarray(w, np.float64), device=dev)
        self.ec = torch.as_tensor(graph.edge_child, device=dev)
        self.ep = torch.as_tensor(graph.edge_parent, device=dev)
        self.layers = [torch.as_tensor(L.astype(np.int32), device=dev)
                       for L in graph.layers(I)]
        self.S = torch.zeros(I, dtype=torch.float32, device=dev)
        self.T = torch.zeros(I, engine.ld, dtype=torch.float32, device=dev)
        self.tau = hyper.lam3 + hyper.lam4

    def solve_layer(self, k: int):
        """Layer k of the item half-step: S/T from the current Q, then the
        layer's rows solved exactly."""
        eng, h = self.eng, self.hyper
        rows = self.layers[k]
        if rows.numel() == 0:
            return
        check(_lib.lib().mcf_taxonomy_terms(ptr(self.inc_ptr), ptr(self.inc_edge),
                                            ptr(self.inc_other), ptr(self.w), ptr(eng.Q),
                                            eng.r.num_items, eng.D, ptr(rows), rows.numel(),
                                            ptr(self.S), ptr(self.T), stream_ptr(eng.device)),
              "mcf_taxonomy_terms")
        eng.half_step("items", 0.0, h.lam2, self.mu, self.S, self.T, self.tau, rows=rows,
                      rows_key=("layer", k))

    def item_layers(self):
        for k in range(len(self.layers)):
            self.solve_layer(k)

    def users(self):
        self.eng.half_step("users", 0.0, self.hyper.lam2, self.mu)

    def sweep(self):
        self.item_layers()
        self.users()

    def loss(self) -> torch.Tensor:
        """loss_mfitr with biases/q_a at 0 and time off (mfitr.py:219-242)."""
        eng, h = self.eng, self.hyper
        lay = eng.r.by_user
        if getattr(eng, "_rows_of_records", None) is None:
            eng._rows_of_records = torch.repeat_interleave(
                torch.arange(eng.r.num_users, device=eng.device, dtype=torch.int32),
                lay.degrees())
        _, sse = eng.predict(eng._rows_of_records, lay.idx, lay.val, want_pred=False,
                             mu=self.mu, clip=(-3.0e38, 3.0e38))
        reg = eng.sq_norms(eng.P, eng.r.by_user.ptr) + eng.sq_norms(eng.Q, eng.r.by_item.ptr)
        Q = eng.Q[:, : eng.D].double()
        d2 = ((Q[self.ec] - Q[self.ep]) ** 2).sum(1)
        graph = self.tau * (self.w64 * d2).sum()
        return sse + h.lam2 * reg + graph


class MfitrFullSolver:
    """Every MFITR parameter block on device (time terms off), SURVEY §8(f)1:
    block-coordinate descent on loss_mfitr (mfitr.py:226-242) over augmented
    unknowns [f | b] (factor columns 0..D-1, bias in column D):

      items   [q_i | b_i] layer by layer (tracks, albums, artists, rest; no
              edge joins two items of one layer, taxonomy.py:102-103), with
              the taxonomy term on q only;
      artists [q_a | b_a] over the ratings of each artist's items (q_a, b_a
              indexed by the artist's item id, mfitr.py:92-149);
      users   [p_u | b_u].

    Each block is one exact least-squares solve (mcf_als_half_step_bias):
    lam2 * n on the factor coordinates and lam1 * n on the bias -- the
    per-observation regularisers of loss_mfitr -- with the block's fixed
    terms folded into per-rating targets (mcf_mfitr_targets) and the
    gathered rows [x | 1] built by mcf_mfitr_fixed.  mu stays the train mean
    (the reference never updates mu, mfitr.py:142 / factor.py:161)."""

    def __init__(self, ratings, graph: TaxonomyGraph, w: np.ndarray, hyper: MfitrHyper, mu: float,
                 art: np.ndarray, P0, Q0, Qa0=None, b_u=None, b_i=None, b_a=None,
                 chunk: int | None = None):
        from .device import LayoutSolver, SideLayout
        dev = ratings.device
        self.r, self.hyper, self.mu, self.device = ratings, hyper, float(mu), dev
        U, I, D = ratings.num_users, ratings.num_items, int(hyper.D)
        self.U, self.I, self.D = U, I, D
        self.ld = _lib.factor_ld(D + 1)
        z = lambda n: torch.zeros(n, self.ld, dtype=torch.float32, device=dev)  # noqa: E731
        self.Pa, self.Qa, self.Aa = z(U), z(I), z(I)
        f32 = lambda a: torch.as_tensor(np.asarray(_host(a), np.float32), device=dev)  # noqa: E731
        self.Pa[:, :D] = f32(P0)
        self.Qa[:, :D] = f32(Q0)
        if Qa0 is not None:
            self.Aa[:, :D] = f32(Qa0)
        for t, b in ((self.Pa, b_u), (self.Qa, b_i), (self.Aa, b_a)):
            if b is not None:
                t[:, D] = f32(b)
        self.art_np = np.asarray(art, np.int64)
        self.art = torch.as_tensor(self.art_np.astype(np.int32), device=dev)
        self.Xu, self.Xi = z(U), z(I)
        self.t_items = torch.empty(ratings.nnz, dtype=torch.float32, device=dev)
        # item id of every rating of the items layout (the targets kernel runs
        # thread per rating)
        self.item_rows = torch.repeat_interleave(torch.arange(I, device=dev, dtype=torch.int32),
                                                 ratings.by_item.degrees())
        self.t_users = torch.empty(ratings.nnz, dtype=torch.float32, device=dev)
        lay = ratings.by_user
        # fused item / artist steps (D + 1 <= 21, the Schur pair path): the item
        # layers emit their row systems and drop the artist terms from their rhs
        # through their own Gram; the artist block is solved from the emitted
        # systems (mcf_mfitr_artist_step) -- no per-rating artist passes
        self.fused = (D + 1 <= 21 and not os.environ.get("MCF_MFITR_LEGACY")
                      and not os.environ.get("MCF_NO_SCHUR"))
        has_i = self.art >= 0
        deg_i = ratings.by_item.degrees()
        cnt = torch.zeros(I, dtype=torch.int64, device=dev)
        cnt.index_add_(0, self.art[has_i].long(), deg_i[has_i])
        self.cnt_a = cnt.double()
        if self.fused:
            self.cnt_ptr = torch.zeros(I + 1, dtype=torch.int64, device=dev)
            self.cnt_ptr[1:] = torch.cumsum(cnt, 0)
            items = torch.nonzero(has_i).flatten()
            order = torch.argsort(self.art[items].long(), stable=True)
            self.art_items = items[order].to(torch.int32).contiguous()
            arts_sorted = self.art[self.art_items.long()].long()
            self.artist_row, counts = torch.unique_consecutive(arts_sorted, return_counts=True)
            self.artist_row = self.artist_row.to(torch.int32).contiguous()
            self.art_ptr = torch.zeros(self.artist_row.numel() + 1, dtype=torch.int64, device=dev)
            self.art_ptr[1:] = torch.cumsum(counts, 0)
            self.emit = torch.zeros(I, 256, dtype=torch.float32, device=dev)
            # rows of q_a / b_a that are not an artist have no ratings: the
            # block solve leaves them 0 (the per-rating path does the same)
            not_artist = torch.ones(I, dtype=torch.bool, device=dev)
            not_artist[self.artist_row.long()] = False
            self.not_artist = torch.nonzero(not_artist).flatten()
            n_art = int(self.artist_row.numel())
            self.art_ws = torch.empty(max(int(_lib.lib().mcf_mfitr_artist_workspace_bytes(n_art)),
                                          256), dtype=torch.uint8, device=dev)
        else:
            # artist layout: the records whose item has an artist, keyed by
            # artist, partner = user, aux = item (records rebuilt from the users layout)
            rec_u = torch.repeat_interleave(torch.arange(U, device=dev, dtype=torch.int32),
                                            lay.degrees())
            rec_i, rec_s = lay.idx, lay.val
            a_of = self.art[rec_i.long()]
            has = a_of >= 0
            hu, hi, hs, ha = rec_u[has], rec_i[has], rec_s[has], a_of[has]
            self.by_artist = SideLayout(ha.contiguous(), hu.contiguous(), hs.contiguous(), I,
                                        keep_perm=True)
            self.art_item = hi[self.by_artist.perm.long()].contiguous()
            self.t_art = torch.empty(self.by_artist.nnz, dtype=torch.float32, device=dev)
        self.cnt_u = lay.degrees().double()
        self.cnt_i = deg_i.double()
        # taxonomy
        inc_ptr, inc_edge, inc_other = graph.incident_edges(I)
        self.inc_ptr = torch.as_tensor(inc_ptr, device=dev)
        self.inc_edge = torch.as_tensor(inc_edge.astype(np.int32), device=dev)
        self.inc_other = torch.as_tensor(inc_other.astype(np.int32), device=dev)
        self.w = torch.as_tensor(np.asarray(w, np.float32), device=dev)
        self.w64 = torch.as_tensor(np.asarray(w, np.float64), device=dev)
        self.ec = torch.as_tensor(graph.edge_child, device=dev)
        self.ep = torch.as_tensor(graph.edge_parent, device=dev)
        self.layers = [torch.as_tensor(L.astype(np.int32), device=dev) for L in graph.layers(I)]
        self.S = torch.zeros(I, dtype=torch.float32, device=dev)
        self.T = torch.zeros(I, self.ld, dtype=torch.float32, device=dev)
        self.tau = hyper.lam3 + hyper.lam4
        self.solver = LayoutSolver(D + 1, chunk)
        self.fail = torch.full((1,), -1, dtype=torch.int64, device=dev)
        # every solve resets `fail`; the first failing row of each block
        # (items layers, artists, users) since the last check() is kept here
        self._fail_acc = torch.full((3,), -1, dtype=torch.int64, device=dev)

    BLOCKS = ("items", "artists", "users")

    def _fold(self, block: int):
        acc = self._fail_acc[block:block + 1]
        torch.where(acc < 0, self.fail, acc, out=acc)

    def _bias(self):
        return (self.D, 0.0, self.hyper.lam1)

    def _fixed(self, main, add, art, n, out):
        check(_lib.lib().mcf_mfitr_fixed(ptr(main), ptr(add), ptr(art), n, self.D, ptr(out),
                                         stream_ptr(self.device)), "mcf_mfitr_fixed")

    def _targets(self, mode, lay, aux, out):
        check(_lib.lib().mcf_mfitr_targets(mode, ptr(lay.ptr), ptr(lay.idx), ptr(lay.val),
                                           ptr(aux), lay.n_rows, ptr(self.Pa), ptr(self.Qa),
                                           ptr(self.Aa), ptr(self.art), self.mu, self.D, ptr(out),
                                           stream_ptr(self.device)), "mcf_mfitr_targets")

    def _fixed_bsub(self, main, add, art, n, out):
        check(_lib.lib().mcf_mfitr_fixed_bsub(ptr(main), ptr(add), ptr(art), n, self.D, ptr(out),
                                              stream_ptr(self.device)), "mcf_mfitr_fixed_bsub")

    def _item_prep(self):
        # [p_u | 1] and the item targets depend only on user / artist blocks
        if self.fused:   # [p_u | 1 | b_u]: the targets are formed in the solve's gather
            self._fixed_bsub(self.Pa, None, None, self.U, self.Xu)
            return
        self._fixed(self.Pa, None, None, self.U, self.Xu)
        self._targets(1, self.r.by_item, self.item_rows, self.t_items)

    def item_layers(self):
        self._item_prep()
        for k in range(len(self.layers)):
            self._solve_layer(k)

    def item_layer(self, k: int):
        """One taxonomy layer on its own (tests / diagnostics)."""
        self._item_prep()
        self._solve_layer(k)

    def _solve_layer(self, k: int):
        L, h = _lib.lib(), self.hyper
        rows = self.layers[k]
        if rows.numel():
            check(L.mcf_taxonomy_terms(ptr(self.inc_ptr), ptr(self.inc_edge), ptr(self.inc_other),
                                       ptr(self.w), ptr(self.Qa), self.I, self.D + 1, ptr(rows),
                                       rows.numel(), ptr(self.S), ptr(self.T),
                                       stream_ptr(self.device)), "mcf_taxonomy_terms")
            if self.fused:   # raw ratings - mu - b_u (gather); artist terms from the Gram
                self.solver.solve(self.r.by_item, self.Xu, self.Qa, 0.0, h.lam2, self.mu, self.S,
                                  self.T, self.tau, rows, ("layer", k), None, self.fail, None,
                                  bias=self._bias(), emit=(self.emit, self.Aa, self.art, True))
            else:
                self.solver.solve(self.r.by_item, self.Xu, self.Qa, 0.0, h.lam2, 0.0, self.S,
                                  self.T, self.tau, rows, ("layer", k), None, self.fail, None,
                                  val=self.t_items, bias=self._bias())
            self._fold(0)

    def artists(self):
        if self.fused:   # from the item layers' emitted systems
            check(_lib.lib().mcf_mfitr_artist_step(
                ptr(self.art_ptr), ptr(self.art_items), ptr(self.artist_row),
                int(self.artist_row.numel()), ptr(self.cnt_ptr), ptr(self.emit), ptr(self.Qa),
                ptr(self.Aa), self.D + 1, float(self.hyper.lam2), float(self.hyper.lam1),
                ptr(self.fail), ptr(self.art_ws), self.art_ws.numel(), stream_ptr(self.device)),
                "mcf_mfitr_artist_step")
            self.Aa.index_fill_(0, self.not_artist, 0.0)
            self._fold(1)
            return
        self._fixed(self.Pa, None, None, self.U, self.Xu)
        self._targets(2, self.by_artist, self.art_item, self.t_art)
        self.solver.solve(self.by_artist, self.Xu, self.Aa, 0.0, self.hyper.lam2, fail=self.fail,
                          val=self.t_art, bias=self._bias())
        self._fold(1)

    def users(self):
        if self.fused:   # [q_i + q_a | 1 | b_i + b_a]: targets formed in the gather
            self._fixed_bsub(self.Qa, self.Aa, self.art, self.I, self.Xi)
            self.solver.solve(self.r.by_user, self.Xi, self.Pa, 0.0, self.hyper.lam2, self.mu,
                              fail=self.fail, bias=self._bias(), emit=(None, None, None, True))
            self._fold(2)
            return
        self._fixed(self.Qa, self.Aa, self.art, self.I, self.Xi)
        self._targets(0, self.r.by_user, None, self.t_users)
        self.solver.solve(self.r.by_user, self.Xi, self.Pa, 0.0, self.hyper.lam2, fail=self.fail,
                          val=self.t_users, bias=self._bias())
        self._fold(2)

    def sweep(self):
        self.item_layers()
        self.artists()
        self.users()

    def check(self):
        """Raise SingularSystemError for the first block (in sweep order)
        that had a failing row since the last check."""
        rows = [int(x) for x in self._fail_acc.tolist()]
        self._fail_acc.fill_(-1)
        for block, row in zip(self.BLOCKS, rows):
            if row >= 0:
                from .errors import SingularSystemError
                raise SingularSystemError(f"singular MFITR block system at {block} row {row}")

    def params(self):
        """(P, Q, b_u, b_i, b_a, Q_a) device views."""
        D = self.D
        return (self.Pa[:, :D], self.Qa[:, :D], self.Pa[:, D], self.Qa[:, D], self.Aa[:, D],
                self.Aa[:, :D])

    def _predictor(self):
        pe = getattr(self, "_pe", None)
        if pe is None:
            from .device import DeviceRatings
            z = torch.zeros(0, dtype=torch.int32, device=self.device)
            pe = self._pe = AlsEngine(DeviceRatings(z, z, z.float(), self.U, self.I, self.device),
                                      self.D)
            pe.Qa_t = torch.zeros_like(pe.Q)
        P, Q, _, _, _, Qa = self.params()
        pe.P[:, : self.D] = P
        pe.Q[:, : self.D] = Q
        pe.Qa_t[:, : self.D] = Qa
        return pe

    def predict(self, users, items, truth=None, clip=(-3.0e38, 3.0e38)):
        """(pred, sse) of the full model through mcf_predict_sse."""
        pe = self._predictor()
        bu, bi, ba = (x.contiguous() for x in self.params()[2:5])
        return pe.predict(users, items, truth, want_pred=truth is None, mu=self.mu, b_u=bu, b_i=bi,
                          art=self.art, b_a=ba, Q_a=pe.Qa_t, clip=clip)

    def loss(self) -> torch.Tensor:
        """loss_mfitr with time off (mfitr.py:226-242), on device: the data
        term through mcf_predict_sse, the per-observation regularisers as
        count-weighted squared norms, the graph term over the edges."""
        h, D = self.hyper, self.D
        lay = self.r.by_user
        P, Q, bu, bi, ba, Qa = self.params()
        rec_u = getattr(self, "_rec_u", None)
        if rec_u is None:
            rec_u = self._rec_u = torch.repeat_interleave(
                torch.arange(self.U, device=self.device, dtype=torch.int32), lay.degrees())
        _, sse = self.predict(rec_u, lay.idx, lay.val)
        d = lambda x: x.double()  # noqa: E731
        reg1 = ((self.cnt_u * d(bu) ** 2).sum() + (self.cnt_i * d(bi) ** 2).sum()
                + (self.cnt_a * d(ba) ** 2).sum())
        reg2 = ((self.cnt_u * (d(P) ** 2).sum(1)).sum() + (self.cnt_i * (d(Q) ** 2).sum(1)).sum()
                + (self.cnt_a * (d(Qa) ** 2).sum(1)).sum())
        d2 = ((d(Q)[self.ec] - d(Q)[self.ep]) ** 2).sum(1)
        return sse + h.lam1 * reg1 + h.lam2 * reg2 + self.tau * (self.w64 * d2).sum()


def train_mfitr_sgd(kind: str, train_data: Dataset, validation: Dataset | None,
                    graph: TaxonomyGraph, hyper: MfitrHyper, seed: int = 0,
                    ew: TaxonomyEdgeWeights | None = None, num_users: int | None = None,
                    num_items: int | None = None, *, device=None, objective: bool = True,
                    workers: int = 0, conflicts: str = "locks") -> tuple[MfitrModel, list[EpochStats]]:
    """The reference's own MFITR trainer on device:
    mfitr.train_mfitr (mfitr.py:347-371) with sgd_epoch_mfitr per epoch --
    the same seeded init (init_mfitr), the same per-epoch user shuffle
    (default_rng([seed, 2]), factor.py:166, 408), rate_update over each
    user's ratings then the edge pass (mcf_mfitr_sgd_epoch, Hogwild across
    users), gamma *= decay after every epoch; one EpochStats row per epoch
    with loss_mfitr and the clipped validation RMSE.  workers: concurrent
    user warps -- 0 (default) the whole GPU, 1 the reference's single-thread
    order exactly.  conflicts: "locks" (default) keeps the reference's
    LockTable contract across concurrent users (one lock per item id, the
    (item, artist) pair in ascending order per rating, both endpoints per
    edge -- parallel.py:21-49, mcf_mfitr_sgd_epoch_locked); "hogwild" updates
    shared item state without locks."""
    if conflicts not in ("locks", "hogwild"):
        raise ConfigError(f"conflicts must be 'locks' or 'hogwild', got {conflicts!r}")
    hyper = dataclasses.replace(hyper)
    model = init_mfitr(kind, train_data, graph, hyper, seed, num_users=num_users,
                       num_items=num_items)
    base = model.base
    r = _ratings_for(train_data, device, False, base.num_users, base.num_items)
    if ew is None:
        ew = edge_weights(graph, train_data, device=r.device, num_items=base.num_items)
    dev = r.device
    D = base.D
    ld = _lib.factor_ld(D)
    f32 = lambda a: torch.as_tensor(np.asarray(_host(a), np.float32), device=dev)  # noqa: E731
    P = torch.zeros(base.num_users, ld, dtype=torch.float32, device=dev)
    Q = torch.zeros(base.num_items, ld, dtype=torch.float32, device=dev)
    Qa = torch.zeros(base.num_items, ld, dtype=torch.float32, device=dev)
    P[:, :D], Q[:, :D], Qa[:, :D] = f32(base.p), f32(base.q), f32(model.q_a)
    bu, bi, ba = f32(base.b_u), f32(base.b_i), f32(model.b_a)
    art = torch.as_tensor(model.artist_of_item.astype(np.int32), device=dev)
    ec = torch.as_tensor(np.asarray(ew.edge_child, np.int64), device=dev)
    ep = torch.as_tensor(np.asarray(ew.edge_parent, np.int64), device=dev)
    w = torch.as_tensor(np.asarray(ew.w, np.float64), device=dev)
    lay = r.by_user
    deg = lay.degrees().cpu().numpy()
    counter = torch.zeros(1, dtype=torch.int32, device=dev)
    locks = (torch.zeros(base.num_items, dtype=torch.int32, device=dev)
             if conflicts == "locks" else None)
    shuffle = np.random.default_rng([seed, 2])
    eng = AlsEngine(r, D)            # prediction / loss helpers
    vu = vi = vs = None
    if validation is not None and len(validation):
        vu = torch.as_tensor(validation.users.astype(np.int32), device=dev)
        vi = torch.as_tensor(validation.items.astype(np.int32), device=dev)
        vs = torch.as_tensor(validation.scores.astype(np.float32), device=dev)
    rec_u = torch.repeat_interleave(torch.arange(base.num_users, device=dev, dtype=torch.int32),
                                    lay.degrees())
    cnt_u, cnt_i = lay.degrees().double(), r.by_item.degrees().double()
    has = art >= 0
    cnt_a = torch.zeros(base.num_items, dtype=torch.float64, device=dev)
    cnt_a.index_add_(0, art[lay.idx.long()][has[lay.idx.long()]].long(),
                     torch.ones(int(has[lay.idx.long()].sum()), dtype=torch.float64, device=dev))
    report = []
    L = _lib.lib()
    for ep_i in range(hyper.iters):
        gamma_used = hyper.gamma
        perm = shuffle.permutation(base.num_users)
        active = perm[deg[perm] > 0].astype(np.int32)
        order = torch.as_tensor(active, device=dev)
        args = (ptr(lay.ptr), ptr(lay.idx), ptr(lay.val), ptr(order), int(order.numel()),
                ptr(counter), ptr(P), ptr(Q), ptr(bu), ptr(bi), ptr(art), ptr(ba), ptr(Qa),
                float(base.mu), D, float(hyper.gamma), float(hyper.lam1), float(hyper.lam2),
                ptr(ec), ptr(ep), ptr(w), int(ec.numel()), float(hyper.lam3), float(hyper.lam4),
                int(workers))
        if locks is not None:
            check(L.mcf_mfitr_sgd_epoch_locked(*args, ptr(locks), stream_ptr(dev)),
                  "mcf_mfitr_sgd_epoch_locked")
        else:
            check(L.mcf_mfitr_sgd_epoch(*args, stream_ptr(dev)), "mcf_mfitr_sgd_epoch")
        base.epochs_done += 1
        hyper.gamma *= hyper.decay
        obj = float("nan")
        if objective:
            _, sse = eng.predict(rec_u, lay.idx, lay.val, want_pred=False, mu=base.mu, b_u=bu,
                                 b_i=bi, art=art, b_a=ba, Q_a=Qa, P=P, Q=Q,
                                 clip=(-3.0e38, 3.0e38))
            d = lambda x: x.double()  # noqa: E731
            reg1 = ((cnt_u * d(bu) ** 2).sum() + (cnt_i * d(bi) ** 2).sum()
                    + (cnt_a * d(ba) ** 2).sum())
            reg2 = ((cnt_u * (d(P[:, :D]) ** 2).sum(1)).sum()
                    + (cnt_i * (d(Q[:, :D]) ** 2).sum(1)).sum()
                    + (cnt_a * (d(Qa[:, :D]) ** 2).sum(1)).sum())
            d2 = ((d(Q[:, :D])[ec] - d(Q[:, :D])[ep]) ** 2).sum(1)
            graph_t = (hyper.lam3 + hyper.lam4) * (w * d2).sum()
            obj = float((sse + hyper.lam1 * reg1 + hyper.lam2 * reg2 + graph_t).item())
        rm = float("nan")
        if vu is not None:
            _, sse = eng.predict(vu, vi, vs, want_pred=False, mu=base.mu, b_u=bu, b_i=bi,
                                 art=art, b_a=ba, Q_a=Qa, P=P, Q=Q,
                                 clip=(train_data.scale.lo, train_data.scale.hi))
            rm = float(torch.sqrt(sse / vu.numel()).item())
        if not (np.isfinite(obj) if objective else True):
            raise DivergenceError(f"MFITR SGD diverged at epoch {ep_i}")
        report.append(EpochStats(ep_i, gamma_used, obj, rm))
    host = lambda t: t.double().cpu().numpy()  # noqa: E731
    base.p, base.q, model.q_a = host(P[:, :D]), host(Q[:, :D]), host(Qa[:, :D])
    base.b_u, base.b_i, model.b_a = host(bu), host(bi), host(ba)
    eng.set_factors(P[:, :D], Q[:, :D])
    base.engine = eng
    model.ew = ew
    return model, report


def train_mfitr(kind: str, train_data: Dataset, validation: Dataset | None,
                graph: TaxonomyGraph, hyper: MfitrHyper, threads: int = 1, seed: int = 0,
                binner=None, ew: TaxonomyEdgeWeights | None = None,
                num_users: int | None = None, num_items: int | None = None, *, init=None,
                device=None, as_torch: bool = False, objective: bool = True,
                blocks: str = "full", method: str = "als", sgd_workers: int = 0,
                sgd_conflicts: str = "locks", devices=None) -> tuple[MfitrModel, list[EpochStats]]:
    """hyper.iters ALS-MFITR sweeps; one EpochStats row per sweep with
    loss_mfitr and the clipped validation RMSE (mfitr.py:347-371 signature).

    method="sgd": the reference's own SGD trainer instead (train_mfitr_sgd;
    sgd_workers concurrent user warps, sgd_conflicts "locks" = the
    reference's per-item LockTable contract, or "hogwild").
    blocks="full" (default): every parameter of the reference's MFITR model
    (mfitr.py:92-149) -- [q_i|b_i] per taxonomy layer, [q_a|b_a] per artist,
    [p_u|b_u] (MfitrFullSolver); blocks="q": factors only, biases and q_a
    frozen at 0 (MfitrSolver, the benchmark's configs 2 and 4).
    devices=N > 1 (blocks="q"): the factor blocks sharded over N GPUs, one
    process per GPU calling train_mfitr(..., devices=N) on the same data --
    users by nnz, items by whole taxonomy subtree (parallel.ShardedMfitr);
    identical results for any N."""
    if kind == "time-mfitr":
        raise ConfigError("time-mfitr is outside the device path (no time terms)")
    if method == "sgd":   # the reference's own trainer (mfitr.py:347-371), on device
        return train_mfitr_sgd(kind, train_data, validation, graph, hyper, seed, ew,
                               num_users, num_items, device=device, objective=objective,
                               workers=sgd_workers, conflicts=sgd_conflicts)
    if method != "als":
        raise ConfigError(f"method must be 'als' or 'sgd', got {method!r}")
    if blocks not in ("full", "q"):
        raise ConfigError(f"blocks must be 'full' or 'q', got {blocks!r}")
    from .factor import sharded_world
    world = sharded_world(devices)
    if world > 1 and blocks != "q":
        raise ConfigError("the sharded ALS-MFITR fit covers the factor blocks (blocks='q')")
    hyper = dataclasses.replace(hyper)
    model = init_mfitr(kind, train_data, graph, hyper, seed, num_users=num_users,
                       num_items=num_items)
    if blocks == "q":
        model.q_a = np.zeros_like(model.q_a)      # artist factors frozen at 0
    base = model.base
    if init is not None:
        base.p, base.q = np.asarray(init[0], np.float64), np.asarray(init[1], np.float64)
    r = _ratings_for(train_data, device, False, base.num_users, base.num_items)
    if ew is None:
        ew = edge_weights(graph, train_data, device=r.device, num_items=base.num_items)
    dev = r.device
    vu = vi = vs = None
    if validation is not None and len(validation):
        vu = torch.as_tensor(validation.users.astype(np.int32), device=dev)
        vi = torch.as_tensor(validation.items.astype(np.int32), device=dev)
        vs = torch.as_tensor(validation.scores.astype(np.float32), device=dev)
    clip = (train_data.scale.lo, train_data.scale.hi)
    report = []
    if world > 1:
        return _train_mfitr_sharded(model, train_data, graph, ew, hyper, dev, (vu, vi, vs), clip,
                                    objective, as_torch)
    if blocks == "full":
        solver = MfitrFullSolver(r, graph, ew.w, hyper, base.mu, model.artist_of_item, base.p,
                                 base.q, model.q_a, base.b_u, base.b_i, model.b_a)
        for ep in range(hyper.iters):
            solver.sweep()
            base.epochs_done += 1
            obj = solver.loss() if objective else None
            rm = None
            if vu is not None:
                _, sse = solver.predict(vu, vi, vs, clip=clip)
                rm = torch.sqrt(sse / vu.numel())
            solver.check()
            report.append(EpochStats(ep, hyper.gamma,
                                     float(obj.item()) if obj is not None else float("nan"),
                                     float(rm.item()) if rm is not None else float("nan")))
        P, Q, bu, bi, ba, Qa = solver.params()
        host = (lambda t: t.clone()) if as_torch else (lambda t: t.double().cpu().numpy())
        base.p, base.q, model.q_a = host(P), host(Q), host(Qa)
        base.b_u, base.b_i, model.b_a = (t.double().cpu().numpy() for t in (bu, bi, ba))
        eng = AlsEngine(r, base.D)       # prediction engine of the fitted model
        eng.set_factors(P, Q)
        base.engine = eng
        model.ew = ew
        return model, report
    eng = AlsEngine(r, base.D)
    eng.set_factors(base.p, base.q)
    base.engine = eng
    solver = MfitrSolver(eng, graph, ew.w, hyper, base.mu)
    art = torch.as_tensor(model.artist_of_item.astype(np.int32), device=dev)
    for ep in range(hyper.iters):
        solver.sweep()
        base.epochs_done += 1
        obj = solver.loss() if objective else None
        rm = None
        if vu is not None:
            _, sse = eng.predict(vu, vi, vs, want_pred=False, mu=base.mu, art=art,
                                 Q_a=torch.zeros_like(eng.Q), clip=clip)
            rm = torch.sqrt(sse / vu.numel())
        eng.check()
        report.append(EpochStats(ep, hyper.gamma,
                                 float(obj.item()) if obj is not None else float("nan"),
                                 float(rm.item()) if rm is not None else float("nan")))
    if as_torch:
        base.p, base.q = eng.factors()
    else:
        P, Q = eng.factors()
        base.p, base.q = P.double().cpu().numpy(), Q.double().cpu().numpy()
    model.ew = ew
    return model, report


def _train_mfitr_sharded(model: MfitrModel, train_data: Dataset, graph: TaxonomyGraph,
                         ew: TaxonomyEdgeWeights, hyper: MfitrHyper, dev, valid, clip,
                         objective: bool, as_torch: bool):
    """train_mfitr(blocks='q') over the ranks of the default process group
    (parallel.ShardedMfitr).  Per sweep: loss_mfitr (time off, biases and q_a
    at 0) from the replicated factors, the clipped held-out RMSE, and the
    failure check reduced over ranks."""
    from .factor import _standalone_engine_for
    from .parallel import ShardedMfitr
    base = model.base
    U, I, D = base.num_users, base.num_items, base.D
    run = ShardedMfitr(train_data.users, train_data.items, train_data.scores, U, I, D, graph,
                       ew.w, hyper.lam2, hyper.lam3 + hyper.lam4, base.mu, device=dev)
    run.set_factors(base.p, base.q)
    ev = _standalone_engine_for(U, I, D, dev)
    art = torch.as_tensor(model.artist_of_item.astype(np.int32), device=dev)
    vu, vi, vs = valid
    w64 = torch.as_tensor(np.asarray(ew.w, np.float64), device=dev)
    ec = torch.as_tensor(graph.edge_child, device=dev)
    ep = torch.as_tensor(graph.edge_parent, device=dev)
    report = []
    for it in range(hyper.iters):
        run.sweep()
        base.epochs_done += 1
        run.check()
        P, Q = run.factors()
        ev.set_factors(P, Q)
        obj = float("nan")
        if objective:
            obj = float(_loss_q(ev, train_data, dev, base.mu, hyper, w64, ec, ep).item())
        rm = float("nan")
        if vu is not None:
            _, sse = ev.predict(vu, vi, vs, want_pred=False, mu=base.mu, art=art,
                                Q_a=torch.zeros_like(ev.Q), clip=clip)
            rm = float(torch.sqrt(sse / vu.numel()).item())
        report.append(EpochStats(it, hyper.gamma, obj, rm))
    base.engine = ev
    if as_torch:
        base.p, base.q = ev.factors()
    else:
        P, Q = ev.factors()
        base.p, base.q = P.double().cpu().numpy(), Q.double().cpu().numpy()
    model.ew = ew
    return model, report


def _loss_q(ev: AlsEngine, train_data: Dataset, dev, mu: float, hyper: MfitrHyper, w64, ec, ep):
    """loss_mfitr with biases / q_a at 0 and time off (mfitr.py:219-242) from
    replicated factors over the full training split."""
    cache = train_data.__dict__.setdefault("_loss_q_cache", {})
    key = str(dev)
    if key not in cache:
        u = torch.as_tensor(np.asarray(train_data.users, np.int32), device=dev)
        i = torch.as_tensor(np.asarray(train_data.items, np.int32), device=dev)
        s = torch.as_tensor(np.asarray(train_data.scores, np.float32), device=dev)
        cu = torch.bincount(u.long(), minlength=ev.P.shape[0]).double()
        ci = torch.bincount(i.long(), minlength=ev.Q.shape[0]).double()
        cache[key] = (u, i, s, cu, ci)
    u, i, s, cu, ci = cache[key]
    _, sse = ev.predict(u, i, s, want_pred=False, mu=mu, clip=(-3.0e38, 3.0e38))
    P, Q = (t.double() for t in ev.factors())
    reg = (cu * (P ** 2).sum(1)).sum() + (ci * (Q ** 2).sum(1)).sum()
    d2 = ((Q[ec] - Q[ep]) ** 2).sum(1)
    return sse + hyper.lam2 * reg + (hyper.lam3 + hyper.lam4) * (w64 * d2).sum()
