"""Resident device state of the ALS sweep: rating layouts, factor tables,
work plans, workspaces -- everything the C-ABI needs, allocated through
PyTorch (device memory + streams are plumbing; the compute is libmcf).

HBM layout (per GPU):
  * users layout (CSR by user) and items layout (CSC by item): ptr int64
    [n+1], idx int32 [nnz] (the partner id), val float32 [nnz] (the rating),
    perm int32 [nnz] (record index, kept only when per-observation weights
    must be permuted);  8 B per rating per layout.
  * factor tables P [U][ld], Q [I][ld] float32, ld = mcf_factor_ld(D) (round_up(D, 8)
    for D > 4) with zero padding, so every partner row is sector-aligned.
  * per (layout, row set) a work plan (int32 chunk offsets, partial-Gram
    slot offsets, item->row map) and the partial-Gram workspace.
"""
from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from ._lib import check, ptr
from .errors import ConfigError, DeviceError, SingularSystemError

DEFAULT_CHUNK = 2048
TC_CHUNK = int(os.environ.get("MCF_TC_CHUNK", 2048))   # tensor-core wide path: ratings per hot-row chunk (a
                                     # chunk's partial Gram is DP^2 floats, ~6 B per rating)
PAIR_CHUNK_CAP = 8192                # pair path: longest task (config 1: 11.5 -> 11.3 ms)
TASKS_IN_FLIGHT = 2 * 148 * 8 * 16   # 2 x (SMs x pair-kernel warps x lane pairs)


def adaptive_chunk(nnz_rows: int, cap: int = PAIR_CHUNK_CAP) -> int:
    """Task length of the pair path for rows holding nnz_rows ratings: long
    tasks (fewer hot-row chunk partials, fewer group boundaries) but at
    least ~2 tasks per lane pair in flight, multiples of 32, 128..cap
    (MCF_PAIR_CHUNK_MIN; config 2: 64 / 128 / 256 / 512 -> 11.725 / 11.713 / 11.718 / 11.778 ms)."""
    return max(int(os.environ.get("MCF_PAIR_CHUNK_MIN", 128)), min(cap, nnz_rows // TASKS_IN_FLIGHT // 32 * 32))
PLAN_INFO_LEN = 6   # MCF_PLAN_INFO_LEN


def tc_path(D: int, weighted: bool = False) -> bool:
    """mcf_als_half_step runs the tensor-core wide path (als_tc.cu) for this
    dimension: 64 <= D <= 128 without per-observation weights (MCF_NO_TC=1
    selects the CUDA-core kernels instead)."""
    lo = max(49, int(os.environ.get("MCF_TC_MIN_D", 64)))   # must agree with tc_min_d() (als_tc.cu)
    return lo <= D <= 128 and not weighted and not os.environ.get("MCF_NO_TC")


def cuda_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the ALS sweep runs only on the GPU (no CPU fallback)")
    dev = torch.device(device if device is not None else "cuda")
    if dev.type != "cuda":
        raise DeviceError(f"device must be a CUDA device, got {dev}")
    return dev


def stream_ptr(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


class SideLayout:
    """CSR of one side: rows keyed by `keys`, partners `cols`, values `vals`
    -- in-row order == record order (reference factor.py:502)."""

    def __init__(self, keys: torch.Tensor, cols: torch.Tensor, vals: torch.Tensor, n_rows: int,
                 keep_perm: bool = False):
        dev = keys.device
        L = _lib.lib()
        nnz = int(keys.numel())
        self.n_rows, self.nnz, self.device = int(n_rows), nnz, dev
        self.ptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
        self.idx = torch.empty(nnz, dtype=torch.int32, device=dev)
        self.val = torch.empty(nnz, dtype=torch.float32, device=dev)
        self.perm = torch.empty(nnz, dtype=torch.int32, device=dev) if keep_perm else None
        ws = torch.empty(int(L.mcf_csr_workspace_bytes(nnz, n_rows)), dtype=torch.uint8, device=dev)
        check(L.mcf_csr_build(ptr(keys), ptr(cols), ptr(vals), nnz, n_rows, ptr(self.ptr),
                              ptr(self.idx), ptr(self.val), ptr(self.perm), ptr(ws), ws.numel(),
                              stream_ptr(dev)), "mcf_csr_build")
        del ws
        self._plans = {}

    def degrees(self) -> torch.Tensor:
        return self.ptr[1:] - self.ptr[:-1]

    def plan(self, rows: torch.Tensor | None = None, key=None, chunk: int = DEFAULT_CHUNK,
             adaptive: bool = False):
        """(plan buffer, plan_info, row list, n_list, chunk) for all rows, or
        for the int32 row list `rows` (cached under `key`).  adaptive=True (the
        pair path): `chunk` is a cap and the task length follows the rows'
        rating count (adaptive_chunk) -- e.g. a small taxonomy layer with a
        few Zipf-hot items would otherwise end on one long task."""
        k = (key if rows is not None else "all", chunk, adaptive)
        if k not in self._plans:
            L = _lib.lib()
            n_list = self.n_rows if rows is None else int(rows.numel())
            if adaptive:
                nnz_rows = self.nnz if rows is None else (
                    int(self.degrees()[rows.long()].sum()) if n_list else 0)
                chunk = adaptive_chunk(nnz_rows, chunk)
            buf = torch.empty(int(L.mcf_als_plan_bytes(n_list, self.nnz, chunk)), dtype=torch.uint8,
                              device=self.device)
            info = (_lib.c_i64 * PLAN_INFO_LEN)()
            check(L.mcf_als_plan(ptr(self.ptr), ptr(rows), n_list, 0, chunk, self.nnz, ptr(buf),
                                 buf.numel(), info, stream_ptr(self.device)), "mcf_als_plan")
            self._plans[k] = (buf, info, rows, n_list, chunk)
        return self._plans[k]


def _as_i32(x, dev):
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.int32, non_blocking=True).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int32)).to(dev, non_blocking=True)


def _as_f32(x, dev):
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.float32, non_blocking=True).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev, non_blocking=True)


class DeviceRatings:
    """Both layouts of one training split, resident on one GPU."""

    def __init__(self, users, items, scores, num_users: int, num_items: int, device=None,
                 keep_perm: bool = False):
        dev = cuda_device(device)
        u, i, s = _as_i32(users, dev), _as_i32(items, dev), _as_f32(scores, dev)
        self.device, self.num_users, self.num_items = dev, int(num_users), int(num_items)
        self.nnz = int(u.numel())
        self.by_user = SideLayout(u, i, s, num_users, keep_perm)
        self.by_item = SideLayout(i, u, s, num_items, keep_perm)
        # float64 sum without a float64 copy of the ratings
        self.global_mean = float(torch.sum(s, dtype=torch.float64)) / self.nnz if self.nnz else 0.0

    @classmethod
    def from_dataset(cls, ds, device=None, keep_perm: bool = False) -> "DeviceRatings":
        return cls(ds.users, ds.items, ds.scores, ds.num_users, ds.num_items, device, keep_perm)

    def layout(self, side: str) -> SideLayout:
        if side == "users":
            return self.by_user
        if side == "items":
            return self.by_item
        raise ConfigError(f"side must be 'users' or 'items', got {side!r}")


class LayoutSolver:
    """mcf_als_half_step over one SideLayout with caller-chosen fixed / out
    tables (used by AlsEngine and by the row-sharded multi-GPU runner)."""

    def __init__(self, D: int, chunk: int | None = None):
        """chunk: fixed task length, or None -- adaptive up to PAIR_CHUNK_CAP
        on the pair path (D <= 20), DEFAULT_CHUNK on the wide paths."""
        self.D, self.chunk = int(D), (None if chunk is None else int(chunk))
        self._ws = {}
        self.fail = None

    def solve(self, lay: SideLayout, fixed: torch.Tensor, out: torch.Tensor, lam_c=0.0, lam_n=0.0,
              y_shift=0.0, tax_S=None, tax_T=None, tau=0.0, rows=None, rows_key=None, wts=None,
              fail: torch.Tensor | None = None, obj_out: torch.Tensor | None = None,
              val: torch.Tensor | None = None, bias=None, peers: torch.Tensor | None = None,
              chunk: int | None = None, multicast: int | None = None, emit=None):
        """bias = (dim, lam_c, lam_n): coordinate `dim` is a bias with its own
        regulariser (mcf_als_half_step_bias); val: per-rating targets in the
        layout's CSR order instead of the ratings; peers: device int64 tensor
        of peer replica pointers -- the kernel stores every solved row there
        too (mcf_als_half_step_peers, the fused all-gather); multicast: the
        NVLS multicast address of the replicated table at this shard -- one
        multimem store per element reaches every replica
        (mcf_als_half_step_multicast)."""
        dev = lay.device
        if fail is None:
            if self.fail is None:
                self.fail = torch.full((1,), -1, dtype=torch.int64, device=dev)
            fail = self.fail
        if chunk is None:
            chunk = self.chunk
        if chunk is not None:       # fixed task length (tests, G-invariant sharded runs)
            buf, info, rl, n_list, chunk = lay.plan(rows, rows_key, chunk)
        elif self.D <= 20:          # pair path: adaptive task length
            buf, info, rl, n_list, chunk = lay.plan(rows, rows_key, PAIR_CHUNK_CAP, adaptive=True)
        elif tc_path(self.D, wts is not None):   # tensor-core wide path: long chunks
            buf, info, rl, n_list, chunk = lay.plan(rows, rows_key, TC_CHUNK)
        else:
            buf, info, rl, n_list, chunk = lay.plan(rows, rows_key, DEFAULT_CHUNK)
        slots = max(info[1], info[3])   # hot-chunk slots (pair path / warp+CTA paths)
        k = (id(lay), rows_key)
        need = int(_lib.lib().mcf_als_workspace_bytes_fixed(n_list, slots, self.D,
                                                            int(fixed.shape[0]), int(info[5])))
        if k not in self._ws or self._ws[k].numel() < need:
            self._ws[k] = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
        ws = self._ws[k]
        vals = lay.val if val is None else val
        if multicast is not None:
            if bias is not None or peers is not None:
                raise ConfigError("multicast stores exclude bias blocks and peer stores")
            check(_lib.lib().mcf_als_half_step_multicast(
                ptr(lay.ptr), ptr(lay.idx), ptr(vals), ptr(wts), ptr(fixed), fixed.shape[0],
                ptr(out), self.D, float(lam_c), float(lam_n), float(y_shift), ptr(tax_S),
                ptr(tax_T), float(tau), ptr(rl), n_list, 0, chunk, ptr(buf), info, ptr(fail),
                ptr(obj_out), ptr(ws), ws.numel(), int(multicast), stream_ptr(dev)),
                "mcf_als_half_step_multicast")
            return fail
        if peers is not None:
            if bias is not None:
                raise ConfigError("bias blocks and peer stores are not combined")
            check(_lib.lib().mcf_als_half_step_peers(
                ptr(lay.ptr), ptr(lay.idx), ptr(vals), ptr(wts), ptr(fixed), fixed.shape[0],
                ptr(out), self.D, float(lam_c), float(lam_n), float(y_shift), ptr(tax_S),
                ptr(tax_T), float(tau), ptr(rl), n_list, 0, chunk, ptr(buf), info, ptr(fail),
                ptr(obj_out), ptr(ws), ws.numel(), ptr(peers), int(peers.numel()),
                stream_ptr(dev)), "mcf_als_half_step_peers")
            return fail
        if emit is not None:   # MFITR block: (emit, corr_tab, corr_idx, ysub), Schur pair path
            if bias is None or wts is not None or lam_c != 0.0 or bias[1] != 0.0:
                raise ConfigError("emit= needs a bias block without weights or lam_c")
            e, corr_tab, corr_idx, ysub = emit
            check(_lib.lib().mcf_als_half_step_mfitr(
                ptr(lay.ptr), ptr(lay.idx), ptr(vals), ptr(fixed), fixed.shape[0], ptr(out),
                self.D, float(lam_n), float(y_shift), ptr(tax_S), ptr(tax_T), float(tau), ptr(rl),
                n_list, chunk, ptr(buf), info, ptr(fail), ptr(ws), ws.numel(), float(bias[2]),
                ptr(e), ptr(corr_tab), ptr(corr_idx), int(bool(ysub)), stream_ptr(dev)),
                "mcf_als_half_step_mfitr")
            return fail
        if bias is not None:
            check(_lib.lib().mcf_als_half_step_bias(
                ptr(lay.ptr), ptr(lay.idx), ptr(vals), ptr(wts), ptr(fixed), fixed.shape[0],
                ptr(out), self.D, float(lam_c), float(lam_n), float(y_shift), ptr(tax_S),
                ptr(tax_T), float(tau), ptr(rl), n_list, 0, chunk, ptr(buf), info, ptr(fail),
                ptr(ws), ws.numel(), int(bias[0]), float(bias[1]), float(bias[2]),
                stream_ptr(dev)), "mcf_als_half_step_bias")
            return fail
        check(_lib.lib().mcf_als_half_step(
            ptr(lay.ptr), ptr(lay.idx), ptr(vals), ptr(wts), ptr(fixed), fixed.shape[0],
            ptr(out), self.D,
            float(lam_c), float(lam_n), float(y_shift), ptr(tax_S), ptr(tax_T), float(tau),
            ptr(rl), n_list, 0, chunk, ptr(buf), info, ptr(fail), ptr(obj_out), ptr(ws),
            ws.numel(), stream_ptr(dev)), "mcf_als_half_step")
        return fail


class AlsEngine:
    """Factor tables + plans + workspaces for repeated half-steps of one
    ratings split.  All calls are asynchronous on the current stream; row
    failures accumulate in a device scalar read by `check()`."""

    def __init__(self, ratings: DeviceRatings, D: int, chunk: int | None = None):
        if not 1 <= D <= 128:
            raise ConfigError("D must be in [1, 128] on the device path")
        self.r, self.D, self.ld, self.chunk = ratings, int(D), _lib.factor_ld(D), chunk
        dev = ratings.device
        self.device = dev
        self.P = torch.zeros(ratings.num_users, self.ld, dtype=torch.float32, device=dev)
        self.Q = torch.zeros(ratings.num_items, self.ld, dtype=torch.float32, device=dev)
        self.fail = torch.full((1,), -1, dtype=torch.int64, device=dev)
        # first failing row per side since the last check()
        self._fail_acc = torch.full((2,), -1, dtype=torch.int64, device=dev)
        self._solver = LayoutSolver(D, chunk)
        self._wts = {}
        self._red = None

    # -- factors -------------------------------------------------------------
    def set_factors(self, P=None, Q=None):
        for dst, src in ((self.P, P), (self.Q, Q)):
            if src is None:
                continue
            t = src if isinstance(src, torch.Tensor) else torch.from_numpy(np.asarray(src))
            if t.shape != (dst.shape[0], self.D):
                raise ConfigError(f"factor shape {tuple(t.shape)} != {(dst.shape[0], self.D)}")
            if t.device.type == "cpu" and t.dtype != torch.float32:
                t = t.to(torch.float32)
            dst[:, : self.D].copy_(t, non_blocking=True)
            if self.ld > self.D:
                dst[:, self.D:].zero_()

    def factors(self):
        return self.P[:, : self.D], self.Q[:, : self.D]

    # -- weights -------------------------------------------------------------
    def set_weights(self, weights):
        """Per-observation weights in record order (the reference's wALS
        hook, factor.py:506-509): permuted into each layout's CSR order."""
        if weights is None:
            self._wts = {}
            return
        w = _as_f32(weights, self.device)
        for side in ("users", "items"):
            lay = self.r.layout(side)
            if lay.perm is None:
                raise ConfigError("per-observation weights need DeviceRatings(keep_perm=True)")
            self._wts[side] = w[lay.perm.long()]

    # -- half-step -----------------------------------------------------------
    def half_step(self, side: str, lam_c: float = 0.0, lam_n: float = 0.0, y_shift: float = 0.0,
                  tax_S=None, tax_T=None, tau: float = 0.0, rows: torch.Tensor | None = None,
                  rows_key=None, fixed: torch.Tensor | None = None, obj_out=None):
        lay = self.r.layout(side)
        out = self.P if side == "users" else self.Q
        if fixed is None:
            fixed = self.Q if side == "users" else self.P
        self._solver.solve(lay, fixed, out, lam_c, lam_n, y_shift, tax_S, tax_T, tau, rows,
                           rows_key, self._wts.get(side), self.fail, obj_out)
        acc = self._fail_acc[0:1] if side == "items" else self._fail_acc[1:2]
        torch.where(acc < 0, self.fail, acc, out=acc)
        return out

    @property
    def fused_objective(self) -> bool:
        """The solve epilogue can report the objective (D <= 20 path)."""
        return self.D <= 20

    def sweep(self, lam_c: float = 0.0, lam_n: float = 0.0, obj: torch.Tensor | None = None):
        """One full iteration: items half-step, then users (factor.py:550-555).
        With `obj` (device double[4], D <= 20) the half-steps also report
        their objective terms: (items sse, items reg, users sse, users reg)."""
        self.half_step("items", lam_c, lam_n, obj_out=None if obj is None else obj[0:2])
        self.half_step("users", lam_c, lam_n, obj_out=None if obj is None else obj[2:4])

    @staticmethod
    def sweep_objective(obj: torch.Tensor) -> torch.Tensor:
        """Objective after a sweep: the users half-step's data term with the
        final factors, plus both sides' regularisers."""
        return obj[2:3] + obj[3:4] + obj[1:2]

    def check_with(self, *values):
        """check() and read device scalars in ONE host synchronisation: the
        per-sweep metrics of train() ride along with the failure flags."""
        parts = [v.reshape(-1)[:1].double() for v in values if v is not None]
        flat = torch.cat(parts + [self._fail_acc.double()]).tolist()
        items_row, users_row = int(flat[-2]), int(flat[-1])
        self._fail_acc.fill_(-1)
        for side, row in (("items", items_row), ("users", users_row)):
            if row >= 0:
                raise SingularSystemError(
                    f"singular normal equations at {side} row {row}; use lam > 0")
        it = iter(flat[:-2])
        return [next(it) if v is not None else None for v in values]

    def check(self):
        """Synchronise and raise SingularSystemError for a failed row
        (factor.py:535-537); the items half-step runs first in a sweep, so
        its failure is reported first."""
        items_row, users_row = (int(x) for x in self._fail_acc.tolist())
        self._fail_acc.fill_(-1)
        for side, row in (("items", items_row), ("users", users_row)):
            if row >= 0:
                raise SingularSystemError(
                    f"singular normal equations at {side} row {row}; use lam > 0")

    # -- metrics ---------------------------------------------------------------
    def _reduction_ws(self, n):
        need = int(_lib.lib().mcf_predict_workspace_bytes(n))
        if self._red is None or self._red.numel() < need:
            self._red = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
        return self._red

    def predict(self, users: torch.Tensor, items: torch.Tensor, truth: torch.Tensor | None = None,
                want_pred: bool = True, mu: float = 0.0, b_u=None, b_i=None, art=None, b_a=None,
                Q_a=None, clip=(0.0, 100.0), P=None, Q=None):
        """(pred or None, sse device double or None)."""
        n = int(users.numel())
        pred = torch.empty(n, dtype=torch.float32, device=self.device) if want_pred else None
        sse = torch.zeros(1, dtype=torch.float64, device=self.device) if truth is not None else None
        ws = self._reduction_ws(n)
        P = self.P if P is None else P
        Q = self.Q if Q is None else Q
        check(_lib.lib().mcf_predict_sse(
            ptr(users), ptr(items), ptr(truth), n, ptr(P), P.shape[0], ptr(Q), Q.shape[0],
            self.D, float(mu), ptr(b_u), ptr(b_i), ptr(art), ptr(b_a), ptr(Q_a),
            float(clip[0]), float(clip[1]), ptr(pred), ptr(sse), ptr(ws), ws.numel(),
            stream_ptr(self.device)), "mcf_predict_sse")
        return pred, sse

    def rmse(self, users, items, truth, clip=(0.0, 100.0)) -> torch.Tensor:
        _, sse = self.predict(users, items, truth, want_pred=False, clip=clip)
        return torch.sqrt(sse / max(int(users.numel()), 1))

    def sq_norms(self, F: torch.Tensor, counts_ptr=None) -> torch.Tensor:
        out = torch.zeros(1, dtype=torch.float64, device=self.device)
        ws = self._reduction_ws(F.shape[0])
        check(_lib.lib().mcf_sq_norms(ptr(F), F.shape[0], self.D, ptr(counts_ptr), ptr(out),
                                      ptr(ws), ws.numel(), stream_ptr(self.device)),
              "mcf_sq_norms")
        return out

    def objective(self, lam: float, reg: str = "plain", users=None, items=None, scores=None):
        """Training objective on device: sum (r - q.p)^2 + lam (|P|^2 + |Q|^2)
        (plain, factor.py:541-547) or + lam sum_r n_r |f_r|^2 (weighted,
        factor.loss_mf with mu = b = 0, factor.py:270-278).  Evaluated
        through the users layout (its idx/val are the records in CSR order)."""
        lay = self.r.by_user
        if users is None:
            if getattr(self, "_rows_of_records", None) is None:
                self._rows_of_records = torch.repeat_interleave(
                    torch.arange(self.r.num_users, device=self.device, dtype=torch.int32),
                    lay.degrees())
            users, items, scores = self._rows_of_records, lay.idx, lay.val
            w = self._wts.get("users")      # record weights in the users layout's order
        else:
            w = None
        if w is not None:
            # the reference's weighted data term sum w (r - q.p)^2 (factor.py:541-547)
            pred, _ = self.predict(users, items, None, want_pred=True)
            sse = (w.double() * (scores.double() - pred.double()) ** 2).sum().reshape(1)
        else:
            _, sse = self.predict(users, items, scores, want_pred=False, clip=(-3.0e38, 3.0e38))
        if reg == "weighted":
            regp = self.sq_norms(self.P, self.r.by_user.ptr)
            regq = self.sq_norms(self.Q, self.r.by_item.ptr)
        else:
            regp, regq = self.sq_norms(self.P), self.sq_norms(self.Q)
        return sse + lam * (regp + regq)
