"""Row-sharded multi-GPU ALS: one process per GPU, NCCL all-gather of the
freshly solved factor shard after every half-step.

The reference parallelises a half-step over static equal-row blocks of
Python threads (parallel.run_blocks / even_bounds, reference
parallel.py:134-145); rows are independent given the fixed side, so its
output is identical for any thread count (factor.py:528-534).
The device analogue:

* users and items are cut into `world` CONTIGUOUS row ranges at the nnz
  prefix-sum quantiles of their layout (not equal row counts: degrees are
  log-normal / Zipf);
* each rank keeps only its own rows' CSR (users) and CSC (items) -- built
  from the records whose user (item) falls in its range -- and the FULL
  opposite factor table;
* factor tables use a PADDED shard layout: shard s occupies rows
  [s*S, s*S + n_s) of a [world*S, ld] table (S = the largest shard), and
  partner ids in the local layouts are stored in that padded numbering, so
  the solve writes its rows in place and the all-gather is NCCL's in-place
  form (sendbuff == recvbuff + rank*S*ld) -- no copies, no index remap at
  run time;
* every row is solved with the same chunking and reduction order as on one
  GPU, so factors are bit-identical for any world size (G-invariance, the
  device analogue of the reference's thread-count invariance).

`solver` is pluggable so the host-side logic (cuts, padded numbering,
gather) can be exercised on CPU ranks over gloo; the product path uses the
device solver (libmcf) and NCCL.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .errors import ConfigError


def nnz_balanced_cuts(degrees: torch.Tensor, world: int) -> torch.Tensor:
    """Contiguous row ranges with ~equal ratings: cut k is the first row
    whose nnz prefix reaches k/world of the total.  int64 [world + 1]."""
    n = int(degrees.numel())
    pre = torch.cumsum(degrees.to(torch.int64), 0)
    total = int(pre[-1]) if n else 0
    targets = torch.tensor([(total * k + world - 1) // world for k in range(1, world)],
                           dtype=torch.int64, device=degrees.device)
    inner = torch.searchsorted(pre, targets, right=False) + 1 if n else targets * 0
    cuts = torch.cat([torch.zeros(1, dtype=torch.int64, device=degrees.device),
                      inner.clamp(max=n),
                      torch.full((1,), n, dtype=torch.int64, device=degrees.device)])
    return torch.cummax(cuts, 0).values


class ShardMap:
    """Global row id <-> padded shard numbering."""

    def __init__(self, cuts: torch.Tensor):
        self.cuts = cuts
        self.world = int(cuts.numel()) - 1
        sizes = cuts[1:] - cuts[:-1]
        self.sizes = sizes
        self.S = max(1, int(sizes.max())) if self.world else 1
        self.rows = self.world * self.S

    def range(self, r: int):
        return int(self.cuts[r]), int(self.cuts[r + 1])

    def to_padded(self, ids: torch.Tensor) -> torch.Tensor:
        ids64 = ids.to(torch.int64)
        shard = torch.searchsorted(self.cuts[1:], ids64, right=True)
        return (shard * self.S + ids64 - self.cuts[shard]).to(torch.int32)

    def padded_index(self) -> torch.Tensor:
        """For each global row, its padded row (int64 [n])."""
        n = int(self.cuts[-1])
        return self.to_padded(torch.arange(n, device=self.cuts.device)).to(torch.int64)


class ShardedAls:
    """One rank's part of a row-sharded ALS fit."""

    def __init__(self, users, items, scores, num_users: int, num_items: int, D: int, *,
                 group=None, solver="device", device=None, chunk: int | None = None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.D, self.ld = int(D), _lib.factor_ld(D)
        if solver == "device":
            from .device import DEFAULT_CHUNK, LayoutSolver, cuda_device
            dev = cuda_device(device)
            self._solver = LayoutSolver(D, chunk or DEFAULT_CHUNK)
        else:
            dev = torch.device(device or "cpu")
            self._solver = solver
        self.device = dev
        u = torch.as_tensor(users).to(dev, torch.int64)
        it = torch.as_tensor(items).to(dev, torch.int64)
        s = torch.as_tensor(scores).to(dev, torch.float32)
        self.num_users, self.num_items = int(num_users), int(num_items)
        self.umap = ShardMap(nnz_balanced_cuts(torch.bincount(u, minlength=num_users), self.world))
        self.imap = ShardMap(nnz_balanced_cuts(torch.bincount(it, minlength=num_items), self.world))
        self.P = torch.zeros(self.umap.rows, self.ld, dtype=torch.float32, device=dev)
        self.Q = torch.zeros(self.imap.rows, self.ld, dtype=torch.float32, device=dev)
        # local layouts: my users (partners = padded item ids), my items
        self.local = {}
        for side, keys, cols, kmap, cmap in (("users", u, it, self.umap, self.imap),
                                             ("items", it, u, self.imap, self.umap)):
            lo, hi = kmap.range(self.rank)
            m = (keys >= lo) & (keys < hi)
            k_loc = (keys[m] - lo).to(torch.int32)
            c_pad = cmap.to_padded(cols[m])
            self.local[side] = self._make_layout(k_loc, c_pad, s[m], hi - lo)
        self.nnz_local = {k: int(v.nnz) for k, v in self.local.items()}

    def _make_layout(self, keys, cols, vals, n_rows):
        if self._solver.__class__.__name__ == "LayoutSolver":
            from .device import SideLayout
            return SideLayout(keys, cols, vals, n_rows)
        return _HostLayout(keys, cols, vals, n_rows)

    # -- factors -------------------------------------------------------------
    def set_factors(self, P=None, Q=None):
        for dst, src, mp in ((self.P, P, self.umap), (self.Q, Q, self.imap)):
            if src is None:
                continue
            t = torch.as_tensor(np.asarray(src) if not isinstance(src, torch.Tensor) else src)
            t = t.to(self.device, torch.float32)
            dst.zero_()
            dst[mp.padded_index(), : self.D] = t

    def factors(self):
        """(P, Q) in global row order, [n, D] views gathered from the padded tables."""
        return (self.P[self.umap.padded_index(), : self.D],
                self.Q[self.imap.padded_index(), : self.D])

    # -- sweep ---------------------------------------------------------------
    def half_step(self, side: str, lam_c: float = 0.0, lam_n: float = 0.0, gather: bool = True):
        if side not in ("users", "items"):
            raise ConfigError(f"side must be 'users' or 'items', got {side!r}")
        out_full, fixed, mp = ((self.P, self.Q, self.umap) if side == "users"
                               else (self.Q, self.P, self.imap))
        S = mp.S
        mine = out_full[self.rank * S:(self.rank + 1) * S]
        self._solver.solve(self.local[side], fixed, mine, lam_c, lam_n)
        if gather and self.world > 1:
            # in place: my shard already sits at rank*S inside out_full
            dist.all_gather_into_tensor(out_full, mine, group=self.group)
        return out_full

    def sweep(self, lam_c: float = 0.0, lam_n: float = 0.0):
        self.half_step("items", lam_c, lam_n)
        self.half_step("users", lam_c, lam_n)

    def check(self):
        f = getattr(self._solver, "fail", None)
        if isinstance(f, torch.Tensor):
            row = int(f.item())
            if row >= 0:
                from .errors import SingularSystemError
                raise SingularSystemError(f"singular normal equations at local row {row} "
                                          f"on rank {self.rank}; use lam > 0")


class _HostLayout:
    """CPU stand-in for SideLayout (host-logic tests over gloo)."""

    def __init__(self, keys, cols, vals, n_rows):
        order = torch.sort(keys.to(torch.int64), stable=True).indices
        self.n_rows = int(n_rows)
        self.ptr = torch.zeros(n_rows + 1, dtype=torch.int64)
        self.ptr[1:] = torch.cumsum(torch.bincount(keys.to(torch.int64), minlength=n_rows), 0)
        self.idx = cols[order]
        self.val = vals[order]
        self.nnz = int(keys.numel())
