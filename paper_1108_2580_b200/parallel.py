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


def global_chunk(nnz_total: int, D: int, chunk: int | None) -> int:
    """Task length of a sharded run, from the GLOBAL rating count: every rank
    and every world size chunks the hot rows identically, so the chunk-order
    sums -- and the factors -- do not depend on the world size."""
    from .device import DEFAULT_CHUNK, adaptive_chunk
    if chunk is not None:
        return int(chunk)
    return adaptive_chunk(nnz_total) if D <= 20 else DEFAULT_CHUNK


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
                 group=None, solver="device", device=None, chunk: int | None = None,
                 collective: str = "nccl"):
        """collective: "nccl" -- in-place ncclAllGather after each half-step;
        "peer" -- the fused form: P and Q live in symmetric memory
        (torch.distributed._symmetric_memory, NVLink peer mappings) and the
        solve kernel itself stores every row into each peer's replica
        (mcf_als_half_step_peers), followed by a device barrier."""
        if collective not in ("nccl", "peer"):
            raise ConfigError(f"collective must be 'nccl' or 'peer', got {collective!r}")
        self.collective = collective
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.D, self.ld = int(D), _lib.factor_ld(D)
        if solver == "device":
            from .device import LayoutSolver, cuda_device
            dev = cuda_device(device)
            self._solver = LayoutSolver(D, chunk)
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
        self._peers, self._handles = {}, {}
        if collective == "peer":
            self.P, self.Q = self._symmetric_tables(dev)
        else:
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
        self.fixed_chunk = global_chunk(int(u.numel()), self.D, chunk)

    def _symmetric_tables(self, dev):
        """P, Q in symmetric memory; per side the device array of the peers'
        replica pointers, offset to this rank's shard."""
        import torch.distributed._symmetric_memory as symm_mem
        group = self.group if self.group is not None else dist.group.WORLD
        name = group.group_name
        if hasattr(symm_mem, "enable_symm_mem_for_group"):
            symm_mem.enable_symm_mem_for_group(name)
        tabs = []
        for side, mp in (("users", self.umap), ("items", self.imap)):
            t = symm_mem.empty(mp.rows, self.ld, dtype=torch.float32, device=dev)
            t.zero_()
            h = symm_mem.rendezvous(t, name)
            off = self.rank * mp.S * self.ld * 4
            ptrs = [int(h.buffer_ptrs[k]) + off for k in range(self.world) if k != self.rank]
            self._peers[side] = torch.tensor(ptrs, dtype=torch.int64, device=dev)
            self._handles[side] = h
            tabs.append(t)
        return tabs

    def _is_device(self):
        return self._solver.__class__.__name__ == "LayoutSolver"

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
        if self.collective == "peer":
            # fused: the kernel also stores each solved row into every peer's
            # replica; the barrier orders the next half-step after all stores
            self._solver.solve(self.local[side], fixed, mine, lam_c, lam_n,
                               peers=self._peers[side], chunk=self.fixed_chunk)
            if gather and self.world > 1:
                self._handles[side].barrier(channel=0)
            return out_full
        kw = {"chunk": self.fixed_chunk} if self._is_device() else {}
        self._solver.solve(self.local[side], fixed, mine, lam_c, lam_n, **kw)
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


# ---------------------------------------------------------------------------
# ALS-MFITR sharding: items cut at taxonomy-subtree boundaries

def subtree_components(graph, num_items: int) -> np.ndarray:
    """Component label per item of the taxonomy forest (an artist with its
    albums and tracks; items off the graph are singletons).  Every edge of
    the graph term (taxonomy.py:106-118) stays inside one component, so a
    rank that owns whole components solves its layered item half-step
    without any cross-rank exchange."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    E = int(graph.edge_child.size)
    A = coo_matrix((np.ones(E, dtype=np.int8), (graph.edge_child, graph.edge_parent)),
                   shape=(num_items, num_items))
    _, lab = connected_components(A, directed=False)
    return lab.astype(np.int64)


def lpt_owner(weights: np.ndarray, world: int) -> np.ndarray:
    """Longest-processing-time assignment of weighted units to `world`
    ranks (heaviest first onto the least-loaded rank; ties by unit id and
    rank id), deterministic."""
    import heapq
    n = int(weights.size)
    order = np.lexsort((np.arange(n), -weights))
    heap = [(0, r) for r in range(world)]
    owner = np.empty(n, dtype=np.int64)
    for c in order:
        load, r = heapq.heappop(heap)
        owner[c] = r
        heapq.heappush(heap, (load + int(weights[c]), r))
    return owner


class PermMap:
    """Padded shard numbering for an arbitrary row -> rank assignment: rank
    r's rows (ascending id) occupy [r*S, r*S + n_r) of a [world*S] table."""

    def __init__(self, owner: np.ndarray, world: int, device):
        owner = np.asarray(owner, np.int64)
        self.world, self.n = int(world), int(owner.size)
        counts = np.bincount(owner, minlength=world)
        self.counts = counts
        self.S = max(1, int(counts.max())) if self.n else 1
        self.rows = self.world * self.S
        order = np.lexsort((np.arange(self.n), owner))           # by rank, then id
        local = np.empty(self.n, dtype=np.int64)
        starts = np.concatenate([[0], np.cumsum(counts)[:-1]])
        local[order] = np.arange(self.n) - np.repeat(starts, counts)
        self.owner, self.local = owner, local
        self.padded_np = owner * self.S + local
        self.padded = torch.as_tensor(self.padded_np, device=device)

    def to_padded(self, ids: torch.Tensor) -> torch.Tensor:
        return self.padded[ids.to(torch.int64)].to(torch.int32)

    def padded_index(self) -> torch.Tensor:
        return self.padded


class ShardedMfitr:
    """One rank's part of a sharded ALS-MFITR fit (factor blocks; biases and
    q_a at 0, as MfitrSolver): users cut at nnz quantiles, items assigned by
    whole taxonomy subtree (LPT on their ratings), the layered item
    half-step solved locally with S/T from the local subtrees, one in-place
    all-gather per half-step.  Results are identical for any world size."""

    def __init__(self, users, items, scores, num_users: int, num_items: int, D: int, graph,
                 w, lam2: float, tau: float, mu: float, *, group=None, solver="device",
                 device=None, chunk: int | None = None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.D, self.ld = int(D), _lib.factor_ld(D)
        self.lam2, self.tau, self.mu = float(lam2), float(tau), float(mu)
        if solver == "device":
            from .device import LayoutSolver, cuda_device
            dev = cuda_device(device)
            self._solver = LayoutSolver(D, chunk)
        else:
            dev = torch.device(device or "cpu")
            self._solver = solver
        self.device = dev
        u = torch.as_tensor(users).to(dev, torch.int64)
        it = torch.as_tensor(items).to(dev, torch.int64)
        s = torch.as_tensor(scores).to(dev, torch.float32)
        self.num_users, self.num_items = int(num_users), int(num_items)
        self.umap = ShardMap(nnz_balanced_cuts(torch.bincount(u, minlength=num_users), self.world))
        comp = subtree_components(graph, num_items)
        deg = torch.bincount(it, minlength=num_items).cpu().numpy()
        cw = np.bincount(comp, weights=deg, minlength=int(comp.max()) + 1 if comp.size else 0)
        self.imap = PermMap(lpt_owner(cw.astype(np.int64), self.world)[comp], self.world, dev)
        self.P = torch.zeros(self.umap.rows, self.ld, dtype=torch.float32, device=dev)
        self.Q = torch.zeros(self.imap.rows, self.ld, dtype=torch.float32, device=dev)
        lo, hi = self.umap.range(self.rank)
        m = (u >= lo) & (u < hi)
        mk = ShardedAls._make_layout
        self.local = {"users": mk(self, (u[m] - lo).to(torch.int32), self.imap.to_padded(it[m]),
                                  s[m], hi - lo)}
        own = torch.as_tensor(self.imap.owner, device=dev)[it] == self.rank
        loc = torch.as_tensor(self.imap.local, device=dev)
        n_mine = int(self.imap.counts[self.rank])
        self.local["items"] = mk(self, loc[it[own]].to(torch.int32), self.umap.to_padded(u[own]),
                                 s[own], n_mine)
        self.nnz_local = {k: int(v.nnz) for k, v in self.local.items()}
        # taxonomy in padded item ids: incident-edge CSR (edge-list order per
        # item, as TaxonomyGraph.incident_edges), edge weights
        pc, pp = self.imap.padded_np[graph.edge_child], self.imap.padded_np[graph.edge_parent]
        E = int(pc.size)
        ends, other = np.concatenate([pc, pp]), np.concatenate([pp, pc])
        eid = np.concatenate([np.arange(E), np.arange(E)])
        order = np.argsort(ends, kind="stable")
        inc_ptr = np.zeros(self.imap.rows + 1, dtype=np.int64)
        np.cumsum(np.bincount(ends, minlength=self.imap.rows), out=inc_ptr[1:])
        self.inc = (torch.as_tensor(inc_ptr, device=dev),
                    torch.as_tensor(eid[order].astype(np.int32), device=dev),
                    torch.as_tensor(other[order].astype(np.int32), device=dev))
        self.w = torch.as_tensor(np.asarray(w, np.float32), device=dev)
        self.edges_padded = (pc, pp, np.asarray(w, np.float64))
        # my rows of each layer: local and padded indices
        mine = self.imap.owner == self.rank
        self.layers, self.layer_chunk = [], []
        self.users_chunk = global_chunk(int(u.numel()), self.D, chunk)
        for L in graph.layers(num_items):
            # task length from the GLOBAL layer size: identical on every rank,
            # so hot-row chunk sums (and results) do not depend on world size
            self.layer_chunk.append(global_chunk(int(deg[L].sum()), self.D, chunk))
            Lm = L[mine[L]]
            loc_rows = np.sort(self.imap.local[Lm])
            self.layers.append((torch.as_tensor(loc_rows.astype(np.int32), device=dev),
                                torch.as_tensor((self.rank * self.imap.S + loc_rows)
                                                .astype(np.int32), device=dev)))
        self.S_t = torch.zeros(self.imap.rows, dtype=torch.float32, device=dev)
        self.T_t = torch.zeros(self.imap.rows, self.ld, dtype=torch.float32, device=dev)

    # -- factors -------------------------------------------------------------
    def set_factors(self, P=None, Q=None):
        for dst, src, idx in ((self.P, P, self.umap.padded_index()),
                              (self.Q, Q, self.imap.padded_index())):
            if src is None:
                continue
            t = torch.as_tensor(np.asarray(src) if not isinstance(src, torch.Tensor) else src)
            dst.zero_()
            dst[idx, : self.D] = t.to(self.device, torch.float32)

    def factors(self):
        return (self.P[self.umap.padded_index(), : self.D],
                self.Q[self.imap.padded_index(), : self.D])

    # -- sweep ---------------------------------------------------------------
    def _terms(self, padded_rows):
        if self._solver.__class__.__name__ == "LayoutSolver":
            from ._lib import check, ptr
            from .device import stream_ptr
            ip, ie, io = self.inc
            check(_lib.lib().mcf_taxonomy_terms(ptr(ip), ptr(ie), ptr(io), ptr(self.w),
                                                ptr(self.Q), self.imap.rows, self.D,
                                                ptr(padded_rows), padded_rows.numel(),
                                                ptr(self.S_t), ptr(self.T_t),
                                                stream_ptr(self.device)), "mcf_taxonomy_terms")
        else:   # host stand-in (tests): the same sums, float32 tables
            self._solver.terms(self, padded_rows)

    def item_layers(self):
        S0 = self.rank * self.imap.S
        mine = self.Q[S0:S0 + self.imap.S]
        for k, (rows_loc, rows_pad) in enumerate(self.layers):
            if rows_loc.numel():
                self._terms(rows_pad)
                kw = {"chunk": self.layer_chunk[k]} if self._is_device() else {}
                self._solver.solve(self.local["items"], self.P, mine, 0.0, self.lam2, self.mu,
                                   self.S_t[S0:], self.T_t[S0:], self.tau, rows_loc,
                                   ("layer", k), **kw)
        if self.world > 1:
            dist.all_gather_into_tensor(self.Q, mine, group=self.group)

    def users(self):
        S0 = self.rank * self.umap.S
        mine = self.P[S0:S0 + self.umap.S]
        kw = {"chunk": self.users_chunk} if self._is_device() else {}
        self._solver.solve(self.local["users"], self.Q, mine, 0.0, self.lam2, self.mu, **kw)
        if self.world > 1:
            dist.all_gather_into_tensor(self.P, mine, group=self.group)

    def sweep(self):
        self.item_layers()
        self.users()

    check = ShardedAls.check
    _is_device = ShardedAls._is_device
