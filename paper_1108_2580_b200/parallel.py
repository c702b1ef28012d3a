"""Row-sharded multi-GPU ALS: one process per GPU, the freshly solved factor
rows of each rank all-gathered after every half-step.

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
* factor tables are EXACT: shard s occupies rows [off_s, off_s + n_s) of the
  [n, ld] table (ALS: the natural row numbering, off_s = cut s), so each
  rank solves its rows in place and the all-gather moves exactly n rows --
  grouped broadcasts of uneven shards, no padding;
* collectives (`collective=`):
    "nccl"      torch.distributed all_gather of the uneven row slices
                (NCCL groups one broadcast per rank);
    "mcf"       the same grouped broadcasts through libmcf's own C-ABI
                communicator (mcf_comm_init / mcf_allgather_rows) -- what a
                non-torch C caller uses;
    "peer"      fused: P/Q in torch symmetric memory and the solve kernel
                stores every solved row into each peer's replica
                (mcf_als_half_step_peers), then a device barrier;
    "multicast" fused: one NVLS multimem store per element into the
                multicast mapping of the symmetric tables
                (mcf_als_half_step_multicast), then a device barrier;
* every row is solved with the same chunking and reduction order as on one
  GPU, so factors are bit-identical for any world size (G-invariance, the
  device analogue of the reference's thread-count invariance);
* a failing row is folded into a per-side accumulator as its GLOBAL row id
  and `check()` all-reduces the minimum over ranks, so every rank raises the
  same SingularSystemError (no rank left waiting in the next collective).

`solver` is pluggable so the host-side logic (cuts, numbering, gather,
failure reduction) can be exercised on CPU ranks over gloo; the product path
uses the device solver (libmcf) and NCCL.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .errors import ConfigError, SingularSystemError

NO_FAIL = torch.iinfo(torch.int64).max
COLLECTIVES = ("nccl", "mcf", "peer", "multicast")


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
    """Contiguous row ranges in the natural numbering: shard s = rows
    [cuts[s], cuts[s+1]); the factor table is indexed by global row id."""

    def __init__(self, cuts: torch.Tensor):
        self.cuts = cuts
        self.world = int(cuts.numel()) - 1
        c = [int(x) for x in cuts.tolist()]
        self.offsets = c[:-1]
        self.sizes = [c[k + 1] - c[k] for k in range(self.world)]
        self.rows = c[-1]

    def range(self, r: int):
        return self.offsets[r], self.offsets[r] + self.sizes[r]

    def to_table(self, ids: torch.Tensor) -> torch.Tensor:
        return ids.to(torch.int32)

    def table_index(self) -> torch.Tensor:
        """Table row of every global row (int64 [n])."""
        return torch.arange(self.rows, device=self.cuts.device)

    def global_rows(self, r: int) -> torch.Tensor:
        lo, hi = self.range(r)
        return torch.arange(lo, hi, device=self.cuts.device)


class PermMap:
    """Exact rank-major numbering for an arbitrary row -> rank assignment:
    rank r's rows (ascending id) occupy [off_r, off_r + n_r) of an [n] table."""

    def __init__(self, owner: np.ndarray, world: int, device):
        owner = np.asarray(owner, np.int64)
        self.world, self.n = int(world), int(owner.size)
        counts = np.bincount(owner, minlength=world)
        self.counts = counts
        self.sizes = [int(x) for x in counts]
        starts = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
        self.offsets = [int(x) for x in starts]
        self.rows = self.n
        order = np.lexsort((np.arange(self.n), owner))           # by rank, then id
        local = np.empty(self.n, dtype=np.int64)
        local[order] = np.arange(self.n) - np.repeat(starts, counts)
        self.owner, self.local = owner, local
        self.table_np = starts[owner] + local
        self.table = torch.as_tensor(self.table_np, device=device)
        self._by_rank = order          # global ids in table order

    def range(self, r: int):
        return self.offsets[r], self.offsets[r] + self.sizes[r]

    def to_table(self, ids: torch.Tensor) -> torch.Tensor:
        return self.table[ids.to(torch.int64)].to(torch.int32)

    def table_index(self) -> torch.Tensor:
        return self.table

    def global_rows(self, r: int) -> torch.Tensor:
        lo, hi = self.range(r)
        return torch.as_tensor(self._by_rank[lo:hi], device=self.table.device)


def allgather_rows(table: torch.Tensor, mp, group=None, comm=None) -> None:
    """Every rank's rows [off_r, off_r + n_r) of `table` to every rank, in
    place and exact (uneven shards, no padding)."""
    world = mp.world
    if world <= 1:
        return
    if comm is not None:            # libmcf's own communicator (C-ABI)
        comm.allgather_rows(table, mp.offsets, mp.sizes)
        return
    parts = [table[o:o + n] for o, n in zip(mp.offsets, mp.sizes)]
    rank = dist.get_rank(group)
    if dist.get_backend(group) == "nccl":
        # NCCL: uneven all_gather = one grouped ncclBroadcast per rank
        dist.all_gather(parts, parts[rank], group=group)
    else:                           # gloo (host-logic tests): broadcast per rank
        for k in range(world):
            if mp.sizes[k]:
                dist.broadcast(parts[k], src=dist.get_global_rank(group, k)
                               if group is not None else k, group=group)


class _FailAcc:
    """Per-side first failing GLOBAL row since the last check()."""

    def __init__(self, device):
        self.acc = torch.full((2,), NO_FAIL, dtype=torch.int64, device=device)

    def fold(self, k: int, fail, global_rows: torch.Tensor):
        if not isinstance(fail, torch.Tensor):
            return
        f = fail.reshape(-1)[:1].to(self.acc.device)
        g = global_rows[f.clamp(min=0)] if global_rows.numel() else f
        g = torch.where(f >= 0, g, torch.full_like(f, NO_FAIL))
        torch.minimum(self.acc[k:k + 1], g, out=self.acc[k:k + 1])

    def check(self, group, world, sides=("items", "users")):
        acc = self.acc.clone()
        self.acc.fill_(NO_FAIL)
        if world > 1:
            dist.all_reduce(acc, op=dist.ReduceOp.MIN, group=group)
        for side, row in zip(sides, acc.tolist()):
            if row != NO_FAIL:
                raise SingularSystemError(
                    f"singular normal equations at {side} row {row}; use lam > 0")


class ShardedAls:
    """One rank's part of a row-sharded ALS fit."""

    def __init__(self, users, items, scores, num_users: int, num_items: int, D: int, *,
                 group=None, solver="device", device=None, chunk: int | None = None,
                 collective: str = "nccl", comm=None):
        if collective not in COLLECTIVES:
            raise ConfigError(f"collective must be one of {COLLECTIVES}, got {collective!r}")
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
        self.comm = comm
        if collective == "mcf" and comm is None and self.world > 1:
            self.comm = MfcComm.from_group(group, dev)
        self._peers, self._handles, self._mc = {}, {}, {}
        if collective in ("peer", "multicast"):
            self.P, self.Q = self._symmetric_tables(dev)
        else:
            self.P = torch.zeros(self.umap.rows, self.ld, dtype=torch.float32, device=dev)
            self.Q = torch.zeros(self.imap.rows, self.ld, dtype=torch.float32, device=dev)
        # local layouts: my users (partners = item table rows), my items
        self.local = {}
        for side, keys, cols, kmap, cmap in (("users", u, it, self.umap, self.imap),
                                             ("items", it, u, self.imap, self.umap)):
            lo, hi = kmap.range(self.rank)
            m = (keys >= lo) & (keys < hi)
            k_loc = (keys[m] - lo).to(torch.int32)
            self.local[side] = self._make_layout(k_loc, cmap.to_table(cols[m]), s[m], hi - lo)
        self.nnz_local = {k: int(v.nnz) for k, v in self.local.items()}
        self.fixed_chunk = global_chunk(int(u.numel()), self.D, chunk)
        self._rows = {"users": self.umap.global_rows(self.rank),
                      "items": self.imap.global_rows(self.rank)}
        self._fail = _FailAcc(dev)

    def _symmetric_tables(self, dev):
        """P, Q in symmetric memory; per side the device array of the peers'
        replica pointers (peer) or the multicast address (multicast), offset
        to this rank's shard."""
        import torch.distributed._symmetric_memory as symm_mem
        group = self.group if self.group is not None else dist.group.WORLD
        name = group.group_name
        if hasattr(symm_mem, "enable_symm_mem_for_group"):
            symm_mem.enable_symm_mem_for_group(name)
        tabs = []
        for side, mp in (("users", self.umap), ("items", self.imap)):
            t = symm_mem.empty(max(mp.rows, 1), self.ld, dtype=torch.float32, device=dev)
            t.zero_()
            h = symm_mem.rendezvous(t, name)
            off = mp.offsets[self.rank] * self.ld * 4
            if self.collective == "multicast":
                mc = int(getattr(h, "multicast_ptr", 0) or 0)
                if not mc:
                    raise ConfigError("collective='multicast' needs NVLS multicast support "
                                      "(symmetric memory reports none on this system)")
                self._mc[side] = mc + off
            ptrs = [int(h.buffer_ptrs[k]) + off for k in range(self.world) if k != self.rank]
            self._peers[side] = torch.tensor(ptrs, dtype=torch.int64, device=dev)
            self._handles[side] = h
            tabs.append(t[: mp.rows])
        return tabs

    def _is_device(self):
        return self._solver.__class__.__name__ == "LayoutSolver"

    def _make_layout(self, keys, cols, vals, n_rows):
        if self._is_device():
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
            dst[mp.table_index(), : self.D] = t

    def factors(self):
        """(P, Q) in global row order, [n, D] views of the tables."""
        return (self.P[self.umap.table_index(), : self.D],
                self.Q[self.imap.table_index(), : self.D])

    # -- sweep ---------------------------------------------------------------
    def half_step(self, side: str, lam_c: float = 0.0, lam_n: float = 0.0, gather: bool = True,
                  obj_out: torch.Tensor | None = None):
        if side not in ("users", "items"):
            raise ConfigError(f"side must be 'users' or 'items', got {side!r}")
        out_full, fixed, mp = ((self.P, self.Q, self.umap) if side == "users"
                               else (self.Q, self.P, self.imap))
        lo, hi = mp.range(self.rank)
        mine = out_full[lo:hi]
        if self.collective in ("peer", "multicast"):
            # fused: the kernel itself writes every solved row into each
            # replica (peer stores or one multimem store); the barrier orders
            # the next half-step after all ranks' stores
            kw = ({"multicast": self._mc[side]} if self.collective == "multicast"
                  else {"peers": self._peers[side]})
            fail = self._solver.solve(self.local[side], fixed, mine, lam_c, lam_n,
                                      chunk=self.fixed_chunk, obj_out=obj_out, **kw)
            self._fail.fold(0 if side == "items" else 1, fail, self._rows[side])
            if gather and self.world > 1:
                self._handles[side].barrier(channel=0)
            return out_full
        kw = {"chunk": self.fixed_chunk, "obj_out": obj_out} if self._is_device() else {}
        fail = self._solver.solve(self.local[side], fixed, mine, lam_c, lam_n, **kw)
        self._fail.fold(0 if side == "items" else 1, fail, self._rows[side])
        if gather and self.world > 1:
            allgather_rows(out_full, mp, self.group, self.comm)
        return out_full

    def sweep(self, lam_c: float = 0.0, lam_n: float = 0.0, obj: torch.Tensor | None = None):
        self.half_step("items", lam_c, lam_n, obj_out=None if obj is None else obj[0:2])
        self.half_step("users", lam_c, lam_n, obj_out=None if obj is None else obj[2:4])

    def check(self):
        """Raise SingularSystemError with the minimum failing global row of
        the first failing side, on every rank (all-reduce MIN)."""
        self._fail.check(self.group, self.world)


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
# libmcf's own communicator (C-ABI mcf_comm_*; NCCL loaded by libmcf)

class MfcComm:
    """Thin owner of an mcf_comm_t: NCCL communicator created by libmcf from
    a unique id (rank 0 creates it, torch.distributed or any other channel
    ships the 128 bytes), used for the exact-size row all-gather."""

    def __init__(self, unique_id: bytes, world: int, rank: int, device):
        import ctypes
        from ._lib import check
        self.world, self.rank, self.device = int(world), int(rank), device
        self._h = ctypes.c_void_p()
        buf = (ctypes.c_char * len(unique_id)).from_buffer_copy(unique_id)
        with torch.cuda.device(device):
            check(_lib.lib().mcf_comm_init(buf, len(unique_id), self.world, self.rank,
                                           ctypes.byref(self._h)), "mcf_comm_init")

    @classmethod
    def unique_id(cls) -> bytes:
        import ctypes
        from ._lib import check
        n = int(_lib.lib().mcf_comm_id_bytes())
        buf = (ctypes.c_char * n)()
        check(_lib.lib().mcf_comm_get_unique_id(buf, n), "mcf_comm_get_unique_id")
        return bytes(buf)

    @classmethod
    def from_group(cls, group, device) -> "MfcComm":
        rank = dist.get_rank(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None
                                   else 0, group=group)
        return cls(obj[0], dist.get_world_size(group), rank, device)

    def allgather_rows(self, table: torch.Tensor, offsets, sizes):
        import ctypes
        from ._lib import check
        from .device import stream_ptr
        off = (ctypes.c_int64 * len(offsets))(*offsets)
        cnt = (ctypes.c_int64 * len(sizes))(*sizes)
        check(_lib.lib().mcf_allgather_rows(self._h, table.data_ptr(), table.shape[1], off, cnt,
                                            stream_ptr(self.device)), "mcf_allgather_rows")

    def __del__(self):
        try:
            if self._h:
                _lib.lib().mcf_comm_destroy(self._h)
        except Exception:
            pass


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


class ShardedMfitr:
    """One rank's part of a sharded ALS-MFITR fit (factor blocks; biases and
    q_a at 0, as MfitrSolver): users cut at nnz quantiles, items assigned by
    whole taxonomy subtree (LPT on their ratings) in an exact rank-major
    numbering, the layered item half-step solved locally with S/T from the
    local subtrees, one exact all-gather per half-step.  Results are
    identical for any world size."""

    def __init__(self, users, items, scores, num_users: int, num_items: int, D: int, graph,
                 w, lam2: float, tau: float, mu: float, *, group=None, solver="device",
                 device=None, chunk: int | None = None, comm=None):
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
        self.comm = comm
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
        self.local = {"users": mk(self, (u[m] - lo).to(torch.int32), self.imap.to_table(it[m]),
                                  s[m], hi - lo)}
        own = torch.as_tensor(self.imap.owner, device=dev)[it] == self.rank
        loc = torch.as_tensor(self.imap.local, device=dev)
        n_mine = int(self.imap.counts[self.rank])
        self.local["items"] = mk(self, loc[it[own]].to(torch.int32), self.umap.to_table(u[own]),
                                 s[own], n_mine)
        self.nnz_local = {k: int(v.nnz) for k, v in self.local.items()}
        # taxonomy in item-table rows: incident-edge CSR (edge-list order per
        # item, as TaxonomyGraph.incident_edges), edge weights
        pc, pp = self.imap.table_np[graph.edge_child], self.imap.table_np[graph.edge_parent]
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
        self.edges_table = (pc, pp, np.asarray(w, np.float64))
        # my rows of each layer: local and table indices
        mine = self.imap.owner == self.rank
        self.layers, self.layer_chunk = [], []
        self.users_chunk = global_chunk(int(u.numel()), self.D, chunk)
        off = self.imap.offsets[self.rank]
        for L in graph.layers(num_items):
            # task length from the GLOBAL layer size: identical on every rank,
            # so hot-row chunk sums (and results) do not depend on world size
            self.layer_chunk.append(global_chunk(int(deg[L].sum()), self.D, chunk))
            Lm = L[mine[L]]
            loc_rows = np.sort(self.imap.local[Lm])
            self.layers.append((torch.as_tensor(loc_rows.astype(np.int32), device=dev),
                                torch.as_tensor((off + loc_rows).astype(np.int32), device=dev)))
        self.S_t = torch.zeros(self.imap.rows, dtype=torch.float32, device=dev)
        self.T_t = torch.zeros(self.imap.rows, self.ld, dtype=torch.float32, device=dev)
        self._rows = {"users": self.umap.global_rows(self.rank),
                      "items": self.imap.global_rows(self.rank)}
        self._fail = _FailAcc(dev)

    # -- factors -------------------------------------------------------------
    def set_factors(self, P=None, Q=None):
        for dst, src, idx in ((self.P, P, self.umap.table_index()),
                              (self.Q, Q, self.imap.table_index())):
            if src is None:
                continue
            t = torch.as_tensor(np.asarray(src) if not isinstance(src, torch.Tensor) else src)
            dst.zero_()
            dst[idx, : self.D] = t.to(self.device, torch.float32)

    def factors(self):
        return (self.P[self.umap.table_index(), : self.D],
                self.Q[self.imap.table_index(), : self.D])

    # -- sweep ---------------------------------------------------------------
    def _terms(self, table_rows):
        if self._is_device():
            from ._lib import check, ptr
            from .device import stream_ptr
            ip, ie, io = self.inc
            check(_lib.lib().mcf_taxonomy_terms(ptr(ip), ptr(ie), ptr(io), ptr(self.w),
                                                ptr(self.Q), self.imap.rows, self.D,
                                                ptr(table_rows), table_rows.numel(),
                                                ptr(self.S_t), ptr(self.T_t),
                                                stream_ptr(self.device)), "mcf_taxonomy_terms")
        else:   # host stand-in (tests): the same sums, float32 tables
            self._solver.terms(self, table_rows)

    def item_layers(self):
        S0, n = self.imap.range(self.rank)
        mine = self.Q[S0:n]
        for k, (rows_loc, rows_tab) in enumerate(self.layers):
            if rows_loc.numel():
                self._terms(rows_tab)
                kw = {"chunk": self.layer_chunk[k]} if self._is_device() else {}
                fail = self._solver.solve(self.local["items"], self.P, mine, 0.0, self.lam2,
                                          self.mu, self.S_t[S0:], self.T_t[S0:], self.tau,
                                          rows_loc, ("layer", k), **kw)
                self._fail.fold(0, fail, self._rows["items"])
        if self.world > 1:
            allgather_rows(self.Q, self.imap, self.group, self.comm)

    def users(self):
        S0, n = self.umap.range(self.rank)
        mine = self.P[S0:n]
        kw = {"chunk": self.users_chunk} if self._is_device() else {}
        fail = self._solver.solve(self.local["users"], self.Q, mine, 0.0, self.lam2, self.mu,
                                  **kw)
        self._fail.fold(1, fail, self._rows["users"])
        if self.world > 1:
            allgather_rows(self.P, self.umap, self.group, self.comm)

    def sweep(self):
        self.item_layers()
        self.users()

    check = ShardedAls.check
    _is_device = ShardedAls._is_device
