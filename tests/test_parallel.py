"""Multi-rank host logic of the row-sharded sweep on CPU ranks over gloo
(world_size 2): nnz-balanced cuts, the padded shard numbering, the in-place
all-gather, and G-invariance (2 ranks == 1 rank, bit for bit).  The per-row
solve is the CPU oracle here (injected; the product uses libmcf + NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1108_2580_b200.parallel import ShardedAls, ShardMap, nnz_balanced_cuts


class OracleSolver:
    """Test-only: solves a local CSR with the float64 oracle."""

    def __init__(self):
        self.fail = None

    def solve(self, lay, fixed, out, lam_c, lam_n):
        csr = (lay.ptr.numpy(), lay.idx.numpy().astype(np.int64),
               lay.val.numpy().astype(np.float64), None)
        D = out.shape[1]
        res, failed = oracle.solve_rows(csr, fixed.double().numpy(), lay.n_rows, lam_c, lam_n)
        assert failed == -1
        out[: lay.n_rows] = torch.from_numpy(res[:, :D]).float()


def _data(seed=0, U=60, I=45, nnz=900, D=6):
    rng = np.random.default_rng(seed)
    keys = rng.choice(U * I, size=nnz, replace=False)
    keys[:40] = np.arange(40) * I + 3            # a hot item
    keys = np.unique(keys)
    rng.shuffle(keys)
    u, i = keys // I, keys % I
    s = rng.integers(0, 101, keys.size).astype(np.float32)
    P0 = rng.normal(0, 0.1, (U, D)).astype(np.float32)
    Q0 = rng.normal(0, 0.1, (I, D)).astype(np.float32)
    return u, i, s, U, I, D, P0, Q0


def test_cuts_balanced_and_cover():
    deg = torch.tensor([5, 1, 1, 1, 9, 0, 0, 3, 2, 2, 8, 1], dtype=torch.int64)
    for w in (1, 2, 3, 4, 8, 20):
        c = nnz_balanced_cuts(deg, w)
        assert c.numel() == w + 1 and c[0] == 0 and c[-1] == deg.numel()
        assert torch.all(c[1:] >= c[:-1])
        loads = [int(deg[c[k]:c[k + 1]].sum()) for k in range(w)]
        assert sum(loads) == int(deg.sum())
        assert max(loads) <= int(deg.sum()) // w + int(deg.max())
    m = ShardMap(nnz_balanced_cuts(deg, 3))
    assert sum(m.sizes) == m.rows == deg.numel()
    assert torch.equal(m.table_index(), torch.arange(deg.numel()))


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u, i, s, U, I, D, P0, Q0 = _data()
        run = ShardedAls(u, i, s, U, I, D, solver=OracleSolver(), device="cpu")
        run.set_factors(P0, Q0)
        for _ in range(2):
            run.sweep(0.0, 0.065)
        P, Q = run.factors()
        if rank == 0:
            results["P"], results["Q"] = P.numpy().copy(), Q.numpy().copy()
            results["nnz_local"] = run.nnz_local
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_sharded_sweep_g_invariant(world):
    # single rank (no process group)
    u, i, s, U, I, D, P0, Q0 = _data()
    run1 = ShardedAls(u, i, s, U, I, D, solver=OracleSolver(), device="cpu")
    run1.set_factors(P0, Q0)
    for _ in range(2):
        run1.sweep(0.0, 0.065)
    P1, Q1 = (t.numpy() for t in run1.factors())
    with mp.Manager() as man:
        res = man.dict()
        mp.spawn(_worker, args=(world, _free_port(), res), nprocs=world, join=True)
        assert np.array_equal(res["P"], P1) and np.array_equal(res["Q"], Q1)
    # and both equal a plain oracle sweep (float32 storage between half-steps)
    P, Q = P0.astype(np.float64), Q0.astype(np.float64)
    for _ in range(2):
        Q, _ = oracle.als_half_step(P, Q, u, i, s, "items", lam_n=0.065)
        Q = Q.astype(np.float32).astype(np.float64)
        P, _ = oracle.als_half_step(P, Q, u, i, s, "users", lam_n=0.065)
        P = P.astype(np.float32).astype(np.float64)
    assert np.array_equal(P1, P.astype(np.float32)) and np.array_equal(Q1, Q.astype(np.float32))


# ---------------------------------------------------------------------------
# ALS-MFITR sharded by taxonomy subtree

class OracleMfitrSolver:
    """Test-only host stand-in for LayoutSolver + mcf_taxonomy_terms (float64
    oracle arithmetic, float32 factor tables)."""

    def __init__(self):
        self.fail = None

    def terms(self, run, table_rows):
        pc, pp, w = run.edges_table
        S, T = oracle.taxonomy_terms(pc, pp, w, run.Q[:, : run.D].double().numpy(), run.imap.rows)
        r = table_rows.to(torch.int64)
        run.S_t[r] = torch.from_numpy(S[r.numpy()]).float()
        run.T_t[r, : run.D] = torch.from_numpy(T[r.numpy()]).float()

    def solve(self, lay, fixed, out, lam_c, lam_n, y_shift=0.0, tax_S=None, tax_T=None, tau=0.0,
              rows=None, rows_key=None):
        csr = (lay.ptr.numpy(), lay.idx.numpy().astype(np.int64),
               lay.val.numpy().astype(np.float64) - y_shift, None)
        D = out.shape[1] if tax_T is None else tax_T.shape[1]
        D = fixed.shape[1] if D is None else D
        n = lay.n_rows
        S = None if tax_S is None else tax_S[:n].double().numpy()
        T = None if tax_T is None else tax_T[:n].double().numpy()
        res, failed = oracle.solve_rows(csr, fixed.double().numpy(), n, lam_c, lam_n,
                                        tax_S=S, tax_T=T, tau=tau)
        assert failed == -1
        sel = torch.arange(n) if rows is None else rows.to(torch.int64)
        out[sel] = torch.from_numpy(res[sel.numpy()]).float()


def _mfitr_data(golden_dir):
    g = np.load(os.path.join(golden_dir, "mfitr_cfg2s.npz"))
    from paper_1108_2580_b200.taxonomy import build_graph_arrays
    graph = build_graph_arrays(g["kind"], g["album_of"], g["artist_link"])
    U, I = int(g["U"]), int(g["I"])
    D = 6
    rng = np.random.default_rng(3)
    P0 = rng.normal(0, 0.1, (U, D)).astype(np.float32)
    Q0 = rng.normal(0, 0.1, (I, D)).astype(np.float32)
    return g, graph, U, I, D, P0, Q0


def _mfitr_run(world_rank_group, golden_dir):
    from paper_1108_2580_b200.parallel import ShardedMfitr
    g, graph, U, I, D, P0, Q0 = _mfitr_data(golden_dir)
    run = ShardedMfitr(g["users"], g["items"], g["scores"], U, I, D, graph, g["w"],
                       float(g["lam2"]), float(g["lam3"]) + float(g["lam4"]), float(g["mu"]),
                       solver=OracleMfitrSolver(), device="cpu")
    run.set_factors(P0, Q0)
    for _ in range(2):
        run.sweep()
    return run


def _mfitr_worker(rank, world, port, golden_dir, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        run = _mfitr_run(None, golden_dir)
        P, Q = run.factors()
        if rank == 0:
            results["P"], results["Q"] = P.numpy().copy(), Q.numpy().copy()
        results[f"nnz{rank}"] = run.nnz_local
        results[f"own{rank}"] = run.imap.owner.copy()
    finally:
        dist.destroy_process_group()


def test_subtree_cuts_keep_every_edge_local():
    from paper_1108_2580_b200.parallel import PermMap, lpt_owner, subtree_components
    from conftest import REPO
    g, graph, U, I, D, P0, Q0 = _mfitr_data(os.path.join(REPO, "tests", "golden"))
    comp = subtree_components(graph, I)
    assert np.all(comp[graph.edge_child] == comp[graph.edge_parent])
    deg = np.bincount(g["items"].astype(np.int64), minlength=I)
    cw = np.bincount(comp, weights=deg).astype(np.int64)
    for world in (1, 2, 3, 8):
        owner = lpt_owner(cw, world)[comp]
        assert np.all(owner[graph.edge_child] == owner[graph.edge_parent])
        loads = np.bincount(owner, weights=deg, minlength=world)
        assert loads.max() <= deg.sum() / world + cw.max()     # LPT bound
        m = PermMap(owner, world, "cpu")
        assert np.array_equal(np.sort(m.table_np), np.arange(I))      # exact, no padding
        for r in range(world):                                         # rank-major blocks
            lo, hi = m.range(r)
            assert np.all(owner[m.global_rows(r).numpy()] == r) and hi - lo == m.counts[r]


@pytest.mark.parametrize("world", [2])
def test_sharded_mfitr_g_invariant_and_oracle(world):
    """2 ranks over gloo == 1 rank, bit for bit; and == the unsharded layered
    ALS-MFITR sweep computed directly with the oracle."""
    from conftest import REPO
    gd = os.path.join(REPO, "tests", "golden")
    run1 = _mfitr_run(None, gd)
    P1, Q1 = (t.numpy() for t in run1.factors())
    with mp.Manager() as man:
        res = man.dict()
        mp.spawn(_mfitr_worker, args=(world, _free_port(), gd, res), nprocs=world, join=True)
        assert np.array_equal(res["P"], P1) and np.array_equal(res["Q"], Q1)
        own = res["own0"]
        assert set(np.unique(own)) == set(range(world))
    # unsharded reference: layered item solves then users, float32 storage
    g, graph, U, I, D, P0, Q0 = _mfitr_data(gd)
    u, i = g["users"].astype(np.int64), g["items"].astype(np.int64)
    s = g["scores"].astype(np.float64) - float(g["mu"])
    lam2, tau = float(g["lam2"]), float(g["lam3"]) + float(g["lam4"])
    icsr = oracle.side_csr(i, u, s, I)
    ucsr = oracle.side_csr(u, i, s, U)
    P, Q = P0.astype(np.float64), Q0.astype(np.float64)
    for _ in range(2):
        for L in graph.layers(I):
            if L.size == 0:
                continue
            S, T = oracle.taxonomy_terms(graph.edge_child, graph.edge_parent, g["w"], Q, I)
            f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731  (S/T tables)
            res, f = oracle.solve_rows(icsr, P, I, 0.0, lam2, tax_S=f32(S), tax_T=f32(T), tau=tau)
            assert f == -1
            Q = Q.copy()
            Q[L] = res[L].astype(np.float32)
        res, f = oracle.solve_rows(ucsr, Q, U, 0.0, lam2)
        P = res.astype(np.float32).astype(np.float64)
    assert np.array_equal(P1, P.astype(np.float32)) and np.array_equal(Q1, Q.astype(np.float32))


# ---------------------------------------------------------------------------
# a failing row on one rank is raised on every rank, as its global row id

class FailingSolver(OracleSolver):
    """Reports local row 1 of the items layout of rank 1 as singular."""

    def __init__(self, rank):
        super().__init__()
        self.rank = rank

    def solve(self, lay, fixed, out, lam_c, lam_n):
        super().solve(lay, fixed, out, lam_c, lam_n)
        bad = self.rank == 1 and out.shape[0] == lay.n_rows and getattr(lay, "side", "") == "items"
        return torch.tensor([1 if bad else -1], dtype=torch.int64)


def _fail_worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1108_2580_b200.errors import SingularSystemError
        u, i, s, U, I, D, P0, Q0 = _data()
        run = ShardedAls(u, i, s, U, I, D, solver=FailingSolver(rank), device="cpu")
        for side, lay in run.local.items():
            lay.side = side
        run.set_factors(P0, Q0)
        run.sweep(0.0, 0.065)
        try:
            run.check()
            results[f"r{rank}"] = "no error"
        except SingularSystemError as e:
            results[f"r{rank}"] = str(e)
        results[f"lo{rank}"] = run.imap.range(1)[0]
    finally:
        dist.destroy_process_group()


def test_sharded_failure_raised_on_every_rank():
    with mp.Manager() as man:
        res = man.dict()
        mp.spawn(_fail_worker, args=(2, _free_port(), res), nprocs=2, join=True)
        row = res["lo0"] + 1                       # rank 1's local row 1, global id
        assert res["r0"] == res["r1"]
        assert f"items row {row}" in res["r0"], res["r0"]
