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
    pad = m.padded_index()
    assert pad.unique().numel() == deg.numel() and int(pad.max()) < m.rows


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
