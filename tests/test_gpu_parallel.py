"""The sharded fit on one GPU (a one-rank NCCL group): the public
factor.train / mfitr.train_mfitr sharded path equals the single-GPU path bit
for bit, libmcf's own communicator initialises and all-gathers, and the
exact-size tables cover every row once.  (Two-GPU G-invariance:
tests/test_multigpu.py, skipped on one-GPU boxes.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture
def one_rank_group():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    yield
    dist.destroy_process_group()


def _split(seed=0, U=3000, I=500, nnz=90_000, D=20):
    rng = np.random.default_rng(seed)
    keys = np.unique(rng.integers(0, U * I, nnz))
    keys = np.unique(np.concatenate([keys, np.arange(U) * I + 7]))     # a hot item
    rng.shuffle(keys)
    u, i = (keys // I).astype(np.int32), (keys % I).astype(np.int32)
    s = rng.integers(0, 101, keys.size).astype(np.float32)
    return u, i, s, U, I, D, rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D))


@pytest.mark.parametrize("D", [20, 32])
def test_sharded_train_equals_train(one_rank_group, D):
    from paper_1108_2580_b200 import factor
    from paper_1108_2580_b200.data import Dataset
    u, i, s, U, I, _, P0, Q0 = _split(D=D)
    P0, Q0 = np.random.default_rng(1).normal(0, 0.1, (U, D)), np.random.default_rng(2).normal(
        0, 0.1, (I, D))
    tr = Dataset.from_arrays(u, i, s, num_users=U, num_items=I)
    va = Dataset.from_arrays(u[:500], i[:500], s[:500], num_users=U, num_items=I)
    hp = factor.HyperParams(lam=0.065, D=D, iters=3)
    m1, r1 = factor.train("wals", tr, va, hp, reg="weighted", init=(P0, Q0))
    model = factor.init_model("wals", tr, hp, 0)
    m2, r2 = factor._train_sharded(model, tr, va, hp, "weighted", (P0, Q0), None, False, True,
                                   "nccl")
    assert np.array_equal(m1.p, m2.p) and np.array_equal(m1.q, m2.q)
    for a, b in zip(r1, r2):
        assert abs(a.valid_rmse - b.valid_rmse) < 1e-12
        assert abs(a.objective - b.objective) <= 1e-9 * abs(a.objective)


def test_mcf_comm_single_rank(one_rank_group):
    """libmcf's communicator (C-ABI mcf_comm_*): unique id, init on this
    device, an all-gather over one rank (no-op), destroy."""
    from paper_1108_2580_b200.parallel import MfcComm, ShardedAls
    comm = MfcComm.from_group(None, torch.device("cuda", torch.cuda.current_device()))
    t = torch.arange(24, dtype=torch.float32, device="cuda").reshape(3, 8)
    before = t.clone()
    comm.allgather_rows(t, [0], [3])
    torch.cuda.synchronize()
    assert torch.equal(t, before)
    u, i, s, U, I, D, P0, Q0 = _split()
    outs = []
    for coll in ("nccl", "mcf"):
        run = ShardedAls(u, i, s, U, I, D, collective=coll, comm=comm if coll == "mcf" else None)
        run.set_factors(P0, Q0)
        run.sweep(0.0, 0.065)
        run.check()
        outs.append([x.clone() for x in run.factors()])
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    del comm


def test_sharded_mfitr_train_equals_single(one_rank_group):
    from paper_1108_2580_b200 import mfitr
    from paper_1108_2580_b200.data import Dataset
    from paper_1108_2580_b200.taxonomy import build_graph_arrays
    g = np.load(os.path.join(HERE, "golden", "mfitr_cfg2s.npz"))
    graph = build_graph_arrays(g["kind"], g["album_of"], g["artist_link"])
    U, I, D = int(g["U"]), int(g["I"]), 8
    tr = Dataset.from_arrays(g["users"], g["items"], g["scores"], num_users=U, num_items=I)
    h = mfitr.MfitrHyper(D=D, lam1=0.0, lam2=float(g["lam2"]), lam3=float(g["lam3"]),
                         lam4=float(g["lam4"]), iters=2)
    rng = np.random.default_rng(4)
    init = (rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D)))
    m1, r1 = mfitr.train_mfitr("mfitr", tr, tr, graph, h, init=init, blocks="q")
    model = mfitr.init_mfitr("mfitr", tr, graph, h, 0)
    model.base.p, model.base.q = init
    ew = mfitr.edge_weights(graph, tr, num_items=I)
    m2, r2 = mfitr._train_mfitr_sharded(
        model, tr, graph, ew, h, torch.device("cuda"),
        tuple(torch.as_tensor(a, device="cuda") for a in (
            tr.users.astype(np.int32), tr.items.astype(np.int32), tr.scores.astype(np.float32))),
        (0.0, 100.0), True, False)
    assert np.array_equal(m1.base.p, m2.base.p) and np.array_equal(m1.base.q, m2.base.q)
    for a, b in zip(r1, r2):
        assert abs(a.objective - b.objective) <= 1e-6 * abs(a.objective)
        assert abs(a.valid_rmse - b.valid_rmse) < 1e-9


def test_multicast_requires_nvls(one_rank_group):
    """collective='multicast' either runs (NVLS present) and equals NCCL, or
    refuses loudly -- never a silent fallback."""
    from paper_1108_2580_b200.errors import ConfigError
    from paper_1108_2580_b200.parallel import ShardedAls
    u, i, s, U, I, D, P0, Q0 = _split(nnz=40_000)
    try:
        run = ShardedAls(u, i, s, U, I, D, collective="multicast")
    except ConfigError as e:
        assert "multicast" in str(e)
        return
    except Exception as e:   # pragma: no cover - symmetric memory unavailable
        pytest.skip(f"symmetric memory unavailable: {e}")
    ref = ShardedAls(u, i, s, U, I, D)
    for r in (run, ref):
        r.set_factors(P0, Q0)
        r.sweep(0.0, 0.065)
        r.check()
    assert torch.equal(run.factors()[0], ref.factors()[0])
