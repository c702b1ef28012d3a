"""GPU parity of the MFITR path: device edge weights (bit-exact), the
segmented S/T reduction, the layered ALS-MFITR item solve (zero gradient on
each solved layer, re-anchored factors within 1e-4), the drop-in trainer."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def dev():
    assert torch.cuda.is_available()
    return torch.device("cuda")


def _graph(g):
    from paper_1108_2580_b200.taxonomy import build_graph_arrays
    return build_graph_arrays(g["kind"], g["album_of"], g["artist_link"])


def _train(g):
    from paper_1108_2580_b200.data import Dataset
    return Dataset.from_arrays(g["users"], g["items"], g["scores"], num_users=int(g["U"]),
                               num_items=int(g["I"]), compact=True)


def test_edge_weights_bit_exact_golden(golden):
    from paper_1108_2580_b200 import mfitr
    g = golden("mfitr_cfg2s.npz")
    graph = _graph(g)
    assert np.array_equal(graph.edge_child, g["ec"]) and np.array_equal(graph.edge_parent, g["ep"])
    ew = mfitr.edge_weights(graph, _train(g), device=dev())
    assert np.array_equal(ew.w, g["w"])          # the reference's own weights, bit for bit


def test_edge_weights_bit_exact_larger():
    from paper_1108_2580_b200 import mfitr, synth
    wl = synth.generate(synth.scaled_config(synth.CONFIGS[2], 0.01), seed=2)
    tr = wl.train_dataset()
    ew = mfitr.edge_weights(wl.graph, tr, device=dev())
    ref = oracle.edge_weights(wl.graph.edge_child, wl.graph.edge_parent, tr.users, tr.items,
                              tr.scores, tr.num_users, tr.num_items)
    assert np.array_equal(ew.w, ref)
    assert (ew.w > 0).mean() > 0.1


def _solver(g, D=None):
    from paper_1108_2580_b200 import mfitr
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings
    U, I = int(g["U"]), int(g["I"])
    r = DeviceRatings(g["users"], g["items"], g["scores"], U, I, dev())
    eng = AlsEngine(r, g["P"].shape[1])
    eng.set_factors(g["P"], g["Q"])
    h = mfitr.MfitrHyper(D=g["P"].shape[1], lam1=0.0, lam2=float(g["lam2"]),
                         lam3=float(g["lam3"]), lam4=float(g["lam4"]))
    return mfitr.MfitrSolver(eng, _graph(g), g["w"], h, float(g["mu"])), eng


def test_taxonomy_terms_match_oracle(golden):
    g = golden("mfitr_cfg2s.npz")
    solver, eng = _solver(g)
    from paper_1108_2580_b200 import _lib
    from paper_1108_2580_b200.device import stream_ptr
    I = int(g["I"])
    _lib.check(_lib.lib().mcf_taxonomy_terms(
        solver.inc_ptr.data_ptr(), solver.inc_edge.data_ptr(), solver.inc_other.data_ptr(),
        solver.w.data_ptr(), eng.Q.data_ptr(), I, eng.D, None, 0, solver.S.data_ptr(),
        solver.T.data_ptr(), stream_ptr(eng.device)), "terms")
    S, T = oracle.taxonomy_terms(g["ec"], g["ep"], g["w"], eng.factors()[1].double().cpu().numpy(), I)
    np.testing.assert_allclose(solver.S.cpu().numpy(), S, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(solver.T[:, : eng.D].cpu().numpy(), T, rtol=1e-5, atol=1e-6)


def test_layered_item_half_step_reanchored(golden):
    g = golden("mfitr_cfg2s.npz")
    solver, eng = _solver(g)
    U, I = int(g["U"]), int(g["I"])
    u, i = g["users"].astype(np.int64), g["items"].astype(np.int64)
    s = g["scores"].astype(np.float64)
    mu, l2 = float(g["mu"]), float(g["lam2"])
    tau = float(g["lam3"]) + float(g["lam4"])
    csr = oracle.side_csr(i, u, s - mu, I)
    z = np.zeros(I)
    for rows_t in solver.layers:
        rows = rows_t.cpu().numpy()
        P, Q = (t.double().cpu().numpy() for t in eng.factors())
        S, T = oracle.taxonomy_terms(g["ec"], g["ep"], g["w"], Q, I)
        ref, failed = oracle.solve_rows(csr, P, I, lam_n=l2, tax_S=S, tax_T=T, tau=tau)
        assert failed == -1
        # one device layer
        from paper_1108_2580_b200 import _lib
        from paper_1108_2580_b200.device import stream_ptr
        _lib.check(_lib.lib().mcf_taxonomy_terms(
            solver.inc_ptr.data_ptr(), solver.inc_edge.data_ptr(), solver.inc_other.data_ptr(),
            solver.w.data_ptr(), eng.Q.data_ptr(), I, eng.D, rows_t.data_ptr(), rows_t.numel(),
            solver.S.data_ptr(), solver.T.data_ptr(), stream_ptr(eng.device)), "terms")
        eng.half_step("items", 0.0, l2, mu, solver.S, solver.T, tau, rows=rows_t,
                      rows_key=("t", rows.size))
        eng.check()
        got = eng.factors()[1].double().cpu().numpy()
        if rows.size:
            d = np.abs(got[rows] - ref[rows]).max() / max(np.abs(ref[rows]).max(), 1e-30)
            assert d < 1e-4, d
        others = np.setdiff1d(np.arange(I), rows)
        assert np.array_equal(got[others], Q[others])     # only the layer moves
        gq = oracle.grad_mfitr(P, got, u, i, s, mu, np.zeros(U), z, g["art"], z,
                               np.zeros_like(got), g["ec"], g["ep"], g["w"], 0.0, l2,
                               float(g["lam3"]), float(g["lam4"]))["q"]
        scale = np.abs(g["grad_q"]).max()
        if rows.size:
            assert np.abs(gq[rows]).max() < 1e-4 * scale


def test_zero_taxonomy_weight_reduces_to_weighted_als(golden):
    g = golden("mfitr_cfg2s.npz")
    solver, eng = _solver(g)
    solver.tau = 0.0
    U, I = int(g["U"]), int(g["I"])
    P, Q = (t.double().cpu().numpy() for t in eng.factors())
    solver.item_layers()
    eng.check()
    u, i = g["users"].astype(np.int64), g["items"].astype(np.int64)
    s = g["scores"].astype(np.float64) - float(g["mu"])
    ref, _ = oracle.als_half_step(P, Q, u, i, s, "items", lam_n=float(g["lam2"]))
    got = eng.factors()[1].double().cpu().numpy()
    assert np.abs(got - ref).max() < 1e-4 * np.abs(ref).max()


def test_train_mfitr_drop_in(golden):
    from paper_1108_2580_b200 import mfitr, registry
    g = golden("mfitr_cfg2s.npz")
    graph = _graph(g)
    tr = _train(g)
    h = mfitr.MfitrHyper(D=8, lam1=0.0, lam2=0.065, lam3=0.1, lam4=0.1, iters=4)
    tm = registry.train_model("mfitr", tr, h, seed=0, taxonomy=graph, validation=tr)
    rep = tm.report
    objs = np.array([r.objective for r in rep])
    assert np.all(np.isfinite(objs)) and np.all(np.diff(objs) <= 1e-5 * objs[:-1])
    m = tm.model
    pred = tm.predict(g["users"][:500], g["items"][:500])
    ref = oracle.predict(m.base.p, m.base.q, g["users"][:500], g["items"][:500], mu=m.base.mu,
                         b_u=m.base.b_u, b_i=m.base.b_i,
                         arts=m.artist_of_item[g["items"][:500]],   # per query (mf_predict_batch)
                         b_a=m.b_a, Q_a=m.q_a)
    assert np.abs(pred - ref).max() < 1e-4 * np.abs(ref).max()
    assert np.array_equal(tm.model.ew.w, g["w"])
    # the full model trains every block (biases and artist offsets move)
    assert np.abs(m.base.b_u).max() > 0 and np.abs(m.q_a).max() > 0
    # the reported objective is the oracle's loss_mfitr of the returned model
    u, i = g["users"].astype(np.int64), g["items"].astype(np.int64)
    ref_loss = oracle.loss_mfitr(m.base.p, m.base.q, u, i, g["scores"], m.base.mu, m.base.b_u,
                                 m.base.b_i, m.artist_of_item, m.b_a, m.q_a, g["ec"], g["ep"],
                                 g["w"], h.lam1, h.lam2, h.lam3, h.lam4)
    assert abs(objs[-1] - ref_loss) < 1e-4 * ref_loss


def test_train_mfitr_q_blocks_only(golden):
    from paper_1108_2580_b200 import mfitr
    g = golden("mfitr_cfg2s.npz")
    h = mfitr.MfitrHyper(D=8, lam1=0.0, lam2=0.065, lam3=0.1, lam4=0.1, iters=3)
    m, rep = mfitr.train_mfitr("mfitr", _train(g), None, _graph(g), h, blocks="q")
    assert np.all(m.base.b_u == 0) and np.all(m.q_a == 0)
    objs = np.array([r.objective for r in rep])
    assert np.all(np.diff(objs) <= 1e-5 * objs[:-1])


def _full_solver(g, D=None):
    from paper_1108_2580_b200.device import DeviceRatings
    from paper_1108_2580_b200 import mfitr
    graph = _graph(g)
    U, I = int(g["U"]), int(g["I"])
    D = D or g["P"].shape[1]
    h = mfitr.MfitrHyper(D=D, lam1=float(g["lam1"]), lam2=float(g["lam2"]),
                         lam3=float(g["lam3"]), lam4=float(g["lam4"]))
    r = DeviceRatings(g["users"], g["items"], g["scores"], U, I, dev())
    return mfitr.MfitrFullSolver(r, graph, g["w"], h, float(g["mu"]), g["art"], g["P"], g["Q"],
                                 g["Qa"], g["bu"], g["bi"], g["ba"], chunk=64)


def _host_params(fs):
    return [t.double().cpu().numpy() for t in fs.params()]


@pytest.mark.parametrize("fixture,D", [("mfitr.npz", None), ("mfitr_cfg2s.npz", None),
                                       ("mfitr_cfg2s.npz", 20), ("mfitr_cfg2s.npz", 24),
                                       ("mfitr_cfg2s.npz", 40)])
def test_full_blocks_zero_gradient_and_monotone(golden, fixture, D):
    """MFITR full blocks: every block solve is exact, so the
    reference's own gradient (grad_mfitr, restated in oracle/ and pinned to
    the reference's values) of the solved block vanishes, and loss_mfitr
    never increases; the device loss matches the oracle's."""
    g = golden(fixture)
    if "Qa" not in g.files:   # cfg2s fixture: start from its factors, biases / q_a at 0
        g = dict(g)
        g["Qa"] = np.zeros_like(g["Q"])
        g["bu"], g["bi"], g["ba"] = np.zeros(int(g["U"])), np.zeros(int(g["I"])), np.zeros(int(g["I"]))
        g["lam1"] = 0.01
    if D is not None:   # wider factors: the warp (D+1 <= 28) and tile-warp paths
        rng = np.random.default_rng(D)
        g["P"] = rng.normal(0, 0.1, (int(g["U"]), D))
        g["Q"] = rng.normal(0, 0.1, (int(g["I"]), D))
        g["Qa"] = np.zeros_like(g["Q"])
    fs = _full_solver(g)
    u, i = g["users"].astype(np.int64), g["items"].astype(np.int64)
    s = g["scores"].astype(np.float64)
    lam = [float(g[k]) for k in ("lam1", "lam2", "lam3", "lam4")]

    def terms():
        P, Q, bu, bi, ba, Qa = _host_params(fs)
        a = (P, Q, u, i, s, float(g["mu"]), bu, bi, g["art"], ba, Qa, g["ec"], g["ep"], g["w"],
             *lam)
        return oracle.loss_mfitr(*a), oracle.grad_mfitr(*a)

    loss0, gr0 = terms()
    scale = {k: max(np.abs(v).max(), 1e-12) for k, v in gr0.items()}
    dev_loss = float(fs.loss().item())
    assert abs(dev_loss - loss0) < 1e-4 * abs(loss0), (dev_loss, loss0)
    prev = loss0
    arts = np.unique(g["art"][g["art"] >= 0])
    for k, layer in enumerate(fs.layers):
        rows = layer.cpu().numpy()
        if rows.size == 0:
            continue
        fs.item_layer(k)
        fs.check()
        loss, gr = terms()
        assert loss <= prev * (1 + 1e-6), ("items layer", loss, prev)
        prev = loss
        assert np.abs(gr["q"][rows]).max() < 1e-4 * scale["q"]
        assert np.abs(gr["b_i"][rows]).max() < 1e-4 * scale["b_i"]
    fs.artists()
    fs.check()
    loss, gr = terms()
    assert loss <= prev * (1 + 1e-6), ("artists", loss, prev)
    prev = loss
    assert np.abs(gr["q_a"][arts]).max() < 1e-4 * scale["q_a"]
    assert np.abs(gr["b_a"][arts]).max() < 1e-4 * scale["b_a"]
    fs.users()
    fs.check()
    loss, gr = terms()
    assert loss <= prev * (1 + 1e-6), ("users", loss, prev)
    assert np.abs(gr["p"]).max() < 1e-4 * scale["p"]
    assert np.abs(gr["b_u"]).max() < 1e-4 * scale["b_u"]
    dev_loss = float(fs.loss().item())
    assert abs(dev_loss - loss) < 1e-4 * abs(loss), (dev_loss, loss)


def test_sharded_mfitr_device_world1_matches_solver(golden):
    """The subtree-sharded runner on one GPU (no process group) reproduces
    MfitrSolver bit for bit (same layouts, plans, kernels)."""
    from paper_1108_2580_b200 import mfitr
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings
    from paper_1108_2580_b200.parallel import ShardedMfitr
    g = golden("mfitr_cfg2s.npz")
    graph = _graph(g)
    U, I, D = int(g["U"]), int(g["I"]), 8
    rng = np.random.default_rng(5)
    P0, Q0 = rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D))
    lam2, tau, mu = float(g["lam2"]), float(g["lam3"]) + float(g["lam4"]), float(g["mu"])
    run = ShardedMfitr(g["users"], g["items"], g["scores"], U, I, D, graph, g["w"], lam2, tau,
                       mu, chunk=64)
    run.set_factors(P0, Q0)
    r = DeviceRatings(g["users"], g["items"], g["scores"], U, I, dev())
    eng = AlsEngine(r, D, chunk=64)
    eng.set_factors(P0, Q0)
    h = mfitr.MfitrHyper(D=D, lam1=0.0, lam2=lam2, lam3=float(g["lam3"]), lam4=float(g["lam4"]))
    solver = mfitr.MfitrSolver(eng, graph, g["w"], h, mu)
    for _ in range(2):
        run.sweep()
        solver.sweep()
    run.check()
    eng.check()
    P1, Q1 = run.factors()
    P2, Q2 = eng.factors()
    assert torch.equal(P1, P2) and torch.equal(Q1, Q2)


def test_schur_bias_equals_coordinate_bias(golden, monkeypatch):
    """The pair kernel's Schur-complement bias (D + 1 <= 21, D = 20 here) and
    the plain bias-coordinate solve (MCF_NO_SCHUR: the 4x4-tile warp kernel
    on D + 1) give the same blocks to fp32 accuracy."""
    g = dict(golden("mfitr_cfg2s.npz"))
    rng = np.random.default_rng(20)
    U, I, D = int(g["U"]), int(g["I"]), 20
    g["P"], g["Q"] = rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D))
    g["Qa"] = rng.normal(0, 0.05, (I, D))
    g["bu"], g["bi"], g["ba"] = rng.normal(0, 1, U), rng.normal(0, 1, I), rng.normal(0, 1, I)
    g["lam1"] = 0.02
    outs = []
    for no_schur in (False, True):
        if no_schur:
            monkeypatch.setenv("MCF_NO_SCHUR", "1")
        fs = _full_solver(g)
        fs.sweep()
        fs.check()
        outs.append(_host_params(fs))
    for a, b in zip(*outs):
        assert np.abs(a - b).max() <= 1e-4 * max(np.abs(b).max(), 1e-6)


def test_mfitr_sgd_trainer_follows_reference(golden):
    """train_mfitr(method="sgd"): the reference's own SGD trainer on device
    (same seeded init and user shuffles, rate_update + edge pass, gamma
    decay; Hogwild across users) tracks the reference trainer's per-epoch
    loss and validation RMSE (tests/golden/mfitr_sgd.npz, made by running
    mfitr.train_mfitr itself)."""
    from paper_1108_2580_b200 import mfitr
    from paper_1108_2580_b200.data import Dataset
    g = golden("mfitr_sgd.npz")
    f = golden("mfitr.npz")
    graph = _graph(f)
    tr = _train(f)
    va = Dataset.from_arrays(g["vu"], g["vi"], g["vs"], num_users=int(f["U"]),
                             num_items=int(f["I"]), compact=True)
    h = mfitr.MfitrHyper(D=4, lam1=float(g["lam1"]), lam2=float(g["lam2"]),
                         lam3=float(g["lam3"]), lam4=float(g["lam4"]), gamma=float(g["gamma0"]),
                         decay=float(g["decay"]), iters=3)
    # one worker: the reference's strictly sequential order -> fp32 rounding only
    m, rep = mfitr.train_mfitr("mfitr", tr, va, graph, h, seed=int(g["seed"]), method="sgd",
                               sgd_workers=1)
    loss = np.array([r.objective for r in rep])
    rmse = np.array([r.valid_rmse for r in rep])
    gam = np.array([r.gamma for r in rep])
    np.testing.assert_allclose(gam, g["gamma"], rtol=1e-6)
    np.testing.assert_allclose(loss, g["loss"], rtol=2e-3)
    np.testing.assert_allclose(rmse, g["rmse"], rtol=2e-3)
    for a, b in ((m.base.p, "P"), (m.base.q, "Q"), (m.b_a, "ba"), (m.base.b_u, "bu")):
        assert np.abs(a - g[b]).max() < 2e-3 * np.abs(g[b]).max(), b
    # the whole GPU, Hogwild across users: still a descent on every epoch
    m2, rep2 = mfitr.train_mfitr("mfitr", tr, va, graph, h, seed=int(g["seed"]), method="sgd",
                                 sgd_conflicts="hogwild")
    loss2 = np.array([r.objective for r in rep2])
    assert np.all(np.isfinite(loss2)) and np.all(np.diff(loss2) < 0)


def test_lock_table_no_lost_updates_no_deadlock():
    """The LockTable contract (reference parallel.py:21-49, SPEC.md:574-575
    and 698): workers increment lock-protected accumulators non-atomically,
    lock pairs taken in ascending id order -- a single shared item under
    heavy contention and many pairs over a few items; every update lands,
    every lock is released, nothing deadlocks."""
    import torch
    from paper_1108_2580_b200 import _lib
    L = _lib.lib()
    for n_items, workers, iters in ((1, 16, 2000), (1, 4096, 20), (8, 4096, 50), (101, 9472, 20)):
        locks = torch.zeros(n_items, dtype=torch.int32, device=dev())
        acc = torch.zeros(n_items, dtype=torch.float32, device=dev())
        _lib.check(L.mcf_lock_stress(_lib.ptr(locks), _lib.ptr(acc), n_items, workers, iters,
                                     torch.cuda.current_stream().cuda_stream), "mcf_lock_stress")
        torch.cuda.synchronize()
        assert float(acc.double().sum()) == 2.0 * workers * iters, (n_items, workers, iters)
        assert int(locks.abs().sum()) == 0


def test_mfitr_sgd_parallel_accuracy_across_workers(golden):
    """SPEC.md:697 (Fig. 4): SGD validation RMSE after 5 epochs with
    concurrent workers stays within 0.5 % of the single-worker run for the
    SPEC's 2, 4 and 8 workers under the per-item locks; 64 and all-GPU user
    warps on this 1000-user problem (far more concurrency per user than the
    SPEC's desk scale) within 2 %."""
    from paper_1108_2580_b200 import mfitr
    from paper_1108_2580_b200.data import Dataset
    f = golden("mfitr_cfg2s.npz")
    graph = _graph(f)
    u, i, s = (np.asarray(f[k]) for k in ("users", "items", "scores"))
    rng = np.random.default_rng(5)
    hold = np.zeros(u.size, bool)
    for usr in np.unique(u):   # 4 held-out ratings per user (BASELINE convention)
        idx = np.flatnonzero(u == usr)
        hold[rng.choice(idx, size=min(4, idx.size - 1), replace=False)] = True
    U, I = int(f["U"]), int(f["I"])
    tr = Dataset.from_arrays(u[~hold], i[~hold], s[~hold], num_users=U, num_items=I, compact=True)
    va = Dataset.from_arrays(u[hold], i[hold], s[hold], num_users=U, num_items=I, compact=True)
    h = mfitr.MfitrHyper(D=8, lam1=0.005, lam2=0.015, lam3=0.05, lam4=0.05, gamma=0.005,
                         decay=0.95, iters=5)
    rm = {}
    for wk in (1, 2, 4, 8, 64, 0):
        _, rep = mfitr.train_mfitr("mfitr", tr, va, graph, h, seed=3, method="sgd",
                                   sgd_workers=wk)
        rm[wk] = rep[-1].valid_rmse
        assert np.isfinite(rm[wk])
    for wk in (2, 4, 8):
        assert abs(rm[wk] - rm[1]) <= 0.005 * rm[1], rm
    for wk in (64, 0):
        assert abs(rm[wk] - rm[1]) <= 0.02 * rm[1], rm
