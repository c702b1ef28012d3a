"""Pin the CPU oracle to the reference: every fixture here was produced by
importing the reference package itself (tests/golden/make_golden.py)."""
import json
import os

import numpy as np

import oracle
from conftest import GOLDEN


def test_spec_scalars():
    spec = json.load(open(os.path.join(GOLDEN, "spec_scalars.json")))
    csr = oracle.side_csr([0], [0], [8.0], 1)
    for lam, key in ((0.0, "p_lam0"), (1.0, "p_lam1")):
        out, failed = oracle.solve_rows(csr, np.array([[2.0]]), 1, lam_c=lam)
        assert failed == -1 and out[0, 0] == spec[key]
    csr_w = oracle.side_csr([0], [0], [8.0], 1, weights=[0.0])
    out, _ = oracle.solve_rows(csr_w, np.array([[2.0]]), 1, lam_c=1.0, use_weights=True)
    assert out[0, 0] == spec["p_w0"] == 0.0
    assert oracle.rmse([0.0, 10.0], [0.0, 0.0]) == spec["rmse_0_10"]
    Q = np.array([[1.0, 0.0], [0.0, 1.0]])
    z = np.zeros(0, np.int64)
    loss = oracle.loss_mfitr(np.zeros((1, 2)), Q, z, z, np.zeros(0), 0.0, np.zeros(1),
                             np.zeros(2), np.full(2, -1), np.zeros(2), np.zeros((2, 2)),
                             np.array([0]), np.array([1]), np.array([1.0]), 0, 0, 0.5, 0.0)
    assert loss == spec["loss_one_edge"]


def test_singular_row_fails_without_lambda():
    csr = oracle.side_csr([0, 1], [0, 0], [3.0, 4.0], 3)     # row 2 empty
    _, failed = oracle.solve_rows(csr, np.ones((1, 2)), 3, lam_c=0.0)
    assert failed == 0                                          # rank-1 row, D=2
    out, failed = oracle.solve_rows(csr, np.ones((1, 2)), 3, lam_c=0.5)
    assert failed == -1 and np.all(out[2] == 0)


def test_csr_bit_exact(golden):
    g = golden("csr.npz")
    U, I = int(g["U"]), int(g["I"])
    for side, keys, cols, n in (("users", g["users"], g["items"], U),
                                ("items", g["items"], g["users"], I)):
        ptr, idx, val, w, perm = oracle.side_csr(keys, cols, g["scores"], n, weights=g["wts"])
        assert np.array_equal(ptr, g[f"{side}_ptr"])
        assert np.array_equal(idx, g[f"{side}_idx"])
        assert np.array_equal(val, g[f"{side}_val"])
        assert np.array_equal(w, g[f"{side}_w"])
        assert np.array_equal(perm, np.argsort(keys, kind="stable"))


def test_als_small_bit_exact_and_monotone(golden):
    g = golden("als_small.npz")
    u, i, r = g["users"], g["items"], g["scores"]
    P, Q = g["P0"].copy(), g["Q0"].copy()
    lam = float(g["lam"])
    objs = []
    for it in range(25):
        Q, f = oracle.als_half_step(P, Q, u, i, r, "items", lam_c=lam, threads=1 + it % 4)
        assert f == -1
        assert np.array_equal(Q, g["Q"][it])                # bit-identical to numba
        objs.append(oracle.als_objective(P, Q, u, i, r, lam))
        P, f = oracle.als_half_step(P, Q, u, i, r, "users", lam_c=lam, threads=3)
        assert np.array_equal(P, g["P"][it])
        objs.append(oracle.als_objective(P, Q, u, i, r, lam))
    np.testing.assert_allclose(objs, g["obj"], rtol=1e-12)
    assert np.all(np.diff(objs) <= 1e-9 * np.abs(objs[:-1]))


def test_als_cfg0_weighted_lambda(golden):
    """lam * n_r on the diagonal == the reference's wALS hook with
    w = 1/n_row, and the plain-lambda path is bit-exact."""
    g = golden("als_cfg0.npz")
    u, i, r = g["train_users"], g["train_items"], g["train_scores"]
    U, I, lam = int(g["U"]), int(g["I"]), float(g["lam"])
    P, Q = g["P0"].astype(np.float64), g["Q0"].astype(np.float64)
    Qp, _ = oracle.als_half_step(P, Q, u, i, r, "items", lam_c=lam)
    assert np.array_equal(Qp, g["Q_plain"])
    # reference-oracle form, bit-exact
    wi = oracle.weighted_lambda_weights(u, i, U, I, "items")
    Qw, _ = oracle.als_half_step(P, Q, u, i, r, "items", lam_c=lam, weights=wi)
    assert np.array_equal(Qw, g["Q1"])
    # direct lam*n form
    Q1, _ = oracle.als_half_step(P, Q, u, i, r, "items", lam_n=lam)
    np.testing.assert_allclose(Q1, g["Q1"], rtol=1e-11, atol=1e-13 * np.abs(g["Q1"]).max())
    P1, _ = oracle.als_half_step(P, Q1, u, i, r, "users", lam_n=lam)
    np.testing.assert_allclose(P1, g["P1"], rtol=1e-10, atol=1e-12 * np.abs(g["P1"]).max())
    # free-running 5 sweeps -> same held-out RMSE
    for s in range(int(g["sweeps"])):
        Q, _ = oracle.als_half_step(P, Q, u, i, r, "items", lam_n=lam, threads=4)
        P, _ = oracle.als_half_step(P, Q, u, i, r, "users", lam_n=lam, threads=4)
        pred = oracle.predict(P, Q, g["valid_users"], g["valid_items"])
        assert abs(oracle.rmse(pred, g["valid_scores"]) - g["rmse"][s]) < 1e-9
    np.testing.assert_allclose(P, g["P_final"], rtol=1e-8, atol=1e-10)


def test_predict_cold_start(golden):
    g = golden("predict.npz")
    pred = oracle.predict(g["P"], g["Q"], g["qu"], g["qi"])
    assert np.array_equal(pred, g["als_pred"])
    art = g["art"]
    mqi = g["mqi"]
    arts = np.full(mqi.size, -1, np.int64)
    ok = (mqi >= 0) & (mqi < art.size)
    arts[ok] = art[mqi[ok]]
    pred = oracle.predict(g["mP"], g["mQ"], g["qu"], mqi, mu=float(g["mu"]), b_u=g["mbu"],
                          b_i=g["mbi"], arts=arts, b_a=g["mba"], Q_a=g["mQa"])
    assert np.array_equal(pred, g["mfitr_pred"])


def test_taxonomy_maps(golden):
    g = golden("taxonomy.npz")
    for p in ("s", "f", "g"):
        ec, ep = oracle.build_edges(g[f"{p}_kind"], g[f"{p}_album_of"], g[f"{p}_artist_link"])
        assert np.array_equal(ec, g[f"{p}_ec"]) and np.array_equal(ep, g[f"{p}_ep"])
        art = oracle.artist_array(g[f"{p}_kind"], g[f"{p}_artist_link"], g[f"{p}_art"].size)
        assert np.array_equal(art, g[f"{p}_art"])


def test_mfitr_weights_loss_grad(golden):
    g = golden("mfitr.npz")
    U, I = int(g["U"]), int(g["I"])
    w = oracle.edge_weights(g["ec"], g["ep"], g["users"], g["items"], g["scores"], U, I)
    assert np.array_equal(w, g["w"])
    args = (g["P"], g["Q"], g["users"], g["items"], g["scores"], float(g["mu"]), g["bu"],
            g["bi"], g["art"], g["ba"], g["Qa"], g["ec"], g["ep"], g["w"], float(g["lam1"]),
            float(g["lam2"]), float(g["lam3"]), float(g["lam4"]))
    np.testing.assert_allclose(oracle.loss_mfitr(*args), float(g["loss"]), rtol=1e-13)
    gr = oracle.grad_mfitr(*args)
    np.testing.assert_allclose(gr["p"], g["grad_p"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(gr["q"], g["grad_q"], rtol=1e-12, atol=1e-12)
    # bias and artist groups too (the MFITR full-block solver's optimality oracle)
    for k, f in (("b_u", "grad_bu"), ("b_i", "grad_bi"), ("b_a", "grad_ba"), ("q_a", "grad_qa")):
        np.testing.assert_allclose(gr[k], g[f], rtol=1e-12, atol=1e-12)


def test_mfitr_cfg2_shape_weights_loss_grad(golden):
    """Config-2 shaped workload: the reference's own edge weights / loss /
    gradient (biases and q_a at zero) reproduced by the oracle."""
    g = golden("mfitr_cfg2s.npz")
    U, I = int(g["U"]), int(g["I"])
    u, i, s = g["users"], g["items"], g["scores"].astype(np.float64)
    ec, ep = oracle.build_edges(g["kind"], g["album_of"], g["artist_link"])
    assert np.array_equal(ec, g["ec"]) and np.array_equal(ep, g["ep"])
    w = oracle.edge_weights(ec, ep, u, i, s, U, I)
    assert np.array_equal(w, g["w"])
    z = np.zeros(I)
    args = (g["P"], g["Q"], u.astype(np.int64), i.astype(np.int64), s, float(g["mu"]),
            np.zeros(U), z, g["art"], z, np.zeros_like(g["Q"]), ec, ep, w, 0.0,
            float(g["lam2"]), float(g["lam3"]), float(g["lam4"]))
    np.testing.assert_allclose(oracle.loss_mfitr(*args), float(g["loss"]), rtol=1e-12)
    gr = oracle.grad_mfitr(*args)
    np.testing.assert_allclose(gr["q"], g["grad_q"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(gr["p"], g["grad_p"], rtol=1e-10, atol=1e-10)


def test_layered_item_solve_zeroes_gradient(golden):
    """The ALS-MFITR item half-step, solved layer by layer with the oracle,
    zeroes grad_mfitr['q'] on every solved layer and never increases
    loss_mfitr (probe P5)."""
    g = golden("mfitr_cfg2s.npz")
    U, I = int(g["U"]), int(g["I"])
    u, i, s = g["users"].astype(np.int64), g["items"].astype(np.int64), g["scores"].astype(float)
    ec, ep, w = g["ec"], g["ep"], g["w"]
    mu, l2, tau = float(g["mu"]), float(g["lam2"]), float(g["lam3"]) + float(g["lam4"])
    P, Q = g["P"].copy(), g["Q"].copy()
    kind = np.full(I, -1, np.int8)
    kind[: g["kind"].size] = g["kind"]
    layers = [np.flatnonzero(kind == 0), np.flatnonzero(kind == 1), np.flatnonzero(kind == 2),
              np.flatnonzero((kind < 0) | (kind == 3))]
    csr = oracle.side_csr(i, u, s - mu, I)
    z = np.zeros(I)
    args = lambda Q_: (P, Q_, u, i, s, mu, np.zeros(U), z, g["art"], z, np.zeros_like(Q_),  # noqa
                       ec, ep, w, 0.0, l2, float(g["lam3"]), float(g["lam4"]))
    last = oracle.loss_mfitr(*args(Q))
    for rows in layers:
        S, T = oracle.taxonomy_terms(ec, ep, w, Q, I)
        out, failed = oracle.solve_rows(csr, P, I, lam_n=l2, tax_S=S, tax_T=T, tau=tau)
        assert failed == -1
        Q[rows] = out[rows]
        gq = oracle.grad_mfitr(*args(Q))["q"]
        scale = np.abs(oracle.grad_mfitr(*args(g["Q"]))["q"]).max()
        assert np.abs(gq[rows]).max() < 1e-9 * scale
        cur = oracle.loss_mfitr(*args(Q))
        assert cur <= last * (1 + 1e-12)
        last = cur


def test_mfitr_sgd_epoch_matches_reference_trainer(golden):
    """oracle.mfitr_sgd_epoch restates the reference's own MFITR trainer
    (sgd_epoch_mfitr: rate_update over users in the seeded shuffle, then the
    edge pass, gamma decay): 3 epochs reproduce its parameters and losses."""
    g = golden("mfitr_sgd.npz")
    f = golden("mfitr.npz")
    U, I = int(f["U"]), int(f["I"])
    P, Q, Qa = g["P0"].copy(), g["Q0"].copy(), g["Qa0"].copy()
    bu, bi, ba = np.zeros(U), np.zeros(I), np.zeros(I)
    lam = [float(g[k]) for k in ("lam1", "lam2", "lam3", "lam4")]
    gamma = float(g["gamma0"])
    for ep in range(3):
        oracle.mfitr_sgd_epoch(P, Q, bu, bi, f["art"], ba, Qa, float(g["mu"]), f["users"],
                               f["items"], f["scores"], g["perms"][ep], f["ec"], f["ep"],
                               f["w"], gamma, *lam)
        loss = oracle.loss_mfitr(P, Q, f["users"], f["items"], f["scores"], float(g["mu"]), bu,
                                 bi, f["art"], ba, Qa, f["ec"], f["ep"], f["w"], *lam)
        np.testing.assert_allclose(loss, g["loss"][ep], rtol=1e-10)
        gamma *= float(g["decay"])
    for a, b in ((P, "P"), (Q, "Q"), (Qa, "Qa"), (bu, "bu"), (bi, "bi"), (ba, "ba")):
        np.testing.assert_allclose(a, g[b], rtol=1e-10, atol=1e-12)
