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
    ref = oracle.predict(m.base.p, m.base.q, g["users"][:500], g["items"][:500], mu=m.base.mu)
    assert np.abs(pred - ref).max() < 1e-4 * np.abs(ref).max()
    assert np.array_equal(tm.model.ew.w, g["w"])
