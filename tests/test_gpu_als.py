"""GPU parity of the ALS path against the CPU oracle (which is itself pinned
bit-exact to the reference, tests/test_oracle.py).

Tolerances (north_star): integer layouts bit-exact; per-half-step factors
within 1e-4 relative (re-anchored: the oracle restarts every half-step from
the device's own input factors); held-out RMSE within 1e-4 absolute after
the configured sweeps."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4


def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda")


def _rel_rows(got, ref):
    """max row-wise |d_r| / max(|ref_r|, 1e-6 max|ref|) and max|d| / max|ref|."""
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    scale = max(np.abs(ref).max(), 1e-30)
    rn = np.linalg.norm(ref, axis=1)
    dn = np.linalg.norm(got - ref, axis=1)
    row = (dn / np.maximum(rn, 1e-6 * np.linalg.norm(ref, axis=1).max() + 1e-30)).max()
    return row, np.abs(got - ref).max() / scale


def _engine(users, items, scores, U, I, D, chunk=2048, keep_perm=False):
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings
    r = DeviceRatings(users, items, scores, U, I, dev(), keep_perm=keep_perm)
    return AlsEngine(r, D, chunk=chunk)


# ---------------------------------------------------------------------------
# layout

def test_csr_build_bit_exact_golden(golden):
    from paper_1108_2580_b200.device import DeviceRatings
    g = golden("csr.npz")
    U, I = int(g["U"]), int(g["I"])
    r = DeviceRatings(g["users"], g["items"], g["scores"].astype(np.float32), U, I, dev(),
                      keep_perm=True)
    for side, lay in (("users", r.by_user), ("items", r.by_item)):
        assert np.array_equal(lay.ptr.cpu().numpy(), g[f"{side}_ptr"])
        assert np.array_equal(lay.idx.cpu().numpy(), g[f"{side}_idx"])
        assert np.array_equal(lay.val.cpu().numpy(), g[f"{side}_val"].astype(np.float32))


@pytest.mark.parametrize("nnz,n_rows", [(0, 5), (1, 1), (3000, 1), (70_001, 300),
                                        (2_500_000, 1_000_000), (1_200_000, 3_000_000)])
def test_csr_build_matches_stable_argsort(nnz, n_rows):
    from paper_1108_2580_b200.device import SideLayout
    rng = np.random.default_rng(nnz + n_rows)
    keys = (rng.zipf(1.3, nnz) * 7919 % n_rows).astype(np.int32)
    cols = rng.integers(0, 1 << 30, nnz).astype(np.int32)
    vals = rng.integers(0, 101, nnz).astype(np.float32)
    d = dev()
    lay = SideLayout(torch.from_numpy(keys).to(d), torch.from_numpy(cols).to(d),
                     torch.from_numpy(vals).to(d), n_rows, keep_perm=True)
    ptr, idx, val, _, perm = oracle.side_csr(keys, cols, vals, n_rows)
    assert np.array_equal(lay.ptr.cpu().numpy(), ptr)
    assert np.array_equal(lay.perm.cpu().numpy(), perm)
    assert np.array_equal(lay.idx.cpu().numpy(), idx)
    assert np.array_equal(lay.val.cpu().numpy(), val.astype(np.float32))


def test_csr_build_rejects_out_of_range_keys():
    from paper_1108_2580_b200.device import SideLayout
    from paper_1108_2580_b200.errors import DeviceError
    d = dev()
    k = torch.tensor([0, 5, 2], dtype=torch.int32, device=d)
    with pytest.raises(DeviceError, match="outside"):
        SideLayout(k, k, k.float(), 5)


# ---------------------------------------------------------------------------
# known answers through the drop-in entry point

def test_spec_scalars_drop_in():
    from paper_1108_2580_b200 import factor
    from paper_1108_2580_b200.data import Dataset
    spec = json.load(open(os.path.join(GOLDEN, "spec_scalars.json")))
    for lam, key in ((0.0, "p_lam0"), (1.0, "p_lam1")):
        ds = Dataset.from_arrays([0], [0], [8.0])
        m = factor.init_model("als", ds, factor.HyperParams(D=1), 0)
        m.q[:] = 2.0
        factor.als_half_step(m, ds, "users", lam)
        assert abs(m.p[0, 0] - spec[key]) < 1e-6
    ds = Dataset.from_arrays([0], [0], [8.0])
    m = factor.init_model("als", ds, factor.HyperParams(D=1), 0)
    m.q[:] = 2.0
    factor.als_half_step(m, ds, "users", 1.0, weights=np.zeros(1))
    assert m.p[0, 0] == spec["p_w0"] == 0.0


def test_singular_row_raises_min_row():
    from paper_1108_2580_b200 import SingularSystemError, factor
    from paper_1108_2580_b200.data import Dataset
    # users 3 and 5 see a single item with D=2 -> rank-1 systems at lam = 0
    ds = Dataset.from_arrays([0, 0, 3, 5, 1, 1], [0, 1, 0, 1, 0, 1], [1, 2, 3, 4, 5, 6.0])
    m = factor.init_model("als", ds, factor.HyperParams(D=2), 0)
    with pytest.raises(SingularSystemError, match="users row 2"):
        factor.als_half_step(m, ds, "users", 0.0)      # row 2 is empty -> min failing row
    m = factor.init_model("als", ds, factor.HyperParams(D=2), 0)
    factor.als_half_step(m, ds, "users", 0.5)          # regularised: fine, empty rows -> 0
    assert np.all(m.p[2] == 0) and np.all(m.p[4] == 0)


# ---------------------------------------------------------------------------
# config 0 parity (re-anchored and free-running)

@pytest.mark.parametrize("chunk", [2048, 64])
def test_cfg0_weighted_lambda_reanchored(golden, chunk):
    g = golden("als_cfg0.npz")
    u, i, s = g["train_users"], g["train_items"], g["train_scores"]
    U, I, D, lam = int(g["U"]), int(g["I"]), int(g["D"]), float(g["lam"])
    eng = _engine(u, i, s, U, I, D, chunk=chunk)
    eng.set_factors(g["P0"], g["Q0"])
    for sweep in range(int(g["sweeps"])):
        for side in ("items", "users"):
            P, Q = (t.double().cpu().numpy() for t in eng.factors())
            ref, failed = oracle.als_half_step(P, Q, u, i, s, side, lam_n=lam)
            assert failed == -1
            eng.half_step(side, 0.0, lam)
            eng.check()
            got = eng.factors()[0 if side == "users" else 1].double().cpu().numpy()
            row, mx = _rel_rows(got, ref)
            assert row < REL_TOL and mx < REL_TOL, (sweep, side, row, mx)
    # free-running held-out RMSE vs the reference's own (golden) RMSE
    vu = torch.as_tensor(g["valid_users"], dtype=torch.int32, device=dev())
    vi = torch.as_tensor(g["valid_items"], dtype=torch.int32, device=dev())
    vs = torch.as_tensor(g["valid_scores"], dtype=torch.float32, device=dev())
    rm = float(eng.rmse(vu, vi, vs).item())
    assert abs(rm - float(g["rmse"][-1])) < 1e-4, (rm, g["rmse"][-1])


def test_cfg0_first_half_steps_vs_reference(golden):
    """Device vs the reference's own factors after the first half-steps
    (fp32 device, f64 reference; same initial factors)."""
    g = golden("als_cfg0.npz")
    eng = _engine(g["train_users"], g["train_items"], g["train_scores"], int(g["U"]),
                  int(g["I"]), int(g["D"]))
    eng.set_factors(g["P0"], g["Q0"])
    lam = float(g["lam"])
    for key in ("Q1", "P1", "Q2", "P2"):
        side = "items" if key[0] == "Q" else "users"
        eng.half_step(side, 0.0, lam)
        got = eng.factors()[0 if side == "users" else 1].double().cpu().numpy()
        row, mx = _rel_rows(got, g[key])
        assert row < REL_TOL and mx < REL_TOL, (key, row, mx)
    eng.check()


def test_train_drop_in_cfg0(golden):
    from paper_1108_2580_b200 import factor
    from paper_1108_2580_b200.data import Dataset
    g = golden("als_cfg0.npz")
    U, I = int(g["U"]), int(g["I"])
    tr = Dataset.from_arrays(g["train_users"], g["train_items"], g["train_scores"],
                             num_users=U, num_items=I)
    va = Dataset.from_arrays(g["valid_users"], g["valid_items"], g["valid_scores"],
                             num_users=U, num_items=I)
    hp = factor.HyperParams(lam=float(g["lam"]), D=int(g["D"]), iters=int(g["sweeps"]))
    model, rep = factor.train("wals", tr, va, hp, reg="weighted", init=(g["P0"], g["Q0"]))
    assert len(rep) == hp.iters
    for s, row in enumerate(rep):
        assert abs(row.valid_rmse - float(g["rmse"][s])) < 1e-4
    assert np.all(np.diff([r.objective for r in rep]) <= 1e-6 * rep[0].objective)
    row, mx = _rel_rows(model.p, g["P_final"])
    assert mx < 1e-3
    pred = factor.predict_batch(model, g["valid_users"], g["valid_items"])
    ref = oracle.predict(g["P_final"], g["Q_final"], g["valid_users"], g["valid_items"])
    assert np.abs(pred - ref).max() < 1e-3 * np.abs(ref).max()


def test_wals_weights_path_reanchored(golden):
    """The reference-oracle form: lam * I with per-observation w = 1/n_row
    (HAS_W kernel), bit-for-bit the reference's wALS hook in f64."""
    g = golden("als_cfg0.npz")
    u, i, s = g["train_users"], g["train_items"], g["train_scores"]
    U, I, D, lam = int(g["U"]), int(g["I"]), int(g["D"]), float(g["lam"])
    eng = _engine(u, i, s, U, I, D, keep_perm=True)
    eng.set_factors(g["P0"], g["Q0"])
    wi = oracle.weighted_lambda_weights(u, i, U, I, "items")
    eng.set_weights(wi)
    eng.half_step("items", lam, 0.0)
    eng.check()
    got = eng.factors()[1].double().cpu().numpy()
    row, mx = _rel_rows(got, g["Q1"])
    assert row < REL_TOL and mx < REL_TOL, (row, mx)


def test_plain_lambda_small_monotone(golden):
    """SPEC.md:346 instance: plain lam = 1, D = 5, 25 iterations; every
    half-step matches the reference and the objective never increases."""
    g = golden("als_small.npz")
    u, i, s = g["users"], g["items"], g["scores"]
    eng = _engine(u, i, s, 20, 30, int(g["D"]))
    eng.set_factors(g["P0"], g["Q0"])
    objs = []
    for it in range(25):
        for side, key in (("items", "Q"), ("users", "P")):
            eng.half_step(side, 1.0, 0.0)
            got = eng.factors()[0 if side == "users" else 1].double().cpu().numpy()
            row, mx = _rel_rows(got, g[key][it])
            assert mx < 1e-3, (it, side, mx)          # free-running fp32 vs f64
            objs.append(float(eng.objective(1.0, "plain").item()))
    eng.check()
    objs = np.array(objs)
    assert np.all(np.diff(objs) <= 1e-5 * objs[:-1])
    np.testing.assert_allclose(objs, g["obj"], rtol=1e-3)


# ---------------------------------------------------------------------------
# dimensions, heavy rows, determinism

def _random_split(U, I, nnz, seed, hot=None):
    rng = np.random.default_rng(seed)
    keys = np.unique(rng.integers(0, U * I, nnz))
    if hot is not None:   # one very hot item rated by every user
        keys = np.unique(np.concatenate([keys, np.arange(U) * I + hot]))
    keys = rng.permutation(keys)
    return ((keys // I).astype(np.int32), (keys % I).astype(np.int32),
            rng.integers(0, 101, keys.size).astype(np.float32))


@pytest.mark.parametrize("D", [1, 3, 5, 8, 16, 20, 21, 28, 29, 32, 50, 56, 64, 96, 100, 103, 104, 128])
@pytest.mark.parametrize("reg", ["plain", "weighted"])
def test_dims_reanchored(D, reg):
    """Every compiled D range (warp path NB <= 7, CTA path above) and both
    regularisers; each half-step starts from fresh N(0, 0.1) factors so the
    comparison measures the kernel, not the conditioning of a free run."""
    U, I = 400, 300
    u, i, s = _random_split(U, I, 30_000, D, hot=7)
    eng = _engine(u, i, s, U, I, D, chunk=256)
    lam = 0.065
    lc, ln = (lam, 0.0) if reg == "plain" else (0.0, lam)
    for k, side in enumerate(("items", "users", "items")):
        rng = np.random.default_rng(k)
        P, Q = rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D))
        eng.set_factors(P, Q)
        P, Q = (t.double().cpu().numpy() for t in eng.factors())
        ref, failed = oracle.als_half_step(P, Q, u, i, s, side, lam_c=lc, lam_n=ln)
        eng.half_step(side, lc, ln)
        eng.check()
        got = eng.factors()[0 if side == "users" else 1].double().cpu().numpy()
        row, mx = _rel_rows(got, ref)
        assert row < REL_TOL and mx < REL_TOL, (D, reg, side, row, mx)
    # padding columns stay zero
    assert torch.all(eng.P[:, D:] == 0) and torch.all(eng.Q[:, D:] == 0)


@pytest.mark.parametrize("D", [64, 100])
def test_wide_ill_conditioned_short_rows(D):
    """The configuration-3 failure mode, small: partner factors with a
    dominant mean direction (cond(A) ~ 1e3-1e4) and rows of every length
    class -- n <= 64 (tensor path, dual n x n form + refinement), 64 < n < D
    (primal + refinement), n >= D, and a row rated by every item --
    re-anchored against the float64 oracle at 1e-4 on the tensor-core path
    (the CUDA-core kernels do not refine: tools/parity_probe.py shows them at
    2-3e-4 on such rows)."""
    rng = np.random.default_rng(D)
    U, I = 3000, 500
    mid = rng.integers(65, D, 900) if D > 66 else rng.integers(3, 65, 900)
    deg = np.concatenate([rng.integers(3, 65, 1200), mid,
                          rng.integers(D, 2 * D + 40, 899), [I]])   # last user: every item
    u = np.repeat(np.arange(U, dtype=np.int32), deg)
    i = np.concatenate([rng.choice(I, size=d, replace=False) for d in deg]).astype(np.int32)
    s = rng.integers(0, 101, u.size).astype(np.float32)
    perm = rng.permutation(u.size)
    u, i, s = u[perm], i[perm], s[perm]
    lam = 0.05
    for mode in ("tc",):
        try:
            eng = _engine(u, i, s, U, I, D, chunk=None)
            # item factors share a dominant direction (the mean of ALS factors)
            Q = rng.normal(0, 0.3, (I, D)) + 1.5
            P = rng.normal(0, 0.1, (U, D))
            eng.set_factors(P, Q)
            P64, Q64 = (t.double().cpu().numpy() for t in eng.factors())
            ref, failed = oracle.als_half_step(P64, Q64, u, i, s, "users", lam_n=lam)
            assert failed == -1
            eng.half_step("users", 0.0, lam)
            eng.check()
            got = eng.factors()[0].double().cpu().numpy()
            row, mx = _rel_rows(got, ref)
            assert row < REL_TOL and mx < REL_TOL, (mode, D, row, mx)
        finally:
            os.environ.pop("MCF_NO_TC", None)


def test_heavy_row_multi_chunk_and_determinism():
    U, I, D = 20_000, 500, 20
    u, i, s = _random_split(U, I, 400_000, 3, hot=11)
    outs = []
    for chunk in (2048, 2048, 128):
        eng = _engine(u, i, s, U, I, D, chunk=chunk)
        rng = np.random.default_rng(2)
        eng.set_factors(rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D)))
        eng.half_step("items", 0.0, 0.065)
        eng.check()
        outs.append(eng.factors()[1].double().cpu().numpy())
    ref, _ = oracle.als_half_step(eng.factors()[0].double().cpu().numpy(), outs[0], u, i, s,
                                  "items", lam_n=0.065)
    assert np.array_equal(outs[0], outs[1])             # run-to-run bit-identical
    for o in outs:
        row, mx = _rel_rows(o, ref)
        assert row < REL_TOL and mx < REL_TOL, (row, mx)


@pytest.mark.parametrize("D,chunk", [(50, None), (56, 512), (63, 2048)])
def test_hybrid_wide_path_long_rows_on_tensor_cores(D, chunk):
    """49 <= D < 64 with MCF_TC_HYBRID_MIN_N=256: rows with >= 256 ratings (and
    every hot-row chunk) take the tensor-core kernel, the others the tile-warp
    kernel; both half-steps vs the float64 oracle, and against the default
    (CUDA-core-only) run."""
    U, I = 6000, 60
    u, i, s = _random_split(U, I, 150_000, 7, hot=5)     # items ~2500 ratings, users ~25
    rng = np.random.default_rng(4)
    P0, Q0 = rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D))
    outs = {}
    for mode in ("hybrid", "cuda"):
        if mode == "hybrid":
            os.environ["MCF_TC_HYBRID_MIN_N"] = "256"   # an experiment knob: off by default
        try:
            eng = _engine(u, i, s, U, I, D, chunk=chunk)
            eng.set_factors(P0, Q0)
            eng.half_step("items", 0.0, 0.065)
            eng.check()
            Q1 = eng.factors()[1].double().cpu().numpy()
            eng.half_step("users", 0.0, 0.065)
            eng.check()
            outs[mode] = (Q1, eng.factors()[0].double().cpu().numpy())
        finally:
            os.environ.pop("MCF_TC_HYBRID_MIN_N", None)
    P32 = torch.as_tensor(P0, dtype=torch.float32).double().numpy()
    refQ, _ = oracle.als_half_step(P32, outs["hybrid"][0], u, i, s, "items", lam_n=0.065)
    refP, _ = oracle.als_half_step(P32, outs["hybrid"][0], u, i, s, "users", lam_n=0.065)
    for mode, (Q1, P1) in outs.items():
        row, mx = _rel_rows(Q1, refQ)
        assert row < REL_TOL and mx < REL_TOL, (mode, "items", row, mx)
    row, mx = _rel_rows(outs["hybrid"][1], refP)
    assert row < REL_TOL and mx < REL_TOL, ("users", row, mx)
    assert not np.array_equal(outs["hybrid"][0], outs["cuda"][0])   # the long rows did change kernels


@pytest.mark.parametrize("D,nnz", [(64, 60_000), (100, 60_000), (100, 150_000), (128, 150_000)])
def test_short_rows_dual_warp_kernel(D, nnz):
    """D >= 64: rows with n <= 32 ratings are solved by k_als_dual<1>, rows with
    33..64 (D > 64) by k_als_dual<2> (dual form, warp per row); checked against
    the float64 oracle and the run without the warp kernels (the tensor-core
    kernel's own dual form)."""
    U, I = 3000, 400
    u, i, s = _random_split(U, I, nnz, 9, hot=3)         # users ~20 / ~50 ratings, items ~150 / ~375
    rng = np.random.default_rng(5)
    P0, Q0 = rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D))
    outs = {}
    for mode in ("dual", "tc"):
        if mode == "tc":
            os.environ["MCF_NO_DUAL_WARP"] = "1"
        else:
            os.environ["MCF_DUAL_WARP_MAX"] = "64"   # also k_als_dual<2> (off by default)
        try:
            eng = _engine(u, i, s, U, I, D)
            eng.set_factors(P0, Q0)
            eng.half_step("users", 0.0, 0.065)
            eng.check()
            outs[mode] = eng.factors()[0].double().cpu().numpy()
        finally:
            os.environ.pop("MCF_NO_DUAL_WARP", None)
            os.environ.pop("MCF_DUAL_WARP_MAX", None)
    Q32 = torch.as_tensor(Q0, dtype=torch.float32).double().numpy()
    ref, _ = oracle.als_half_step(np.zeros((U, D)), Q32, u, i, s, "users", lam_n=0.065)
    for mode, P1 in outs.items():
        row, mx = _rel_rows(P1, ref)
        assert row < REL_TOL and mx < REL_TOL, (mode, row, mx)
    assert not np.array_equal(outs["dual"], outs["tc"])


def test_empty_rows_and_zero_rating_rows():
    U, I, D = 50, 40, 6
    u, i, s = _random_split(U - 10, I - 10, 600, 5)      # last 10 users / items empty
    eng = _engine(u, i, s, U, I, D)
    rng = np.random.default_rng(0)
    eng.set_factors(rng.normal(size=(U, D)), rng.normal(size=(I, D)))
    eng.half_step("users", 0.0, 0.1)
    eng.half_step("items", 0.3, 0.0)
    eng.check()
    P, Q = (t.cpu().numpy() for t in eng.factors())
    assert np.all(P[U - 10:] == 0) and np.all(Q[I - 10:] == 0)


def test_predict_golden_cold_start(golden):
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings
    g = golden("predict.npz")
    P, Q = g["P"], g["Q"]
    z = np.zeros(0, np.int32)
    r = DeviceRatings(z, z, np.zeros(0, np.float32), P.shape[0], Q.shape[0], dev())
    eng = AlsEngine(r, P.shape[1])
    eng.set_factors(P, Q)
    d = dev()
    pred, _ = eng.predict(torch.as_tensor(g["qu"], dtype=torch.int32, device=d),
                          torch.as_tensor(g["qi"], dtype=torch.int32, device=d))
    ref = g["als_pred"]
    assert np.abs(pred.cpu().numpy() - ref).max() < 1e-5 * np.abs(ref).max()
    # MFITR branch: mu + b_u + b_i + b_a + (q_i + q_a) . p_u
    mP, mQ, mQa = g["mP"], g["mQ"], g["mQa"]
    r2 = DeviceRatings(z, z, np.zeros(0, np.float32), mP.shape[0], mQ.shape[0], d)
    e2 = AlsEngine(r2, mP.shape[1])
    e2.set_factors(mP, mQ)
    qa = torch.zeros_like(e2.Q)
    qa[:, : mP.shape[1]] = torch.as_tensor(mQa, dtype=torch.float32)
    f = lambda a: torch.as_tensor(a, dtype=torch.float32, device=d)  # noqa: E731
    pred, _ = e2.predict(torch.as_tensor(g["qu"], dtype=torch.int32, device=d),
                         torch.as_tensor(g["mqi"], dtype=torch.int32, device=d),
                         mu=float(g["mu"]), b_u=f(g["mbu"]), b_i=f(g["mbi"]),
                         art=torch.as_tensor(g["art"], dtype=torch.int32, device=d),
                         b_a=f(g["mba"]), Q_a=qa)
    ref = g["mfitr_pred"]
    assert np.abs(pred.cpu().numpy() - ref).max() < 1e-5 * np.abs(ref).max()


def test_rmse_known_answer():
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings
    z = np.zeros(0, np.int32)
    r = DeviceRatings(z, z, np.zeros(0, np.float32), 2, 2, dev())
    eng = AlsEngine(r, 1)
    eng.set_factors(np.array([[0.0], [2.0]]), np.array([[0.0], [5.0]]))
    d = dev()
    rm = eng.rmse(torch.tensor([0, 1], dtype=torch.int32, device=d),
                  torch.tensor([0, 1], dtype=torch.int32, device=d),
                  torch.tensor([0.0, 0.0], device=d))
    assert abs(float(rm.item()) - np.sqrt(50.0)) < 1e-6


@pytest.mark.parametrize("reg,D", [("weighted", 20), ("plain", 10), ("weighted", 4)])
def test_fused_objective_matches_explicit(golden, reg, D):
    """The objective reported by the solve epilogue equals the explicit
    pass (predict + norms) and the float64 oracle objective."""
    g = golden("als_cfg0.npz")
    u, i, s = g["train_users"], g["train_items"], g["train_scores"]
    U, I = int(g["U"]), int(g["I"])
    eng = _engine(u, i, s, U, I, D, chunk=128)      # small chunk: hot-row path too
    rng = np.random.default_rng(0)
    eng.set_factors(rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D)))
    lam = 0.065
    lc, ln = (lam, 0.0) if reg == "plain" else (0.0, lam)
    obj = torch.zeros(4, dtype=torch.float64, device=dev())
    eng.sweep(lc, ln, obj)
    eng.check()
    fused = float(eng.sweep_objective(obj).item())
    explicit = float(eng.objective(lam, reg).item())
    P, Q = (t.double().cpu().numpy() for t in eng.factors())
    if reg == "plain":
        ref = oracle.als_objective(P, Q, u.astype(np.int64), i.astype(np.int64), s, lam)
    else:
        ref = oracle.weighted_objective(P, Q, u.astype(np.int64), i.astype(np.int64), s, lam)
    assert abs(explicit - ref) < 1e-5 * ref
    assert abs(fused - ref) < 1e-4 * ref, (fused, explicit, ref)


@pytest.mark.parametrize("D", [10, 24])
def test_train_objective_with_observation_weights(golden, D):
    """train(..., weights=w) reports the reference's weighted objective
    sum w (r - q.p)^2 + lam (|P|^2 + |Q|^2) (factor.py:541-547) on both the
    fused (D <= 20) and the explicit (D > 20) objective paths."""
    from paper_1108_2580_b200 import factor
    from paper_1108_2580_b200.data import Dataset
    g = golden("als_cfg0.npz")
    u, i, s = g["train_users"], g["train_items"], g["train_scores"]
    U, I = int(g["U"]), int(g["I"])
    tr = Dataset.from_arrays(u, i, s, num_users=U, num_items=I)
    w = np.random.default_rng(5).uniform(0.2, 2.0, len(tr))
    hp = factor.HyperParams(lam=0.5, D=D, iters=2)
    rng = np.random.default_rng(1)
    init = (rng.normal(0, 0.1, (U, D)).astype(np.float32),
            rng.normal(0, 0.1, (I, D)).astype(np.float32))
    model, rep = factor.train("wals", tr, None, hp, weights=w, init=init)
    ref = factor.als_objective(model, tr, hp.lam, w)
    assert abs(rep[-1].objective - ref) < 1e-4 * ref, (rep[-1].objective, ref)


def test_fused_peer_stores_replicate_every_row():
    """mcf_als_half_step_peers: the solve kernel writes every solved row into
    each peer replica too (the fused all-gather of the sharded sweep) -- two
    'peers' on this GPU receive exactly the local result, for the pair
    (D = 20, hot rows) and tile-warp (D = 50) paths."""
    from paper_1108_2580_b200.device import LayoutSolver
    for D in (20, 50):
        U, I = 3000, 400
        u, i, s = _random_split(U, I, 120_000, 11, hot=5)
        eng = _engine(u, i, s, U, I, D, chunk=256)
        rng = np.random.default_rng(1)
        eng.set_factors(rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D)))
        ref = eng.half_step("items", 0.0, 0.065).clone()
        peers = [torch.full_like(eng.Q, float("nan")) for _ in range(2)]
        ptrs = torch.tensor([t.data_ptr() for t in peers], dtype=torch.int64, device=eng.device)
        out = torch.zeros_like(eng.Q)
        LayoutSolver(D, 256).solve(eng.r.by_item, eng.P, out, 0.0, 0.065, peers=ptrs)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
        for t in peers:
            assert torch.equal(t, ref)


def test_sharded_peer_collective_single_rank():
    """ShardedAls(collective="peer") on a one-rank NCCL group: tables in
    symmetric memory, the fused peer-store path (no peers at world 1) and the
    device barrier; identical to the NCCL-collective runner."""
    import socket
    import torch.distributed as dist
    from paper_1108_2580_b200.parallel import ShardedAls
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        U, I, D = 2000, 300, 20
        u, i, s = _random_split(U, I, 60_000, 4)
        rng = np.random.default_rng(0)
        P0, Q0 = rng.normal(0, 0.1, (U, D)), rng.normal(0, 0.1, (I, D))
        outs = []
        for coll in ("nccl", "peer"):
            try:
                run = ShardedAls(u, i, s, U, I, D, collective=coll)
            except Exception as e:   # pragma: no cover - symmetric memory unavailable
                if coll == "peer":
                    pytest.skip(f"torch symmetric memory unavailable: {e}")
                raise
            run.set_factors(P0, Q0)
            for _ in range(2):
                run.sweep(0.0, 0.065)
            run.check()
            outs.append([t.clone() for t in run.factors()])
        assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    finally:
        dist.destroy_process_group()
