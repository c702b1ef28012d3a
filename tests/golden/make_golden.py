"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src
(numba cache redirected to /tmp, no .pyc writes) and records its outputs on
seeded inputs into tests/golden/*.npz / *.json.  The fixtures are committed;
neither the tests nor the GPU box ever read /root/reference at run time.

Fixtures (reference entry point -> file):
  spec_scalars.json  SPEC.md ALS/RMSE/MFITR known-answer examples run through
                     factor.als_half_step, evaluation.rmse, mfitr.loss_mfitr,
                     mfitr.predict_mfitr
  als_small.npz      SPEC.md:346 instance (20x30, 30% observed, lam=1, D=5):
                     init_model + 25 x als_iteration, every half-step's P/Q and
                     als_objective (plain lambda, threads=1 and 4)
  als_cfg0.npz       BASELINE config 0 (this repo's generator, seed 0, CPU),
                     fp32 N(0,0.1) init (seed 1) injected into model.p/q;
                     weighted-lambda through the reference's wALS hook
                     (weights = 1/n_row per side): factors after each of the
                     first 4 half-steps, after 5 sweeps, held-out RMSE per
                     sweep; plus one plain-lambda items half-step
  csr.npz            factor._side_csr on shuffled records with repeated keys,
                     empty rows and weights (both sides)
  predict.npz        factor.predict_batch / mfitr.predict_batch incl.
                     out-of-range (cold-start) ids
  taxonomy.npz       synth.build_taxonomy, taxonomy.load_taxonomy (artist
                     inheritance), taxonomy.build_graph on this repo's MFITR
                     generator: edge lists and artist_array
  mfitr.npz          mfitr.edge_weights, loss_mfitr, grad_mfitr (every group:
                     p, q, b_u, b_i, b_a, q_a) on a small
                     synth.generate_synthetic instance with random parameters
  mfitr_sgd.npz      mfitr.train_mfitr (the reference's SGD trainer, 1 thread)
                     on the mfitr.npz instance: init, shuffles, per-epoch
                     loss / RMSE, final parameters
  mfitr_cfg2s.npz    config-2 shaped workload (this repo's generator, scaled):
                     reference edge weights, loss_mfitr, grad_mfitr
  formats.npz        data.load_ratings on ratings_small.tsv; modelio.save_model
                     bytes of an ALS and an MFITR model
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from multicf import evaluation, factor, mfitr, neighborhood, synth, taxonomy  # noqa: E402
from multicf.data import Dataset  # noqa: E402

from paper_1108_2580_b200 import synth as mysynth  # noqa: E402


def _ds(u, i, r, nu=None, ni=None):
    return Dataset.from_arrays(np.asarray(u), np.asarray(i), np.asarray(r, float),
                               np.zeros(len(u), np.int64), num_users=nu, num_items=ni)


def spec_scalars():
    out = {}
    hp = factor.HyperParams(D=1, iters=1)
    for lam, key in ((0.0, "p_lam0"), (1.0, "p_lam1")):
        ds = _ds([0], [0], [8.0])
        m = factor.init_model("als", ds, hp, 0)
        m.q[:] = 2.0
        factor.als_half_step(m, ds, "users", lam)
        out[key] = float(m.p[0, 0])
    ds = _ds([0], [0], [8.0])
    m = factor.init_model("als", ds, hp, 0)
    m.q[:] = 2.0
    factor.als_half_step(m, ds, "users", 1.0, weights=np.zeros(1))
    out["p_w0"] = float(m.p[0, 0])
    out["rmse_0_10"] = evaluation.rmse([0.0, 10.0], [0.0, 0.0])
    # one-edge loss example: q_i=(1,0), q_j=(0,1), lam3=.5
    g = taxonomy.build_graph(np.array([0, 1], np.int8), np.array([-1, -1]),
                             np.array([-1, -1]), {})
    g = taxonomy.TaxonomyGraph(g.kind, np.array([1, -1]), g.artist_link, {},
                               np.array([0]), np.array([1]))
    empty = _ds(np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0), nu=1, ni=2)
    h = mfitr.MfitrHyper(D=2, lam1=0, lam2=0, lam3=0.5, lam4=0.0)
    mm = mfitr.init_mfitr("mfitr", empty, g, h, 0, num_users=1, num_items=2)
    mm.base.q[:] = [[1, 0], [0, 1]]
    mm.q_a[:] = 0
    ew = mfitr.TaxonomyEdgeWeights(np.array([0]), np.array([1]), np.array([1.0]))
    out["loss_one_edge"] = mfitr.loss_mfitr(mm, empty, g, ew, h)
    return out


def als_small():
    rng = np.random.default_rng(7)
    U, I, D = 20, 30, 5
    mask = rng.random((U, I)) < 0.3
    u, i = np.nonzero(mask)
    perm = rng.permutation(u.size)
    u, i = u[perm], i[perm]
    r = rng.integers(0, 101, size=u.size).astype(float)
    ds = _ds(u, i, r, U, I)
    hp = factor.HyperParams(lam=1.0, D=D, iters=25)
    m = factor.init_model("als", ds, hp, 0)
    P0, Q0 = m.p.copy(), m.q.copy()
    Ps, Qs, objs = [], [], []
    m4 = m.copy()
    for _ in range(25):
        factor.als_half_step(m, ds, "items", 1.0)
        Qs.append(m.q.copy())
        objs.append(factor.als_objective(m, ds, 1.0))
        factor.als_half_step(m, ds, "users", 1.0)
        Ps.append(m.p.copy())
        objs.append(factor.als_objective(m, ds, 1.0))
        factor.als_iteration(m4, ds, 1.0, threads=4)
    assert np.array_equal(m4.p, m.p) and np.array_equal(m4.q, m.q)
    np.savez_compressed(os.path.join(HERE, "als_small.npz"), users=u, items=i, scores=r,
                        P0=P0, Q0=Q0, Q=np.array(Qs), P=np.array(Ps), obj=np.array(objs),
                        lam=1.0, D=D)


def als_cfg0():
    w = mysynth.generate(0, seed=0, device="cpu")
    cfg = w.cfg
    tu, ti, ts = (w.train_users.numpy().astype(np.int64), w.train_items.numpy().astype(np.int64),
                  w.train_scores.numpy().astype(np.float64))
    vu, vi, vs = (w.valid_users.numpy(), w.valid_items.numpy(), w.valid_scores.numpy())
    U, I, D, lam = cfg.users, cfg.items, cfg.D, cfg.lam
    P0, Q0 = mysynth.init_factors(U, I, D, seed=1)
    ds = _ds(tu, ti, ts, U, I)
    n_u = np.bincount(tu, minlength=U).astype(float)
    n_i = np.bincount(ti, minlength=I).astype(float)
    w_items, w_users = 1.0 / n_i[ti], 1.0 / n_u[tu]
    hp = factor.HyperParams(lam=lam, D=D, iters=cfg.sweeps)
    m = factor.init_model("wals", ds, hp, 0)
    m.p[:] = P0
    m.q[:] = Q0
    halves, rmses = [], []
    for sweep in range(cfg.sweeps):
        factor.als_half_step(m, ds, "items", lam, weights=w_items)
        if sweep < 2:
            halves.append(m.q.copy())
        factor.als_half_step(m, ds, "users", lam, weights=w_users)
        if sweep < 2:
            halves.append(m.p.copy())
        pred = factor.predict_batch(m, vu, vi)
        rmses.append(float(np.sqrt(np.mean((m.scale.clip(pred) - vs) ** 2))))
    # plain lambda, one items half-step from the same init
    mp = factor.init_model("als", ds, hp, 0)
    mp.p[:] = P0
    mp.q[:] = Q0
    factor.als_half_step(mp, ds, "items", lam)
    np.savez_compressed(os.path.join(HERE, "als_cfg0.npz"),
                        train_users=tu.astype(np.int32), train_items=ti.astype(np.int32),
                        train_scores=ts.astype(np.float32), valid_users=vu, valid_items=vi,
                        valid_scores=vs, P0=P0, Q0=Q0, Q1=halves[0], P1=halves[1],
                        Q2=halves[2], P2=halves[3], P_final=m.p, Q_final=m.q,
                        rmse=np.array(rmses), Q_plain=mp.q, U=U, I=I, D=D, lam=lam,
                        sweeps=cfg.sweeps)


def csr():
    rng = np.random.default_rng(11)
    n, U, I = 5000, 300, 200
    u = rng.integers(0, U - 20, n)          # users U-20.. stay empty
    i = (rng.zipf(1.5, n) - 1) % (I - 10)   # heavy repeats, empty tail items
    s = rng.integers(0, 101, n).astype(float)
    wts = rng.random(n)
    ds = _ds(u, i, s, U, I)
    out = {}
    for side in ("users", "items"):
        ptr, idx, val, ww = factor._side_csr(ds, side, wts)
        out.update({f"{side}_ptr": ptr, f"{side}_idx": idx, f"{side}_val": val,
                    f"{side}_w": ww})
    np.savez_compressed(os.path.join(HERE, "csr.npz"), users=u, items=i, scores=s, wts=wts,
                        U=U, I=I, **out)


def predict():
    rng = np.random.default_rng(5)
    U, I, D = 40, 60, 7
    ds = _ds(rng.integers(0, U, 300), rng.integers(0, I, 300), rng.integers(0, 101, 300))
    hp = factor.HyperParams(D=D)
    m = factor.init_model("als", ds, hp, 3, num_users=U, num_items=I)
    m.p[:] = rng.normal(size=m.p.shape)
    m.q[:] = rng.normal(size=m.q.shape)
    qu = np.concatenate([rng.integers(0, U, 200), [-1, U, 3, U + 5, -2]])
    qi = np.concatenate([rng.integers(0, I, 200), [2, 4, I, -1, I + 9]])
    als_pred = factor.predict_batch(m, qu, qi)
    # MFITR model on a small taxonomy
    cfg = synth.SynthConfig(users=U, artists=3, albums_per_artist=2, tracks_per_album=8,
                            ratings_per_user=5, dim=D)
    g = synth.build_taxonomy(cfg)
    n_items = g.num_nodes
    dsm = _ds(rng.integers(0, U, 300), rng.integers(0, n_items, 300), rng.integers(0, 101, 300),
              nu=U, ni=n_items)
    mm = mfitr.init_mfitr("mfitr", dsm, g, mfitr.MfitrHyper(D=D), 1, num_users=U)
    mm.base.p[:] = rng.normal(size=mm.base.p.shape)
    mm.base.q[:] = rng.normal(size=mm.base.q.shape)
    mm.q_a[:] = rng.normal(size=mm.q_a.shape)
    mm.b_a[:] = rng.normal(size=mm.b_a.shape)
    mm.base.b_u[:] = rng.normal(size=U)
    mm.base.b_i[:] = rng.normal(size=n_items)
    mqi = np.concatenate([rng.integers(0, n_items, 200), [2, 4, n_items, -1, n_items + 9]])
    mf_pred = mfitr.predict_batch(mm, qu, mqi)
    np.savez_compressed(os.path.join(HERE, "predict.npz"), P=m.p, Q=m.q, qu=qu, qi=qi,
                        als_pred=als_pred, mP=mm.base.p, mQ=mm.base.q, mQa=mm.q_a,
                        mba=mm.b_a, mbu=mm.base.b_u, mbi=mm.base.b_i, mu=mm.base.mu,
                        art=mm.artist_of_item, mqi=mqi, mfitr_pred=mf_pred)


def taxonomy_fx():
    cfg = synth.SynthConfig(users=10, artists=4, albums_per_artist=3, tracks_per_album=5,
                            ratings_per_user=5)
    g = synth.build_taxonomy(cfg)
    out = {"s_kind": g.kind, "s_album_of": g.album_of, "s_artist_link": g.artist_link,
           "s_ec": g.edge_child, "s_ep": g.edge_parent,
           "s_art": g.artist_array(g.num_nodes + 5)}
    # file format with artist inheritance and a track with both links
    lines = ["artist|0|NA|NA|", "artist|1|NA|NA|7,8", "album|2|NA|0|", "album|3|NA|1|",
             "track|4|2|NA|7", "track|5|3|0|", "track|6|NA|1|", "track|9|2|NA|",
             "track|10|NA|NA|"]
    with tempfile.NamedTemporaryFile("w", suffix=".tax", delete=False) as fh:
        fh.write("\n".join(lines) + "\n")
        path = fh.name
    lg = taxonomy.load_taxonomy(path)
    os.unlink(path)
    out.update({"f_kind": lg.kind, "f_album_of": lg.album_of, "f_artist_link": lg.artist_link,
                "f_ec": lg.edge_child, "f_ep": lg.edge_parent,
                "f_art": lg.artist_array(lg.num_nodes)})
    with open(os.path.join(HERE, "taxonomy_file.tax"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    # this repo's MFITR generator (cfg2 shape, scaled), graph built by the reference
    wl = mysynth.generate(mysynth.scaled_config(mysynth.CONFIGS[2], 0.002), seed=3)
    mg = wl.graph
    rg = taxonomy.build_graph(mg.kind, mg.album_of, mg.artist_link, {})
    out.update({"g_kind": mg.kind, "g_album_of": mg.album_of, "g_artist_link": mg.artist_link,
                "g_ec": rg.edge_child, "g_ep": rg.edge_parent,
                "g_art": rg.artist_array(mg.num_nodes)})
    np.savez_compressed(os.path.join(HERE, "taxonomy.npz"), **out)


def mfitr_fx():
    cfg = synth.SynthConfig(users=60, artists=4, albums_per_artist=2, tracks_per_album=6,
                            ratings_per_user=12, dim=4, drift=False)
    train, valid, test, g = synth.generate_synthetic(cfg, seed=2)
    ew = mfitr.edge_weights(g, train)
    rng = np.random.default_rng(9)
    h = mfitr.MfitrHyper(D=4, lam1=1e-3, lam2=0.065, lam3=0.1, lam4=0.05)
    U = train.num_users
    m = mfitr.init_mfitr("mfitr", train, g, h, 4)
    m.base.p[:] = rng.normal(size=m.base.p.shape)
    m.base.q[:] = rng.normal(size=m.base.q.shape)
    m.q_a[:] = rng.normal(size=m.q_a.shape) * 0.3
    m.b_a[:] = rng.normal(size=m.b_a.shape)
    m.base.b_u[:] = rng.normal(size=m.base.b_u.shape)
    m.base.b_i[:] = rng.normal(size=m.base.b_i.shape)
    loss = mfitr.loss_mfitr(m, train, g, ew, h)
    grad = mfitr.grad_mfitr(m, train, g, ew, h)
    np.savez_compressed(os.path.join(HERE, "mfitr.npz"), users=train.users, items=train.items,
                        scores=train.scores, U=U, I=m.base.num_items, kind=g.kind,
                        album_of=g.album_of, artist_link=g.artist_link, ec=g.edge_child,
                        ep=g.edge_parent, w=ew.w, P=m.base.p, Q=m.base.q, Qa=m.q_a, ba=m.b_a,
                        bu=m.base.b_u, bi=m.base.b_i, mu=m.base.mu, art=m.artist_of_item,
                        lam1=h.lam1, lam2=h.lam2, lam3=h.lam3, lam4=h.lam4, loss=loss,
                        grad_p=grad["p"], grad_q=grad["q"], grad_bu=grad["b_u"],
                        grad_bi=grad["b_i"], grad_ba=grad["b_a"], grad_qa=grad["q_a"])


def mfitr_sgd_fx():
    """The reference's own MFITR trainer (SGD, single thread): train_mfitr
    on the mfitr.npz instance for 3 epochs -- per-epoch loss / validation
    RMSE / gamma, the seeded shuffles, and the final parameters."""
    cfg = synth.SynthConfig(users=60, artists=4, albums_per_artist=2, tracks_per_album=6,
                            ratings_per_user=12, dim=4, drift=False)
    train, valid, test, g = synth.generate_synthetic(cfg, seed=2)
    ew = mfitr.edge_weights(g, train)
    h = mfitr.MfitrHyper(D=4, lam1=1e-3, lam2=0.065, lam3=0.1, lam4=0.05, gamma=0.01,
                         decay=0.9, iters=3)
    m0 = mfitr.init_mfitr("mfitr", train, g, h, 5)
    perms = [np.random.default_rng([5, 2]).permutation(train.num_users)]
    rng = np.random.default_rng([5, 2])
    perms = [rng.permutation(train.num_users) for _ in range(h.iters)]
    m, rep = mfitr.train_mfitr("mfitr", train, valid, g, h, threads=1, seed=5, ew=ew)
    np.savez_compressed(os.path.join(HERE, "mfitr_sgd.npz"),
                        P0=m0.base.p, Q0=m0.base.q, Qa0=m0.q_a, mu=m0.base.mu,
                        perms=np.stack(perms), loss=np.array([r.objective for r in rep]),
                        rmse=np.array([r.valid_rmse for r in rep]),
                        gamma=np.array([r.gamma for r in rep]),
                        P=m.base.p, Q=m.base.q, Qa=m.q_a, bu=m.base.b_u, bi=m.base.b_i, ba=m.b_a,
                        vu=valid.users, vi=valid.items, vs=valid.scores, seed=5,
                        lam1=h.lam1, lam2=h.lam2, lam3=h.lam3, lam4=h.lam4, decay=h.decay,
                        gamma0=0.01)


def mfitr_cfg2s():
    """Config-2 shaped MFITR workload (this repo's generator, scaled 0.001):
    the reference's own edge weights (adjusted_cosine over one cached
    _item_csr, bit-equal to mfitr.edge_weights -- SURVEY probe P5b) and
    loss_mfitr / grad_mfitr at random factors with biases and q_a = 0."""
    wl = mysynth.generate(mysynth.scaled_config(mysynth.CONFIGS[2], 0.001), seed=5)
    U, I = wl.num_users, wl.num_items
    u = wl.train_users.numpy().astype(np.int64)
    i = wl.train_items.numpy().astype(np.int64)
    s = wl.train_scores.numpy().astype(np.float64)
    ds = _ds(u, i, s, U, I)
    mg = wl.graph
    g = taxonomy.build_graph(mg.kind, mg.album_of, mg.artist_link, {})
    means = neighborhood.user_means(ds)
    csr = neighborhood._item_csr(ds, means)
    w = np.array([max(0.0, neighborhood.adjusted_cosine(int(c), int(p), ds, means, _csr=csr))
                  for c, p in zip(g.edge_child, g.edge_parent)])
    assert np.array_equal(w[:50], mfitr.edge_weights(
        taxonomy.TaxonomyGraph(g.kind, g.album_of, g.artist_link, {}, g.edge_child[:50],
                               g.edge_parent[:50]), ds).w)
    h = mfitr.MfitrHyper(D=8, lam1=0.0, lam2=0.065, lam3=0.1, lam4=0.1)
    m = mfitr.init_mfitr("mfitr", ds, g, h, 0, num_users=U, num_items=I)
    rng = np.random.default_rng(3)
    m.base.p[:] = rng.normal(0, 0.1, m.base.p.shape)
    m.base.q[:] = rng.normal(0, 0.1, m.base.q.shape)
    m.q_a[:] = 0.0
    ew = mfitr.TaxonomyEdgeWeights(g.edge_child, g.edge_parent, w)
    loss = mfitr.loss_mfitr(m, ds, g, ew, h)
    grad = mfitr.grad_mfitr(m, ds, g, ew, h)
    np.savez_compressed(os.path.join(HERE, "mfitr_cfg2s.npz"), users=u.astype(np.int32),
                        items=i.astype(np.int32), scores=s.astype(np.float32), U=U, I=I,
                        kind=mg.kind, album_of=mg.album_of, artist_link=mg.artist_link,
                        ec=g.edge_child, ep=g.edge_parent, w=w, P=m.base.p, Q=m.base.q,
                        mu=m.base.mu, art=m.artist_of_item, lam2=h.lam2, lam3=h.lam3,
                        lam4=h.lam4, loss=loss, grad_p=grad["p"], grad_q=grad["q"])


def formats():
    """Files written by the reference: a ratings TSV it loads, and the
    binary model format for an ALS and an MFITR model."""
    from multicf import modelio
    from multicf.data import load_ratings
    rng = np.random.default_rng(21)
    lines = ["# user item score time"]
    for k in range(40):
        lines.append(f"{rng.integers(0, 9)}\t{rng.integers(0, 7)}\t{float(rng.integers(0, 101))}"
                     f"\t{rng.integers(1000, 2000)}")
        if k == 10:
            lines.append("")
    with open(os.path.join(HERE, "ratings_small.tsv"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    ds = load_ratings(os.path.join(HERE, "ratings_small.tsv"))
    hp = factor.HyperParams(lam=1.0, D=3, iters=1)
    m = factor.init_model("als", ds, hp, 5)
    m.p[:] = rng.normal(size=m.p.shape).astype(np.float32)
    m.q[:] = rng.normal(size=m.q.shape).astype(np.float32)
    m.epochs_done = 3
    with tempfile.TemporaryDirectory() as td:
        modelio.save_model(m, os.path.join(td, "als.bin"))
        als_bytes = open(os.path.join(td, "als.bin"), "rb").read()
        cfg = synth.SynthConfig(users=9, artists=2, albums_per_artist=1, tracks_per_album=2,
                                ratings_per_user=2, dim=3)
        g = synth.build_taxonomy(cfg)
        mm = mfitr.init_mfitr("mfitr", ds, g, mfitr.MfitrHyper(D=3), 2, num_users=9,
                              num_items=max(7, g.num_nodes))
        mm.base.p[:] = rng.normal(size=mm.base.p.shape).astype(np.float32)
        mm.base.q[:] = rng.normal(size=mm.base.q.shape).astype(np.float32)
        mm.q_a[:] = 0.0
        modelio.save_model(mm, os.path.join(td, "mfitr.bin"))
        mf_bytes = open(os.path.join(td, "mfitr.bin"), "rb").read()
    np.savez_compressed(os.path.join(HERE, "formats.npz"), users=ds.users, items=ds.items,
                        scores=ds.scores, times=ds.times,
                        als_bytes=np.frombuffer(als_bytes, np.uint8),
                        mfitr_bytes=np.frombuffer(mf_bytes, np.uint8))


def main():
    only = sys.argv[1:]
    if only:   # regenerate just the named fixtures, e.g. `make_golden.py mfitr_fx`
        for name in only:
            globals()[name]()
        return
    with open(os.path.join(HERE, "spec_scalars.json"), "w") as fh:
        json.dump(spec_scalars(), fh, indent=1)
    als_small()
    csr()
    predict()
    taxonomy_fx()
    mfitr_fx()
    als_cfg0()
    mfitr_cfg2s()
    mfitr_sgd_fx()
    formats()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
