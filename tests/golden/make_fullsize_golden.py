"""Full-size golden: the pinned float64 oracle run free over a BASELINE
configuration, on the device-generated workload.

    python tests/golden/make_fullsize_golden.py --config 1 [--sweeps 10]

Runs on a GPU box (the workload is generated there with torch's CUDA RNG --
the same bytes bench.py and the GPU tests generate; torch only, libmcf is
never loaded) and writes tests/golden/fullsize_cfg<N>.json:

* sha256 of the generated train / held-out arrays and of the initial
  factors, so a test can prove it regenerated the identical workload;
* the oracle's held-out RMSE after every sweep (weighted lambda, items then
  users half-step, float64 factors throughout -- the reference's train(),
  factor.py:595-618, with the wALS weighting restated as lam * n_r, equal to
  the reference's weights = 1/n_row hook to <= 1e-13);
* the oracle's objective-free final factors on the hottest rows of each side
  (a record of the long-row sums the device accumulates in fp32 chunks).

The oracle (oracle/als_oracle.c) is pinned bit-exact to the reference's own
numba kernel on the config-0 fixtures (tests/test_oracle.py); rows are solved
with dynamic scheduling over all host cores (identical results).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1108_2580_b200 import synth  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def workload_digest(wl, P0, Q0) -> dict:
    host = lambda t: t.cpu().numpy()  # noqa: E731
    return {"train": sha(host(wl.train_users), host(wl.train_items), host(wl.train_scores)),
            "valid": sha(host(wl.valid_users), host(wl.valid_items), host(wl.valid_scores)),
            "init": sha(P0, Q0)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--sweeps", type=int, default=None)
    ap.add_argument("--hot", type=int, default=16)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    assert cfg.taxonomy is None, "ALS configurations only"
    sweeps = args.sweeps or cfg.sweeps
    threads = os.cpu_count() or 1
    t0 = time.time()
    wl = synth.generate(cfg, seed=0, device="cuda")
    P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
    digest = workload_digest(wl, P0, Q0)
    u = wl.train_users.cpu().numpy().astype(np.int64)
    i = wl.train_items.cpu().numpy().astype(np.int64)
    s = wl.train_scores.cpu().numpy().astype(np.float64)
    vu = wl.valid_users.cpu().numpy().astype(np.int64)
    vi = wl.valid_items.cpu().numpy().astype(np.int64)
    vs = wl.valid_scores.cpu().numpy().astype(np.float64)
    del wl
    torch.cuda.empty_cache()
    print(f"generated in {time.time() - t0:.1f} s; nnz {u.size}", flush=True)
    t0 = time.time()
    ucsr = oracle.side_csr(u, i, s, cfg.users)[:4]
    icsr = oracle.side_csr(i, u, s, cfg.items)[:4]
    deg_u = np.diff(ucsr[0])
    deg_i = np.diff(icsr[0])
    del u, i, s
    print(f"layouts in {time.time() - t0:.1f} s", flush=True)
    P, Q = P0.astype(np.float64), Q0.astype(np.float64)
    rmse, times = [], []
    for sw in range(sweeps):
        t0 = time.time()
        Q, f = oracle.solve_rows(icsr, P, cfg.items, 0.0, cfg.lam, threads=threads, dynamic=True)
        assert f == -1
        P, f = oracle.solve_rows(ucsr, Q, cfg.users, 0.0, cfg.lam, threads=threads, dynamic=True)
        assert f == -1
        rmse.append(oracle.rmse(oracle.predict(P, Q, vu, vi), vs))
        times.append(time.time() - t0)
        print(f"sweep {sw}: {times[-1]:.1f} s  rmse {rmse[-1]:.9f}", flush=True)
    hot_u = np.argsort(-deg_u, kind="stable")[: args.hot]
    hot_i = np.argsort(-deg_i, kind="stable")[: args.hot]
    out = {
        "config": cfg.name, "users": cfg.users, "items": cfg.items, "nnz": int(deg_u.sum()),
        "D": cfg.D, "lambda_weighted": cfg.lam, "sweeps": sweeps, "data_seed": 0, "init_seed": 1,
        "generator": "paper_1108_2580_b200.synth.generate(device='cuda'), torch "
                     + torch.__version__,
        "digest": digest,
        "oracle": "oracle/als_oracle.c float64, weighted lambda as lam*n_r, items then users",
        "oracle_threads": threads, "oracle_seconds_per_sweep": times,
        "valid_rmse": rmse,
        "hot_users": hot_u.tolist(), "hot_users_degree": deg_u[hot_u].tolist(),
        "hot_items": hot_i.tolist(), "hot_items_degree": deg_i[hot_i].tolist(),
        "P_hot_users": P[hot_u].tolist(), "Q_hot_items": Q[hot_i].tolist(),
    }
    path = args.out or os.path.join(HERE, f"fullsize_cfg{args.config}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
