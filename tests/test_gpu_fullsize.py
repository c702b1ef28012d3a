"""Free-running parity at a BASELINE full-size configuration: config 1
(1,000,990 x 624,961, 258.8 M training ratings, D = 20, weighted lambda
0.065), 10 sweeps from the shared N(0, 0.1) init on the device-generated
workload, held-out RMSE after every sweep within 1e-4 (absolute, north_star)
of the float64 oracle's.  The oracle run is recorded in
tests/golden/fullsize_cfg1.json by tests/golden/make_fullsize_golden.py (the
oracle is pinned to the reference itself, tests/test_oracle.py); the test
first proves it regenerated the identical workload (sha256 digests)."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("config", [1, 3])
def test_fullsize_heldout_rmse_vs_oracle(config):
    path = os.path.join(HERE, "golden", f"fullsize_cfg{config}.json")
    if not os.path.exists(path):
        pytest.skip(f"{os.path.basename(path)} not generated")
    g = json.load(open(path))
    from paper_1108_2580_b200 import synth
    from paper_1108_2580_b200.device import AlsEngine, DeviceRatings
    cfg = synth.CONFIGS[config]
    wl = synth.generate(cfg, seed=0, device="cuda")
    P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
    host = lambda t: t.cpu().numpy()  # noqa: E731
    assert _sha(host(wl.train_users), host(wl.train_items), host(wl.train_scores)) == \
        g["digest"]["train"], "regenerated workload differs from the golden's"
    assert _sha(P0, Q0) == g["digest"]["init"]
    r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items)
    eng = AlsEngine(r, cfg.D)
    eng.set_factors(P0, Q0)
    got = []
    for _ in range(g["sweeps"]):
        eng.sweep(0.0, cfg.lam)
        got.append(float(eng.rmse(wl.valid_users, wl.valid_items, wl.valid_scores).item()))
    eng.check()
    diff = np.abs(np.array(got) - np.array(g["valid_rmse"]))
    assert diff.max() <= 1e-4, list(zip(got, g["valid_rmse"]))
