"""Where does re-anchored parity lose accuracy?  Config `CFG` (default 3),
a few sweeps for realistic factors, then one items half-step solved by the
default path and (MCF_NO_TC) the CUDA-core path, both from the same input
factors, against the float64 oracle on the hottest + random rows; prints the
worst rows with their degree and an estimate of cond(A).  GPU box only.
    CFG=3 SWEEPS=2 python tools/parity_probe.py"""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
import oracle  # noqa: E402
from paper_1108_2580_b200 import synth  # noqa: E402
from paper_1108_2580_b200.device import AlsEngine, DeviceRatings  # noqa: E402

cfg_id = int(os.environ.get("CFG", 3))
sweeps = int(os.environ.get("SWEEPS", 2))
wl = synth.generate(cfg_id, seed=0, device="cuda")
cfg = wl.cfg
r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items)
eng = AlsEngine(r, cfg.D)
P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
eng.set_factors(P0, Q0)
for _ in range(sweeps):
    eng.sweep(0.0, cfg.lam)
eng.check()
D = cfg.D
lay = r.by_item
rows = bench.parity_rows(lay, 2000, 64, np.random.default_rng(11))
fixed = eng.P[:, :D].double().cpu().numpy()
sp, idx, val, n = bench.gather_rows(lay, rows)
ref, failed = oracle.solve_rows((sp, idx, val, None), fixed, rows.size, 0.0, cfg.lam,
                                threads=os.cpu_count() or 1, dynamic=True)
deg = lay.degrees()[torch.as_tensor(rows, device="cuda")].cpu().numpy()
Qsave = eng.Q.clone()
for mode in ("default", "MCF_NO_TC"):
    if mode == "MCF_NO_TC":
        os.environ["MCF_NO_TC"] = "1"
    eng.Q.copy_(Qsave)
    eng.half_step("items", 0.0, cfg.lam)
    eng.check()
    os.environ.pop("MCF_NO_TC", None)
    got = eng.Q[torch.as_tensor(rows, device="cuda"), :D].double().cpu().numpy()
    rn = np.linalg.norm(ref, axis=1)
    dn = np.linalg.norm(got - ref, axis=1)
    rel = dn / np.maximum(rn, 1e-6 * rn.max())
    order = np.argsort(-rel)[:8]
    print(f"{mode}: max row rel {rel.max():.3e}, max rel {np.abs(got - ref).max() / np.abs(ref).max():.3e}")
    for lo_, hi_ in ((0, 25), (25, 50), (50, 100), (100, 200), (200, 1000), (1000, 10**9)):
        sel = (deg >= lo_) & (deg < hi_)
        if sel.any():
            print(f"   n in [{lo_},{hi_}): rows {sel.sum()}, max row rel {rel[sel].max():.3e}, median {np.median(rel[sel]):.3e}")
    for k in order[:3]:
        x = fixed[idx[sp[k]:sp[k + 1]]]
        A = x.T @ x + cfg.lam * deg[k] * np.eye(D)
        ev = np.linalg.eigvalsh(A)
        K = x @ x.T + cfg.lam * deg[k] * np.eye(x.shape[0])
        evk = np.linalg.eigvalsh(K)
        print(f"   row {rows[k]} n={deg[k]} rel={rel[k]:.3e} |ref|={rn[k]:.3e} cond={ev[-1] / ev[0]:.3e} "
              f"dual cond={evk[-1] / evk[0]:.3e}")
