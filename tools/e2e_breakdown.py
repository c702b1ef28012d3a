"""Phase timing of the e2e path (factor.train on pinned host arrays) at
config 1: where the non-sweep time goes.  GPU box only."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200 import factor, synth  # noqa: E402
from paper_1108_2580_b200.data import Dataset  # noqa: E402
from paper_1108_2580_b200.device import AlsEngine, DeviceRatings  # noqa: E402


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
dev = torch.device("cuda")
wl = synth.generate(cfg, seed=0, device=dev)
pin = lambda t: t.cpu().pin_memory().numpy()  # noqa: E731
tu, ti, ts = pin(wl.train_users), pin(wl.train_items), pin(wl.train_scores)
vu, vi, vs = pin(wl.valid_users), pin(wl.valid_items), pin(wl.valid_scores)
P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
for rep in range(2):
    t0 = T()
    u = torch.from_numpy(tu).to(dev, non_blocking=True)
    i = torch.from_numpy(ti).to(dev, non_blocking=True)
    s = torch.from_numpy(ts).to(dev, non_blocking=True)
    t1 = T()
    r = DeviceRatings(u, i, s, cfg.users, cfg.items, dev)
    t2 = T()
    eng = AlsEngine(r, cfg.D)
    eng.set_factors(P0, Q0)
    r.by_user.plan()
    r.by_item.plan()
    t3 = T()
    eng.sweep(0.0, cfg.lam)
    t4 = T()
    obj = eng.objective(cfg.lam, "weighted")
    t5 = T()
    vut, vit, vst = (torch.from_numpy(x).to(dev) for x in (vu, vi, vs))
    rm = eng.rmse(vut, vit, vst)
    float(rm.item())
    t6 = T()
    eng.check()
    P, Q = eng.factors()
    Pn, Qn = P.cpu(), Q.cpu()
    t7 = T()
    print(f"rep {rep}: h2d {1e3*(t1-t0):.1f} ms, layouts {1e3*(t2-t1):.1f}, engine+plans {1e3*(t3-t2):.1f}, "
          f"sweep {1e3*(t4-t3):.1f}, objective {1e3*(t5-t4):.1f}, rmse {1e3*(t6-t5):.1f}, d2h {1e3*(t7-t6):.1f}")
    del r, eng, u, i, s
    torch.cuda.empty_cache()
tr = Dataset.from_arrays(tu, ti, ts, num_users=cfg.users, num_items=cfg.items, compact=True)
va = Dataset.from_arrays(vu, vi, vs, num_users=cfg.users, num_items=cfg.items, compact=True)
hp = factor.HyperParams(lam=cfg.lam, D=cfg.D, iters=cfg.sweeps)
for rep in range(2):
    tr.__dict__.pop("_device_cache", None)
    t0 = T()
    m, rep_ = factor.train("wals", tr, va, hp, reg="weighted", init=(P0, Q0), as_torch=True)
    t1 = T()
    print(f"train(): {1e3*(t1-t0):.1f} ms for {cfg.sweeps} sweeps")
