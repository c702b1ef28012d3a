"""Config-2 MFITR: one SGD epoch (the reference's trainer, Hogwild over the
GPU) -- time and ratings/s.  GPU box only."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200 import mfitr, synth  # noqa: E402

cfg = synth.CONFIGS[2]
wl = synth.generate(cfg, seed=0, device="cuda")
tr = wl.train_dataset()
h = mfitr.MfitrHyper(D=cfg.D, lam1=0.005, lam2=cfg.lam, lam3=cfg.tax_weight,
                     lam4=cfg.tax_weight, gamma=5e-4, decay=0.95, iters=1)
mfitr.train_mfitr("mfitr", tr, None, wl.graph, h, method="sgd", objective=False)   # warm-up
for iters in (1, 3):
    h.iters = iters
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m, rep = mfitr.train_mfitr("mfitr", tr, None, wl.graph, h, method="sgd", objective=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{iters} epoch(s): {dt:.3f} s incl. setup; losses {[round(r.objective) for r in rep]}",
          flush=True)
