"""One half-step of a config's ALS sweep after one warm sweep (a target for
ncu: --kernel-name regex:k_als_tc --launch-skip 2 --launch-count 1).
GPU box only.    python tools/run_half_step.py [cfg] [items|users]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1108_2580_b200 import synth  # noqa: E402
from paper_1108_2580_b200.device import AlsEngine, DeviceRatings  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
side = sys.argv[2] if len(sys.argv) > 2 else "items"
dev = torch.device("cuda")
wl = synth.generate(cfg, seed=0, device=dev)
r = DeviceRatings(wl.train_users, wl.train_items, wl.train_scores, cfg.users, cfg.items, dev)
P0, Q0 = synth.init_factors(cfg.users, cfg.items, cfg.D, seed=1)
eng = AlsEngine(r, cfg.D)
eng.set_factors(P0, Q0)
eng.sweep(0.0, cfg.lam)
eng.half_step(side, 0.0, cfg.lam)
torch.cuda.synchronize()
eng.check()
print("ok", side)
